# usage (GPU box): Toeplitz-tile matvec A/B (TDB_MV_TBSR=0 is the CSR-only plan) + GPU tests
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/tbsr_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/tbsr_tests.txt
for c in 2 4; do
  echo "== cfg$c tbsr"; timeout 300 python tools/mv_probe.py $c 2>&1 | grep -i "matvec\|error"
  echo "== cfg$c csr";  TDB_MV_TBSR=0 timeout 300 python tools/mv_probe.py $c 2>&1 | grep matvec
done > gpurun_out/tbsr_mv.txt 2>&1
timeout 300 python tools/solve_probe.py 2 > gpurun_out/tbsr_solve.txt 2>&1
