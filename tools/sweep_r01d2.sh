# usage (GPU box): fill-phase, matvec and solve A/B of the libtdb variants
mkdir -p gpurun_out
bash tools/fill_variants.sh base fb4m2 fb8m2 fb4m3 fb2m3 > gpurun_out/fillsweep.txt 2>&1
for v in base sp4 sp6 sp8; do
  echo "== $v"
  TDB_LIBRARY=tools/_variants/libtdb_$v.so python tools/mv_probe.py 2 2>&1 | grep matvec
  TDB_LIBRARY=tools/_variants/libtdb_$v.so python tools/solve_probe.py 2 2>&1 | grep solve
done > gpurun_out/solvesweep.txt 2>&1
TDB_LIBRARY=tools/_variants/libtdb_sp8.so python -m pytest -q -x tests/test_gpu_krylov.py tests/test_gpu_parity.py > gpurun_out/sp8_tests.txt 2>&1
