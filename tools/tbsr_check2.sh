mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/tbsr_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/tbsr_tests.txt
for c in 2 4; do
  for w in 8 16 32; do echo "== cfg$c tbsr W$w"; TDB_TBSR_WARPS_PER_SM=$w timeout 300 python tools/mv_probe.py $c 2>&1 | grep -i "matvec\|error"; done
  echo "== cfg$c tbsr pred"; TDB_LIBRARY=tools/_variants/libtdb_tpred.so timeout 300 python tools/mv_probe.py $c 2>&1 | grep -i "matvec\|error"
done > gpurun_out/tbsr_mv.txt 2>&1
timeout 300 python tools/solve_probe.py 2 > gpurun_out/tbsr_solve.txt 2>&1
