mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/tbsr_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/tbsr_tests.txt
for c in 2 4; do
  for w in 32 64; do echo "== cfg$c tbsr W$w"; TDB_TBSR_WARPS_PER_SM=$w timeout 300 python tools/mv_probe.py $c 2>&1 | grep -i "matvec\|error"; done
done > gpurun_out/tbsr_mv.txt 2>&1
timeout 300 python tools/solve_probe.py 2 > gpurun_out/tbsr_solve.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mv_launches_t3c4.csv python tools/mv_probe.py 4 1 > /dev/null 2>&1
