mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/mv4_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/mv4_tests.txt
for c in 2 4; do echo "== cfg$c"; timeout 300 python tools/mv_probe.py $c 2>&1 | grep -i "matvec\|error"; done > gpurun_out/mv4.txt 2>&1
timeout 300 python tools/solve_probe.py 2 >> gpurun_out/mv4.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mv_launches_t4c4.csv python tools/mv_probe.py 4 1 > /dev/null 2>&1
