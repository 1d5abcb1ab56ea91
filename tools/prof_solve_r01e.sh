mkdir -p gpurun_out
python -m pytest tests/test_gpu_krylov.py tests/test_gpu_parity.py -x -q > gpurun_out/s_tests.txt 2>&1; echo rc=$? >> gpurun_out/s_tests.txt
python tools/mv_probe.py 2 > gpurun_out/s_mv.txt 2>&1
python tools/solve_probe.py 2 > gpurun_out/s_solve.txt 2>&1
python tools/solve_probe.py 2 4 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_launches_r01e.csv python tools/solve_probe.py 2 4 > /dev/null 2>&1
