# usage (GPU box): bash tools/prof_solve4.sh <tag>  - launch list of 3 outer solve steps on config 4
mkdir -p gpurun_out
python tools/solve_probe.py 4 3 > gpurun_out/solve4_$1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'^(?!k_quad|k_pattern|k_plan|k_finalize)' --log-file gpurun_out/solve4_launches_$1.csv python tools/solve_probe.py 4 3 > /dev/null 2>&1
cat gpurun_out/solve4_$1.log
