# usage (GPU box): bash tools/prof_solve.sh <tag>  - solve timing + launch list of 4 outer steps
mkdir -p gpurun_out
python tools/solve_probe.py 2 > gpurun_out/solve_$1.log 2>&1
cat gpurun_out/solve_$1.log
python tools/solve_probe.py 2 4 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_launches_$1.csv python tools/solve_probe.py 2 4 > /dev/null 2>&1
echo done
