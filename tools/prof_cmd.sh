set -x
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:k_quad -s 1 -c 1 -o gpurun_out/prof_quad $CMD > gpurun_out/ncu_full.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:k_pattern_fill -c 1 -o gpurun_out/prof_fill $CMD > gpurun_out/ncu_fill.log 2>&1
echo done
