# usage: bash tools/prof_round.sh <tag>   (GPU box) - bench line, launch list, ncu of the top kernels
mkdir -p gpurun_out
T=$1
python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
$CMD > gpurun_out/plain_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_quad -s 1 -c 1 -o gpurun_out/prof_quad_$T $CMD > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_pattern_fill -s 1 -c 1 -o gpurun_out/prof_fill_$T $CMD > /dev/null 2>&1
python tools/mv_probe.py 2 > gpurun_out/mvplain_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 2 -c 1 -o gpurun_out/prof_mv_$T python tools/mv_probe.py 2 3 > /dev/null 2>&1
echo done
