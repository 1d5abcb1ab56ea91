# usage: bash tools/prof_quad.sh <tag>   (runs on the GPU box)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_quad -c 1 -o gpurun_out/prof_quad_$1 $CMD > gpurun_out/ncu_$1.log 2>&1
echo done
