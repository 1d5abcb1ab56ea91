# usage (on the GPU box, via gpurun): bash tools/gpu_round.sh <tag> [config]
# bench line, launch list of the same command, one ncu --set full capture each of
# k_quad_cells and k_quad (summarised into gpurun_out/ncu_quad[_cells]_cfg<c>_<tag>.json).
set -u
mkdir -p gpurun_out
T=$1
C=${2:-4}
python bench.py --config $C > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
CMD="python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
$CMD > gpurun_out/plain_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv $CMD > /dev/null 2>&1
# the regular-pair kernel (dominant) and the singular-case kernel, one launch each (the second of the run)
ncu --set full --clock-control none --import-source on -k regex:k_quad_cells -s 1 -c 1 -o gpurun_out/prof_quad_cells_$T $CMD > /dev/null 2>&1 && \
python tools/ncu_json.py gpurun_out/prof_quad_cells_$T.ncu-rep gpurun_out/ncu_quad_cells_cfg${C}_$T.json "config $C" > /dev/null
ncu --set full --clock-control none --import-source on -k "regex:k_quad<" -s 1 -c 1 -o gpurun_out/prof_quad_$T $CMD > /dev/null 2>&1 && \
python tools/ncu_json.py gpurun_out/prof_quad_$T.ncu-rep gpurun_out/ncu_quad_cfg${C}_$T.json "config $C" > /dev/null
echo done
