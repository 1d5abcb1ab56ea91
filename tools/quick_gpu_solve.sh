# usage (GPU box): bash tools/quick_gpu_solve.sh <tag>  - gpu tests + bench line incl. the FGMRES solve
mkdir -p gpurun_out
T=$1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
tail -2 gpurun_out/pytest_$T.log
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$T.json"))
print("value", d["value"], "quad", d["phases_ms"]["ms_quad"], "solve", d["solve"])
PY
tail -3 gpurun_out/bench_$T.err
