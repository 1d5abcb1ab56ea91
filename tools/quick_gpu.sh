# usage (GPU box): bash tools/quick_gpu.sh <tag> [pytest]  - gpu tests (optional) + short bench line
mkdir -p gpurun_out
T=$1
if [ "$2" = "pytest" ]; then
  python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
  tail -2 gpurun_out/pytest_$T.log
fi
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$T.json"))
print("value", d["value"], "ms_step", d["ms_per_step"], "frac", d["roofline"]["frac"], "phases", d["phases_ms"])
PY
