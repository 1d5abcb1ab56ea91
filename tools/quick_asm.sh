# usage (GPU box): GPU tests + a short assembly-only bench (phases)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/q_tests.txt
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python -c "import json; d=json.load(open('gpurun_out/q_bench.json')); print(d['value'], d['phases_ms'], d['matvec']['ms'])"
