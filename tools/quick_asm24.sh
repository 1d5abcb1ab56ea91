mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/q_tests.txt
for c in 2 4; do
python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > gpurun_out/q_bench$c.json 2> gpurun_out/q_bench$c.err
python -c "import json; d=json.load(open('gpurun_out/q_bench$c.json')); print($c, d['value'], d['phases_ms'])"
done
