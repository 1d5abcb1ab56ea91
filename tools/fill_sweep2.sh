mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > gpurun_out/var_main.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/var_main.json')); print('main', d['phases_ms'])"
bash tools/fill_variants.sh fb1m3 fb2m2 fb2m4 fb4m2
