# usage (GPU box): bash tools/fill_variants.sh name...  - pattern-phase ms per libtdb variant
for v in "$@"; do
  TDB_LIBRARY=tools/_variants/libtdb_$v.so python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-solve > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "import json; d=json.load(open('gpurun_out/var_$v.json')); print('$v', d['phases_ms'])" || tail -3 gpurun_out/var_$v.err
done
