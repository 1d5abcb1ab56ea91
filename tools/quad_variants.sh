# usage (GPU box): bash tools/quad_variants.sh name...  - k_quad ms per libtdb variant (bench, 2 steps)
mkdir -p gpurun_out
for v in "$@"; do
  TDB_LIBRARY=tools/_variants/libtdb_$v.so python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-solve > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "import json; d=json.load(open('gpurun_out/var_$v.json')); print('$v', 'quad_ms', round(d['phases_ms']['ms_quad'],2), 'n_in', d['roofline']['n_in'])" || tail -3 gpurun_out/var_$v.err
done
