# usage (GPU box): configs 3/4 bench lines + config-5 8-way rank shares (one GPU, rank by rank)
mkdir -p gpurun_out
for c in 3 4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > gpurun_out/cfg${c}_bench.json 2> gpurun_out/cfg${c}_bench.err
done
: > gpurun_out/cfg5_shares.jsonl
for r in 0 1 2 3 4 5 6 7; do
  timeout 600 python tools/rank_share.py 5 8 $r >> gpurun_out/cfg5_shares.jsonl 2> gpurun_out/cfg5_share_$r.err
done
echo done
