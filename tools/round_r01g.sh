# usage (GPU box): final evidence of the session: tests, smoke, bench + reference arm, launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/g_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/g_smoke.txt
python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
python bench.py --impl reference > gpurun_out/g_bench_ref.json 2> gpurun_out/g_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > /dev/null 2>&1
echo done
