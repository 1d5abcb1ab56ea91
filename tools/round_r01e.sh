# usage (GPU box): tests + smoke + bench + launch list + ncu captures for round r01e
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/e_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/e_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/e_smoke.txt
python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/e_bench_ref.json 2> gpurun_out/e_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tbsr_mv -c 1 -o gpurun_out/e_prof_tbsr \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pattern_fill -c 1 -o gpurun_out/e_prof_fill \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > /dev/null 2>&1
echo done
