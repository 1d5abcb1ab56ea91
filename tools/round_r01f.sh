# usage (GPU box): end-of-session evidence: tests, smoke, bench (ours + reference arm),
# launch list of the bench command, ncu --set full of k_quad, k_tbsr_mv and the largest pattern fill
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/f_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.txt
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > /dev/null 2>&1
Q="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
ncu --set full --clock-control none --import-source on -k regex:k_quad -s 1 -c 1 -o gpurun_out/f_prof_quad $Q > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tbsr_mv -c 1 -o gpurun_out/f_prof_tbsr $Q > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pattern_fill -c 1 -o gpurun_out/f_prof_fill $Q > /dev/null 2>&1
echo done
