# usage (GPU box): bash tools/prof_tbsr.sh <tag> [config] - launch list + ncu full of the tile and CSR matvec kernels
mkdir -p gpurun_out
CMD="python tools/mv_probe.py ${2:-2} 3"
$CMD > gpurun_out/mvplain_$1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mv_launches_$1.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tbsr_mv -c 1 -o gpurun_out/prof_tbsr_$1 $CMD > gpurun_out/ncu_tbsr_$1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_matvec -c 1 -o gpurun_out/prof_mvcsr_$1 $CMD > gpurun_out/ncu_mvcsr_$1.log 2>&1
cat gpurun_out/mvplain_$1.log
echo done
