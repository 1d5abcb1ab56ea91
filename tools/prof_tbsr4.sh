mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_tbsr_mv -c 1 -o gpurun_out/prof_tbsr_c4 python tools/mv_probe.py 4 1 > gpurun_out/ncu_tbsr_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_matvec -c 1 -o gpurun_out/prof_mvcsr_c4 python tools/mv_probe.py 4 1 > gpurun_out/ncu_mvcsr_c4.log 2>&1
