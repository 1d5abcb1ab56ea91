mkdir -p gpurun_out
for w in 32 48 64 96; do for c in 2 4; do echo "== W$w cfg$c"; TDB_TBSR_WARPS_PER_SM=$w python tools/mv_probe.py $c 2>&1 | grep "rows(1, 80) cols(1, 80)\|rows(1, 160)\|rows(41, 80) cols(41\|rows(81, 160) cols(81"; done; done > gpurun_out/tbsr_w.txt 2>&1
