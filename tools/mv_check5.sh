mkdir -p gpurun_out
for c in 2 4; do
 for w in 32 48; do
  echo "== cfg$c W$w"; TDB_TBSR_WARPS_PER_SM=$w timeout 300 python tools/mv_probe.py $c 2>&1 | grep -i "matvec\|error"
  echo "== cfg$c W$w pred"; TDB_TBSR_WARPS_PER_SM=$w TDB_LIBRARY=tools/_variants/libtdb_tpred.so timeout 300 python tools/mv_probe.py $c 2>&1 | grep -i "matvec\|error"
 done
done > gpurun_out/mv5.txt 2>&1
