mkdir -p gpurun_out
for v in base lif16 lif24 mb24 mb24l16 mb12l24; do echo "== $v"; TDB_LIBRARY=tools/_variants/libtdb_$v.so python tools/mv_probe.py 2 2>&1 | grep matvec; done > gpurun_out/mvsweep2.txt
for w in 24 96; do echo "== base W$w"; TDB_MV_WARPS_PER_SM=$w TDB_LIBRARY=tools/_variants/libtdb_base.so python tools/mv_probe.py 2 2>&1 | grep matvec; done >> gpurun_out/mvsweep2.txt
for v in base mb24 mb24l16; do echo "== $v"; TDB_LIBRARY=tools/_variants/libtdb_$v.so python tools/mv_probe.py 4 2>&1 | grep matvec; done > gpurun_out/mvsweep4.txt
