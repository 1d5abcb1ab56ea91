mkdir -p gpurun_out
for v in nc1m24 nc1m32; do echo "== $v"; TDB_LIBRARY=tools/_variants/libtdb_$v.so python tools/mv_probe.py 2 2>&1 | grep "rows(1, 20)"; TDB_LIBRARY=tools/_variants/libtdb_$v.so python tools/mv_probe.py 4 2>&1 | grep "rows(1, 40)"; TDB_LIBRARY=tools/_variants/libtdb_$v.so python tools/solve_probe.py 2 2>&1 | tail -1; done > gpurun_out/nc1.txt 2>&1
echo "== base" >> gpurun_out/nc1.txt; python tools/solve_probe.py 2 2>&1 | tail -1 >> gpurun_out/nc1.txt
