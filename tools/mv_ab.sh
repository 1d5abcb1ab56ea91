# usage (GPU box): bash tools/mv_ab.sh <cfg>  - matvec timings, BSR (TDB_MV_BSR=1) vs CSR (default)
echo "== BSR"; TDB_MV_BSR=1 python tools/mv_quarter.py $1 2>&1; TDB_MV_BSR=1 python tools/mv_probe.py $1 2>&1 | grep "matvec rows(1, " | head -1
echo "== CSR"; python tools/mv_quarter.py $1 2>&1; python tools/mv_probe.py $1 2>&1 | grep "matvec rows(1, " | head -1
