# usage: bash tools/mv_variants.sh config name...   (GPU box)
c=$1; shift
for v in "$@"; do echo "== $v"; TDB_LIBRARY=tools/_variants/libtdb_$v.so python tools/mv_probe.py $c 2>&1 | grep matvec; done
