# usage: bash tools/build_variants.sh name "-DFOO=1 ..." [name "-D..."]...  -> tools/_variants/libtdb_<name>.so
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/_variants
S=paper_1503_07221_b200/csrc
while [ $# -gt 0 ]; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $2 \
    -shared -o tools/_variants/libtdb_$1.so $S/tdb_context.cu $S/tdb_pair.cu $S/tdb_assembly.cu $S/tdb_matvec.cu -lcudart &
  shift 2
done
wait
ls -la tools/_variants
