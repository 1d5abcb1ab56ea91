# usage: bash tools/build_variants.sh name "-DFOO=1 ..." [name "-D..."]...  -> tools/_variants/libtdb_<name>.so
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/_variants/obj
S=paper_1503_07221_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for f in tdb_context tdb_pair tdb_matvec tdb_krylov tdb_bsr tdb_tbsr tdb_potential tdb_rhs tdb_tables; do
  [ tools/_variants/obj/$f.o -nt $S/$f.cu ] || nvcc $F -c -o tools/_variants/obj/$f.o $S/$f.cu &
done
wait
while [ $# -gt 0 ]; do
  ( nvcc $F $2 -c -o tools/_variants/obj/asm_$1.o $S/tdb_assembly.cu && \
    nvcc $F $2 -c -o tools/_variants/obj/mv_$1.o $S/tdb_matvec.cu && \
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/_variants/libtdb_$1.so tools/_variants/obj/asm_$1.o \
      tools/_variants/obj/tdb_context.o tools/_variants/obj/tdb_pair.o tools/_variants/obj/mv_$1.o \
      tools/_variants/obj/tdb_krylov.o tools/_variants/obj/tdb_bsr.o tools/_variants/obj/tdb_tbsr.o tools/_variants/obj/tdb_potential.o tools/_variants/obj/tdb_rhs.o tools/_variants/obj/tdb_tables.o -lcudart ) &
  shift 2
done
wait
ls -la tools/_variants
