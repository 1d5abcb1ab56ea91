"""Build libtdb.so (sm_100a) in-tree with nvcc.

    python -m paper_1503_07221_b200.build [--force]

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtdb.so")
SOURCES = ["tdb_context.cu", "tdb_pair.cu", "tdb_assembly.cu", "tdb_matvec.cu", "tdb_krylov.cu", "tdb_band.cu", "tdb_potential.cu", "tdb_rhs.cu", "tdb_tables.cu"]
HEADERS = ["tdb_common.cuh", "tdb_quad_cells.cuh", "tdb_internal.h", "tdb_band.h", "tdb_async.cuh", "tdb_geometry.cuh", "tdb_basis.cuh", os.path.join("..", "..", "include", "tdb.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS if os.path.exists(os.path.join(CSRC, s))]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra_flags=(), out: str | None = None) -> str:
    """Compile every CUDA source for sm_100a and link libtdb.so (or `out`, a tuning variant
    built with `extra_flags`, e.g. -DTDB_QW=12; load it with TDB_LIBRARY=<path>)."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    objdir = os.path.join(HERE, "build") if out is None else os.path.join("/tmp", "tdb_objs_" + os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    # one nvcc per translation unit, in parallel, then a host link
    procs = []
    objs = []
    for src in srcs:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [_nvcc(), *NVCC_FLAGS, *extra_flags, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    for cmd, pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed ({pr.returncode}): {' '.join(cmd)}\n{out}\n{err}")
        if verbose:
            print(err)
    tmp = lib + ".tmp"
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
