"""ctypes binding of libtdb.so (the C ABI in include/tdb.h).

There is no CPU fallback: importing this module on a machine without the
built library raises, and every call that needs a GPU raises a RuntimeError
carrying the library's own error message when no device is visible.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TDB_LIBRARY") or os.path.join(HERE, "libtdb.so")  # override: tuning variants

i32, i64, f64p, i64p, i32p, u8p = C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_uint8)

TDB_OK = 0
_ERRORS = {
    -1: ValueError,
    -2: RuntimeError,
    -3: MemoryError,
    -4: RuntimeError,
    -5: NotImplementedError,
}


class TdbPsiPack(C.Structure):
    _fields_ = [
        ("p", i32), ("deg", i32), ("max_nsub", i32), ("reserved", i32),
        ("delta", C.c_double),
        ("lo", f64p), ("width", f64p), ("nsub", i64p), ("coeffs", f64p),
        ("sp", f64p), ("sn", f64p), ("fold", u8p), ("active", u8p),
    ]


class TdbMesh(C.Structure):
    _fields_ = [
        ("num_vertices", i64), ("num_triangles", i64),
        ("corners", f64p), ("a2", f64p), ("normals", f64p), ("curls", f64p),
        ("triangles", i64p), ("star_off", i64p), ("star_ids", i64p),
    ]


class TdbFamily(C.Structure):
    _fields_ = [
        ("npos", i32), ("reserved", i32),
        ("delta", f64p), ("slo", f64p), ("shi", f64p),
        ("pack", TdbPsiPack),
    ]


class TdbRule(C.Structure):
    _fields_ = [("nq", i64), ("xhat", f64p), ("yhat", f64p), ("w", f64p)]


class TdbAssemblyDesc(C.Structure):
    _fields_ = [
        ("p", i32), ("num_families", i32),
        ("families", C.POINTER(TdbFamily)),
        ("rules", TdbRule * 4),
        ("num_rows", i64), ("rows", i64p),
    ]


class TdbStats(C.Structure):
    _fields_ = [
        ("units", i64), ("items", i64), ("n_in", i64), ("n_geom", i64), ("nnz_total", i64),
        ("ms_plan", C.c_double), ("ms_quad", C.c_double), ("ms_finalize", C.c_double),
        ("ms_pattern", C.c_double), ("ms_total", C.c_double),
        ("units_case", i64 * 4), ("pairs_case", i64 * 4), ("launches", i64), ("units_primary", i64),
        ("ms_quad_cells", C.c_double), ("n_in_cells", i64), ("pairs_cells", i64),
    ]

    def as_dict(self) -> dict:
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if not isinstance(v, (int, float)) else v
        return out


class TdbMatvecDesc(C.Structure):
    _fields_ = [
        ("N", i32), ("rlo", i32), ("rhi", i32), ("clo", i32), ("chi", i32),
        ("nterms", i32), ("words", i32), ("reserved", i32),
        ("term_family", i32p), ("term_pos", i32p), ("term_d", i32p),
        ("term_mask", C.POINTER(C.c_uint32)),
        ("x_stride", i64), ("x_map", i64p),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1503_07221_b200.build` "
            "(nvcc, sm_100a). There is no CPU fallback."
        )
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "tdb_abi_version": (i32, []),
        "tdb_release_cached_memory": (i32, []),
        "tdb_fp64_peak": (i32, [P, C.c_int, C.POINTER(C.c_double)]),
        "tdb_last_error": (C.c_char_p, []),
        "tdb_device_count": (i32, [C.POINTER(C.c_int)]),
        "tdb_pair_block_contributions": (
            i32, [f64p] * 10 + [i64, i64, C.POINTER(TdbPsiPack), f64p]),
        "tdb_ctx_create": (i32, [C.c_int, C.POINTER(P)]),
        "tdb_ctx_destroy": (i32, [P]),
        "tdb_ctx_set_stream": (i32, [P, P]),
        "tdb_tri_distance_bounds": (i32, [P, C.POINTER(TdbMesh), i64, i64p, f64p, f64p]),
        "tdb_system_assemble": (i32, [P, C.POINTER(TdbMesh), C.POINTER(TdbAssemblyDesc), C.POINTER(P)]),
        "tdb_system_create": (i32, [P, C.POINTER(TdbMesh), C.POINTER(TdbAssemblyDesc), C.POINTER(P)]),
        "tdb_system_run": (i32, [P]),
        "tdb_system_destroy": (i32, [P]),
        "tdb_system_stats": (i32, [P, C.POINTER(TdbStats)]),
        "tdb_system_family_nnz": (i32, [P, i32, C.POINTER(i64)]),
        "tdb_system_copy_family": (i32, [P, i32, i64p, i32p, f64p]),
        "tdb_system_position_units": (i32, [P, i32, i64p]),
        "tdb_system_family_split": (i32, [P, i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
        "tdb_system_family_device": (i32, [P, i32, C.POINTER(P), C.POINTER(P), C.POINTER(P)]),
        "tdb_matvec_plan_create": (i32, [P, C.POINTER(TdbMatvecDesc), C.POINTER(P)]),
        "tdb_matvec_plan_destroy": (i32, [P]),
        "tdb_matvec": (i32, [P, P, P]),
        "tdb_matvec_plan_work": (i32, [P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "tdb_matvec_plan_kind": (i32, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        # device-side GMRES cycle bookkeeping (pointers are device addresses)
        "tdb_krylov_init": (i32, [P, P, C.c_double, P, P]),
        "tdb_krylov_givens": (i32, [P, i32, P, P, i32, P, P, P, P]),
        "tdb_krylov_update": (i32, [P, P, P, i64, i64, P, P, i32, P, i32, P]),
        "tdb_krylov_flag": (i32, [P, P, P]),
        "tdb_krylov_arnoldi": (i32, [P, i64, i64, i32, P, P, P, P, i32, P, P, P, P, P]),
        "tdb_table_node_values": (i32, [P, C.c_double, i32, i32, i32p, f64p, i32, f64p, i32p, f64p, i32, f64p, f64p,
                                        f64p]),
        "tdb_rhs_vertex_gather": (i32, [P, i64, i64, i64, P, P, P, i64, P, P]),
        "tdb_rhs_time_sum": (i32, [P, P, P, i64, i64, P, P]),
        "tdb_dlp_eval": (i32, [P, C.POINTER(TdbMesh), C.c_double, i32, i32, f64p, i64, f64p, i64, f64p, i32,
                               f64p, f64p, i32, f64p, f64p, f64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()

# every symbol include/tdb.h declares (checked by tests/test_capi_symbols.py)
EXPORTED = (
    "tdb_abi_version", "tdb_last_error", "tdb_device_count", "tdb_pair_block_contributions",
    "tdb_ctx_create", "tdb_ctx_destroy", "tdb_ctx_set_stream", "tdb_system_assemble",
    "tdb_system_destroy", "tdb_system_stats", "tdb_system_family_nnz", "tdb_system_copy_family",
    "tdb_system_position_units", "tdb_system_family_split",
    "tdb_system_family_device", "tdb_matvec_plan_create", "tdb_matvec_plan_destroy", "tdb_matvec",
    "tdb_matvec_plan_work", "tdb_matvec_plan_kind", "tdb_tri_distance_bounds", "tdb_system_create", "tdb_system_run",
    "tdb_fp64_peak", "tdb_krylov_init", "tdb_krylov_givens", "tdb_krylov_update", "tdb_krylov_flag",
    "tdb_krylov_arnoldi", "tdb_release_cached_memory", "tdb_dlp_eval",
    "tdb_rhs_vertex_gather", "tdb_rhs_time_sum", "tdb_table_node_values",
)

# TDB_KS_* cycle-state slots (include/tdb.h)
KS_DONE, KS_KDONE, KS_BREAKDOWN, KS_TOL_ABS, KS_BETA, KS_CONVERGED, KS_NSTATE = 0, 1, 2, 3, 4, 5, 8


def check(rc: int, what: str = "") -> None:
    if rc != TDB_OK:
        msg = LIB.tdb_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(f"libtdb {what} failed ({rc}): {msg}")


def ptr(a: np.ndarray, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def device_count() -> int:
    n = C.c_int(0)
    check(LIB.tdb_device_count(C.byref(n)), "device_count")
    return n.value


class Context:
    """One CUDA device + stream (include/tdb.h TdbContext); not thread-safe."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(LIB.tdb_ctx_create(device, C.byref(h)), "ctx_create")
        self.handle = h
        self.device = device

    def set_stream(self, stream_ptr: int) -> None:
        check(LIB.tdb_ctx_set_stream(self.handle, C.c_void_p(stream_ptr)), "ctx_set_stream")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and LIB is not None:  # LIB is None at interpreter exit
            LIB.tdb_ctx_destroy(h)
            self.handle = None


_CTX: dict = {}


def default_context(device: int | None = None) -> Context:
    if device is None:
        device = int(os.environ.get("TDB_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    ctx = _CTX.get(device)
    if ctx is None:
        ctx = _CTX[device] = Context(device)
    return ctx


def fp64_peak_tflops(ctx: "Context | None" = None, repeats: int = 5) -> float:
    """Measured DFMA throughput of the device (TFLOP/s)."""
    ctx = ctx or default_context()
    out = C.c_double()
    check(LIB.tdb_fp64_peak(ctx.handle, repeats, C.byref(out)), "fp64_peak")
    return out.value
