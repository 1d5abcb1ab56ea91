"""Drop-in for the reference plugin point ``tdbem._kernels``.

/root/reference/pkg/src/tdbem/_kernels/__init__.py:1-34 picks a backend at
import time and exports ``pair_block_contributions`` and ``backend_name``.
This module has exactly one backend, the sm_100a kernel in libtdb.so
(csrc/tdb_pair.cu); there is no NumPy or Cython fallback.  Installing it into
a reference process is one assignment:

    import tdbem._kernels as K
    from paper_1503_07221_b200 import _kernels as G
    K.pair_block_contributions = G.pair_block_contributions
"""

from __future__ import annotations

import numpy as np

from . import _lib

backend_name = "cuda-sm100a"

__all__ = ["pair_block_contributions", "backend_name"]


def pair_block_contributions(cx, cy, a2x, a2y, ndot, curly, curlx, xhat, yhat, wq, pack):
    """(npair, p+1, p+1, 3, 3) contributions [pair, m2, m1, a(y), b(x)] of one block position."""
    f = _lib.f64
    cx, cy, curly, curlx = f(cx), f(cy), f(curly), f(curlx)
    a2x, a2y, ndot = f(a2x), f(a2y), f(ndot)
    xhat, yhat, wq = f(xhat), f(yhat), f(wq)
    npair = cx.shape[0]
    for name, arr, shape in (("cx", cx, (npair, 3, 3)), ("cy", cy, (npair, 3, 3)),
                             ("curly", curly, (npair, 3, 3)), ("curlx", curlx, (npair, 3, 3)),
                             ("a2x", a2x, (npair,)), ("a2y", a2y, (npair,)), ("ndot", ndot, (npair,))):
        if arr.shape != shape:
            raise ValueError(f"{name} has shape {arr.shape}, expected {shape}")
    nq = wq.shape[0]
    if xhat.shape != (nq, 2) or yhat.shape != (nq, 2):
        raise ValueError("xhat/yhat must have shape (nq, 2)")
    keep: list = []
    from .assembly import PsiPack

    cpack = PsiPack.to_c(pack, keep) if not isinstance(pack, PsiPack) else pack.to_c(keep)
    np1 = int(pack.p) + 1
    out = np.empty((npair, np1, np1, 3, 3))
    if npair == 0:
        return out
    P = _lib.ptr
    _lib.check(_lib.LIB.tdb_pair_block_contributions(
        P(cx), P(cy), P(a2x), P(a2y), P(ndot), P(curly), P(curlx), P(xhat), P(yhat), P(wq),
        npair, nq, _lib.C.byref(cpack), P(out)), "pair_block_contributions")
    return out
