"""GPU parity of the opt-in tensor-core matvec (TDB_MV_BSR=1, csrc/tdb_bsr.cu).

The switch is read once per process, so the BSR side runs in a subprocess and
its results are compared here with the default CSR kernel (itself pinned to the
reference goldens in test_gpu_parity.py) and with the reference's own p = 0
golden matvec.  Tolerance: 1e-12 relative 2-norm, as for the CSR matvec.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1503_07221_b200.block_system import assemble_system
from paper_1503_07221_b200.mesh import SurfaceMesh, icosphere
from paper_1503_07221_b200.temporal_basis import TimeGrid
out = {}
verts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 1.0, 0.5]])
two = SurfaceMesh(verts, np.array([[0, 1, 2], [1, 3, 2]]))
g = np.load(sys.argv[2])
A = assemble_system(two, TimeGrid(T=2.0, N=3, p=0))
out["two_tri"] = (A @ g["x7"]).tolist()
A = assemble_system(icosphere(2), TimeGrid(T=3.9, N=40, p=0))
x = np.random.default_rng(7).standard_normal(A.shape[1])
out["full"] = (A @ x).tolist()
M = A.M
for lo, hi in [(1, 20), (21, 40), (11, 30)]:
    xs = x[(lo - 1) * M: hi * M]
    out[f"{lo}_{hi}"] = A.matvec(xs, rows=(lo, hi), cols=(lo, hi)).tolist()
out["off"] = A.matvec(x[:20 * M], rows=(21, 40), cols=(1, 20)).tolist()
print(json.dumps(out))
"""


def test_bsr_matvec_matches_csr_and_golden():
    from paper_1503_07221_b200.block_system import assemble_system
    from paper_1503_07221_b200.mesh import SurfaceMesh, icosphere
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    gpath = os.path.join(ROOT, "tests", "golden", "blocks_two_tri_N3_p0.npz")
    env = dict(os.environ, TDB_MV_BSR="1")
    res = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, gpath], capture_output=True, text=True, env=env,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    bsr = json.loads(res.stdout.strip().splitlines()[-1])
    g = golden("blocks_two_tri_N3_p0.npz")
    assert np.linalg.norm(np.array(bsr["two_tri"]) - g["y7"]) <= 1e-12 * np.linalg.norm(g["y7"])
    A = assemble_system(icosphere(2), TimeGrid(T=3.9, N=40, p=0))
    x = np.random.default_rng(7).standard_normal(A.shape[1])
    M = A.M
    ref = {"full": A @ x, "off": A.matvec(x[:20 * M], rows=(21, 40), cols=(1, 20))}
    for lo, hi in [(1, 20), (21, 40), (11, 30)]:
        ref[f"{lo}_{hi}"] = A.matvec(x[(lo - 1) * M: hi * M], rows=(lo, hi), cols=(lo, hi))
    for k, y in ref.items():
        got = np.array(bsr[k])
        assert np.linalg.norm(got - y) <= 1e-12 * np.linalg.norm(y), k
