"""VTU writer golden from the REFERENCE write_vtu (tdbem.cli.write_vtu, cli.py:268-309).

    python tests/golden/make_golden_vtu.py [--refpkg /root/reference/pkg]
"""
import argparse
import os
import sys

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--refpkg", default="/root/reference/pkg")
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(args.refpkg, "src"))
    from tdbem.cli import write_vtu

    rng = np.random.default_rng(3)
    pts = rng.standard_normal((12, 3))
    vals = rng.standard_normal(12)
    write_vtu(os.path.join(OUT, "field_quad_ref.vtu"), pts, vals, (3, 4))
    write_vtu(os.path.join(OUT, "field_vertex_ref.vtu"), pts[:5], vals[:5])
    np.savez(os.path.join(OUT, "vtu_inputs.npz"), pts=pts, vals=vals)


if __name__ == "__main__":
    main()
