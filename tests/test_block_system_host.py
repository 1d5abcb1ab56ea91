"""Host logic of the block system (mirrors reference tests/test_block_system.py:38-106)."""

import numpy as np
import pytest

from paper_1503_07221_b200.block_system import (
    canonical_position,
    canonical_positions,
    inner_nonzero_count,
    is_zero_position,
    n_tilde_z,
    plan_distribution,
)
from paper_1503_07221_b200.temporal_basis import TimeGrid
from conftest import golden

GRID = TimeGrid(T=2.0, N=4, p=1)


def test_inner_count_matches_brute_force():
    for n in range(4, 31):
        for ntz in range(2, n + 1):
            brute = sum(1 for kt in range(2, n) for it in range(2, n) if -1 <= kt - it < ntz)
            assert inner_nonzero_count(n, ntz) == brute


def test_canonical_position():
    assert canonical_position(GRID, 1, 3) is None
    assert canonical_position(GRID, 2, 4) is None
    g = TimeGrid(T=4.0, N=8, p=0)
    assert canonical_position(g, 5, 3) == (4, 2)
    assert canonical_position(g, 4, 4) == (2, 2)
    assert canonical_position(g, 3, 4) == (2, 3)
    assert canonical_position(GRID, 1, 1) == (1, 1)
    assert canonical_position(GRID, GRID.N, 2) == (GRID.N, 2)


def test_plan_distribution(two_tri):
    g = TimeGrid(T=4.0, N=8, p=0)
    with pytest.raises(ValueError):
        plan_distribution(GRID, two_tri, 0)
    plan = plan_distribution(g, two_tri, 3)
    want = {(kt, it) for kt in range(1, 9) for it in range(1, 9) if -1 <= kt - it < plan.n_tilde_z}
    assert set(plan.owners) == want
    for P in (1, 2, 3, 5):
        loads = plan_distribution(g, two_tri, P).rank_loads(g)
        assert loads.sum() == plan_distribution(g, two_tri, P).n_z and loads.max() - loads.min() <= 1
    assert n_tilde_z(TimeGrid(T=2.0, N=4, p=0), 100.0) == 4


def test_light_cone_tie_positions_cfg1(cfg1_mesh):
    # finding 11: the FP64 cut keeps lag 22 at some logical positions only; the canonical
    # set must equal the reference's (golden all_positions)
    g = golden("blocks_cfg1.npz")
    grid = TimeGrid(T=3.9, N=40, p=0)
    pos = canonical_positions(grid, cfg1_mesh.diameter)
    assert pos == [tuple(int(v) for v in r) for r in g["all_positions"]]
    # the cut is decided per logical position with FP64 t_formal differences
    assert all(is_zero_position(grid, cfg1_mesh.diameter, kt, kt - 23) for kt in range(25, 40))
    assert (24, 2) in pos and (25, 2) not in pos
