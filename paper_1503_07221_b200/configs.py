"""The BASELINE.json benchmark configurations (synthetic inputs, built in memory).

Meshes are generated exactly as SURVEY.md 8(d) prescribes: unit-radius
icospheres from icosahedron + refine(project_unit_sphere=True), and the seeded
jittered unit cube (16 x 16 x 2 triangles per face, +-5% h, seed 0).
Temporal order p = 0 (the order BASELINE's storage figures correspond to,
SURVEY finding 3).  T = dt (N - 1).  The reference's quadrature rules are used
(q_reg = 4 -> 256 points per regular pair; SURVEY finding 2: the configs' "7-point
Gauss" does not exist in the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

from .mesh import icosphere, jittered_cube
from .temporal_basis import TimeGrid

__all__ = ["Config", "CONFIGS", "get_config"]


@dataclass(frozen=True)
class Config:
    index: int
    name: str
    mesh_kind: str
    level: int
    dt: float
    N: int
    p: int = 0

    def mesh(self):
        if self.mesh_kind == "icosphere":
            return icosphere(self.level)
        return jittered_cube(16, 0.05, 0)

    def grid(self) -> TimeGrid:
        # T written as its decimal value (3.9, 3.95, ...), as the survey's runs did
        return TimeGrid(T=float(f"{self.dt * (self.N - 1):.12g}"), N=self.N, p=self.p)


CONFIGS = {
    1: Config(1, "icosphere2_E320_dt0.1_N40", "icosphere", 2, 0.1, 40),
    2: Config(2, "icosphere3_E1280_dt0.05_N80", "icosphere", 3, 0.05, 80),
    3: Config(3, "cube16_E3072_dt0.05_N100", "cube", 0, 0.05, 100),
    4: Config(4, "icosphere4_E5120_dt0.025_N160", "icosphere", 4, 0.025, 160),
    5: Config(5, "icosphere5_E20480_dt0.025_N320", "icosphere", 5, 0.025, 320),
}


def get_config(i: int) -> Config:
    return CONFIGS[int(i)]
