"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds none of the method's arithmetic:
  * mesh descriptions (plain numbers: element counts, extents, periodicity,
    deformation flag) for the BASELINE.json configs C1..C5;
  * seeded random nodal fields (numpy default_rng, so both sides see the same
    bytes);
  * closed-form manufactured functions f and exact solutions u*, evaluated at
    caller-supplied coordinates (each side passes its own node coordinates).

Neither `oracle/` nor `paper_2107_01243_b200/` is imported here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class MeshSpec:
    """Hexahedral box mesh ("E non-overlapping hexahedral elements")."""

    ex: int
    ey: int
    ez: int
    x0: float = 0.0
    x1: float = 1.0
    y0: float = 0.0
    y1: float = 1.0
    z0: float = 0.0
    z1: float = 1.0
    periodic: tuple = (0, 0, 0)
    deform: int = 0
    deform_amp: float = 0.15

    @property
    def E(self) -> int:
        return self.ex * self.ey * self.ez

    def n_slots(self, N: int) -> int:
        return self.E * (N + 1) ** 3


def unit_box(ex, ey, ez, periodic=(0, 0, 0)) -> MeshSpec:
    return MeshSpec(ex, ey, ez, periodic=tuple(periodic))


def tgv_box(ex, ey, ez, deform=0, amp=0.15) -> MeshSpec:
    return MeshSpec(ex, ey, ez, 0.0, TWO_PI, 0.0, TWO_PI, 0.0, TWO_PI,
                    periodic=(1, 1, 1), deform=deform, deform_amp=amp)


# BASELINE.json configs (SURVEY.md section 8 table and 8(d) input recipe)
CONFIGS = {
    # C1: 2x2x2 Dirichlet unit box, N=3, manufactured sin solution, PCG to 1e-10
    "C1": (unit_box(2, 2, 2), 3),
    # C2: 8192-element Cartesian box, N=7 (BP5-like, all 6 G stored)
    "C2": (unit_box(32, 16, 16, periodic=(1, 1, 1)), 7),
    # C3: TGV pressure-Poisson, 32^3 elements, N=7, (0,2pi)^3 periodic
    "C3": (tgv_box(32, 32, 32), 7),
    # C4: deformed curvilinear mesh (a=0.15), 64^3 elements, N=7, periodic
    "C4": (tgv_box(64, 64, 64, deform=1), 7),
}


def c5_mesh(N: int) -> MeshSpec:
    """C5 sweep: E_axis = round(1000/(N+1)) in x,y; z rounded to a multiple of 8."""
    ea = int(round(1000.0 / (N + 1)))
    ez = max(8, int(round(ea / 8.0)) * 8)
    return tgv_box(ea, ea, ez)


def weak_scaled(spec: MeshSpec, P: int) -> MeshSpec:
    """Stack P copies of the per-GPU box along z (fixed per-GPU work)."""
    return replace(spec, ez=spec.ez * P, z1=spec.z0 + (spec.z1 - spec.z0) * P)


def random_field(n: int, seed: int = 0) -> np.ndarray:
    """u ~ U[-1, 1) i.i.d. per slot (SURVEY 8(d) C2 recipe)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


# --- manufactured solutions (closed forms) ---------------
def u_sin(x, y, z, xp=np):
    return xp.sin(math.pi * x) * xp.sin(math.pi * y) * xp.sin(math.pi * z)


def f_sin(x, y, z, xp=np):
    """-lap(u_sin) = 3 pi^2 u_sin (Dirichlet unit box, Eqs. 4-5)."""
    return 3.0 * math.pi ** 2 * u_sin(x, y, z, xp)


def p_tgv(x, y, z, xp=np):
    """Closed-form Taylor-Green pressure (reading Q19)."""
    return (xp.cos(2 * x) + xp.cos(2 * y)) * (xp.cos(2 * z) + 2.0) / 16.0


def f_tgv(x, y, z, xp=np):
    """-lap(p_tgv) = 1/2 (cos 2x + cos 2y)(1 + cos 2z); zero mean on the box."""
    return 0.5 * (xp.cos(2 * x) + xp.cos(2 * y)) * (1.0 + xp.cos(2 * z))
