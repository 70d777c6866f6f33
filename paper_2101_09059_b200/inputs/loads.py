"""Prescribed wall traction -> nodal forces (input generation, done once).

One-way coupling: the rigid-wall fluid solution gives the wall traction, t^s = -t^f
(Eq. 20); "at every node ... the shear forces and normal vectors
from adjacent elements are averaged and the nodal pressure added".
The fluid solve itself is out of scope: the Poiseuille pressure
drop on the cylinder is 12.7 Ba over 30 cm against the 17,332 Ba superposed pressure
(SURVEY.md A32), so the load is the uniform superposed pressure.

Reading: consistent piecewise-constant integration
    F_i = sum_{e ni i} (A_e / 3) * p * n_e        (n_e outward unit normal)
which gives an exactly zero net force on a closed surface.

The ens_set_traction contract (include/ens.h) is f(t) = ramp(t) * sum_k g_k(t) F_k with
g_k a periodic piecewise-linear table and ramp(t) = sin(pi t / (2 T_r)) for t < T_r
(SURVEY.md C13 #7).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MMHG = 1333.22           # Ba per mmHg
P_SUPERPOSED = 13.0 * MMHG   # 13 mmHg = MAP - diastolic


def pressure_forces(xyz: np.ndarray, tris: np.ndarray, p: float = 1.0) -> np.ndarray:
    """Nodal forces [V][3] (dyn) of a uniform internal pressure p (Ba)."""
    X = xyz[tris]
    n2 = np.cross(X[:, 1] - X[:, 0], X[:, 2] - X[:, 0])     # = 2 A_e n_e (outward)
    F = np.zeros_like(xyz)
    contrib = (p / 6.0) * n2                                  # (A_e/3) p n_e
    for a in range(3):
        np.add.at(F, tris[:, a], contrib)
    return F


@dataclass
class Traction:
    """Arguments of ens_set_traction."""
    F: np.ndarray          # [K][V][3]
    tab_t: np.ndarray      # [n_tab]
    tab_g: np.ndarray      # [K][n_tab]
    period: float
    ramp_T: float

    @property
    def n_fields(self) -> int:
        return int(self.F.shape[0])


def steady(xyz, tris, p: float = P_SUPERPOSED, ramp_T: float = 0.0) -> Traction:
    """Steady uniform pressure (configs c1, c2)."""
    F = pressure_forces(xyz, tris, p)[None]
    return Traction(np.ascontiguousarray(F), np.zeros(0), np.zeros((1, 0)), 0.0, ramp_T)


def pulsatile(xyz, tris, *, p_base: float = P_SUPERPOSED, p_amp: float = 27.0 * MMHG,
              period: float = 0.8, systole: float = 0.3, n_tab: int = 801,
              ramp_T: float = 0.2) -> Traction:
    """Synthetic pulsatile load (configs c3, c4):
    p(t) = 13 mmHg + 27 mmHg * max(0, sin(pi tau / 0.3 s)), tau = t mod 0.8 s,
    tabulated every 1 ms and interpolated linearly; sine ramp over 0.2 s."""
    F1 = pressure_forces(xyz, tris, 1.0)
    F = np.stack([p_base * F1, p_amp * F1])
    t = np.linspace(0.0, period, n_tab)
    g = np.stack([np.ones(n_tab), np.maximum(0.0, np.sin(np.pi * t / systole))])
    g[1, t >= systole] = 0.0
    return Traction(np.ascontiguousarray(F), t, np.ascontiguousarray(g), period, ramp_T)
