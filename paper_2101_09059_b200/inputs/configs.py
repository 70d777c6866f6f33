"""The BASELINE.json workloads as seeded synthetic inputs.

c1  ideal cylinder ~500 tri (12x23 rings), N_s = 4, steady 13 mmHg, 2,000 steps, fp64
c2  ideal cylinder ~50k tri (96x262), N_s = 64, steady, mode-1 damping 250 1/s (Laplace)
c3  as c2, pulsatile traction over 3 cardiac cycles, undamped
c4  synthetic branched aorta ~500k tri (mesh.aorta), N_s = 128, pulsatile, E 7e6 +- 7e5,
    zeta 0.2 +- 0.02 cm; every realisation an independent GMRF draw
c5  the same generator at ~2M tri, N_s = 512, independent draws too (~1,000 solves on 1M
    nodes in 4-column groups on a thread pool)

Material statistics: E 7.0e6 +- 7.0e5 Ba, zeta 0.4 +- 0.04 cm, rho_corr 3.7 cm
(PAPER.md:436); density 1.06 g/cm^3; nu = 0.5, k = 5/6
(PAPER.md:200).  Seeds: 20210121 + 1000 * config index.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fields, loads, mesh as meshmod

RHO = 1.06
NU = 0.5
K_SHEAR = 5.0 / 6.0
E_MEAN, E_STD = 7.0e6, 7.0e5
H_MEAN, H_STD = 0.4, 0.04
RHO_CORR = 3.7

DAMP_NONE, DAMP_MASS, DAMP_IDENTITY = 0, 1, 2


@dataclass
class Config:
    name: str
    mesh: meshmod.Mesh
    E: np.ndarray            # [n_s][V]
    h: np.ndarray            # [n_s][V]
    traction: loads.Traction
    rho: float = RHO
    nu: float = NU
    k_shear: float = K_SHEAR
    damping: int = DAMP_NONE
    c_d: float = 0.0
    steps: int = 2000
    s_begin: int = 0

    @property
    def n_s(self) -> int:
        return int(self.E.shape[0])

    @property
    def dof(self) -> int:
        return 3 * self.mesh.n_nodes


_RINGS = {"c1": (12, 23), "c2": (96, 262), "c3": (96, 262)}
_AORTA = {"c4": (500_000, 128), "c5": (2_000_000, 512)}


def make_aorta(name: str, n_s: int | None = None, s_begin: int = 0, target_tris: int | None = None) -> Config:
    """Configs c4 / c5: branched aorta, pulsatile, all ends fixed."""
    idx = int(name[1])
    seed = 20210121 + 1000 * idx
    tt, ns_def = _AORTA[name]
    m = meshmod.aorta(target_tris or tt)
    ns = n_s or ns_def
    # every realisation an independent GMRF draw: one sparse LU, then
    # 2 x (N_s - 1) solves in 4-column groups on a thread pool (c4 ~10 s, c5 ~1.5 min)
    E, h, _ = fields.sample_materials(m.xyz, m.tris, ns, E_mean=E_MEAN, E_std=E_STD,
                                      h_mean=0.2, h_std=0.02, rho_corr=RHO_CORR,
                                      seed=seed, s_begin=s_begin)
    tr = loads.pulsatile(m.xyz, m.tris)
    return Config(name, m, E, h, tr, damping=DAMP_NONE, c_d=0.0, steps=2000, s_begin=s_begin)


def make(name: str, n_s: int | None = None, s_begin: int = 0, n_circ: int | None = None,
         n_axial: int | None = None) -> Config:
    """Build config `name` (c1..c5), optionally overriding N_s or the ring counts."""
    if name in _AORTA:
        return make_aorta(name, n_s=n_s, s_begin=s_begin)
    idx = int(name[1])
    seed = 20210121 + 1000 * idx
    nc, na = _RINGS[name]
    nc = n_circ or nc
    na = n_axial or na
    m = meshmod.cylinder(nc, na)
    ns = n_s or {"c1": 4, "c2": 64, "c3": 64}[name]
    E, h, _ = fields.sample_materials(m.xyz, m.tris, ns, E_mean=E_MEAN, E_std=E_STD,
                                      h_mean=H_MEAN, h_std=H_STD, rho_corr=RHO_CORR,
                                      seed=seed, s_begin=s_begin)
    if name == "c3":
        tr = loads.pulsatile(m.xyz, m.tris)
        return Config(name, m, E, h, tr, damping=DAMP_NONE, c_d=0.0, steps=69_600,
                      s_begin=s_begin)
    tr = loads.steady(m.xyz, m.tris)
    if name == "c2":
        return Config(name, m, E, h, tr, damping=DAMP_MASS, c_d=250.0, steps=10_000,
                      s_begin=s_begin)
    return Config(name, m, E, h, tr, damping=DAMP_NONE, c_d=0.0, steps=2000, s_begin=s_begin)
