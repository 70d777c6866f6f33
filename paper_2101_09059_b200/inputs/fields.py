"""Seeded Matérn random fields for E and thickness zeta (input generation, done once).

Paper: nodal vectors E ~ N(E_bar, Q_alpha^-1) and zeta ~ N(zeta_bar, Q_alpha^-1)
(Eq. 11) with the SPDE/GMRF precision of Lindgren et al.
(Eqs. 2-6).  Readings:

* Matérn smoothness nu = 1, d = 2  =>  alpha = nu + d/2 = 2.
* kappa = sqrt(8 nu) / rho_corr.
* Q_2 = A C~^-1 A with A = kappa^2 C~ + G (Eq. 4; C~ the lumped mass,
  PAPER.md:97).  Instead of the Cholesky route x = L^-T z (cholmod is not installed)
  we draw x = A^-1 C~^{1/2} z, whose covariance A^-1 C~ A^-1 = Q_2^-1 is the same.
* Samples are rescaled to the target standard deviation using the SPDE marginal
  variance sigma^2 = Gamma(nu) / (Gamma(nu + d/2) (4 pi)^{d/2} kappa^{2 nu})
   = 1 / (4 pi kappa^2) for nu = 1, d = 2.
* E and zeta are independent draws ("two Matérn random fields").
* z comes from a counter-based generator keyed by (seed, field, s): realisation s is
  the same whatever N_s or the ensemble shard (s_begin) is.
* Realisation s = 0 is homogeneous (E = E_bar, zeta = zeta_bar): it carries the
  closed-form pins (Laplace law).
* Values are clipped at 5% of the mean (never triggered at 10% CV; counted).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

FIELD_E = 0
FIELD_H = 1


def p1_matrices(xyz: np.ndarray, tris: np.ndarray):
    """Lumped P1 mass diag C~ (Eq. 6 lumping) and stiffness G (Eq. 5)."""
    X = xyz[tris]                                   # [F][3][3]
    n = np.cross(X[:, 1] - X[:, 0], X[:, 2] - X[:, 0])
    A = 0.5 * np.linalg.norm(n, axis=1)
    V = xyz.shape[0]
    Cl = np.zeros(V)
    np.add.at(Cl, tris.ravel(), np.repeat(A / 3.0, 3))
    # G_ab = e_a . e_b / (4A), e_a = edge opposite local vertex a
    e = np.stack([X[:, 2] - X[:, 1], X[:, 0] - X[:, 2], X[:, 1] - X[:, 0]], axis=1)
    rows, cols, vals = [], [], []
    for a in range(3):
        for b in range(3):
            rows.append(tris[:, a])
            cols.append(tris[:, b])
            vals.append(np.einsum("ij,ij->i", e[:, a], e[:, b]) / (4.0 * A))
    G = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(V, V)).tocsc()
    return Cl, G


def _z(seed: int, field_id: int, s: int, V: int) -> np.ndarray:
    key = (int(seed) & ((1 << 64) - 1)) | (int(field_id) << 64) | (int(s) << 80)
    return np.random.Generator(np.random.Philox(key=key)).standard_normal(V)


GROUP = 4          # realisations solved together: s in [4g, 4g + 4) always as one 4-column solve


class MaternSampler:
    """Factor A = kappa^2 C~ + G once; draw any realisation index on demand.

    Realisations are solved in aligned groups of GROUP columns (the whole group even when
    only part of it is asked for), so the value of realisation s never depends on which
    other realisations are drawn with it (N_s, shard s_begin); the groups run on a thread
    pool (SuperLU's solve releases the GIL)."""

    def __init__(self, xyz: np.ndarray, tris: np.ndarray, rho_corr: float):
        self.V = xyz.shape[0]
        self.kappa = np.sqrt(8.0 * 1.0) / rho_corr
        Cl, G = p1_matrices(xyz, tris)
        self.sqrtC = np.sqrt(Cl)
        A = (self.kappa ** 2) * sp.diags(Cl) + G
        self.lu = spla.splu(A.tocsc())
        self.sigma_spde = np.sqrt(1.0 / (4.0 * np.pi * self.kappa ** 2))

    def standard(self, seed: int, field_id: int, s_list) -> np.ndarray:
        """Unit-variance GMRF draws, one row per realisation index in s_list: [len][V]."""
        s_list = [int(s) for s in s_list]
        groups = sorted({s // GROUP for s in s_list})

        def solve(g):
            Z = np.stack([_z(seed, field_id, s, self.V) * self.sqrtC for s in range(g * GROUP, (g + 1) * GROUP)],
                         axis=1)
            return g, self.lu.solve(Z)

        with ThreadPoolExecutor(max(1, min(len(groups), os.cpu_count() or 1))) as ex:
            sol = dict(ex.map(solve, groups))
        out = np.empty((len(s_list), self.V))
        for k, s in enumerate(s_list):
            out[k] = sol[s // GROUP][:, s % GROUP]
        return out / self.sigma_spde


def standard_normals(seed: int, field_id: int, s_list, V: int) -> np.ndarray:
    """The counter-based z of realisations s_list: [len(s_list)][V]."""
    return np.stack([_z(seed, field_id, s, V) for s in s_list])


def sample_materials(xyz: np.ndarray, tris: np.ndarray, n_s: int, *, E_mean: float,
                     E_std: float, h_mean: float, h_std: float, rho_corr: float,
                     seed: int, s_begin: int = 0, homogeneous_first: bool = True):
    """Return (E[n_s][V], h[n_s][V], n_clipped) for realisations s_begin .. s_begin+n_s-1,
    every realisation an independent GMRF draw."""
    V = xyz.shape[0]
    E = np.empty((n_s, V))
    h = np.empty((n_s, V))
    s_idx = list(range(s_begin, s_begin + n_s))
    rand = [s for s in s_idx if not (homogeneous_first and s == 0)]
    if rand:
        smp = MaternSampler(xyz, tris, rho_corr)
        xe = smp.standard(seed, FIELD_E, rand)
        xh = smp.standard(seed, FIELD_H, rand)
    k = 0
    for row, s in enumerate(s_idx):
        if homogeneous_first and s == 0:
            E[row] = E_mean
            h[row] = h_mean
        else:
            E[row] = E_mean + E_std * xe[k]
            h[row] = h_mean + h_std * xh[k]
            k += 1
    nclip = int((E < 0.05 * E_mean).sum() + (h < 0.05 * h_mean).sum())
    np.maximum(E, 0.05 * E_mean, out=E)
    np.maximum(h, 0.05 * h_mean, out=h)
    return np.ascontiguousarray(E), np.ascontiguousarray(h), nclip
