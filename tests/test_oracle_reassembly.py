"""Pins of the oracle's selective re-assembly on the updated geometry (SURVEY.md §8(f) N4,
PAPER.md:345) — -m "not gpu"."""
import numpy as np
import pytest

import oracle
from paper_2101_09059_b200.inputs import loads, mesh as meshmod

RHO, NU, KS = 1.06, 0.5, 5.0 / 6.0


def _model(m, n_s=2, seed=0, dt=1e-4):
    rng = np.random.default_rng(seed)
    E = rng.uniform(6e6, 8e6, (n_s, m.n_nodes))
    h = rng.uniform(0.35, 0.45, (n_s, m.n_nodes))
    return oracle.OracleModel(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, dt=dt)


def test_reassembly_at_rest_reproduces_k():
    m = meshmod.perturb(meshmod.cylinder(12, 9), 0.05, 2)
    om = _model(m)
    K0 = om.Kval.copy()
    om.reassemble()
    assert np.max(np.abs(om.Kval - K0)) <= 1e-15 * np.abs(K0).max() * 4


def test_reassembly_invariant_under_rigid_translation():
    """K^_e is translation invariant (it depends on edge vectors only): a rigid shift of
    every realisation's geometry leaves the re-assembled values unchanged to rounding."""
    m = meshmod.perturb(meshmod.cylinder(12, 9), 0.05, 3)
    om = _model(m)
    K0 = om.Kval.copy()
    om.u_n[:] = np.array([0.7, -0.4, 1.3])
    om.reassemble()
    assert np.max(np.abs(om.Kval - K0)) <= 1e-12 * np.abs(K0).max()


def test_reassembly_rigid_rotation_rotates_k():
    """A rigid rotation Q of realisation 1's geometry gives K = (I x Q) K0 (I x Q)^T."""
    m = meshmod.perturb(meshmod.cylinder(10, 7), 0.05, 4)
    om = _model(m)
    th = 0.3
    Q = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1.0]])
    om.u_n[1] = m.xyz @ Q.T - m.xyz
    K0 = om.K_sparse(1).toarray()
    om.reassemble()
    K1 = om.K_sparse(1).toarray()
    T = np.kron(np.eye(m.n_nodes), Q)
    assert np.max(np.abs(K1 - T @ K0 @ T.T)) <= 1e-12 * np.abs(K0).max()


def test_reassembly_small_strain_limit():
    """At small load the geometrically updated run approaches the linear one: the
    difference scales with the load squared (second order in u / L)."""
    m = meshmod.cylinder(12, 23)
    tr = loads.steady(m.xyz, m.tris, p=1.0)
    diffs = []
    for scale in (1e3, 1e4):
        runs = []
        for k in (0, 10):
            om = _model(m, n_s=1, seed=5, dt=2e-4)
            om.set_traction(scale * tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
            om.run(300, reassemble_every=k)
            runs.append(om.u_n[0].copy())
        diffs.append(np.linalg.norm(runs[1] - runs[0]) / np.linalg.norm(runs[0]))
    assert diffs[0] > 0 and diffs[1] / diffs[0] == pytest.approx(10.0, rel=0.1)
