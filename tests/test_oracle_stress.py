"""Pins of the oracle's stress recovery and ensemble statistics (
PAPER.md:319-320, 449-457) — -m "not gpu"."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle
from paper_2101_09059_b200.inputs import loads, mesh as meshmod


def test_rigid_translation_is_stress_free():
    """Translations are in the kernel of every element (the 3-dof shell has no rotational
    dofs, so only translations and the drilling rotation are stress-free, cf. the
    4-dimensional K^_e nullspace pinned in test_oracle_pins)."""
    m = meshmod.perturb(meshmod.cylinder(12, 9), 0.05, 1)
    V = m.n_nodes
    E = np.full((2, V), 7e6)
    u = np.zeros((2, V, 3))
    u[0] += np.array([0.3, -0.2, 0.1])
    u[1] += np.array([-1.0, 2.0, 0.5])
    for frame in (0, 1):
        s = oracle.stress(m.xyz, m.tris, E, u, 0.3, 5 / 6, frame=frame)
        assert np.abs(s).max() <= 1e-8 * 7e6


@pytest.mark.parametrize("nu", [0.0, 0.3, 0.5])
def test_uniaxial_axial_strain_closed_form(nu):
    """Flat patch in the plane y = 0, centreline along z: r = normal, theta = r x z.
    u_z = delta z (uniform axial strain) => s_zz = E delta / (1 - nu^2),
    s_tt = nu E delta / (1 - nu^2), all other components 0 (Eq. 9 plane stress)."""
    nx, nz = 5, 6
    X, Z = np.meshgrid(np.linspace(0, 2, nx), np.linspace(0, 3, nz), indexing="ij")
    xyz = np.stack([X.ravel(), np.zeros(X.size), Z.ravel()], 1)
    tris = []
    for i in range(nx - 1):
        for k in range(nz - 1):
            a, b, c, d = i * nz + k, (i + 1) * nz + k, (i + 1) * nz + k + 1, i * nz + k + 1
            tris += [[a, b, c], [a, c, d]]
    tris = np.array(tris, np.int32)
    V = len(xyz)
    delta, E = 1e-3, 7e6
    u = np.zeros((1, V, 3))
    u[0, :, 2] = delta * xyz[:, 2]
    s = oracle.stress(xyz, tris, np.full((1, V), E), u, nu, 5 / 6, frame=1)[0]
    pre = E / (1 - nu * nu)
    np.testing.assert_allclose(s[:, 2], pre * delta, rtol=1e-12)
    np.testing.assert_allclose(s[:, 1], nu * pre * delta, rtol=1e-12, atol=1e-9 * pre * delta)
    for comp in (0, 3, 4, 5):
        assert np.abs(s[:, comp]).max() <= 1e-9 * pre * delta


def test_cylinder_hoop_stress_laplace():
    """Homogeneous cylinder, fixed ends, 13 mmHg, static: mid-length hoop stress = p R / zeta
    (Laplace / Barlow) within 1e-3; radial stress 0 (eps_zz = 0 shell);
    shear stresses of the homogeneous model vanish to faceting error."""
    m = meshmod.cylinder(96, 262)
    V = m.n_nodes
    E, h, p = 7e6, 0.4, loads.P_SUPERPOSED
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, np.full((1, V), E), np.full((1, V), h),
                            rho=1.06, nu=0.5, k_shear=5 / 6)
    F = loads.pressure_forces(m.xyz, m.tris, p).ravel()
    free = np.repeat(m.fixed == 0, 3)
    K = om.K_sparse(0).tocsc()[free][:, free]
    u = np.zeros(3 * V)
    u[free] = spla.spsolve(K, F[free])
    s = oracle.stress(m.xyz, m.tris, np.full((1, V), E), u.reshape(1, V, 3), 0.5, 5 / 6, frame=1)[0]
    cz = m.xyz[m.tris].mean(1)[:, 2]
    mid = np.abs(cz - 15.0) < 1.0
    hoop = p * 2.0 / h
    assert s[mid, 1].mean() == pytest.approx(hoop, rel=1e-3)
    assert np.abs(s[mid, 0]).max() <= 1e-12 * hoop
    assert np.abs(s[mid, 3:].mean(0)).max() <= 1e-3 * hoop
    assert np.abs(s[mid, 3:]).max() <= 1e-2 * hoop


def test_ensemble_stats_match_library_percentile():
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 64, 100):
        v = rng.standard_normal((n, 13, 6))
        mean, q05, q95 = oracle.ensemble_stats(v)
        np.testing.assert_allclose(mean, v.mean(0), rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(q05, np.percentile(v, 5, axis=0), rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(q95, np.percentile(v, 95, axis=0), rtol=1e-14, atol=1e-15)


def test_centerline_polyline_tangent():
    """A bent centreline: for elements near the second segment, z follows that segment."""
    m = meshmod.cylinder(16, 10)
    V = m.n_nodes
    u = np.zeros((1, V, 3))
    u[0, :, 2] = 1e-3 * m.xyz[:, 2]                           # axial stretch along global z
    E = np.full((1, V), 7e6)
    straight = oracle.stress(m.xyz, m.tris, E, u, 0.0, 5 / 6, frame=1, centerline=[[0, 0, -1], [0, 0, 40]])
    ref = oracle.stress(m.xyz, m.tris, E, u, 0.0, 5 / 6, frame=1)
    np.testing.assert_allclose(straight, ref, rtol=1e-13, atol=1e-9)
    # centreline along x: the axial stretch now reads as circumferential stress
    sideways = oracle.stress(m.xyz, m.tris, E, u, 0.0, 5 / 6, frame=1, centerline=[[-50, 0, 15], [50, 0, 15]])
    cz = m.xyz[m.tris].mean(1)
    top = np.abs(cz[:, 1]) > 1.9                              # elements facing +-y: x axis is in-plane
    assert np.abs(sideways[0, top, 2]).max() <= 1e-4 * 7e3      # facets are not exactly y-normal
    np.testing.assert_allclose(sideways[0, top, 1], 7e6 * 1e-3, rtol=1e-2)
