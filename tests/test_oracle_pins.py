"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Every pin is something other than the oracle itself: a number printed in the paper
(tests/golden/paper_values.json, cited), a closed form, an exact invariant, a special
case with a textbook solution, or brute force on tiny inputs.
maps each oracle function to the pins below.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from paper_2101_09059_b200.inputs import loads, mesh as meshmod

NU, KS, RHO = 0.5, 5.0 / 6.0, 1.06


def paper_count_mesh():
    """An annulus with exactly the paper's coarse counts V = 2,565, F = 5,074
    (PAPER.md:381): cylinder(28, 91) has V = 2,548, F = 5,040 and 56 boundary nodes
    (F = 2V - b); 17 interior triangles are split at their centroid (+1 node, +2 tris)."""
    m = meshmod.cylinder(28, 91)
    xyz = list(m.xyz)
    tris = [list(t) for t in m.tris]
    for k in range(17):
        t = 200 + 250 * k
        a, b, c = tris[t]
        n = len(xyz)
        xyz.append((m.xyz[a] + m.xyz[b] + m.xyz[c]) / 3.0)
        tris[t] = [a, b, n]
        tris.append([b, c, n])
        tris.append([c, a, n])
    xyz = np.array(xyz)
    return meshmod.Mesh(xyz, np.array(tris, np.int32), np.zeros(len(xyz), np.uint8))


# ---------------------------------------------------------------------------------
# S0: pattern
# ---------------------------------------------------------------------------------

def test_paper_nnz_exact(golden):
    """9 * nnzb equals the paper's printed nnz = 160,587 on a mesh with its counts."""
    m = paper_count_mesh()
    assert m.n_nodes == golden["coarse_mesh"]["n_nodes"]
    assert m.n_tris == golden["coarse_mesh"]["n_tris"]
    assert oracle.validate_mesh(m.xyz, m.tris) == (0, -1)
    row_ptr, col = oracle.csr(m.n_nodes, m.tris)
    assert 9 * len(col) == golden["coarse_mesh_nnz"]["nnz"]


@pytest.mark.parametrize("nc,na", [(3, 2), (12, 23), (17, 9), (96, 30)])
def test_nnz_identity_annulus(nc, na):
    """nnzb = V + 2 #edges = 3V + 2F - 2 chi, chi = 0 for a tube (Euler)."""
    m = meshmod.cylinder(nc, na)
    _, col = oracle.csr(m.n_nodes, m.tris)
    assert len(col) == 3 * m.n_nodes + 2 * m.n_tris


def _dense_pattern(V, tris):
    P = np.eye(V, dtype=bool)
    for t in tris:
        for a in t:
            for b in t:
                P[a, b] = True
    return P


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_csr_bruteforce(seed):
    m = meshmod.shuffle_nodes(meshmod.cylinder(6, 7), seed)
    V = m.n_nodes
    P = _dense_pattern(V, m.tris)
    perm = oracle.rcm(V, m.tris)
    for pp in (None, perm):
        row_ptr, col = oracle.csr(V, m.tris, pp)
        Q = np.zeros((V, V), bool)
        for i in range(V):
            cols = col[row_ptr[i]:row_ptr[i + 1]]
            assert np.all(np.diff(cols) > 0)      # ascending, unique
            Q[i, cols] = True
        ref = P if pp is None else P[np.ix_(pp, pp)]
        assert np.array_equal(Q, ref)
        assert np.array_equal(Q, Q.T)


def _bfs_ecc(adj, r):
    lev = {r: 0}
    q = [r]
    for v in q:
        for w in adj[v]:
            if w not in lev:
                lev[w] = lev[v] + 1
                q.append(w)
    return max(lev.values()), lev


@pytest.mark.parametrize("seed", [0, 5, 11])
def test_rcm_properties(seed):
    """Properties any reverse Cuthill-McKee order has."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(9, 14), 0.05, seed), seed)
    V = m.n_nodes
    perm = oracle.rcm(V, m.tris)
    assert sorted(perm.tolist()) == list(range(V))
    adj = [set() for _ in range(V)]
    for t in m.tris:
        for a in t:
            for b in t:
                if a != b:
                    adj[a].add(int(b))
    deg = np.array([len(a) for a in adj])
    cm = perm[::-1].tolist()           # Cuthill-McKee order
    pos = {v: k for k, v in enumerate(cm)}
    # BFS order: the parent (earliest-placed neighbour) positions never decrease ...
    parents = [min(pos[w] for w in adj[v]) if k > 0 else -1 for k, v in enumerate(cm)]
    assert all(parents[k] <= parents[k + 1] for k in range(1, V - 1))
    assert all(parents[k] < k for k in range(1, V))
    # ... and siblings are placed by (degree, original index) ascending
    for k in range(1, V - 1):
        if parents[k] == parents[k + 1]:
            assert (deg[cm[k]], cm[k]) < (deg[cm[k + 1]], cm[k + 1])
    # start node is pseudo-peripheral: its eccentricity is at least that of the
    # minimum-degree node, and no last-level node of its BFS has a larger one
    e0, lev = _bfs_ecc(adj, cm[0])
    mind = min(range(V), key=lambda i: (deg[i], i))
    assert e0 >= _bfs_ecc(adj, mind)[0]
    last = [v for v, l in lev.items() if l == e0]
    x = min(last, key=lambda i: (deg[i], i))
    assert _bfs_ecc(adj, x)[0] <= e0


def test_rcm_two_components():
    a = meshmod.cylinder(5, 4)
    b = meshmod.cylinder(6, 3)
    tris = np.concatenate([a.tris, b.tris + a.n_nodes])
    V = a.n_nodes + b.n_nodes
    perm = oracle.rcm(V, tris)
    cm = perm[::-1]
    # the component of node 0 is numbered first in CM order (last after reversal)
    assert set(cm[:a.n_nodes].tolist()) == set(range(a.n_nodes))


def _bandwidth(V, tris, perm):
    row_ptr, col = oracle.csr(V, tris, perm)
    rows = np.repeat(np.arange(V), np.diff(row_ptr))
    return int(np.max(np.abs(col - rows)))


@pytest.mark.parametrize("nc,na,bw", [(12, 23, 18), (24, 50, 36), (96, 262, 144), (96, 40, 120)])
def test_rcm_bandwidth_vs_library(nc, na, bw):
    """Bandwidth of our RCM == that of scipy.sparse.csgraph.reverse_cuthill_mckee (an
    independent library implementation) and == 1.5 n_circ on long offset-ring cylinders
    (18 on 12x23, 144 on 96x262)."""
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    m = meshmod.cylinder(nc, na)
    perm = oracle.rcm(m.n_nodes, m.tris)
    rp0, col0 = oracle.csr(m.n_nodes, m.tris)
    A = sp.csr_matrix((np.ones(len(col0)), col0, rp0))
    ref = reverse_cuthill_mckee(A, symmetric_mode=True).astype(np.int32)
    assert _bandwidth(m.n_nodes, m.tris, perm) == _bandwidth(m.n_nodes, m.tris, ref) == bw
    if (nc, na) == (12, 23):          # same start and no degree ties => identical order
        assert np.array_equal(perm, ref)


def test_validate_mesh_errors():
    m = meshmod.cylinder(6, 3)
    t = m.tris.copy(); t[3, 1] = m.n_nodes
    assert oracle.validate_mesh(m.xyz, t) == (1, 3)
    t = m.tris.copy(); t[4, 2] = t[4, 0]
    assert oracle.validate_mesh(m.xyz, t) == (2, 4)
    x = m.xyz.copy(); x[m.tris[5, 2]] = x[m.tris[5, 0]] + 0.5 * (x[m.tris[5, 1]] - x[m.tris[5, 0]])
    assert oracle.validate_mesh(x, m.tris)[0] == 3
    t = np.concatenate([m.tris, m.tris[:1]])
    assert oracle.validate_mesh(m.xyz, t)[0] == 4
    # a node in no triangle (zero lumped mass)
    x = np.concatenate([m.xyz, [[9.0, 9.0, 9.0]]])
    assert oracle.validate_mesh(x, m.tris) == (5, m.n_nodes)


# ---------------------------------------------------------------------------------
# S1: element stiffness (Eq. 7-10)
# ---------------------------------------------------------------------------------

def _rand_tri(rng):
    return rng.uniform(-1.0, 1.0, (3, 3)) * np.array([1.0, 2.0, 0.5])


def _rot(rng):
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    return q * np.sign(np.linalg.det(q))


@pytest.mark.parametrize("seed", range(5))
def test_khat_nullspace_and_symmetry(seed):
    rng = np.random.default_rng(seed)
    X = _rand_tri(rng)
    for nu in (0.0, 0.3, 0.5):
        K, A = oracle.element_khat(X, nu, KS)
        assert np.array_equal(K, K.T)
        w = np.linalg.eigvalsh(K)
        scale = w[-1]
        assert np.sum(np.abs(w) < 1e-12 * scale) == 4       # 3 translations + drilling
        assert np.all(w > -1e-12 * scale)
        n = np.cross(X[1] - X[0], X[2] - X[0])
        assert A == pytest.approx(0.5 * np.linalg.norm(n), rel=1e-14)
        n /= np.linalg.norm(n)
        for tvec in np.eye(3):
            assert np.linalg.norm(K @ np.tile(tvec, 3)) < 1e-12 * scale
        c = X.mean(0)
        rot = np.concatenate([np.cross(n, X[a] - c) for a in range(3)])
        assert np.linalg.norm(K @ rot) < 1e-12 * scale * np.linalg.norm(rot)


@pytest.mark.parametrize("seed", range(5))
def test_khat_frame_independence(seed):
    """Choosing another edge for e1 (cyclic renumbering) or rigidly rotating the
    element changes K^ only by the corresponding permutation / rotation."""
    rng = np.random.default_rng(100 + seed)
    X = _rand_tri(rng)
    K, _ = oracle.element_khat(X, 0.3, KS)
    Kc, _ = oracle.element_khat(X[[1, 2, 0]], 0.3, KS)
    p = np.r_[3:6, 6:9, 0:3]          # original dofs of the cycled element's nodes 0,1,2
    Kback = np.empty_like(K)
    Kback[np.ix_(p, p)] = Kc
    assert np.max(np.abs(Kback - K)) <= 4e-15 * np.max(np.abs(K))
    Q = _rot(rng)
    Kr, _ = oracle.element_khat(X @ Q.T, 0.3, KS)
    T = np.kron(np.eye(3), Q)
    assert np.max(np.abs(T.T @ Kr @ T - K)) <= 4e-15 * np.max(np.abs(K))


def _energy_density(eps, nu, k):
    """Plane-stress + transverse-shear strain energy per unit area and unit E*zeta,
    written out from the constitutive law:
    W = 1/(2(1-nu^2)) [exx^2 + eyy^2 + 2 nu exx eyy + (1-nu)/2 gxy^2 + k(1-nu)/2 (gxz^2 + gyz^2)]."""
    exx, eyy, gxy, gxz, gyz = eps
    return (exx ** 2 + eyy ** 2 + 2 * nu * exx * eyy + 0.5 * (1 - nu) * gxy ** 2
            + 0.5 * k * (1 - nu) * (gxz ** 2 + gyz ** 2)) / (2 * (1 - nu * nu))


@pytest.mark.parametrize("seed", range(4))
def test_khat_constant_strain_energy(seed):
    """Patch test: a linear displacement field u = G x in the element plane gives a
    constant strain; 1/2 u^T K^ u must equal A * W(strain) exactly (up to rounding)."""
    rng = np.random.default_rng(200 + seed)
    X = _rand_tri(rng)
    e1 = (X[1] - X[0]) / np.linalg.norm(X[1] - X[0])
    n = np.cross(X[1] - X[0], X[2] - X[0]); e3 = n / np.linalg.norm(n)
    e2 = np.cross(e3, e1)
    A = 0.5 * np.linalg.norm(n)
    G = rng.standard_normal((3, 2))   # (u_x, u_y, u_z)_local = G (x, y)_local
    u = []
    for a in range(3):
        xy = np.array([(X[a] - X[0]) @ e1, (X[a] - X[0]) @ e2])
        ul = G @ xy
        u.append(ul[0] * e1 + ul[1] * e2 + ul[2] * e3)
    u = np.concatenate(u)
    eps = (G[0, 0], G[1, 1], G[0, 1] + G[1, 0], G[2, 0], G[2, 1])
    for nu in (0.0, 0.3, 0.5):
        for k in (1.0, KS):
            K, _ = oracle.element_khat(X, nu, k)
            assert 0.5 * u @ K @ u == pytest.approx(A * _energy_density(eps, nu, k), rel=1e-12)


# ---------------------------------------------------------------------------------
# S1: Gauss-point material scaling, mass, CFL
# ---------------------------------------------------------------------------------

def test_alpha_closed_form_and_rule_independence():
    """alpha = (1/12)[(sum E)(sum zeta) + sum E zeta] (degree-2 exactness of the
    3-point rule on a product of two linear fields) = the mid-edge rule value."""
    rng = np.random.default_rng(7)
    m = meshmod.cylinder(7, 5)
    V = m.n_nodes
    E = rng.uniform(5e6, 9e6, (3, V))
    h = rng.uniform(0.3, 0.5, (3, V))
    al = oracle.alpha(V, m.tris, E, h)
    Et, ht = E[:, m.tris], h[:, m.tris]                       # [s][F][3]
    closed = (Et.sum(-1) * ht.sum(-1) + (Et * ht).sum(-1)) / 12.0
    np.testing.assert_allclose(al, closed, rtol=1e-14)
    mid = np.zeros_like(closed)
    for a, b in ((0, 1), (1, 2), (2, 0)):
        mid += (Et[..., a] + Et[..., b]) * (ht[..., a] + ht[..., b]) / 4.0 / 3.0
    np.testing.assert_allclose(al, mid, rtol=1e-14)
    # constant fields: alpha = E zeta exactly
    al1 = oracle.alpha(V, m.tris, np.full((1, V), 7e6), np.full((1, V), 0.4))
    np.testing.assert_allclose(al1, 7e6 * 0.4, rtol=1e-15)


def test_mass_totals():
    m = meshmod.cylinder(96, 31)
    h = np.full((1, m.n_nodes), 0.4)
    mm = oracle.mass(m.xyz, m.tris, h, RHO)
    _, area = oracle.all_khat(m.xyz, m.tris, NU, KS)
    assert mm.sum() == pytest.approx(RHO * 0.4 * area.sum(), rel=1e-13)
    # lateral surface of the cylinder: rho pi D L zeta (polygonal deficit (pi/n)^2/6)
    assert mm.sum() == pytest.approx(RHO * math.pi * 4.0 * 30.0 * 0.4, rel=2e-4)
    rng = np.random.default_rng(3)
    hr = rng.uniform(0.3, 0.5, (2, m.n_nodes))
    mr = oracle.mass(m.xyz, m.tris, hr, RHO)
    hbar = hr[:, m.tris].mean(-1)
    np.testing.assert_allclose(mr.sum(1), RHO * (area * hbar).sum(1), rtol=1e-13)
    assert np.all(mr > 0)


def test_cfl_paper_example(golden):
    """l = 1e-3 m, E = 0.7 MPa, rho = 1.06 kg/m^3 -> 0.9 * 1.2e-6 s.
    Equilateral triangle whose inscribed-circle diameter is l (side l*sqrt(3))."""
    g = golden["cfl_example"]
    l_cm = g["l_e_min_m"] * 100.0
    E = g["E_MPa"] * 1e7                    # Ba
    rho = g["rho_kg_m3"] * 1e-3             # g/cm^3 (literal value)
    s = l_cm * math.sqrt(3.0)
    xyz = np.array([[0, 0, 0], [s, 0, 0], [s / 2, s * math.sqrt(3) / 2, 0]], float)
    tris = np.array([[0, 1, 2]], np.int32)
    dt = oracle.cfl(xyz, tris, np.full((1, 3), E), rho, g["safety"])
    assert round(dt / g["safety"], 7) == g["dt_unscaled_s"]
    # E x 4 => dt / 2 exactly (c = sqrt(E/rho))
    assert oracle.cfl(xyz, tris, np.full((1, 3), 4 * E), rho, 0.9) == pytest.approx(dt / 2, rel=1e-15)


# ---------------------------------------------------------------------------------
# S2: loads
# ---------------------------------------------------------------------------------

def test_load_coeffs_ramp_and_table():
    tab_t = np.array([0.0, 0.1, 0.4])
    tab_g = np.array([[0.0, 1.0, 4.0], [2.0, 2.0, 2.0]])
    f = lambda t: oracle.load_coeffs(t, 2, tab_t, tab_g, 0.4, 0.2)
    np.testing.assert_array_equal(f(0.0), [0.0, 0.0])                     # sin(0) = 0
    assert f(0.05)[0] == pytest.approx(math.sin(math.pi * 0.05 / 0.4) * 0.5, rel=1e-15)
    assert f(0.2)[1] == 2.0                                                # ramp finished
    assert f(0.25)[0] == pytest.approx(2.5, rel=1e-14)                     # between stamps
    assert f(0.4 + 0.25)[0] == pytest.approx(2.5, rel=1e-12)               # periodic wrap
    np.testing.assert_array_equal(oracle.load_coeffs(3.0, 1, [], np.zeros((1, 0)), 0.0, 0.0), [1.0])


def test_pressure_forces_closed_surface():
    """Zero net force on a closed surface (octahedron); |F_i| = p * (A_i tributary) on a
    flat patch.  (Loads are inputs — this pins the fixture used by both sides.)"""
    xyz = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], float)
    tris = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4],
                     [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]], np.int32)
    F = loads.pressure_forces(xyz, tris, 17331.86)
    assert np.linalg.norm(F.sum(0)) < 1e-10 * 17331.86
    assert np.all(np.einsum("ij,ij->i", F, xyz) > 0)       # outward


# ---------------------------------------------------------------------------------
# S3/S4: assembly, SpMM, central-difference dynamics
# ---------------------------------------------------------------------------------

def _model(m, n_s=2, seed=0, nu=NU, damping=0, c_d=0.0, dt=None, homog=False):
    rng = np.random.default_rng(seed)
    V = m.n_nodes
    if homog:
        E = np.full((n_s, V), 7e6); h = np.full((n_s, V), 0.4)
    else:
        E = rng.uniform(6e6, 8e6, (n_s, V)); h = rng.uniform(0.35, 0.45, (n_s, V))
    return oracle.OracleModel(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=nu, k_shear=KS,
                              damping=damping, c_d=c_d, dt=dt)


def test_assembly_dense_bruteforce():
    m = meshmod.perturb(meshmod.cylinder(6, 6), 0.1, 4)
    om = _model(m, n_s=2)
    V = m.n_nodes
    for s in range(2):
        Kd = np.zeros((3 * V, 3 * V))
        for e, t in enumerate(m.tris):
            dofs = np.concatenate([[3 * a, 3 * a + 1, 3 * a + 2] for a in t])
            Kd[np.ix_(dofs, dofs)] += om.alpha[s, e] * om.Khat[e]
        Ks = om.K_sparse(s).toarray()
        assert np.max(np.abs(Ks - Kd)) <= 1e-15 * np.max(np.abs(Kd)) * 8
        assert np.array_equal(Ks, Ks.T)
        for tv in np.eye(3):
            assert np.linalg.norm(Ks @ np.tile(tv, V)) <= 1e-12 * np.abs(Ks).max()


def test_spmm_against_dense_and_ensemble_independence():
    m = meshmod.perturb(meshmod.cylinder(8, 7), 0.05, 9)
    om = _model(m, n_s=3)
    rng = np.random.default_rng(1)
    u = rng.uniform(-1, 1, (3, m.n_nodes, 3))
    y = om.spmm(u)
    for s in range(3):
        ref = om.K_sparse(s).toarray() @ u[s].ravel()
        np.testing.assert_allclose(y[s].ravel(), ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    # perturb realisation 1's values: others bit-unchanged
    K2 = om.Kval.copy(); K2[1] *= 1.5
    y2 = oracle.spmm(om.row_ptr, om.col, K2, u)
    assert np.array_equal(y2[0], y[0]) and np.array_equal(y2[2], y[2])
    assert not np.array_equal(y2[1], y[1])


def _sdof(m, k, f, dt, n):
    row_ptr = np.array([0, 1]); col = np.array([0], np.int32)
    Kval = np.diag([k, k, k]).reshape(1, 1, 9).astype(float)
    c1, c2, c3 = oracle.coeffs(np.array([[m]]), dt, 0, 0.0)
    un = np.zeros((1, 1, 3)); unm1 = np.zeros((1, 1, 3))
    F = np.array([[[f, 0.0, -f]]])
    out = []
    for _ in range(n):
        oracle.run_raw(row_ptr, col, Kval, c1, c2, c3, None, un, unm1, dt=dt, nsteps=1, F=F)
        out.append(un[0, 0, 0])
        assert un[0, 0, 2] == -un[0, 0, 0]
    return np.array(out)


def test_sdof_closed_form_recurrence():
    """u_n = (f/k)[1 - cos n th + tan(th/2) sin n th], cos th = 1 - w^2 dt^2 / 2 — the
    exact solution of Eq. 22's recurrence for one DOF from rest; u_1 = f dt^2 / m."""
    m, k, f = 2.0, 50.0, 3.0
    w = math.sqrt(k / m)
    dt = 0.9 * 2.0 / w
    n = 10_000
    u = _sdof(m, k, f, dt, n)
    # reference in extended precision with the fp64 coefficient the recurrence uses
    # (c1 = dt^2/m rounded): u_{n+1} - (2 - c1 k) u_n + u_{n-1} = c1 f
    L = np.longdouble
    c1 = oracle.coeffs(np.array([[m]]), dt, 0, 0.0)[0][0, 0]
    assert c1 == pytest.approx(dt * dt / m, rel=1e-16)
    th = np.arccos(1 - L(c1) * L(k) / 2)
    idx = np.arange(1, n + 1).astype(L)
    ref = (L(f) / L(k)) * (1 - np.cos(idx * th) + np.tan(th / 2) * np.sin(idx * th))
    assert u[0] == pytest.approx(f * dt * dt / m, rel=1e-15)
    err = np.max(np.abs(u.astype(L) - ref)) / np.max(np.abs(ref))
    assert err <= 2e-13, float(err)


def test_sdof_damped_mode1():
    """Mode-1 damping (C = c_d M): steady state f/k and the discrete decay rate."""
    row_ptr = np.array([0, 1]); col = np.array([0], np.int32)
    k, m, f, cd = 40.0, 1.0, 1.0, 3.0
    Kval = np.diag([k] * 3).reshape(1, 1, 9)
    dt = 0.01
    c1, c2, c3 = oracle.coeffs(np.array([[m]]), dt, 1, cd)
    D = m * (1 + dt * cd / 2)
    assert c1[0, 0] == pytest.approx(dt * dt / D, rel=1e-15)
    un = np.zeros((1, 1, 3)); unm1 = np.zeros((1, 1, 3))
    oracle.run_raw(row_ptr, col, Kval, c1, c2, c3, None, un, unm1, dt=dt, nsteps=5000,
                   F=np.full((1, 1, 3), f))
    assert un[0, 0, 0] == pytest.approx(f / k, rel=1e-12)


def _damped_sdof_closed_form(m, k, f, c, dt, n):
    """Exact solution of the damped central-difference recurrence of Eq. 22
    for one DOF from rest (u_{-1} = u_0 = 0), in extended precision and from the physical
    parameters only: D u_{n+1} = dt^2 f - (dt^2 k - 2m) u_n - (m - dt c/2) u_{n-1},
    D = m + dt c/2.  Characteristic roots of D l^2 - (2m - dt^2 k) l + (m - dt c/2) = 0 are
    r e^{+-i th} (underdamped), so u_n = u* + r^n (C1 cos n th + C2 sin n th) with
    u* = f/k, C1 = -u*, C2 = u* (r - cos th) / sin th."""
    L = np.longdouble
    m, k, f, c, dt = L(m), L(k), L(f), L(c), L(dt)
    D = m + dt * c / 2
    q = m - dt * c / 2
    b = 2 * m - dt * dt * k
    assert b * b < 4 * D * q, "underdamped case only"
    r = np.sqrt(q / D)
    th = np.arccos(b / (2 * D * r))
    us = f / k
    C1, C2 = -us, us * (r - np.cos(th)) / np.sin(th)
    idx = np.arange(1, n + 1).astype(L)
    return us + r ** idx * (C1 * np.cos(idx * th) + C2 * np.sin(idx * th))


@pytest.mark.parametrize("m", [0.5, 3.0])
def test_sdof_damped_modes_trajectory(m):
    """orc_coeffs' damping forms (DESIGN.md §2 #4): mode 1 C~ = c_d M~
    (c = c_d m), mode 2 C~ = c_d I (c = c_d, the literal f_v = -c_d u').
    The whole 10^4-step oracle trajectory of a damped SDOF with m != 1 (where the two modes
    differ) must match the closed form of the damped recurrence in extended precision; a
    swapped mode, a mis-scaled c or a wrong sign in c2/c3 fails it."""
    k, f, cd = 40.0, 1.0, 0.8
    dt = 0.5 * 2.0 / math.sqrt(k / m)
    n = 10_000
    row_ptr = np.array([0, 1]); col = np.array([0], np.int32)
    Kval = np.diag([k] * 3).reshape(1, 1, 9)
    traj = {}
    for mode, c in ((1, cd * m), (2, cd)):
        c1, c2, c3 = oracle.coeffs(np.array([[m]]), dt, mode, cd)
        un = np.zeros((1, 1, 3)); unm1 = np.zeros((1, 1, 3))
        out = np.empty(n)
        for t in range(n):
            oracle.run_raw(row_ptr, col, Kval, c1, c2, c3, None, un, unm1, dt=dt, nsteps=1,
                           step0=t, F=np.full((1, 1, 3), f))
            out[t] = un[0, 0, 0]
        ref = _damped_sdof_closed_form(m, k, f, c, dt, n)
        err = np.max(np.abs(out.astype(np.longdouble) - ref)) / np.max(np.abs(ref))
        assert err <= 1e-12, (mode, float(err))
        # the decay: the transient shrinks by r^n; after 10^4 steps only f/k is left
        assert out[-1] == pytest.approx(f / k, rel=1e-9)
        traj[mode] = out
    # the two forms differ when m != 1 (they coincide at m = 1, the old pin's case)
    assert np.max(np.abs(traj[1][:200] - traj[2][:200])) > 1e-3 * f / k


def _crit_dt(om, s):
    free = np.repeat(om.fixed == 0, 3)
    K = om.K_sparse(s).toarray()[np.ix_(free, free)]
    mi = np.repeat(om.m[s], 3)[free]
    Ms = 1.0 / np.sqrt(mi)
    lam = sla.eigvalsh(Ms[:, None] * K * Ms[None, :])
    return 2.0 / math.sqrt(lam[-1]), math.sqrt(max(lam[lam > 1e-6 * lam[-1]][0], 0))


def _energy(om, s, u1, u0, f):
    """Shadow energy of central differences: H = 1/2 v M v + 1/2 u1 K u0 - 1/2 f (u1+u0)."""
    K = om.K_sparse(s)
    v = (u1 - u0) / om.dt
    mm = np.repeat(om.m[s], 3)
    return 0.5 * v @ (mm * v) + 0.5 * u1 @ (K @ u0) - 0.5 * f @ (u1 + u0), 0.5 * v @ (mm * v)


def test_shadow_energy_and_stability_dichotomy():
    """c_d = 0, constant load: H_{n+1/2} is exactly conserved at 0.9 dt_crit over 10^4
    steps; at 1.05 dt_crit the solution grows by > 1e6 within 500 steps."""
    m = meshmod.cylinder(12, 23)
    om0 = _model(m, n_s=1, seed=3)
    dtc, _ = _crit_dt(om0, 0)
    tr = loads.steady(m.xyz, m.tris)
    om = _model(m, n_s=1, seed=3, dt=0.9 * dtc)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
    f = tr.F[0].ravel() * np.repeat(om.fixed == 0, 3)
    Hs, KEmax = [], 0.0
    prev = om.u_n[0].ravel().copy()
    for n in range(10_000):
        om.run(1)
        cur = om.u_n[0].ravel().copy()
        if n % 50 == 0 or n > 9990:
            H, KE = _energy(om, 0, cur, prev, f)
            Hs.append(H)
            KEmax = max(KEmax, KE)
        prev = cur
    Hs = np.array(Hs)
    assert np.max(np.abs(Hs - Hs[0])) <= 1e-10 * KEmax
    om2 = _model(m, n_s=1, seed=3, dt=1.05 * dtc)
    om2.set_traction(tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
    om2.run(1)
    a0 = np.abs(om2.u_n).max()
    om2.run(499)
    assert np.abs(om2.u_n).max() > 1e6 * a0


def test_cfl_estimate_is_conservative():
    """The paper's CFL estimate is below the exact dt_crit on the c1 mesh."""
    m = meshmod.cylinder(12, 23)
    om = _model(m, n_s=1, homog=True)
    dtc, wmin = _crit_dt(om, 0)
    assert om.dt_cfl < dtc
    # unscaled estimate l/c over the exact threshold: 0.831 on 12x23
    assert om.dt_cfl / 0.9 / dtc == pytest.approx(0.831, abs=0.002)
    assert dtc == pytest.approx(3.35e-4, rel=2e-3)


def test_ensemble_equivalence_bitexact():
    """Running N_s realisations together == each alone — bit for bit."""
    m = meshmod.cylinder(12, 23)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    rng = np.random.default_rng(5)
    V = m.n_nodes
    E = rng.uniform(6e6, 8e6, (4, V)); h = rng.uniform(0.35, 0.45, (4, V))
    kw = dict(rho=RHO, nu=NU, k_shear=KS, damping=2, c_d=0.5, dt=2e-4)
    allm = oracle.OracleModel(m.xyz, m.tris, m.fixed, E, h, **kw)
    allm.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    allm.run(300)
    for s in range(4):
        one = oracle.OracleModel(m.xyz, m.tris, m.fixed, E[s:s + 1], h[s:s + 1], **kw)
        one.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        one.run(300)
        assert np.array_equal(one.u_n[0], allm.u_n[s])
        assert np.array_equal(one.u_nm1[0], allm.u_nm1[s])


def test_dirichlet_and_zero_load():
    m = meshmod.cylinder(12, 23)
    om = _model(m, n_s=2, dt=1e-4)
    om.run(50)
    assert not om.u_n.any()                      # zero load, rest => zero trajectory
    tr = loads.steady(m.xyz, m.tris)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
    om.run(100)
    fixed = om.fixed == 7
    assert not om.u_n[:, fixed].any() and not om.u_nm1[:, fixed].any()
    assert om.u_n[:, ~fixed].any()


def test_free_particle_kick():
    """K = 0, c_d = 0, constant f, from rest: u_1 = dt^2 f / m exactly."""
    V = 4
    row_ptr = np.arange(V + 1); col = np.arange(V, dtype=np.int32)
    Kval = np.zeros((1, V, 9))
    mm = np.array([[1.0, 2.0, 3.0, 4.0]])
    dt = 1e-3
    c1, c2, c3 = oracle.coeffs(mm, dt, 0, 0.0)
    F = np.arange(12, dtype=float).reshape(1, V, 3)
    un = np.zeros((1, V, 3)); unm1 = np.zeros((1, V, 3))
    oracle.run_raw(row_ptr, col, Kval, c1, c2, c3, None, un, unm1, dt=dt, nsteps=1, F=F)
    np.testing.assert_allclose(un[0], dt * dt * F[0] / mm[0][:, None], rtol=1e-15)


def test_damped_run_reaches_static_solution():
    """Mode-1 damping c_d ~ 2 w_min: the explicit run converges to K_ff u = f_f."""
    m = meshmod.cylinder(12, 23)
    om0 = _model(m, n_s=1, seed=8)
    dtc, wmin = _crit_dt(om0, 0)
    om = _model(m, n_s=1, seed=8, dt=0.9 * dtc, damping=1, c_d=2 * wmin)
    tr = loads.steady(m.xyz, m.tris)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
    om.run(10_000)
    free = np.repeat(om.fixed == 0, 3)
    K = om.K_sparse(0).tocsc()[free][:, free]
    us = spla.spsolve(K, tr.F[0].ravel()[free])
    got = om.u_n[0].ravel()[free]
    assert np.linalg.norm(got - us) <= 1e-8 * np.linalg.norm(us)


@pytest.mark.parametrize("nu", [0.0, 0.5])
def test_laplace_law_static(nu):
    """Homogeneous cylinder, fixed ends, uniform 13 mmHg: mid-length radial displacement
    u_r = (1-nu^2) p R^2 / (E zeta) / (1 - 2 nu^2 l / L), l = R sqrt(k / (2(1+nu)))
    (thin-cylinder Laplace law with the fixed-end correction; PAPER.md:450 'consistent
    with an homogeneous solution'); <= 1e-3 relative on the 96 x 262 mesh (c2)."""
    m = meshmod.cylinder(96, 262)
    V = m.n_nodes
    E, h = 7e6, 0.4
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, np.full((1, V), E), np.full((1, V), h),
                            rho=RHO, nu=nu, k_shear=KS)
    p = loads.P_SUPERPOSED
    F = loads.pressure_forces(m.xyz, m.tris, p).ravel()
    free = np.repeat(m.fixed == 0, 3)
    K = om.K_sparse(0).tocsc()[free][:, free]
    u = np.zeros(3 * V)
    u[free] = spla.spsolve(K, F[free])
    u = u.reshape(V, 3)
    ring = 131
    nodes = np.arange(ring * 96, (ring + 1) * 96)
    rhat = m.xyz[nodes, :2] / np.linalg.norm(m.xyz[nodes, :2], axis=1, keepdims=True)
    ur = np.mean(np.einsum("ij,ij->i", u[nodes, :2], rhat))
    R, L = 2.0, 30.0
    ell = R * math.sqrt(KS / (2 * (1 + nu)))
    ref = (1 - nu * nu) * p * R * R / (E * h) / (1 - 2 * nu * nu * ell / L)
    assert ur == pytest.approx(ref, rel=1e-3)


# ---------------------------------------------------------------------------------
# S5: partition and halo maps (integer) — brute force
# ---------------------------------------------------------------------------------

@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_maps_bruteforce(P):
    m = meshmod.shuffle_nodes(meshmod.cylinder(10, 13), 3)
    V = m.n_nodes
    perm = oracle.rcm(V, m.tris)
    row_ptr, col = oracle.csr(V, m.tris, perm)
    b, gh, send = oracle.halo_maps(row_ptr, col, P)
    nnzb = int(row_ptr[-1])
    assert b[0] == 0 and b[-1] == V and np.all(np.diff(b) >= 0)
    for p in range(1, P):
        ok = [r for r in range(V + 1) if P * row_ptr[r] >= p * nnzb]
        assert b[p] == ok[0]
    P_dense = _dense_pattern(V, m.tris)[np.ix_(perm, perm)]
    for p in range(P):
        lo, hi = b[p], b[p + 1]
        mine = np.zeros(V, bool); mine[lo:hi] = True
        expect = np.where(P_dense[mine].any(0) & ~mine)[0]
        assert np.array_equal(gh[p], expect)
        for q in range(P):
            if q != p:
                assert np.array_equal(send[p][q], np.intersect1d(gh[q], np.arange(lo, hi)))
