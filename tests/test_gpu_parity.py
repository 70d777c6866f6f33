"""Parity of the CUDA path (through the C ABI) with the CPU oracle, on a B200 (-m gpu).

Tolerances (north star): one SpMM <= 1e-12 relative L2 and
|dy| <= 4 nnz_row eps (|K||u|) per entry; displacement after 10^4 steps <= 1e-9
relative L2; ensemble equivalence, Dirichlet zeros, state round trips: bit-exact.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200._ffi import ENS_E_DIVERGED, ENS_E_STATE, EnsError
from paper_2101_09059_b200.inputs import configs, fields, loads, mesh as meshmod

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps
RHO, NU, KS = 1.06, 0.5, 5.0 / 6.0


def _mats(m, n_s, seed, s_begin=0):
    E, h, _ = fields.sample_materials(m.xyz, m.tris, n_s, E_mean=7e6, E_std=7e5, h_mean=0.4,
                                      h_std=0.04, rho_corr=3.7, seed=seed, s_begin=s_begin)
    return E, h


def _pair(m, E, h, kernel="assembled", **kw):
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, kernel=kernel, **kw)
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS,
                            damping=solver.DAMPING[kw.get("damping", 0)], c_d=kw.get("c_d", 0.0),
                            dt=ens.info()["dt"])
    return ens, om


def _check_spmm(ens, om, u):
    y = ens.apply_stiffness(u)
    yo = om.spmm(u)
    assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)
    # per entry: 4 * nnz_row * eps * (|K| |u|)_i
    absKu = oracle.spmm(om.row_ptr, om.col, np.abs(om.Kval), np.abs(u))
    nnz_row = np.diff(om.row_ptr).max() * 3
    assert np.all(np.abs(y - yo) <= 4 * nnz_row * EPS * absKu + 1e-300)


@pytest.mark.parametrize("kernel", ["assembled", "assembled_sym", "matrix_free"])
@pytest.mark.parametrize("n_s", [1, 3, 4, 6, 64, 128])
def test_spmm_parity(kernel, n_s):
    """Several tiles and a ragged tail: 40 x 51 rings, V = 2,040, N_s odd/even/x4."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(40, 51), 0.02, 1), 1)
    E, h = _mats(m, n_s, 11)
    ens, om = _pair(m, E, h, kernel=kernel)
    rng = np.random.default_rng(n_s)
    _check_spmm(ens, om, rng.uniform(-1, 1, (n_s, m.n_nodes, 3)))
    ens.close()


def _crit_dt(om):
    """Exact stability threshold 2 / sqrt(lambda_max(M^-1/2 K_ff M^-1/2)), min over s."""
    free = np.repeat(om.fixed == 0, 3)
    best = np.inf
    for s in range(om.n_s):
        K = om.K_sparse(s).toarray()[np.ix_(free, free)]
        d = 1.0 / np.sqrt(np.repeat(om.m[s], 3)[free])
        lam = sla.eigvalsh(d[:, None] * K * d[None, :], subset_by_index=[K.shape[0] - 1, K.shape[0] - 1])
        best = min(best, 2.0 / math.sqrt(lam[-1]))
    return best


def test_c1_1e4_steps_parity():
    """Config c1 (12 x 23 rings, N_s = 4, steady 13 mmHg, undamped), 10^4 steps at
    0.9 dt_crit: relative L2 <= 1e-9 at step 10^4."""
    cfg = configs.make("c1")
    m = cfg.mesh
    om0 = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=RHO, nu=NU, k_shear=KS)
    dt = 0.9 * _crit_dt(om0)
    ens, om = _pair(m, cfg.E, cfg.h, dt=dt)
    tr = cfg.traction
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    for chunk in (1, 99, 900, 9000):
        ens.step(chunk)
        om.run(chunk)
        u, up, t, step = ens.get_state()
        assert step == om.step
        for a, b in ((u, om.u_n), (up, om.u_nm1)):
            assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b)
    assert t == pytest.approx(1e4 * dt, rel=1e-15)
    ens.close()


@pytest.mark.parametrize("damping,c_d", [("mass", 250.0), ("identity", 0.5)])
def test_pulsatile_damped_parity(damping, c_d):
    """Pulsatile table + sine ramp + period wrap + both damping forms, 3,000 steps."""
    m = meshmod.cylinder(16, 31)
    E, h = _mats(m, 6, 21)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.05, systole=0.02, n_tab=51, ramp_T=0.03)
    ens, om = _pair(m, E, h, damping=damping, c_d=c_d)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(3000)
    om.run(3000)
    u, up, _, _ = ens.get_state()
    assert np.linalg.norm(u - om.u_n) <= 1e-9 * np.linalg.norm(om.u_n)
    ens.close()


@pytest.mark.parametrize("kernel", ["assembled", "assembled_sym", "matrix_free"])
def test_ensemble_equivalence_bitexact(kernel):
    """N_s = 8 together (VEC = 2 lanes) == each realisation alone (VEC = 1): bit for bit."""
    m = meshmod.cylinder(24, 40)
    E, h = _mats(m, 8, 31)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel=kernel, dt=5e-5, damping="identity", c_d=0.3)
    allr = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    allr.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    allr.step(500)
    u_all, up_all, _, _ = allr.get_state()
    for s in (0, 3, 7):
        one = solver.Ensemble(m.xyz, m.tris, m.fixed, E[s:s + 1], h[s:s + 1], **kw)
        one.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        one.step(500)
        u1, up1, _, _ = one.get_state()
        assert np.array_equal(u1[0], u_all[s]) and np.array_equal(up1[0], up_all[s])
        one.close()
    # and an N_s = 128 run (two warps per row) whose first 8 realisations are the same fields
    E2 = np.concatenate([E] * 16)
    h2 = np.concatenate([h] * 16)
    big = solver.Ensemble(m.xyz, m.tris, m.fixed, E2, h2, **kw)
    big.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    big.step(500)
    ub, _, _, _ = big.get_state(want_prev=False)
    for r in range(16):
        assert np.array_equal(ub[8 * r:8 * r + 8], u_all)
    big.close()
    allr.close()


def test_dirichlet_zero_load_and_state_roundtrip():
    m = meshmod.cylinder(16, 21)
    E, h = _mats(m, 4, 41)
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS)
    ens.step(100)
    u, up, _, _ = ens.get_state()
    assert not u.any() and not up.any()            # zero load from rest => zero
    tr = loads.steady(m.xyz, m.tris)
    ens.set_traction(tr.F)
    ens.step(137)
    u, up, _, step = ens.get_state()
    fixed = m.fixed == 7
    assert not u[:, fixed].any() and not up[:, fixed].any() and u[:, ~fixed].any()
    ens.step(50)
    ref, _, _, _ = ens.get_state()
    # resume from the checkpoint in a fresh context: bit-identical continuation
    ens2 = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS)
    ens2.set_traction(tr.F)
    ens2.set_state(u, up, step)
    ens2.step(50)
    got, _, _, step2 = ens2.get_state()
    assert step2 == step + 50 and np.array_equal(got, ref)
    ens.close(); ens2.close()


def test_divergence_detected_and_latched():
    m = meshmod.cylinder(12, 23)
    E, h = _mats(m, 2, 51)
    om0 = oracle.OracleModel(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS)
    dt = 3.0 * _crit_dt(om0)
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, dt=dt)
    ens.set_traction(loads.steady(m.xyz, m.tris).F)
    ens.step(3000)
    with pytest.raises(EnsError) as ei:
        ens.sync()
    assert ei.value.code == ENS_E_DIVERGED and "step" in str(ei.value)
    with pytest.raises(EnsError) as ei:
        ens.step(1)
    assert ei.value.code == ENS_E_STATE
    ens.set_state(None, None, 0)
    ens.step(1)
    ens.sync()
    ens.close()


def test_sdof_closed_form_on_gpu():
    """ens_create_csr with one 3x3 diagonal block: the kernel reproduces the closed-form
    solution of the central-difference recurrence (same pin as the oracle's)."""
    m_, k, f = 2.0, 50.0, 3.0
    dt = 0.9 * 2.0 / math.sqrt(k / m_)
    c1, c2, c3 = oracle.coeffs(np.array([[m_]]), dt, 0, 0.0)
    ens = solver.Ensemble.from_csr([0, 1], [0], np.diag([k] * 3).reshape(1, 1, 9), c1, c2, c3, dt=dt)
    ens.set_traction(np.array([[[f, 0.0, -f]]]))
    n = 10_000
    ens.step(n)
    u, _, _, _ = ens.get_state()
    L = np.longdouble
    th = np.arccos(1 - L(c1[0, 0]) * L(k) / 2)
    ref = (L(f) / L(k)) * (1 - np.cos(L(n) * th) + np.tan(th / 2) * np.sin(L(n) * th))
    assert abs(L(u[0, 0, 0]) - ref) <= 1e-12 * (f / k) * 3
    assert u[0, 0, 2] == -u[0, 0, 0] and u[0, 0, 1] == 0.0
    ens.close()


def test_c2_full_size_sampled_realisations():
    """Config c2 at full size (96 x 262, N_s = 64, mode-1 damping 250/s) in the bench's
    launch configuration; the oracle recomputes a sample of realisations one by one."""
    cfg = configs.make("c2")
    m = cfg.mesh
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=RHO, nu=NU, k_shear=KS,
                          damping="mass", c_d=cfg.c_d)
    dt = ens.info()["dt"]
    tr = cfg.traction
    ens.set_traction(tr.F)
    ens.step(1000)
    u, _, _, _ = ens.get_state(want_prev=False)
    for s in (0, 17, 63):
        om = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E[s:s + 1], cfg.h[s:s + 1], rho=RHO,
                                nu=NU, k_shear=KS, damping=1, c_d=cfg.c_d, dt=dt)
        om.set_traction(tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
        om.run(1000)
        assert np.linalg.norm(u[s] - om.u_n[0]) <= 1e-9 * np.linalg.norm(om.u_n[0])
    ens.close()


def test_c2_laplace_law_on_gpu():
    """BASELINE config 2: steady pressure to static equilibrium, 10^4 steps; the
    homogeneous member s = 0 matches the Laplace law with the fixed-end correction."""
    cfg = configs.make("c2")
    m = cfg.mesh
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=RHO, nu=NU, k_shear=KS,
                          damping="mass", c_d=cfg.c_d)
    ens.set_traction(cfg.traction.F)
    ens.step(10_000)
    u, up, _, _ = ens.get_state()
    assert np.linalg.norm(u - up) <= 1e-10 * np.linalg.norm(u)    # at rest
    ring = 131
    nodes = np.arange(ring * 96, (ring + 1) * 96)
    rhat = m.xyz[nodes, :2] / np.linalg.norm(m.xyz[nodes, :2], axis=1, keepdims=True)
    ur = np.mean(np.einsum("ij,ij->i", u[0, nodes, :2], rhat))
    R, L, p = 2.0, 30.0, loads.P_SUPERPOSED
    ell = R * math.sqrt(KS / (2 * (1 + NU)))
    ref = (1 - NU ** 2) * p * R * R / (7e6 * 0.4) / (1 - 2 * NU ** 2 * ell / L)
    assert ur == pytest.approx(ref, rel=1e-3)
    # realisations with random fields: displacement spread around the homogeneous value
    urs = np.mean(np.einsum("sij,ij->si", u[:, nodes, :2], rhat), axis=1)
    assert np.all(np.abs(urs / ref - 1) < 0.5)
    ens.close()


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
@pytest.mark.parametrize("kernel", ["assembled", "assembled_sym", "matrix_free"])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_node_partition_bitexact(kernel, P, halo):
    """ENS_DIST_NODE (all P parts in one context): halo "nccl" = boundary rows, pack,
    device copies, interior rows; halo "p2p" = boundary rows storing u_{n+1} straight into
    the neighbours' ghost rows + release/acquire step flags, in CUDA graphs.  Both are
    bit-identical to the unpartitioned run, since each row keeps its global summation
    order."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 2)
    E, h = _mats(m, 6, 61)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel=kernel, dt=5e-5, damping="identity", c_d=0.3)
    ref = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    par = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, dist="node", world=P, halo=halo, **kw)
    inf = par.info()
    assert inf["n_owned"] == m.n_nodes and inf["halo_bytes_per_step"] > 0
    assert inf["halo"] == solver.HALO[halo] and inf["graph_steps"] > 0     # both halos captured in graphs
    for e in (ref, par):
        e.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    par.prepare()                   # both parities' graphs (with the halo) built ahead of ens_step
    for e in (ref, par):
        e.step(257)
    u0, p0, _, s0 = ref.get_state()
    u1, p1, _, s1 = par.get_state()
    assert s0 == s1 and np.array_equal(u0, u1) and np.array_equal(p0, p1)
    for e in (ref, par):            # graph replays starting at an odd step (the other parity's graph)
        e.step(130)
    u0, p0, _, s0 = ref.get_state()
    u1, p1, _, s1 = par.get_state()
    assert s0 == s1 == 387 and np.array_equal(u0, u1) and np.array_equal(p0, p1)
    rng = np.random.default_rng(P)
    x = rng.uniform(-1, 1, u0.shape)
    assert np.array_equal(ref.apply_stiffness(x), par.apply_stiffness(x))
    # checkpoint into the partitioned context, continue both
    par.set_state(u0, p0, s0)
    for e in (ref, par):
        e.step(40)
    assert np.array_equal(ref.get_state()[0], par.get_state()[0])
    ref.close(); par.close()


@pytest.mark.parametrize("kernel", ["assembled_sym", "matrix_free"])
def test_prepare_builds_graphs_without_stepping(kernel):
    """ens_prepare captures the step-loop graphs of both parities and executes nothing: the
    state and step are unchanged, and the run afterwards (graph replays from both parities,
    a traction change that drops the graphs, prepare again) is bit-identical to one without."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(20, 40), 0.01, 3), 5)
    E, h = _mats(m, 64, 17)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel=kernel, dt=5e-5, damping="mass", c_d=100.0)
    a = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    b = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    for e in (a, b):
        e.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    b.prepare()
    u, p, t, s = b.get_state()
    assert s == 0 and not u.any() and not p.any()
    for e in (a, b):
        e.step(1)
    b.prepare()
    for e in (a, b):
        e.step(200)
        e.set_traction(tr.F, tr.tab_t, tr.tab_g, 2 * tr.period, tr.ramp_T)   # new period: graphs dropped
    b.prepare()
    for e in (a, b):
        e.step(129)
    ua, pa, _, sa = a.get_state()
    ub, pb, _, sb = b.get_state()
    assert sa == sb == 330 and np.array_equal(ua, ub) and np.array_equal(pa, pb)
    a.close(); b.close()


@pytest.mark.parametrize("kernel", ["assembled", "assembled_sym"])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_node_partition_persistent_bitexact(kernel, P):
    """N2 (ens_options.persistent): all P parts advanced by one persistent cooperative kernel
    per ens_step (grid-wide barrier per step, u_{n+1} of send rows stored into the neighbours'
    ghost rows): bit-identical to the unpartitioned run, across calls, a checkpoint restart
    and a traction change."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 2)
    E, h = _mats(m, 6, 61)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel=kernel, dt=5e-5, damping="identity", c_d=0.3)
    ref = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    par = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, dist="node", world=P, halo="p2p", persistent=True, **kw)
    assert par.info()["launches_per_step"] == 1 and par.info()["graph_steps"] == 0
    for e in (ref, par):
        e.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        e.step(257)
        e.step(3)
    u0, p0, _, s0 = ref.get_state()
    u1, p1, _, s1 = par.get_state()
    assert s0 == s1 == 260 and np.array_equal(u0, u1) and np.array_equal(p0, p1)
    par.set_state(u0, p0, s0)
    F2 = np.concatenate([tr.F, 0.5 * tr.F])
    for e in (ref, par):
        e.set_traction(F2, tr.tab_t, np.concatenate([tr.tab_g, tr.tab_g[::-1]]), tr.period, tr.ramp_T)
        e.step(50)
    assert np.array_equal(ref.get_state()[0], par.get_state()[0])
    ref.close(); par.close()


def test_persistent_rejected_elsewhere():
    m = meshmod.cylinder(12, 23)
    E, h = _mats(m, 4, 3)
    for kw in (dict(dist="node", world=2, halo="nccl"), dict(dist="node", world=2, halo="p2p", kernel="matrix_free"),
               dict(dist="single")):
        with pytest.raises(EnsError) as ei:
            solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, persistent=True, **kw)
        assert ei.value.code == -8                      # ENS_E_UNSUPPORTED


def test_symmetric_storage_bitexact_vs_full():
    """ASSEMBLED_SYM stores only blocks (i, j >= i) and reads (j, i)^T for j < i, in the
    full row's column order: bit-identical to ASSEMBLED, with fewer value bytes."""
    m = meshmod.shuffle_nodes(meshmod.cylinder(32, 41), 5)
    E, h = _mats(m, 64, 71)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    out = []
    for kernel in ("assembled", "assembled_sym"):
        e = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, kernel=kernel,
                            damping="mass", c_d=100.0)
        e.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        e.step(300)
        out.append((e.get_state(), e.info()))
        e.close()
    (a, ia), (b, ib) = out
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert ib["bytes_per_step"] < 0.7 * ia["bytes_per_step"]


def test_c3_pulsatile_three_cycles_stable():
    """Config c3: pulsatile traction over 3 cardiac cycles (0.8 s each), undamped, at the
    CFL step — no divergence, displacement follows the load, and a sampled
    realisation matches the oracle after the first 2,000 steps (ramp still active)."""
    cfg = configs.make("c3", n_s=8)
    m = cfg.mesh
    tr = cfg.traction
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=RHO, nu=NU, k_shear=KS)
    dt = ens.info()["dt"]
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(2000)
    u, _, _, _ = ens.get_state(want_prev=False)
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E[3:4], cfg.h[3:4], rho=RHO, nu=NU, k_shear=KS, dt=dt)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.run(2000)
    assert np.linalg.norm(u[3] - om.u_n[0]) <= 1e-9 * np.linalg.norm(om.u_n[0])
    n_total = int(round(3 * 0.8 / dt))
    ring = 131
    nodes = np.arange(ring * 96, (ring + 1) * 96)
    rhat = m.xyz[nodes, :2] / np.linalg.norm(m.xyz[nodes, :2], axis=1, keepdims=True)
    rad = []
    done = 2000
    while done < n_total:
        k = min(2000, n_total - done)
        ens.step(k)
        done += k
        u, _, t, _ = ens.get_state(want_prev=False)
        assert np.all(np.isfinite(u))
        rad.append((t, np.mean(np.einsum("ij,ij->i", u[0, nodes, :2], rhat))))
    rad = np.array(rad)
    static = 13 * 1333.22 * 4 / (7e6 * 0.4)          # Laplace scale of the 13 mmHg baseline
    assert np.all(np.abs(rad[:, 1]) < 10 * static)
    # peak systole (40 mmHg) vs diastole (13 mmHg): the radius follows the load
    tau = rad[:, 0] % 0.8
    sys_ = rad[(tau > 0.12) & (tau < 0.18) & (rad[:, 0] > 0.8), 1]
    dia = rad[(tau > 0.5) & (tau < 0.75) & (rad[:, 0] > 0.8), 1]
    assert sys_.mean() > 1.5 * dia.mean() > 0
    ens.close()


def test_c4_aorta_sampled_parity():
    """Config c4 mesh (synthetic branched aorta, ~500k triangles) with N_s = 8: every
    kernel against the oracle on sampled realisations after 100 steps."""
    cfg = configs.make("c4", n_s=8)
    m = cfg.mesh
    tr = cfg.traction
    out = {}
    for kernel in ("assembled", "assembled_sym", "matrix_free"):
        ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=RHO, nu=NU, k_shear=KS, kernel=kernel)
        dt = ens.info()["dt"]
        ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        ens.step(100)
        out[kernel] = ens.get_state(want_prev=False)[0]
        ens.close()
    assert np.array_equal(out["assembled"], out["assembled_sym"])
    for s in (1, 6):
        om = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E[s:s + 1], cfg.h[s:s + 1], rho=RHO, nu=NU,
                                k_shear=KS, dt=dt)
        om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        om.run(100)
        for kernel in out:
            ref = om.u_n[0]
            assert np.linalg.norm(out[kernel][s] - ref) <= 1e-9 * np.linalg.norm(ref), kernel


@pytest.mark.parametrize("frame,centerline", [(0, None), (1, None), (1, [[0.5, -0.3, -5.0], [-0.2, 0.4, 12.0], [0.1, 0.0, 40.0]])])
def test_stress_and_statistics_parity(frame, centerline):
    """ens_stress / ens_displacement_stats against the oracle on a
    jittered, renumbered mesh with a random state: per-realisation stresses, their
    ensemble mean and 5%/95% quantiles."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(20, 31), 0.03, 4), 4)
    n_s = 37
    E, h = _mats(m, n_s, 81)
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS)
    rng = np.random.default_rng(frame)
    u = rng.uniform(-1e-2, 1e-2, (n_s, m.n_nodes, 3))
    ens.set_state(u, u, 0)
    got = ens.stress(frame=frame, centerline=centerline)
    ref = oracle.stress(m.xyz, m.tris, E, u, NU, KS, frame=frame, centerline=centerline)
    scale = np.abs(ref).max()
    assert np.abs(got["sigma"] - ref).max() <= 1e-12 * scale
    rm, r5, r95 = oracle.ensemble_stats(ref)
    for key, r in (("mean", rm), ("q05", r5), ("q95", r95)):
        assert np.abs(got[key] - r).max() <= 1e-12 * scale, key
    dm, d5, d95 = ens.displacement_stats()
    vals = np.concatenate([u, np.linalg.norm(u, axis=2)[..., None]], axis=2)
    om, o5, o95 = oracle.ensemble_stats(vals)
    for g, r in ((dm, om), (d5, o5), (d95, o95)):
        assert np.abs(g - r).max() <= 1e-14
    ens.close()


def test_c2_hoop_stress_statistics_on_gpu():
    """c2 to static equilibrium: mid-length hoop stress of the homogeneous member = p R /
    zeta (1e-3); the 5-95% band brackets the ensemble mean."""
    cfg = configs.make("c2")
    m = cfg.mesh
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=RHO, nu=NU, k_shear=KS,
                          damping="mass", c_d=cfg.c_d)
    ens.set_traction(cfg.traction.F)
    ens.step(10_000)
    st = ens.stress(frame=1)
    cz = m.xyz[m.tris].mean(1)[:, 2]
    mid = np.abs(cz - 15.0) < 1.0
    hoop = loads.P_SUPERPOSED * 2.0 / 0.4
    assert st["sigma"][0, mid, 1].mean() == pytest.approx(hoop, rel=1e-3)
    assert np.all(st["q05"][mid, 1] <= st["mean"][mid, 1]) and np.all(st["mean"][mid, 1] <= st["q95"][mid, 1])
    assert np.all(st["q95"][mid, 1] - st["q05"][mid, 1] > 0)
    ens.close()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_gpu_matern_sampler_matches_sparse_lu(name):
    """ens_matern_fields (multi-RHS Jacobi-PCG on the GPU) reproduces the
    host sampler's draws (scipy sparse LU of A = kappa^2 C~ + G, same z) to 1e-9."""
    nc, na = {"c1": (12, 23), "c2": (96, 262)}[name]
    m = meshmod.cylinder(nc, na)
    smp = fields.MaternSampler(m.xyz, m.tris, 3.7)
    ref = smp.standard(20210121, fields.FIELD_E, range(1, 17))
    z = fields.standard_normals(20210121, fields.FIELD_E, range(1, 17), m.n_nodes)
    x, iters, res = solver.matern_fields(m.xyz, m.tris, 3.7, z)
    assert res <= 1e-13 and iters > 0
    assert np.linalg.norm(x - ref) <= 1e-9 * np.linalg.norm(ref)


def test_gpu_matern_correlation_follows_matern():
    """Fig. 5: the empirical correlation of the generated field along the
    cylinder follows the Matérn model r(d) = (kappa d) K_1(kappa d), kappa = sqrt(8)/rho
    (nu = 1), in the interior of the 96 x 262 cylinder (4,096 draws)."""
    from scipy.special import k1
    m = meshmod.cylinder(96, 262)
    z = fields.standard_normals(7, 0, range(4096), m.n_nodes)
    x, _, _ = solver.matern_fields(m.xyz, m.tris, 3.7, z)
    kappa = math.sqrt(8.0) / 3.7
    nc = 96
    base_rings = range(100, 160, 6)
    for dr in (5, 10, 20, 32):                                  # axial ring offsets
        d = 30.0 * dr / 261
        cs = []
        for r0 in base_rings:
            a = x[:, r0 * nc:(r0 + 1) * nc]
            b = x[:, (r0 + dr) * nc:(r0 + dr + 1) * nc]
            cs.append(np.mean([np.corrcoef(a[:, k], b[:, k])[0, 1] for k in range(0, nc, 8)]))
        model = kappa * d * k1(kappa * d)
        assert np.mean(cs) == pytest.approx(model, abs=0.06), (d, np.mean(cs), model)


@pytest.mark.parametrize("kernel", ["assembled", "assembled_sym"])
def test_geometry_reassembly_parity(kernel):
    """reassemble_every = k: every k steps each
    realisation's stiffness is rebuilt on X + u; a large pressure makes the geometric
    update visible.  GPU vs oracle <= 1e-9; full vs half storage bit-identical."""
    m = meshmod.shuffle_nodes(meshmod.cylinder(16, 25), 6)
    E, h = _mats(m, 4, 91)
    tr = loads.steady(m.xyz, m.tris, p=5 * loads.P_SUPERPOSED)     # u ~ 0.13 cm: 10% geometric effect
    dt, k, n = 1e-4, 25, 400
    outs = {}
    for kern in ("assembled", kernel):
        ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, kernel=kern, dt=dt,
                              damping="mass", c_d=100.0, reassemble_every=k)
        assert ens.info()["reassemble_every"] == k and ens.info()["graph_steps"] == 0
        ens.set_traction(tr.F)
        ens.step(n)
        outs[kern] = ens.get_state()[0]
        ens.close()
    assert np.array_equal(outs["assembled"], outs[kernel])
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, damping=1, c_d=100.0, dt=dt)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
    om.run(n, reassemble_every=k)
    assert np.linalg.norm(outs[kernel] - om.u_n) <= 1e-9 * np.linalg.norm(om.u_n)
    lin = oracle.OracleModel(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, damping=1, c_d=100.0, dt=dt)
    lin.set_traction(tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
    lin.run(n)
    assert np.linalg.norm(om.u_n - lin.u_n) > 1e-6 * np.linalg.norm(lin.u_n)    # the update matters


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
def test_geometry_reassembly_node_partition_bitexact(halo):
    """Re-assembly reads the ghost rows' u as well: partitioned runs (P = 3) stay
    bit-identical to the single-part run."""
    m = meshmod.shuffle_nodes(meshmod.cylinder(16, 25), 6)
    E, h = _mats(m, 4, 92)
    tr = loads.steady(m.xyz, m.tris, p=5 * loads.P_SUPERPOSED)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel="assembled", dt=1e-4, damping="mass", c_d=100.0,
              reassemble_every=20)
    out = []
    for extra in ({}, dict(dist="node", world=3, halo=halo)):
        ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw, **extra)
        ens.set_traction(tr.F)
        ens.step(150)
        out.append(ens.get_state()[0])
        ens.close()
    assert np.array_equal(out[0], out[1])


def test_reassembly_rejected_for_matrix_free():
    m = meshmod.cylinder(8, 5)
    E, h = _mats(m, 2, 1)
    with pytest.raises(EnsError):
        solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, kernel="matrix_free",
                        reassemble_every=10)


def test_async_traction_update_and_observe():
    """Same-shape ens_set_traction is enqueued after the running steps (no sync, no graph
    rebuild) and ens_observe snapshots u_n while later steps run: the results equal the
    oracle run with the traction switched at the same step, and the snapshot equals the
    state at its step."""
    import torch
    m = meshmod.shuffle_nodes(meshmod.cylinder(16, 25), 8)
    E, h = _mats(m, 4, 93)
    tr1 = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    tr2 = loads.pulsatile(m.xyz, m.tris, p_base=1.5 * loads.P_SUPERPOSED, period=0.012, systole=0.005,
                          ramp_T=0.003)
    ens, om = _pair(m, E, h, kernel="assembled_sym", damping="mass", c_d=80.0, dt=5e-5)
    ens.set_traction(tr1.F, tr1.tab_t, tr1.tab_g, tr1.period, tr1.ramp_T)
    ens.step(150)                                    # graph replays + direct steps
    snap = torch.empty((4, m.n_nodes, 3), dtype=torch.float64).pin_memory()
    ens.observe(snap)
    ens.set_traction(2 * tr1.F, tr1.tab_t, 0.5 * tr1.tab_g, tr1.period, tr1.ramp_T)    # same shape: async
    ens.step(130)
    assert ens.observe_wait() == 150
    ens.set_traction(tr2.F, tr2.tab_t, tr2.tab_g, tr2.period, tr2.ramp_T)              # period changes
    ens.step(70)
    u, up, _, st = ens.get_state()
    om.set_traction(tr1.F, tr1.tab_t, tr1.tab_g, tr1.period, tr1.ramp_T)
    om.run(150)
    assert np.linalg.norm(snap.numpy() - om.u_n) <= 1e-12 * np.linalg.norm(om.u_n)
    om.set_traction(2 * tr1.F, tr1.tab_t, 0.5 * tr1.tab_g, tr1.period, tr1.ramp_T)
    om.run(130)
    om.set_traction(tr2.F, tr2.tab_t, tr2.tab_g, tr2.period, tr2.ramp_T)
    om.run(70)
    assert st == 350
    assert np.linalg.norm(u - om.u_n) <= 1e-11 * np.linalg.norm(om.u_n)
    assert np.linalg.norm(up - om.u_nm1) <= 1e-11 * np.linalg.norm(om.u_nm1)
    with pytest.raises(EnsError):
        ens.observe_wait()                           # nothing in flight
    ens.close()


def test_fp64_fma_probe_is_plausible():
    """ens_measure_fp64 (the ALU roofline of a2): a B200 has ~37 TFLOP/s of FP64 FMA
    (148 SMs x 64 DFMA/clk x 2 x ~1.9 GHz); the probe must land in a plausible band."""
    tf = solver.measure_fp64_tflops(0)
    assert 15.0 < tf < 80.0, tf


@pytest.mark.parametrize("name,kernel,steps,samples", [
    ("c4", "assembled_sym", 100, (0, 77, 127)),        # bench --config c4 (N_s = 128, the default kernel)
    ("c5", "matrix_free", 30, (0, 311, 511)),          # bench --config c5 (N_s = 512, one GPU)
])
def test_full_size_launch_configuration_sampled(name, kernel, steps, samples):
    """The aorta configs at their full size and in the launch configuration bench.py times
    (N_s = 128 / 512 on one device): sampled realisations recomputed one by one by the
    oracle (ensemble equivalence makes the single-realisation run the reference), <= 1e-9."""
    cfg = configs.make(name)
    m, tr = cfg.mesh, cfg.traction
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, k_shear=cfg.k_shear,
                          damping=cfg.damping, c_d=cfg.c_d, kernel=kernel)
    dt = ens.info()["dt"]
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(steps)
    u = ens.get_state(want_prev=False)[0]
    ens.close()
    for s in samples:
        om = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E[s:s + 1], cfg.h[s:s + 1], rho=cfg.rho, nu=cfg.nu,
                                k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d, dt=dt)
        om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        om.run(steps)
        ref = om.u_n[0]
        assert np.linalg.norm(u[s] - ref) <= 1e-9 * np.linalg.norm(ref), s


def _nonmanifold_mesh():
    """A cylinder with (a) a flap of 5 triangles fanned around one of its vertices (a bowtie
    vertex: two incidence chains), (b) a second flap sharing only a vertex with the first
    one, and (c) a separate 2-triangle patch (a second component)."""
    m = meshmod.cylinder(16, 9)
    xyz, tris = list(m.xyz), [tuple(t) for t in m.tris]
    fixed = list(m.fixed)
    hub = 4 * 16 + 3                                # a mid-length vertex
    c = m.xyz[hub]
    nrm = np.array([c[0], c[1], 0.0]) / np.hypot(c[0], c[1])
    ring = []
    for k in range(6):                              # open fan: 6 rim nodes, 5 triangles
        a = 0.9 * k / 5 - 0.45
        p = c + 0.6 * nrm + 0.5 * np.array([np.cos(a) * nrm[1], -np.sin(a) * 0 + 0.0, np.sin(a)]) \
            + 0.3 * np.array([-nrm[1], nrm[0], 0.0]) * np.cos(a)
        ring.append(len(xyz))
        xyz.append(p)
        fixed.append(0)
    for k in range(5):
        tris.append((hub, ring[k], ring[k + 1]))
    tip = ring[5]                                   # second flap around the first flap's tip
    ring2 = []
    for k in range(3):
        p = xyz[tip] + np.array([0.2 * k, 0.3, 0.1 + 0.05 * k])
        ring2.append(len(xyz))
        xyz.append(p)
        fixed.append(0)
    tris.append((tip, ring2[0], ring2[1]))
    tris.append((tip, ring2[1], ring2[2]))
    q = len(xyz)                                    # separate component
    for p in ([5.0, 5.0, 0.0], [6.0, 5.0, 0.0], [5.0, 6.0, 0.0], [6.0, 6.2, 0.3]):
        xyz.append(np.array(p))
        fixed.append(0)
    tris.append((q, q + 1, q + 2))
    tris.append((q + 1, q + 3, q + 2))
    return meshmod.Mesh(np.array(xyz, dtype=np.float64), np.array(tris, dtype=np.int32),
                        np.array(fixed, dtype=np.uint8), name="nonmanifold")


@pytest.mark.parametrize("kernel", ["assembled", "assembled_sym", "matrix_free"])
def test_nonmanifold_vertex_and_components(kernel):
    """Non-manifold (bowtie) vertices make the matrix-free fans restart (several incidence
    chains per node) and a separate component makes RCM restart: SpMM <= 1e-12 and 300
    steps <= 1e-9 against the oracle, for every kernel."""
    m = meshmod.shuffle_nodes(_nonmanifold_mesh(), 9)
    E, h = _mats(m, 6, 41)
    ens, om = _pair(m, E, h, kernel=kernel, damping="mass", c_d=200.0)
    rng = np.random.default_rng(3)
    _check_spmm(ens, om, rng.uniform(-1, 1, (6, m.n_nodes, 3)))
    tr = loads.steady(m.xyz, m.tris)
    ens.set_traction(tr.F)
    ens.step(300)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, 0.0, 0.0)
    om.run(300)
    u = ens.get_state()[0]
    assert np.linalg.norm(u - om.u_n) <= 1e-9 * np.linalg.norm(om.u_n)
    ens.close()


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
@pytest.mark.parametrize("kernel", ["assembled_sym", "matrix_free"])
def test_many_small_parts_bitexact(kernel, halo):
    """P = 8 parts of a 157-node mesh: parts whose every row is a boundary row, parts with
    several (not only adjacent) neighbours, a part holding a whole component — still
    bit-identical to the single-part run."""
    m = meshmod.shuffle_nodes(_nonmanifold_mesh(), 10)
    E, h = _mats(m, 4, 42)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel=kernel, dt=2e-5, damping="mass", c_d=100.0)
    out = []
    for extra in ({}, dict(dist="node", world=8, halo=halo)):
        ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw, **extra)
        ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        ens.step(150)
        out.append(ens.get_state())
        ens.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
