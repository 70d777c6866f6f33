"""The three device data paths of the matrix-free step (ens.h ENS_MF_*) on a B200 (-m gpu).

TILES (k_step_matrix_free), WARP (k_step_mf_warp) and STAGED (k_step_mf_staged: warp-
specialised tile stages, the default for N_s % 64 == 0) compute the same sums in the same
order per row, so they are held to the oracle's bars (SpMM <= 1e-12, steps
<= 1e-9 relative L2) and to bit-identity with each other; node partitions stay bit-identical
to the unpartitioned run (each row keeps its global summation order).
"""
import os

import numpy as np
import pytest

import oracle
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200._ffi import ENS_E_UNSUPPORTED, EnsError
from paper_2101_09059_b200.inputs import fields, loads, mesh as meshmod

from test_gpu_parity import _check_spmm, _nonmanifold_mesh, _pair

pytestmark = pytest.mark.gpu
RHO, NU, KS = 1.06, 0.5, 5.0 / 6.0
MFV = solver.MF_VARIANT


def _mats(m, n_s, seed):
    E, h, _ = fields.sample_materials(m.xyz, m.tris, n_s, E_mean=7e6, E_std=7e5, h_mean=0.4,
                                      h_std=0.04, rho_corr=3.7, seed=seed)
    return E, h


def _run(m, E, h, variant, damping="mass", c_d=120.0, steps=400, **kw):
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, kernel="matrix_free",
                          dt=5e-5, damping=damping, c_d=c_d, mf_variant=variant, **kw)
    assert ens.info()["mf_variant"] == MFV[variant]
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(steps)
    u, p, _, s = ens.get_state()
    x = np.random.default_rng(1).uniform(-1, 1, u.shape)
    y = ens.apply_stiffness(x)
    ens.close()
    assert s == steps
    return u, p, y


@pytest.mark.parametrize("n_s", [64, 128, 192, 256, 320])
def test_variants_bitexact_and_oracle_spmm(n_s):
    """N_s >= 256 takes STAGED's sliced stages (2-D tensor copies of 64-realisation slices)."""
    """States after 400 pulsatile steps (two load fields: ramp + table) and one product
    y = K x through TILES, WARP and STAGED: bit for bit; STAGED's product against the oracle."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 2)
    E, h = _mats(m, n_s, 77)
    res = {v: _run(m, E, h, v) for v in ("tiles", "warp", "staged")}
    for v in ("warp", "staged"):
        for k in range(3):
            assert np.array_equal(res["tiles"][k], res[v][k]), (v, k)
    ens, om = _pair(m, E, h, kernel="matrix_free", mf_variant="staged")
    _check_spmm(ens, om, np.random.default_rng(n_s).uniform(-1, 1, (n_s, m.n_nodes, 3)))
    ens.close()


@pytest.mark.parametrize("n_s,damping", [(66, "mass"), (100, "identity"), (200, "mass"), (258, "mass"),
                                         (500, "identity")])
def test_staged_ragged_ensemble(n_s, damping):
    """Any even N_s >= 64 takes STAGED: the last unit (or sliced stage) of a row is partial,
    its lanes past N_s address realisation N_s - 2 and store nothing.  States and products
    bit-identical to TILES (which handles any N_s), the product against the oracle.  N_s = 66,
    100, 200: two-slice units (66 or 100 of 128; 128 + 72); 258: sliced, 64-wide slices (5, the
    last 2 wide); 500: sliced, 128-wide (4, the last 116 wide)."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 9)
    E, h = _mats(m, n_s, 31)
    c_d = 120.0 if damping == "mass" else 0.3
    ref = _run(m, E, h, "tiles", damping=damping, c_d=c_d, steps=200)
    got = _run(m, E, h, "staged", damping=damping, c_d=c_d, steps=200)
    for k in range(3):
        assert np.array_equal(ref[k], got[k]), k
    ens, om = _pair(m, E, h, kernel="matrix_free")
    assert ens.info()["mf_variant"] == MFV["staged"]             # AUTO takes it
    _check_spmm(ens, om, np.random.default_rng(n_s).uniform(-1, 1, (n_s, m.n_nodes, 3)))
    ens.close()


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
def test_staged_ragged_node_partition(halo):
    """A ragged N_s (100: one two-slice unit per row with 100 of its 128 lanes' realisations
    valid) in a node partition with P2P forwarding of the partial unit: bit-identical to one
    part."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 4)
    E, h = _mats(m, 100, 62)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel="matrix_free", dt=5e-5, damping="mass", c_d=80.0,
              mf_variant="staged")
    ref = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    par = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, dist="node", world=3, halo=halo, **kw)
    for e in (ref, par):
        e.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        e.step(201)
    u0, p0, _, s0 = ref.get_state()
    u1, p1, _, s1 = par.get_state()
    assert s0 == s1 and np.array_equal(u0, u1) and np.array_equal(p0, p1)
    ref.close(); par.close()


def test_staged_identity_damping_bitexact():
    """Per-row c2, c3 arrays (damping mode 2) in the staged kernel (the C23 instance)."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(20, 40), 0.01, 5), 3)
    E, h = _mats(m, 64, 5)
    a = _run(m, E, h, "tiles", damping="identity", c_d=0.3)
    b = _run(m, E, h, "staged", damping="identity", c_d=0.3)
    for k in range(3):
        assert np.array_equal(a[k], b[k]), k


def test_staged_nonmanifold_vs_oracle():
    """Fan restarts (bowtie vertices) and a second component through the staged records."""
    m = meshmod.shuffle_nodes(_nonmanifold_mesh(), 11)
    E, h = _mats(m, 64, 43)
    ens, om = _pair(m, E, h, kernel="matrix_free", damping="mass", c_d=150.0, mf_variant="staged")
    rng = np.random.default_rng(5)
    _check_spmm(ens, om, rng.uniform(-1, 1, (64, m.n_nodes, 3)))
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(300)
    om.run(300)
    u = ens.get_state()[0]
    assert np.linalg.norm(u - om.u_n) <= 1e-9 * np.linalg.norm(om.u_n)
    ens.close()


@pytest.mark.parametrize("sliced", ["0", "1"])
@pytest.mark.parametrize("tiling", ["strip", "patch"])
@pytest.mark.parametrize("n_s", [64, 128])
def test_staged_tilings_bitexact(n_s, tiling, sliced, monkeypatch):
    """Strips of consecutive rows and compact patches (ENS_MFS_TILING, read at create) only
    change which rows share a stage: bit-identical results."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 6)
    E, h = _mats(m, n_s, 9)
    ref = _run(m, E, h, "tiles", steps=150)
    monkeypatch.setenv("ENS_MFS_TILING", tiling)
    monkeypatch.setenv("ENS_MFS_SLICED", sliced)        # N_s = 128 in 64-realisation slices too
    got = _run(m, E, h, "staged", steps=150)
    for k in range(3):
        assert np.array_equal(ref[k], got[k]), k


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("n_s", [64, 128, 256])
def test_staged_node_partition_bitexact(n_s, P, halo):
    """Boundary / interior launches each with their own tile set, ghost rows in the stages,
    P2P forwarding from the update: bit-identical to the single-part run."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 4)
    E, h = _mats(m, n_s, 62)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel="matrix_free", dt=5e-5, damping="mass", c_d=80.0,
              mf_variant="staged")
    ref = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    par = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, dist="node", world=P, halo=halo, **kw)
    for e in (ref, par):
        e.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        e.step(201)
    u0, p0, _, s0 = ref.get_state()
    u1, p1, _, s1 = par.get_state()
    assert s0 == s1 and np.array_equal(u0, u1) and np.array_equal(p0, p1)
    x = np.random.default_rng(P).uniform(-1, 1, u0.shape)
    assert np.array_equal(ref.apply_stiffness(x), par.apply_stiffness(x))
    ref.close(); par.close()


@pytest.mark.parametrize("damping", ["mass", "identity"])
@pytest.mark.parametrize("n_s", [128, 256])
def test_staged_shapes_bitexact(n_s, damping, monkeypatch):
    """Consumer shapes (ENS_MFS_SHAPE, read at create): one 64-realisation slice per unit
    (11x3, 15x3) or two (7x3w, the default at N_s % 128 == 0; 11x3w) change only which warp
    computes a realisation, not its operations: bit-identical states and products (N_s = 256
    takes the sliced stages: 64-realisation slices for 11x3 / 15x3, 128 for the wide shapes)."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 8)
    E, h = _mats(m, n_s, 21)
    c_d = 120.0 if damping == "mass" else 0.3
    ref = _run(m, E, h, "tiles", damping=damping, c_d=c_d, steps=200)
    for shape in ("11x3", "15x3", "7x3w", "11x3w"):
        monkeypatch.setenv("ENS_MFS_SHAPE", shape)
        got = _run(m, E, h, "staged", damping=damping, c_d=c_d, steps=200)
        for k in range(3):
            assert np.array_equal(ref[k], got[k]), (shape, k)


def test_variant_selection_and_rejection():
    """AUTO takes STAGED where it applies (even N_s >= 64) and TILES elsewhere; asking for a
    path that does not apply is ENS_E_UNSUPPORTED."""
    m = meshmod.cylinder(12, 23)
    # the staged shape the plan picks (ens_info): consumers, unit width, stage-row width
    shapes = {64: (11, 64, 64), 128: (7, 128, 128), 100: (7, 128, 100), 192: (11, 64, 192), 500: (7, 128, 128),
              66: (7, 128, 66)}
    for n_s, want in ((64, "staged"), (128, "staged"), (100, "staged"), (192, "staged"), (500, "staged"), (66, "staged"),
                      (48, "tiles"), (5, "tiles"), (101, "tiles")):
        E, h = _mats(m, n_s, 3)
        ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, kernel="matrix_free")
        inf = ens.info()
        assert inf["mf_variant"] == MFV[want]
        if want == "staged":
            assert (inf["mfs_consumers"], inf["mfs_unit_width"], inf["mfs_stage_width"]) == shapes[n_s], n_s
            assert inf["mfs_stages"] == 3
        else:
            assert inf["mfs_consumers"] == 0
        ens.close()
    for n_s, damping, variant in ((48, "mass", "staged"), (64, "identity", "warp"), (96, "none", "warp")):
        E, h = _mats(m, n_s, 3)
        with pytest.raises(EnsError) as ei:
            solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, kernel="matrix_free",
                            damping=damping, c_d=10.0, mf_variant=variant)
        assert ei.value.code == ENS_E_UNSUPPORTED
    E, h = _mats(m, 64, 3)                         # assembled kernels ignore the option
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, kernel="assembled_sym", mf_variant="staged")
    assert ens.info()["mf_variant"] == 0
    ens.close()


@pytest.mark.parametrize("n_s", [64, 128])
def test_staged_divergence_detected(n_s):
    """A step 3x above the stability limit blows up: the staged kernel's non-finite check
    (all-ones exponent per realisation; at N_s = 128 in the two-slice units) raises
    ENS_E_DIVERGED and latches the context."""
    from paper_2101_09059_b200._ffi import ENS_E_DIVERGED, ENS_E_STATE
    m = meshmod.cylinder(12, 23)
    E, h = _mats(m, n_s, 51)
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, kernel="matrix_free",
                          mf_variant="staged")
    dt = 3.0 * ens.info()["dt"] / 0.9 * 1.3
    ens.close()
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, k_shear=KS, kernel="matrix_free",
                          mf_variant="staged", dt=dt)
    ens.set_traction(loads.steady(m.xyz, m.tris).F)
    ens.step(3000)
    with pytest.raises(EnsError) as ei:
        ens.sync()
    assert ei.value.code == ENS_E_DIVERGED
    with pytest.raises(EnsError) as ei:
        ens.step(1)
    assert ei.value.code == ENS_E_STATE
    ens.close()
