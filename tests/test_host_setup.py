"""CPU tests of the product's host setup (libens.so ens_host_* entry points) against the
oracle: integer maps bit-exact, floating-point setup within rounding (-m "not gpu")."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from paper_2101_09059_b200 import _ffi, solver
from paper_2101_09059_b200.inputs import mesh as meshmod

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "ens.h")).read()
    declared = set(re.findall(r"\b(ens_[a-z0-9_]+)\s*\(", header))
    declared -= {"ens_ctx"}
    L = _ffi.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(_ffi.EXPORTS)


MESHES = [
    lambda: meshmod.cylinder(12, 23),
    lambda: meshmod.shuffle_nodes(meshmod.cylinder(12, 23), 1),
    lambda: meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(17, 11), 0.05, 2), 2),
    lambda: meshmod.shuffle_nodes(meshmod.cylinder(96, 40), 3),
]


@pytest.mark.parametrize("mk", MESHES)
def test_pattern_bitexact_vs_oracle(mk):
    m = mk()
    perm, row_ptr, col = solver.host_pattern(m.n_nodes, m.tris)
    operm = oracle.rcm(m.n_nodes, m.tris)
    orow, ocol = oracle.csr(m.n_nodes, m.tris, operm)
    assert np.array_equal(perm, operm)
    assert np.array_equal(row_ptr, orow)
    assert np.array_equal(col, ocol)


def test_pattern_two_components_bitexact():
    a = meshmod.cylinder(5, 4)
    b = meshmod.cylinder(6, 3)
    tris = np.concatenate([b.tris + a.n_nodes, a.tris])
    V = a.n_nodes + b.n_nodes
    perm, row_ptr, col = solver.host_pattern(V, tris)
    assert np.array_equal(perm, oracle.rcm(V, tris))


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_and_ghosts_bitexact(P):
    m = meshmod.shuffle_nodes(meshmod.cylinder(24, 30), 7)
    perm, row_ptr, col = solver.host_pattern(m.n_nodes, m.tris)
    b = solver.host_partition(row_ptr, P)
    ob, ogh, _ = oracle.halo_maps(row_ptr, col, P)
    assert np.array_equal(b, ob)
    for p in range(P):
        assert np.array_equal(solver.host_ghosts(row_ptr, col, b[p], b[p + 1]), ogh[p])


def test_validate_codes_match_oracle():
    m = meshmod.cylinder(6, 3)
    cases = []
    t = m.tris.copy(); t[3, 1] = m.n_nodes; cases.append((m.xyz, t))
    t = m.tris.copy(); t[4, 2] = t[4, 0]; cases.append((m.xyz, t))
    x = m.xyz.copy(); x[m.tris[5, 2]] = x[m.tris[5, 0]] + 0.5 * (x[m.tris[5, 1]] - x[m.tris[5, 0]])
    cases.append((x, m.tris))
    cases.append((m.xyz, np.concatenate([m.tris, m.tris[:1]])))
    cases.append((np.concatenate([m.xyz, [[9.0, 9.0, 9.0]]]), m.tris))     # node in no triangle
    cases.append((m.xyz, m.tris))
    for xyz, tris in cases:
        assert solver.host_validate(xyz, tris) == oracle.validate_mesh(xyz, tris)


def test_element_stiffness_vs_oracle():
    m = meshmod.perturb(meshmod.cylinder(16, 12), 0.1, 5)
    for nu in (0.0, 0.3, 0.5):
        K, A = solver.host_element_stiffness(m.xyz, m.tris, nu, 5 / 6)
        Ko, Ao = oracle.all_khat(m.xyz, m.tris, nu, 5 / 6)
        scale = np.abs(Ko).max(axis=(1, 2), keepdims=True)
        assert np.max(np.abs(K - Ko) / scale) < 1e-13
        np.testing.assert_allclose(A, Ao, rtol=1e-14)
        assert np.array_equal(K, np.transpose(K, (0, 2, 1)))


def test_materials_vs_oracle():
    m = meshmod.perturb(meshmod.cylinder(16, 12), 0.1, 6)
    rng = np.random.default_rng(0)
    E = rng.uniform(5e6, 9e6, (3, m.n_nodes))
    h = rng.uniform(0.3, 0.5, (3, m.n_nodes))
    al, ms, dt = solver.host_materials(m.xyz, m.tris, E, h, 1.06, 0.9)
    np.testing.assert_allclose(al, oracle.alpha(m.n_nodes, m.tris, E, h), rtol=1e-14)
    np.testing.assert_allclose(ms, oracle.mass(m.xyz, m.tris, h, 1.06), rtol=1e-13)
    assert dt == pytest.approx(oracle.cfl(m.xyz, m.tris, E, 1.06, 0.9), rel=1e-14)


def test_create_without_gpu_fails_loudly():
    """On a box without a device, ens_create must fail with ENS_E_CUDA — never fall back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    m = meshmod.cylinder(6, 3)
    E = np.full((1, m.n_nodes), 7e6)
    h = np.full((1, m.n_nodes), 0.4)
    with pytest.raises(_ffi.EnsError) as ei:
        solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=1.06, nu=0.5)
    assert ei.value.code in (_ffi.ENS_E_CUDA, _ffi.ENS_E_OOM)


def test_fp64_probe_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_ffi.EnsError) as ei:
        solver.measure_fp64_tflops()
    assert ei.value.code == _ffi.ENS_E_CUDA


@pytest.mark.parametrize("bad", ["E", "h", "nu", "rho", "mesh"])
def test_create_argument_errors(bad):
    m = meshmod.cylinder(6, 3)
    E = np.full((1, m.n_nodes), 7e6)
    h = np.full((1, m.n_nodes), 0.4)
    kw = dict(rho=1.06, nu=0.5)
    tris = m.tris
    if bad == "E":
        E[0, 3] = -1
    elif bad == "h":
        h[0, 2] = 0
    elif bad == "nu":
        kw["nu"] = 0.7
    elif bad == "rho":
        kw["rho"] = 0.0
    else:
        tris = m.tris.copy(); tris[0, 0] = 999
    with pytest.raises(_ffi.EnsError) as ei:
        solver.Ensemble(m.xyz, tris, m.fixed, E, h, torch_alloc=False, **kw)
    assert ei.value.code == (_ffi.ENS_E_MESH if bad == "mesh" else _ffi.ENS_E_ARG)


@pytest.mark.parametrize("P", [2, 3, 5])
def test_halo_plan_vs_oracle(P):
    """The product's halo plan (ens_host_halo_plan) against the oracle's C11 maps: owned
    ranges, ghost counts, send lists (as local rows) and receive slices, bit-exact; every
    row with a ghost column inside the boundary launch ranges."""
    m = meshmod.shuffle_nodes(meshmod.cylinder(20, 33), 4)
    perm, row_ptr, col = solver.host_pattern(m.n_nodes, m.tris)
    ob, ogh, osend = oracle.halo_maps(row_ptr, col, P)
    for p in range(P):
        pl = solver.host_halo_plan(row_ptr, col, P, p)
        lo, hi = pl["lo"], pl["hi"]
        assert (lo, hi) == (ob[p], ob[p + 1]) and pl["n_ghost"] == len(ogh[p])
        peers = {q: (so, sn, rr, rn) for q, so, sn, rr, rn in pl["peers"]}
        for q in range(P):
            if q == p:
                continue
            exp_send = osend[p][q] - lo
            exp_recv = ogh[p][(ogh[p] >= ob[q]) & (ogh[p] < ob[q + 1])]
            if len(exp_send) == 0 and len(exp_recv) == 0:
                assert q not in peers
                continue
            so, sn, rr, rn = peers[q]
            assert np.array_equal(pl["send_rows"][so:so + sn], exp_send)
            assert rn == len(exp_recv)
            if rn:
                first = np.searchsorted(ogh[p], exp_recv[0])
                assert rr == (hi - lo) + first
        n_own = hi - lo
        for i in range(lo, hi):
            cols = col[row_ptr[i]:row_ptr[i + 1]]
            if np.any((cols < lo) | (cols >= hi)):
                li = i - lo
                assert li < pl["b_lo"] or li >= n_own - pl["b_hi"]


def test_null_context_is_an_argument_error():
    """Every context call rejects a NULL context with ENS_E_ARG and a message (no crash);
    ens_destroy(NULL) is a no-op."""
    L = _ffi.lib()
    i64 = C.c_int64()
    calls = {
        "ens_step": lambda: L.ens_step(None, 1),
        "ens_sync": lambda: L.ens_sync(None),
        "ens_get_state": lambda: L.ens_get_state(None, None, None, None, None),
        "ens_get_owned": lambda: L.ens_get_owned(None, None, C.byref(i64)),
        "ens_set_state": lambda: L.ens_set_state(None, None, None, 0.0, 0),
        "ens_set_traction": lambda: L.ens_set_traction(None, 0, None, 0, None, None, 0.0, 0.0),
        "ens_apply_stiffness": lambda: L.ens_apply_stiffness(None, None, None),
        "ens_stress": lambda: L.ens_stress(None, 0, None, 0, None, None, None, None),
        "ens_displacement_stats": lambda: L.ens_displacement_stats(None, None, None, None),
        "ens_observe": lambda: L.ens_observe(None, None),
        "ens_observe_wait": lambda: L.ens_observe_wait(None, C.byref(i64)),
        "ens_p2p_export": lambda: L.ens_p2p_export(None, None),
        "ens_p2p_connect": lambda: L.ens_p2p_connect(None, None),
        "ens_query": lambda: L.ens_query(None, None),
        "ens_measure_fp64": lambda: L.ens_measure_fp64(-1, None),
    }
    for name, call in calls.items():
        assert call() == _ffi.ENS_E_ARG, name
        assert L.ens_last_error(None), name
    L.ens_destroy(None)


@pytest.mark.parametrize("n_s", [64, 128])
def test_mf_staged_tiles_partition_and_budget(n_s):
    """The STAGED matrix-free tiling (ens_host_mf_tiles): every RCM row in exactly one tile,
    strips are runs of consecutive rows, every tile's stage image (+ the F_k budget) fits the
    stage and moves in <= 96 bulk copies; compact patches move fewer bytes per row than
    strips at the same budget (each patch's 1-ring is smaller than a strip's)."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(48, 80), 0.02, 4), 3)
    V = m.n_nodes
    per_row = {}
    for patches in (False, True):
        tile_of, tb, te, budget = solver.host_mf_tiles(m.xyz, m.tris, n_s, patches=patches, max_rows=32,
                                                       stage_bytes=77312)
        n = len(tb)
        assert budget == 77312 and n > 0
        assert tile_of.min() == 0 and tile_of.max() == n - 1
        rows_per = np.bincount(tile_of, minlength=n)
        assert rows_per.sum() == V and rows_per.min() >= 1 and rows_per.max() <= 32
        assert np.all(tb + 4 * 32 * rows_per <= budget) and np.all(te <= 96) and np.all(te >= 3)
        if not patches:
            assert np.all(np.diff(tile_of) >= 0)          # consecutive rows, tiles in row order
        per_row[patches] = tb.sum() / V
    assert per_row[True] < per_row[False]
