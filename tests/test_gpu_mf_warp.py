"""The per-warp TMA item-stream form of the matrix-free step (kernels.cu F2w,
k_step_mf_warp; the library's choice at N_s = 64 without identity damping; ENS_MF_WARP=1
takes it for any N_s % 64 == 0, exercised here in subprocesses) on a B200 (-m gpu).

F2w computes exactly F2's arithmetic in F2's order, so it is held to the
oracle's bars (SpMM <= 1e-12, steps <= 1e-9 relative L2) and, against F2 itself
(ENS_MF_WARP=0 in a subprocess), to bit-identity; node partitions stay bit-identical to the
unpartitioned run (each row keeps its global summation order).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import fields, loads, mesh as meshmod

from test_gpu_parity import _check_spmm, _nonmanifold_mesh, _pair

pytestmark = pytest.mark.gpu
RHO, NU, KS = 1.06, 0.5, 5.0 / 6.0
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _mats(m, n_s, seed):
    E, h, _ = fields.sample_materials(m.xyz, m.tris, n_s, E_mean=7e6, E_std=7e5, h_mean=0.4,
                                      h_std=0.04, rho_corr=3.7, seed=seed)
    return E, h


@pytest.mark.parametrize("n_s", [64])
def test_mf_warp_vs_oracle_nonmanifold(n_s):
    """Fan restarts (bowtie vertices) and a second component through the item programs:
    PREV items at every chain start."""
    m = meshmod.shuffle_nodes(_nonmanifold_mesh(), 11)
    E, h = _mats(m, n_s, 43)
    ens, om = _pair(m, E, h, kernel="matrix_free", damping="mass", c_d=150.0)
    assert ens.info()["mf_variant"] == 1
    rng = np.random.default_rng(5)
    _check_spmm(ens, om, rng.uniform(-1, 1, (n_s, m.n_nodes, 3)))
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(300)
    om.run(300)
    u = ens.get_state()[0]
    assert np.linalg.norm(u - om.u_n) <= 1e-9 * np.linalg.norm(om.u_n)
    ens.close()


_SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import fields, loads, mesh as meshmod
n_s = {n_s}
m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 2)
E, h, _ = fields.sample_materials(m.xyz, m.tris, n_s, E_mean=7e6, E_std=7e5, h_mean=0.4,
                                  h_std=0.04, rho_corr=3.7, seed=77)
ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=1.06, nu=0.5, k_shear=5.0 / 6.0,
                      kernel="matrix_free", dt=5e-5, damping="mass", c_d=120.0)
tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
ens.step(400)
u, p, _, s = ens.get_state()
x = np.random.default_rng(1).uniform(-1, 1, u.shape)
y = ens.apply_stiffness(x)
np.savez({out!r}, u=u, p=p, y=y)
print(json.dumps({{"mf_variant": ens.info()["mf_variant"], "step": s}}))
"""


@pytest.mark.parametrize("n_s", [64, 128, 192])
def test_mf_warp_bitexact_vs_tile_kernel(n_s, tmp_path):
    """Same inputs through F2 (ENS_MF_WARP=0) and F2w (ENS_MF_WARP=1; N_s > 64 takes the
    2-D tensor copies of u): states after 400 pulsatile steps (two load fields staged per
    OWN item) and one product y = K x, bit for bit."""
    res = {}
    for flag in ("0", "1"):
        out = str(tmp_path / f"mf{flag}.npz")
        env = dict(os.environ, ENS_MF_WARP=flag)
        r = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"),
                                                                n_s=n_s, out=out)],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        meta = json.loads(r.stdout.strip().splitlines()[-1])
        assert meta["mf_variant"] == int(flag) and meta["step"] == 400
        res[flag] = np.load(out)
    for k in ("u", "p", "y"):
        assert np.array_equal(res["0"][k], res["1"][k]), k


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_mf_warp_node_partition_bitexact(P, halo):
    """Row ranges [row0, row0 + V) of boundary / interior launches, ghost rows in the item
    programs, P2P forwarding from the update: bit-identical to the single-part run."""
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 4)
    E, h = _mats(m, 64, 62)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel="matrix_free", dt=5e-5, damping="mass", c_d=80.0)
    ref = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    par = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, dist="node", world=P, halo=halo, **kw)
    assert ref.info()["mf_variant"] == 1 and par.info()["mf_variant"] == 1
    for e in (ref, par):
        e.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        e.step(201)
    u0, p0, _, s0 = ref.get_state()
    u1, p1, _, s1 = par.get_state()
    assert s0 == s1 and np.array_equal(u0, u1) and np.array_equal(p0, p1)
    x = np.random.default_rng(P).uniform(-1, 1, u0.shape)
    assert np.array_equal(ref.apply_stiffness(x), par.apply_stiffness(x))
    ref.close(); par.close()


def test_mf_warp_not_used_for_identity_damping_or_odd_ns():
    """The launcher falls back to F2 where F2w does not apply (mode-2 damping stages c2, c3;
    N_s not a multiple of 64)."""
    m = meshmod.cylinder(12, 23)
    for n_s, damping in ((64, "identity"), (48, "mass"), (96, "none")):
        E, h = _mats(m, n_s, 3)
        ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=RHO, nu=NU, kernel="matrix_free",
                              damping=damping, c_d=10.0)
        assert ens.info()["mf_variant"] == 0
        ens.close()
