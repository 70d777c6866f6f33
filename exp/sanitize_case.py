"""One small run of a kernel / data path for compute-sanitizer (memcheck, racecheck, synccheck):
    python exp/sanitize_case.py <kernel> <mf_variant> [P] [halo] [N_s]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import fields, loads, mesh as meshmod

kernel, variant = sys.argv[1], sys.argv[2]
P = int(sys.argv[3]) if len(sys.argv) > 3 else 1
halo = sys.argv[4] if len(sys.argv) > 4 else "nccl"
m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(16, 30), 0.01, 3), 2)
n_s = int(sys.argv[5]) if len(sys.argv) > 5 else 64
E, h, _ = fields.sample_materials(m.xyz, m.tris, n_s, E_mean=7e6, E_std=7e5, h_mean=0.4, h_std=0.04,
                                  rho_corr=3.7, seed=5)
kw = dict(dist="node", world=P, halo=halo) if P > 1 else {}
ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=1.06, nu=0.5, kernel=kernel, mf_variant=variant,
                      dt=5e-5, damping="mass", c_d=100.0, torch_alloc=False, **kw)
tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
ens.step(70)                      # one graph replay (64) + 6 direct steps
u = ens.get_state()[0]
y = ens.apply_stiffness(np.random.default_rng(0).uniform(-1, 1, u.shape))
print(kernel, variant, P, halo, n_s, "ok", float(np.linalg.norm(u)), float(np.linalg.norm(y)), ens.info()["mf_variant"])
ens.close()
