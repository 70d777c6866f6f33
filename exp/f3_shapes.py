"""F3 consumer shapes: bit-identity against the default shape on a small mesh, then timing per
shape on a config.  python exp/f3_shapes.py c4 11x3 7x3w 11x3w"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import configs, fields, loads, mesh as meshmod
name, shapes = sys.argv[1], sys.argv[2:]

def run_small(n_s, shape, damping):
    os.environ["ENS_MFS_SHAPE"] = shape
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 2)
    E, h, _ = fields.sample_materials(m.xyz, m.tris, n_s, E_mean=7e6, E_std=7e5, h_mean=0.4, h_std=0.04,
                                      rho_corr=3.7, seed=77)
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=1.06, nu=0.5, k_shear=5 / 6, kernel="matrix_free",
                          dt=5e-5, damping=damping, c_d=120.0 if damping == "mass" else 0.3, mf_variant="staged")
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(200)
    u, p, _, _ = ens.get_state()
    y = ens.apply_stiffness(np.random.default_rng(1).uniform(-1, 1, u.shape))
    ens.close()
    return u, p, y

for n_s in (128, 256):
    for damping in ("mass", "identity"):
        ref = run_small(n_s, "11x3", damping)
        for sh in shapes:
            got = run_small(n_s, sh, damping)
            print("bitexact", n_s, damping, sh, all(np.array_equal(a, b) for a, b in zip(ref, got)), flush=True)

cfg = configs.make(name)
m, tr = cfg.mesh, cfg.traction
K = 500 if name in ("c2", "c3") else 100
for rep in range(2):
    for sh in shapes:
        os.environ["ENS_MFS_SHAPE"] = sh
        ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, k_shear=cfg.k_shear,
                              damping=cfg.damping, c_d=cfg.c_d, kernel="matrix_free", mf_variant="staged")
        ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        ens.step(20); ens.sync()
        st = torch.cuda.current_stream()
        best = 1e9
        for r in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); ens.step(K); e1.record(st); e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / K)
        inf = ens.info()
        print(f"{name} {sh} {best*1e3:.1f} us/step frac={inf['bytes_per_step']/best/1e6/6547.2:.3f} "
              f"{cfg.n_s*3*m.n_nodes/best*1e3:.3e} DOF/s", flush=True)
        ens.close()
