"""Quick F3 sanity: SpMM parity vs oracle, bit-identity vs F2, and c2 timing per variant."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import configs, fields, loads, mesh as meshmod

def mats(m, n_s, seed):
    E, h, _ = fields.sample_materials(m.xyz, m.tris, n_s, E_mean=7e6, E_std=7e5, h_mean=0.4, h_std=0.04, rho_corr=3.7, seed=seed)
    return E, h

for n_s in (64, 128):
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(40, 51), 0.02, 1), 1)
    E, h = mats(m, n_s, 11)
    res = {}
    for var in ("tiles", "warp", "staged"):
        ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, rho=1.06, nu=0.5, kernel="matrix_free", mf_variant=var,
                              damping="mass", c_d=100.0, dt=2e-5)
        print(n_s, var, ens.info()["mf_variant"], flush=True)
        x = np.random.default_rng(1).uniform(-1, 1, (n_s, m.n_nodes, 3))
        y = ens.apply_stiffness(x)
        tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
        ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        ens.step(300)
        u = ens.get_state()[0]
        res[var] = (y, u)
        ens.close()
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, E, h, rho=1.06, nu=0.5, k_shear=5/6)
    yo = om.spmm(x)
    for var in res:
        print(n_s, var, "spmm rel", np.linalg.norm(res[var][0] - yo) / np.linalg.norm(yo),
              "bitexact y", np.array_equal(res[var][0], res["tiles"][0]), "bitexact u", np.array_equal(res[var][1], res["tiles"][1]), flush=True)

for name in ():
    cfg = configs.make(name)
    m, tr = cfg.mesh, cfg.traction
    for var in ("tiles", "warp", "staged"):
        if var == "warp" and name == "c4": continue
        try:
            ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, k_shear=cfg.k_shear,
                                  damping=cfg.damping, c_d=cfg.c_d, kernel="matrix_free", mf_variant=var)
        except Exception as e:
            print(name, var, "ERR", e); continue
        ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        ens.step(20); ens.sync()
        st = torch.cuda.current_stream()
        K = 500 if name == "c2" else 100
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); ens.step(K); e1.record(st); e1.synchronize()
        ms = e0.elapsed_time(e1) / K
        inf = ens.info()
        print(name, var, f"{ms*1e3:.1f} us/step", f"{inf['bytes_per_step']/ms/1e6:.0f} GB/s", f"{cfg.n_s*3*m.n_nodes/ms*1e3:.3e} DOF/s", flush=True)
        u = ens.get_state(want_prev=False)[0]
        print("   norm", float(np.linalg.norm(u)))
        ens.close()
