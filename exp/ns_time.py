"""Step time of each path at a given N_s on a config: python exp/ns_time.py <config> <n_s> [steps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import configs
name, n_s = sys.argv[1], int(sys.argv[2])
K = int(sys.argv[3]) if len(sys.argv) > 3 else 200
cfg = configs.make(name, n_s=n_s)
m, tr = cfg.mesh, cfg.traction
for kernel, var in (("matrix_free", "staged"), ("matrix_free", "tiles"), ("assembled_sym", "auto")):
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, k_shear=cfg.k_shear,
                          damping=cfg.damping, c_d=cfg.c_d, kernel=kernel, mf_variant=var)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.prepare(); ens.step(20); ens.sync()
    st = torch.cuda.current_stream()
    best = 1e9
    for r in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); ens.step(K); e1.record(st); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / K)
    inf = ens.info()
    print(f"{name} N_s={n_s} {kernel}/{var} {best*1e3:.1f} us/step frac={inf['bytes_per_step']/best/1e6/6547.2:.3f} "
          f"{n_s*3*m.n_nodes/best*1e3:.3e} DOF/s", flush=True)
    ens.close()
