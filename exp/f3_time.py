"""Time one matrix-free variant on a config: python exp/f3_time.py c2 staged [steps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import configs
name, var = sys.argv[1], sys.argv[2]
K = int(sys.argv[3]) if len(sys.argv) > 3 else (500 if name in ("c2", "c3") else 100)
kernel = sys.argv[4] if len(sys.argv) > 4 else "matrix_free"
cfg = configs.make(name)
m, tr = cfg.mesh, cfg.traction
ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, k_shear=cfg.k_shear,
                      damping=cfg.damping, c_d=cfg.c_d, kernel=kernel, mf_variant=var)
ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
ens.step(20); ens.sync()
st = torch.cuda.current_stream()
best = 1e9
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); ens.step(K); e1.record(st); e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / K)
inf = ens.info()
print(f"{name} {kernel}/{var} shape={os.environ.get('ENS_MFS_SHAPE','default')} {best*1e3:.1f} us/step "
      f"{inf['bytes_per_step']/best/1e6:.0f} GB/s frac={inf['bytes_per_step']/best/1e6/6547.2:.3f} "
      f"{cfg.n_s*3*m.n_nodes/best*1e3:.3e} DOF/s", flush=True)
ens.close()
