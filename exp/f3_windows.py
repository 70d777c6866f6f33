"""Per-window step times (CUDA events) to look for intermittent slow windows:
python exp/f3_windows.py <config> <kernel> <windows> <steps>"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import configs
name, kernel, W, K = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cfg = configs.make(name)
m, tr = cfg.mesh, cfg.traction
ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, k_shear=cfg.k_shear,
                      damping=cfg.damping, c_d=cfg.c_d, kernel=kernel)
ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
ens.step(3); ens.sync()
st = torch.cuda.current_stream()
ts = []
for w in range(W):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); ens.step(K); e1.record(st); e1.synchronize()
    ts.append(e0.elapsed_time(e1) / K * 1e3)
print(name, kernel, " ".join(f"{t:.1f}" for t in ts), flush=True)
ens.close()
