"""Time the staged matrix-free step on c2 alone and after other contexts in the same process."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import configs

def timed(cfg, kernel, K):
    m, tr = cfg.mesh, cfg.traction
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, k_shear=cfg.k_shear,
                          damping=cfg.damping, c_d=cfg.c_d, kernel=kernel)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(20); ens.sync()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); ens.step(K); e1.record(st); e1.synchronize()
    inf = ens.info()
    ens.close()
    return e0.elapsed_time(e1) / K * 1e3, inf

c2 = configs.make("c2")
print("c2 mf first", timed(c2, "matrix_free", 500)[0], flush=True)
seq = sys.argv[1:] or ["c4:matrix_free"]
big = {}
for item in seq:
    name, kernel = item.split(":")
    if name not in big: big[name] = configs.make(name)
    us, inf = timed(big[name], kernel, 50)
    print(name, kernel, us, "graph_steps", inf.get("graph_steps"), flush=True)
    print("c2 mf after", item, timed(c2, "matrix_free", 500)[0], flush=True)
