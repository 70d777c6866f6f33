"""A/B bit-identity of matrix-free variants: python exp/mfw_check.py <config> <n_s> <steps> <out.npy>"""
import sys, numpy as np
from paper_2101_09059_b200 import Ensemble
from paper_2101_09059_b200.inputs import configs
cfg = configs.make(sys.argv[1], n_s=int(sys.argv[2]))
n_s = int(sys.argv[2]); steps = int(sys.argv[3])
E, h = cfg.E[:n_s], cfg.h[:n_s]
ens = Ensemble(cfg.mesh.xyz, cfg.mesh.tris, cfg.mesh.fixed, E, h, rho=1.06, nu=0.5,
               damping="mass", c_d=250.0, kernel="matrix_free")
ens.set_traction(cfg.traction.F)
ens.step(steps)
u_n, u_nm1, t, step = ens.get_state()
np.save(sys.argv[4], np.asarray(u_n))
print("saved", sys.argv[4], np.abs(np.asarray(u_n)).max())
