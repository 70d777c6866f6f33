"""Tiny staged run (progress printed) to debug a checked (-DENS_CHECKS) build."""
import sys, os, faulthandler
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2101_09059_b200 import solver
from paper_2101_09059_b200.inputs import configs
print("import ok", flush=True)
cfg = configs.make("c1", n_s=64)
m = cfg.mesh
ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, kernel="matrix_free")
print("created", ens.info()["mf_variant"], flush=True)
ens.set_traction(cfg.traction.F)
print("traction", flush=True)
ens.step(1)
print("stepped", flush=True)
ens.sync()
print("synced", flush=True)
ens.step(100); ens.sync()
print("100 ok", flush=True)
