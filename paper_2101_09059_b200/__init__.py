"""B200-native ensemble explicit shell solver (arXiv 2101.09059 hot path).

    from paper_2101_09059_b200 import Ensemble
    ens = Ensemble(xyz, tris, fixed, E, h, rho=1.06, nu=0.5)
    ens.set_traction(F)            # [K][V][3] nodal forces
    ens.step(1000)                 # fused sm_100a steps, asynchronous
    u_n, u_nm1, t, step = ens.get_state()

The C ABI is include/ens.h (libens.so); this package is its thin ctypes binding plus the
seeded input generators (paper_2101_09059_b200.inputs).  Importing the package does
not load the library; the first call does, and fails loudly if it is missing.
"""
__all__ = ["Ensemble", "EnsError"]


def __getattr__(name):
    if name in ("Ensemble", "EnsError"):
        from . import solver
        return getattr(solver, name)
    raise AttributeError(name)
