"""CPU fp64 oracle for arXiv 2101.09059's ensemble explicit shell step — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import this package.  It loads oracle/liboracle.so (plain C, -O2 -ffp-contract=off,
oracle/oracle.c) through ctypes; it shares no code with paper_2101_09059_b200/.

`OracleModel` composes the C functions in the paper's order (§2.2.1, §2.3):
element stiffness (Eq. 7-10) -> Gauss-point E*zeta scaling -> assembly -> lumped mass ->
central-difference coefficients (Eq. 22) -> time loop.  Everything is in the caller's
original node numbering, realisation-outermost ([n_s][V][3]).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11",
          "-D_DEFAULT_SOURCE"]


def build(force: bool = False) -> str:
    """Compile oracle/oracle.c into oracle/liboracle.so (gcc)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        i64, i32, f64, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
        sig = {
            "orc_validate_mesh": (C.c_int, [i64, i64, vp, vp, vp]),
            "orc_adjacency": (i64, [i64, i64, vp, vp, vp]),
            "orc_rcm": (None, [i64, vp, vp, vp]),
            "orc_csr": (i64, [i64, vp, vp, vp, vp, vp]),
            "orc_element_khat": (None, [vp, f64, f64, vp, vp]),
            "orc_all_khat": (None, [i64, vp, vp, f64, f64, vp, vp]),
            "orc_alpha": (None, [i64, i64, vp, i32, vp, vp, vp]),
            "orc_assemble": (C.c_int, [i64, i64, vp, vp, vp, vp, i32, vp, vp]),
            "orc_mass": (None, [i64, i64, vp, vp, i32, vp, f64, vp]),
            "orc_coeffs": (None, [i64, i32, vp, f64, i32, f64, vp, vp, vp]),
            "orc_cfl": (f64, [i64, i64, vp, vp, i32, vp, f64, f64]),
            "orc_load_coeffs": (None, [f64, i32, i32, vp, vp, f64, f64, vp]),
            "orc_spmm": (None, [i64, vp, vp, i32, vp, vp, vp]),
            "orc_run": (i64, [i64, vp, vp, i32, vp, vp, vp, vp, vp, i32, vp, i32, vp, vp, f64, f64,
                              f64, i64, i64, vp, vp]),
            "orc_partition_bounds": (None, [i64, vp, i32, vp]),
            "orc_stress": (None, [i64, i64, vp, vp, i32, vp, vp, f64, f64, i32, vp, i32, vp]),
            "orc_ghosts": (i64, [i64, vp, vp, i64, i64, vp]),
            "orc_set_threads": (C.c_int, [C.c_int]),
            "orc_reassemble": (C.c_int, [i64, i64, vp, vp, vp, vp, f64, f64, i32, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's loops over realisations (results are independent)."""
    return int(lib().orc_set_threads(int(n)))


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------------------------
# integer maps
# ------------------------------------------------------------------------------------

def validate_mesh(xyz, tris):
    xyz, tris = _c(xyz, np.float64), _c(tris, np.int32)
    bad = np.zeros(1, np.int64)
    rc = lib().orc_validate_mesh(xyz.shape[0], tris.shape[0], _p(xyz), _p(tris), _p(bad))
    return int(rc), int(bad[0])


def adjacency(V, tris):
    tris = _c(tris, np.int32)
    ptr = np.zeros(V + 1, np.int64)
    adj = np.zeros(max(1, 6 * tris.shape[0]), np.int32)
    m = lib().orc_adjacency(V, tris.shape[0], _p(tris), _p(ptr), _p(adj))
    return ptr, adj[:m].copy()


def rcm(V, tris) -> np.ndarray:
    """perm[new] = old."""
    ptr, adj = adjacency(V, tris)
    perm = np.zeros(V, np.int32)
    lib().orc_rcm(V, _p(ptr), _p(adj), _p(perm))
    return perm


def csr(V, tris, perm=None):
    """(row_ptr int64[V+1], col int32[nnzb]) in the numbering perm (None = original)."""
    ptr, adj = adjacency(V, tris)
    row_ptr = np.zeros(V + 1, np.int64)
    col = np.zeros(V + len(adj), np.int32)
    pp = None if perm is None else _c(perm, np.int32)
    n = lib().orc_csr(V, _p(ptr), _p(adj), _p(pp), _p(row_ptr), _p(col))
    return row_ptr, col[:n].copy()


def partition_bounds(row_ptr, P):
    row_ptr = _c(row_ptr, np.int64)
    b = np.zeros(P + 1, np.int64)
    lib().orc_partition_bounds(len(row_ptr) - 1, _p(row_ptr), P, _p(b))
    return b


def ghosts(row_ptr, col, lo, hi):
    row_ptr, col = _c(row_ptr, np.int64), _c(col, np.int32)
    V = len(row_ptr) - 1
    g = np.zeros(V, np.int32)
    n = lib().orc_ghosts(V, _p(row_ptr), _p(col), lo, hi, _p(g))
    return g[:n].copy()


def halo_maps(row_ptr, col, P):
    """bounds, ghosts[p], send[p][q] (sorted rows of p that are ghosts of q) — C11."""
    b = partition_bounds(row_ptr, P)
    gh = [ghosts(row_ptr, col, int(b[p]), int(b[p + 1])) for p in range(P)]
    send = [[gh[q][(gh[q] >= b[p]) & (gh[q] < b[p + 1])] if q != p else np.zeros(0, np.int32)
             for q in range(P)] for p in range(P)]
    return b, gh, send


# ------------------------------------------------------------------------------------
# floating-point setup
# ------------------------------------------------------------------------------------

def element_khat(X, nu, k):
    X = _c(X, np.float64).reshape(9)
    K = np.zeros(81)
    A = np.zeros(1)
    lib().orc_element_khat(_p(X), nu, k, _p(K), _p(A))
    return K.reshape(9, 9), float(A[0])


def all_khat(xyz, tris, nu, k):
    xyz, tris = _c(xyz, np.float64), _c(tris, np.int32)
    F = tris.shape[0]
    K = np.zeros((F, 9, 9))
    A = np.zeros(F)
    lib().orc_all_khat(F, _p(xyz), _p(tris), nu, k, _p(K), _p(A))
    return K, A


def alpha(V, tris, E, h):
    tris, E, h = _c(tris, np.int32), _c(E, np.float64), _c(h, np.float64)
    n_s, F = E.shape[0], tris.shape[0]
    out = np.zeros((n_s, F))
    lib().orc_alpha(V, F, _p(tris), n_s, _p(E), _p(h), _p(out))
    return out


def mass(xyz, tris, h, rho):
    xyz, tris, h = _c(xyz, np.float64), _c(tris, np.int32), _c(h, np.float64)
    out = np.zeros(h.shape)
    lib().orc_mass(xyz.shape[0], tris.shape[0], _p(xyz), _p(tris), h.shape[0], _p(h), rho, _p(out))
    return out


def coeffs(m, dt, damping, c_d):
    m = _c(m, np.float64)
    c1, c2, c3 = np.zeros(m.shape), np.zeros(m.shape), np.zeros(m.shape)
    lib().orc_coeffs(m.shape[1], m.shape[0], _p(m), dt, damping, c_d, _p(c1), _p(c2), _p(c3))
    return c1, c2, c3


def cfl(xyz, tris, E, rho, safety=0.9):
    xyz, tris, E = _c(xyz, np.float64), _c(tris, np.int32), _c(E, np.float64)
    return float(lib().orc_cfl(xyz.shape[0], tris.shape[0], _p(xyz), _p(tris), E.shape[0], _p(E),
                               rho, safety))


def load_coeffs(t, n_fields, tab_t, tab_g, period, ramp_T):
    tab_t = _c(tab_t, np.float64)
    tab_g = _c(tab_g, np.float64)
    out = np.zeros(n_fields)
    lib().orc_load_coeffs(t, n_fields, len(tab_t), _p(tab_t), _p(tab_g), period, ramp_T, _p(out))
    return out


def spmm(row_ptr, col, Kval, u):
    row_ptr, col, Kval, u = _c(row_ptr, np.int64), _c(col, np.int32), _c(Kval, np.float64), _c(u, np.float64)
    y = np.zeros_like(u)
    lib().orc_spmm(len(row_ptr) - 1, _p(row_ptr), _p(col), u.shape[0], _p(Kval), _p(u), _p(y))
    return y


def stress(xyz, tris, E, u, nu, k_shear, frame=1, centerline=None):
    """Element stresses [n_s][F][6] (orc_stress; frame 0 local shell, 1 cylindrical)."""
    xyz, tris, E, u = _c(xyz, np.float64), _c(tris, np.int32), _c(E, np.float64), _c(u, np.float64)
    cl = None if centerline is None else _c(centerline, np.float64)
    n_s, F = E.shape[0], tris.shape[0]
    out = np.zeros((n_s, F, 6))
    lib().orc_stress(xyz.shape[0], F, _p(xyz), _p(tris), n_s, _p(E), _p(u), nu, k_shear, frame,
                     _p(cl), 0 if cl is None else cl.shape[0], _p(out))
    return out


def ensemble_stats(values, q=(0.05, 0.95)):
    """Mean and quantiles over realisations (axis 0).  Quantile p of n sorted values v:
    h = (n - 1) p, v[floor h] + (h - floor h) (v[floor h + 1] - v[floor h]) (the 5%-95%
    bands of PAPER.md:452; linear interpolation between order statistics)."""
    v = np.sort(np.asarray(values, dtype=np.float64), axis=0)
    n = v.shape[0]
    out = [v.mean(axis=0)]
    for p in q:
        h = (n - 1) * p
        lo = int(np.floor(h))
        hi = min(lo + 1, n - 1)
        out.append(v[lo] + (h - lo) * (v[hi] - v[lo]))
    return out


def run_raw(row_ptr, col, Kval, c1, c2, c3, fixed, u_n, u_nm1, *, dt, nsteps, step0=0,
            F=None, tab_t=None, tab_g=None, period=0.0, ramp_T=0.0):
    """orc_run on caller-supplied CSR / values / coefficients (SDOF and synthetic tests).
    Kval [n_s][nnzb][9], c* [n_s][V], u_* [n_s][V][3] (updated in place)."""
    row_ptr, col = _c(row_ptr, np.int64), _c(col, np.int32)
    V = len(row_ptr) - 1
    Kval = _c(Kval, np.float64)
    c1, c2, c3 = _c(c1, np.float64), _c(c2, np.float64), _c(c3, np.float64)
    fixed = None if fixed is None else _c(fixed, np.uint8)
    F = np.zeros((1, V, 3)) if F is None else _c(F, np.float64)
    tab_t = np.zeros(0) if tab_t is None else _c(tab_t, np.float64)
    tab_g = np.zeros((F.shape[0], 0)) if tab_g is None else _c(tab_g, np.float64)
    assert u_n.flags.c_contiguous and u_nm1.flags.c_contiguous
    return int(lib().orc_run(V, _p(row_ptr), _p(col), u_n.shape[0], _p(Kval), _p(c1), _p(c2), _p(c3),
                             _p(fixed), F.shape[0], _p(F), len(tab_t), _p(tab_t), _p(tab_g),
                             float(period), float(ramp_T), float(dt), int(step0), int(nsteps),
                             _p(u_n), _p(u_nm1)))


class OracleModel:
    """The whole per-realisation pipeline, in the paper's order, original numbering."""

    def __init__(self, xyz, tris, fixed, E, h, *, rho, nu, k_shear, damping=0, c_d=0.0,
                 dt=None, cfl_safety=0.9, with_K=True):
        self.xyz = _c(xyz, np.float64)
        self.tris = _c(tris, np.int32)
        self.V = self.xyz.shape[0]
        self.F = self.tris.shape[0]
        self.fixed = _c(fixed if fixed is not None else np.zeros(self.V), np.uint8)
        self.E = _c(E, np.float64)
        self.h = _c(h, np.float64)
        self.n_s = self.E.shape[0]
        self.rho, self.nu, self.k_shear = rho, nu, k_shear
        self.dt_cfl = cfl(self.xyz, self.tris, self.E, rho, cfl_safety)
        self.dt = float(dt) if dt is not None and dt > 0 else self.dt_cfl
        self.row_ptr, self.col = csr(self.V, self.tris, None)
        self.Khat, self.area = all_khat(self.xyz, self.tris, nu, k_shear)
        self.alpha = alpha(self.V, self.tris, self.E, self.h)
        self.Kval = None
        if with_K:
            self.Kval = np.zeros((self.n_s, len(self.col), 9))
            rc = lib().orc_assemble(self.V, self.F, _p(self.tris), _p(self.row_ptr), _p(self.col),
                                    _p(self.Khat), self.n_s, _p(self.alpha), _p(self.Kval))
            assert rc == 0
        self.m = mass(self.xyz, self.tris, self.h, rho)
        self.c1, self.c2, self.c3 = coeffs(self.m, self.dt, damping, c_d)
        self.u_n = np.zeros((self.n_s, self.V, 3))
        self.u_nm1 = np.zeros((self.n_s, self.V, 3))
        self.step = 0
        self.set_traction(np.zeros((1, self.V, 3)), np.zeros(0), np.zeros((1, 0)), 0.0, 0.0)

    def set_traction(self, F, tab_t, tab_g, period, ramp_T):
        self.Fk = _c(F, np.float64)
        self.tab_t = _c(tab_t, np.float64)
        self.tab_g = _c(np.asarray(tab_g).reshape(self.Fk.shape[0], len(self.tab_t)), np.float64)
        self.period, self.ramp_T = float(period), float(ramp_T)

    def reassemble(self):
        """Kval from the deformed geometry X + u_n (orc_reassemble)."""
        rc = lib().orc_reassemble(self.V, self.F, _p(self.xyz), _p(self.tris), _p(self.row_ptr), _p(self.col),
                                  self.nu, self.k_shear, self.n_s, _p(self.alpha), _p(self.u_n), _p(self.Kval))
        assert rc == 0

    def run(self, n: int, reassemble_every: int = 0) -> int:
        """n steps; with reassemble_every = k > 0 the stiffness is rebuilt on X + u_m
        before every step index m >= 1 with m % k == 0."""
        if reassemble_every <= 0:
            return self._run(n)
        bad, done = -1, 0
        while done < n:
            m = self.step
            if m > 0 and m % reassemble_every == 0:
                self.reassemble()
            nxt = (m // reassemble_every + 1) * reassemble_every
            chunk = min(n - done, nxt - m)
            b = self._run(chunk)
            bad = b if bad < 0 else bad
            done += chunk
        return bad

    def _run(self, n: int) -> int:
        bad = lib().orc_run(self.V, _p(self.row_ptr), _p(self.col), self.n_s, _p(self.Kval),
                            _p(self.c1), _p(self.c2), _p(self.c3), _p(self.fixed),
                            self.Fk.shape[0], _p(self.Fk), len(self.tab_t), _p(self.tab_t),
                            _p(self.tab_g), self.period, self.ramp_T, self.dt, self.step, n,
                            _p(self.u_n), _p(self.u_nm1))
        self.step += n
        return int(bad)

    def spmm(self, u):
        return spmm(self.row_ptr, self.col, self.Kval, u)

    def K_sparse(self, s: int):
        """K_s as a scipy CSR matrix (3V x 3V), for the pins."""
        import scipy.sparse as sp
        rows, cols, vals = [], [], []
        for i in range(self.V):
            for b in range(self.row_ptr[i], self.row_ptr[i + 1]):
                j = self.col[b]
                blk = self.Kval[s, b].reshape(3, 3)
                for c in range(3):
                    for d in range(3):
                        rows.append(3 * i + c)
                        cols.append(3 * j + d)
                        vals.append(blk[c, d])
        return sp.csr_matrix((vals, (rows, cols)), shape=(3 * self.V, 3 * self.V))
