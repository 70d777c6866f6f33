"""Python binding of the C ABI (include/ens.h): argument marshalling only.

Every step of the hot path runs in libens.so's sm_100a kernels.  PyTorch supplies the
device memory (its caching allocator, through the ABI's dev_alloc/dev_free callbacks)
and the CUDA stream; nothing here computes any part of the method.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _ffi
from ._ffi import EnsError, check, lib

DAMPING = {"none": 0, "mass": 1, "identity": 2, 0: 0, 1: 1, 2: 2}
KERNEL = {"assembled": 0, "matrix_free": 1, "assembled_sym": 2, 0: 0, 1: 1, 2: 2}
DIST = {"single": 0, "node": 1, "ensemble": 2, 0: 0, 1: 1, 2: 2}
HALO = {"nccl": 0, "p2p": 1, 0: 0, 1: 1}
# matrix-free data paths (ens.h ENS_MF_*): same arithmetic, different data movement
MF_VARIANT = {"auto": 0, "tiles": 1, "warp": 2, "staged": 3, 0: 0, 1: 1, 2: 2, 3: 3}
MF_KERNEL_FN = {1: "k_step_matrix_free", 2: "k_step_mf_warp", 3: "k_step_mf_staged"}


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _TorchAllocator:
    """dev_alloc / dev_free callbacks backed by torch's CUDA caching allocator."""

    def __init__(self, device):
        import torch
        self.torch = torch
        self.device = device
        self.live = {}
        self.alloc_cb = _ffi.DEV_ALLOC(self._alloc)
        self.free_cb = _ffi.DEV_FREE(self._free)

    def _alloc(self, nbytes, _user):
        try:
            t = self.torch.empty(int(nbytes), dtype=self.torch.uint8, device=self.device)
        except Exception:     # OOM -> NULL -> ENS_E_OOM
            return None
        self.live[t.data_ptr()] = t
        return t.data_ptr()

    def _free(self, ptr, _user):
        self.live.pop(ptr, None)


class Ensemble:
    """N_s realisations of the wall, advanced together by the fused sm_100a step.

    Arrays crossing this API are realisation-outermost in the caller's node numbering:
    E, h: [n_s][V]; u: [n_s][V][3]; F: [K][V][3].
    """

    def __init__(self, xyz, tris, fixed, E, h, *, rho, nu, k_shear=5.0 / 6.0, dt=0.0,
                 cfl_safety=0.9, c_d=0.0, damping="none", kernel="assembled", dist="single",
                 s_begin=0, rank=0, world=1, nccl_comm=None, device=None, stream=None,
                 torch_alloc=True, reassemble_every=0, halo="nccl", p2p_procs=False, group=None,
                 mf_variant="auto", persistent=False, _ctx=None):
        """dist="node" splits the RCM rows into `world` parts.  halo="nccl": NCCL
        send/recv with nccl_comm (one part per process) or, without it, device copies
        between all parts held here.  halo="p2p": device-initiated stores into the
        neighbours' ghost rows; p2p_procs=True => one part per process, connected to the
        other ranks of `group` (torch.distributed, default group) through CUDA IPC.
        mf_variant ("auto", "tiles", "warp", "staged"): the matrix-free data path (ens.h).
        persistent=True (node partition, P2P halo, assembled kernels): one persistent kernel per
        ens_step call instead of per-step launches (ens.h ens_options.persistent)."""
        self._ctx = None
        self._alloc = None
        self._p2p_group, self._p2p_multi = None, False
        if _ctx is not None:                      # from_csr
            self._ctx, self._alloc, self.n_s, self.V = _ctx
            return
        xyz, tris = _c(xyz, np.float64), _c(tris, np.int32)
        E, h = _c(E, np.float64), _c(h, np.float64)
        fixed = None if fixed is None else _c(fixed, np.uint8)
        self.V, self.n_s = xyz.shape[0], E.shape[0]
        mesh = _ffi.EnsMesh(self.V, tris.shape[0], _p(xyz), _p(tris), _p(fixed))
        mat = _ffi.EnsMaterials(self.n_s, _p(E), _p(h), rho, nu, k_shear, s_begin)
        opt, self._alloc = _options(dt, cfl_safety, c_d, damping, kernel, dist, rank, world,
                                    device, stream, torch_alloc)
        if nccl_comm is not None:
            opt.nccl_comm = C.c_void_p(int(nccl_comm))
        opt.reassemble_every = int(reassemble_every)
        opt.halo = HALO[halo]
        opt.p2p_procs = int(bool(p2p_procs))
        opt.mf_variant = MF_VARIANT[mf_variant]
        opt.persistent = int(bool(persistent))
        ctx = C.c_void_p()
        check(lib().ens_create(C.byref(mesh), C.byref(mat), C.byref(opt), C.byref(ctx)))
        self._ctx = ctx
        self._p2p_multi = bool(p2p_procs) and int(world) > 1
        if self._p2p_multi:
            self._p2p_group = group
            self._p2p_connect(group)

    def _p2p_connect(self, group):
        """All-gather the CUDA IPC blobs of every rank (ens_p2p_export) and connect."""
        import torch.distributed as dist
        blob = (C.c_char * _ffi.P2P_BLOB_BYTES)()
        check(lib().ens_p2p_export(self._ctx, blob), self._ctx)
        world = dist.get_world_size(group)
        objs = [None] * world
        dist.all_gather_object(objs, bytes(blob), group=group)
        allb = b"".join(objs)
        check(lib().ens_p2p_connect(self._ctx, allb), self._ctx)

    @classmethod
    def from_csr(cls, row_ptr, col, Kval, c1, c2, c3, fixed=None, dt=1.0, *, device=None,
                 stream=None, torch_alloc=True):
        """Test-only: synthetic operator (ens_create_csr).  Kval [n_s][nnzb][9], c* [n_s][V]."""
        row_ptr, col = _c(row_ptr, np.int64), _c(col, np.int32)
        Kval = _c(Kval, np.float64)
        c1, c2, c3 = _c(c1, np.float64), _c(c2, np.float64), _c(c3, np.float64)
        fixed = None if fixed is None else _c(fixed, np.uint8)
        V, n_s = len(row_ptr) - 1, Kval.shape[0]
        opt, alloc = _options(dt, 0.9, 0.0, 0, 0, 0, 0, 1, device, stream, torch_alloc)
        ctx = C.c_void_p()
        check(lib().ens_create_csr(V, _p(row_ptr), _p(col), n_s, _p(Kval), _p(c1), _p(c2), _p(c3),
                                   _p(fixed), float(dt), C.byref(opt), C.byref(ctx)))
        return cls(None, None, None, None, None, rho=0, nu=0, _ctx=(ctx, alloc, n_s, V))

    # ---- lifecycle ------------------------------------------------------------------
    def close(self):
        if self._ctx:
            lib().ens_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- the ABI calls --------------------------------------------------------------
    def set_traction(self, F, tab_t=None, tab_g=None, period=0.0, ramp_T=0.0):
        F = _c(F, np.float64)
        K = F.shape[0]
        tab_t = np.zeros(0) if tab_t is None else _c(tab_t, np.float64)
        tab_g = np.zeros((K, 0)) if tab_g is None else _c(tab_g, np.float64)
        check(lib().ens_set_traction(self._ctx, K, _p(F), len(tab_t), _p(tab_t), _p(tab_g),
                                     float(period), float(ramp_T)), self._ctx)

    def step(self, n: int = 1):
        check(lib().ens_step(self._ctx, int(n)), self._ctx)

    def prepare(self):
        """Build the step-loop CUDA graphs now (setup; ens_prepare), not in the first ens_step."""
        check(lib().ens_prepare(self._ctx), self._ctx)

    def sync(self):
        check(lib().ens_sync(self._ctx), self._ctx)

    def owned(self) -> np.ndarray:
        """Caller node ids of the rows get_state returns (all nodes unless NODE on NCCL)."""
        n = C.c_int64()
        check(lib().ens_get_owned(self._ctx, None, C.byref(n)), self._ctx)
        ids = np.zeros(n.value, np.int32)
        check(lib().ens_get_owned(self._ctx, _p(ids), C.byref(n)), self._ctx)
        return ids

    def get_state(self, u_n=None, u_nm1=None, want_prev=True):
        """Returns (u_n, u_nm1, t, step); fills the given host buffers if provided."""
        n = C.c_int64()
        check(lib().ens_get_owned(self._ctx, None, C.byref(n)), self._ctx)
        shape = (self.n_s, n.value, 3)
        if u_n is None:
            u_n = np.empty(shape)
        if want_prev and u_nm1 is None:
            u_nm1 = np.empty(shape)
        t = C.c_double()
        st = C.c_int64()
        check(lib().ens_get_state(self._ctx, _ptr(u_n), _ptr(u_nm1), C.byref(t), C.byref(st)), self._ctx)
        return u_n, u_nm1, t.value, st.value

    def observe(self, out=None):
        """Enqueue a snapshot of u_n into `out` ([n_s][R][3] float64, a pinned CPU torch
        tensor or a numpy array) and return it at once; the copy overlaps later steps.
        observe_wait() completes it (ens_observe / ens_observe_wait)."""
        if out is None:
            n = C.c_int64()
            check(lib().ens_get_owned(self._ctx, None, C.byref(n)), self._ctx)
            out = np.empty((self.n_s, n.value, 3))
        self._obs_out = out                      # keep the buffer alive while in flight
        check(lib().ens_observe(self._ctx, _ptr(out)), self._ctx)
        return out

    def observe_wait(self) -> int:
        """Block until the last observe() copy is done; returns its step."""
        st = C.c_int64()
        check(lib().ens_observe_wait(self._ctx, C.byref(st)), self._ctx)
        return st.value

    def set_state(self, u_n=None, u_nm1=None, step=0):
        u_n = None if u_n is None else _c(u_n, np.float64)
        u_nm1 = None if u_nm1 is None else _c(u_nm1, np.float64)
        check(lib().ens_set_state(self._ctx, _p(u_n), _p(u_nm1), 0.0, int(step)), self._ctx)
        if getattr(self, "_p2p_multi", False):
            import torch.distributed as dist      # neighbours must not step before every reset
            dist.barrier(group=self._p2p_group)

    def apply_stiffness(self, u):
        u = _c(u, np.float64)
        n = C.c_int64()
        check(lib().ens_get_owned(self._ctx, None, C.byref(n)), self._ctx)
        y = np.empty((u.shape[0], n.value, 3))
        check(lib().ens_apply_stiffness(self._ctx, _p(u), _p(y)), self._ctx)
        return y

    def stress(self, frame: int = 1, centerline=None, per_realisation: bool = True, stats: bool = True):
        """Element stresses of u_n (ens_stress): dict with 'sigma' [n_s][F][6] and/or
        'mean', 'q05', 'q95' [F][6]."""
        F = int(self.info()["n_tris"])
        cl = None if centerline is None else _c(centerline, np.float64)
        out = {}
        sig = np.empty((self.n_s, F, 6)) if per_realisation else None
        st = [np.empty((F, 6)) for _ in range(3)] if stats else [None] * 3
        check(lib().ens_stress(self._ctx, int(frame), _p(cl), 0 if cl is None else cl.shape[0], _p(sig),
                               *[_p(a) for a in st]), self._ctx)
        if per_realisation:
            out["sigma"] = sig
        if stats:
            out["mean"], out["q05"], out["q95"] = st
        return out

    def displacement_stats(self):
        """(mean, q05, q95), each [V][4] = (u_x, u_y, u_z, |u|) over the realisations."""
        st = [np.empty((self.V, 4)) for _ in range(3)]
        check(lib().ens_displacement_stats(self._ctx, *[_p(a) for a in st]), self._ctx)
        return tuple(st)

    def info(self) -> dict:
        inf = _ffi.EnsInfo()
        check(lib().ens_query(self._ctx, C.byref(inf)), self._ctx)
        return {k: getattr(inf, k) for k, _ in _ffi.EnsInfo._fields_}


def _ptr(a):
    """Host pointer of a numpy array or a (pinned) CPU torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous and a.dtype == np.float64
        return a.ctypes.data_as(C.c_void_p)
    assert a.is_contiguous() and a.device.type == "cpu"
    return C.c_void_p(a.data_ptr())


def _options(dt, cfl_safety, c_d, damping, kernel, dist, rank, world, device, stream, torch_alloc):
    opt = _ffi.EnsOptions()
    opt.dt = float(dt or 0.0)
    opt.cfl_safety = float(cfl_safety)
    opt.c_d = float(c_d)
    opt.damping = DAMPING[damping]
    opt.kernel = KERNEL[kernel]
    opt.dist = DIST[dist]
    opt.rank, opt.world = int(rank), int(world)
    opt.device = -1 if device is None else int(device)
    alloc = None
    if stream is not None:
        opt.stream = C.c_void_p(int(stream))
    if torch_alloc:
        import torch
        if torch.cuda.is_available():
            dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
            if stream is None:
                opt.stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
            alloc = _TorchAllocator(dev)
            opt.dev_alloc = alloc.alloc_cb
            opt.dev_free = alloc.free_cb
    return opt, alloc


# ---- host-side maps (no GPU) ----------------------------------------------------------

def host_validate(xyz, tris):
    xyz, tris = _c(xyz, np.float64), _c(tris, np.int32)
    code, bad = C.c_int32(), C.c_int64()
    lib().ens_host_validate(xyz.shape[0], tris.shape[0], _p(xyz), _p(tris), C.byref(code), C.byref(bad))
    return code.value, bad.value


def host_pattern(V, tris):
    """(perm, row_ptr, col) exactly as ens_create builds them."""
    tris = _c(tris, np.int32)
    perm = np.zeros(V, np.int32)
    row_ptr = np.zeros(V + 1, np.int64)
    cap = V + 6 * tris.shape[0]
    col = np.zeros(cap, np.int32)
    n = C.c_int64()
    check(lib().ens_host_pattern(V, tris.shape[0], _p(tris), _p(perm), _p(row_ptr), _p(col), cap, C.byref(n)))
    return perm, row_ptr, col[:n.value].copy()


def host_partition(row_ptr, P):
    row_ptr = _c(row_ptr, np.int64)
    b = np.zeros(P + 1, np.int64)
    check(lib().ens_host_partition(len(row_ptr) - 1, _p(row_ptr), P, _p(b)))
    return b


def host_ghosts(row_ptr, col, lo, hi):
    row_ptr, col = _c(row_ptr, np.int64), _c(col, np.int32)
    V = len(row_ptr) - 1
    g = np.zeros(V, np.int32)
    n = C.c_int64()
    check(lib().ens_host_ghosts(V, _p(row_ptr), _p(col), int(lo), int(hi), _p(g), V, C.byref(n)))
    return g[:n.value].copy()


def host_mf_tiles(xyz, tris, n_s, patches=True, max_rows=32, stage_bytes=0):
    """The STAGED matrix-free tiling of the whole row range (ens_host_mf_tiles): returns
    (tile_of[V] in RCM order, tile_bytes[n_tiles], tile_entries[n_tiles], budget)."""
    xyz, tris = _c(xyz, np.float64), _c(tris, np.int32)
    V = xyz.shape[0]
    tile_of = np.empty(V, np.int32)
    tb = np.empty(V, np.int64)
    te = np.empty(V, np.int32)
    n, budget = C.c_int64(), C.c_int64()
    check(lib().ens_host_mf_tiles(V, tris.shape[0], _p(xyz), _p(tris), int(n_s), int(bool(patches)), int(max_rows),
                                  int(stage_bytes), _p(tile_of), _p(tb), _p(te), C.byref(n), C.byref(budget)))
    return tile_of, tb[:n.value].copy(), te[:n.value].copy(), budget.value


def host_element_stiffness(xyz, tris, nu, k_shear):
    xyz, tris = _c(xyz, np.float64), _c(tris, np.int32)
    F = tris.shape[0]
    K = np.zeros((F, 9, 9))
    A = np.zeros(F)
    check(lib().ens_host_element_stiffness(xyz.shape[0], F, _p(xyz), _p(tris), nu, k_shear, _p(K), _p(A)))
    return K, A


def host_materials(xyz, tris, E, h, rho, cfl_safety=0.9):
    xyz, tris, E, h = _c(xyz, np.float64), _c(tris, np.int32), _c(E, np.float64), _c(h, np.float64)
    n_s, V, F = E.shape[0], xyz.shape[0], tris.shape[0]
    alpha = np.zeros((n_s, F))
    mass = np.zeros((n_s, V))
    dt = C.c_double()
    check(lib().ens_host_materials(V, F, _p(xyz), _p(tris), n_s, _p(E), _p(h), rho, cfl_safety,
                                   _p(alpha), _p(mass), C.byref(dt)))
    return alpha, mass, dt.value


def host_halo_plan(row_ptr, col, P, part):
    """Halo plan of `part` (ens_host_halo_plan): dict lo, hi, b_lo, b_hi, n_ghost, peers
    [(q, send_off, send_n, recv_row, recv_n)], send_rows."""
    row_ptr, col = _c(row_ptr, np.int64), _c(col, np.int32)
    V = len(row_ptr) - 1
    lhb = np.zeros(5, np.int64)
    peers = np.zeros(P, np.int32)
    info = np.zeros((P, 4), np.int64)
    cap = V
    send = np.zeros(cap, np.int32)
    npe, ns = C.c_int64(), C.c_int64()
    check(lib().ens_host_halo_plan(V, _p(row_ptr), _p(col), P, part, _p(lhb), _p(peers), _p(info), _p(send),
                                   cap, C.byref(npe), C.byref(ns)))
    return {"lo": int(lhb[0]), "hi": int(lhb[1]), "b_lo": int(lhb[2]), "b_hi": int(lhb[3]),
            "n_ghost": int(lhb[4]),
            "peers": [(int(peers[k]), *map(int, info[k])) for k in range(npe.value)],
            "send_rows": send[:ns.value].copy()}


def nccl_comm_of(group=None, device=None) -> int:
    """ncclComm_t (as an int) of torch's ProcessGroupNCCL for `group` (default group): the
    communicator ENS_DIST_NODE exchanges its halo on.  The group must be initialised with
    device_id (eager NCCL init) or have run a collective."""
    import torch
    import torch.distributed as dist
    pg = group or dist.distributed_c10d._get_default_group()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    return int(pg._get_backend(dev)._comm_ptr())


def measure_fp64_tflops(device=None) -> float:
    """Measured FP64 FMA throughput of the device (ens_measure_fp64), TFLOP/s."""
    v = C.c_double()
    check(lib().ens_measure_fp64(-1 if device is None else int(device), C.byref(v)))
    return v.value


def matern_fields(xyz, tris, rho_corr, z, tol=1e-13, max_iter=5000, device=None):
    """GPU GMRF draws x[k] = A^-1 C~^{1/2} z[k] / sigma (ens_matern_fields); z [n][V]."""
    xyz, tris, z = _c(xyz, np.float64), _c(tris, np.int32), _c(z, np.float64)
    mesh = _ffi.EnsMesh(xyz.shape[0], tris.shape[0], _p(xyz), _p(tris), None)
    opt, alloc = _options(0.0, 0.9, 0.0, 0, 0, 0, 0, 1, device, None, True)
    x = np.empty_like(z)
    it, res = C.c_int32(), C.c_double()
    check(lib().ens_matern_fields(C.byref(mesh), float(rho_corr), z.shape[0], _p(z), _p(x), float(tol),
                                  int(max_iter), C.byref(opt), C.byref(it), C.byref(res)))
    return x, it.value, res.value
