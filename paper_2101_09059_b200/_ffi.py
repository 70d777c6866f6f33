"""ctypes declarations of include/ens.h (argument marshalling only).

Loads paper_2101_09059_b200/libens.so — the sm_100a library.  There is no fallback:
if the library is missing or cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ENS_LIB_PATH") or os.path.join(_HERE, "libens.so")   # override: A/B builds only

ENS_OK, ENS_E_ARG, ENS_E_MESH, ENS_E_OOM, ENS_E_CUDA, ENS_E_NCCL, ENS_E_DIVERGED, ENS_E_STATE, \
    ENS_E_UNSUPPORTED = 0, -1, -2, -3, -4, -5, -6, -7, -8
ERROR_NAMES = {ENS_E_ARG: "ENS_E_ARG", ENS_E_MESH: "ENS_E_MESH", ENS_E_OOM: "ENS_E_OOM",
               ENS_E_CUDA: "ENS_E_CUDA", ENS_E_NCCL: "ENS_E_NCCL", ENS_E_DIVERGED: "ENS_E_DIVERGED",
               ENS_E_STATE: "ENS_E_STATE", ENS_E_UNSUPPORTED: "ENS_E_UNSUPPORTED"}

DEV_ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
DEV_FREE = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class EnsMesh(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_tris", C.c_int64), ("xyz", C.c_void_p),
                ("tris", C.c_void_p), ("fixed", C.c_void_p)]


class EnsMaterials(C.Structure):
    _fields_ = [("n_s", C.c_int32), ("E", C.c_void_p), ("h", C.c_void_p), ("rho", C.c_double),
                ("nu", C.c_double), ("k_shear", C.c_double), ("s_begin", C.c_int32)]


class EnsOptions(C.Structure):
    _fields_ = [("dt", C.c_double), ("cfl_safety", C.c_double), ("c_d", C.c_double),
                ("damping", C.c_int32), ("kernel", C.c_int32), ("dist", C.c_int32),
                ("rank", C.c_int32), ("world", C.c_int32), ("nccl_comm", C.c_void_p),
                ("stream", C.c_void_p), ("dev_alloc", DEV_ALLOC), ("dev_free", DEV_FREE),
                ("alloc_user", C.c_void_p), ("device", C.c_int32), ("reassemble_every", C.c_int32),
                ("halo", C.c_int32), ("p2p_procs", C.c_int32), ("mf_variant", C.c_int32),
                ("persistent", C.c_int32)]


class EnsInfo(C.Structure):
    _fields_ = [("dt", C.c_double), ("dt_cfl", C.c_double), ("n_nodes", C.c_int64),
                ("n_tris", C.c_int64), ("nnzb", C.c_int64), ("n_s", C.c_int32),
                ("kernel", C.c_int32), ("damping", C.c_int32), ("dist", C.c_int32),
                ("step", C.c_int64), ("bytes_per_step", C.c_int64), ("flops_per_step", C.c_int64),
                ("device_bytes", C.c_int64), ("rcm_bandwidth", C.c_int32),
                ("n_owned", C.c_int64), ("halo_bytes_per_step", C.c_int64),
                ("launches_per_step", C.c_int32), ("reassemble_every", C.c_int32), ("graph_steps", C.c_int32),
                ("halo", C.c_int32), ("mf_variant", C.c_int32), ("comm_rank", C.c_int32),
                ("comm_nranks", C.c_int32), ("mfs_consumers", C.c_int32), ("mfs_unit_width", C.c_int32),
                ("mfs_stage_width", C.c_int32), ("mfs_stages", C.c_int32)]


EXPORTS = [
    "ens_create", "ens_set_traction", "ens_step", "ens_prepare", "ens_sync", "ens_get_state", "ens_set_state",
    "ens_apply_stiffness", "ens_query", "ens_destroy", "ens_last_error", "ens_host_validate",
    "ens_host_pattern", "ens_host_partition", "ens_host_ghosts", "ens_host_element_stiffness",
    "ens_host_materials", "ens_create_csr", "ens_get_owned", "ens_host_halo_plan", "ens_stress",
    "ens_displacement_stats", "ens_matern_fields", "ens_p2p_export", "ens_p2p_connect", "ens_observe",
    "ens_observe_wait", "ens_measure_fp64", "ens_host_mf_tiles",
]
P2P_BLOB_BYTES = 256

_lib = None


class EnsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


def lib():
    """Load libens.so (building it first if the sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    if LIB_PATH == _build.LIB and _build.stale() and os.path.exists(_build.NVCC):
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "ens_create": (C.c_int, [P(EnsMesh), P(EnsMaterials), P(EnsOptions), P(vp)]),
        "ens_set_traction": (C.c_int, [vp, i32, vp, i32, vp, vp, f64, f64]),
        "ens_step": (C.c_int, [vp, i64]),
        "ens_prepare": (C.c_int, [vp]),
        "ens_sync": (C.c_int, [vp]),
        "ens_get_state": (C.c_int, [vp, vp, vp, P(f64), P(i64)]),
        "ens_set_state": (C.c_int, [vp, vp, vp, f64, i64]),
        "ens_apply_stiffness": (C.c_int, [vp, vp, vp]),
        "ens_query": (C.c_int, [vp, P(EnsInfo)]),
        "ens_destroy": (None, [vp]),
        "ens_last_error": (C.c_char_p, [vp]),
        "ens_host_validate": (C.c_int, [i64, i64, vp, vp, P(i32), P(i64)]),
        "ens_host_pattern": (C.c_int, [i64, i64, vp, vp, vp, vp, i64, P(i64)]),
        "ens_host_partition": (C.c_int, [i64, vp, i32, vp]),
        "ens_host_ghosts": (C.c_int, [i64, vp, vp, i64, i64, vp, i64, P(i64)]),
        "ens_host_element_stiffness": (C.c_int, [i64, i64, vp, vp, f64, f64, vp, vp]),
        "ens_host_materials": (C.c_int, [i64, i64, vp, vp, i32, vp, vp, f64, f64, vp, vp, P(f64)]),
        "ens_create_csr": (C.c_int, [i64, vp, vp, i32, vp, vp, vp, vp, vp, f64, P(EnsOptions), P(vp)]),
        "ens_get_owned": (C.c_int, [vp, vp, P(i64)]),
        "ens_stress": (C.c_int, [vp, i32, vp, i32, vp, vp, vp, vp]),
        "ens_displacement_stats": (C.c_int, [vp, vp, vp, vp]),
        "ens_matern_fields": (C.c_int, [P(EnsMesh), f64, i32, vp, vp, f64, i32, P(EnsOptions), P(i32), P(f64)]),
        "ens_host_halo_plan": (C.c_int, [i64, vp, vp, i32, i32, vp, vp, vp, vp, i64, P(i64), P(i64)]),
        "ens_p2p_export": (C.c_int, [vp, vp]),
        "ens_p2p_connect": (C.c_int, [vp, vp]),
        "ens_observe": (C.c_int, [vp, vp]),
        "ens_observe_wait": (C.c_int, [vp, P(i64)]),
        "ens_measure_fp64": (C.c_int, [i32, P(f64)]),
        "ens_host_mf_tiles": (C.c_int, [i64, i64, vp, vp, i32, i32, i32, i64, vp, vp, vp, P(i64), P(i64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int, ctx=None):
    if rc != ENS_OK:
        msg = lib().ens_last_error(ctx)
        raise EnsError(rc, msg.decode() if msg else "")
    return rc
