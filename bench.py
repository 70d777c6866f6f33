#!/usr/bin/env python
"""Benchmark of the fused ensemble step (arXiv 2101.09059 hot path) on B200.

    python bench.py [--gpus N --steps K --warmup W --config c2 --kernel assembled_sym|assembled|matrix_free]
    python bench.py --impl reference ...        # the CPU oracle, timed on the host cores

One "step" = one explicit central-difference step of all N_s realisations (S2 load +
S3 ensemble SpMM + S4 update, one fused kernel launch).  Default kernel: the assembled
per-realisation block-CSR values in symmetric half storage (a1s, the fastest assembled
path); the full-storage a1 and the matrix-free a2 are timed alongside ("alternatives").  Metric (BASELINE.json):
ensemble DOF-updates/s = N_s * 3V * steps / time, plus the fused step's HBM GB/s against
the measured peak.  Multi-GPU (torchrun): ensemble sharding, N_s per GPU fixed (weak
scaling), no collective on the data path; timing = max over ranks (CUDA events).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# the device function each --kernel runs (matrix-free: the data path the library chose,
# ens_info.mf_variant)
_KERNEL_FN = {"assembled": lambda info: "k_step_assembled",
              "assembled_sym": lambda info: "k_step_assembled_sym",
              "matrix_free": lambda info: {1: "k_step_matrix_free", 2: "k_step_mf_warp",
                                           3: "k_step_mf_staged"}.get(info.get("mf_variant"), "?")}
METRIC = ("ensemble DOF-updates/s (N_s×DOF×steps/s) and fused-step HBM GB/s vs peak")
FALLBACK_HBM_GBS = 6650.0      # /opt/skills/guides/B200_PROFILING.md fallback


def _workload_desc(cfg, n_s_total, world):
    m = cfg.mesh
    geo = (f"ideal cylinder D=4 L=30 cm, {m.meta['n_circ']}x{m.meta['n_axial']} rings"
           if m.meta.get("kind") == "cylinder" else "synthetic branched aorta (7 branches)")
    return (f"{cfg.name}: {geo} "
            f"(V={m.n_nodes}, F={m.n_tris}), N_s={n_s_total} ({cfg.n_s}/GPU), "
            + ("steady 13 mmHg" if len(cfg.traction.tab_t) == 0 else "pulsatile 13+27 mmHg")
            + (f", mode-1 damping {cfg.c_d:g}/s" if cfg.damping == 1 else ", undamped"))


def _peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during the timed region."""

    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
             "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.NAMES.items():
                    if r & getattr(nv, attr, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _max_over_ranks(x: float) -> float:
    """Max of a host float over the ranks (NCCL: a CUDA tensor; gloo: a CPU tensor)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _launch_count(n: int, G: int) -> int:
    """Kernels ens_step(n) enqueues: n fused steps + one counter advance per graph replay
    (G steps each) and one for the directly launched remainder."""
    if G > 0 and n >= G:
        q, r = divmod(n, G)
        return q * (G + 1) + (r + 1 if r else 0)
    return n + (1 if n else 0)


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cpu_baseline(cfg, budget_s: float = 12.0, max_steps: int = 40):
    """The oracle as it stands (oracle/oracle.c), timed on this host's cores on a bounded
    sample of the same workload: the same mesh and all N_s realisations, a few steps."""
    cores = len(os.sched_getaffinity(0))
    import oracle
    cores = oracle.set_threads(cores)        # torchrun exports OMP_NUM_THREADS=1: override
    m = cfg.mesh
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu,
                            k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d)
    tr = cfg.traction
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.run(1)
    n, t0 = 0, time.perf_counter()
    while n < max_steps and time.perf_counter() - t0 < budget_s:
        om.run(1)
        n += 1
    el = time.perf_counter() - t0
    return {"value": cfg.n_s * 3 * m.n_nodes * n / el, "unit": "DOF-updates/s",
            "cores": cores, "kind": "oracle",
            "sample": f"{cfg.name} mesh, all {cfg.n_s} realisations, {n} steps ({el:.1f} s)",
            "s_per_step": el / n}


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    from paper_2101_09059_b200.inputs import configs
    cfg = configs.make(args.config, n_s=args.n_s)
    # each "step" of this arm is one oracle time step on the full workload (bounded: the
    # oracle steps a few hundred ms per step on 16 cores)
    import oracle
    cores = oracle.set_threads(len(os.sched_getaffinity(0)))   # all host cores (torchrun sets 1)
    m = cfg.mesh
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu,
                            k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d)
    tr = cfg.traction
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.run(args.warmup)
    t0 = time.perf_counter()
    om.run(args.steps)
    el = time.perf_counter() - t0
    value = cfg.n_s * 3 * m.n_nodes * args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "DOF-updates/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload_desc(cfg, cfg.n_s, 1), "impl_detail": "oracle/oracle.c, OpenMP over realisations"},
            "cpu_baseline": {"value": value, "unit": "DOF-updates/s", "cores": cores,
                             "kind": "oracle", "sample": f"{cfg.name}, all {cfg.n_s} realisations, {args.steps} steps"},
            "e2e": {"value": value, "unit": "DOF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _node_partition_run(args, cfg, base, m, tr, rank, world, local, stream, barrier, n_s, halo):
    """Node partition (strong scaling of the full config): every rank holds the same N_s
    realisations, the RCM rows are split across ranks; halo "nccl" = NCCL send/recv of the
    packed interface rows, "p2p" = device-initiated stores into the neighbours' ghost rows
    over NVLink (CUDA IPC) with step flags, graph-captured."""
    import torch
    from paper_2101_09059_b200 import solver
    extra = dict(nccl_comm=solver.nccl_comm_of()) if halo == "nccl" else dict(halo="p2p", p2p_procs=True)
    npar = solver.Ensemble(m.xyz, m.tris, m.fixed, base.E, base.h, rho=cfg.rho, nu=cfg.nu,
                           k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d,
                           kernel=args.kernel, dist="node", rank=rank, world=world,
                           device=local, **extra)
    npar.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    npar.step(max(3, args.warmup))
    npar.sync()
    barrier()
    n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0.record(stream)
    npar.step(args.steps)
    n1.record(stream)
    n1.synchronize()
    barrier()
    npar.sync()
    tmax = _max_over_ranks(n0.elapsed_time(n1) / 1e3)
    ninf = npar.info()
    node = {"value": n_s * 3 * m.n_nodes * args.steps / tmax, "unit": "DOF-updates/s",
            "ms_per_step": 1e3 * tmax / args.steps, "scaling": "strong",
            "n_s_total": n_s, "rows_rank0": ninf["n_owned"],
            "halo_bytes_per_step_rank0": ninf["halo_bytes_per_step"],
            "launches_per_step": ninf["launches_per_step"], "halo": halo,
            "graph_steps": ninf["graph_steps"]}
    npar.close()

    return node


def _emulated_partition_run(args, cfg, m, tr, local, stream, halo, single_value):
    """ENS_DIST_NODE with all P parts in this one context on this one GPU: the per-step cost
    of the partitioned schedule (boundary / interior launches, halo by device copies or by
    the P2P forwarding stores + step flags) against the unpartitioned step.  Not a
    multi-GPU number: the parts run one after another on the same device."""
    import torch
    from paper_2101_09059_b200 import solver
    P = args.emulate_partition
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu, k_shear=cfg.k_shear,
                          damping=cfg.damping, c_d=cfg.c_d, kernel=args.kernel, dist="node", world=P, halo=halo,
                          device=local)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(max(3, args.warmup))
    ens.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ens.step(args.steps)
    e1.record(stream)
    e1.synchronize()
    el = e0.elapsed_time(e1) / 1e3
    inf = ens.info()
    ens.close()
    v = cfg.n_s * 3 * m.n_nodes * args.steps / el
    return {"value": v, "unit": "DOF-updates/s", "ms_per_step": 1e3 * el / args.steps,
            "of_unpartitioned": v / single_value, "launches_per_step": inf["launches_per_step"],
            "graph_steps": inf["graph_steps"], "halo_bytes_per_step": inf["halo_bytes_per_step"]}


def _read_stream_gbs(gib: float = 4.0, reps: int = 10) -> float:
    """Practical ceiling of a read-dominated kernel on this box: torch.sum over a 4 GiB fp64
    tensor, best of `reps`, CUDA events."""
    import torch
    x = torch.ones(int(gib * (1 << 30)) // 8, dtype=torch.float64, device="cuda")
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x.sum()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    n = x.numel() * 8
    del x
    torch.cuda.empty_cache()
    return n / best / 1e9


def _time_kernel(kernel, args, cfg, m, tr, world, rank, local, stream, barrier, peak):
    """Time `kernel` on the same workload exactly like the headline (CUDA events around
    ens_step(K) on the context stream, max over ranks)."""
    import torch
    from paper_2101_09059_b200 import solver
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu,
                          k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d, kernel=kernel,
                          dist="ensemble" if world > 1 else "single", s_begin=cfg.s_begin,
                          rank=rank, world=world, device=local)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    info = ens.info()
    ens.step(max(3, args.warmup))
    ens.sync()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ens.step(args.steps)
    e1.record(stream)
    e1.synchronize()
    barrier()
    ens.sync()
    el = e0.elapsed_time(e1) / 1e3
    el = _max_over_ranks(el)
    ens.close()
    ach = info["bytes_per_step"] / (el / args.steps) / 1e9
    tf = info["flops_per_step"] / (el / args.steps) / 1e12
    return {"value": world * cfg.n_s * 3 * m.n_nodes * args.steps / el, "unit": "DOF-updates/s",
            "ms_per_step": 1e3 * el / args.steps, "achieved_GBs": ach, "frac": ach / peak,
            "algorithmic_bytes_per_launch": info["bytes_per_step"], "achieved_fp64_TFLOPs": tf,
            "kernel_fn": _KERNEL_FN[kernel](info),
            "algorithmic_flops_per_launch": info["flops_per_step"]}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--n-s", type=int, default=None, help="realisations per GPU (default: the config's)")
    ap.add_argument("--kernel", default="assembled_sym", choices=["assembled", "assembled_sym", "matrix_free"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alternatives", action="store_true", help="do not time the other kernels")
    ap.add_argument("--node-partition", action="store_true",
                    help="at N > 1 also time ENS_DIST_NODE (RCM rows split; NCCL and P2P halos; strong scaling)")
    ap.add_argument("--emulate-partition", type=int, default=0,
                    help="at N = 1 also time ENS_DIST_NODE with this many parts in one context (schedule overhead)")
    ap.add_argument("--e2e-windows", type=int, default=10)
    ap.add_argument("--obs-every", type=int, default=100)
    args = ap.parse_args(argv)
    if args.impl == "reference":
        if args.steps > 50:          # the driver's K for our arm; the oracle is ~10^3x slower
            args.steps, args.warmup = 5, 1
        return run_reference(args)

    import torch
    world, rank, local = _dist()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    # one process per GPU; ENS_BENCH_BACKEND=gloo lets several ranks share one device to
    # exercise the multi-process plumbing on a single-GPU box (timings then meaningless)
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("ENS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2101_09059_b200 import solver
    from paper_2101_09059_b200.inputs import configs
    base = configs.make(args.config, n_s=args.n_s, n_circ=None)
    n_s = base.n_s
    cfg = configs.make(args.config, n_s=n_s, s_begin=rank * n_s) if world > 1 else base
    m = cfg.mesh
    stream = torch.cuda.current_stream()
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu,
                          k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d, kernel=args.kernel,
                          dist="ensemble" if world > 1 else "single", s_begin=cfg.s_begin,
                          rank=rank, world=world, device=local)
    tr = cfg.traction
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    info = ens.info()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    ens.step(max(3, args.warmup))
    ens.sync()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        ens.step(args.steps)
        e1.record(stream)
        e1.synchronize()
    barrier()
    ens.sync()                                   # raises on divergence
    el = e0.elapsed_time(e1) / 1e3
    el_max = _max_over_ranks(el)
    dof_updates = world * n_s * 3 * m.n_nodes * args.steps
    value = dof_updates / el_max
    per_launch = el / args.steps
    peak, peak_src = _peak_hbm()
    achieved = info["bytes_per_step"] / per_launch / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        key = f"{args.config}/{args.kernel}/{n_s}"
        traffic = tj.get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        pass

    # end to end through the public API with host buffers: per observation window of
    # obs_every steps, H2D of the traction (from pinned memory, ens_set_traction's
    # asynchronous same-shape update) + the steps + D2H of u_n into pinned memory
    # (ens_observe: the copy of window w overlaps the steps of window w + 1; the last one
    # is waited for inside the timed region)
    Fp = torch.from_numpy(np.ascontiguousarray(tr.F)).pin_memory()
    outs = [torch.empty((n_s, m.n_nodes, 3), dtype=torch.float64).pin_memory() for _ in range(2)]
    out = outs[0]
    win = args.obs_every
    barrier()
    t0 = time.perf_counter()
    for w in range(args.e2e_windows):
        ens.set_traction(Fp.numpy(), tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        ens.step(win)
        if w > 0:
            ens.observe_wait()
        ens.observe(outs[w % 2])
    ens.observe_wait()
    e2e_el = time.perf_counter() - t0
    e2e_el = _max_over_ranks(e2e_el)
    e2e_value = world * n_s * 3 * m.n_nodes * win * args.e2e_windows / e2e_el
    h2d = Fp.numel() * 8 + tr.tab_t.size * 8 + tr.tab_g.size * 8
    d2h = out.numel() * 8

    # node partition (strong scaling of the full config): the same N_s realisations on
    # every rank, RCM rows split across ranks, NCCL halo of the interface rows per step
    node = None
    if world > 1 and args.node_partition:
        node = {}
        for halo in ("nccl", "p2p"):
            try:
                node[halo] = _node_partition_run(args, cfg, base, m, tr, rank, world, local, stream, barrier,
                                                 n_s, halo)
            except Exception as e:      # reported, never fatal for the primary (sharded) line
                node[halo] = {"error": repr(e)[:300]}
    elif world == 1 and args.emulate_partition > 1:
        node = {"emulated_parts": args.emulate_partition}
        for halo in ("nccl", "p2p"):
            try:
                node[halo] = _emulated_partition_run(args, cfg, m, tr, local, stream, halo, value)
            except Exception as e:
                node[halo] = {"error": repr(e)[:300]}

    # the other kernels of the same step, same inputs, same launch protocol (reported
    # alongside; the headline is --kernel)
    alts = {}
    if not args.no_alternatives:
        for k in ("assembled", "assembled_sym", "matrix_free"):
            if k == args.kernel:
                continue
            try:
                alts[k] = _time_kernel(k, args, cfg, m, tr, world, rank, local, stream, barrier, peak)
            except Exception as e:
                alts[k] = {"error": repr(e)[:200]}

    read_gbs = _read_stream_gbs() if rank == 0 else None
    try:                         # FP64 FMA probe: the ALU roofline
        from paper_2101_09059_b200 import solver as _solver
        fp64_peak = _solver.measure_fp64_tflops(local) if rank == 0 else None
    except Exception:
        fp64_peak = None
    if fp64_peak:
        for a in alts.values():
            if "achieved_fp64_TFLOPs" in a:
                a["fp64_frac"] = a["achieved_fp64_TFLOPs"] / fp64_peak
    tf_head = info["flops_per_step"] / (el_max / args.steps) / 1e12

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(base)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "DOF-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": _workload_desc(cfg, world * n_s, world), "kernel": args.kernel,
                       "n_s_per_gpu": n_s, "V": m.n_nodes, "F": m.n_tris, "nnzb": info["nnzb"],
                       "dt": info["dt"], "parallelism": f"ensemble-shard x{world}",
                       "l2": f"inputs larger than L2: {info['bytes_per_step'] / 1e9:.3f} GB streamed per step vs 126 MB L2 (no flush)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": _KERNEL_FN[args.kernel](info),
                         "algorithmic_bytes_per_launch": info["bytes_per_step"],
                         "read_stream_GBs": read_gbs, "frac_of_read_stream": achieved / read_gbs if read_gbs else None,
                         "fp64": {"achieved_TFLOPs": tf_head, "peak_TFLOPs": fp64_peak,
                                  "peak_source": "measured (ens_measure_fp64: DFMA probe, this run)",
                                  "frac": tf_head / fp64_peak if fp64_peak else None}},
            "cpu_baseline": cpu,
            "alternatives": alts,
            "node_partition": node,
            "e2e": {"value": e2e_value, "unit": "DOF-updates/s", "h2d_bytes_per_step": h2d / win,
                    "d2h_bytes_per_step": d2h / win,
                    "window": f"{win} steps + ens_set_traction (H2D {h2d} B) + ens_observe u_n (D2H {d2h} B, overlapped with the next window)"},
            "gpu_launches": _launch_count(args.steps, info.get("graph_steps", 0)),
            "clocks": clk.summary(),
            "paper_best_context": {"value": 7.27e8, "unit": "DOF-updates/s",
                                   "hardware": "4x RTX 2080 Ti, OpenCL, 131,552-tri cylinder, 500 realisations (PAPER.md:665)"},
        }
        print(json.dumps(line), flush=True)
    ens.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
