#!/usr/bin/env python
"""Benchmark of the fused ensemble step (arXiv 2101.09059 hot path) on B200.

    python bench.py [--gpus N --steps K --warmup W --config c4 --kernel assembled_sym|assembled|matrix_free]
    python bench.py --impl reference ...        # the CPU oracle, timed on the host cores

One "step" = one explicit central-difference step of all N_s realisations (S2 load +
S3 ensemble SpMM + S4 update, one fused kernel launch).  Workload: config c4 by default, the
largest BASELINE.json configuration that fits one GPU (synthetic branched aorta, ~500k
triangles, N_s = 128, pulsatile traction).  Default kernel: the assembled per-realisation
block-CSR values in symmetric half storage (a1s); the full-storage a1 and the matrix-free a2
(warp-specialised tile stages) are timed alongside ("alternatives"), and so is the c2
cylinder.  Metric (BASELINE.json): ensemble DOF-updates/s = N_s * 3V * steps / time, plus
the fused step's HBM GB/s against the measured peak.
Multi-GPU (torchrun): the RCM rows of the same workload are split across the ranks (node
partition, strong scaling) with the halo of the interface rows exchanged every step by NCCL
send/recv (or, with ENS_BENCH_BACKEND=gloo, by device-initiated P2P stores through CUDA IPC);
the communication-free ensemble sharding (weak scaling) is reported alongside.  Timing =
max over ranks of CUDA-event time.
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

    def __init__(self, device_index: int, period_s: float = 0.005):
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


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_rate(cfg, idx, threads: int, steps: int = 5):
    """The oracle (oracle/oracle.c, as it stands) on realisations idx of cfg with `threads`
    OpenMP threads: median over `steps` individually timed steps (after one untimed)."""
    import oracle
    used = oracle.set_threads(threads)
    m = cfg.mesh
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E[idx], cfg.h[idx], rho=cfg.rho, nu=cfg.nu,
                            k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d)
    tr = cfg.traction
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.run(1)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        om.run(1)
        ts.append(time.perf_counter() - t0)
    per = statistics.median(ts)
    return len(idx) * 3 * m.n_nodes / per, per, used


def _cpu_baseline(cfg):
    """The oracle timed on this host: all cores on all N_s realisations, and one core on a
    subset of 8 (the rate in DOF-updates/s does not depend on how many realisations)."""
    cores = len(os.sched_getaffinity(0))
    v_all, per_all, used = _oracle_rate(cfg, list(range(cfg.n_s)), cores)
    v_one, per_one, _ = _oracle_rate(cfg, list(range(min(8, cfg.n_s))), 1)
    import oracle
    oracle.set_threads(cores)
    return {"value": v_all, "unit": "DOF-updates/s", "cores": used, "kind": "oracle",
            "sample": (f"{cfg.name} mesh (V={cfg.mesh.n_nodes}), all {cfg.n_s} realisations, median of 5 "
                       f"timed steps ({per_all:.3f} s/step on {used} threads); 1 core: 8 realisations, "
                       f"median of 5 steps ({per_one:.3f} s/step)"),
            "s_per_step": per_all, "one_core": {"value": v_one, "s_per_step": per_one, "realisations": 8},
            "cpu_model": _cpu_model()}


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    from paper_2101_09059_b200.inputs import configs
    cfg = configs.make(args.config, n_s=args.n_s)
    # each "step" of this arm is one oracle time step on the full workload (c4: ~0.4 s on 16
    # cores), bounded so that the run ends within a few minutes
    steps, warmup = min(args.steps, 20), min(args.warmup, 2)
    import oracle
    cores = oracle.set_threads(len(os.sched_getaffinity(0)))   # all host cores (torchrun sets 1)
    m = cfg.mesh
    om = oracle.OracleModel(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu,
                            k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d)
    tr = cfg.traction
    om.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    om.run(warmup)
    t0 = time.perf_counter()
    om.run(steps)
    el = time.perf_counter() - t0
    value = cfg.n_s * 3 * m.n_nodes * steps / el
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "DOF-updates/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
            "ms_per_step": 1e3 * el / steps, "higher_is_better": True,
            "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": _workload_desc(cfg, cfg.n_s, 1),
                       "impl_detail": "oracle/oracle.c (plain fp64 C, the CPU reference), OpenMP over realisations"},
            "cpu_baseline": {"value": value, "unit": "DOF-updates/s", "cores": cores, "kind": "oracle",
                             "sample": f"{cfg.name}, all {cfg.n_s} realisations, {steps} steps", "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": "DOF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


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


class Run:
    """One context on this rank: the step timed like the headline (CUDA events around
    ens_step(K) on the context stream, barriers on both sides, max over ranks)."""

    def __init__(self, cfg, kernel, world, rank, local, dist_mode="single", halo="nccl", mf_variant="auto"):
        from paper_2101_09059_b200 import solver
        extra = {}
        if dist_mode == "node" and world > 1:
            extra = dict(nccl_comm=solver.nccl_comm_of()) if halo == "nccl" else dict(halo="p2p", p2p_procs=True)
        m = cfg.mesh
        self.cfg, self.kernel = cfg, kernel
        self.ens = solver.Ensemble(m.xyz, m.tris, m.fixed, cfg.E, cfg.h, rho=cfg.rho, nu=cfg.nu,
                                   k_shear=cfg.k_shear, damping=cfg.damping, c_d=cfg.c_d, kernel=kernel,
                                   dist=dist_mode if world > 1 else "single", s_begin=cfg.s_begin,
                                   rank=rank, world=world if world > 1 else 1, device=local,
                                   mf_variant=mf_variant, **extra)
        tr = cfg.traction
        self.ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        self.info = self.ens.info()

    def time(self, steps, warmup, stream, barrier, clocks=None):
        import torch
        self.ens.prepare()              # step-loop graphs built as setup (ens_prepare), not timed
        self.ens.step(max(3, warmup))
        self.ens.sync()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if clocks:
            clocks.__enter__()
        e0.record(stream)
        self.ens.step(steps)
        e1.record(stream)
        e1.synchronize()
        if clocks:
            clocks.__exit__(None, None, None)
        barrier()
        self.ens.sync()                                   # raises on divergence
        self.el_local = e0.elapsed_time(e1) / 1e3
        self.el = _max_over_ranks(self.el_local)
        return self.el

    def time_median(self, steps, warmup, stream, barrier, reps=3):
        """Alternatives: the median of `reps` timed windows (one window once read 3x slow on
        a box and never again; the headline is always one window of exactly K steps)."""
        els, locs = [], []
        for _ in range(reps):
            els.append(self.time(steps, warmup if not els else 0, stream, barrier))
            locs.append(self.el_local)
        self.el = statistics.median(els)
        self.el_local = statistics.median(locs)
        return self.el

    def close(self):
        self.ens.close()


def _line_item(run, steps, units, peak):
    """Throughput and roofline numbers of a timed Run (units = DOF-updates of all ranks)."""
    info = run.info
    per = run.el / steps
    ach = info["bytes_per_step"] / (run.el_local / steps) / 1e9     # this rank's kernel bytes / its time
    extra = {}
    if info.get("mfs_consumers"):
        extra["staged_shape"] = {k: info[k] for k in ("mfs_consumers", "mfs_unit_width", "mfs_stage_width", "mfs_stages")}
    return {**extra, "value": units / run.el, "unit": "DOF-updates/s", "ms_per_step": 1e3 * per,
            "achieved_GBs": ach, "frac": ach / peak, "algorithmic_bytes_per_launch": info["bytes_per_step"],
            "achieved_fp64_TFLOPs": info["flops_per_step"] / (run.el_local / steps) / 1e12,
            "algorithmic_flops_per_launch": info["flops_per_step"], "kernel_fn": _KERNEL_FN[run.kernel](info)}


def _e2e(run, windows, win, world, barrier):
    """End to end through the public API with host buffers: per window of `win` steps, the
    H2D of the traction from pinned memory (ens_set_traction's asynchronous same-shape
    update), the steps, and the D2H of u_n into pinned memory (ens_observe: window w's copy
    overlaps window w + 1's steps; the last one is waited for inside the timed region)."""
    import torch
    tr = run.cfg.traction
    rows = run.info["n_owned"]
    Fp = torch.from_numpy(np.ascontiguousarray(tr.F)).pin_memory()
    outs = [torch.empty((run.cfg.n_s, rows, 3), dtype=torch.float64).pin_memory() for _ in range(2)]
    barrier()
    t0 = time.perf_counter()
    for w in range(windows):
        run.ens.set_traction(Fp.numpy(), tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
        run.ens.step(win)
        if w > 0:
            run.ens.observe_wait()
        run.ens.observe(outs[w % 2])
    run.ens.observe_wait()
    el = _max_over_ranks(time.perf_counter() - t0)
    h2d = (Fp.numel() + tr.tab_t.size + tr.tab_g.size) * 8
    d2h = outs[0].numel() * 8
    h2d_all, d2h_all = _sum_over_ranks(h2d), _sum_over_ranks(d2h)
    return el, {"h2d_bytes_per_step": h2d_all / win, "d2h_bytes_per_step": d2h_all / win,
                "window": f"{win} steps + ens_set_traction (H2D {h2d} B per rank) + ens_observe u_n "
                          f"(D2H {d2h} B per rank, overlapped with the next window)"}


def _sum_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def _traffic(config, kernel_fn, n_s):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        return tj.get(f"{config}/{kernel_fn}/{n_s}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--n-s", type=int, default=None, help="realisations per GPU (default: the config's)")
    ap.add_argument("--kernel", default="assembled_sym", choices=["assembled", "assembled_sym", "matrix_free"])
    ap.add_argument("--mf-variant", default="auto", choices=["auto", "tiles", "warp", "staged"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alternatives", action="store_true", help="do not time the other kernels / configs")
    ap.add_argument("--emulate-partition", type=int, default=0,
                    help="at N = 1 also time ENS_DIST_NODE with this many parts in one context (schedule overhead)")
    ap.add_argument("--e2e-windows", type=int, default=10)
    ap.add_argument("--obs-every", type=int, default=100)
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world, rank, local = _dist()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    # one process per GPU; ENS_BENCH_BACKEND=gloo lets several ranks share one device to
    # exercise the multi-process plumbing on a single-GPU box (timings then meaningless; the
    # node-partition halo is then the P2P one, NCCL refuses two ranks on one device)
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    backend = os.environ.get("ENS_BENCH_BACKEND", "nccl")
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2101_09059_b200 import solver
    from paper_2101_09059_b200.inputs import configs
    base = configs.make(args.config, n_s=args.n_s)
    n_s = base.n_s
    m = base.mesh
    stream = torch.cuda.current_stream()
    peak, peak_src = _peak_hbm()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    K = args.steps
    alts, node_emul, comm, repeat = {}, None, None, None
    if world == 1:
        # headline: the whole config on this GPU
        head = Run(base, args.kernel, 1, 0, local, mf_variant=args.mf_variant)
        clk = ClockSampler(local)
        head.time(K, args.warmup, stream, barrier, clocks=clk)
        units = n_s * 3 * m.n_nodes * K
        item = _line_item(head, K, units, peak)
        # SURVEY.md §8(d) asks for the median of 5: four more windows of K steps, reported
        # beside the headline (which stays the first window, as the contract times it)
        el0, loc0 = head.el, head.el_local
        wins = [el0]
        for _ in range(4):
            wins.append(head.time(K, 0, stream, barrier))
        head.el, head.el_local = el0, loc0
        repeat = {"ms_per_step": [1e3 * w / K for w in wins], "median_ms_per_step": 1e3 * statistics.median(wins) / K,
                  "median_value": units / statistics.median(wins)}
        scaling, parallelism = "weak", "single GPU"
        e2e_el, e2e_meta = _e2e(head, args.e2e_windows, args.obs_every, world, barrier)
        e2e_units = n_s * 3 * m.n_nodes * args.obs_every * args.e2e_windows
        launches = _launch_count(K, head.info.get("graph_steps", 0))
        head_info = head.info
        head.close()
        if args.emulate_partition > 1:
            node_emul = {"emulated_parts": args.emulate_partition}
            variants = ["nccl", "p2p"] + (["p2p_persistent"] if args.kernel != "matrix_free" else [])
            for halo in variants:
                try:
                    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, base.E, base.h, rho=base.rho, nu=base.nu,
                                          k_shear=base.k_shear, damping=base.damping, c_d=base.c_d,
                                          kernel=args.kernel, dist="node", world=args.emulate_partition,
                                          halo=halo.split("_")[0], persistent=halo.endswith("persistent"),
                                          device=local)
                    r = Run.__new__(Run)
                    r.cfg, r.kernel, r.ens = base, args.kernel, ens
                    tr = base.traction
                    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
                    r.info = ens.info()
                    r.time(K, args.warmup, stream, barrier)
                    node_emul[halo] = {"value": units / r.el, "ms_per_step": 1e3 * r.el / K,
                                       "of_unpartitioned": (units / r.el) / item["value"],
                                       "launches_per_step": r.info["launches_per_step"],
                                       "graph_steps": r.info["graph_steps"]}
                    r.close()
                except Exception as e:
                    node_emul[halo] = {"error": repr(e)[:300]}
        if not args.no_alternatives:
            for k in ("assembled", "assembled_sym", "matrix_free"):
                if k == args.kernel:
                    continue
                try:
                    r = Run(base, k, 1, 0, local)
                    r.time_median(K, args.warmup, stream, barrier)
                    alts[k] = _line_item(r, K, units, peak)
                    r.close()
                except Exception as e:
                    alts[k] = {"error": repr(e)[:200]}
            if args.config != "c2":       # the c2 cylinder (BASELINE configs[1]) alongside
                c2 = configs.make("c2")
                for k in ("assembled_sym", "matrix_free"):
                    try:
                        r = Run(c2, k, 1, 0, local)
                        K2 = max(K, 500)
                        r.time_median(K2, max(args.warmup, 20), stream, barrier)
                        it = _line_item(r, K2, c2.n_s * 3 * c2.mesh.n_nodes * K2, peak)
                        it["workload"] = _workload_desc(c2, c2.n_s, 1)
                        it["steps"] = K2
                        alts[f"c2/{k}"] = it
                        r.close()
                    except Exception as e:
                        alts[f"c2/{k}"] = {"error": repr(e)[:200]}
    else:
        # headline: node partition of the whole config (strong scaling), halo every step
        halo = "nccl" if backend == "nccl" else "p2p"
        try:
            head = Run(base, args.kernel, world, rank, local, dist_mode="node", halo=halo, mf_variant=args.mf_variant)
        except Exception as e:           # never lose the whole line: fall back to the ensemble shard
            print(f"node partition failed ({e!r}); ensemble shard as the headline", file=sys.stderr, flush=True)
            head = None
    if world > 1 and head is None:
        shard = configs.make(args.config, n_s=n_s, s_begin=rank * n_s)
        head = Run(shard, args.kernel, world, rank, local, dist_mode="ensemble")
        clk = ClockSampler(local)
        head.time(K, args.warmup, stream, barrier, clocks=clk)
        units = world * n_s * 3 * m.n_nodes * K
        item = _line_item(head, K, units, peak)
        item.update(rows_rank=head.info["n_owned"], halo="none", halo_bytes_per_step_rank=0,
                    launches_per_step=head.info["launches_per_step"])
        scaling, parallelism = "weak", f"ensemble shard x{world} (node partition failed)"
        e2e_el, e2e_meta = _e2e(head, args.e2e_windows, args.obs_every, world, barrier)
        e2e_units = world * n_s * 3 * m.n_nodes * args.obs_every * args.e2e_windows
        launches = _launch_count(K, head.info.get("graph_steps", 0))
        head_info = head.info
        head.close()
    elif world > 1:
        if head.info.get("comm_nranks", -1) > 0:
            comm = {"backend": "nccl", "rank": head.info["comm_rank"], "nranks": head.info["comm_nranks"],
                    "source": "ncclCommUserRank / ncclCommCount of the halo's communicator"}
            print(f"NCCL communicator: rank {comm['rank']} nRanks {comm['nranks']} "
                  f"(halo of ENS_DIST_NODE, torch ProcessGroupNCCL comm)", file=sys.stderr, flush=True)
        clk = ClockSampler(local)
        head.time(K, args.warmup, stream, barrier, clocks=clk)
        units = n_s * 3 * m.n_nodes * K              # the same total work as one GPU
        item = _line_item(head, K, units, peak)
        item["rows_rank"] = head.info["n_owned"]
        item["halo"] = halo
        item["halo_bytes_per_step_rank"] = head.info["halo_bytes_per_step"]
        item["launches_per_step"] = head.info["launches_per_step"]
        scaling, parallelism = "strong", f"node partition x{world} ({halo} halo)"
        e2e_el, e2e_meta = _e2e(head, args.e2e_windows, args.obs_every, world, barrier)
        e2e_units = n_s * 3 * m.n_nodes * args.obs_every * args.e2e_windows
        # kernels per step (boundary rows, pack / signal / wait, interior) + counter advances
        launches = head.info["launches_per_step"] * K + (_launch_count(K, head.info.get("graph_steps", 0)) - K)
        head_info = head.info
        head.close()
        if not args.no_alternatives:
            if halo == "nccl":
                try:
                    r = Run(base, args.kernel, world, rank, local, dist_mode="node", halo="p2p")
                    r.time(K, args.warmup, stream, barrier)
                    alts["node_partition_p2p"] = _line_item(r, K, units, peak)
                    r.close()
                except Exception as e:
                    alts["node_partition_p2p"] = {"error": repr(e)[:300]}
            try:                               # ensemble sharding: N_s per GPU fixed (weak)
                shard = configs.make(args.config, n_s=n_s, s_begin=rank * n_s)
                r = Run(shard, args.kernel, world, rank, local, dist_mode="ensemble")
                r.time(K, args.warmup, stream, barrier)
                it = _line_item(r, K, world * n_s * 3 * m.n_nodes * K, peak)
                it["scaling"] = "weak"
                it["n_s_total"] = world * n_s
                alts["ensemble_shard"] = it
                r.close()
            except Exception as e:
                alts["ensemble_shard"] = {"error": repr(e)[:300]}
            if n_s % world == 0 and n_s // world >= 1:
                # the same N_s realisations split across the ranks (strong scaling): the
                # communication-free counterpart of the node partition (BASELINE config c5:
                # "node-partitioned vs ensemble-sharded")
                try:
                    per = n_s // world
                    shard = configs.make(args.config, n_s=per, s_begin=rank * per)
                    r = Run(shard, args.kernel, world, rank, local, dist_mode="ensemble")
                    r.time(K, args.warmup, stream, barrier)
                    it = _line_item(r, K, n_s * 3 * m.n_nodes * K, peak)
                    it["scaling"] = "strong"
                    it["n_s_per_gpu"] = per
                    alts["ensemble_shard_strong"] = it
                    r.close()
                except Exception as e:
                    alts["ensemble_shard_strong"] = {"error": repr(e)[:300]}

    read_gbs = _read_stream_gbs() if rank == 0 else None
    try:                         # FP64 FMA probe: the ALU roofline
        fp64_peak = solver.measure_fp64_tflops(local) if rank == 0 else None
    except Exception:
        fp64_peak = None
    if fp64_peak:
        for a in alts.values():
            if "achieved_fp64_TFLOPs" in a:
                a["fp64_frac"] = a["achieved_fp64_TFLOPs"] / fp64_peak
    cpu = cpu_c2 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(base)
        if args.config != "c2" and not args.no_alternatives:     # c2 and c4
            cpu_c2 = _cpu_baseline(configs.make("c2"))

    if rank == 0:
        kfn = item["kernel_fn"]
        line = {
            "metric": METRIC, "value": item["value"], "unit": "DOF-updates/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": item["ms_per_step"],
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": _workload_desc(base, n_s, world), "kernel": args.kernel,
                       "n_s": n_s, "V": m.n_nodes, "F": m.n_tris, "nnzb": head_info["nnzb"],
                       "dt": head_info["dt"], "parallelism": parallelism,
                       "l2": f"inputs larger than L2: {head_info['bytes_per_step'] / 1e9:.3f} GB streamed per step "
                             f"and launch vs 126 MB L2 (no flush)"},
            "roofline": {"bound": "hbm", "achieved": item["achieved_GBs"], "peak": peak, "unit": "GB/s",
                         "frac": item["frac"], "traffic": _traffic(args.config, kfn, n_s) if world == 1 else None,
                         "peak_source": peak_src, "kernel": kfn,
                         "algorithmic_bytes_per_launch": head_info["bytes_per_step"],
                         "frac_of_nominal_8TBs": item["achieved_GBs"] / 8000.0,
                         "read_stream_GBs": read_gbs,
                         "frac_of_read_stream": item["achieved_GBs"] / read_gbs if read_gbs else None,
                         "fp64": {"achieved_TFLOPs": item["achieved_fp64_TFLOPs"], "peak_TFLOPs": fp64_peak,
                                  "peak_source": "measured (ens_measure_fp64: DFMA probe, this run)",
                                  "frac": item["achieved_fp64_TFLOPs"] / fp64_peak if fp64_peak else None}},
            "cpu_baseline": cpu,
            "alternatives": alts,
            "cpu_baseline_c2": cpu_c2,
            "e2e": {"value": e2e_units / e2e_el, "unit": "DOF-updates/s", **e2e_meta},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "paper_best_context": {"value": 7.27e8, "unit": "DOF-updates/s",
                                   "hardware": "4x RTX 2080 Ti, OpenCL, 131,552-tri cylinder, 500 realisations (PAPER.md:665)"},
        }
        if world > 1:
            line["config"]["rows_rank0"] = item["rows_rank"]
            line["config"]["halo_bytes_per_step_rank0"] = item["halo_bytes_per_step_rank"]
            line["config"]["launches_per_step"] = item["launches_per_step"]
            line["config"]["nccl"] = comm
        if node_emul:
            line["node_partition_emulated"] = node_emul
        if repeat:
            line["headline_windows"] = repeat
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
