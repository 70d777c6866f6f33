"""bench.py's JSON-line contract on a B200 (-m gpu): the N = 1 line (c1 for speed) and the
N > 1 line, whose headline is the node partition of the whole workload (strong scaling).
The N = 2 run puts two ranks on the one GPU of the box (ENS_BENCH_BACKEND=gloo: NCCL refuses
two ranks on one device, so the halo is the device-initiated P2P one through CUDA IPC);
its timings are meaningless, the plumbing and the line are what is checked."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_bench_n1_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "64",
                        "--warmup", "3", "--e2e-windows", "2", "--obs-every", "10"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 64 and d["dtype"] == "f64" and d["value"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["kernel"] == "k_step_assembled_sym" and rf["frac"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["one_core"]["value"] > 0 and cb["cpu_model"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    alts = d["alternatives"]
    assert alts["matrix_free"]["kernel_fn"] == "k_step_matrix_free"       # c1: N_s = 4 -> TILES
    assert alts["c2/matrix_free"]["kernel_fn"] == "k_step_mf_staged" and alts["c2/matrix_free"]["value"] > 0
    assert d["gpu_launches"] >= 64


def test_bench_n2_node_partition_headline():
    port = _free_port()
    env = dict(os.environ, ENS_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", "c1", "--steps", "40", "--warmup", "3", "--e2e-windows", "2",
           "--obs-every", "10"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout[-2000:]                  # rank 0 only
    d = lines[0]
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["parallelism"].startswith("node partition x2")
    assert 0 < d["config"]["rows_rank0"] < d["config"]["V"] and d["config"]["halo_bytes_per_step_rank0"] > 0
    assert d["cpu_baseline"] is None                          # rank 0 at N = 1 only
    assert d["alternatives"]["ensemble_shard"]["scaling"] == "weak"
    assert d["alternatives"]["ensemble_shard"]["n_s_total"] == 2 * 4
    strong = d["alternatives"]["ensemble_shard_strong"]            # the 4 realisations split 2 + 2
    assert strong["scaling"] == "strong" and strong["n_s_per_gpu"] == 2 and strong["value"] > 0
