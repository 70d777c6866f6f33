"""World-size-2 (and 3) CPU tests of the multi-process paths with the gloo backend.

* Node partition: every rank builds the halo plan with the product library
  (ens_host_halo_plan) and executes it as a real point-to-point exchange (gloo
  isend/irecv of the send rows' payload); each rank must receive exactly its ghost rows,
  in its ghost order — the same message schedule ens_step runs over NCCL.
* Ensemble sharding: the per-rank realisation slices are disjoint and cover N_s, and the
  shard inputs (Matérn draws keyed by (seed, field, s)) equal the matching slice of the
  unsharded draw.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _halo_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        from paper_2101_09059_b200 import solver
        from paper_2101_09059_b200.inputs import mesh as meshmod
        m = meshmod.shuffle_nodes(meshmod.cylinder(18, 41), 9)
        perm, row_ptr, col = solver.host_pattern(m.n_nodes, m.tris)
        pl = solver.host_halo_plan(row_ptr, col, world, rank)
        lo, hi = pl["lo"], pl["hi"]
        n_own = hi - lo
        W = 5                          # payload width (stands for 3 * N_s)
        # payload of global row g: (g, g + 0.25, ...) so receivers can check identity
        send = torch.tensor([[lo + r + 0.25 * k for k in range(W)] for r in pl["send_rows"]],
                            dtype=torch.float64).reshape(-1, W)
        ghosts = torch.full((pl["n_ghost"], W), -1.0, dtype=torch.float64)
        reqs = []
        for (qq, so, sn, rr, rn) in pl["peers"]:
            if sn:
                reqs.append(dist.isend(send[so:so + sn].contiguous(), qq))
            if rn:
                buf = torch.empty((rn, W), dtype=torch.float64)
                reqs.append((dist.irecv(buf, qq), buf, rr - n_own))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                ghosts[r[2]:r[2] + r[1].shape[0]] = r[1]
            else:
                r.wait()
        # expected ghosts: sorted global columns outside [lo, hi) of the owned rows
        cols = col[row_ptr[lo]:row_ptr[hi]]
        exp = np.unique(cols[(cols < lo) | (cols >= hi)])
        got = ghosts[:, 0].numpy()
        ok = np.array_equal(got, exp.astype(float)) and np.allclose(ghosts[:, 3].numpy(), exp + 0.75)
        q.put((rank, bool(ok), len(exp)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), -1))


@pytest.mark.parametrize("world", [2, 3])
def test_halo_plan_executes_as_p2p_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, n in res:
        assert ok is True, (rank, ok)
        assert n > 0


def _shard_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        from paper_2101_09059_b200.inputs import configs
        n_s = 4
        cfg = configs.make("c1", n_s=n_s, s_begin=rank * n_s)
        t = torch.from_numpy(np.ascontiguousarray(cfg.E))
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        full = configs.make("c1", n_s=n_s * world)
        ok = np.array_equal(torch.cat(out).numpy(), full.E)
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_ensemble_shards_match_unsharded_draws():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok is True for _, ok in res), res
