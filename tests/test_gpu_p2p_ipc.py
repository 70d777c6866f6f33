"""ENS_HALO_P2P across processes: two ranks, one part each, connected
through CUDA IPC (ens_p2p_export / ens_p2p_connect, blobs all-gathered over a gloo
group).  On the one-GPU test box both ranks share cuda:0, so the peer stores are plain
device stores between two contexts; on an NVSwitch box the same code stores over NVLink.
The owned rows of each rank must equal the single-process run bit for bit (-m gpu)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RHO, NU, KS = 1.06, 0.5, 5.0 / 6.0
STEPS = 70          # one graph replay (64) + 6 direct steps


def _problem():
    from paper_2101_09059_b200.inputs import fields, loads, mesh as meshmod
    m = meshmod.shuffle_nodes(meshmod.perturb(meshmod.cylinder(24, 60), 0.01, 3), 2)
    E, h, _ = fields.sample_materials(m.xyz, m.tris, 8, E_mean=7e6, E_std=7e5, h_mean=0.4, h_std=0.04,
                                      rho_corr=3.7, seed=77)
    tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
    kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel="assembled", dt=5e-5, damping="identity", c_d=0.3)
    return m, E, h, tr, kw


def _rank_main(rank, world, port, outdir, persistent=False, steps=STEPS):
    import torch
    import torch.distributed as dist
    from paper_2101_09059_b200 import solver
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    m, E, h, tr, kw = _problem()
    ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, dist="node", world=world, rank=rank, halo="p2p",
                          p2p_procs=True, persistent=persistent, **kw)
    ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ens.step(steps)
    u, um, _, st = ens.get_state()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), u=u, um=um, ids=ens.owned(), step=st,
             launches=ens.info()["launches_per_step"])
    dist.barrier()
    ens.close()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("persistent", [False, True])
def test_p2p_two_processes_bitexact(tmp_path, persistent):
    """persistent=True: each rank advances its part in ONE cooperative kernel per ens_step
    (N2), waiting for / publishing the step flags inside it; the two kernels share the one
    GPU by time slicing here (a few steps only), across NVLink on a multi-GPU box."""
    import torch.multiprocessing as mp
    from paper_2101_09059_b200 import solver
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    steps = 12 if persistent else STEPS
    mp.start_processes(_rank_main, args=(world, port, str(tmp_path), persistent, steps), nprocs=world, join=True,
                       start_method="spawn")
    m, E, h, tr, kw = _problem()
    ref = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw)
    ref.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
    ref.step(steps)
    u, um, _, st = ref.get_state()
    seen = np.zeros(m.n_nodes, bool)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert int(d["step"]) == st == steps
        ids = d["ids"]
        assert np.array_equal(d["u"], u[:, ids]) and np.array_equal(d["um"], um[:, ids])
        seen[ids] = True
    assert seen.all()
    ref.close()
