"""The NCCL leg of ENS_DIST_NODE in a real process group (-m gpu).  A one-GPU box allows
only world_size = 1 (NCCL rejects two ranks on one device), so this checks the plumbing a
multi-GPU run depends on: torch's communicator pointer (ProcessGroupNCCL._comm_ptr), the
in-process libnccl.so.2 symbols (ncclGroupStart/End, ncclSend/Recv) resolved by
nccl_dl.cpp, the comm-stream / event ordering of enqueue_step — and that the result is
bit-identical to the single-device path."""
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RHO, NU, KS = 1.06, 0.5, 5.0 / 6.0


def test_nccl_world1_bitexact():
    import torch
    import torch.distributed as dist
    from paper_2101_09059_b200 import solver
    from paper_2101_09059_b200.inputs import fields, loads, mesh as meshmod
    torch.cuda.set_device(0)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        x = torch.ones(4, device="cuda")
        dist.all_reduce(x)                                   # the communicator exists
        comm = solver.nccl_comm_of()
        assert comm != 0
        m = meshmod.shuffle_nodes(meshmod.cylinder(24, 40), 4)
        E, h, _ = fields.sample_materials(m.xyz, m.tris, 8, E_mean=7e6, E_std=7e5, h_mean=0.4, h_std=0.04,
                                          rho_corr=3.7, seed=5)
        tr = loads.pulsatile(m.xyz, m.tris, period=0.01, systole=0.004, ramp_T=0.003)
        kw = dict(rho=RHO, nu=NU, k_shear=KS, kernel="assembled_sym", dt=5e-5, damping="mass", c_d=50.0)
        out = []
        for extra in ({}, dict(dist="node", world=1, rank=0, nccl_comm=comm)):
            ens = solver.Ensemble(m.xyz, m.tris, m.fixed, E, h, **kw, **extra)
            ens.set_traction(tr.F, tr.tab_t, tr.tab_g, tr.period, tr.ramp_T)
            ens.step(90)
            u, up, _, st = ens.get_state()
            out.append((u, ens.owned(), st))
            ens.close()
        # the NODE context reports its owned rows in local order (ens_get_owned gives node ids)
        (u0, _, s0), (u1, ids, s1) = out
        assert s0 == s1 == 90 and len(ids) == m.n_nodes
        assert np.array_equal(u0[:, ids], u1)
    finally:
        dist.destroy_process_group()
