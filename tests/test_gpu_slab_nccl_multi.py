"""Slab decomposition over REAL NCCL ranks (mode 2, one process per GPU): every
rank steps its own rows [r n, (r+1) n) of the global field with halos and the distributed-FFT all-to-alls
going through ncclSend / ncclRecv, and the gathered result equals the single-domain step (Pin-14: relL2
1e-5).  Needs >= 2 visible GPUs: skipped otherwise (the 1-rank NCCL path and the all-ranks-in-one-process
emulation are covered by tests/test_gpu_slab.py; the multi-process host logic by tests/test_slab_gloo.py)."""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, outdir, name, n, B, steps):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist
    from ldgen.configs import get_config
    from paper_2507_01975_b200 import ldsolver as L
    from tests.helpers import setup
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    cfg = get_config(name, n=n, batch=B, conv_precision=1)
    cfg, u0, params = setup(cfg, init="stress")
    uid = L.nccl_unique_id() if rank == 0 else bytes(128)
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    comm = L.nccl_comm_init(obj[0], world, rank)
    rows = n // world
    try:
        s = L.Solver(L.make_config(cfg), params, dist=L.ld_dist(mode=2, rank=rank, world=world, nccl_comm=comm))
        u = torch.from_numpy(np.ascontiguousarray(u0[:, :, rank * rows:(rank + 1) * rows], dtype=np.float32)).cuda()
        s.ld_rollout(u, steps)
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"r{rank}.npy"), u.cpu().numpy())
        s.close()
    finally:
        L.nccl_comm_destroy(comm)
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,n,B,steps", [("c3", 256, 2, 2), ("c4", 512, 1, 1)])
def test_slab_nccl_two_ranks_equals_single_domain(name, n, B, steps):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (one rank per GPU)")
    from ldgen.configs import get_config
    from tests.helpers import gpu_solver, rel_l2, setup, to_dev
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank_main, args=(world, _free_port(), d, name, n, B, steps), nprocs=world,
                           start_method="spawn")
        got = np.concatenate([np.load(os.path.join(d, f"r{r}.npy")) for r in range(world)], axis=2)
    cfg = get_config(name, n=n, batch=B, conv_precision=1)
    cfg, u0, params = setup(cfg, init="stress")
    ref = to_dev(u0)
    gpu_solver(cfg, params).ld_rollout(ref, steps)
    assert rel_l2(got, ref.cpu().numpy()) < 1e-5
