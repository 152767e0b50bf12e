"""Multi-process (world_size 2, gloo on CPU) checks of the ensemble host logic that the
N>1 bench path uses: shard assignment, bitwise-consistent seeded
inputs per shard, max-over-ranks timing, whole-job throughput and result gathering.
The GPU data path has no collective, so this covers everything multi-rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from ldgen.configs import get_config
from ldgen.ic import make_config_ic
from paper_2507_01975_b200 import ensemble as E


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    d = E.init_process_group("gloo")
    assert d is not None and d.get_world_size() == world
    cfg = get_config("c2", batch=3)
    idx = E.shard(rank, world, cfg.batch)
    local = torch.from_numpy(make_config_ic(cfg, elements=idx).astype(np.float32))
    full = E.gather_fields(local, d)
    t = E.max_over_ranks(10.0 + rank, d)
    v = E.aggregate_throughput(world, cfg.batch * cfg.n * cfg.n, 5, t)
    d.barrier()
    if rank == 0:
        out.put((full.numpy(), t, v, list(idx)))
    d.destroy_process_group()


@pytest.mark.timeout(300)
def test_ensemble_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, t, v, idx0 = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = get_config("c2", batch=6)
    ref = make_config_ic(cfg).astype(np.float32)         # the same 6 elements generated at once
    np.testing.assert_array_equal(full, ref)              # shards concatenate to the global batch
    assert t == 11.0                                      # max over ranks
    assert v == pytest.approx(2 * 3 * 64 * 64 * 5 / 11.0e-3)
    assert idx0 == [0, 1, 2]


def test_shard_helpers():
    assert list(E.shard(1, 4, 8)) == list(range(8, 16))
    parts = [list(E.shard_of_global(r, 3, 10)) for r in range(3)]
    assert sum(parts, []) == list(range(10)) and [len(p) for p in parts] == [4, 3, 3]
    with pytest.raises(ValueError):
        E.shard(2, 2, 4)
    assert E.max_over_ranks(3.5, None) == 3.5
