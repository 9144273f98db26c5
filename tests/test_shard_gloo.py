"""World-size-2 gloo test of the receiver-tile partition + gather (shard.py) on CPU."""
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
    port = s.getsockname()[1]
    s.close()
    return port


def field_of(idx, F):
    """Stand-in per-receiver result: depends only on the global receiver index."""
    i = idx.double()[:, None]
    f = torch.arange(F, dtype=torch.float64)[None, :]
    return torch.complex(torch.sin(i * 0.37 + f), torch.cos(i * 0.11 - f)), (idx * 3 + 1)


def _worker(rank, world, port, n, F, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_13382_b200 import shard
    # a deterministic stand-in for the device Hilbert order
    order = torch.from_numpy(np.random.default_rng(7).permutation(n)).long()
    mine = shard.rank_indices(order, rank, world, tile=64)
    acc, ev = field_of(mine, F)
    plan = shard.GatherPlan(order, world, n, tile=64) if F > 1 else None
    full, evf = shard.gather_field(acc, ev.long(), order, rank, world, n, tile=64, plan=plan)
    if rank == 0:
        want, want_ev = field_of(torch.arange(n), F)
        q.put((bool(torch.equal(full, want)), bool(torch.equal(evf, want_ev))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,F,world", [(1000, 1, 2), (333, 5, 2), (1000, 3, 3)])
def test_gather_field_world2(n, F, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, F, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) == (True, True)
