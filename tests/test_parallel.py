"""Multi-process host logic of the sharded path (gloo, world size 2, CPU)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_20384_b200.parallel import gather_rows, shard


def test_shard_covers_all_units_once():
    for total in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, c = shard(total, r, world)
                seen.extend(range(s, s + c))
            assert seen == list(range(total))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, c = shard(total, rank, world)
    # each rank "computes" its directions: row i = i * (1+2j) (a stand-in for Hess_R rows)
    local = torch.stack([torch.full((3, 4), complex(i, 2 * i), dtype=torch.complex128) for i in range(s, s + c)]) \
        if c else torch.zeros((0, 3, 4), dtype=torch.complex128)
    full = gather_rows(local, total)
    realv = gather_rows(torch.arange(s, s + c, dtype=torch.float64)[:, None], total)
    if rank == 0:
        q.put((full.numpy(), realv.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [7, 8])
def test_gather_rows_world2_gloo(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, realv = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert full.shape == (total, 3, 4)
    for i in range(total):
        assert (full[i] == complex(i, 2 * i)).all()
    assert (realv[:, 0] == range(total)).all()
