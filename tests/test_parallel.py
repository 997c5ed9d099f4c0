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


class _StandInEngine:
    """Host-side stand-in of api.HVPEngine for the CPU choreography tests: the
    'primal store' (uint8, like the real one) is a function of the gates, its
    two halves are the bottom / top sweep regions, apply needs a valid store."""

    def __init__(self):
        self.store = torch.zeros(64, dtype=torch.uint8)
        self.scalars = torch.zeros(8, dtype=torch.float64)
        self.valid = False
        self.calls = []

    @staticmethod
    def _primal(gates):
        return (gates.real.reshape(-1)[:8].clone() + 1.0).view(torch.uint8)

    def environments(self, gates):
        self.calls.append("environments")
        self.store.copy_(self._primal(gates))
        self.scalars.copy_(2 * self.store.view(torch.float64))
        self.valid = True

    def environments_part(self, gates, part):
        self.calls.append(f"part{part}")
        self.valid = False
        off, nb = self.primal_region(part)
        self.store[off:off + nb] = self._primal(gates)[off:off + nb]

    def primal_region(self, part):
        return (0, 32) if part == 0 else (32, 32)

    def environments_finish(self, gates):
        self.calls.append("finish")
        assert torch.equal(self.store, self._primal(gates)), "store regions do not match the point"
        self.scalars.copy_(2 * self.store.view(torch.float64))
        self.valid = True
        return self.scalars, None

    def primal_store(self):
        return self.store

    def invalidate_primal(self):
        self.calls.append("invalidate")
        self.valid = False

    def primal_imported(self, gates):
        self.calls.append("imported")
        assert torch.equal(self.store, self._primal(gates)), "store does not match the point"
        self.valid = True

    def apply(self, dirs):
        assert self.valid
        self.calls.append(f"apply{dirs.shape[0]}")
        return dirs * complex(float(self.store.view(torch.float64).sum()), 0.5)


def _step_worker(rank, world, port, B, split, q):
    from paper_2604_20384_b200.parallel import sharded_step
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(3)
    gates = torch.randn(5, 4, 4, dtype=torch.complex128, generator=g)
    dirs = torch.randn(B, 5, 4, 4, dtype=torch.complex128, generator=g)
    eng = _StandInEngine()
    sc, full = sharded_step(eng, gates, dirs, split=split)
    p = _StandInEngine._primal(gates).view(torch.float64)
    want = dirs * complex(float(p.sum()), 0.5)
    q.put((rank, bool(torch.equal(full, want)), bool(torch.equal(sc, 2 * p)), eng.calls))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, B, split):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, B, split, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("B", [5, 1])
def test_sharded_step_broadcast_world2_gloo(B):
    """split=False: primal once on rank 0 -> in-place broadcast of the whole
    store -> import check on rank 1 -> B/2 directions per rank -> all_gather."""
    (r0, ok0, sc0, calls0), (r1, ok1, sc1, calls1) = _run(2, B, False)
    assert ok0 and ok1 and sc0 and sc1
    assert calls0[0] == "environments" and "imported" not in calls0
    assert calls1[:2] == ["invalidate", "imported"] and "environments" not in calls1
    n0 = (B + 1) // 2
    assert calls0[-1] == f"apply{n0}"
    assert (calls1[-1] == f"apply{B - n0}") if B - n0 else calls1[-1] == "imported"


def test_sharded_step_split_primal_world3_gloo():
    """split=True (the default): bottom sweep on rank 0, top sweep on rank 1,
    both store regions broadcast, every rank finishes the environments itself
    (rank 2 only receives), then 7 directions in shares 3/2/2 and all_gather."""
    res = _run(3, 7, True)
    for rank, ok, sc, calls in res:
        assert ok and sc, rank
        assert calls[-2] == "finish" and "environments" not in calls and "imported" not in calls
    assert res[0][3][0] == "part0" and res[1][3][0] == "part1" and res[2][3][0] == "invalidate"
    assert [c[-1] for _, _, _, c in res] == ["apply3", "apply2", "apply2"]
