"""Multi-GPU plumbing (torch.distributed; NCCL on the box, gloo in CPU tests).

The HVP path shards by independent units: tangent
directions of one point, or whole trust-region problems.  Nothing inside an
HVP is exchanged; the collectives here are outside the hot loop:
  * shard(total, rank, world)        -- contiguous balanced split of units;
  * gather_rows(local, total, group) -- all_gather of per-rank results
                                        (padded to equal length) in rank order;
  * broadcast_primal(eng, gates, src) -- primal store of rank `src` to all
                                        ranks, in place (one primal pass, many
                                        ranks applying);
  * split_primal(eng, gates)          -- bottom sweep on rank 0, top sweep on
                                        rank 1, both store regions broadcast,
                                        environments finished on every rank;
  * sharded_step(eng, gates, dirs)    -- the strong-scaling step bench.py
                                        times for N > 1: primal once (split),
                                        B/N directions per rank, all_gather.
Every function only needs the engine's methods (environments, apply,
primal_store, invalidate_primal, primal_imported, environments_part,
primal_region, environments_finish, scalars), so the CPU tests
drive the same choreography over gloo with a stand-in engine.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(total: int, rank: int, world: int):
    """(start, count) of rank's share: the first total % world ranks get one more."""
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def gather_rows(local: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather per-rank row blocks (dim 0, sizes from `shard`) into [total, ...]."""
    world = dist.get_world_size(group)
    width = -(-total // world)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    if local.dtype.is_complex:
        pad_r = torch.view_as_real(pad).contiguous()
        outs = [torch.empty_like(pad_r) for _ in range(world)]
        dist.all_gather(outs, pad_r, group=group)
        outs = [torch.view_as_complex(o) for o in outs]
    else:
        outs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
    rows = []
    for r in range(world):
        _, c = shard(total, r, world)
        rows.append(outs[r][:c])
    return torch.cat(rows, 0)


def broadcast_primal(eng, gates: torch.Tensor, src: int = 0, group=None):
    """Rank `src` has run eng.environments(gates) (or eng.step); every other
    rank receives the primal store IN PLACE (the store is the engine's
    caller-owned torch buffer, eng.primal_store()) and marks it valid
    (eng.primal_imported -> tn_hvp_primal_imported, which checks that the
    received store's point is `gates`).  Returns the store."""
    buf = eng.primal_store()
    receiver = dist.get_rank(group) != src
    if receiver:
        eng.invalidate_primal()   # the old point's caches must not outlive the overwrite
    dist.broadcast(buf, src=src, group=group)
    if receiver:
        eng.primal_imported(gates)
    return buf


def split_primal(eng, gates: torch.Tensor, group=None):
    """The primal pass over two ranks: rank 0 runs the bottom
    sweep and rank 1 the top sweep at the same time, each writing its side's
    region of the primal store; both regions are broadcast in place (bottom
    from rank 0, top from rank 1) to every rank, which then finishes the pass
    (layer environments, E, f, grad_R) on its own GPU.  One GPU: the ordinary
    primal pass.  Returns (scalars, grad_R)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world < 2:
        return eng.environments(gates)
    rank = dist.get_rank(group)
    if rank < 2:
        eng.environments_part(gates, rank)
    else:
        eng.invalidate_primal()
    store = eng.primal_store()
    for part in (0, 1):
        off, nbytes = eng.primal_region(part)
        dist.broadcast(store[off:off + nbytes], src=part, group=group)
    return eng.environments_finish(gates)


def sharded_step(eng, gates: torch.Tensor, dirs: torch.Tensor, src: int = 0, group=None, out=None,
                 split: bool = True):
    """One strong-scaling step of the hot path (north_star):
    the primal pass once -- split over ranks 0 and 1 (split_primal: the two
    sweeps at the same time, their store regions broadcast, every rank
    finishing the environments), or with split=False on rank `src` with the
    whole store broadcast in place (broadcast_primal) -- each rank applying its
    contiguous share of the B directions (shard), the Riemannian HVPs
    all-gathered in direction order (gather_rows).  Every rank passes the same
    gates and all B directions; returns (scalars [8], Hess_R [B, K, 4, 4]) on
    every rank (scalars broadcast from `src`).  `out`: optional [B,K,4,4]
    buffer for the gathered result."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if split and world >= 2:
        split_primal(eng, gates, group)          # every rank ends with the full store
    else:
        if rank == src:
            eng.environments(gates)
        broadcast_primal(eng, gates, src, group)
        dist.broadcast(eng.scalars, src=src, group=group)
    B = dirs.shape[0]
    start, count = shard(B, rank, world)
    if count:
        local = eng.apply(dirs[start:start + count])
    else:
        local = dirs.new_zeros((0,) + tuple(dirs.shape[1:]))
    full = gather_rows(local, B, group)
    if out is not None:
        out.copy_(full)
        full = out
    return eng.scalars, full
