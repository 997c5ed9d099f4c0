"""Multi-GPU plumbing (torch.distributed; NCCL on the box, gloo in CPU tests).

The HVP path shards by independent units: tangent
directions of one point, or whole trust-region problems.  Nothing inside an
HVP is exchanged; the collectives here are outside the hot loop:
  * shard(total, rank, world)        -- contiguous balanced split of units;
  * gather_rows(local, total, group) -- all_gather of per-rank results
                                        (padded to equal length) in rank order;
  * broadcast_primal(eng, gates, src) -- primal store of rank `src` to all
                                        ranks (strong-scaling use: one primal
                                        pass, many ranks applying).
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
    """Rank `src` has run eng.environments(gates); every other rank receives
    its primal store over NCCL and marks it valid (tn_hvp_primal_imported)."""
    from .api import primal_export, primal_import
    _, nbytes = eng.primal_blob()
    if dist.get_rank(group) == src:
        buf = primal_export(eng)
    else:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=eng.device)
    dist.broadcast(buf, src=src, group=group)
    if dist.get_rank(group) != src:
        primal_import(eng, buf, gates)
    return buf
