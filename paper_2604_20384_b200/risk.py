"""N1: the sampled-state empirical risk on the GPU.

PAPER.md:525-554 (eq:costHS): C_hat(G) = 1 - (1/S) sum_s |<phi_s| W(G) |psi_s>|^2
over S Haar product states psi_s with labels phi_s = U_ref psi_s, "embarrassingly
parallel" over samples.  One state-mode context (site_dim = 2:
product-state bottom start, label-MPS top start) per sample holds that
sample's primal store; the risk, its Riemannian gradient and Riemannian HVPs
are sample means, accumulated by the library's tangent axpby kernel
(tn_tangent_axpby) -- App. E's maps are linear in (grad f, H_f), so the mean of
the per-sample Riemannian outputs is the Riemannian output of the mean.  With a
process group the samples are sharded over ranks (parallel.shard) and the
partial means are summed with one all_reduce per call (the path's real
exchange step).  This module only marshals arguments; all arithmetic runs in
libtn_hvp.so.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import torch

from .api import HVPEngine, axpby
from .parallel import shard


class EmpiricalRisk:
    """labels: S label MPS (lists of [b][2][b'] tensors, right-canonical, the
    same bonds for every sample); psis: [S, n, 2] product states."""

    def __init__(self, n, depth, chi, labels, psis, first_offset=0, max_batch=64, device=None, group=None,
                 concurrency=4):
        self.group = group
        S = len(labels)
        if group is not None:
            import torch.distributed as dist
            start, count = shard(S, dist.get_rank(group), dist.get_world_size(group))
        else:
            start, count = 0, S
        self.S, self.mine = S, range(start, start + count)
        self.engines = []
        for s in self.mine:
            eng = HVPEngine(n, depth, chi, labels[s], first_offset, max_batch, device, site_dim=2)
            eng.set_product_state(torch.as_tensor(psis[s], dtype=torch.complex128, device=eng.device).contiguous())
            self.engines.append(eng)
        self.device = self.engines[0].device if self.engines else torch.device("cuda", torch.cuda.current_device())
        self.K = self.engines[0].K if self.engines else None
        # samples are independent: each engine runs on its own stream from its
        # own host thread, so their latency-bound primal sweeps overlap on the
        # GPU (ctypes releases the GIL inside the library calls)
        self.streams = [torch.cuda.Stream(device=self.device) for _ in self.engines]
        # the engines share the device: split the per-point cache memory
        # (chains + memo) evenly, keeping room for each sample's tangent state
        if self.engines:
            free, _ = torch.cuda.mem_get_info(self.device)
            work = 2 * min(concurrency, len(self.engines)) * max(e.per_direction_bytes * e.max_batch
                                                                for e in self.engines)
            share = max(0, int(0.8 * (free - work))) // len(self.engines)
            for e in self.engines:
                e.set_cache_budget(max(share, 1))
        # at most `concurrency` samples in flight (their transient tangent and
        # environment buffers must fit beside all samples' primal stores)
        self.pool = ThreadPoolExecutor(max_workers=max(1, min(concurrency, len(self.engines))))

    def _each(self, fn):
        """fn(engine) for every local sample, concurrently on per-sample
        streams; returns the results once the caller's stream is ordered after
        all of them."""
        cur = torch.cuda.current_stream(self.device)
        ev = cur.record_event()

        def run(i):
            with torch.cuda.stream(self.streams[i]):
                self.streams[i].wait_event(ev)
                return fn(self.engines[i])

        outs = list(self.pool.map(run, range(len(self.engines))))
        for st in self.streams:
            cur.wait_stream(st)
        for o in outs:                  # made on a sample stream, consumed on the caller's
            for t in (o if isinstance(o, tuple) else (o,)):
                t.record_stream(cur)
        return outs

    def _reduce(self, t):
        if self.group is not None:
            import torch.distributed as dist
            dist.all_reduce(torch.view_as_real(t), group=self.group)
        return t

    def environments(self, gates: torch.Tensor):
        """-> (risk [1] float64 device = 1 + mean_s f_s, grad_R [K,4,4] of the risk)."""
        K = gates.shape[0]
        acc = torch.zeros(4, dtype=torch.complex128, device=self.device)     # (f, T) pairs of scalars[0:2]
        g = torch.zeros(K, 4, 4, dtype=torch.complex128, device=self.device)
        for sc, gR in self._each(lambda eng: tuple(t.clone() for t in eng.environments(gates))):
            axpby(1.0 / self.S, torch.view_as_complex(sc.view(4, 2)), 1.0, acc)
            axpby(1.0 / self.S, gR, 1.0, g)
        self._reduce(acc)
        self._reduce(g)
        risk = torch.ones(1, dtype=torch.complex128, device=self.device)
        axpby(1.0, acc[:1], 1.0, risk)              # 1 + mean f  (real part)
        return torch.view_as_real(risk)[:, 0], g

    def cost(self, gates: torch.Tensor):
        """Risk at trial gates (per-sample top sweeps only, tn_hvp_cost; the
        stored points are untouched) -> [1] float64 = 1 + mean_s f_s."""
        acc = torch.zeros(4, dtype=torch.complex128, device=self.device)
        for sc in self._each(lambda eng: eng.cost(gates)):
            axpby(1.0 / self.S, torch.view_as_complex(sc.view(4, 2)), 1.0, acc)
        self._reduce(acc)
        risk = torch.ones(1, dtype=torch.complex128, device=self.device)
        axpby(1.0, acc[:1], 1.0, risk)
        return torch.view_as_real(risk)[:, 0]

    def apply(self, dirs: torch.Tensor):
        """Riemannian HVPs of the risk for dirs [B,K,4,4] -> [B,K,4,4]."""
        H = torch.zeros_like(dirs)
        for Hs in self._each(lambda eng: eng.apply(dirs)):
            axpby(1.0 / self.S, Hs, 1.0, H)
        return self._reduce(H)

    def close(self):
        torch.cuda.synchronize(self.device)
        for eng in self.engines:
            eng.close()
        self.engines = []
        self.pool.shutdown()
