"""Benchmark of the HVP hot path (BASELINE.json metric: HVPs/sec, complex128,
and the fraction of the FP64 roofline) on 1..N B200s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of the whole hot path over one
batch of the config's B tangent directions (C4: 64): the primal pass
(tn_hvp_environments: sweeps, layer environments, f, grad_R) and the Riemannian
HVPs of all B directions.
  * N = 1: the fused tn_hvp_step (the first sub-batch's forward tangents
    overlap the primal pass).
  * N > 1 (torchrun, one process per GPU): strong scaling as north_star and
    SURVEY.md §8(e) describe -- the primal pass once on rank 0, its store
    broadcast in place with NCCL, B/N directions applied per rank, Hess_R
    all-gathered with NCCL (parallel.sharded_step).
value = B / max-over-ranks step time.  Phase times (primal, broadcast,
apply, gather), the apply-only HVPs/s of SURVEY.md §8(d) and the broadcast
bytes are measured after the timed region and reported beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from tn_inputs import configs as C  # noqa: E402

METRIC = "HVPs/sec (complex128) and fraction of FP64/HBM roofline at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=int(os.environ.get("TN_BENCH_CONFIG", 4)))
    ap.add_argument("--batch", type=int, default=None, help="directions per GPU (default: the config's)")
    ap.add_argument("--max-batch", type=int, default=None, help="internal sub-batch (memory)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--unfused", action="store_true",
                    help="time tn_hvp_environments + tn_hvp_apply instead of the fused tn_hvp_step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="config", choices=["config", "n1"],
                    help="config: the BASELINE.json config (default); n1: the sampled-state empirical risk "
                         "(SURVEY.md 8(f) N1) at the config's width")
    ap.add_argument("--samples", type=int, default=4, help="N1: product states S")
    ap.add_argument("--concurrency", type=int, default=2, help="N1: samples in flight per GPU")
    return ap.parse_args()


# ------------------------------------------------------------ helpers --
class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4) if r[2 + j].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def fp64_peak():
    """Measured DMMA peak (TF/s): live probe, else the committed measurement."""
    exe = os.path.join(ROOT, "paper_2604_20384_b200", "bin", "fp64_peak")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
        d = json.loads(out)
        return d["dmma_tflops"], "live bin/fp64_peak DMMA loop (MEASURED_PEAKS.json has no FP64 entry)"
    except Exception:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak_probe.json")) as f:
            d = json.load(f)
        return d["loops"]["dmma_tflops"], "profiles/r01_fp64_peak_probe.json DMMA loop"


def dist_init(n):
    if n <= 1 and "WORLD_SIZE" not in os.environ:
        return 0, 1, 0
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------- oracle sample --
def oracle_sample(cfg, ref_cpu, G, budget_s=20.0):
    """The CPU oracle (O3) as it stands, on a bounded sample of the workload:
    its sweep steps (two-site SVD truncation + channel-tangent update for one
    direction) on the first-processed top layer (full reference bonds), run
    gate by gate for ~budget_s.  HVPs/s = 1 / (t_gate x 2K) -- an UPPER bound
    on the oracle's rate: it leaves out the per-layer environment/extraction
    work (and the primal E), which the GPU's work model puts at ~3-4x the
    tangent-step work."""
    from oracle import common as cm
    from oracle import mpo as M
    K = C.num_gates(cfg.n, cfg.depth, cfg.first_offset)
    V = C.tangent_directions(cfg.cid, G, 1)
    sw = M.MPOSweep(ref_cpu, cfg.chi, 1)
    ly = cm.layers(cfg.n, cfg.depth, cfg.first_offset)[cfg.depth - 1]
    t0 = time.time()
    done = 0
    for k, s in ly:
        sw.pair_step(s, G[k].conj().T, [V[0, k].conj().T], True)
        done += 1
        if time.time() - t0 > budget_s:
            break
    dt = time.time() - t0
    t_gate = dt / done
    return 1.0 / (t_gate * 2 * K), dt, done


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_baseline(cfg, ref_cpu, G, budget_s=10.0):
    """cpu_baseline object: the oracle sample at 1 BLAS thread and at all
    cores of this host (threadpoolctl), plus the full-size oracle timings
    recorded when tests/golden/ was generated (tools/golden_full.py)."""
    from threadpoolctl import threadpool_limits
    ncores = os.cpu_count()
    with threadpool_limits(limits=1):
        r1, dt1, n1 = oracle_sample(cfg, ref_cpu, G, budget_s)
    with threadpool_limits(limits=ncores):
        ra, dta, na = oracle_sample(cfg, ref_cpu, G, budget_s)
    out = {"value": ra, "unit": "HVPs/s", "cores": ncores, "kind": "oracle",
           "sample": (f"O3 numpy oracle sweep steps (SVD truncation + tangent update, 1 direction) on the first "
                      f"top layer at full bonds: {na} gates in {dta:.1f} s at {ncores} threads, {n1} gates in "
                      f"{dt1:.1f} s at 1 thread; HVPs/s = 1/(t_gate x 2K), an upper bound (excludes the layer "
                      f"environment / extraction work)"),
           "hvps_per_s_1thread": r1, "hvps_per_s_all_cores": ra, "nproc": ncores, "cpu_model": cpu_model(),
           "s_per_hvp_1thread_upper_bound": 1 / r1, "s_per_hvp_all_cores_upper_bound": 1 / ra}
    gpath = os.path.join(ROOT, "tests", "golden", f"full_c{cfg.cid}.json")
    if not os.path.exists(gpath):   # per-direction oracle runs (tools/golden_full.py --only b)
        gpath = os.path.join(ROOT, "tests", "golden", f"full_c{cfg.cid}_d0.json")
    if os.path.exists(gpath):
        with open(gpath) as f:
            g = json.load(f)
        td = g.get("t_dir_s") or []
        out["oracle_full_size"] = {
            "what": "measured full oracle run that wrote tests/golden (tools/golden_full.py), on the build "
                    "container, not this host", "primal_s": g.get("t_primal_s"), "primal_and_E_s": g.get("t_env_s"),
            "per_hvp_s": (sum(td) / len(td)) if td else None, "threads": g.get("threads"), "nproc": g.get("nproc"),
            "hvps_per_s": (len(td) / sum(td)) if td else None}
    return out


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    ref = C.reference_mpo(cfg, device="cuda" if torch.cuda.is_available() else "cpu")
    ref_cpu = [a.detach().resolve_conj().cpu().numpy() for a in ref]
    G = C.haar_gates(cfg.cid, C.num_gates(cfg.n, cfg.depth, cfg.first_offset))
    rates, times = [], []
    done = 0
    for _ in range(args.steps):
        r, dt, done = oracle_sample(cfg, ref_cpu, G)
        rates.append(r)
        times.append(dt)
    v = statistics.median(rates)
    cores = os.cpu_count()
    sample = (f"O3 numpy oracle sweep steps (SVD truncation + tangent update, 1 direction) on {done} gates of the "
              f"first top layer at full bonds, ~20 s, {cores} cores ({cpu_model()}); HVPs/s = 1/(t_gate x 2K): upper "
              f"bound, excludes the layer environment/extraction work")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "HVPs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": cfg.name, "n": cfg.n, "depth": cfg.depth, "chi": cfg.chi},
        "cpu_baseline": {"value": v, "unit": "HVPs/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "HVPs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


class Phase:
    """CUDA-event interval on the current stream (synchronised on exit)."""

    def __enter__(self):
        self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.e0.record()
        return self

    def __exit__(self, *a):
        self.e1.record()
        self.e1.synchronize()
        self.ms = self.e0.elapsed_time(self.e1)


# ------------------------------------------------------------------ N1 --
def run_n1(args, cfg, rank, world, local):
    """N1: risk HVPs/s = directions / step, a step being the
    risk's primal pass over all S samples (concurrent per-sample streams) and
    its Riemannian HVPs for B directions; samples sharded over ranks with one
    all_reduce per call (risk.EmpiricalRisk)."""
    import torch.distributed as dist
    from paper_2604_20384_b200 import _native as N
    from paper_2604_20384_b200.risk import EmpiricalRisk
    from tn_inputs import samples as SMP
    dev = torch.device("cuda", torch.cuda.current_device())
    S, B = args.samples, args.batch or 8
    K = C.num_gates(cfg.n, cfg.depth, cfg.first_offset)
    ref = [a.detach().resolve_conj().cpu().numpy() for a in C.reference_mpo(cfg, device=dev)]
    psis = SMP.haar_product_states(cfg.cid, S, cfg.n)
    labels = [[torch.tensor(a, device=dev) for a in SMP.label_mps(ref, p)] for p in psis]
    Gnp = C.haar_gates(cfg.cid, K)
    G = torch.tensor(Gnp, device=dev)
    V = torch.tensor(C.tangent_directions(cfg.cid, Gnp, B), device=dev)
    er = EmpiricalRisk(cfg.n, cfg.depth, cfg.chi, labels, psis, cfg.first_offset, max_batch=B,
                       group=dist.group.WORLD if world > 1 else None, concurrency=args.concurrency)

    def step():
        er.environments(G)
        return er.apply(V)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    N.tn_gemm_profile(1)
    er.apply(V)
    torch.cuda.synchronize()
    gemm_ms, gemm_cmac = N.tn_gemm_profile(0)
    barrier(world)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        l0 = N.tn_hvp_launch_count()
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        torch.cuda.synchronize()
        launches = N.tn_hvp_launch_count() - l0
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    with Phase() as p_env:
        er.environments(G)
    with Phase() as p_ap:
        er.apply(V)
    peak, peak_src = fp64_peak()
    achieved = 8 * gemm_cmac / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    line = {
        "metric": "risk HVPs/sec of the N1 sampled-state empirical risk (complex128)", "value": B / (ms / 1e3),
        "unit": "risk HVPs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"N1-{cfg.name}-S{S}", "n": cfg.n, "depth": cfg.depth, "chi": cfg.chi,
                   "samples": S, "directions_per_step": B,
                   "parallelism": f"samples over {world} rank(s), concurrent per-sample streams, all_reduce",
                   "l2": "working set > 126 MB L2; no flush"},
        "sample_hvps_per_s": S * B / (ms / 1e3),
        "phases": {"primal_all_samples_ms": max_over_ranks(p_env.ms, world),
                   "apply_all_samples_ms": max_over_ranks(p_ap.ms, world)},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if achieved else None, "traffic": None,
                     "kernel": "tn::zgemm3m_kernel over one risk apply (per-launch CUDA events, concurrent streams)",
                     "peak_source": peak_src},
        "clocks": clk.summary(), "gpu_launches": int(launches)}
    if rank == 0:
        print(json.dumps(line))
    er.close()


# ----------------------------------------------------------------- ours --
def main():
    args = parse()
    cfg = C.CONFIGS[args.config]
    rank, world, local = dist_init(args.gpus)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if args.workload == "n1":
        run_n1(args, cfg, rank, world, local)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    from paper_2604_20384_b200 import _native as N
    from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine
    from paper_2604_20384_b200.parallel import broadcast_primal, gather_rows, shard, sharded_step, split_primal

    dev = torch.device("cuda", torch.cuda.current_device())
    B = args.batch or cfg.batch                       # directions per step (all ranks together)
    mb = args.max_batch or SUB_BATCH[cfg.cid]
    K = C.num_gates(cfg.n, cfg.depth, cfg.first_offset)
    # N4: the reference MPO is built on the GPU by the library's TEBD (tn_mpo_tebd)
    from paper_2604_20384_b200.api import mpo_tebd
    torch.cuda.synchronize()
    t_ref0 = time.time()
    ref = mpo_tebd(cfg.n, C.reference_layers(cfg), cfg.chi)
    if world > 1:   # every rank uses rank 0's reference bits (the imported primal store was built on it)
        import torch.distributed as dist
        for a in ref:
            dist.broadcast(a, src=0)
    torch.cuda.synchronize()
    t_ref = time.time() - t_ref0
    Gnp = C.haar_gates(cfg.cid, K)
    Vnp = C.tangent_directions(cfg.cid, Gnp, B)
    G = torch.tensor(Gnp, device=dev)
    V = torch.tensor(Vnp, device=dev)
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, cfg.first_offset, max_batch=mb)
    out = torch.empty_like(V)
    s0, cnt = shard(B, rank, world)
    Vmine = V[s0:s0 + cnt].contiguous()

    def step(Gd=G, Vd=V):
        if world > 1:
            return sharded_step(eng, Gd, Vd, out=out)
        if args.unfused:
            sc, _ = eng.environments(Gd)
            eng.apply(Vd, out=out)
            return sc, out
        sc, _, _ = eng.step(Gd, Vd, out=out)
        return sc, out

    for _ in range(max(args.warmup - 1, 0)):
        step()
    torch.cuda.synchronize()
    # the last warm-up step is instrumented (untimed) and unfused, so that the
    # apply phase's GEMMs run alone on one stream: per-launch GEMM time (CUDA
    # events around every GEMM) and exact complex MACs of each phase
    barrier(world)
    N.tn_gemm_profile(1)
    split_primal(eng, G)                       # one GPU: tn_hvp_environments
    torch.cuda.synchronize()
    env_gemm_ms, env_gemm_cmac = N.tn_gemm_profile(0)
    N.tn_gemm_profile(1)
    if cnt:
        eng.apply(Vmine)
    torch.cuda.synchronize()
    gemm_ms, gemm_cmac = N.tn_gemm_profile(0)
    cmac_dir, cmac_primal = eng.work()
    if rank != 0:
        cmac_primal = 0.0

    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        l0 = N.tn_hvp_launch_count()
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        torch.cuda.synchronize()
        launches = N.tn_hvp_launch_count() - l0
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    value = B / (ms / 1e3)

    # end-to-end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        Gh = torch.tensor(Gnp).pin_memory()
        Vh = torch.tensor(Vnp).pin_memory()
        Hh = torch.empty(Vh.shape, dtype=Vh.dtype).pin_memory()
        Sh = torch.empty(8, dtype=torch.float64).pin_memory()
        Gd, Vd = torch.empty_like(G), torch.empty_like(V)

        def step_e2e():
            Gd.copy_(Gh, non_blocking=True)
            Vd.copy_(Vh, non_blocking=True)
            sc, H = step(Gd, Vd)
            Hh.copy_(H, non_blocking=True)
            Sh.copy_(sc, non_blocking=True)

        torch.cuda.synchronize()
        barrier(world)
        e0.record(st)
        for _ in range(args.steps):
            step_e2e()
        e1.record(st)
        torch.cuda.synchronize()
        barrier(world)
        ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        e2e = {"value": B / (ms_e2e / 1e3), "unit": "HVPs/s",
               "h2d_bytes_per_step": int(Gh.numel() * 16 + Vh.numel() * 16),
               "d2h_bytes_per_step": int(Hh.numel() * 16 + 8 * 8)}

    # phases of one (untimed) step, each bracketed by a barrier: the primal
    # pass (N > 1: split over ranks 0 / 1 with the region exchange and every
    # rank's finish), the alternative whole-store broadcast from rank 0, the
    # apply of this rank's share, the all_gather
    if cfg.chi <= 128 and cnt:
        # small configurations replay the apply from a point-free CUDA graph captured at the first
        # un-instrumented apply after a primal pass: capture it here, outside the timed phases
        split_primal(eng, G)
        eng.apply(Vmine)
        torch.cuda.synchronize()
    barrier(world)
    with Phase() as p_env:
        split_primal(eng, G)
    t_env = max_over_ranks(p_env.ms, world)
    barrier(world)
    with Phase() as p_bc:
        if world > 1:
            broadcast_primal(eng, G)
    t_bc = max_over_ranks(p_bc.ms, world)
    barrier(world)
    with Phase() as p_ap:
        local_H = eng.apply(Vmine) if cnt else V[:0]
    t_ap = max_over_ranks(p_ap.ms, world)
    barrier(world)
    with Phase() as p_ga:
        if world > 1:
            gather_rows(local_H, B)
    t_ga = max_over_ranks(p_ga.ms, world)
    xbytes = sum(eng.primal_region(p)[1] for p in (0, 1))
    phases = {"primal_ms": t_env,
              "primal": ("split over ranks 0/1 (bottom | top sweep), both store regions broadcast "
                         f"({xbytes} bytes), environments finished on every rank") if world > 1 else
                        "tn_hvp_environments",
              "broadcast_ms": t_bc if world > 1 else 0.0,
              "broadcast_bytes": int(eng.primal_bytes) if world > 1 else 0,
              "broadcast": "whole-store NCCL broadcast from rank 0 (the unsplit alternative), timed for reference",
              "apply_ms": t_ap,
              "gather_ms": t_ga if world > 1 else 0.0, "directions_per_rank": cnt,
              "apply_only_hvps_per_s": B / (t_ap / 1e3),
              "apply_only": "SURVEY.md §8(d) HVPs/s: B directions / max-over-ranks apply time of the rank shares, "
                            "primal built once and excluded",
              "apply_plus_broadcast_hvps_per_s": B / ((t_ap + (t_bc if world > 1 else 0.0)) / 1e3),
              "primal_split_paths": eng.split_stats()}

    peak, peak_src = fp64_peak()
    achieved = 8 * gemm_cmac / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    traffic = traffic_alg = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_c{cfg.cid}.json")  # ncu dram bytes/launch (committed)
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_launch")
        traffic_alg = tj.get("algorithmic_bytes_per_launch")
    flops_step = 8 * (cmac_dir * B + max_over_ranks(cmac_primal, world))
    line = {
        "metric": METRIC, "value": value, "unit": "HVPs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": cfg.name, "n": cfg.n, "depth": cfg.depth, "chi": cfg.chi, "gates": K,
                   "directions_per_step": B, "sub_batch": mb,
                   "parallelism": ("strong: primal once, its two sweeps split over ranks 0/1 with an NCCL "
                                   f"exchange of the store regions, {B}/{world} directions per rank, NCCL "
                                   "all_gather of Hess_R") if world > 1
                                  else "1 GPU",
                   "step": ("parallel.sharded_step" if world > 1 else
                            "tn_hvp_environments + tn_hvp_apply" if args.unfused else
                            "tn_hvp_step (fused: first sub-batch's forward tangents overlap the primal pass)"),
                   "l2": "working set (primal store, tangent caches: GBs) > 126 MB L2; no flush",
                   "reference": f"tn_mpo_tebd (library TEBD of the {cfg.order}-order Trotter circuit, N4), "
                                f"built in {t_ref:.1f} s before timing"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "traffic_algorithmic_bytes_per_launch": traffic_alg,
                     "traffic_source": f"profiles/traffic_c{cfg.cid}.json (ncu dram__bytes_read+write per "
                                       f"zgemm3m launch over a sample of APPLY launches, same population as "
                                       f"'achieved')",
                     "kernel": "tn::zgemm3m_kernel (DMMA m8n8k4 f64, 3M: 3 real DMMA per complex k-step; "
                               "algorithmic 8 flop per complex MAC, so frac can exceed 1 up to 4/3)",
                     "peak_source": peak_src,
                     "measured_on": "apply phase of an instrumented unfused warm-up step (GEMMs serialised on "
                                    "one stream; CUDA events around every GEMM launch)",
                     "apply_gemm_ms": gemm_ms, "primal_gemm_ms": env_gemm_ms,
                     "gemm_share_of_step": gemm_ms / ms if ms else None,   # apply-phase GEMM time / step
                     "flops_per_step": flops_step, "apply_cmac_per_direction": cmac_dir,
                     "primal_cmac": cmac_primal,
                     "step_frac": flops_step / (ms / 1e3) / 1e12 / peak / world},
        "phases": phases,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),      # library kernel launches inside the timed region (all steps)
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref_cpu = [a.detach().resolve_conj().cpu().numpy() for a in ref]
        line["cpu_baseline"] = oracle_baseline(cfg, ref_cpu, Gnp)
    if rank == 0:
        print(json.dumps(line))
    eng.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
