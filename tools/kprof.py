"""Kernel-time breakdown of one environments / apply call via torch.profiler (CUPTI)."""
import argparse
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--max-batch", type=int, default=64)
ap.add_argument("--what", default="apply", choices=["apply", "env", "step"])
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
dev = torch.device("cuda")
ref = C.reference_mpo(cfg, device=dev)
K = C.num_gates(cfg.n, cfg.depth)
Gn = C.haar_gates(cfg.cid, K)
G = torch.tensor(Gn, device=dev)
V = torch.tensor(C.tangent_directions(cfg.cid, Gn, a.batch), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=a.max_batch)
eng.environments(G)
eng.apply(V)
torch.cuda.synchronize()
import time  # noqa: E402
t0 = time.time()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if a.what == "env":
        eng.environments(G)
    elif a.what == "step":       # bench.py's step: fused tn_hvp_step
        eng.step(G, V)
    else:
        eng.apply(V)
    torch.cuda.synchronize()
wall = time.time() - t0
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        full = ev.name.replace("(anonymous namespace)::", "").replace("void ", "")
        name = full.split("(")[0]
        if "zgemm3m_kernel" in full:
            name = "tn::zgemm3m_kernel (DMMA complex GEMM)"
        elif "<" in name:
            name = name[:name.find("<")]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(f"{a.what} config {cfg.name} batch {a.batch} (sub-batch {a.max_batch}): kernels {sum(v[0] for v in agg.values())}, "
      f"summed kernel time {tot/1e3:.1f} ms, wall {wall*1e3:.1f} ms (streams overlap in the primal pass)")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{k[:70]:70s} {n:7d} {t/1e3:9.2f} ms {100*t/tot:5.1f}%")
