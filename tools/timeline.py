"""GPU timeline of one tn_hvp_environments (or fused step) call via CUPTI
(torch.profiler): wall time, union of busy intervals over all streams (how
idle the GPU is during the latency-bound primal sweeps), per-stream busy time,
kernel-time shares and the idle gaps of the busiest stream.

  python tools/timeline.py --config 4 [--what env|step] > profiles/<name>.json
"""
import argparse
import collections
import json
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--what", default="env", choices=["env", "step"])
ap.add_argument("--batch", type=int, default=None)
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
dev = torch.device("cuda")
ref = C.reference_mpo(cfg, device=dev)
K = C.num_gates(cfg.n, cfg.depth)
Gn = C.haar_gates(cfg.cid, K)
G = torch.tensor(Gn, device=dev)
B = a.batch or cfg.batch
V = torch.tensor(C.tangent_directions(cfg.cid, Gn, B), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=SUB_BATCH[cfg.cid])
run = (lambda: eng.environments(G)) if a.what == "env" else (lambda: eng.step(G, V))
run()
torch.cuda.synchronize()
t0 = time.time()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
wall = time.time() - t0
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
        ev.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0), e.name))
ev.sort()
t_first, t_last = ev[0][0], max(x[1] for x in ev)
# union of busy intervals
busy, cur_s, cur_e = 0.0, None, None
for s, e, _, _ in ev:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
per_stream = collections.defaultdict(float)
per_kernel = collections.defaultdict(lambda: [0, 0.0])
for s, e, sid, name in ev:
    per_stream[sid] += e - s
    short = name.replace("void ", "").split("(")[0]
    if "zgemm3m" in short:
        short = "tn::zgemm3m_kernel"
    elif "<" in short:
        short = short[:short.find("<")]
    per_kernel[short][0] += 1
    per_kernel[short][1] += e - s
span = t_last - t_first
top_sid = max(per_stream, key=per_stream.get)
gaps = []
prev = None
for s, e, sid, _ in ev:
    if sid != top_sid:
        continue
    if prev is not None and s > prev:
        gaps.append(s - prev)
    prev = e if prev is None else max(prev, e)
gaps.sort()
out = {
    "config": cfg.name, "what": a.what, "directions": B if a.what == "step" else 0,
    "wall_s_under_profiler": wall, "gpu_span_ms": span / 1e3, "gpu_busy_union_ms": busy / 1e3,
    "busy_fraction": busy / span, "kernels": len(ev),
    "per_stream_busy_ms": {str(k): v / 1e3 for k, v in sorted(per_stream.items(), key=lambda kv: -kv[1])},
    "busiest_stream_gaps": {"count": len(gaps), "sum_ms": sum(gaps) / 1e3,
                            "median_us": gaps[len(gaps) // 2] if gaps else None,
                            "p90_us": gaps[int(0.9 * len(gaps))] if gaps else None},
    "kernel_ms": {k: [n, t / 1e3] for k, (n, t) in sorted(per_kernel.items(), key=lambda kv: -kv[1][1])[:20]},
}
print(json.dumps(out, indent=1))
