"""Time the fused step (tn_hvp_step) and its unfused parts at a config: A/B tool for engine switches
(environment variables are read by the library at engine creation)."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--max-batch", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--gates", default="haar")
ap.add_argument("--tag", default="")
ap.add_argument("--ref", default="torch", choices=["torch", "tebd"], help="reference built by tn_inputs (torch, GPU) or the library TEBD (bench.py)")
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
dev = torch.device("cuda")
if a.ref == "tebd":
    from paper_2604_20384_b200.api import mpo_tebd
    ref = mpo_tebd(cfg.n, C.reference_layers(cfg), cfg.chi)
else:
    ref = C.reference_mpo(cfg, device=dev)
B = a.batch or cfg.batch
K = C.num_gates(cfg.n, cfg.depth)
Gn = C.haar_gates(cfg.cid, K) if a.gates == "haar" else C.trotter_init_gates(cfg, 0)
G = torch.tensor(Gn, device=dev)
V = torch.tensor(C.tangent_directions(cfg.cid, Gn, B), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=a.max_batch or SUB_BATCH[cfg.cid])


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3, r


out = {"config": cfg.name, "tag": a.tag, "batch": B, "step_s": [], "env_s": [], "apply_s": [],
       "env": {k: v for k, v in os.environ.items() if k.startswith("TN_")}}
from paper_2604_20384_b200 import _native as N  # noqa: E402
eng.step(G, V)
out["stats_first"] = eng.split_stats()
out["launches"] = []
for _ in range(a.reps):
    l0 = N.tn_hvp_launch_count()
    t, r = timed(lambda: eng.step(G, V))
    out["step_s"].append(round(t, 4))
    out["launches"].append(N.tn_hvp_launch_count() - l0)
out["stats"] = eng.split_stats()
for _ in range(a.reps):
    t, r = timed(lambda: eng.environments(G))
    out["env_s"].append(round(t, 4))
    sc = r[0]
    t, _ = timed(lambda: eng.apply(V))
    out["apply_s"].append(round(t, 4))
out.update({"f": sc[0].item(), "fallbacks": sc[6].item(), "deflations": sc[7].item(),
            "hvps_per_s": B / min(out["step_s"])})
print(json.dumps(out))
