"""Per-step times of a series of fused steps with the device's free memory after each (diagnostic)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine, mpo_tebd  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=8)
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
dev = torch.device("cuda")
ref = mpo_tebd(cfg.n, C.reference_layers(cfg), cfg.chi)
K = C.num_gates(cfg.n, cfg.depth)
Gn = C.haar_gates(cfg.cid, K)
G = torch.tensor(Gn, device=dev)
V = torch.tensor(C.tangent_directions(cfg.cid, Gn, cfg.batch), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=SUB_BATCH[cfg.cid])
out = torch.empty_like(V)
rows = []
for i in range(a.n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.step(G, V, out=out)
    e1.record()
    torch.cuda.synchronize()
    fr, tot = torch.cuda.mem_get_info()
    rows.append({"step": i, "s": round(e0.elapsed_time(e1) / 1e3, 4), "free_gb": round(fr / 2**30, 2)})
print(json.dumps({"config": cfg.name, "env": {k: v for k, v in os.environ.items() if k.startswith("TN_")}, "steps": rows}))
