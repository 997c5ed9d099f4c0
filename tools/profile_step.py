"""One profiled step (environments + apply) between cudaProfilerStart/Stop, for ncu."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--apply-only", action="store_true")
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
dev = torch.device("cuda")
ref = C.reference_mpo(cfg, device=dev)
K = C.num_gates(cfg.n, cfg.depth)
Gn = C.haar_gates(cfg.cid, K)
G = torch.tensor(Gn, device=dev)
V = torch.tensor(C.tangent_directions(cfg.cid, Gn, a.batch), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=a.batch)
eng.environments(G)
eng.apply(V)
torch.cuda.synchronize()
torch.cuda.profiler.start()
if not a.apply_only:
    eng.environments(G)
eng.apply(V)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
