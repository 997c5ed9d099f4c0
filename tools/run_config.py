"""Time one config end to end on the GPU: reference build, environments, apply."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--max-batch", type=int, default=64)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
dev = torch.device("cuda")
t0 = time.time()
ref = C.reference_mpo(cfg, device=dev)
torch.cuda.synchronize()
t_ref = time.time() - t0
B = a.batch or cfg.batch
K = C.num_gates(cfg.n, cfg.depth)
G = torch.tensor(C.haar_gates(cfg.cid, K), device=dev)
V = torch.tensor(C.tangent_directions(cfg.cid, C.haar_gates(cfg.cid, K), B), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=a.max_batch)
out = {"config": cfg.name, "t_ref_build_s": t_ref, "ref_bonds_max": max(eng.ref_bonds)}
for rep in range(a.reps + 1):
    torch.cuda.synchronize()
    t0 = time.time()
    sc, gR = eng.environments(G)
    torch.cuda.synchronize()
    t1 = time.time()
    H = eng.apply(V)
    torch.cuda.synchronize()
    t2 = time.time()
out.update({"t_env_s": t1 - t0, "t_apply_s": t2 - t1, "batch": B, "f": sc[0].item(), "diag": sc[3:6].tolist()})
w_dir, w_pr = eng.work()
out.update({"cmac_per_dir": w_dir, "cmac_primal": w_pr,
            "apply_tflops": 8 * w_dir * B / (t2 - t1) / 1e12, "hvp_per_s": B / (t2 - t1),
            "step_hvp_per_s": B / (t2 - t0), "mem_gb": torch.cuda.max_memory_allocated() / 1e9,
            "device_used_gb": (torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9})
print(json.dumps(out))
