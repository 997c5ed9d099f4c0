"""Time tn_hvp_environments for a config and gate family; print split statistics."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
kind = sys.argv[2] if len(sys.argv) > 2 else "haar"
cfg = C.CONFIGS[cid]
dev = torch.device("cuda")
t = time.time()
ref = C.reference_mpo(cfg, device=dev)
torch.cuda.synchronize()
t_ref = time.time() - t
K = C.num_gates(cfg.n, cfg.depth)
G = C.haar_gates(cid, K) if kind == "haar" else C.trotter_init_gates(cfg, 0)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=1)
out = {"config": cfg.name, "gates": kind, "t_ref": t_ref}
for rep in range(2):
    torch.cuda.synchronize()
    t = time.time()
    sc, _ = eng.environments(torch.tensor(G, device=dev))
    torch.cuda.synchronize()
    out[f"t_env_{rep}"] = time.time() - t
out.update({"f": sc[0].item(), "fallbacks": sc[6].item(), "deflations": sc[7].item(), "min_gap": sc[4].item()})
V = torch.tensor(C.tangent_directions(cid, G, 1), device=dev)
t = time.time()
eng.apply(V)
torch.cuda.synchronize()
out["t_apply_1dir"] = time.time() - t
print(json.dumps(out))
