"""GPU side of the sampled full-size parity (tools/oracle_full.py wrote the
oracle outputs): the same seeded inputs, the reference MPO rebuilt with the
CPU path of tn_inputs.reference, the engine in bench.py's launch
configuration (the config's full direction batch in SUB_BATCH sub-batches,
fused tn_hvp_step); compares f, grad_R and Hess_R of the oracle's directions
(the first `dirs` of the batch).  Prints one JSON line."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--file", default=None)
ap.add_argument("--ref", default=None, help="reference sites saved by oracle_full.py --save-ref (same CPU build)")
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
path = a.file or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                              f"r01_oracle_c{cfg.cid}.npz")
o = np.load(path)
t0 = time.time()
if a.ref:
    ref_cpu = [torch.from_numpy(x) for x in np.load(a.ref, allow_pickle=True)]
else:
    ref_cpu = C.reference_mpo(cfg, device="cpu")
t_ref = time.time() - t0
ref_sum = np.array([float(x.abs().sum()) for x in ref_cpu])
dev = torch.device("cuda")
ref = [x.to(dev) for x in ref_cpu]
K = C.num_gates(cfg.n, cfg.depth)
G = C.haar_gates(cfg.cid, K)
V = C.tangent_directions(cfg.cid, G, cfg.batch)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=SUB_BATCH[cfg.cid])
sc, gR, H = eng.step(torch.tensor(G, device=dev), torch.tensor(V, device=dev))
torch.cuda.synchronize()
f = sc[0].item()
gR, H = gR.cpu().numpy(), H.cpu().numpy()


def rel(x, y):
    return float(np.linalg.norm(np.ravel(x - y)) / np.linalg.norm(np.ravel(y)))


nd = int(o["dirs"])
print(json.dumps({
    "config": cfg.name, "launch": {"directions": cfg.batch, "sub_batch": SUB_BATCH[cfg.cid], "call": "tn_hvp_step"},
    "reference_rebuild_rel_diff": float(np.abs(ref_sum - o["ref_sum"]).max() / np.abs(o["ref_sum"]).max()),
    "t_reference_cpu_s": t_ref, "oracle_f": float(o["f"]), "gpu_f": f,
    "f_rel": abs(f - float(o["f"])) / abs(float(o["f"])), "grad_R_rel": rel(gR, o["grad_R"]),
    "hess_R_rel": [rel(H[b], o["HR"][b]) for b in range(nd)] if nd else None,
    "diag": sc[3:8].cpu().tolist()}))
