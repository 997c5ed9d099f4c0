"""GPU vs oracle at a full config (sampled directions).  Prints one JSON line."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import common as cm  # noqa: E402
from oracle import mpo as M  # noqa: E402
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--dirs", type=int, default=1)
ap.add_argument("--no-hvp", action="store_true")
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
dev = torch.device("cuda")
ref = C.reference_mpo(cfg, device=dev)
K = C.num_gates(cfg.n, cfg.depth)
G = C.haar_gates(cfg.cid, K)
V = C.tangent_directions(cfg.cid, G, a.dirs)
out = {"config": cfg.name}
for m in ("eigh",):
    os.environ["TN_SVD"] = m
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=a.dirs)
    sc, gR = eng.environments(torch.tensor(G, device=dev))
    H = eng.apply(torch.tensor(V, device=dev))
    torch.cuda.synchronize()
    out[m] = {"f": sc[0].item(), "gR": gR.cpu().numpy(), "H": H.cpu().numpy(), "diag": sc[3:8].tolist()}
    eng.close()
t0 = time.time()
o = M.MPOOracle(cfg.n, cfg.depth, cfg.chi, G, [x.detach().resolve_conj().cpu().numpy() for x in ref], V)
E = o.gradient_T()
f, gf, _ = cm.postprocess_gradient(o.T, E)
gR = cm.riemannian_gradient(G, gf)
HR = []
if not a.no_hvp:
    for b in range(a.dirs):
        Hf, _ = cm.postprocess_hvp(o.T, E, o.hvp_T(b), V[b])
        HR.append(cm.riemannian_hvp(G, gf, Hf, V[b]))
out["oracle_s"] = time.time() - t0
rel = lambda x, y: float(np.linalg.norm(np.ravel(x - y)) / np.linalg.norm(np.ravel(y)))
res = {"config": cfg.name, "oracle_f": f, "oracle_seconds": out["oracle_s"]}
for m in ("eigh",):
    r = {"f_rel": abs(out[m]["f"] - f) / abs(f), "grad_R_rel": rel(out[m]["gR"], gR), "diag": out[m]["diag"]}
    if HR:
        r["hess_R_rel"] = max(rel(out[m]["H"][b], HR[b]) for b in range(a.dirs))
    res[m] = r
print(json.dumps(res))
