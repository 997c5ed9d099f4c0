"""Timings for the NEXT rows built this round (one B200, CUDA events on the
current stream, after a warm-up call):
  N2  translation-invariant HVPs at config 3 (tied layer gates, 64 directions)
  N3  the full Pauli-basis Riemannian Hessian at config 2 (16K = 960 HVPs),
      its symmetric-part spectrum, and a 10-step CG probe
Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine, sym_eig  # noqa: E402
from paper_2604_20384_b200.spectrum import cg_probe, hessian_matrix  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

dev = torch.device("cuda")


def timed(fn):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    out = fn()
    e1.record(st)
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / 1e3


res = {}
# ---- N2 at config 3
cfg = C.CONFIGS[3]
ref = C.reference_mpo(cfg, device=dev)
g = torch.tensor(C.haar_gates(3000, cfg.depth), device=dev)
v = torch.tensor(C.tangent_directions(3000, g.cpu().numpy(), cfg.batch), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=SUB_BATCH[3])
eng.ti_environments(g)
eng.ti_apply(v[:2])
(_, _), t_env = timed(lambda: eng.ti_environments(g))
_, t_app = timed(lambda: eng.ti_apply(v))
res["N2_ti_config3"] = {"workload": cfg.name, "layers": cfg.depth, "directions": cfg.batch,
                        "t_environments_s": t_env, "t_apply_s": t_app, "hvps_per_s": cfg.batch / t_app,
                        "step_hvps_per_s": cfg.batch / (t_env + t_app)}
eng.close()
del ref
torch.cuda.empty_cache()

# ---- N3 at config 2
cfg = C.CONFIGS[2]
ref = C.reference_mpo(cfg, device=dev)
K = C.num_gates(cfg.n, cfg.depth)
G = torch.tensor(C.haar_gates(2, K), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=64)
_, gR = eng.environments(G)
hessian_matrix(eng, G, chunk=64)
Mt, t_mat = timed(lambda: hessian_matrix(eng, G, chunk=64))
(w, asym), t_eig = timed(lambda: sym_eig(Mt))
(_, resid), t_cg = timed(lambda: cg_probe(eng, -gR, 10))
w = w.cpu().numpy()
a = asym.cpu().numpy()
res["N3_spectrum_config2"] = {
    "workload": cfg.name, "dim": 16 * K, "t_matrix_s": t_mat, "hvps_per_s": 16 * K / t_mat,
    "t_sym_eig_s": t_eig, "t_cg10_s": t_cg, "asymmetry": float(a[0] / a[1]),
    "eig_min": float(w[0]), "eig_max": float(w[-1]), "n_negative": int((w < -1e-12 * abs(w).max()).sum()),
    "cg_residuals": [float(x) for x in resid]}
eng.close()
print(json.dumps(res))
