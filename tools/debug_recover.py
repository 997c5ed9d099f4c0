"""Diagnose recovery after a failed (NaN) primal pass (tests/test_gpu_kernels.py::test_error_statuses)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200 import _native as N  # noqa: E402
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402
from tn_inputs.reference import reference_mpo  # noqa: E402

cfg = C.small_case(81, 6, 4, 8, batch=1)
ref = reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)
K = C.num_gates(cfg.n, cfg.depth)
G = C.haar_gates(81, K)
dev = torch.device("cuda")
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=1)
V = torch.tensor(C.tangent_directions(81, G, 1), device=dev)
sc, gR = eng.environments(torch.tensor(G, device=dev))
H0 = eng.apply(V).clone()
E0 = eng.gradient_T().clone()
print("clean: f", sc[0].item(), "finite H", bool(torch.isfinite(H0).all()))
Gbad = G.copy()
Gbad[3, 1, 2] = np.nan
try:
    eng.environments(torch.tensor(Gbad, device=dev))
except N.TNError as e:
    print("nan run:", e)
sc, gR = eng.environments(torch.tensor(G, device=dev))
torch.cuda.synchronize()
E1 = eng.gradient_T()
print("recovered: f", sc[0].item(), "grad finite", bool(torch.isfinite(gR).all()), "E equal", bool(torch.equal(E0, E1)))
H1 = eng.apply(V)
print("H finite", bool(torch.isfinite(H1).all()), "H equal", bool(torch.equal(H0, H1)),
      "nonfinite gates", torch.nonzero(~torch.isfinite(H1[0]).all(-1).all(-1)).flatten().tolist())
