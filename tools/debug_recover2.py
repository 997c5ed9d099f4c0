"""Narrow the post-failure recovery bug: which pass (failed / good) must be threaded."""
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
V = torch.tensor(C.tangent_directions(81, G, 1), device=dev)
Gbad = G.copy()
Gbad[3, 1, 2] = np.nan


def mode(serial):
    if serial:
        os.environ["TN_SERIAL_PRIMAL"] = "1"
    else:
        os.environ.pop("TN_SERIAL_PRIMAL", None)


def run(nan_serial, good_serial, good_twice=False, clean_first=True):
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=1)
    mode(False)
    H0 = None
    if clean_first:
        eng.environments(torch.tensor(G, device=dev))
        H0 = eng.apply(V).clone()
    mode(nan_serial)
    try:
        eng.environments(torch.tensor(Gbad, device=dev))
    except N.TNError:
        pass
    mode(good_serial)
    eng.environments(torch.tensor(G, device=dev))
    if good_twice:
        eng.environments(torch.tensor(G, device=dev))
    H, HT, OM = eng.apply(V, aux=True)
    torch.cuda.synchronize()
    r = {"nan_serial": nan_serial, "good_serial": good_serial, "good_twice": good_twice,
         "H_finite": bool(torch.isfinite(H).all()), "HT_finite": bool(torch.isfinite(HT).all()),
         "OM_finite": bool(torch.isfinite(OM).all())}
    if H0 is not None:
        r["H_equal_clean"] = bool(torch.equal(H, H0))
    H2 = eng.apply(V)
    r["second_apply_finite"] = bool(torch.isfinite(H2).all())
    print(r, flush=True)
    eng.close()
    mode(False)


for ns, gs, tw in [(False, False, False), (False, False, True), (True, False, False), (False, True, False),
                   (True, True, False)]:
    run(ns, gs, tw)
run(False, False, False, clean_first=False)
