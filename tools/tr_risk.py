"""The paper's training experiment in miniature:
compress the config's Trotter reference into its brickwall circuit by a
Riemannian trust region on the sampled-state empirical risk (S Haar product
training states), then evaluate the risk on fresh test states.  Every f,
gradient and HVP comes from the state-mode engines (risk.EmpiricalRisk).
One JSON line.

  python tools/tr_risk.py --config 3 --train 8 --test 8 --outer 10
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import mpo_tebd  # noqa: E402
from paper_2604_20384_b200.risk import EmpiricalRisk  # noqa: E402
from paper_2604_20384_b200.trust_region import TRParams, TrustRegion  # noqa: E402
from tn_inputs import configs as C  # noqa: E402
from tn_inputs import samples as SMP  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--train", type=int, default=8)
ap.add_argument("--test", type=int, default=8)
ap.add_argument("--outer", type=int, default=10)
ap.add_argument("--max-hvp", type=int, default=20)
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
dev = torch.device("cuda")
t0 = time.time()
ref = [x.cpu().numpy() for x in mpo_tebd(cfg.n, C.reference_layers(cfg), cfg.chi)]
psis = SMP.haar_product_states(cfg.cid, a.train + a.test, cfg.n)


def risk_engine(ps):
    labels = [[torch.tensor(x, device=dev) for x in SMP.label_mps(ref, p)] for p in ps]
    return EmpiricalRisk(cfg.n, cfg.depth, cfg.chi, labels, ps, cfg.first_offset, max_batch=1)


train = risk_engine(psis[:a.train])
x0 = torch.tensor(C.trotter_init_gates(cfg, 0), device=dev)
tp = time.time()
x, f, tr = TrustRegion(train, TRParams(outer=a.outer, max_hvp=a.max_hvp)).run(x0)
torch.cuda.synchronize()
t_tr = time.time() - tp
train.close()
test = risk_engine(psis[a.train:])
test_0 = float(test.cost(x0).item())
test_1 = float(test.cost(x).item())
test.close()
print(json.dumps({
    "config": cfg.name, "train_states": a.train, "test_states": a.test, "outer": a.outer,
    "train_risk": [tr.records[0]["f"]] + [r["f_trial"] for r in tr.records if r.get("accepted")],
    "test_risk_start": test_0, "test_risk_end": test_1, "hvps": tr.hvps, "grads": tr.grads,
    "tr_seconds": t_tr, "wall_s": time.time() - t0,
    "trace": [{k: v for k, v in r.items() if k in ("iter", "f", "rho", "accepted", "n_hvp", "delta", "tcg_stop")}
              for r in tr.records]}))
