"""Oracle outputs at a full BASELINE.json config, for sampled full-size parity.

Calls only oracle/ and tn_inputs/ (no CUDA path): the reference MPO is built
with the CPU path of tn_inputs.reference, the circuit and directions are the
config's seeded inputs, and O3 gives f, T, E, grad_R and Hess_R for `--dirs`
directions.  Writes profiles/r01_oracle_c<cid>.npz plus a JSON line with the
oracle's own timing.  tools/parity_from_file.py runs the GPU side on the
same inputs and compares.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import common as cm  # noqa: E402
from oracle import mpo as M  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--dirs", type=int, default=1)
ap.add_argument("--out", default=None)
ap.add_argument("--save-ref", default=None, help="also np.save the reference sites (object array) here")
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
t0 = time.time()
ref = [x.detach().resolve_conj().cpu().numpy() for x in C.reference_mpo(cfg, device="cpu")]
t_ref = time.time() - t0
if a.save_ref:
    arr = np.empty(len(ref), dtype=object)
    arr[:] = ref
    np.save(a.save_ref, arr, allow_pickle=True)
K = C.num_gates(cfg.n, cfg.depth)
G = C.haar_gates(cfg.cid, K)
V = C.tangent_directions(cfg.cid, G, a.dirs)
t1 = time.time()
o = M.MPOOracle(cfg.n, cfg.depth, cfg.chi, G, ref, V)
E = o.gradient_T()
f, gf, _ = cm.postprocess_gradient(o.T, E)
gR = cm.riemannian_gradient(G, gf)
HR = []
for b in range(a.dirs):
    Hf, _ = cm.postprocess_hvp(o.T, E, o.hvp_T(b), V[b])
    HR.append(cm.riemannian_hvp(G, gf, Hf, V[b]))
t_or = time.time() - t1
out = a.out or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            f"r01_oracle_c{cfg.cid}.npz")
np.savez(out, f=f, T=o.T, E=E, grad_R=gR, HR=np.array(HR), dirs=a.dirs,
         ref_sum=np.array([np.abs(x).sum() for x in ref]))
print(json.dumps({"config": cfg.name, "dirs": a.dirs, "t_reference_s": t_ref, "t_oracle_s": t_or, "f": f,
                  "file": out}))
