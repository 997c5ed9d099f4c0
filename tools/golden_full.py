"""Stored oracle outputs for the default-on full-size parity tests.

Writes tests/golden/full_<name>.npz (+ .json: command, timing, citation).
Calls only oracle/ and tn_inputs/ -- nothing of the CUDA path -- so every
expected value in those files comes from the oracle O3 (oracle/mpo.py, the
truncated definition of SURVEY.md §8(c.2), readings X7-X9; the HVP
definition checked is the fixed-projector one) on the
config's seeded inputs:

  * the reference MPO is rebuilt by tn_inputs.reference on the CPU (its hash
    of bonds and site norms is stored so the GPU test can check that it
    rebuilt the same input);
  * gates: Haar (stream (cid, "gates", k)) for C3/C4; the X17 Trotter start
    for the reduced-depth C5 case "c5r" (n=128, chi=256, D=4, C5's reference);
  * directions: the first --dirs of the config's seeded batch, i.e. the same
    directions the bench launch configuration processes first.

Usage: python tools/golden_full.py --case c4 --dirs 2
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import common as cm  # noqa: E402
from oracle import mpo as M  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="c4", choices=sorted(C.FULL_PARITY_CASES))
ap.add_argument("--dirs", type=int, default=2)
ap.add_argument("--only", type=int, default=None,
                help="compute just direction ONLY (its tangent alone in the sweeps) -> full_<case>_d<ONLY>.npz")
a = ap.parse_args()

cfg, G, V = C.full_parity_inputs(a.case, a.dirs if a.only is None else a.only + 1)
if a.only is not None:
    V = V[a.only:a.only + 1]
t0 = time.time()
ref = [x.detach().resolve_conj().cpu().numpy() for x in C.reference_mpo(cfg, device="cpu")]
t_ref = time.time() - t0
print(json.dumps({"case": a.case, "t_reference_s": t_ref, "bonds": [int(x.shape[2]) for x in ref]}), flush=True)
t1 = time.time()
o = M.MPOOracle(cfg.n, cfg.depth, cfg.chi, G, ref, V, cfg.first_offset)
t_primal = time.time() - t1
E = o.gradient_T()
f, gf, _ = cm.postprocess_gradient(o.T, E)
gR = cm.riemannian_gradient(G, gf)
t_env = time.time() - t1
print(json.dumps({"case": a.case, "t_primal_s": t_primal, "t_env_s": t_env, "f": f}), flush=True)
HR, t_dirs = [], []
for b in range(V.shape[0]):
    tb = time.time()
    Hf, _ = cm.postprocess_hvp(o.T, E, o.hvp_T(b), V[b])
    HR.append(cm.riemannian_hvp(G, gf, Hf, V[b]))
    t_dirs.append(time.time() - tb)
    print(json.dumps({"case": a.case, "dir": b, "t_s": t_dirs[-1]}), flush=True)
out = os.path.join(ROOT, "tests", "golden",
                   f"full_{a.case}.npz" if a.only is None else f"full_{a.case}_d{a.only}.npz")
np.savez_compressed(out, f=f, T=o.T, grad_R=gR, HR=np.array(HR).reshape(V.shape[0], -1, 4, 4),
                    ref_bonds=np.array(C.ref_fingerprint(ref)[0]), ref_norms=C.ref_fingerprint(ref)[1])
meta = {"case": a.case, "config": cfg.name, "n": cfg.n, "depth": cfg.depth, "chi": cfg.chi,
        "dirs": V.shape[0], "first_dir": 0 if a.only is None else a.only,
        "command": f"python tools/golden_full.py --case {a.case} " + (f"--dirs {a.dirs}" if a.only is None
                                                                       else f"--only {a.only}"),
        "oracle": "oracle/mpo.py MPOOracle (O3), oracle/common.py postprocessing",
        "definition": "truncated fixed-projector HVP, SURVEY.md 8(c.2), readings X7-X9; PAPER.md:1019-1023",
        "t_reference_s": t_ref, "t_primal_s": t_primal, "t_env_s": t_env, "t_dir_s": t_dirs,
        "f": f, "T": [o.T.real, o.T.imag], "remainder": o.diag["remainder"],
        "min_gap": min(d["gap"] for d in o.diag["bottom"] + o.diag["top"]),
        "threads": os.environ.get("OMP_NUM_THREADS", "all"), "nproc": os.cpu_count()}
with open(out.replace(".npz", ".json"), "w") as fh:
    json.dump(meta, fh, indent=1)
print(json.dumps(meta), flush=True)
