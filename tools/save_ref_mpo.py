"""Save the CPU-built reference MPO of a full-size parity case next to the stored oracle outputs
(tests/golden/local/, git-ignored: 210 MB at C4) so that a GPU run from THIS checkout uses bit for bit the
input the oracle used.  The test checks its fingerprints against tests/golden/full_<case>_ref.npz and the
per-site norms stored with the oracle outputs.  Usage: python tools/save_ref_mpo.py --case c4"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="c4", choices=sorted(C.FULL_PARITY_CASES))
a = ap.parse_args()
cfg = C.full_parity_config(a.case)
ref = [x.detach().resolve_conj().cpu().numpy() for x in C.reference_mpo(cfg, device="cpu")]
bonds, norms = C.ref_fingerprint(ref)
g = [f for f in sorted(os.listdir(os.path.join(ROOT, "tests", "golden"))) if f.startswith(f"full_{a.case}") and f.endswith(".npz") and "_ref" not in f]
o = np.load(os.path.join(ROOT, "tests", "golden", g[0]))
print("bonds equal:", bonds == [int(b) for b in o["ref_bonds"]], " per-site norms max rel diff vs the oracle's:",
      float(np.max(np.abs(norms - o["ref_norms"]) / o["ref_norms"])))
os.makedirs(os.path.join(ROOT, "tests", "golden", "local"), exist_ok=True)
np.savez(os.path.join(ROOT, "tests", "golden", "local", f"full_{a.case}_refmpo.npz"), **{f"s{j}": x for j, x in enumerate(ref)})
print("saved", len(ref), "sites")
