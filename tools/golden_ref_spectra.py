"""Gauge-invariant fingerprint of the reference MPO a full-size parity case was
generated on: its operator Schmidt values at every cut (tn_inputs.configs.
ref_schmidt_spectra), written to tests/golden/full_<case>_ref.npz.  The GPU test
rebuilds the reference on the GPU box's CPU (other LAPACK rounding, so another
bond gauge) and checks it is the same operator before comparing outputs.
Calls only tn_inputs/.  Usage: python tools/golden_ref_spectra.py --case c4"""
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
spec = C.ref_schmidt_spectra(ref)
probe_m, probe_l = C.ref_probe_overlaps(ref)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"full_{a.case}_ref.npz"),
                    bonds=np.array([1] + [x.shape[2] for x in ref]), probe_mantissa=probe_m, probe_log10=probe_l,
                    **{f"cut{j + 1}": s for j, s in enumerate(spec)})
print(a.case, "cuts", len(spec), "max bond", max(x.shape[2] for x in ref))
