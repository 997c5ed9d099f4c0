"""Full-size parity, default on: the CUDA path at C3, C4 and a full-width C5
case against oracle outputs stored in tests/golden/ by tools/golden_full.py
(which calls only oracle/ and tn_inputs/; commands and oracle timings in the
.json beside each .npz).

Definition checked: the truncated fixed-projector HVP (SURVEY.md §8(c.2),
readings X7-X9).  Launch configuration: bench.py's --
the config's full direction batch in SUB_BATCH sub-batches through the fused
tn_hvp_step; the stored directions are the first of that batch.  Bar
(north_star): relative error <= 1e-10 for f, grad_R and every stored
direction's Hess_R, whole-output and per gate (tests/helpers.gatewise).

"c5r" is config 5 at full width and bond cap (n = 128, chi = 256, C5's
reference MPO, X17 trust-region start) at depth 4: the full-depth C5 oracle
does not fit the oracle machine's memory.  It reaches the noise-floor /
deflation split paths of the trust-region regime; the full-depth C5 engine is
covered by the identities of test_gpu_parity.py::test_full_size_properties_config5.

The reference MPO is rebuilt with the CPU path of tn_inputs.reference (the
same input the oracle used); its bonds and its operator Schmidt values at every
cut (gauge invariant) are checked against tests/golden/full_<case>_ref.npz.
"""
import json
import os
import time

import numpy as np
import pytest
import torch

from tests.helpers import gatewise, rel
from tn_inputs import configs as C

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
TOL = 1e-10


def _load(case):
    """Stored oracle outputs: full_<case>.npz (the first `dirs` directions) and/or
    per-direction files full_<case>_d<b>.npz (tools/golden_full.py --only b).
    -> (f, T, grad_R, {direction index: Hess_R})."""
    files = [os.path.join(GOLDEN, f"full_{case}.npz")] + sorted(
        os.path.join(GOLDEN, x) for x in os.listdir(GOLDEN) if x.startswith(f"full_{case}_d") and x.endswith(".npz"))
    files = [x for x in files if os.path.exists(x)]
    if not files:
        pytest.skip(f"no stored oracle outputs for {case} in tests/golden (python tools/golden_full.py --case {case})")
    HR, base = {}, None
    for path in files:
        o = np.load(path)
        with open(path.replace(".npz", ".json")) as fh:
            meta = json.load(fh)
        first = int(meta.get("first_dir", 0))
        for j in range(int(meta["dirs"])):
            HR[first + j] = o["HR"][j]
        if base is None:
            base = o
        else:                                  # the pieces were computed at the same point and reference
            assert abs(float(o["f"]) - float(base["f"])) <= 1e-13 * abs(float(base["f"]))
    return base, HR


@pytest.mark.parametrize("case", list(C.FULL_PARITY_CASES))
def test_full_size_parity(case):
    from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine, riemannian_project
    o, HRo = _load(case)
    nd = max(HRo) + 1
    cfg, G, V0 = C.full_parity_inputs(case, nd)
    t0 = time.time()
    # the oracle's own input when this checkout has it (tools/save_ref_mpo.py; git-ignored), else a CPU rebuild
    local = os.path.join(GOLDEN, "local", f"full_{case}_refmpo.npz")
    if os.path.exists(local):
        z = np.load(local)
        ref_cpu = [torch.tensor(z[f"s{j}"]) for j in range(cfg.n)]
        ref_source = "tests/golden/local (the oracle's input)"
    else:
        ref_cpu = C.reference_mpo(cfg, device="cpu")
        ref_source = "rebuilt on this machine's CPU"
    t_ref = time.time() - t0
    # Same input as the oracle's?  Bonds, operator Schmidt values at every cut and overlaps with fixed probe
    # MPOs (all gauge invariant; tools/golden_ref_spectra.py).  The truncated reference of a symmetric model
    # (C4: XXZ) has near-degenerate Schmidt values at its bond cap, where the kept vectors depend on the SVD
    # routine's rounding: a rebuild on another machine can be ANOTHER operator (reading X25).  That is a
    # difference of inputs, not of outputs, so the comparison is skipped with the evidence, not failed.
    ref_np = [x.numpy() for x in ref_cpu]
    bonds, _ = C.ref_fingerprint(ref_np)
    rs = np.load(os.path.join(GOLDEN, f"full_{case}_ref.npz"))
    mismatch = None
    if bonds != [int(b) for b in o["ref_bonds"]]:
        mismatch = "bonds differ"
    else:
        worst = max(float(np.abs(sv - rs[f"cut{j + 1}"]).max() / rs[f"cut{j + 1}"][0])
                    for j, sv in enumerate(C.ref_schmidt_spectra(ref_np)))
        if worst > 1e-10:
            mismatch = f"operator Schmidt values differ by {worst:.1e} of the largest"
        elif "probe_mantissa" in rs.files:
            pm, pl = C.ref_probe_overlaps(ref_np)
            if not (np.abs(pl - rs["probe_log10"]).max() <= 1e-8
                    and np.abs(pm - rs["probe_mantissa"]).max() <= 1e-8 * np.abs(rs["probe_mantissa"]).max()):
                mismatch = "overlaps with the probe MPOs differ"
    if mismatch:
        pytest.skip(f"{case}: the reference MPO {ref_source} is another operator than the one the stored oracle "
                    f"outputs were computed on ({mismatch}): inputs differ, nothing to compare")
    dev = torch.device("cuda")
    batch = max(cfg.batch, nd)
    V = C.tangent_directions(cfg.cid, G, batch)
    assert np.array_equal(V[:nd], V0)
    mb = SUB_BATCH[cfg.cid] if case != "c5r" else 1
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [x.to(dev) for x in ref_cpu], cfg.first_offset, max_batch=mb)
    Gt, Vt = torch.tensor(G, device=dev), torch.tensor(V, device=dev)
    sc, gR, H = eng.step(Gt, Vt)                       # bench.py's step
    torch.cuda.synchronize()
    split_stats = eng.split_stats()
    f = sc[0].item()
    T = complex(sc[1].item(), sc[2].item())
    gR, Hn = gR.cpu().numpy(), H.cpu().numpy()
    report = {"case": case, "reference": ref_source, "t_reference_cpu_s": t_ref, "f_rel": abs(f - float(o["f"])) / abs(float(o["f"])),
              "T_rel": abs(T - complex(o["T"])) / abs(complex(o["T"])), "grad_R_rel": rel(gR, o["grad_R"]),
              "grad_R_gate": gatewise(gR, o["grad_R"], TOL), "diag": sc[3:8].cpu().tolist(),
              "split_stats": split_stats}
    assert report["f_rel"] <= TOL and report["T_rel"] <= TOL
    assert report["grad_R_rel"] <= TOL
    report["hess_R_rel"], report["hess_R_gate"] = {}, {}
    for b in sorted(HRo):
        report["hess_R_rel"][b] = rel(Hn[b], HRo[b])
        report["hess_R_gate"][b] = gatewise(Hn[b], HRo[b], TOL)
        assert report["hess_R_rel"][b] <= TOL, b
    print(json.dumps(report))
    # identities at full size on the same engine (any-size properties):
    # every output in the tangent space, Hess_R real-linear in V
    assert rel(riemannian_project(Gt, torch.tensor(gR, device=dev)).cpu().numpy(), gR) < 1e-13
    assert rel(riemannian_project(Gt, H).cpu().numpy(), Hn) < 1e-13
    comb = torch.stack([Vt[0] + 2.5 * Vt[1 % batch], Vt[1 % batch]]).contiguous()
    Hc = eng.apply(comb).cpu().numpy()
    assert rel(Hc[0], Hn[0] + 2.5 * Hn[1 % batch]) < 1e-11
    eng.close()
