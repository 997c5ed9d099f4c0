"""Shared test helpers: build a workload from tn_inputs and run the oracle (O3, or O2
for the dense plain definition), plus the per-gate comparison."""
import numpy as np

from oracle import common as cm
from oracle import mpo as M
from tn_inputs import configs as C
from tn_inputs.reference import mpo_bonds, reference_mpo


def workload(cfg, nb=None, ref_device="cpu", ref_chi=None):
    ref = reference_mpo(C.reference_layers(cfg), cfg.n, ref_chi or cfg.chi, device=ref_device)
    K = C.num_gates(cfg.n, cfg.depth, cfg.first_offset)
    G = C.haar_gates(cfg.cid, K)
    V = C.tangent_directions(cfg.cid, G, nb if nb is not None else cfg.batch)
    return ref, G, V


def oracle_outputs(cfg, ref, G, V, dirs=None):
    """f, grad_R, Hess_R[V_b] (b in dirs), H_T, Omega from O3."""
    refs = [a.detach().resolve_conj().cpu().numpy() for a in ref]
    o3 = M.MPOOracle(cfg.n, cfg.depth, cfg.chi, G, refs, V, cfg.first_offset)
    E = o3.gradient_T()
    f, grad_f, _ = cm.postprocess_gradient(o3.T, E)
    gR = cm.riemannian_gradient(G, grad_f)
    dirs = range(V.shape[0]) if dirs is None else dirs
    HR, HT, OM = {}, {}, {}
    for b in dirs:
        H = o3.hvp_T(b)
        Hf, om = cm.postprocess_hvp(o3.T, E, H, V[b])
        HR[b] = cm.riemannian_hvp(G, grad_f, Hf, V[b])
        HT[b], OM[b] = H, om
    return {"T": o3.T, "f": f, "E": E, "grad_R": gR, "HR": HR, "HT": HT, "OM": OM, "oracle": o3}


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def o2_outputs(cfg, ref, G, V, dirs=None):
    """The same outputs from O2 (oracle/dense.py DenseTruncated): the truncated
    definition written out on 4^n vectors with explicit Schmidt projectors
    (the plain definition; n <= 8)."""
    from oracle import dense as O
    from tn_inputs.reference import mpo_to_dense_operator
    n = cfg.n
    U = mpo_to_dense_operator(ref)                      # U_ref / 2^{n/2} (normalised MPO)
    o2 = O.DenseTruncated(n, cfg.depth, cfg.chi, G, O.op_to_vec(U, n), mpo_bonds(ref), V, cfg.first_offset)
    E = o2.gradient_T()
    f, grad_f, _ = cm.postprocess_gradient(o2.T, E)
    gR = cm.riemannian_gradient(G, grad_f)
    dirs = range(V.shape[0]) if dirs is None else dirs
    HR, HT, OM = {}, {}, {}
    for b in dirs:
        H = o2.hvp_T(b)
        Hf, om = cm.postprocess_hvp(o2.T, E, H, V[b])
        HR[b] = cm.riemannian_hvp(G, grad_f, Hf, V[b])
        HT[b], OM[b] = H, om
    return {"T": o2.T, "f": f, "E": E, "grad_R": gR, "HR": HR, "HT": HT, "OM": OM}


def gatewise(g, o, tol, floor=1e-3):
    """Per-gate relative error of [K][4][4] outputs: max_k ||g_k - o_k|| /
    max(||o_k||, floor * rms_k ||o_k||) -- each gate against its own norm, with
    an absolute floor at 1e-3 of the average gate norm so that a gate whose
    exact value is ~0 is judged on the output's scale (X18 per-gate reading).
    Asserts <= tol and returns (worst error, worst gate)."""
    g = np.asarray(g).reshape(-1, 16)
    o = np.asarray(o).reshape(-1, 16)
    on = np.linalg.norm(o, axis=1)
    rms = float(np.sqrt(np.mean(on ** 2)))
    err = np.linalg.norm(g - o, axis=1) / np.maximum(on, floor * rms)
    k = int(np.argmax(err))
    assert err[k] <= tol, f"gate {k}: per-gate relative error {err[k]:.3e} > {tol:.0e} (|o_k| = {on[k]:.3e}, rms {rms:.3e})"
    return float(err[k]), k
