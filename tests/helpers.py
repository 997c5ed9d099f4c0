"""Shared test helpers: build a workload from tn_inputs and run the oracle."""
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
