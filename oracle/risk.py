"""N1: the sampled-state empirical risk -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:525-554, eq:costHS:
    C_hat(G) = 1 - (1/S) sum_s |<phi_s| W(G) |psi_s>|^2,   phi_s = U_ref psi_s,
over S Haar-random product states psi_s.  Each summand is the
state-mode overlap T_s = <phi_s|W|psi_s> of PAPER.md:325-331 (the paper's MPS
setting), so per sample the oracle runs O3 in state mode (oracle/mpo.py with
site dimension 2: product-state bottom start, label MPS top start, the same
truncation rule X7 with the state-site bound) and Alg. 2 / App. E
postprocessing; the risk and its derivatives are sample means (eq:costHS is a
mean of the L_HS^(s); the Riemannian maps of App. E are linear in (grad f,
H_f), so projecting the means equals averaging the projections).

Readings: R1 -- the risk is reported as C_hat = 1 + mean_s f_s with the
per-sample f_s = -|T_s|^2 of X2 (its gradient and HVP are those of
mean_s f_s); R2 -- the truncation rule per sample is X7 with P = 2:
r = min(chi, 4 m, 2 b_l, 2 b_r).
"""
from __future__ import annotations

import numpy as np

from . import common as cm
from . import mpo as M


def empirical_risk(n, depth, chi, G, labels, psis, V=None, first_offset=0, dirs=None):
    """labels: S label MPS (lists of [b][2][b']); psis [S][n][2]; V [B][K][4][4].

    Returns dict: risk, T [S], grad_f (Euclidean, mean), grad_R, H_f [dirs],
    Hess_R [dirs] and the per-sample O3 objects."""
    G = np.asarray(G)
    S = len(labels)
    K = G.shape[0]
    dirs = [] if V is None else (range(V.shape[0]) if dirs is None else dirs)
    Ts, fs = [], []
    grad_f = np.zeros((K, 4, 4), dtype=np.complex128)
    H_f = {b: np.zeros((K, 4, 4), dtype=np.complex128) for b in dirs}
    per = []
    for s in range(S):
        o = M.MPOOracle(n, depth, chi, G, labels[s], V, first_offset, psi=psis[s])
        E = o.gradient_T()
        f, gf, _ = cm.postprocess_gradient(o.T, E)
        Ts.append(o.T)
        fs.append(f)
        grad_f += gf / S
        for b in dirs:
            Hf, _ = cm.postprocess_hvp(o.T, E, o.hvp_T(b), V[b])
            H_f[b] += Hf / S
        per.append(o)
    out = {"risk": 1.0 + float(np.mean(fs)), "T": np.array(Ts), "grad_f": grad_f,
           "grad_R": cm.riemannian_gradient(G, grad_f), "H_f": H_f, "oracles": per}
    out["HR"] = {b: cm.riemannian_hvp(G, grad_f, H_f[b], V[b]) for b in dirs}
    return out
