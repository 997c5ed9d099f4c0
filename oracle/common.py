"""Layout, Alg. 2 postprocessing and Riemannian projections (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------- layout --
def layers(n: int, depth: int, first_offset: int = 0):
    """Brickwall layers: list (ell = 1..D) of lists of (k, left site).

    X5 reading: layer 1 acts on
    pairs (off, off+1), (off+2, off+3), ...; layers alternate the offset; the
    gate index k runs layer-major, left -> right.
    """
    out, k = [], 0
    for ell in range(1, depth + 1):
        off = (first_offset + ell - 1) % 2
        ly = []
        for s in range(off, n - 1, 2):
            ly.append((k, s))
            k += 1
        out.append(ly)
    return out


def bottom_order_lr(ell: int) -> bool:
    """Bottom sweep of layer ell runs left->right for odd ell (X7)."""
    return ell % 2 == 1


def top_order_lr(ell: int, depth: int) -> bool:
    """Top sweep processes layer D first, left->right, then alternates (X7)."""
    return (depth - ell) % 2 == 0


def apply_out_gate(x: np.ndarray, g: np.ndarray) -> np.ndarray:
    """(G (x) I_in) on a two-site block x[..., p1, p2, ...] with p = 2*o + i.

    x has shape (bl, 4, 4, br); returns the same shape.  G[(o1 o2), (o1' o2')]
    acts on the OUT legs only (SURVEY.md §0 mapping, X6).
    """
    bl, _, _, br = x.shape
    t = x.reshape(bl, 2, 2, 2, 2, br)
    gg = g.reshape(2, 2, 2, 2)
    return np.einsum("abcd,xcidjy->xaibjy", gg, t).reshape(bl, 4, 4, br)


def apply_pair_gate(x: np.ndarray, g: np.ndarray) -> np.ndarray:
    """The gate on the OUT legs of a two-site block x[bl, p, p, br]: operator
    sites p = 4 (p = 2 out + in, apply_out_gate) or state sites p = 2 (p = out;
    the N1 MPS setting of PAPER.md:325-336)."""
    if x.shape[1] == 4:
        return apply_out_gate(x, g)
    bl, _, _, br = x.shape
    return np.einsum("ab,xby->xay", g, x.reshape(bl, 4, br)).reshape(bl, 2, 2, br)


# ------------------------------------------------------ Alg. 2 postprocess --
def postprocess_gradient(T: complex, E: np.ndarray):
    """f and the Euclidean gradient from (T, grad T = E).

    PAPER.md:492-499 (Alg. 2): grad L_F = -conj(grad T).  The cost is the
    config's f = -|T|^2 = -Tr(U_ref^dag W)^2/4^n.  Reading X2: Alg. 2's gradient
    line (-2 T grad L_F) is the gradient of +|T|^2, so
    grad f = +2 T grad L_F = -2 T conj(E) (pinned by finite differences).
    """
    grad_LF = -np.conj(E)
    f = -abs(T) ** 2
    grad_f = 2.0 * T * grad_LF
    return f, grad_f, grad_LF


def omega(E: np.ndarray, V: np.ndarray) -> complex:
    """Omega = -sum_k <grad_k L_F, V_k> = sum_k sum_ab E_k[a,b] V_k[a,b].

    PAPER.md:426-439 (eq:Omega), App. B; <A,B> = Tr(A^dag B).
    """
    grad_LF = -np.conj(E)
    return -np.sum(np.conj(grad_LF) * V)


def postprocess_hvp(T: complex, E: np.ndarray, H_T: np.ndarray, V: np.ndarray):
    """H_f[V] = 2 [Omega grad L_F + T H_F[V]],  H_F = -conj(H_T).

    PAPER.md:501-505 (Alg. 2) and eq:hvp-costHS as printed; with
    f = -|T|^2 this is D(grad f)[V] (X2; pinned by finite differences).
    """
    grad_LF = -np.conj(E)
    om = omega(E, V)
    H_LF = -np.conj(H_T)
    return 2.0 * (om * grad_LF + T * H_LF), om


# ------------------------------------------------------ App. E projections --
def project(G: np.ndarray, Z: np.ndarray) -> np.ndarray:
    """P_G(Z) = 1/2 Z - 1/2 G Z^dag G, gate-wise."""
    return 0.5 * Z - 0.5 * G @ np.conj(np.swapaxes(Z, -1, -2)) @ G


def riemannian_gradient(G: np.ndarray, grad_f: np.ndarray) -> np.ndarray:
    """grad_R f = [P_{G_k}(grad_k f)]_k."""
    return project(G, grad_f)


def riemannian_hvp(G: np.ndarray, grad_f: np.ndarray, H_f: np.ndarray, V: np.ndarray) -> np.ndarray:
    """H_R[V]_k = P_G(H_f[V]_k - 1/2 V_k grad_k f^dag G_k - 1/2 G_k grad_k f^dag V_k).

    PAPER.md:1152-1157 (App. E, gate-wise).
    """
    gh = np.conj(np.swapaxes(grad_f, -1, -2))
    return project(G, H_f - 0.5 * V @ gh @ G - 0.5 * G @ gh @ V)


def inner(A: np.ndarray, B: np.ndarray) -> float:
    """Riemannian metric Re sum_k Tr(A_k^dag B_k) (X15)."""
    return float(np.real(np.sum(np.conj(A) * B)))


def full_outputs(G, T, E, H_T, V):
    """(f, grad_R, Hess_R[V] per direction, Omega per direction, H_f)."""
    f, grad_f, _ = postprocess_gradient(T, E)
    gR = riemannian_gradient(G, grad_f)
    HR, OM, HF = [], [], []
    for b in range(V.shape[0]):
        Hf, om = postprocess_hvp(T, E, H_T[b], V[b])
        HF.append(Hf)
        OM.append(om)
        HR.append(riemannian_hvp(G, grad_f, Hf, V[b]))
    return f, gR, np.array(HR), np.array(OM), np.array(HF), grad_f
