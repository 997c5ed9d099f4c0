"""N2: translation-invariant brickwall circuits (App. "Modified HVP kernel for
translationally invariant brickwall circuits").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every gate of layer ell is the same layer gate g_ell, and
directions are layer-wise constant, V_k = v_ell for k in I_ell.
Reading X20: the quantities are those of the per-gate kernel composed with
the tying map (chain rule), as the equations before Alg. 3 state:
  dT/dg_ell = sum_{k in I_ell} dT/dG_k
  Omega = sum_ell Tr[v_ell^T dT/dg_ell]
  H_T[v]_ell = sum_{k in I_ell} D_V(dT/dG_k)
with D_V taken along the broadcast direction.  Alg. 3's listing (:1071-1104)
sums the same per-gate terms; its gradient line carries a stray minus sign and
shifted state indices (garbled), so it is not followed literally.  f, the
Euclidean gradient / HVP (Alg. 2, eq:grad-costHS, eq:hvp-costHS) and the
Riemannian projections (App. E) then act on U(4)^L exactly as on U(4)^K.
A layer with no gate (n = 2, even layer) has dT/dg_ell = 0.
"""
from __future__ import annotations

import numpy as np

from . import common as cm


def layer_of_gates(n: int, depth: int, first_offset: int = 0) -> np.ndarray:
    """ell - 1 for every gate k (layer-major gate order, X5)."""
    out = []
    for li, ly in enumerate(cm.layers(n, depth, first_offset)):
        out += [li] * len(ly)
    return np.array(out, dtype=np.int64)


def expand(x: np.ndarray, layer_of: np.ndarray) -> np.ndarray:
    """[..., L, 4, 4] layer quantities -> [..., K, 4, 4] per gate (G_k = g_ell)."""
    return np.take(x, layer_of, axis=-3)


def reduce(x: np.ndarray, layer_of: np.ndarray, L: int) -> np.ndarray:
    """sum_{k in I_ell} x_k: [..., K, 4, 4] -> [..., L, 4, 4]."""
    out = np.zeros(x.shape[:-3] + (L, 4, 4), dtype=x.dtype)
    for k, li in enumerate(layer_of):
        out[..., li, :, :] += x[..., k, :, :]
    return out


def gradient(T: complex, E: np.ndarray, g: np.ndarray, layer_of: np.ndarray):
    """From the per-gate (T, E_k) at G = expand(g): (f, grad_f_ell, grad_R_ell, E_ell)."""
    E_l = reduce(E, layer_of, g.shape[0])
    f, grad_f, _ = cm.postprocess_gradient(T, E_l)
    return f, grad_f, cm.riemannian_gradient(g, grad_f), E_l


def hvp(T: complex, E: np.ndarray, H_T: np.ndarray, g: np.ndarray, v: np.ndarray, layer_of: np.ndarray):
    """From the per-gate H_T[expand(v)]_k: (Hess_R[v]_ell, H_f[v]_ell, Omega)."""
    L = g.shape[0]
    E_l = reduce(E, layer_of, L)
    H_l = reduce(H_T, layer_of, L)
    _, grad_f, _ = cm.postprocess_gradient(T, E_l)
    Hf, om = cm.postprocess_hvp(T, E_l, H_l, v)
    return cm.riemannian_hvp(g, grad_f, Hf, v), Hf, om
