"""N3: the dense Riemannian Hessian in the Pauli tangent basis, its spectrum
and a CG probe (App. "Spectral analysis").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Basis: for gate k and Paulis P_a, P_b in {I, X, Y, Z},
  B_{16k + 4a + b} = (0, .., i G_k (P_a (x) P_b)/2, .., 0).  16K vectors,
  orthonormal under the metric Re sum_k Tr(A_k^dag B_k).
* Matrix: (H_R)_ij = <B_i, H_R[B_j]>; with an orthonormal
  basis the HVP of B_j gives column j directly.
* Spectrum: H_R is self-adjoint, so its eigenvalues are
  real.  Reading X19: under truncation the fixed-projector HVP is only
  approximately self-adjoint, so the spectrum reported is
  that of the symmetric part (M + M^T)/2 and the asymmetry ||M - M^T||/||M||
  is reported beside it.
* CG probe (fig:cg): plain conjugate gradients on
  H_R x = -grad_R with the full (matrix-free) Hessian, residual per iteration.
"""
from __future__ import annotations

import numpy as np

_P = (np.eye(2, dtype=np.complex128),
      np.array([[0, 1], [1, 0]], dtype=np.complex128),
      np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
      np.array([[1, 0], [0, -1]], dtype=np.complex128))


def pauli_pair(a: int, b: int) -> np.ndarray:
    """P_a (x) P_b in the gate's 4x4 index 2 q_i + q_{i+1} (X6)."""
    return np.kron(_P[a], _P[b])


def pauli_basis(G: np.ndarray) -> np.ndarray:
    """[16K][K][4][4]: B_{16k+4a+b} = i G_k (P_a (x) P_b) / 2 at gate k."""
    K = G.shape[0]
    out = np.zeros((16 * K, K, 4, 4), dtype=np.complex128)
    for k in range(K):
        for a in range(4):
            for b in range(4):
                out[16 * k + 4 * a + b, k] = 1j * G[k] @ pauli_pair(a, b) / 2
    return out


def coordinates(basis: np.ndarray, X: np.ndarray) -> np.ndarray:
    """<B_i, X> = Re sum Tr(B_i^dag X) for every basis vector."""
    return np.real(np.einsum("ikab,kab->i", np.conj(basis), X))


def hessian_matrix(basis: np.ndarray, hvp) -> np.ndarray:
    """(H_R)_ij = <B_i, H_R[B_j]>; hvp(V) -> H_R[V]."""
    cols = [coordinates(basis, hvp(Bj)) for Bj in basis]
    return np.array(cols).T


def spectrum(M: np.ndarray):
    """Eigenvalues (ascending) of the symmetric part and the relative asymmetry (X19)."""
    asym = float(np.linalg.norm(M - M.T) / np.linalg.norm(M)) if np.any(M) else 0.0
    return np.linalg.eigvalsh(0.5 * (M + M.T)), asym


def cg_probe(hvp, inner, b: np.ndarray, iters: int):
    """Conjugate gradients for H x = b from x = 0 (Hestenes-Stiefel), no
    truncation: returns x and the residual norms ||b - H x_j||, j = 0..iters
    (the recurrence residual, as plotted in fig:cg)."""
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = inner(r, r)
    res = [np.sqrt(rr)]
    for _ in range(iters):
        Hp = hvp(p)
        pHp = inner(p, Hp)
        if pHp == 0 or rr == 0:
            break
        alpha = rr / pHp
        x = x + alpha * p
        r = r - alpha * Hp
        rr_new = inner(r, r)
        res.append(np.sqrt(rr_new))
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, np.array(res)
