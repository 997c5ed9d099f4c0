"""N3: the dense Riemannian Hessian in the Pauli tangent basis, its spectrum
and a CG probe (App. "Spectral analysis").

(H_R)_ij = <B_i, H_R[B_j]> with the orthonormal basis
B_{16k+4a+b} = i G_k (P_a (x) P_b)/2 at gate k.  Every
step is a library call: tn_pauli_basis generates a window of basis vectors,
tn_hvp_apply takes them as a batch of directions, tn_pauli_coords turns the
HVPs into matrix rows, tn_sym_eig returns the spectrum of the symmetric part
(reading X19).  The CG probe (fig:cg) is plain
conjugate gradients on H_R x = -grad_R with matrix-free HVPs, the tangent
algebra in tn_tangent_dot / tn_tangent_axpby.  Only control flow runs here.
"""
from __future__ import annotations

import math

import torch

from .api import HVPEngine, axpby, pauli_basis, pauli_coords, sym_eig, tangent_dot


def hessian_matrix(eng: HVPEngine, gates: torch.Tensor, chunk: int | None = None) -> torch.Tensor:
    """H_R^T as a float64 [16K, 16K] device tensor (row j = coordinates of
    H_R[B_j]); eng must hold the primal pass for `gates` (tn_hvp_environments)."""
    K = gates.shape[0]
    n = 16 * K
    chunk = chunk or eng.max_batch
    Mt = torch.empty((n, n), dtype=torch.float64, device=gates.device)
    for j0 in range(0, n, chunk):
        c = min(chunk, n - j0)
        B = pauli_basis(gates, j0, c)
        H = eng.apply(B)
        pauli_coords(gates, H, out=Mt[j0:j0 + c])
    return Mt


def hessian_spectrum(eng: HVPEngine, gates: torch.Tensor, chunk: int | None = None):
    """(eigenvalues ascending [16K], relative asymmetry ||M - M^T|| / ||M||)."""
    Mt = hessian_matrix(eng, gates, chunk)
    w, asym = sym_eig(Mt)
    a = asym.cpu()
    return w, (float(a[0] / a[1]) if a[1] > 0 else 0.0)


def cg_probe(eng: HVPEngine, b: torch.Tensor, iters: int):
    """Conjugate gradients for H_R x = b from x = 0 (no truncation radius):
    returns x and the recurrence residual norms ||r_j||, j = 0..iters."""
    def dot(u, v):
        return float(tangent_dot(u[None], v[None]).item())

    x = torch.zeros_like(b)
    r = b.clone()
    p = r.clone()
    rr = dot(r, r)
    res = [math.sqrt(rr)]
    for _ in range(iters):
        Hp = eng.apply(p[None])[0]
        pHp = dot(p, Hp)
        if pHp == 0 or rr == 0:
            break
        alpha = rr / pHp
        axpby(alpha, p, 1.0, x)
        axpby(-alpha, Hp, 1.0, r)
        rr_new = dot(r, r)
        res.append(math.sqrt(rr_new))
        axpby(1.0, r, rr_new / rr, p)
        rr = rr_new
    return x, res
