"""Reference MPO U_ref / 2^{n/2} built from a Trotter circuit (input generation).

SURVEY.md §8(c.4) X11: the paper gives no construction for "a reference MPO
truncated to chi"; this harness runs a plain TEBD of the Trotter layers on the
identity operator I/2^{n/2} (site tensor delta_{oi}/sqrt(2), bond 1), gates on
the OUT legs, mixed-canonical sweeps with QR centre moves, keep
min(chi, #{sigma > 1e-14 sigma_max}) singular values per two-site split (a cap
that would cut a cluster of equal values drops the whole cluster) and
rescale the kept values to the pre-truncation norm.  The result is returned
right-canonical with the orthogonality centre at site 0 and unit Frobenius
norm (a1: "U_ref/2^{n/2}, right-canonical, centre at site 0").

It is input DATA to both the oracle and the CUDA path; it uses torch linear
algebra on whatever device it is given (CPU in the CPU test-suite, the GPU on
the box so large configs are generated in seconds).  The MPO site layout is
[b_left][p][b_right] with p = 2*out + in.
"""
from __future__ import annotations

import math

import numpy as np
import torch


def _apply_out_gate(theta: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    bl, _, _, br = theta.shape
    t = theta.reshape(bl, 2, 2, 2, 2, br)          # [bl][o1][i1][o2][i2][br]
    gg = g.reshape(2, 2, 2, 2)                      # [o1][o2][o1'][o2']
    t = torch.einsum("abcd,xcidjy->xaibjy", gg, t)
    return t.reshape(bl, 4, 4, br)


def identity_mpo(n: int, device="cpu"):
    a = torch.zeros(1, 4, 1, dtype=torch.complex128, device=device)
    a[0, 0, 0] = a[0, 3, 0] = 1.0 / math.sqrt(2.0)
    return [a.clone() for _ in range(n)]


def _move_right(sites, c):
    b, _, bp = sites[c].shape
    q, r = torch.linalg.qr(sites[c].reshape(b * 4, bp))
    sites[c] = q.reshape(b, 4, q.shape[1])
    sites[c + 1] = torch.einsum("ab,bpc->apc", r, sites[c + 1])


def _move_left(sites, c):
    b, _, bp = sites[c].shape
    q, r = torch.linalg.qr(sites[c].reshape(b, 4 * bp).mH)
    sites[c] = q.mH.reshape(q.shape[1], 4, bp)
    sites[c - 1] = torch.einsum("apb,bc->apc", sites[c - 1], r.mH)


CLUSTER_GAP = 1e-8


def _keep_whole_multiplets(s, keep: int) -> int:
    """A bond cut that falls inside a cluster of (numerically) equal singular
    values -- the Schmidt multiplets of a symmetric model (XXZ: U(1)) -- keeps an
    arbitrary part of the multiplet: WHICH operator comes out then depends on
    the SVD routine's rounding, i.e. on the machine.  When the cap chi cuts such
    a cluster (relative gap s[keep-1] - s[keep] <= CLUSTER_GAP s[keep-1]) the
    whole cluster is dropped instead, so the generated reference is the same
    operator on every machine (stored oracle outputs depend on it)."""
    while 1 < keep < s.numel() and float(s[keep - 1] - s[keep]) <= CLUSTER_GAP * float(s[keep - 1]):
        keep -= 1
    return keep


def tebd_out_legs(sites, layers, chi: int, tol: float = 1e-14):
    """Apply layers [(i, G), ...] to an MPO (centre at 0), truncating to chi."""
    dev = sites[0].device
    c = 0
    for layer in layers:
        for i, g in layer:
            while c < i:
                _move_right(sites, c); c += 1
            while c > i:
                _move_left(sites, c); c -= 1
            gt = torch.as_tensor(np.asarray(g), dtype=torch.complex128, device=dev)
            bl, br = sites[i].shape[0], sites[i + 1].shape[2]
            th = torch.einsum("apb,bqc->apqc", sites[i], sites[i + 1])
            th = _apply_out_gate(th, gt).reshape(bl * 4, 4 * br)
            nrm = torch.linalg.vector_norm(th)
            if th.is_cuda:
                # GPU input generation: split through the Gram matrix (eigh is
                # ~15x faster than the GPU SVD at 1024^2); values below ~1e-7
                # of the largest are resolved only roughly, which only changes
                # WHICH reference MPO is generated, not its use downstream.
                w, v = torch.linalg.eigh(th @ th.mH)
                w, v = w.flip(0).clamp_min(0.0), v.flip(1)
                above = int((w > (max(tol, 1e-7) ** 2) * w[0]).sum().item())
                keep = max(1, min(chi, above))
                if keep < above:
                    keep = _keep_whole_multiplets(w.sqrt().cpu(), keep)
                u = v[:, :keep]
                right = u.mH @ th
            else:
                u, s, vh = torch.linalg.svd(th, full_matrices=False)
                above = int((s > tol * s[0]).sum().item())
                keep = max(1, min(chi, above))
                if keep < above:                      # the cap cuts: never through a multiplet
                    keep = _keep_whole_multiplets(s, keep)
                u = u[:, :keep]
                right = s[:keep, None].to(vh.dtype) * vh[:keep]
            right = right * (nrm / torch.linalg.vector_norm(right))
            sites[i] = u.reshape(bl, 4, keep)
            sites[i + 1] = right.reshape(keep, 4, br)
            c = i + 1
    while c > 0:
        _move_left(sites, c); c -= 1
    nrm = torch.linalg.vector_norm(sites[0])
    sites[0] = sites[0] / nrm
    return [a.resolve_conj().contiguous() for a in sites]


def reference_mpo(layers, n: int, chi: int, device="cpu"):
    """U_ref/2^{n/2} as a right-canonical MPO (list of [b][4][b'] tensors)."""
    sites = identity_mpo(n, device)
    return tebd_out_legs(sites, layers, chi)


def mpo_bonds(sites):
    return [1] + [int(a.shape[2]) for a in sites]


def mpo_to_dense_operator(sites) -> np.ndarray:
    """Contract an MPO (n <= 10) into its 2^n x 2^n operator (times 1, no rescale)."""
    n = len(sites)

    def host(x):
        return x if isinstance(x, np.ndarray) else x.detach().resolve_conj().cpu().numpy()

    t = host(sites[0])                                           # [1][4][b]
    for s in range(1, n):
        a = host(sites[s])
        t = np.tensordot(t, a, axes=([t.ndim - 1], [0]))
    t = t.reshape((4,) * n)                         # drop boundary bonds
    t = t.reshape((2, 2) * n)                       # o0 i0 o1 i1 ...
    perm = list(range(0, 2 * n, 2)) + list(range(1, 2 * n, 2))
    return t.transpose(perm).reshape(2 ** n, 2 ** n)
