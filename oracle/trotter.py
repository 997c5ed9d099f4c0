"""N4: reference construction -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reading X11: the reference U_ref / 2^{n/2} "truncated to chi" is the TEBD of the
Trotter circuit's gates applied to I/2^{n/2} on the OUT legs, each two-site
split keeping r = min(chi, #{sigma_j > tol sigma_1}) singular values rescaled to
the pre-truncation norm, gates in the circuit's order, centre moved by QR;
the result is right-canonical with its centre at site 0 and unit norm.

  * dense_product: the untruncated definition, the 2^n x 2^n product of the
    gate sequence (n <= 10) -- what TEBD reaches exactly when nothing is cut;
  * tebd: the truncated definition, written out with numpy SVD / QR.
"""
from __future__ import annotations

import numpy as np

from .common import apply_out_gate


def dense_product(n, gate_seq):
    """W = G_last ... G_first for gate_seq = [(left site, 4x4 gate), ...]."""
    W = np.eye(2 ** n, dtype=np.complex128)
    for i, g in gate_seq:
        W = np.kron(np.kron(np.eye(2 ** i), g), np.eye(2 ** (n - i - 2))) @ W
    return W


def tebd(n, gate_seq, chi, tol):
    """Sites [b][4][b'] (p = 2 out + in) of U / 2^{n/2}, right-canonical, centre 0."""
    a = []
    for _ in range(n):
        t = np.zeros((1, 4, 1), dtype=np.complex128)
        t[0, 0, 0] = t[0, 3, 0] = 1.0 / np.sqrt(2.0)
        a.append(t)
    c = 0

    def right():
        nonlocal c
        b, _, bp = a[c].shape
        q, r = np.linalg.qr(a[c].reshape(b * 4, bp))
        a[c] = q.reshape(b, 4, q.shape[1])
        a[c + 1] = np.einsum("ab,bpc->apc", r, a[c + 1])
        c += 1

    def left():
        nonlocal c
        b, _, bp = a[c].shape
        qh, rh = np.linalg.qr(a[c].reshape(b, 4 * bp).conj().T)
        a[c] = qh.conj().T.reshape(qh.shape[1], 4, bp)
        a[c - 1] = np.einsum("apb,bc->apc", a[c - 1], rh.conj().T)
        c -= 1

    for i, g in gate_seq:
        while c < i:
            right()
        while c > i:
            left()
        bl, br = a[i].shape[0], a[i + 1].shape[2]
        th = apply_out_gate(np.einsum("apb,bqc->apqc", a[i], a[i + 1]), g).reshape(bl * 4, 4 * br)
        u, s, vh = np.linalg.svd(th, full_matrices=False)
        r = max(1, min(chi, int(np.sum(s > tol * s[0]))))
        right_f = s[:r, None] * vh[:r]
        right_f *= np.linalg.norm(th) / np.linalg.norm(right_f)
        a[i] = u[:, :r].reshape(bl, 4, r)
        a[i + 1] = right_f.reshape(r, 4, br)
        c = i + 1
    while c > 0:
        left()
    a[0] = a[0] / np.linalg.norm(a[0])
    return a
