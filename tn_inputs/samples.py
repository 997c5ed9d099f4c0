"""Training samples of the sampled-state empirical risk.

Input generation only: no arithmetic of the method.
(eq:costHS): S Haar-random product states psi_s (each qubit an independent
Haar-random state) and their labels phi_s = U_ref psi_s
(PAPER.md:326), here as MPS:

  * haar_product_states: site vectors psi_s[j] = z / ||z||, z complex Gaussian
    from the SplitMix64 stream (cid, "samples", s * n + j) (X14 conventions);
  * label_mps: contract the reference MPO (U_ref / 2^{n/2}, site layout
    [b][2 out + in][b']) with psi on its in legs and restore the 2^{n/2}
    (sqrt 2 per site), then bring the MPS to right-canonical form with its
    centre at site 0 by exact QR sweeps (left-to-right QR, right-to-left LQ;
    no truncation) -- the form and structural bonds b_{s+1} <= 2 b_s the
    engine's state mode expects of a top start.
"""
from __future__ import annotations

import numpy as np

from . import rng


def haar_product_states(cid: int, S: int, n: int) -> np.ndarray:
    """[S][n][2] complex128, each site a normalised Haar-random qubit state."""
    out = np.empty((S, n, 2), dtype=np.complex128)
    for s in range(S):
        for j in range(n):
            z = rng.complex_normal(rng.stream_key(cid, "samples", s * n + j), 2)
            out[s, j] = z / np.linalg.norm(z)
    return out


def label_mps(ref_sites, psi: np.ndarray):
    """phi = U_ref |psi> as a right-canonical MPS (list of [b][2][b'])."""
    n = len(ref_sites)
    sites = []
    for j in range(n):
        u = np.asarray(ref_sites[j], dtype=np.complex128)
        b, _, bp = u.shape
        u = u.reshape(b, 2, 2, bp)                     # [b][out][in][b']
        sites.append(np.sqrt(2.0) * np.einsum("aoib,i->aob", u, psi[j]))
    for j in range(n - 1):                             # left-to-right QR (exact)
        b, _, bp = sites[j].shape
        q, r = np.linalg.qr(sites[j].reshape(b * 2, bp))
        sites[j] = q.reshape(b, 2, q.shape[1])
        sites[j + 1] = np.einsum("ab,bpc->apc", r, sites[j + 1])
    for j in range(n - 1, 0, -1):                      # right-to-left LQ (exact)
        b, _, bp = sites[j].shape
        qh, rh = np.linalg.qr(sites[j].reshape(b, 2 * bp).conj().T)
        sites[j] = qh.conj().T.reshape(qh.shape[1], 2, bp)
        sites[j - 1] = np.einsum("apb,bc->apc", sites[j - 1], rh.conj().T)
    return sites


def mps_bonds(sites):
    return [1] + [int(a.shape[2]) for a in sites]
