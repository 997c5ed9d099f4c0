"""O1 (exact dense Algorithm 1) and O2 (dense truncated definition).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Operator <-> state mapping (reading X1): a circuit W = G_K...G_1
acts on operators X by X -> G_k X (gate on the OUT legs of its qubit pair); the
inner product is <<X|Y>> = Tr(X^dag Y).  With psi^(0) = I/2^{n/2} and
phi^(0) = U_ref/2^{n/2} the paper's overlap T = phi^dag A_K...A_1 psi
 is T = Tr(U_ref^dag W)/2^n.  Qubit order big-endian, site 0
most significant; a gate's 4x4 index is 2 q_i + q_{i+1} (X6).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as _sla


def _svd(a):
    """Thin SVD (LAPACK gesdd); if divide-and-conquer does not converge (seen
    on blocks with many singular values at the noise floor), the QR-iteration
    driver gesvd computes the same decomposition."""
    try:
        return np.linalg.svd(a, full_matrices=False)
    except np.linalg.LinAlgError:
        return _sla.svd(a, full_matrices=False, lapack_driver="gesvd")

from .common import apply_pair_gate, bottom_order_lr, layers, top_order_lr

# ====================================================================== O1 ==


def apply_op(X: np.ndarray, n: int, s: int, G: np.ndarray) -> np.ndarray:
    """(G on qubits s, s+1) @ X for a 2^n x m matrix X (m = 2^n: an operator;
    m = 1: a state vector, the N1 setting)."""
    d, m = 2 ** n, X.shape[1]
    t = X.reshape(2 ** s, 4, 2 ** (n - s - 2), m)
    return np.einsum("ab,xbyz->xayz", G, t).reshape(d, m)


def env_op(phi: np.ndarray, psi: np.ndarray, n: int, s: int) -> np.ndarray:
    """sum_alpha conj(phi)_{a alpha} psi_{b alpha}: the gate environment.

    eq:environment: a, b run over the OUT indices of the
    pair (s, s+1); alpha over all other out indices and every in index.
    Reading X4: row = gate output index a, column = gate input index b, so that
    T = sum_ab G_ab E_ab (Euler identity).
    """
    m = psi.shape[1]
    f = phi.reshape(2 ** s, 4, 2 ** (n - s - 2), m)
    p = psi.reshape(2 ** s, 4, 2 ** (n - s - 2), m)
    return np.einsum("xayz,xbyz->ab", np.conj(f), p)


def overlap(phi: np.ndarray, psi: np.ndarray) -> complex:
    return complex(np.vdot(phi.ravel(), psi.ravel()))


def alg1(n, sites, G, Uref, V=None, psi0=None, phi0=None):
    """Algorithm 1 HVP_Kernel, forward pass first.

    Forward pass (lines 278-281) caches psi^(k) and Dpsi^(k) (eq:fis, eq:dfis);
    backward pass (lines 286-291) accumulates grad_k T = conj(phi^(K-k)) (x)
    psi^(k-1) (eq:general-doverlap) and [H_T]_k = conj(Dphi^(K-k)) (x) psi^(k-1)
    + conj(phi^(K-k)) (x) Dpsi^(k-1) (eq:overlap-hvp), then updates phi, Dphi.
    Reading X3: the accumulation at step k uses the PRE-update Dphi and phi
    (line 289 is written with Dphi^(K-k)); line 287's update is applied after.
    T = <phi^(K)|psi^(0)> at the boundary (line 292).
    Returns (T, E[K,4,4], H[K,4,4] or None).
    State mode (N1): psi0 = |psi> and phi0 = U_ref |psi> as
    2^n x 1 columns (then Uref is unused), T = <phi| W |psi>.
    """
    K = len(sites)
    d = 2 ** n
    if psi0 is None:
        psi0, phi0 = np.eye(d, dtype=np.complex128) / 2 ** (n / 2), Uref / 2 ** (n / 2)
    psi = [np.asarray(psi0, dtype=np.complex128)]
    dpsi = [np.zeros_like(psi[0])]
    for k in range(K):                                   # forward pass
        if V is not None:
            dpsi.append(apply_op(dpsi[k], n, sites[k], G[k]) + apply_op(psi[k], n, sites[k], V[k]))
        psi.append(apply_op(psi[k], n, sites[k], G[k]))
    phi = np.asarray(phi0, dtype=np.complex128)
    dphi = np.zeros_like(phi)
    E = np.zeros((K, 4, 4), dtype=np.complex128)
    H = np.zeros((K, 4, 4), dtype=np.complex128) if V is not None else None
    for k in reversed(range(K)):                         # backward pass
        E[k] = env_op(phi, psi[k], n, sites[k])
        if V is not None:
            H[k] = env_op(dphi, psi[k], n, sites[k]) + env_op(phi, dpsi[k], n, sites[k])
            dphi = apply_op(dphi, n, sites[k], G[k].conj().T) + apply_op(phi, n, sites[k], V[k].conj().T)
        phi = apply_op(phi, n, sites[k], G[k].conj().T)
    T = overlap(phi, psi[0])
    return T, E, H


def alg1_backward_first(n, sites, G, Uref, V):
    """The mirrored pass order (App. C): cache the backward
    states phi, Dphi first, then sweep forward computing psi, Dpsi on the fly.
    FoR == RoR means it must return the same (T, E, H) as alg1."""
    K = len(sites)
    d = 2 ** n
    phis = [Uref / 2 ** (n / 2)]
    dphis = [np.zeros((d, d), dtype=np.complex128)]
    for j in range(1, K + 1):                              # phi^(j), j = 1..K
        k = K - j
        dphis.append(apply_op(dphis[j - 1], n, sites[k], G[k].conj().T)
                     + apply_op(phis[j - 1], n, sites[k], V[k].conj().T))
        phis.append(apply_op(phis[j - 1], n, sites[k], G[k].conj().T))
    psi = np.eye(d, dtype=np.complex128) / 2 ** (n / 2)
    dpsi = np.zeros_like(psi)
    E = np.zeros((K, 4, 4), dtype=np.complex128)
    H = np.zeros((K, 4, 4), dtype=np.complex128)
    for k in range(K):
        j = K - k - 1                                       # phi^(K-k) index
        E[k] = env_op(phis[j], psi, n, sites[k])
        H[k] = env_op(dphis[j], psi, n, sites[k]) + env_op(phis[j], dpsi, n, sites[k])
        dpsi = apply_op(dpsi, n, sites[k], G[k]) + apply_op(psi, n, sites[k], V[k])
        psi = apply_op(psi, n, sites[k], G[k])
    T = overlap(phis[K], np.eye(d) / 2 ** (n / 2))
    return T, E, H


def substitution_hvp(n, sites, G, Uref, V):
    """[H_T[V]]_k = sum_{k' != k} E_k[G_{k'} -> V_{k'}].

    Brute force: one gradient evaluation per substituted gate.
    """
    K = len(sites)
    H = np.zeros((K, 4, 4), dtype=np.complex128)
    for kp in range(K):
        Gs = G.copy()
        Gs[kp] = V[kp]
        _, Es, _ = alg1(n, sites, Gs, Uref)
        for k in range(K):
            if k != kp:
                H[k] += Es[k]
    return H


def dense_circuit(n, sites, G) -> np.ndarray:
    W = np.eye(2 ** n, dtype=np.complex128)
    for k, s in enumerate(sites):
        W = apply_op(W, n, s, G[k])
    return W


def cost_T(n, sites, G, Uref) -> complex:
    """T = Tr(U_ref^dag W)/2^n directly from the dense circuit."""
    return complex(np.trace(Uref.conj().T @ dense_circuit(n, sites, G)) / 2 ** n)


# ====================================================================== O2 ==
# Operators as 4^n vectors, site index p = 2*out + in (layout of the MPO).


def op_to_vec(X: np.ndarray, n: int) -> np.ndarray:
    t = X.reshape((2,) * (2 * n))                       # o0..o_{n-1}, i0..i_{n-1}
    perm = []
    for s in range(n):
        perm += [s, n + s]
    return t.transpose(perm).reshape((4,) * n)


def vec_apply(x: np.ndarray, n: int, s: int, M: np.ndarray) -> np.ndarray:
    """Gate on the out legs of sites (s, s+1) of a p^n vector: p = 4 operator
    (p = 2 out + in), p = 2 state (N1)."""
    p = x.shape[0]
    t = x.reshape(p ** s, p, p, p ** (n - s - 2))
    return apply_pair_gate(t, M).reshape((p,) * n)


def vec_env(top: np.ndarray, bot: np.ndarray, n: int, s: int) -> np.ndarray:
    """E[(o1 o2), (o1' o2')] = sum conj(top[.., o1 i1, o2 i2, ..]) bot[.., o1' i1, o2' i2, ..]
    (state vectors: no in legs)."""
    p = top.shape[0]
    if p == 2:
        t = top.reshape(2 ** s, 4, 2 ** (n - s - 2))
        b = bot.reshape(2 ** s, 4, 2 ** (n - s - 2))
        return np.einsum("xay,xby->ab", np.conj(t), b)
    t = top.reshape(4 ** s, 2, 2, 2, 2, 4 ** (n - s - 2))
    b = bot.reshape(4 ** s, 2, 2, 2, 2, 4 ** (n - s - 2))
    return np.einsum("xaibjy,xcidjy->abcd", np.conj(t), b).reshape(4, 4)


def tangent_project(D: np.ndarray, Ur: np.ndarray, Vr: np.ndarray) -> np.ndarray:
    """P_T D = (P^L (x) I + I (x) P^R - P^L (x) P^R) D for the matricised state D
    (rows: sites left of the cut), P^L = Ur Ur^dag, P^R = Vr^dag Vr: the orthogonal
    projection onto the tangent space of the bond-r manifold at the kept
    Schmidt spaces (PAPER.md:1019-1023 fixed projectors; reading X8)."""
    PLD = Ur @ (Ur.conj().T @ D)
    return PLD + (D @ Vr.conj().T) @ Vr - (PLD @ Vr.conj().T) @ Vr


class DenseTruncated:
    """O2: the truncated definition of SURVEY.md §8(c.2), written out densely.

    Per gate k at cut c (between sites s and s+1), on the state X after
    applying M = G_k (bottom) or G_k^dag (top):
      * Schmidt decomposition X = sum sigma_a l_a (x) r_a (sigma descending);
      * keep r = min(chi, 4 m_c, 4 b_{c-1}, 4 b_{c+1}) (structural rule, X7);
      * P^L = sum_{a<r} l_a l_a^dag, P^R = sum_{a<r} r_a r_a^dag;
      * Y = s (P^L (x) I) X with frozen s = ||X|| / ||(P^L (x) I) X||;
      * tangent DY = s (P^L(x)I + I(x)P^R - P^L(x)P^R)(M DX_prev + V_M X_prev)
        -- PAPER.md:1019-1023 "SVD performed exclusively on the unperturbed
        2-site tensor ... isometries act as fixed projectors applied linearly to
        the tangent block" (reading X8).
    Gates of a layer are processed in the sweep order of X7; E_k and H_T are
    taken layer-wise with the layer's own gates exact (X9); T = <<T_0|B_0>>.
    """

    def __init__(self, n, depth, chi, G, Uref_vec, ref_bonds, V=None, first_offset=0, psi=None):
        """Operator mode: Uref_vec = U_ref/2^{n/2} as a 4^n vector.  State mode
        (N1): psi [n][2] the product state and Uref_vec the label phi = U_ref psi
        as a 2^n vector (bottom start psi, T = <phi|W|psi>)."""
        self.n, self.D, self.chi = n, depth, chi
        self.G = np.asarray(G)
        self.V = None if V is None else np.asarray(V)
        self.layers = layers(n, depth, first_offset)
        self.diag = []
        nb = 0 if V is None else self.V.shape[0]
        # bottom sweep: B_0 = I/2^{n/2} (operator) or the product state psi (state)
        if psi is None:
            x = op_to_vec(np.eye(2 ** n, dtype=np.complex128) / 2 ** (n / 2), n)
        else:
            x = np.asarray(psi[0], dtype=np.complex128)
            for s in range(1, n):
                x = np.kron(x, psi[s])
            x = x.reshape((2,) * n)
        self.p = x.shape[0]
        dx = [np.zeros_like(x) for _ in range(nb)]
        bonds = [1] * (n + 1)
        self.B, self.DB = [], []
        for ell in range(1, depth + 1):
            self.B.append(x.copy())
            self.DB.append([v.copy() for v in dx])
            order = self.layers[ell - 1] if bottom_order_lr(ell) else self.layers[ell - 1][::-1]
            for k, s in order:
                vm = [self.V[b, k] for b in range(nb)]
                x, dx = self._step(x, dx, s, self.G[k], vm, bonds)
        # top sweep: T_D = U_ref/2^{n/2}
        x = np.asarray(Uref_vec).copy()
        dx = [np.zeros_like(x) for _ in range(nb)]
        bonds = list(ref_bonds)
        self.Ttop = [None] * (depth + 1)
        self.DT = [None] * (depth + 1)
        for ell in range(depth, 0, -1):
            self.Ttop[ell] = x.copy()
            self.DT[ell] = [v.copy() for v in dx]
            ly = self.layers[ell - 1]
            order = ly if top_order_lr(ell, depth) else ly[::-1]
            for k, s in order:
                vm = [self.V[b, k].conj().T for b in range(nb)]
                x, dx = self._step(x, dx, s, self.G[k].conj().T, vm, bonds)
        self.Ttop[0] = x
        self.T = complex(np.vdot(self.Ttop[0].ravel(), self.B[0].ravel()))

    def _step(self, x, dx, s, M, VM, bonds):
        n, c, p = self.n, s + 1, self.p
        xp = vec_apply(x, n, s, M)
        dxp = [vec_apply(d, n, s, M) + vec_apply(x, n, s, vm) for d, vm in zip(dx, VM)]
        mat = xp.reshape(p ** c, -1)
        U, S, Vh = _svd(mat)
        # X7: r = min(chi, 4 m_c, p b_{c-1}, p b_{c+1}) (gate operator-Schmidt rank <= 4)
        r = min(self.chi, 4 * bonds[c], p * bonds[c - 1], p * bonds[c + 1], len(S))
        Ur, Vr = U[:, :r], Vh[:r]
        y = Ur @ (Ur.conj().T @ mat)
        sc = np.linalg.norm(mat) / np.linalg.norm(y)
        out = [(sc * tangent_project(d.reshape(mat.shape), Ur, Vr)).reshape(x.shape) for d in dxp]
        bonds[c] = r
        self.diag.append({"cut": c, "r": r, "sigma": S, "s": sc})
        return (sc * y).reshape(x.shape), out

    # -------------------------------------------------- layer-wise E and H_T
    def _layer_env(self, ell, top, bot, subst=None):
        """E_k for all gates k of layer ell for <<top| L_ell |bot>>.

        subst = (k', M) replaces gate k' by M (used for the in-layer V terms).
        """
        n = self.n
        ly = self.layers[ell - 1]
        gates = {k: self.G[k] for k, _ in ly}
        if subst is not None:
            gates[subst[0]] = subst[1]
        E = {}
        for k, s in ly:
            z = bot
            for kk, ss in ly:
                if kk != k:
                    z = vec_apply(z, n, ss, gates[kk])
            E[k] = vec_env(top, z, n, s)
        return E

    def gradient_T(self):
        K = self.G.shape[0]
        E = np.zeros((K, 4, 4), dtype=np.complex128)
        for ell in range(1, self.D + 1):
            for k, v in self._layer_env(ell, self.Ttop[ell], self.B[ell - 1]).items():
                E[k] = v
        return E

    def hvp_T(self, b):
        """H_T[V_b]: future (DT) + past (DB) + in-layer (k' != k) channels."""
        K = self.G.shape[0]
        H = np.zeros((K, 4, 4), dtype=np.complex128)
        for ell in range(1, self.D + 1):
            T_, B_ = self.Ttop[ell], self.B[ell - 1]
            for k, v in self._layer_env(ell, self.DT[ell][b], B_).items():
                H[k] += v
            for k, v in self._layer_env(ell, T_, self.DB[ell - 1][b]).items():
                H[k] += v
            for kp, _ in self.layers[ell - 1]:
                for k, v in self._layer_env(ell, T_, B_, subst=(kp, self.V[b, kp])).items():
                    if k != kp:
                        H[k] += v
        return H

    def layer_T(self, ell):
        """Per-layer overlap T^(ell) = <<T_ell|L_ell B_{ell-1}>> (diagnostic)."""
        z = self.B[ell - 1]
        for k, s in self.layers[ell - 1]:
            z = vec_apply(z, self.n, s, self.G[k])
        return complex(np.vdot(self.Ttop[ell].ravel(), z.ravel()))
