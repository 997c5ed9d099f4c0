"""O3: the truncated definition realised with MPO sweeps.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

MPO site tensors are numpy arrays [b_left][p][b_right], p = 2*out + in.

Tangent representation (App. D; reading X8): the tangent of
an MPO state is kept in "channel" form
    DX = sum_j Ab_0 ... Ab_{j-1} B_j Aa_{j+1} ... Aa_{n-1},
i.e. the augmented MPO [[Ab, B], [0, Aa]] of bond <= 2 chi.
The before-chain Ab and after-chain Aa are direction independent; only the
blocks B_j depend on the direction.  The paper's "optimal" truncation -- SVD on
the unperturbed two-site tensor only, its isometries applied as fixed
projectors to the tangent block -- becomes, per gate with
G Theta ~= U S W^dag kept to r:
    DTheta = M (B_i Aa_{i+1} + Ab_i B_{i+1}) + V_M Theta
    LR sweep: B_i <- s (1 - U U^dag) DTheta W,  B_{i+1} <- s U^dag DTheta
    RL sweep: B_i <- s DTheta W,                B_{i+1} <- s U^dag DTheta (1 - W W^dag)
    Aa_i <- s M(Aa_i Aa_{i+1}) W, Aa_{i+1} <- W^dag
    Ab_{i+1} <- s U^dag M(Ab_i Ab_{i+1}), Ab_i <- U
which is DY = s (P^L(x)I + I(x)P^R - P^L(x)P^R)(M DX + V_M X) of O2 with the
projectors frozen from the primal SVD.  Centre moves (QR right / LQ left)
re-gauge the blocks so the gauge conditions hold at every step; no inverse of
S or of a QR factor is ever formed.
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


def _c(a):
    return np.conj(a)


# ---------------------------------------------------------------- sweeps --
class MPOSweep:
    """Primal MPO + channel-form tangents for a batch of directions."""

    def __init__(self, sites, chi, nb):
        self.n = len(sites)
        self.p = int(np.asarray(sites[0]).shape[1])   # 4: operator sites, 2: state sites (N1)
        self.chi = chi
        self.P = [np.array(a, dtype=np.complex128) for a in sites]
        self.c = 0
        self.Ab = [a.copy() for a in self.P]
        self.Aa = [a.copy() for a in self.P]
        self.Bd = [[np.zeros_like(a) for a in self.P] for _ in range(nb)]
        self.diag = []
        self.remainder = 0.0

    # -- centre moves -------------------------------------------------------
    def move_right(self):
        c = self.c
        P = self.P
        b, _, bp = P[c].shape
        Q, R = np.linalg.qr(P[c].reshape(b * self.p, bp))
        k = Q.shape[1]
        P[c] = Q.reshape(b, self.p, k)
        P[c + 1] = np.einsum("ab,bpc->apc", R, P[c + 1])
        # before-chain reduction Ab_c = Q X (remainder zero in exact arithmetic)
        Abc = self.Ab[c].reshape(b * self.p, -1)
        X = Q.conj().T @ Abc
        self.remainder = max(self.remainder, float(np.linalg.norm(Abc - Q @ X)))
        self.Ab[c] = Q.reshape(b, self.p, k)
        self.Ab[c + 1] = np.einsum("ab,bpc->apc", X, self.Ab[c + 1])
        for Bd in self.Bd:
            Bc = Bd[c].reshape(b * self.p, -1)
            Y = Q.conj().T @ Bc
            Bd[c] = (Bc - Q @ Y).reshape(b, self.p, -1)
            Bd[c + 1] = (np.einsum("ab,bpc->apc", X, Bd[c + 1])
                         + np.einsum("ab,bpc->apc", Y, self.Aa[c + 1]))
        self.c = c + 1

    def move_left(self):
        c = self.c
        P = self.P
        b, _, bp = P[c].shape
        Qh, Rh = np.linalg.qr(P[c].reshape(b, self.p * bp).conj().T)
        Q, L = Qh.conj().T, Rh.conj().T          # P_c = L Q, Q row-orthonormal
        k = Q.shape[0]
        P[c] = Q.reshape(k, self.p, bp)
        P[c - 1] = np.einsum("apb,bc->apc", P[c - 1], L)
        Aac = self.Aa[c].reshape(-1, self.p * bp)
        X = Aac @ Q.conj().T
        self.remainder = max(self.remainder, float(np.linalg.norm(Aac - X @ Q)))
        self.Aa[c] = Q.reshape(k, self.p, bp)
        self.Aa[c - 1] = np.einsum("apb,bc->apc", self.Aa[c - 1], X)
        for Bd in self.Bd:
            Bc = Bd[c].reshape(-1, self.p * bp)
            Y = Bc @ Q.conj().T
            Bd[c] = (Bc - Y @ Q).reshape(-1, self.p, bp)
            Bd[c - 1] = (np.einsum("apb,bc->apc", Bd[c - 1], X)
                         + np.einsum("apb,bc->apc", self.Ab[c - 1], Y))
        self.c = c - 1

    def move_to(self, target):
        while self.c < target:
            self.move_right()
        while self.c > target:
            self.move_left()

    # -- one gate -----------------------------------------------------------
    def pair_step(self, i, M, VM, lr):
        P = self.P
        self.move_to(i if lr else i + 1)
        bl, m, br = P[i].shape[0], P[i].shape[2], P[i + 1].shape[2]
        theta = np.einsum("apb,bqc->apqc", P[i], P[i + 1])
        p = self.p
        thp = apply_pair_gate(theta, M).reshape(bl * p, p * br)
        U, S, Vh = _svd(thp)
        r = min(self.chi, 4 * m, p * bl, p * br, len(S))   # gate operator-Schmidt rank <= 4
        Ur, Sr, Vr = U[:, :r], S[:r], Vh[:r]
        W = Vr.conj().T
        s = float(np.linalg.norm(S) / np.linalg.norm(Sr))
        self.diag.append({"site": i, "r": r, "sigma": S, "s": s,
                          "gap": float((S[r - 1] - S[r]) / S[0]) if r < len(S) else 1.0})
        # per-direction blocks (use the chains as they stand before this gate)
        for Bd, vm in zip(self.Bd, VM):
            d1 = np.einsum("apb,bqc->apqc", Bd[i], self.Aa[i + 1])
            d2 = np.einsum("apb,bqc->apqc", self.Ab[i], Bd[i + 1])
            dth = (apply_pair_gate(d1 + d2, M) + apply_pair_gate(theta, vm)).reshape(bl * p, p * br)
            if lr:
                UD = Ur.conj().T @ dth
                Bd[i] = (s * ((dth - Ur @ UD) @ W)).reshape(bl, p, r)
                Bd[i + 1] = (s * UD).reshape(r, p, br)
            else:
                DW = dth @ W
                Bd[i] = (s * DW).reshape(bl, p, r)
                Bd[i + 1] = (s * (Ur.conj().T @ (dth - DW @ W.conj().T))).reshape(r, p, br)
        # direction-independent chain pass-throughs
        ba_i = self.Aa[i].shape[0]
        aa = apply_pair_gate(np.einsum("apb,bqc->apqc", self.Aa[i], self.Aa[i + 1]), M)
        self.Aa[i] = (s * (aa.reshape(ba_i * p, p * br) @ W)).reshape(ba_i, p, r)
        self.Aa[i + 1] = Vr.reshape(r, p, br)
        bb_n = self.Ab[i + 1].shape[2]
        ab = apply_pair_gate(np.einsum("apb,bqc->apqc", self.Ab[i], self.Ab[i + 1]), M)
        self.Ab[i + 1] = (s * (Ur.conj().T @ ab.reshape(bl * p, p * bb_n))).reshape(r, p, bb_n)
        self.Ab[i] = Ur.reshape(bl, p, r)
        # primal
        if lr:
            P[i] = Ur.reshape(bl, p, r)
            P[i + 1] = (s * (Sr[:, None] * Vr)).reshape(r, p, br)
            self.c = i + 1
        else:
            P[i] = (s * (Ur * Sr[None, :])).reshape(bl, p, r)
            P[i + 1] = Vr.reshape(r, p, br)
            self.c = i

    def snapshot(self):
        return ([a.copy() for a in self.P], [a.copy() for a in self.Ab],
                [a.copy() for a in self.Aa], [[a.copy() for a in Bd] for Bd in self.Bd])


def augmented(Ab, Aa, B):
    """Sites of the augmented MPO [[Ab, B], [0, Aa]] with boundary vectors
    selecting the before-chain at site 0 and the after-chain at site n-1 --
    exactly sum_j Ab..B_j..Aa."""
    n = len(Ab)
    out = []
    for s in range(n):
        bb, _, bbn = Ab[s].shape
        ba, _, ban = Aa[s].shape
        M = np.zeros((bb + ba, Ab[s].shape[1], bbn + ban), dtype=np.complex128)
        M[:bb, :, :bbn] = Ab[s]
        M[:bb, :, bbn:] = B[s]
        M[bb:, :, bbn:] = Aa[s]
        if s == 0:
            M = M[:bb]
        if s == n - 1:
            M = M[:, :, bbn:]
        out.append(M)
    return out


# --------------------------------------------------- layer environments --
def _blocks(n, layer_gates):
    left = {s: (k, G) for k, s, G in layer_gates}
    out, s = [], 0
    while s < n:
        if s in left:
            out.append((s, left[s][0], left[s][1]))
            s += 2
        else:
            out.append((s, None, None))
            s += 1
    return out


def _upd_left(L, top, bot, blk, G):
    s, k, _ = blk
    if k is None:
        return np.einsum("tb,tpu,bpv->uv", L, _c(top[s]), bot[s], optimize=True)
    tt = np.einsum("apb,bqc->apqc", top[s], top[s + 1])
    bb = apply_pair_gate(np.einsum("apb,bqc->apqc", bot[s], bot[s + 1]), G)
    return np.einsum("tb,tpqu,bpqv->uv", L, _c(tt), bb, optimize=True)


def _upd_right(R, top, bot, blk, G):
    s, k, _ = blk
    if k is None:
        return np.einsum("uv,tpu,bpv->tb", R, _c(top[s]), bot[s], optimize=True)
    tt = np.einsum("apb,bqc->apqc", top[s], top[s + 1])
    bb = apply_pair_gate(np.einsum("apb,bqc->apqc", bot[s], bot[s + 1]), G)
    return np.einsum("uv,tpqu,bpqv->tb", R, _c(tt), bb, optimize=True)


def _extract(L, R, top, bot, blk):
    """E[(o1 o2),(o1' o2')] with the gate slot of block blk opened (eq:environment)."""
    s = blk[0]
    tt = np.einsum("apb,bqc->apqc", top[s], top[s + 1])
    bb = np.einsum("apb,bqc->apqc", bot[s], bot[s + 1])
    if tt.shape[1] == 2:        # state sites: p = out
        return np.einsum("XY,XabU,YcdV,UV->abcd", L, _c(tt), bb, R, optimize=True).reshape(4, 4)
    t6 = tt.reshape(tt.shape[0], 2, 2, 2, 2, tt.shape[3])
    b6 = bb.reshape(bb.shape[0], 2, 2, 2, 2, bb.shape[3])
    return np.einsum("XY,XaibjU,YcidjV,UV->abcd", L, _c(t6), b6, R, optimize=True).reshape(4, 4)


def layer_gradient(top, bot, layer_gates):
    """{k: d/dG_k <<top| L(G) |bot>>} for the gates of one layer (exact in-layer)."""
    n = len(top)
    blks = _blocks(n, layer_gates)
    Ls = [np.ones((1, 1), dtype=np.complex128)]
    for blk in blks:
        Ls.append(_upd_left(Ls[-1], top, bot, blk, blk[2]))
    Rs = [np.ones((1, 1), dtype=np.complex128)]
    for blk in reversed(blks):
        Rs.append(_upd_right(Rs[-1], top, bot, blk, blk[2]))
    Rs = Rs[::-1]
    return {blk[1]: _extract(Ls[j], Rs[j + 1], top, bot, blk)
            for j, blk in enumerate(blks) if blk[1] is not None}, Ls[-1][0, 0]


def layer_gradient_dual(top, bot, layer_gates, Vdir):
    """{k: sum_{k' != k} E_k[G_{k'} -> V_{k'}]} (in-layer channel of H_T).

    First-order (dual-number) environments: L1' = L1 o G + L0 o V.
    """
    n = len(top)
    blks = _blocks(n, layer_gates)
    L0 = [np.ones((1, 1), dtype=np.complex128)]
    L1 = [np.zeros((1, 1), dtype=np.complex128)]
    for blk in blks:
        L0.append(_upd_left(L0[-1], top, bot, blk, blk[2]))
        nxt = _upd_left(L1[-1], top, bot, blk, blk[2])
        if blk[1] is not None:
            nxt = nxt + _upd_left(L0[-2], top, bot, blk, Vdir[blk[1]])
        L1.append(nxt)
    R0 = [np.ones((1, 1), dtype=np.complex128)]
    R1 = [np.zeros((1, 1), dtype=np.complex128)]
    for blk in reversed(blks):
        R0.append(_upd_right(R0[-1], top, bot, blk, blk[2]))
        nxt = _upd_right(R1[-1], top, bot, blk, blk[2])
        if blk[1] is not None:
            nxt = nxt + _upd_right(R0[-2], top, bot, blk, Vdir[blk[1]])
        R1.append(nxt)
    R0, R1 = R0[::-1], R1[::-1]
    return {blk[1]: _extract(L1[j], R0[j + 1], top, bot, blk) + _extract(L0[j], R1[j + 1], top, bot, blk)
            for j, blk in enumerate(blks) if blk[1] is not None}


def overlap(top, bot):
    L = np.ones((1, 1), dtype=np.complex128)
    for a, b in zip(top, bot):
        L = np.einsum("tb,tpu,bpv->uv", L, _c(a), b, optimize=True)
    return complex(L[0, 0])


# ------------------------------------------------------------- driver --
class MPOOracle:
    """Bottom sweep (a2, a6), top sweep (a3, a7), layer environments (a4, a8).

    Algorithm 1's two passes at layer granularity: the
    forward pass caches B_ell and DB_ell; the backward pass produces T_ell and
    DT_ell and, per layer, E_k (eq:environment) and H_T[V]_k (eq:overlap-hvp:
    future variations via DT, past via DB, plus the in-layer k' != k gates).
    """

    def __init__(self, n, depth, chi, G, ref_sites, V=None, first_offset=0, psi=None):
        """Operator mode: ref_sites the MPO of U_ref / 2^{n/2} ([b][4][b']), bottom
        start I/2^{n/2}.  State mode (N1): ref_sites the label
        MPS phi = U_ref psi ([b][2][b']) and psi [n][2] the product state, so
        T = <phi| W |psi>."""
        self.n, self.D, self.chi = n, depth, chi
        self.G = np.asarray(G)
        self.V = None if V is None else np.asarray(V)
        nb = 0 if V is None else self.V.shape[0]
        self.layers = layers(n, depth, first_offset)
        if np.asarray(ref_sites[0]).shape[1] == 2:
            psi = np.asarray(psi, dtype=np.complex128)
            start = [psi[s].reshape(1, 2, 1) for s in range(n)]
        else:
            ident = np.zeros((1, 4, 1), dtype=np.complex128)
            ident[0, 0, 0] = ident[0, 3, 0] = 1.0 / np.sqrt(2.0)
            start = [ident] * n
        bot = MPOSweep(start, chi, nb)
        self.Bs = []
        for ell in range(1, depth + 1):
            self.Bs.append(bot.snapshot())
            ly = self.layers[ell - 1]
            lr = bottom_order_lr(ell)
            for k, s in (ly if lr else ly[::-1]):
                bot.pair_step(s, self.G[k], [self.V[b, k] for b in range(nb)], lr)
        top = MPOSweep([np.asarray(a) for a in ref_sites], chi, nb)
        self.Ts = [None] * (depth + 1)
        for ell in range(depth, 0, -1):
            self.Ts[ell] = top.snapshot()
            ly = self.layers[ell - 1]
            lr = top_order_lr(ell, depth)
            for k, s in (ly if lr else ly[::-1]):
                top.pair_step(s, self.G[k].conj().T, [self.V[b, k].conj().T for b in range(nb)], lr)
        self.Ts[0] = top.snapshot()
        self.T = overlap(self.Ts[0][0], self.Bs[0][0])
        self.diag = {"bottom": bot.diag, "top": top.diag,
                     "remainder": max(bot.remainder, top.remainder)}

    def _lg(self, ell):
        return [(k, s, self.G[k]) for k, s in self.layers[ell - 1]]

    def gradient_T(self):
        K = self.G.shape[0]
        E = np.zeros((K, 4, 4), dtype=np.complex128)
        self.layer_T = []
        for ell in range(1, self.D + 1):
            Ed, tl = layer_gradient(self.Ts[ell][0], self.Bs[ell - 1][0], self._lg(ell))
            self.layer_T.append(tl)
            for k, v in Ed.items():
                E[k] = v
        return E

    def hvp_T(self, b):
        K = self.G.shape[0]
        H = np.zeros((K, 4, 4), dtype=np.complex128)
        for ell in range(1, self.D + 1):
            Tp, TAb, TAa, TB = self.Ts[ell]
            Bp, BAb, BAa, BB = self.Bs[ell - 1]
            lg = self._lg(ell)
            dT = augmented(TAb, TAa, TB[b])
            dB = augmented(BAb, BAa, BB[b])
            for src in (layer_gradient(dT, Bp, lg)[0], layer_gradient(Tp, dB, lg)[0],
                        layer_gradient_dual(Tp, Bp, lg, {k: self.V[b, k] for k, _, _ in lg})):
                for k, v in src.items():
                    H[k] += v
        return H
