"""ctypes front of the plain C++ complex128 oracle (oracle/cpp/tn_oracle.cpp).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  north_star subsystem (1):
a CPU oracle in plain C++ complex128 sharing no code with the GPU path --
Algorithm 1 on dense matrices (exact) and the truncated definition on dense
vectors with its own one-sided Jacobi SVD, plus Alg. 2 / App. E
postprocessing, all in std::complex<double> loops.  The numpy oracles (O1, O2,
O3) are a second, independent realisation that this one is checked against.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .common import layers


def _lib():
    from .cpp.build import build
    L = C.CDLL(build())
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
    L.tno_alg1.argtypes = [C.c_int, C.c_int, ip, dp, C.c_int, dp, dp, C.c_int, dp, dp, dp, dp]
    L.tno_dense_truncated.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, dp, ip, C.c_int, dp, dp,
                                      dp, dp]
    L.tno_postprocess.argtypes = [C.c_int, C.c_int, dp, dp, dp, dp, dp, dp, dp, dp]
    return L


_L = None


def lib():
    global _L
    if _L is None:
        _L = _lib()
    return _L


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def alg1(n, sites, G, psi0, phi0, V=None):
    """Exact Algorithm 1: psi0, phi0 [2^n][m] (operators: I/2^{n/2}, U/2^{n/2}; states: columns).
    -> (T, E [K,4,4], H_T [B,K,4,4] or None)."""
    K = len(sites)
    nb = 0 if V is None else V.shape[0]
    G, gp = _d(G)
    psi0, pp = _d(psi0)
    phi0, fp = _d(phi0)
    V, vp = _d(np.zeros((1, K, 4, 4)) if V is None else V)
    s = (C.c_int * K)(*sites)
    T = np.zeros(2)
    E = np.zeros((K, 4, 4), dtype=np.complex128)
    H = np.zeros((max(nb, 1), K, 4, 4), dtype=np.complex128)
    lib().tno_alg1(n, K, s, gp, psi0.shape[1], pp, fp, nb, vp, T.ctypes.data_as(C.POINTER(C.c_double)),
                   _d(E)[1], _d(H)[1])
    return complex(T[0], T[1]), E, (H[:nb] if nb else None)


def dense_truncated(n, depth, chi, G, x0, top0, ref_bonds, V=None, first_offset=0):
    """The truncated definition on p^n vectors (x0: bottom start, top0: top start,
    p = 4 operators or 2 states, inferred from the length) -> (T, E, H_T)."""
    x0 = np.ravel(x0)
    p = 4 if x0.size == 4 ** n else 2
    K = sum(len(ly) for ly in layers(n, depth, first_offset))
    nb = 0 if V is None else V.shape[0]
    G, gp = _d(G)
    x0, xp = _d(x0)
    top0, tp = _d(np.ravel(top0))
    V, vp = _d(np.zeros((1, K, 4, 4)) if V is None else V)
    rb = (C.c_int * (n + 1))(*[int(b) for b in ref_bonds])
    T = np.zeros(2)
    E = np.zeros((K, 4, 4), dtype=np.complex128)
    H = np.zeros((max(nb, 1), K, 4, 4), dtype=np.complex128)
    lib().tno_dense_truncated(n, depth, chi, first_offset, p, gp, xp, tp, rb, nb, vp,
                              T.ctypes.data_as(C.POINTER(C.c_double)), _d(E)[1], _d(H)[1])
    return complex(T[0], T[1]), E, (H[:nb] if nb else None)


def postprocess(G, T, E, HT, V):
    """-> (f, grad_R [K,4,4], Hess_R [B,K,4,4]) by Alg. 2 (X2) and App. E."""
    K = G.shape[0]
    nb = HT.shape[0]
    G, gp = _d(G)
    E, ep = _d(E)
    HT, hp = _d(HT)
    V, vp = _d(V)
    T2 = np.array([T.real, T.imag])
    f = np.zeros(1)
    gR = np.zeros((K, 4, 4), dtype=np.complex128)
    hR = np.zeros((nb, K, 4, 4), dtype=np.complex128)
    lib().tno_postprocess(K, nb, gp, T2.ctypes.data_as(C.POINTER(C.c_double)), ep, hp, vp,
                          f.ctypes.data_as(C.POINTER(C.c_double)), _d(gR)[1], _d(hR)[1])
    return float(f[0]), gR, hR
