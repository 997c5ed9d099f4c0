"""Counter-based SplitMix64 streams and the seeded draws built on them.

Seeded synthetic inputs only.  This module holds none
of the method's arithmetic: it turns (base seed, config id, kind, index) into
reproducible uniforms / Gaussians / Haar U(4) matrices.  Both the oracle
(`oracle/`) and the CUDA path's tests consume what it produces.

Stream definition (X14): state_j = key + (j+1)*0x9E3779B97F4A7C15 (mod 2^64),
z_j = mix(state_j) with the SplitMix64 finaliser (multipliers 0xBF58476D1CE4E5B9,
0x94D049BB133111EB; shifts 30/27/31).  u = ((z >> 11) + 1) * 2^-53 in (0, 1].
Box-Muller uses consecutive uniform pairs (u1, u2): g = sqrt(-2 ln u1) *
(cos 2 pi u2, sin 2 pi u2), the two outputs taken as (re, im) in that order.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 20260419
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

KIND = {"gates": 1, "directions": 2, "init": 3, "samples": 4, "misc": 5}


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def stream_key(cfg_id: int, kind: str | int, index: int, base: int = BASE_SEED) -> np.uint64:
    k = KIND[kind] if isinstance(kind, str) else int(kind)
    a = _mix(np.array([base], dtype=np.uint64))
    b = _mix(np.array([(int(cfg_id) << 40) ^ (k << 32) ^ int(index)], dtype=np.uint64))
    with np.errstate(over="ignore"):
        return (a ^ (b * np.uint64(3)))[0]


def raw(key: np.uint64, count: int) -> np.ndarray:
    j = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = np.uint64(key) + j * _GOLDEN
    return _mix(st)


def uniform(key: np.uint64, count: int) -> np.ndarray:
    z = raw(key, count)
    return ((z >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)


def complex_normal(key: np.uint64, count: int) -> np.ndarray:
    """count complex numbers with re, im ~ N(0, 1) independently."""
    u = uniform(key, 2 * count).reshape(count, 2)
    rad = np.sqrt(-2.0 * np.log(u[:, 0]))
    ang = 2.0 * np.pi * u[:, 1]
    return rad * np.cos(ang) + 1j * rad * np.sin(ang)


def haar_u4(key: np.uint64) -> np.ndarray:
    """Haar-random U(4): QR of a Ginibre matrix with the R-diagonal phase fix."""
    z = complex_normal(key, 16).reshape(4, 4)
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    return q * (d / np.abs(d))[None, :]


def skew_gaussian(key: np.uint64) -> np.ndarray:
    """S = (A - A^dag)/2 with A complex Gaussian 4x4 (skew-Hermitian)."""
    a = complex_normal(key, 16).reshape(4, 4)
    return 0.5 * (a - a.conj().T)
