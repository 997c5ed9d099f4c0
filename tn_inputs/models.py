"""Spin-chain Hamiltonians and Trotter circuits used to synthesise U_ref.

Input generation only.  Conventions:
  * two-qubit index = 2*q_i + q_{i+1}, site i the left (most significant) qubit;
  * bond term h_{i,i+1} carries the coupling plus the single-site fields of its
    two sites with weight 1/2, full weight at the chain ends;
  * H_A = sum over pairs (0,1),(2,3),... ; H_B = sum over (1,2),(3,4),... ;
  * 1st order: U(d) = e^{-i d H_B} e^{-i d H_A} (H_A applied first);
  * 2nd order (Strang): e^{-i d H_A/2} e^{-i d H_B} e^{-i d H_A/2}, adjacent
    half layers merged -> 2*steps+1 layers.
Models follow the BASELINE.json configs' letters (X12):
  TFIM:  H = -J sum ZZ - h sum X - g sum Z     (PAPER.md:585 has other letters)
  XXX:   H =  J sum (XX + YY + ZZ)
  XXZ:   H =  sum (XX + YY + Delta ZZ) + hz sum Z
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

I2 = np.eye(2, dtype=np.complex128)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
PAULI = (I2, X, Y, Z)


@dataclass(frozen=True)
class Model:
    kind: str                     # "tfim" | "xxx" | "xxz"
    params: dict = field(default_factory=dict)

    def couplings(self):
        """(two-site coupling 4x4, single-site field 2x2)."""
        p = self.params
        if self.kind == "tfim":
            J, h, g = p.get("J", 1.0), p.get("h", 0.0), p.get("g", 0.0)
            return -J * np.kron(Z, Z), -h * X - g * Z
        if self.kind == "xxx":
            J = p.get("J", 1.0)
            return J * (np.kron(X, X) + np.kron(Y, Y) + np.kron(Z, Z)), 0.0 * I2
        if self.kind == "xxz":
            d, hz = p.get("Delta", 1.0), p.get("hz", 0.0)
            return np.kron(X, X) + np.kron(Y, Y) + d * np.kron(Z, Z), hz * Z
        raise ValueError(self.kind)


def bond_term(model: Model, n: int, i: int) -> np.ndarray:
    """h_{i,i+1}: coupling + split single-site fields (full weight at ends)."""
    c, f = model.couplings()
    wl = 1.0 if i == 0 else 0.5
    wr = 1.0 if i + 1 == n - 1 else 0.5
    return c + wl * np.kron(f, I2) + wr * np.kron(I2, f)


def expm_herm(h: np.ndarray, dt: float) -> np.ndarray:
    """exp(-i dt h) for Hermitian h, via its eigendecomposition."""
    w, v = np.linalg.eigh(h)
    return (v * np.exp(-1j * dt * w)[None, :]) @ v.conj().T


def dense_hamiltonian(model: Model, n: int) -> np.ndarray:
    """Full 2^n x 2^n H = sum of bond terms (for n <= 10 checks)."""
    dim = 2 ** n
    H = np.zeros((dim, dim), dtype=np.complex128)
    for i in range(n - 1):
        hb = bond_term(model, n, i)
        H += np.kron(np.kron(np.eye(2 ** i), hb), np.eye(2 ** (n - i - 2)))
    return H


def layer_pairs(n: int, offset: int):
    return [(s, s + 1) for s in range(offset, n - 1, 2)]


def trotter_layers(model: Model, n: int, t: float, steps: int, order: int):
    """List of layers; each layer a list of (left site, 4x4 gate), applied in order."""
    d = t / steps

    def layer(offset, dt):
        return [(i, expm_herm(bond_term(model, n, i), dt)) for i, _ in layer_pairs(n, offset)]

    layers = []
    if order == 1:
        for _ in range(steps):
            layers.append(layer(0, d))
            layers.append(layer(1, d))
    elif order == 2:
        layers.append(layer(0, d / 2))
        for s in range(steps):
            layers.append(layer(1, d))
            layers.append(layer(0, d if s + 1 < steps else d / 2))
    elif order == 4:
        # Suzuki's fourth-order fractal (PAPER.md:589, :601 use a 4th-order
        # reference): S4(d) = S2(p d)^2 S2((1 - 4p) d) S2(p d)^2, p = 1/(4 - 4^{1/3}),
        # S2(x) = e^{-i x H_A/2} e^{-i x H_B} e^{-i x H_A/2}; adjacent H_A half
        # steps are merged into one layer (as for order 2)
        p = 1.0 / (4.0 - 4.0 ** (1.0 / 3.0))
        seq = []                                   # (offset, dt) factors, applied in order
        for _ in range(steps):
            for x in (p, p, 1 - 4 * p, p, p):
                seq += [(0, x * d / 2), (1, x * d), (0, x * d / 2)]
        merged = []
        for off, dt in seq:
            if merged and merged[-1][0] == off:
                merged[-1] = (off, merged[-1][1] + dt)
            else:
                merged.append((off, dt))
        layers = [layer(off, dt) for off, dt in merged]
    else:
        raise ValueError("order must be 1, 2 or 4")
    return [ly for ly in layers if ly]
