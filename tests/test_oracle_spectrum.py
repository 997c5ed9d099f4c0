"""Pins for oracle/spectrum.py (N3) against mathematics
the paper fixes: orthonormal spanning basis, the exact Hessian's symmetry,
phase null vectors, second derivatives along geodesics, CG on an SPD system."""
import numpy as np
from scipy.linalg import expm

from oracle import common as cm
from oracle import spectrum as S
from tests.test_oracle_exact import dense_riemannian_hessian, f_of, problem


def test_basis_is_an_orthonormal_basis_of_the_tangent_space():
    _, _, G, _, V = problem(n=3, D=2)
    B = S.pauli_basis(G)
    gram = np.array([[cm.inner(a, b) for b in B] for a in B])
    assert np.abs(gram - np.eye(len(B))).max() < 1e-14
    for b in B:                                          # each B_i is tangent: P_G(B) = B
        assert np.abs(cm.project(G, b) - b).max() < 1e-15
    c = S.coordinates(B, V[0])                           # V tangent -> V = sum c_i B_i
    assert np.abs(np.einsum("i,ikab->kab", c, B) - V[0]).max() < 1e-14


def test_phase_directions_are_exact_null_vectors():
    """f is invariant under G_k -> e^{i theta} G_k and i*I is central, so
    H_R[i G_k / 2] = 0 at ANY point (App. E formula; derivation in DESIGN.md
    X19), column and row 16k of the exact matrix vanish."""
    n, sites, G, U, _ = problem(n=4, D=3)
    M = dense_riemannian_hessian(n, sites, G, U)
    scale = np.abs(M).max()
    ph = np.arange(0, M.shape[0], 16)
    assert np.abs(M[:, ph]).max() < 1e-13 * scale
    assert np.abs(M[ph, :]).max() < 1e-13 * scale
    w, asym = S.spectrum(M)
    assert asym < 1e-13
    assert np.sum(np.abs(w) < 1e-12 * scale) >= len(ph)


def test_entries_are_second_derivatives_along_geodesics():
    """<u, H_R v> = (q(u+v) - q(u) - q(v))/2 with q(w) = d^2/dt^2 f(Exp_G(t w)),
    Exp_G(t w)_k = G_k expm(t G_k^dag w_k) (bi-invariant metric)."""
    n, sites, G, U, _ = problem(n=3, D=3)
    M = dense_riemannian_hessian(n, sites, G, U)
    B = S.pauli_basis(G)
    f0 = f_of(n, sites, G, U)

    def q(w, h=1e-4):
        def f_t(t):
            return f_of(n, sites, np.stack([G[k] @ expm(t * G[k].conj().T @ w[k]) for k in range(len(G))]), U)
        return (f_t(h) - 2 * f0 + f_t(-h)) / h ** 2

    rng = np.random.default_rng(5)
    for i, j in [(1, 1), (3, 20), (17, 40)] + [tuple(rng.integers(0, len(B), 2)) for _ in range(3)]:
        est = 0.5 * (q(B[i] + B[j]) - q(B[i]) - q(B[j]))
        assert abs(est - M[i, j]) < 2e-6 * max(1.0, np.abs(M).max())


def test_cg_probe_solves_an_spd_system():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((12, 12))
    A = A @ A.T + 0.5 * np.eye(12)
    b = rng.standard_normal(12)
    xs = np.linalg.solve(A, b)
    x, res = S.cg_probe(lambda v: A @ v, lambda a, c: float(a @ c), b, 12)   # n steps: exact up to rounding
    assert len(res) == 13 and res[-1] < 1e-6 * res[0]
    assert np.linalg.norm(x - xs) < 1e-6 * np.linalg.norm(xs)
    x, res = S.cg_probe(lambda v: A @ v, lambda a, c: float(a @ c), b, 24)
    assert np.linalg.norm(x - xs) < 1e-12 * np.linalg.norm(xs)
