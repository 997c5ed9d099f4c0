"""Pins for the exact oracle O1 (dense Algorithm 1) and the postprocessing.

Everything here is checked against mathematics the paper fixes, not against
the oracle itself: closed forms, finite differences, the substitution sum,
pass-order equivalence, invariants of the projections.
"""
import numpy as np
import pytest
from scipy.linalg import expm

from oracle import common as cm
from oracle import dense as O
from oracle import spectrum as S
from tn_inputs import configs as C
from tn_inputs.reference import mpo_to_dense_operator, reference_mpo


def problem(n=4, D=4, cid=11, nb=2):
    cfg = C.small_case(cid, n, D, 4096, batch=nb)
    U = mpo_to_dense_operator(reference_mpo(C.reference_layers(cfg), n, 4096)) * 2 ** (n / 2)
    sites = C.brickwall_sites(n, D)
    G = C.haar_gates(cid, len(sites))
    V = C.tangent_directions(cid, G, nb)
    return n, sites, G, U, V


def f_of(n, sites, G, U):
    return -abs(O.cost_T(n, sites, G, U)) ** 2


def grad_f_of(n, sites, G, U):
    T, E, _ = O.alg1(n, sites, G, U)
    return cm.postprocess_gradient(T, E)[1]


# ---------------------------------------------------------- closed forms --
def test_closed_form_two_qubits_two_gates():
    """n=2, W = G2 G1, U_ref = I: T = Tr(G2 G1)/4, E1 = G2^T/4, E2 = G1^T/4,
    H_T[V]_1 = V2^T/4, H_T[V]_2 = V1^T/4 (SURVEY.md §8(c.5) closed form (i))."""
    G = C.haar_gates(21, 2)
    V = C.tangent_directions(21, G, 1)[0]
    T, E, H = O.alg1(2, [0, 0], G, np.eye(4), V)
    assert abs(T - np.trace(G[1] @ G[0]) / 4) < 1e-15
    assert np.abs(E[0] - G[1].T / 4).max() < 1e-15
    assert np.abs(E[1] - G[0].T / 4).max() < 1e-15
    assert np.abs(H[0] - V[1].T / 4).max() < 1e-15
    assert np.abs(H[1] - V[0].T / 4).max() < 1e-15


def test_closed_form_identity_circuit():
    """Identity circuit vs U_ref = I: T = 1, E_k = I/4 (closed form (ii))."""
    n, D = 5, 4
    sites = C.brickwall_sites(n, D)
    G = np.stack([np.eye(4, dtype=complex)] * len(sites))
    T, E, _ = O.alg1(n, sites, G, np.eye(2 ** n))
    assert abs(T - 1) < 1e-14
    assert np.abs(E - np.eye(4) / 4).max() < 1e-15


def test_zero_direction_and_single_gate():
    n, sites, G, U, V = problem()
    _, _, H = O.alg1(n, sites, G, U, np.zeros_like(V[0]))
    assert np.abs(H).max() == 0.0
    _, _, H1 = O.alg1(3, [0], G[:1], np.eye(8), V[0][:1])      # K = 1 -> H_T = 0
    assert np.abs(H1).max() == 0.0


def test_global_minimum_when_circuit_is_the_reference():
    """W = U_ref: f = -1, grad_R = 0, Riemannian Hessian PSD (closed form (iii))."""
    n, sites, G, _, V = problem(n=4, D=3)
    U = O.dense_circuit(n, sites, G)
    T, E, _ = O.alg1(n, sites, G, U)
    f, grad_f, _ = cm.postprocess_gradient(T, E)
    assert abs(f + 1) < 1e-13
    assert np.abs(cm.riemannian_gradient(G, grad_f)).max() < 1e-13
    Hd = dense_riemannian_hessian(n, sites, G, U)
    assert np.linalg.eigvalsh(0.5 * (Hd + Hd.T)).min() > -1e-12


# --------------------------------------------------------------- identities --
def test_euler_identity_and_depth_invariance():
    """T = sum_ab G_ab E_ab for every k (eq:overlap-2, X4) and
    T = phi^(K-k)^dag psi^(k) at every depth k (eq:overlap-general)."""
    n, sites, G, U, _ = problem()
    T, E, _ = O.alg1(n, sites, G, U)
    for k in range(len(sites)):
        assert abs(np.sum(G[k] * E[k]) - T) < 1e-14
    K = len(sites)
    for k in range(K + 1):
        psi = np.eye(2 ** n) / 2 ** (n / 2)
        for j in range(k):
            psi = O.apply_op(psi, n, sites[j], G[j])
        phi = U / 2 ** (n / 2)
        for j in reversed(range(k, K)):
            phi = O.apply_op(phi, n, sites[j], G[j].conj().T)
        assert abs(O.overlap(phi, psi) - T) < 1e-14


def test_T_matches_trace_definition():
    n, sites, G, U, _ = problem()
    T, _, _ = O.alg1(n, sites, G, U)
    assert abs(T - np.trace(U.conj().T @ O.dense_circuit(n, sites, G)) / 2 ** n) < 1e-15


def test_holomorphic_derivative_by_finite_differences():
    """dT/dRe G = E, dT/dIm G = i E, i.e. dT/dG* = 0."""
    n, sites, G, U, _ = problem()
    _, E, _ = O.alg1(n, sites, G, U)
    eps = 1e-6
    for k, (a, b) in [(0, (1, 2)), (3, (3, 0)), (5, (2, 2))]:
        for dz, fac in ((1.0, 1.0), (1j, 1j)):
            Gp, Gm = G.copy(), G.copy()
            Gp[k, a, b] += eps * dz
            Gm[k, a, b] -= eps * dz
            fd = (O.cost_T(n, sites, Gp, U) - O.cost_T(n, sites, Gm, U)) / (2 * eps)
            assert abs(fd - fac * E[k, a, b]) < 1e-9


def test_omega_is_directional_derivative_of_T():
    n, sites, G, U, V = problem()
    T, E, _ = O.alg1(n, sites, G, U)
    eps = 1e-6
    fd = (O.cost_T(n, sites, G + eps * V[0], U) - O.cost_T(n, sites, G - eps * V[0], U)) / (2 * eps)
    assert abs(fd - cm.omega(E, V[0])) < 1e-9


def test_gradient_by_finite_differences():
    """Df[Z] = Re sum Tr(grad f^dag Z) for arbitrary complex Z (eq:grad-real)."""
    n, sites, G, U, _ = problem()
    Z = np.random.default_rng(1).standard_normal(G.shape) + 1j * np.random.default_rng(2).standard_normal(G.shape)
    gf = grad_f_of(n, sites, G, U)
    eps = 1e-5
    fd = (f_of(n, sites, G + eps * Z, U) - f_of(n, sites, G - eps * Z, U)) / (2 * eps)
    assert abs(fd - cm.inner(gf, Z)) < 1e-9 * max(1, abs(fd))


def test_hvp_by_finite_differences_of_the_gradient():
    """H_f[V] = D(grad f)[V] (eq:FoR); signs of Alg. 2 under reading X2."""
    n, sites, G, U, V = problem()
    T, E, H = O.alg1(n, sites, G, U, V[0])
    Hf, _ = cm.postprocess_hvp(T, E, H, V[0])
    eps = 1e-5
    fd = (grad_f_of(n, sites, G + eps * V[0], U) - grad_f_of(n, sites, G - eps * V[0], U)) / (2 * eps)
    assert np.abs(fd - Hf).max() < 1e-8 * max(1.0, np.abs(Hf).max())


def test_pass_order_and_substitution():
    """FoR == RoR (App. C): forward-first and backward-first passes agree, and
    both equal the O(K^2) substitution sum of the paper's definition."""
    n, sites, G, U, V = problem()
    T1, E1, H1 = O.alg1(n, sites, G, U, V[1])
    T2, E2, H2 = O.alg1_backward_first(n, sites, G, U, V[1])
    Hs = O.substitution_hvp(n, sites, G, U, V[1])
    assert abs(T1 - T2) < 1e-15
    assert np.abs(E1 - E2).max() < 1e-15
    assert np.abs(H1 - H2).max() < 1e-14
    assert np.abs(H1 - Hs).max() < 1e-14


def test_alg1_reading_x3_matches_substitution():
    """Reading X3 (accumulate with the pre-update Dphi) gives
    exactly the substitution sum, which has no k' = k term."""
    n, sites, G, U, V = problem()
    _, _, H = O.alg1(n, sites, G, U, V[0])
    Hs = O.substitution_hvp(n, sites, G, U, V[0])
    assert np.abs(H - Hs).max() < 1e-14          # the reading X3 matches the definition


# ---------------------------------------------------------- Riemannian --
def test_projection_invariants():
    G = C.haar_gates(31, 6)
    rng_ = np.random.default_rng(3)
    Z = rng_.standard_normal(G.shape) + 1j * rng_.standard_normal(G.shape)
    W = rng_.standard_normal(G.shape) + 1j * rng_.standard_normal(G.shape)
    P = cm.project(G, Z)
    assert np.abs(cm.project(G, P) - P).max() < 1e-14                      # idempotent
    assert abs(cm.inner(P, W) - cm.inner(Z, cm.project(G, W))) < 1e-12     # orthogonal
    A = rng_.standard_normal(G.shape) + 1j * rng_.standard_normal(G.shape)
    S = 0.5 * (A - np.conj(np.swapaxes(A, -1, -2)))
    Hm = 0.5 * (A + np.conj(np.swapaxes(A, -1, -2)))
    assert np.abs(cm.project(G, G @ S) - G @ S).max() < 1e-14              # tangent kept
    assert np.abs(cm.project(G, G @ Hm)).max() < 1e-14                     # normal killed


def test_riemannian_hessian_self_adjoint():
    n, sites, G, U, V = problem(nb=2)
    T, E, _ = O.alg1(n, sites, G, U)
    _, grad_f, _ = cm.postprocess_gradient(T, E)
    out = []
    for b in range(2):
        _, _, H = O.alg1(n, sites, G, U, V[b])
        Hf, _ = cm.postprocess_hvp(T, E, H, V[b])
        out.append(cm.riemannian_hvp(G, grad_f, Hf, V[b]))
    a, b_ = cm.inner(V[0], out[1]), cm.inner(out[0], V[1])
    assert abs(a - b_) < 1e-13 * max(1, abs(a))


def test_geodesic_derivatives():
    """Along the geodesic gamma(t) = G exp(t G^dag V): d/dt f = <grad_R, V>,
    d^2/dt^2 f = <V, Hess_R[V]> (App. E)."""
    n, sites, G, U, V = problem()
    Vd = V[0]
    T, E, H = O.alg1(n, sites, G, U, Vd)
    f0, grad_f, _ = cm.postprocess_gradient(T, E)
    Hf, _ = cm.postprocess_hvp(T, E, H, Vd)
    HR = cm.riemannian_hvp(G, grad_f, Hf, Vd)
    gR = cm.riemannian_gradient(G, grad_f)

    def f_t(t):
        Gt = np.stack([G[k] @ expm(t * G[k].conj().T @ Vd[k]) for k in range(len(G))])
        return f_of(n, sites, Gt, U)

    h = 1e-4
    d1 = (f_t(h) - f_t(-h)) / (2 * h)
    d2 = (f_t(h) - 2 * f0 + f_t(-h)) / h ** 2
    assert abs(d1 - cm.inner(gR, Vd)) < 1e-8
    assert abs(d2 - cm.inner(Vd, HR)) < 1e-5 * max(1, abs(d2))


def pauli_basis(G):
    return list(S.pauli_basis(G))


def dense_riemannian_hessian(n, sites, G, U):
    """(H_R)_ij = <B_i, H_R[B_j]> from the exact O1 HVP (oracle.spectrum)."""
    T, E, _ = O.alg1(n, sites, G, U)
    _, grad_f, _ = cm.postprocess_gradient(T, E)

    def hvp(V):
        _, _, H = O.alg1(n, sites, G, U, V)
        Hf, _ = cm.postprocess_hvp(T, E, H, V)
        return cm.riemannian_hvp(G, grad_f, Hf, V)
    return S.hessian_matrix(S.pauli_basis(G), hvp)


def test_pauli_basis_orthonormal_and_dense_hessian_symmetric():
    n, sites, G, U, _ = problem(n=3, D=2)
    basis = pauli_basis(G)
    gram = np.array([[cm.inner(a, b) for b in basis] for a in basis])
    assert np.abs(gram - np.eye(len(basis))).max() < 1e-14
    Hd = dense_riemannian_hessian(n, sites, G, U)
    assert np.abs(Hd - Hd.T).max() < 1e-13
