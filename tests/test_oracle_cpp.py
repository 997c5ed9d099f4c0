"""Pins for the plain C++ complex128 oracle (oracle/cpp/tn_oracle.cpp, north_star
subsystem (1)): closed forms, finite differences, the Euler identity and
self-adjointness of the Riemannian Hessian (mathematics), then agreement with
the independent numpy realisations O1 / O2 / O3 (operator and state mode,
untruncated and truncated)."""
import numpy as np
import pytest

from oracle import common as cm
from oracle import cpp_oracle as X
from oracle import dense as O
from oracle import mpo as M
from tn_inputs import configs as C
from tn_inputs import samples as SMP
from tn_inputs.reference import mpo_bonds, mpo_to_dense_operator, reference_mpo


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b))


def problem(n, D, cid, nb=2, offset=0, ref_chi=4096):
    cfg = C.small_case(cid, n, D, ref_chi, batch=nb, first_offset=offset)
    ref = reference_mpo(C.reference_layers(cfg), n, ref_chi)
    U = mpo_to_dense_operator(ref) * 2 ** (n / 2)
    sites = C.brickwall_sites(n, D, offset)
    G = C.haar_gates(cid, len(sites))
    V = C.tangent_directions(cid, G, nb)
    return ref, U, sites, G, V


def test_closed_form_two_qubits():
    """n=2, W = G2 G1, U_ref = I: T = Tr(G2 G1)/4, E1 = G2^T/4, E2 = G1^T/4,
    H_T[V]_1 = V2^T/4, H_T[V]_2 = V1^T/4 (SURVEY.md §8(c.5) closed form (i))."""
    G = C.haar_gates(601, 2)
    V = C.tangent_directions(601, G, 1)
    I4 = np.eye(4, dtype=np.complex128) / 2
    T, E, H = X.alg1(2, [0, 0], G, I4, I4, V)
    assert abs(T - np.trace(G[1] @ G[0]) / 4) < 1e-15
    assert np.abs(E[0] - G[1].T / 4).max() < 1e-15 and np.abs(E[1] - G[0].T / 4).max() < 1e-15
    assert np.abs(H[0, 0] - V[0, 1].T / 4).max() < 1e-15 and np.abs(H[0, 1] - V[0, 0].T / 4).max() < 1e-15


def test_euler_identity_fd_and_self_adjointness():
    n, D = 4, 4
    ref, U, sites, G, V = problem(n, D, 602)
    d = 2 ** n
    psi0, phi0 = np.eye(d) / 2 ** (n / 2), U / 2 ** (n / 2)
    T, E, H = X.alg1(n, sites, G, psi0, phi0, V)
    for k in range(len(sites)):                       # Euler: T = sum G_k o E_k for every k
        assert abs(np.sum(G[k] * E[k]) - T) < 1e-14
    assert abs(T - np.trace(U.conj().T @ O.dense_circuit(n, sites, G)) / d) < 1e-14
    eps = 1e-6                                        # Omega = D_V T (FD)
    Tp = X.alg1(n, sites, G + eps * V[0], psi0, phi0)[0]
    Tm = X.alg1(n, sites, G - eps * V[0], psi0, phi0)[0]
    assert abs((Tp - Tm) / (2 * eps) - np.sum(E * V[0])) < 1e-9
    f, gR, HR = X.postprocess(G, T, E, H, V)           # <w, Hess v> = <Hess w, v> (exact regime)
    assert abs(cm.inner(V[0], HR[1]) - cm.inner(HR[0], V[1])) < 1e-12 * max(1.0, np.abs(HR).max())
    # f by FD along a Euclidean direction: d f = Re <grad f, Z>
    Z = np.random.default_rng(3).standard_normal(G.shape) + 0j
    fp = -abs(X.alg1(n, sites, G + 1e-5 * Z, psi0, phi0)[0]) ** 2
    fm = -abs(X.alg1(n, sites, G - 1e-5 * Z, psi0, phi0)[0]) ** 2
    gf = -2 * T * np.conj(E)
    assert abs((fp - fm) / 2e-5 - cm.inner(gf, Z)) < 1e-9


@pytest.mark.parametrize("n,D,offset", [(4, 4, 0), (5, 3, 1)])
def test_cpp_equals_numpy_exact(n, D, offset):
    ref, U, sites, G, V = problem(n, D, 610 + n, offset=offset)
    d = 2 ** n
    T, E, H = X.alg1(n, sites, G, np.eye(d) / 2 ** (n / 2), U / 2 ** (n / 2), V)
    Tn, En, Hn = O.alg1(n, sites, G, U, V[0])
    assert abs(T - Tn) < 1e-14 and rel(E, En) < 1e-13 and rel(H[0], Hn) < 1e-13
    # the truncated routine with no cap reaches the exact result
    Tt, Et, Ht = X.dense_truncated(n, D, 10 ** 6, G, O.op_to_vec(np.eye(d) / 2 ** (n / 2), n),
                                   O.op_to_vec(U / 2 ** (n / 2), n), mpo_bonds(ref), V, offset)
    assert abs(Tt - Tn) < 1e-13 and rel(Et, En) < 1e-12 and rel(Ht[0], Hn) < 1e-12
    # postprocessing equals oracle/common
    f, gR, HR = X.postprocess(G, T, E, H, V)
    f2, gf2, _ = cm.postprocess_gradient(Tn, En)
    assert abs(f - f2) < 1e-15 and rel(gR, cm.riemannian_gradient(G, gf2)) < 1e-13
    Hf, _ = cm.postprocess_hvp(Tn, En, Hn, V[0])
    assert rel(HR[0], cm.riemannian_hvp(G, gf2, Hf, V[0])) < 1e-12


@pytest.mark.parametrize("n,D,chi,offset", [(6, 4, 4, 0), (7, 4, 8, 1)])
def test_cpp_truncated_equals_numpy_o2_and_o3(n, D, chi, offset):
    ref, U, sites, G, V = problem(n, D, 620 + n + chi, offset=offset)
    d = 2 ** n
    Uv = O.op_to_vec(U / 2 ** (n / 2), n)
    T, E, H = X.dense_truncated(n, D, chi, G, O.op_to_vec(np.eye(d) / 2 ** (n / 2), n), Uv, mpo_bonds(ref), V,
                                offset)
    o2 = O.DenseTruncated(n, D, chi, G, Uv, mpo_bonds(ref), V, offset)
    o3 = M.MPOOracle(n, D, chi, G, [a.numpy() for a in ref], V, offset)
    for o in (o2, o3):
        assert abs(T - o.T) < 1e-12 * max(1, abs(o.T))
        assert rel(E, o.gradient_T()) < 1e-11
        for b in range(2):
            assert rel(H[b], o.hvp_T(b)) < 1e-10


def test_cpp_state_mode():
    n, D, chi = 6, 4, 2
    ref, U, sites, G, V = problem(n, D, 631)
    psi = SMP.haar_product_states(631, 1, n)[0]
    lab = SMP.label_mps([a.numpy() for a in ref], psi)
    x = psi[0]
    for q in psi[1:]:
        x = np.kron(x, q)
    phi = U @ x
    # exact: state columns in Alg. 1 vs the truncated routine with no cap vs numpy O1
    T, E, H = X.alg1(n, sites, G, x[:, None], phi[:, None], V)
    Tn, En, Hn = O.alg1(n, sites, G, None, V[0], psi0=x[:, None], phi0=phi[:, None])
    assert abs(T - Tn) < 1e-14 and rel(E, En) < 1e-13 and rel(H[0], Hn) < 1e-13
    # truncated state mode vs numpy O3 state mode
    Tt, Et, Ht = X.dense_truncated(n, D, chi, G, x, phi, SMP.mps_bonds(lab), V)
    o3 = M.MPOOracle(n, D, chi, G, lab, V, psi=psi)
    assert abs(Tt - o3.T) < 1e-12 * max(1, abs(o3.T))
    assert rel(Et, o3.gradient_T()) < 1e-11 and rel(Ht[1], o3.hvp_T(1)) < 1e-10
