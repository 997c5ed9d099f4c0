"""Pins for oracle/ti.py (N2) against mathematics the paper
fixes: geodesic derivatives of the tied cost on U(4)^L, self-adjointness,
Euler homogeneity of degree |I_ell|, the one-gate-per-layer special case,
phase null vectors."""
import numpy as np
from scipy.linalg import expm

from oracle import common as cm
from oracle import dense as O
from oracle import spectrum as S
from oracle import ti
from tests.test_oracle_exact import f_of, problem
from tn_inputs import configs as C


def ti_problem(n=4, D=4, cid=11, nb=2):
    n, sites, _, U, _ = problem(n=n, D=D, cid=cid)
    g = C.haar_gates(cid + 1000, D)
    lay = ti.layer_of_gates(n, D)
    v = C.tangent_directions(cid + 1000, g, nb)
    return n, sites, g, lay, U, v


def ti_all(n, sites, g, lay, U, v):
    G = ti.expand(g, lay)
    T, E, _ = O.alg1(n, sites, G, U)
    f, grad_f, gR, E_l = ti.gradient(T, E, g, lay)
    HR = []
    for vb in v:
        _, _, H = O.alg1(n, sites, G, U, ti.expand(vb, lay))
        HR.append(ti.hvp(T, E, H, g, vb, lay)[0])
    return T, f, gR, E_l, np.array(HR)


def test_geodesic_derivatives_of_the_tied_cost():
    n, sites, g, lay, U, v = ti_problem()
    _, f0, gR, _, HR = ti_all(n, sites, g, lay, U, v)

    def f_t(t, w):
        gt = np.stack([g[l] @ expm(t * g[l].conj().T @ w[l]) for l in range(len(g))])
        return f_of(n, sites, ti.expand(gt, lay), U)
    h, h1 = 1e-4, 1e-5             # tied gates raise the degree: smaller step for d1 (O(h^2) error)
    for b in range(len(v)):
        d1 = (f_t(h1, v[b]) - f_t(-h1, v[b])) / (2 * h1)
        d2 = (f_t(h, v[b]) - 2 * f0 + f_t(-h, v[b])) / h ** 2
        assert abs(d1 - cm.inner(gR, v[b])) < 1e-8
        assert abs(d2 - cm.inner(v[b], HR[b])) < 1e-5 * max(1, abs(d2))


def test_self_adjoint_and_tangent():
    n, sites, g, lay, U, v = ti_problem(n=5, D=3)
    _, _, gR, _, HR = ti_all(n, sites, g, lay, U, v)
    a, b = cm.inner(v[0], HR[1]), cm.inner(HR[0], v[1])
    assert abs(a - b) < 1e-13 * max(1, abs(a))
    assert np.abs(cm.project(g, gR) - gR).max() < 1e-15
    assert np.abs(cm.project(g, HR) - HR).max() < 1e-15


def test_euler_homogeneity_degree_is_gates_per_layer():
    """T(e^{i t} g_ell) = e^{i t |I_ell|} T, so sum_ab (g_ell)_ab (dT/dg_ell)_ab = |I_ell| T."""
    n, sites, g, lay, U, v = ti_problem(n=5, D=4)
    T, _, _, E_l, _ = ti_all(n, sites, g, lay, U, v[:0])
    counts = np.bincount(lay, minlength=len(g))
    assert sorted(set(counts)) == [2]                    # n = 5: two gates in every layer
    for l in range(len(g)):
        assert abs(np.sum(g[l] * E_l[l]) - counts[l] * T) < 1e-14


def test_one_gate_per_layer_is_the_per_gate_kernel():
    n, sites, g, lay, U, v = ti_problem(n=3, D=4)
    assert list(lay) == [0, 1, 2, 3]
    T, f, gR, _, HR = ti_all(n, sites, g, lay, U, v)
    T2, E, _ = O.alg1(n, sites, g, U)
    _, grad_f, _ = cm.postprocess_gradient(T2, E)
    assert abs(T - T2) < 1e-15
    assert np.abs(gR - cm.riemannian_gradient(g, grad_f)).max() < 1e-15
    _, _, H = O.alg1(n, sites, g, U, v[0])
    Hf, _ = cm.postprocess_hvp(T2, E, H, v[0])
    assert np.abs(HR[0] - cm.riemannian_hvp(g, grad_f, Hf, v[0])).max() < 1e-15


def test_phase_null_vectors():
    n, sites, g, lay, U, _ = ti_problem(n=4, D=3)
    B = S.pauli_basis(g)
    _, _, _, _, HR = ti_all(n, sites, g, lay, U, B[::16])
    assert np.abs(HR).max() < 1e-13
