"""Pins for the trust-region / truncated-CG driver (oracle twin, CPU) and the
GPU driver's agreement with it (gpu-marked)."""
import math

import numpy as np
import pytest

from oracle import common as cm
from oracle import dense as O
from oracle import mpo as M
from oracle import trust as TR
from tn_inputs import configs as C
from tn_inputs.reference import mpo_to_dense_operator, reference_mpo

inner_r = lambda a, b: float(np.real(np.vdot(a, b)))


def test_tcg_identity_hessian_is_one_newton_step():
    g = np.random.default_rng(0).standard_normal(16)
    eta, _, n, stop, bnd = TR.tcg(g, lambda v: v, inner_r, delta=1e3)
    assert n == 1 and stop == "converged" and not bnd
    assert np.abs(eta + g).max() < 1e-14


def test_tcg_negative_curvature_goes_to_the_boundary():
    g = np.random.default_rng(1).standard_normal(16)
    eta, _, n, stop, bnd = TR.tcg(g, lambda v: -v, inner_r, delta=0.3)
    assert stop == "negative curvature" and bnd and n == 1
    assert abs(np.linalg.norm(eta) - 0.3) < 1e-14
    assert np.abs(eta / np.linalg.norm(eta) + g / np.linalg.norm(g)).max() < 1e-14


def test_tcg_spd_matches_dense_solve():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((16, 16))
    H = A @ A.T + 16 * np.eye(16)
    g = rng.standard_normal(16)
    eta, _, n, stop, _ = TR.tcg(g, lambda v: H @ v, inner_r, delta=1e6, kappa=1e-14, theta=1.0, max_iter=200)
    assert np.abs(eta - np.linalg.solve(H, -g)).max() < 1e-8


def test_rtr_quadratic_surrogate_converges():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((12, 12))
    H = A @ A.T + np.eye(12)
    b = rng.standard_normal(12)

    class Q:
        f = staticmethod(lambda x: 0.5 * x @ H @ x - b @ x)
        grad = staticmethod(lambda x: H @ x - b)
        hess = staticmethod(lambda x, v: H @ v)
        retract = staticmethod(lambda x, e: x + e)
        inner = staticmethod(inner_r)

    x, f, tr = TR.rtr(Q, np.zeros(12), delta0=0.5, delta_max=50, outer=60, max_hvp=12, kappa=1e-3)
    assert np.abs(x - np.linalg.solve(H, b)).max() < 1e-6
    fs = [r["f"] for r in tr]
    assert all(fs[i + 1] <= fs[i] + 1e-12 for i in range(len(fs) - 1))


class CircuitProblem:
    """f = -|Tr(U_ref^dag W)|^2/4^n on U(4)^K with Riemannian derivatives (O3 oracle)."""

    def __init__(self, n, D, chi, refs):
        self.n, self.D, self.chi, self.refs = n, D, chi, refs

    def _o(self, x, V=None):
        return M.MPOOracle(self.n, self.D, self.chi, x, self.refs, V)

    def f(self, x):
        return -abs(self._o(x).T) ** 2

    def grad(self, x):
        o = self._o(x)
        _, gf, _ = cm.postprocess_gradient(o.T, o.gradient_T())
        return cm.riemannian_gradient(x, gf)

    def hess(self, x, v):
        o = self._o(x, v[None])
        E = o.gradient_T()
        _, gf, _ = cm.postprocess_gradient(o.T, E)
        Hf, _ = cm.postprocess_hvp(o.T, E, o.hvp_T(0), v)
        return cm.riemannian_hvp(x, gf, Hf, v)

    retract = staticmethod(lambda x, e: np.stack([TR.polar(x[k] + e[k]) for k in range(len(x))]))
    inner = staticmethod(cm.inner)


def circuit_case(cid=601, n=6, D=4, chi=8):
    cfg = C.small_case(cid, n, D, chi, batch=1)
    ref = reference_mpo(C.reference_layers(cfg), n, chi)
    K = C.num_gates(n, D)
    # start near the reference: a Trotter-like circuit perturbed (X17 spirit)
    G = C.haar_gates(cid, K)
    return cfg, ref, G


def test_rtr_on_a_circuit_decreases_and_stays_unitary():
    cfg, ref, G = circuit_case()
    P = CircuitProblem(cfg.n, cfg.depth, cfg.chi, [a.numpy() for a in ref])
    K = G.shape[0]
    x, f, tr = TR.rtr(P, G, delta0=0.01 * math.sqrt(16 * K), delta_max=math.sqrt(16 * K), outer=4, max_hvp=8)
    acc = [r["f"] for r in tr if r["accepted"]]
    assert f <= tr[0]["f"]
    for k in range(K):
        assert np.abs(x[k].conj().T @ x[k] - np.eye(4)).max() < 1e-12


@pytest.mark.gpu
def test_gpu_trust_region_matches_oracle_trajectory():
    import torch

    from paper_2604_20384_b200.api import HVPEngine
    from paper_2604_20384_b200.trust_region import TRParams, TrustRegion
    cfg, ref, G = circuit_case()
    K = G.shape[0]
    P = CircuitProblem(cfg.n, cfg.depth, cfg.chi, [a.numpy() for a in ref])
    d0 = 0.01 * math.sqrt(16 * K)
    x_o, f_o, tr_o = TR.rtr(P, G, delta0=d0, delta_max=100 * d0, outer=3, max_hvp=8)
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=1)
    x_g, f_g, tr_g = TrustRegion(eng, TRParams(delta0=d0, outer=3, max_hvp=8)).run(torch.tensor(G, device=dev))
    for a, b in zip(tr_o, tr_g.records):
        assert a["accepted"] == b["accepted"] and a["n_hvp"] == b["n_hvp"] and a["tcg_stop"] == b["tcg_stop"]
        assert abs(a["f"] - b["f"]) <= 1e-9 * abs(a["f"])
    assert np.abs(x_g.cpu().numpy() - x_o).max() < 1e-8
    xg = x_g.cpu().numpy()
    for k in range(K):
        assert np.abs(xg[k].conj().T @ xg[k] - np.eye(4)).max() < 1e-12
