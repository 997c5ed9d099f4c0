"""Riemannian trust region + truncated CG (oracle twin of the GPU driver).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Absil, Mahony & Sepulchre
Alg. 10 (RTR) with Alg. 11 (Steihaug-Toint truncated CG), as cited by
PAPER.md:516; written from the textbook algorithm, not from the GPU driver.
The objective is a provider with f(x), grad(x), hess(x, v), retract(x, xi),
inner(a, b) -- e.g. the O3 oracle on U(4)^K, or a quadratic surrogate.
"""
from __future__ import annotations

import math

import numpy as np


def tcg(g, hess, inner, delta, kappa=0.1, theta=1.0, max_iter=20):
    eta = np.zeros_like(g)
    Heta = np.zeros_like(g)
    r = g.copy()
    delta_vec = -r
    rr = inner(r, r)
    r0 = math.sqrt(rr)
    for j in range(max_iter):
        Hd = hess(delta_vec)
        dHd = inner(delta_vec, Hd)
        if dHd <= 0:
            tau = _to_boundary(eta, delta_vec, delta, inner)
            return eta + tau * delta_vec, Heta + tau * Hd, j + 1, "negative curvature", True
        alpha = rr / dHd
        eta_new = eta + alpha * delta_vec
        if math.sqrt(inner(eta_new, eta_new)) >= delta:
            tau = _to_boundary(eta, delta_vec, delta, inner)
            return eta + tau * delta_vec, Heta + tau * Hd, j + 1, "exceeded trust region", True
        eta, Heta = eta_new, Heta + alpha * Hd
        r = r + alpha * Hd
        rr_new = inner(r, r)
        if math.sqrt(rr_new) <= r0 * min(r0 ** theta, kappa):
            return eta, Heta, j + 1, "converged", False
        delta_vec = -r + (rr_new / rr) * delta_vec
        rr = rr_new
    return eta, Heta, max_iter, "maxiter", False


def _to_boundary(eta, d, delta, inner):
    """tau >= 0 with ||eta + tau d|| = delta."""
    a = inner(d, d)
    b = 2 * inner(eta, d)
    c = inner(eta, eta) - delta * delta
    return (-b + math.sqrt(b * b - 4 * a * c)) / (2 * a)


def rtr(problem, x0, delta0, delta_max, outer=10, max_hvp=20, rho_accept=0.1, kappa=0.1, theta=1.0):
    x = x0
    f = problem.f(x)
    g = problem.grad(x)
    delta = delta0
    trace = []
    for it in range(outer):
        eta, Heta, nh, stop, boundary = tcg(g, lambda v: problem.hess(x, v), problem.inner, delta, kappa, theta,
                                            max_hvp)
        mdec = -(problem.inner(g, eta) + 0.5 * problem.inner(eta, Heta))
        x_new = problem.retract(x, eta)
        f_new = problem.f(x_new)
        rho = (f - f_new) / mdec if mdec > 0 else -math.inf
        rec = {"iter": it, "f": f, "delta": delta, "rho": rho, "n_hvp": nh, "tcg_stop": stop, "boundary": boundary}
        if rho < 0.25:
            delta /= 4
        elif rho > 0.75 and boundary:
            delta = min(2 * delta, delta_max)
        rec["accepted"] = rho > rho_accept
        if rec["accepted"]:
            x, f, g = x_new, f_new, problem.grad(x_new)
        trace.append(rec)
    return x, f, trace


def polar(M):
    u, _, vh = np.linalg.svd(M)
    return u @ vh
