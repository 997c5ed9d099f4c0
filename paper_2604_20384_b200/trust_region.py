"""Riemannian trust region with truncated CG on U(4)^K (a11).

PAPER.md:516 (Absil Alg. 10 + Alg. 11, truncated CG), :615 (several HVPs per
TR step).  Objective, gradient and Hessian-vector products come from the C ABI
(HVPEngine: tn_hvp_environments / tn_hvp_apply / tn_hvp_cost); the retraction
(polar factor) and the tangent-vector algebra (metric
Re sum Tr(A^dag B), X15) are library kernels too (tn_retract,
tn_tangent_dot, tn_tangent_axpby).  Only the scalar control flow runs here.
Defaults (X16): Delta0 = 0.01 sqrt(16K), Delta_max = 100 Delta0,
rho' = 0.1, kappa = 0.1, theta = 1, at most max_hvp HVPs per outer step.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from .api import axpby, retract, tangent_dot


@dataclass
class TRParams:
    delta0: float | None = None
    delta_max_factor: float = 100.0
    rho_accept: float = 0.1
    kappa: float = 0.1
    theta: float = 1.0
    max_hvp: int = 20
    outer: int = 10
    grad_tol: float = 0.0


@dataclass
class TRTrace:
    records: list = field(default_factory=list)
    hvps: int = 0
    grads: int = 0


def _dot(a, b):
    return float(tangent_dot(a[None], b[None]).item())


def truncated_cg(g, hvp, delta, kappa, theta, max_hvp):
    """Steihaug-Toint tCG (Absil Alg. 11, no preconditioner) for
    min <g,eta> + 1/2 <eta, H eta>, ||eta|| <= delta.  Returns
    (eta, H eta, n_hvp, stop, boundary)."""
    eta = torch.zeros_like(g)
    Heta = torch.zeros_like(g)
    r = g.clone()
    d = -r
    r_r = _dot(r, r)
    norm_r0 = math.sqrt(r_r)
    e_Pe, e_Pd, d_Pd = 0.0, 0.0, r_r
    stop, n = "maxiter", 0
    for _ in range(max_hvp):
        Hd = hvp(d)
        n += 1
        d_Hd = _dot(d, Hd)
        alpha = r_r / d_Hd if d_Hd != 0 else math.inf
        e_Pe_new = e_Pe + 2 * alpha * e_Pd + alpha * alpha * d_Pd
        if d_Hd <= 0 or e_Pe_new >= delta * delta:
            tau = (-e_Pd + math.sqrt(e_Pd * e_Pd + d_Pd * (delta * delta - e_Pe))) / d_Pd
            axpby(tau, d, 1.0, eta)
            axpby(tau, Hd, 1.0, Heta)
            return eta, Heta, n, ("negative curvature" if d_Hd <= 0 else "exceeded trust region"), True
        axpby(alpha, d, 1.0, eta)
        axpby(alpha, Hd, 1.0, Heta)
        e_Pe = e_Pe_new
        axpby(alpha, Hd, 1.0, r)
        r_r_new = _dot(r, r)
        if math.sqrt(r_r_new) <= norm_r0 * min(norm_r0 ** theta, kappa):
            stop = "converged"
            break
        beta = r_r_new / r_r
        r_r = r_r_new
        axpby(-1.0, r, beta, d)          # d = -r + beta d
        e_Pd = beta * (e_Pd + alpha * d_Pd)
        d_Pd = r_r + beta * beta * d_Pd
    return eta, Heta, n, stop, False


class TrustRegion:
    """Drive one problem: engine = HVPEngine set up for (n, D, chi, U_ref)."""

    def __init__(self, engine, params: TRParams | None = None):
        self.eng = engine
        self.p = params or TRParams()

    def _env(self, x):
        sc, gR = self.eng.environments(x)
        return float(sc[0].item()), gR

    def run(self, x0: torch.Tensor):
        p = self.p
        K = x0.shape[0]
        delta = p.delta0 if p.delta0 is not None else 0.01 * math.sqrt(16 * K)
        delta_max = p.delta_max_factor * delta
        x = x0.clone()
        tr = TRTrace()
        f, g = self._env(x)
        tr.grads += 1
        for it in range(p.outer):
            gn = math.sqrt(_dot(g, g))
            if gn <= p.grad_tol:
                tr.records.append({"iter": it, "f": f, "grad_norm": gn, "stop": "grad_tol"})
                break
            hvp = lambda v: self.eng.apply(v[None].contiguous())[0]
            eta, Heta, nh, stop, boundary = truncated_cg(g, hvp, delta, p.kappa, p.theta, p.max_hvp)
            tr.hvps += nh
            model_dec = -(_dot(g, eta) + 0.5 * _dot(eta, Heta))
            x_new = retract(x, eta)
            f_new = float(self.eng.cost(x_new)[0].item())
            rho = (f - f_new) / model_dec if model_dec > 0 else -math.inf
            rec = {"iter": it, "f": f, "grad_norm": gn, "delta": delta, "rho": rho, "f_trial": f_new,
                   "n_hvp": nh, "tcg_stop": stop, "boundary": boundary, "eta_norm": math.sqrt(_dot(eta, eta))}
            if rho < 0.25:
                delta = delta / 4
            elif rho > 0.75 and boundary:
                delta = min(2 * delta, delta_max)
            rec["accepted"] = bool(rho > p.rho_accept)
            if rec["accepted"]:
                x = x_new
                f, g = self._env(x)
                tr.grads += 1
            rec["cum_hvp"], rec["cum_grad"] = tr.hvps, tr.grads
            tr.records.append(rec)
        return x, f, tr
