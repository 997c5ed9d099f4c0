"""The five BASELINE.json workloads (C1..C5) and the seeded inputs they need.

Recipe: U_ref = Trotter circuit of the config's spin
chain compressed to chi (tn_inputs.reference); circuit gates G_k Haar-random
U(4) from stream (cfg, "gates", k); tangent directions V_k = G_k S_k with S_k
skew-Hermitian Gaussian from stream (cfg, "directions", b*K + k) -- a tangent
vector by construction, same law as P_G(Z) for Gaussian Z (X14).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import rng
from .models import Model, layer_pairs, trotter_layers


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    n: int
    depth: int
    chi: int
    model: Model
    t: float
    steps: int
    order: int
    batch: int
    first_offset: int = 0
    extra: dict = field(default_factory=dict)


CONFIGS = {
    1: Config(1, "C1-tfim-n6", 6, 4, 64, Model("tfim", {"J": 1.0, "h": 0.75}), 1.0, 12, 1, 1),
    2: Config(2, "C2-xxx-n16", 16, 8, 64, Model("xxx", {"J": 1.0}), 0.5, 10, 2, 16),
    3: Config(3, "C3-tfim-n32", 32, 12, 128, Model("tfim", {"J": 1.0, "h": 1.0, "g": 0.3}), 1.0, 20, 2, 64),
    4: Config(4, "C4-xxz-n50", 50, 16, 256, Model("xxz", {"Delta": 0.5, "hz": 0.2}), 1.0, 25, 2, 64),
    5: Config(5, "C5-tfim-n128", 128, 24, 256, Model("tfim", {"J": 1.0, "h": 0.9, "g": 0.4}), 2.0, 40, 2, 1,
              extra={"problems": 32, "outer": 10, "max_hvp": 20}),
}


def brickwall_sites(n: int, depth: int, first_offset: int = 0):
    """Left site of every gate, layer-major, left->right (X5)."""
    out = []
    for ell in range(1, depth + 1):
        off = (first_offset + ell - 1) % 2
        out.extend(i for i, _ in layer_pairs(n, off))
    return out


def num_gates(n: int, depth: int, first_offset: int = 0) -> int:
    return len(brickwall_sites(n, depth, first_offset))


def haar_gates(cid: int, K: int) -> np.ndarray:
    return np.stack([rng.haar_u4(rng.stream_key(cid, "gates", k)) for k in range(K)])


def tangent_directions(cid: int, gates: np.ndarray, batch: int, offset: int = 0) -> np.ndarray:
    K = gates.shape[0]
    out = np.empty((batch, K, 4, 4), dtype=np.complex128)
    for b in range(batch):
        for k in range(K):
            s = rng.skew_gaussian(rng.stream_key(cid, "directions", (offset + b) * K + k))
            out[b, k] = gates[k] @ s
    return out


def reference_layers(cfg: Config):
    return trotter_layers(cfg.model, cfg.n, cfg.t, cfg.steps, cfg.order)


def reference_mpo(cfg: Config, device="cpu"):
    from .reference import reference_mpo as _build
    return _build(reference_layers(cfg), cfg.n, cfg.chi, device=device)


def small_case(cid: int, n: int, depth: int, chi: int, batch: int = 2, model: Model | None = None,
               t: float = 0.6, steps: int = 3, order: int = 2, first_offset: int = 0) -> Config:
    """A reduced workload for oracle-speed tests (same recipe, smaller sizes)."""
    m = model or Model("tfim", {"J": 1.0, "h": 0.9, "g": 0.4})
    return Config(cid, f"small-{cid}-n{n}-D{depth}-chi{chi}", n, depth, chi, m, t, steps, order, batch,
                  first_offset)


def trotter_init_gates(cfg: Config, problem: int, steps: int | None = None, eps: float = 0.05) -> np.ndarray:
    """Config-5 starting circuits: the 1st-order Trotter circuit
    of the config's H with D/2 steps (one A and one B layer per step = the
    brickwall layout), each gate multiplied by exp(-i eps H_s) with H_s a
    seeded GUE 4x4 from stream (cfg, "init", problem*K + k)."""
    from .models import bond_term, expm_herm
    steps = steps or cfg.depth // 2
    dt = cfg.t / steps
    sites = brickwall_sites(cfg.n, cfg.depth, cfg.first_offset)
    K = len(sites)
    out = np.empty((K, 4, 4), dtype=np.complex128)
    for k, s in enumerate(sites):
        a = rng.complex_normal(rng.stream_key(cfg.cid, "init", problem * K + k), 16).reshape(4, 4)
        hs = 0.5 * (a + a.conj().T)
        out[k] = expm_herm(bond_term(cfg.model, cfg.n, s), dt) @ expm_herm(hs, eps)
    return out


# Full-size parity cases with stored oracle outputs (tests/golden/full_*.npz,
# written by tools/golden_full.py).  "c5r" is config 5 at full width and
# bond cap (n = 128, chi = 256, C5's reference MPO) with a reduced depth D = 4
# and the X17 Trotter start of problem 0 (the trust-region regime whose cuts
# fall in the noise floor); the full-depth C5 oracle does not fit this
# container's memory.
FULL_PARITY_CASES = ("c3", "c4", "c5r")


def full_parity_config(case: str) -> Config:
    if case == "c3":
        return CONFIGS[3]
    if case == "c4":
        return CONFIGS[4]
    if case == "c5r":
        c5 = CONFIGS[5]
        return Config(5, "C5r-tfim-n128-D4", c5.n, 4, c5.chi, c5.model, c5.t, c5.steps, c5.order, 1)
    raise ValueError(case)


def full_parity_inputs(case: str, dirs: int):
    """(config, gates, first `dirs` directions) of a full-size parity case."""
    cfg = full_parity_config(case)
    K = num_gates(cfg.n, cfg.depth, cfg.first_offset)
    if case == "c5r":
        G = trotter_init_gates(cfg, 0)
    else:
        G = haar_gates(cfg.cid, K)
    return cfg, G, tangent_directions(cfg.cid, G, dirs)


def ref_fingerprint(sites):
    """(bonds, per-site sum |x|) of a reference MPO (gauge dependent)."""
    import numpy as _np
    bonds = [1] + [int(x.shape[2]) for x in sites]
    norms = _np.array([float(_np.abs(_np.asarray(x)).sum()) for x in sites])
    return bonds, norms


def ref_schmidt_spectra(sites):
    """Operator Schmidt values of a right-canonical MPO at every cut c = 1..n-1
    (singular values of the bond matrix after moving the centre there by QR):
    a gauge-invariant fingerprint of the operator, so a reference rebuilt on
    another machine (different LAPACK rounding, different bond gauge) can be
    checked to be the same input.  Returns a list of descending arrays."""
    import numpy as _np
    a = [_np.asarray(x, dtype=_np.complex128) for x in sites]
    out = []
    c = a[0]
    for j in range(len(a) - 1):
        b, p, bp = c.shape
        q, r = _np.linalg.qr(c.reshape(b * p, bp))
        out.append(_np.linalg.svd(r, compute_uv=False))
        c = _np.einsum("ab,bpc->apc", r, a[j + 1])
    return out


def ref_probe_overlaps(sites, nprobe: int = 4, bond: int = 3):
    """Overlaps <<X_j|R>> of an MPO R with `nprobe` fixed pseudo-random MPOs X_j of
    bond dimension `bond` (numpy default_rng(1000 + j), one site tensor reused at
    every site): gauge invariant like the Schmidt values, but they also tell
    apart two operators with equal Schmidt values (e.g. different kept parts of a
    degenerate multiplet).  Returns (unit-modulus-scaled complex mantissas,
    log10 magnitudes) so that long chains neither overflow nor underflow."""
    import numpy as _np
    a = [_np.asarray(x, dtype=_np.complex128) for x in sites]
    mant, logs = [], []
    for j in range(nprobe):
        rng = _np.random.default_rng(1000 + j)
        x = (rng.standard_normal((bond, 4, bond)) + 1j * rng.standard_normal((bond, 4, bond))) / _np.sqrt(8.0 * bond)
        env = _np.zeros((bond, a[0].shape[0]), dtype=_np.complex128)
        env[0, :] = 1.0
        lg = 0.0
        for t in a:                                   # env[x, r] <- sum conj(X[x, p, x']) env[x, r] R[r, p, r']
            env = _np.einsum("xr,xpy,rpq->yq", env, x.conj(), t, optimize=True)
            nrm = _np.linalg.norm(env)
            env /= nrm
            lg += _np.log10(nrm)
        mant.append(env[0, :].sum())
        logs.append(lg)
    return _np.array(mant), _np.array(logs)
