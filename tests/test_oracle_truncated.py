"""Pins for the truncated definition: O2 (dense, explicit Schmidt projectors)
and O3 (MPO sweeps, channel-form tangents) -- two structurally independent
realisations of SURVEY.md §8(c.2) -- plus reduction to the exact O1."""
import numpy as np
import pytest

from oracle import common as cm
from oracle import dense as O
from oracle import mpo as M
from tn_inputs import configs as C
from tn_inputs.reference import mpo_bonds, mpo_to_dense_operator, reference_mpo


def setup(n, D, cid, nb=2, offset=0, ref_chi=4096):
    cfg = C.small_case(cid, n, D, ref_chi, batch=nb, first_offset=offset)
    ref = reference_mpo(C.reference_layers(cfg), n, ref_chi)
    refs = [a.numpy() for a in ref]
    U = mpo_to_dense_operator(ref) * 2 ** (n / 2)
    sites = C.brickwall_sites(n, D, offset)
    G = C.haar_gates(cid, len(sites))
    V = C.tangent_directions(cid, G, nb)
    return refs, mpo_bonds(ref), U, sites, G, V


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b))


@pytest.mark.parametrize("n,D,offset", [(4, 4, 0), (5, 4, 1), (6, 3, 0)])
def test_untruncated_equals_exact(n, D, offset):
    refs, bonds, U, sites, G, V = setup(n, D, 40 + n, offset=offset)
    T, E, H = O.alg1(n, sites, G, U, V[0])
    o2 = O.DenseTruncated(n, D, 10 ** 6, G, O.op_to_vec(U / 2 ** (n / 2), n), bonds, V, offset)
    o3 = M.MPOOracle(n, D, 10 ** 6, G, refs, V, offset)
    for o in (o2, o3):
        assert abs(o.T - T) < 1e-14
        assert rel(o.gradient_T(), E) < 1e-13
        assert rel(o.hvp_T(0), H) < 1e-13


@pytest.mark.parametrize("n,D,chi,offset", [(6, 4, 4, 0), (7, 5, 8, 0), (6, 5, 6, 1), (8, 4, 16, 0)])
def test_mpo_sweeps_equal_dense_definition_with_truncation(n, D, chi, offset):
    refs, bonds, U, sites, G, V = setup(n, D, 50 + n + chi, offset=offset)
    o2 = O.DenseTruncated(n, D, chi, G, O.op_to_vec(U / 2 ** (n / 2), n), bonds, V, offset)
    o3 = M.MPOOracle(n, D, chi, G, refs, V, offset)
    disc = [1 - np.sum(d["sigma"][:d["r"]] ** 2) / np.sum(d["sigma"] ** 2) for d in o2.diag]
    assert max(disc) > 1e-3                      # truncation really active
    assert abs(o2.T - o3.T) < 1e-13 * max(1, abs(o2.T))
    assert rel(o3.gradient_T(), o2.gradient_T()) < 1e-12
    for b in range(2):
        assert rel(o3.hvp_T(b), o2.hvp_T(b)) < 1e-11
    assert o3.diag["remainder"] < 1e-10         # before/after-chain reduction exact


def test_truncated_hvp_is_linear_in_the_direction():
    n, D, chi = 7, 4, 8
    refs, bonds, U, sites, G, V = setup(n, D, 61, nb=2)
    a, b = 0.7 - 0.2j, -1.3
    Vc = np.concatenate([V, (a * V[0] + b * V[1])[None]], 0)
    o3 = M.MPOOracle(n, D, chi, G, refs, Vc)
    H = [o3.hvp_T(i) for i in range(3)]
    assert rel(H[2], a * H[0] + b * H[1]) < 1e-13


def test_tangent_bond_bound_two_chi():
    """Tangent Schmidt rank <= 2 chi at every cut (App. D),
    chi = the intermediate states' maximum bond: the reference
    is compressed to chi as in the configs."""
    n, D, chi = 7, 6, 4
    refs, bonds, U, sites, G, V = setup(n, D, 62, ref_chi=chi)
    o2 = O.DenseTruncated(n, D, chi, G, O.op_to_vec(U / 2 ** (n / 2), n), bonds, V)
    for states in (o2.DB[1:], [o2.DT[ell] for ell in range(1, D)]):
        for st in states:
            for x in st:
                for c in range(1, n):
                    s = np.linalg.svd(x.reshape(4 ** c, -1), compute_uv=False)
                    assert np.sum(s > 1e-12 * s[0]) <= 2 * chi


def test_layer_euler_identity_under_truncation():
    """Layer-wise environments are exact within the layer (X9): for each layer
    T^(ell) = sum_ab G_k E_k for every gate k of that layer."""
    n, D, chi = 8, 6, 8
    refs, bonds, U, sites, G, V = setup(n, D, 63, nb=1)
    o3 = M.MPOOracle(n, D, chi, G, refs, V)
    E = o3.gradient_T()
    for ell, ly in enumerate(cm.layers(n, D), start=1):
        vals = [np.sum(G[k] * E[k]) for k, _ in ly]
        assert np.abs(np.array(vals) - o3.layer_T[ell - 1]).max() < 1e-14


def test_chi_convergence_to_exact():
    """O3 -> O1 as chi -> the structural maximum (exact at 4^(n/2))."""
    n, D = 8, 6
    refs, bonds, U, sites, G, V = setup(n, D, 64, nb=1)
    T, E, H = O.alg1(n, sites, G, U, V[0])
    errs = []
    for chi in (8, 32, 256):
        o3 = M.MPOOracle(n, D, chi, G, refs, V)
        errs.append(rel(o3.hvp_T(0), H))
    assert errs[0] > errs[1] > 1e-9
    assert errs[2] < 1e-12


def test_insensitive_to_noise_floor_directions():
    """Reading X10: with chi above the reference's numerical rank the cut falls
    inside the ~1e-14 noise floor (kept directions there are arbitrary); the
    outputs nevertheless move only at roundoff level under 1e-15 gate jitter."""
    n, D, chi = 8, 4, 128
    cfg = C.Config(3, "noise", n, D, chi, C.CONFIGS[3].model, 1.0, 20, 2, 1)
    ref = reference_mpo(C.reference_layers(cfg), n, 1024)
    refs = [a.numpy() for a in ref]
    G = C.haar_gates(3, C.num_gates(n, D))
    V = C.tangent_directions(3, G, 1)
    rng = np.random.default_rng(5)
    P = 1e-15 * (rng.standard_normal(G.shape) + 1j * rng.standard_normal(G.shape))
    outs = []
    for Gx in (G, G + P):
        o = M.MPOOracle(n, D, chi, Gx, refs, V)
        outs.append((o.T, o.gradient_T(), o.hvp_T(0), o.diag))
    sig = [d["sigma"][d["r"] - 1] / d["sigma"][0] for d in outs[0][3]["top"]]
    assert min(sig) < 1e-13                      # the cut really is in the noise floor
    assert abs(outs[0][0] - outs[1][0]) < 1e-12 * abs(outs[0][0])
    assert rel(outs[1][2], outs[0][2]) < 1e-12


def test_tangent_projector_is_the_orthogonal_tangent_projection():
    """O2's frozen-projector map P_T = P^L(x)I + I(x)P^R - P^L(x)P^R (SURVEY.md
    §8(c.5)(iii)): idempotent, self-adjoint in the
    Frobenius inner product, identity on tangent vectors Ur A + B Vr, and its
    complement is (1 - P^L) D (1 - P^R).  A sign error on the -P^L(x)P^R term
    (or a dropped term) breaks idempotence and the complement identity."""
    rng = np.random.default_rng(7)

    def cn(*s):
        return rng.standard_normal(s) + 1j * rng.standard_normal(s)

    for (m, n_, r) in ((12, 10, 3), (16, 16, 5), (8, 20, 8)):
        Ur = np.linalg.qr(cn(m, r))[0]
        Vr = np.linalg.qr(cn(n_, r))[0].conj().T          # rows orthonormal (r x n)
        D, E = cn(m, n_), cn(m, n_)
        P = O.tangent_project(D, Ur, Vr)
        assert np.abs(O.tangent_project(P, Ur, Vr) - P).max() < 1e-13
        assert abs(np.vdot(E, P) - np.vdot(O.tangent_project(E, Ur, Vr), D)) < 1e-12 * np.abs(D).sum()
        Y = Ur @ cn(r, n_) + cn(m, r) @ Vr
        assert np.abs(O.tangent_project(Y, Ur, Vr) - Y).max() < 1e-12
        PL, PR = Ur @ Ur.conj().T, Vr.conj().T @ Vr
        comp = (np.eye(m) - PL) @ D @ (np.eye(n_) - PR)
        assert np.abs(D - P - comp).max() < 1e-12
        # rank of the projection <= 2 r (the 2-chi tangent bound)
        assert np.linalg.matrix_rank(P, tol=1e-10) <= 2 * r
    # the wrong-sign variant fails idempotence (the pin is sensitive to it)
    def wrong(X):
        PLX = Ur @ (Ur.conj().T @ X)
        return PLX + (X @ Vr.conj().T) @ Vr + (PLX @ Vr.conj().T) @ Vr
    assert np.abs(wrong(wrong(D)) - wrong(D)).max() > 1e-3
