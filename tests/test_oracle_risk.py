"""Pins for the N1 oracle (oracle/risk.py, state mode of O1/O2/O3): the
sampled-state empirical risk of PAPER.md:525-554 (eq:costHS).

Pinned against mathematics the paper fixes, not against the oracle itself:
the label MPS equals U_ref psi densely; per sample T_s = <psi| U_ref^dag W |psi>
 from the dense circuit; the state-mode MPO sweeps equal the
exact dense Algorithm 1 on vectors when untruncated and the dense
explicit-projector definition O2 when truncated; the risk's gradient and HVP
equal finite differences of the risk; the risk is the sample mean."""
import numpy as np
import pytest

from oracle import common as cm
from oracle import dense as O
from oracle import mpo as M
from oracle import risk as R
from tn_inputs import configs as C
from tn_inputs import samples as SMP
from tn_inputs.reference import mpo_bonds, mpo_to_dense_operator, reference_mpo


def setup(n, D, cid, S=2, nb=2, offset=0, ref_chi=4096):
    cfg = C.small_case(cid, n, D, ref_chi, batch=nb, first_offset=offset)
    ref = reference_mpo(C.reference_layers(cfg), n, ref_chi)
    refs = [a.numpy() for a in ref]
    U = mpo_to_dense_operator(ref) * 2 ** (n / 2)
    psis = SMP.haar_product_states(cid, S, n)
    labels = [SMP.label_mps(refs, p) for p in psis]
    sites = C.brickwall_sites(n, D, offset)
    G = C.haar_gates(cid, len(sites))
    V = C.tangent_directions(cid, G, nb)
    return refs, U, psis, labels, sites, G, V


def dense_state(psi):
    x = psi[0]
    for p in psi[1:]:
        x = np.kron(x, p)
    return x


def mps_to_vector(sites):
    t = sites[0]
    for a in sites[1:]:
        t = np.tensordot(t, a, axes=([t.ndim - 1], [0]))
    return t.reshape(-1)


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b))


def test_product_states_and_labels():
    refs, U, psis, labels, *_ = setup(5, 3, 401, S=3)
    for p, lab in zip(psis, labels):
        assert np.allclose(np.linalg.norm(p, axis=1), 1.0, atol=1e-15)
        assert rel(mps_to_vector(lab), U @ dense_state(p)) < 1e-13       # phi = U_ref psi
        bonds = SMP.mps_bonds(lab)
        assert all(bonds[j + 1] <= 2 * bonds[j] and bonds[j] <= 2 * bonds[j + 1] for j in range(len(lab)))
        for a in lab[1:]:                                                   # right-canonical, centre at 0
            m = a.reshape(a.shape[0], -1)
            assert np.abs(m @ m.conj().T - np.eye(m.shape[0])).max() < 1e-13


@pytest.mark.parametrize("n,D,offset", [(4, 4, 0), (5, 3, 1), (6, 3, 0)])
def test_state_mode_untruncated_equals_exact(n, D, offset):
    refs, U, psis, labels, sites, G, V = setup(n, D, 410 + n, offset=offset)
    psi = dense_state(psis[0])
    phi = U @ psi
    T, E, H = O.alg1(n, sites, G, None, V[0], psi0=psi[:, None], phi0=phi[:, None])
    # closed form of the overlap: <psi| U_ref^dag W |psi>
    assert abs(T - np.vdot(phi, O.dense_circuit(n, sites, G) @ psi)) < 1e-13
    o3 = M.MPOOracle(n, D, 10 ** 6, G, labels[0], V, offset, psi=psis[0])
    assert abs(o3.T - T) < 1e-13
    assert rel(o3.gradient_T(), E) < 1e-12
    assert rel(o3.hvp_T(0), H) < 1e-12
    # and the O(K^2) substitution sum of the exact HVP
    Hs = np.zeros_like(H)
    for kp in range(len(sites)):
        Gs = G.copy()
        Gs[kp] = V[0, kp]
        _, Es, _ = O.alg1(n, sites, Gs, None, psi0=psi[:, None], phi0=phi[:, None])
        Hs += Es
        Hs[kp] -= Es[kp]
    assert rel(H, Hs) < 1e-12


@pytest.mark.parametrize("n,D,chi,offset", [(6, 4, 2, 0), (7, 5, 4, 1), (8, 4, 4, 0)])
def test_state_mode_mpo_equals_dense_definition_with_truncation(n, D, chi, offset):
    refs, U, psis, labels, sites, G, V = setup(n, D, 420 + n + chi, offset=offset)
    lab = labels[0]
    o2 = O.DenseTruncated(n, D, chi, G, mps_to_vector(lab).reshape((2,) * n), SMP.mps_bonds(lab), V, offset,
                          psi=psis[0])
    o3 = M.MPOOracle(n, D, chi, G, lab, V, offset, psi=psis[0])
    disc = [1 - np.sum(d["sigma"][:d["r"]] ** 2) / np.sum(d["sigma"] ** 2) for d in o2.diag]
    assert max(disc) > 1e-3                                 # truncation really active
    assert abs(o2.T - o3.T) < 1e-12 * max(1, abs(o2.T))
    assert rel(o3.gradient_T(), o2.gradient_T()) < 1e-11
    for b in range(2):
        assert rel(o3.hvp_T(b), o2.hvp_T(b)) < 1e-10
    assert o3.diag["remainder"] < 1e-10


def _risk_dense(n, sites, G, U, psis):
    W = O.dense_circuit(n, sites, G)
    vals = []
    for p in psis:
        x = dense_state(p)
        vals.append(abs(np.vdot(U @ x, W @ x)) ** 2)
    return 1.0 - float(np.mean(vals))


def test_risk_gradient_and_hvp_by_finite_differences():
    n, D = 4, 4
    refs, U, psis, labels, sites, G, V = setup(n, D, 431, S=3, nb=1)
    out = R.empirical_risk(n, D, 10 ** 6, G, labels, psis, V)
    assert abs(out["risk"] - _risk_dense(n, sites, G, U, psis)) < 1e-13
    Z = (np.random.default_rng(5).standard_normal(G.shape) + 1j * np.random.default_rng(6).standard_normal(G.shape))
    eps = 1e-5
    fd = (_risk_dense(n, sites, G + eps * Z, U, psis) - _risk_dense(n, sites, G - eps * Z, U, psis)) / (2 * eps)
    assert abs(fd - cm.inner(out["grad_f"], Z)) < 1e-9 * max(1.0, abs(fd))
    gp = R.empirical_risk(n, D, 10 ** 6, G + eps * V[0], labels, psis)["grad_f"]
    gm = R.empirical_risk(n, D, 10 ** 6, G - eps * V[0], labels, psis)["grad_f"]
    assert np.abs((gp - gm) / (2 * eps) - out["H_f"][0]).max() < 1e-8 * max(1.0, np.abs(out["H_f"][0]).max())
    # Riemannian outputs live in the tangent space
    assert rel(cm.project(G, out["grad_R"]), out["grad_R"]) < 1e-13
    assert rel(cm.project(G, out["HR"][0]), out["HR"][0]) < 1e-13


def test_risk_is_the_sample_mean():
    n, D, chi = 6, 4, 4
    refs, U, psis, labels, sites, G, V = setup(n, D, 441, S=3, nb=1)
    all3 = R.empirical_risk(n, D, chi, G, labels, psis, V)
    one = [R.empirical_risk(n, D, chi, G, [labels[s]], psis[s:s + 1], V) for s in range(3)]
    assert abs(all3["risk"] - np.mean([o["risk"] for o in one])) < 1e-14
    assert rel(all3["grad_R"], sum(o["grad_R"] for o in one) / 3) < 1e-13
    assert rel(all3["HR"][0], sum(o["HR"][0] for o in one) / 3) < 1e-13
