"""Pins for the seeded input generator (tn_inputs)."""
import numpy as np
import pytest

from tn_inputs import configs as C
from tn_inputs import rng
from tn_inputs.models import Model, dense_hamiltonian, expm_herm, trotter_layers, bond_term
from tn_inputs.reference import mpo_bonds, mpo_to_dense_operator, reference_mpo


def test_splitmix_reference_values():
    # SplitMix64 with state0 = 0: the first outputs of the published generator
    # (Steele/Lea/Flood 2014; same constants as X14).
    z = rng.raw(np.uint64(0), 3)
    assert [int(v) for v in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_uniform_range_and_gaussian_moments():
    u = rng.uniform(rng.stream_key(9, "misc", 0), 200000)
    assert u.min() > 0.0 and u.max() <= 1.0
    g = rng.complex_normal(rng.stream_key(9, "misc", 1), 200000)
    assert abs(g.real.mean()) < 0.01 and abs(g.imag.mean()) < 0.01
    assert abs(g.real.var() - 1) < 0.02 and abs(g.imag.var() - 1) < 0.02
    assert abs(np.mean(g.real * g.imag)) < 0.01


def test_determinism_and_stream_separation():
    a = C.haar_gates(3, 5)
    b = C.haar_gates(3, 5)
    assert np.array_equal(a, b)
    c = C.haar_gates(4, 5)
    assert not np.allclose(a, c)


def test_haar_unitary_and_tangent_directions():
    G = C.haar_gates(2, 7)
    for g in G:
        assert np.abs(g.conj().T @ g - np.eye(4)).max() < 1e-13
    V = C.tangent_directions(2, G, 3)
    for b in range(3):
        for k in range(7):
            S = G[k].conj().T @ V[b, k]
            assert np.abs(S + S.conj().T).max() < 1e-13     # G^dag V skew-Hermitian


def test_brickwall_counts():
    # K = D/2 * floor(n/2) + D/2 * floor((n-1)/2) for even D, offset 0
    for cid, cfg in C.CONFIGS.items():
        K = C.num_gates(cfg.n, cfg.depth)
        exp = (cfg.depth // 2) * (cfg.n // 2) + (cfg.depth // 2) * ((cfg.n - 1) // 2)
        assert K == exp
    assert [C.num_gates(c.n, c.depth) for c in C.CONFIGS.values()] == [10, 60, 186, 392, 1524]


def test_strang_layer_count_matches_paper():
    # PAPER.md:611 "11 layers"; n_steps=5 -> 11 layers
    ly = trotter_layers(Model("tfim", {"J": 1, "h": 0.75, "g": 0.6}), 6, 1.0, 5, 2)
    assert len(ly) == 11


def test_trotter_gate_closed_form_zz():
    # Ising J=1, g=h=0 -> diagonal gate with phases e^{-+ i dt}
    m = Model("tfim", {"J": 1.0, "h": 0.0, "g": 0.0})
    g = expm_herm(bond_term(m, 4, 1), 0.3)
    assert np.allclose(g, np.diag(np.exp(1j * 0.3 * np.array([1, -1, -1, 1]))), atol=1e-15)


@pytest.mark.parametrize("order,slope", [(1, 2.0), (2, 4.0), (4, 16.0)])
def test_trotter_order(order, slope):
    n, t = 5, 0.5
    m = Model("tfim", {"J": 1.0, "h": 0.9, "g": 0.4})
    ex = expm_herm(dense_hamiltonian(m, n), t)
    errs = []
    for steps in (4, 8):
        W = np.eye(2 ** n, dtype=complex)
        for layer in trotter_layers(m, n, t, steps, order):
            for i, g in layer:
                W = np.kron(np.kron(np.eye(2 ** i), g), np.eye(2 ** (n - i - 2))) @ W
        errs.append(np.linalg.norm(W - ex, 2))
    assert abs(errs[0] / errs[1] - slope) < 0.35 * slope


def test_reference_mpo_is_the_trotter_product():
    n = 5
    cfg = C.small_case(7, n, 4, 1024)
    sites = reference_mpo(C.reference_layers(cfg), n, 1024)
    U = mpo_to_dense_operator(sites) * 2 ** (n / 2)
    W = np.eye(2 ** n, dtype=complex)
    for layer in C.reference_layers(cfg):
        for i, g in layer:
            W = np.kron(np.kron(np.eye(2 ** i), g), np.eye(2 ** (n - i - 2))) @ W
    assert np.abs(U - W).max() < 1e-12
    # right-canonical, centre at 0
    for a in sites[1:]:
        a = a.numpy()
        m = a.reshape(a.shape[0], -1)
        assert np.abs(m @ m.conj().T - np.eye(a.shape[0])).max() < 1e-12
    assert mpo_bonds(sites)[0] == 1 and mpo_bonds(sites)[-1] == 1


def test_reference_cap_never_cuts_a_multiplet():
    """X25: a bond cap that would fall inside a cluster of equal singular
    values drops the whole cluster (the truncated reference must be the same
    operator on every machine).  Unit rule + a Heisenberg chain, whose SU(2)
    multiplets are exactly degenerate: every kept bond spectrum ends at a gap."""
    import torch
    from tn_inputs import configs as C
    from tn_inputs.reference import CLUSTER_GAP, _keep_whole_multiplets, reference_mpo
    s = torch.tensor([1.0, 0.5, 0.5, 0.5 * (1 - 1e-12), 0.2, 0.1])
    assert _keep_whole_multiplets(s, 3) == 1          # cap inside the 0.5 triplet: drop all of it
    assert _keep_whole_multiplets(s, 4) == 4          # cap at the gap after the triplet
    assert _keep_whole_multiplets(s, 5) == 5
    assert _keep_whole_multiplets(s, 6) == 6          # nothing beyond: not a cut
    cfg = C.small_case(77, 8, 2, 10, model=C.CONFIGS[2].model, t=0.5, steps=4)
    full = reference_mpo(C.reference_layers(cfg), cfg.n, 256)
    capped = reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)
    sf, sc = C.ref_schmidt_spectra([a.numpy() for a in full]), C.ref_schmidt_spectra([a.numpy() for a in capped])
    shrunk = 0
    for a, b in zip(sf, sc):
        k = len(b)
        assert k <= cfg.chi
        shrunk += k < min(cfg.chi, len(a))
        if k < len(a):                                # a real cut: it sits at a gap of the full spectrum
            assert a[k - 1] - a[k] > CLUSTER_GAP * a[k - 1]
    assert shrunk > 0                                 # the rule was exercised (chi = 10 cuts SU(2) multiplets)
