"""GPU parity: f, T, gradient and Riemannian HVPs of libtn_hvp.so vs the oracle.

Bar (BASELINE.json north_star): relative error <= 1e-10 in complex128 on the
same seeded inputs (X18: rel = ||x_gpu - x_ref|| / ||x_ref|| per output; for
Hess_R the max over directions)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from tests.helpers import gatewise, o2_outputs, oracle_outputs, rel, workload  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

TOL = 1e-10


def gpu_outputs(cfg, ref, G, V, max_batch=64):
    from paper_2604_20384_b200.api import HVPEngine
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], cfg.first_offset, max_batch=max_batch)
    sc, gR = eng.environments(torch.tensor(G, device=dev))
    E = eng.gradient_T()
    H, HT, OM = eng.apply(torch.tensor(V, device=dev), aux=True)
    torch.cuda.synchronize()
    out = {"f": sc[0].item(), "T": complex(sc[1].item(), sc[2].item()), "grad_R": gR.cpu().numpy(),
           "E": E.cpu().numpy(), "HR": H.cpu().numpy(), "HT": HT.cpu().numpy(), "OM": OM.cpu().numpy(),
           "diag": sc.cpu().numpy()}
    eng.close()
    return out


CASES = [
    C.small_case(201, 4, 4, 64, batch=2),                 # untruncated
    C.small_case(202, 6, 5, 8, batch=3),                  # truncation active, odd depth
    C.small_case(203, 7, 4, 6, batch=2, first_offset=1),  # odd n, offset 1
    C.small_case(204, 8, 6, 16, batch=2),
]


def cpp_outputs(cfg, ref, G, V):
    """The plain C++ complex128 oracle (oracle/cpp): the dense truncated
    definition with its own Jacobi SVD, Alg. 2 / App. E postprocessing."""
    from oracle import cpp_oracle as X
    from oracle import dense as O
    from tn_inputs.reference import mpo_bonds, mpo_to_dense_operator
    n = cfg.n
    x0 = O.op_to_vec(np.eye(2 ** n) / 2 ** (n / 2), n)
    top0 = O.op_to_vec(mpo_to_dense_operator(ref), n)
    T, E, H = X.dense_truncated(n, cfg.depth, cfg.chi, G, x0, top0, mpo_bonds(ref), V, cfg.first_offset)
    f, gR, HR = X.postprocess(G, T, E, H, V)
    return {"T": T, "f": f, "E": E, "grad_R": gR, "HR": HR, "HT": H,
            "OM": np.array([np.sum(E * V[b]) for b in range(V.shape[0])])}


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
def test_parity_small(cfg):
    """Against O3 (MPO sweeps), O2 (the dense plain definition with explicit
    Schmidt projectors, n <= 8) AND the plain C++ oracle, whole-output and per
    gate."""
    ref, G, V = workload(cfg, ref_chi=max(cfg.chi, 4))
    g = gpu_outputs(cfg, ref, G, V)
    for o in (oracle_outputs(cfg, ref, G, V), o2_outputs(cfg, ref, G, V), cpp_outputs(cfg, ref, G, V)):
        assert abs(g["T"] - o["T"]) <= TOL * abs(o["T"])
        assert abs(g["f"] - o["f"]) <= TOL * abs(o["f"])
        assert rel(g["E"], o["E"]) < TOL
        gatewise(g["E"], o["E"], TOL)
        assert rel(g["grad_R"], o["grad_R"]) < TOL
        gatewise(g["grad_R"], o["grad_R"], TOL)
        for b in range(V.shape[0]):
            assert rel(g["HT"][b], o["HT"][b]) < TOL, b
            assert rel(g["HR"][b], o["HR"][b]) < TOL, b
            gatewise(g["HR"][b], o["HR"][b], TOL)
            assert abs(g["OM"][b] - o["OM"][b]) <= TOL * abs(o["OM"][b])


def test_parity_low_entanglement_start():
    """Trotter-initialised circuits (the X17 trust-region start, low
    entanglement): many two-site blocks have numerical rank <= the kept rank
    and are split by the range probe instead of an eigendecomposition
    (tn_hvp_split_stats counts them).  Same parity bar against O3; a second
    primal pass at the same point (hints learnt) gives the same outputs."""
    from paper_2604_20384_b200.api import HVPEngine
    cfg = C.small_case(205, 10, 6, 32, batch=2, t=0.3, steps=2)
    ref, _, _ = workload(cfg)
    K = C.num_gates(cfg.n, cfg.depth)
    G = C.trotter_init_gates(cfg, 0)
    V = C.tangent_directions(cfg.cid, G, 2)
    o = oracle_outputs(cfg, ref, G, V)
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], cfg.first_offset, max_batch=2)
    Gt, Vt = torch.tensor(G, device=dev), torch.tensor(V, device=dev)
    for rep in range(2):
        sc, gR = eng.environments(Gt)
        H = eng.apply(Vt)
        st = eng.split_stats()
        assert st["low_rank_splits"] > 0 and st["pair_steps"] == 2 * K, st
        assert abs(sc[0].item() - o["f"]) <= TOL * abs(o["f"])
        assert rel(gR.cpu().numpy(), o["grad_R"]) < TOL
        gatewise(gR.cpu().numpy(), o["grad_R"], TOL)
        for b in range(2):
            assert rel(H[b].cpu().numpy(), o["HR"][b]) < TOL, (rep, b)
            gatewise(H[b].cpu().numpy(), o["HR"][b], TOL)
    eng.close()


def test_parity_config1():
    """C1 (n = 6, exact MPO) against O3 and O2."""
    cfg = C.CONFIGS[1]
    ref, G, V = workload(cfg)
    g = gpu_outputs(cfg, ref, G, V)
    for o in (oracle_outputs(cfg, ref, G, V), o2_outputs(cfg, ref, G, V)):
        assert abs(g["f"] - o["f"]) <= TOL * abs(o["f"])
        assert rel(g["grad_R"], o["grad_R"]) < TOL
        gatewise(g["grad_R"], o["grad_R"], TOL)
        assert rel(g["HR"][0], o["HR"][0]) < TOL
        gatewise(g["HR"][0], o["HR"][0], TOL)


def test_parity_config2():
    cfg = C.CONFIGS[2]
    ref, G, V = workload(cfg)
    o = oracle_outputs(cfg, ref, G, V, dirs=[0, 7, 15])
    g = gpu_outputs(cfg, ref, G, V, max_batch=6)   # ragged sub-batches
    assert abs(g["f"] - o["f"]) <= TOL * abs(o["f"])
    assert rel(g["grad_R"], o["grad_R"]) < TOL
    gatewise(g["grad_R"], o["grad_R"], TOL)
    for b in (0, 7, 15):
        assert rel(g["HR"][b], o["HR"][b]) < TOL, b
        gatewise(g["HR"][b], o["HR"][b], TOL)


def test_apply_is_linear_and_batch_independent():
    cfg = C.small_case(205, 8, 6, 8, batch=3)
    ref, G, V = workload(cfg)
    a, b = 0.6, -1.7                    # Hess_R is real-linear (H_f has conj(H_T))
    Vc = np.concatenate([V[:2], (a * V[0] + b * V[1])[None]], 0)
    g = gpu_outputs(cfg, ref, G, Vc, max_batch=2)
    assert rel(g["HR"][2], a * g["HR"][0] + b * g["HR"][1]) < 1e-12
    g1 = gpu_outputs(cfg, ref, G, Vc[1:2])
    assert rel(g1["HR"][0], g["HR"][1]) < 1e-13


def _layer_sites(cfg):
    from oracle.common import layers
    return layers(cfg.n, cfg.depth, cfg.first_offset)


@pytest.mark.parametrize("cid", [3])
def test_full_size_properties(cid):
    """Properties that hold at any size, at the full config and in the launch
    configuration bench.py times (cfg.batch directions in SUB_BATCH sub-batches):
    per-layer Euler identity of E (X9), grad_R and Hess_R in the tangent space,
    Hess_R real-linear in V, results independent of the direction's position in
    the batch (bitwise)."""
    cfg = C.CONFIGS[cid]
    from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine, riemannian_project
    dev = torch.device("cuda")
    ref = C.reference_mpo(cfg, device=dev)
    K = C.num_gates(cfg.n, cfg.depth)
    G = C.haar_gates(cfg.cid, K)
    V = C.tangent_directions(cfg.cid, G, cfg.batch)
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=SUB_BATCH[cid])
    Gt = torch.tensor(G, device=dev)
    sc, gR = eng.environments(Gt)
    E = eng.gradient_T().cpu().numpy()
    for ly in _layer_sites(cfg):
        vals = np.array([np.sum(G[k] * E[k]) for k, _ in ly])
        assert np.abs(vals - vals[0]).max() <= 1e-12 * np.abs(vals[0])
    assert rel(riemannian_project(Gt, gR).cpu().numpy(), gR.cpu().numpy()) < 1e-13
    Vt = torch.tensor(V, device=dev)
    H = eng.apply(Vt).cpu().numpy()
    Hp = riemannian_project(Gt, torch.tensor(H, device=dev)).cpu().numpy()
    assert rel(Hp, H) < 1e-13
    comb = torch.tensor(np.stack([V[0] + 2.5 * V[1], V[1]]), device=dev)
    Hc = eng.apply(comb).cpu().numpy()
    assert rel(Hc[0], H[0] + 2.5 * H[1]) < 1e-11
    assert rel(Hc[1], H[1]) < 1e-13                     # other batch size (split-K choices may differ)
    Hr = eng.apply(torch.flip(Vt, [0]).contiguous()).cpu().numpy()[::-1]
    assert np.array_equal(Hr, H)                        # same batch size, reversed order: bitwise
    eng.close()


def test_full_size_properties_config5():
    """Config 5 (n=128, D=24, chi=256) at a trust-region starting point (X17),
    max_batch 1 as in truncated CG: the identities of test_full_size_properties
    (Euler per layer, tangency, real linearity)."""
    cfg = C.CONFIGS[5]
    from paper_2604_20384_b200.api import HVPEngine, riemannian_project
    dev = torch.device("cuda")
    ref = C.reference_mpo(cfg, device=dev)
    G = C.trotter_init_gates(cfg, 0)
    V = C.tangent_directions(cfg.cid, G, 2)
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=1)
    Gt = torch.tensor(G, device=dev)
    sc, gR = eng.environments(Gt)
    assert np.isfinite(sc.cpu().numpy()[:6]).all()
    E = eng.gradient_T().cpu().numpy()
    for ly in _layer_sites(cfg):
        vals = np.array([np.sum(G[k] * E[k]) for k, _ in ly])
        assert np.abs(vals - vals[0]).max() <= 1e-11 * np.abs(vals[0])
    assert rel(riemannian_project(Gt, gR).cpu().numpy(), gR.cpu().numpy()) < 1e-13
    comb = np.stack([V[0], V[1], V[0] + 3.0 * V[1]])
    H = eng.apply(torch.tensor(comb, device=dev)).cpu().numpy()
    assert rel(riemannian_project(Gt, torch.tensor(H, device=dev)).cpu().numpy(), H) < 1e-13
    assert rel(H[2], H[0] + 3.0 * H[1]) < 1e-11
    eng.close()


@pytest.mark.parametrize("cid,max_batch", [(2, 8), (3, 64)])
def test_fused_step_equals_environments_plus_apply(cid, max_batch):
    """tn_hvp_step (first sub-batch's forward tangents replayed during the
    primal pass) gives bitwise the results of tn_hvp_environments + tn_hvp_apply."""
    from paper_2604_20384_b200.api import HVPEngine
    cfg = C.CONFIGS[cid]
    dev = torch.device("cuda")
    ref = C.reference_mpo(cfg, device=dev)
    K = C.num_gates(cfg.n, cfg.depth)
    G = torch.tensor(C.haar_gates(cfg.cid, K), device=dev)
    V = torch.tensor(C.tangent_directions(cfg.cid, G.cpu().numpy(), 16), device=dev)
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=max_batch)
    sc1, gR1 = eng.environments(G)
    sc1, gR1 = sc1.clone(), gR1.clone()
    H1 = eng.apply(V)
    sc2, gR2, H2 = eng.step(G, V)
    torch.cuda.synchronize()
    assert torch.equal(sc1[:6], sc2[:6]) and torch.equal(gR1, gR2) and torch.equal(H1, H2)
    H3 = eng.apply(V)                                  # state after the fused step is the same
    assert torch.equal(H3, H1)
    eng.close()


EDGE = [
    C.small_case(231, 2, 3, 4, batch=2),                  # n = 2: layer 2 has no gate (K = 2)
    C.small_case(232, 2, 2, 4, batch=1, first_offset=1),  # n = 2, offset 1: layer 1 empty (K = 1)
    C.small_case(233, 3, 1, 16, batch=2),                 # depth 1
    C.small_case(234, 3, 2, 2, batch=3, first_offset=1),  # odd n, chi = 2 (heavy truncation)
]


@pytest.mark.parametrize("cfg", EDGE, ids=lambda c: c.name)
def test_parity_edge_cases(cfg):
    """Degenerate layouts (empty layers, a single gate, depth 1, chi = 2)
    against O3 and the plain C++ oracle, whole output and per gate."""
    ref, G, V = workload(cfg, ref_chi=max(cfg.chi, 4))
    g = gpu_outputs(cfg, ref, G, V, max_batch=2)           # ragged sub-batches for batch 3
    for o in (oracle_outputs(cfg, ref, G, V), cpp_outputs(cfg, ref, G, V)):
        assert abs(g["f"] - o["f"]) <= TOL * abs(o["f"])
        gatewise(g["grad_R"], o["grad_R"], TOL)
        for b in range(V.shape[0]):
            gatewise(g["HR"][b], o["HR"][b], TOL)


def test_empty_batch_and_zero_direction():
    """batch 0 is a no-op; the zero direction gives a zero Hessian (V = 0 closed form)."""
    from paper_2604_20384_b200.api import HVPEngine
    cfg = C.small_case(235, 4, 3, 8, batch=1)
    ref, G, V = workload(cfg)
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=2)
    eng.environments(torch.tensor(G, device=dev))
    H0 = eng.apply(torch.zeros((0,) + V.shape[1:], dtype=torch.complex128, device=dev))
    assert H0.shape[0] == 0
    Hz = eng.apply(torch.zeros_like(torch.tensor(V, device=dev)))
    assert float(Hz.abs().max()) == 0.0
    eng.close()
