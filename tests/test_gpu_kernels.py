"""GPU: the DMMA complex GEMM and the projection kernel vs CPU references."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import common as cm  # noqa: E402
from tn_inputs import configs as C  # noqa: E402


def _rand(shape, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal(shape) + 1j * g.standard_normal(shape)


@pytest.mark.parametrize("opa,opb", [(a, b) for a in "NTC" for b in "NTC"])
@pytest.mark.parametrize("M,N,K,batch", [(64, 64, 16, 1), (70, 33, 29, 3), (1, 1, 1, 2), (130, 257, 200, 2),
                                         (64, 96, 1000, 1), (100, 64, 2050, 3)])  # last two: split-K
def test_zgemm_ops_ragged(opa, opb, M, N, K, batch):
    from paper_2604_20384_b200.api import zgemm
    As = (batch, M, K) if opa == "N" else (batch, K, M)
    Bs = (batch, K, N) if opb == "N" else (batch, N, K)
    A, B, Cm = _rand(As, 1), _rand(Bs, 2), _rand((batch, M, N), 3)
    op = {"N": lambda x: x, "T": lambda x: np.swapaxes(x, -1, -2), "C": lambda x: np.conj(np.swapaxes(x, -1, -2))}
    ref = (0.3 - 0.7j) * op[opa](A) @ op[opb](B) + (1.1 + 0.2j) * Cm
    dev = torch.device("cuda")
    Ct = torch.tensor(Cm, device=dev)
    out = zgemm(torch.tensor(A, device=dev), torch.tensor(B, device=dev), opa, opb, 0.3 - 0.7j, 1.1 + 0.2j, Ct)
    err = np.abs(out.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err < 1e-14


def test_zgemm_shared_operand_and_stacking():
    from paper_2604_20384_b200.api import zgemm
    dev = torch.device("cuda")
    A, B = _rand((5, 48, 40), 4), _rand((1, 40, 72), 5)
    out = zgemm(torch.tensor(A, device=dev), torch.tensor(B, device=dev)).cpu().numpy()
    assert np.abs(out - A @ B[0]).max() < 1e-12
    A1, B5 = _rand((1, 24, 40), 6), _rand((5, 40, 72), 7)
    out = zgemm(torch.tensor(A1, device=dev), torch.tensor(B5, device=dev)).cpu().numpy()
    assert np.abs(out - A1[0] @ B5).max() < 1e-12


def test_projection_kernel_matches_oracle():
    from paper_2604_20384_b200.api import riemannian_project
    G = C.haar_gates(77, 9)
    Z = _rand((3, 9, 4, 4), 8)
    dev = torch.device("cuda")
    out = riemannian_project(torch.tensor(G, device=dev), torch.tensor(Z, device=dev)).cpu().numpy()
    ref = np.stack([cm.project(G, Z[b]) for b in range(3)])
    assert np.abs(out - ref).max() < 1e-15


def test_retraction_is_the_polar_factor():
    from paper_2604_20384_b200.api import retract
    G = C.haar_gates(78, 7)
    xi = 0.3 * _rand(G.shape, 9)
    dev = torch.device("cuda")
    out = retract(torch.tensor(G, device=dev), torch.tensor(xi, device=dev)).cpu().numpy()
    for k in range(7):
        u, _, vh = np.linalg.svd(G[k] + xi[k])
        assert np.abs(out[k] - u @ vh).max() < 1e-13
        assert np.abs(out[k].conj().T @ out[k] - np.eye(4)).max() < 1e-14


def test_tangent_algebra():
    from paper_2604_20384_b200.api import axpby, tangent_dot
    dev = torch.device("cuda")
    A, B = _rand((3, 5, 4, 4), 10), _rand((3, 5, 4, 4), 11)
    d = tangent_dot(torch.tensor(A, device=dev), torch.tensor(B, device=dev)).cpu().numpy()
    assert np.abs(d - np.real(np.sum(np.conj(A) * B, axis=(1, 2, 3)))).max() < 1e-12
    y = torch.tensor(B, device=dev)
    axpby(0.5 - 1j, torch.tensor(A, device=dev), 2.0, y)
    assert np.abs(y.cpu().numpy() - ((0.5 - 1j) * A + 2.0 * B)).max() < 1e-14


def test_primal_export_import_roundtrip():
    from paper_2604_20384_b200.api import HVPEngine, primal_export, primal_import
    from tn_inputs.reference import reference_mpo
    cfg = C.small_case(79, 6, 4, 8, batch=2)
    ref = reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)
    K = C.num_gates(cfg.n, cfg.depth)
    G1, G2 = C.haar_gates(79, K), C.haar_gates(80, K)
    V = C.tangent_directions(79, G1, 2)
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=2)
    g1 = torch.tensor(G1, device=dev)
    eng.environments(g1)
    H1 = eng.apply(torch.tensor(V, device=dev)).cpu().numpy()
    blob = primal_export(eng).clone()
    eng.environments(torch.tensor(G2, device=dev))
    primal_import(eng, blob, g1)
    H2 = eng.apply(torch.tensor(V, device=dev)).cpu().numpy()
    assert np.array_equal(H1, H2)


def test_error_statuses():
    """TN_ESTATE before a primal pass; TN_ENUMERIC on non-finite gates."""
    from paper_2604_20384_b200 import _native as N
    from paper_2604_20384_b200.api import HVPEngine
    from tn_inputs.reference import reference_mpo
    cfg = C.small_case(81, 6, 4, 8, batch=1)
    ref = reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)
    K = C.num_gates(cfg.n, cfg.depth)
    G = C.haar_gates(81, K)
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=1)
    V = torch.tensor(C.tangent_directions(81, G, 1), device=dev)
    with pytest.raises(N.TNError) as e:
        eng.apply(V)
    assert e.value.status == N.TN_ESTATE
    Gbad = G.copy()
    Gbad[3, 1, 2] = np.nan
    with pytest.raises(N.TNError) as e:
        eng.environments(torch.tensor(Gbad, device=dev))
    assert e.value.status == N.TN_ENUMERIC
    eng.environments(torch.tensor(G, device=dev))         # recovers
    assert torch.isfinite(eng.apply(V)).all()


def test_no_uninitialised_reads_under_nan_poison():
    """TN_POISON=1 fills every new device buffer (pools, owned tensors, arena,
    reduction partials) with NaN bytes: any read of uninitialised memory that
    reaches an output turns it into NaN.  The small parity cases must still
    pass (the library reads the flag at load, hence the subprocess)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TN_POISON="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"), "-k", "small or config1 or linear"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_apply_graph_replay_is_bitwise_eager():
    """Repeated same-batch tn_hvp_apply calls (tCG) run eagerly, then are
    captured into a CUDA graph and replayed: results bitwise equal, launch and
    work counters credited per replay, graphs dropped by the next primal pass."""
    from paper_2604_20384_b200 import _native as N
    from paper_2604_20384_b200.api import HVPEngine
    from tn_inputs.reference import reference_mpo
    cfg = C.small_case(82, 8, 5, 16, batch=3)
    ref = reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)
    K = C.num_gates(cfg.n, cfg.depth)
    G = C.haar_gates(82, K)
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=2)
    V = torch.tensor(C.tangent_directions(82, G, 3), device=dev)
    for rep in range(2):                                   # second primal pass drops and re-captures
        eng.environments(torch.tensor(G, device=dev))
        outs, counts, works = [], [], []
        for call in range(4):
            l0 = N.tn_hvp_launch_count()
            Vc = V.clone()                                 # fresh input buffer each call, as in tCG
            outs.append(eng.apply(Vc).clone())
            torch.cuda.synchronize()
            counts.append(N.tn_hvp_launch_count() - l0)
            works.append(eng.work()[0])
        for o in outs[1:]:
            assert torch.equal(o, outs[0])
        # call 0 replays the point-free graph (captured at the first point, no
        # caches), call 1 runs eagerly and records the point's caches, calls 2
        # (capture + launch) and 3 (replay) run the cached schedule and are
        # credited the same
        assert counts[2] == counts[3] and 0 < counts[2] <= counts[1] <= counts[0]
        assert works[2] == works[3]
        H1 = eng.apply(V[1:2].contiguous())                # other batch size: its own key
        assert torch.equal(H1, eng.apply(V[1:2].contiguous()))
    eng.close()


def test_chain_cache_is_bitwise_uncached():
    """The per-point cache of direction-independent tangent chains (recorded by
    the first apply after a primal pass, borrowed afterwards) changes no bit:
    same HVPs as an engine built with TN_NO_CHAIN_CACHE=1, over several
    sub-batches, repeated calls and two primal passes."""
    import os
    from paper_2604_20384_b200.api import HVPEngine
    from tn_inputs.reference import reference_mpo
    cfg = C.small_case(83, 8, 6, 12, batch=5, first_offset=1)
    ref = [a.to("cuda") for a in reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)]
    K = C.num_gates(cfg.n, cfg.depth, 1)
    dev = torch.device("cuda")
    os.environ["TN_NO_CHAIN_CACHE"] = "1"
    try:
        plain = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, 1, max_batch=2)
    finally:
        del os.environ["TN_NO_CHAIN_CACHE"]
    cached = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, 1, max_batch=2)
    for seed in (83, 84):
        G = torch.tensor(C.haar_gates(seed, K), device=dev)
        V = torch.tensor(C.tangent_directions(seed, G.cpu().numpy(), 5), device=dev)
        plain.environments(G)
        cached.environments(G)
        want = plain.apply(V)
        for _ in range(3):
            assert torch.equal(cached.apply(V), want)
        assert torch.equal(cached.apply(V[2:3].contiguous()), want[2:3])
    plain.close()
    cached.close()


def test_gemm_orthonormalisations_match_householder():
    """The GEMM-rich orthonormalisations of the primal sweeps -- CholeskyQR2 for
    the centre moves and Newton-Schulz steps on the sigma-scaled rows of
    Y = U_r^H A for W_r^H -- give the same outputs (f, grad_R, Hess_R are gauge
    invariant) as an engine built with the Householder factorisations
    (TN_NO_CHOLQR, TN_NO_LOWDIN_LQ), at C2 (chi = 64, truncating) and on a
    small exact case; outputs also match with the kept-only Loewdin step."""
    import os
    from paper_2604_20384_b200.api import HVPEngine
    from tests.helpers import rel
    dev = torch.device("cuda")
    cases = [(C.CONFIGS[2], C.reference_mpo(C.CONFIGS[2], device=dev), 0)]
    from tn_inputs.reference import reference_mpo
    small = C.small_case(85, 10, 6, 16, batch=3, first_offset=1)
    cases.append((small, [a.to(dev) for a in reference_mpo(C.reference_layers(small), small.n, small.chi)], 1))
    for cfg, ref, off in cases:
        K = C.num_gates(cfg.n, cfg.depth, off)
        Gn = C.haar_gates(cfg.cid, K)
        G = torch.tensor(Gn, device=dev)
        V = torch.tensor(C.tangent_directions(cfg.cid, Gn, 3), device=dev)
        os.environ["TN_NO_CHOLQR"] = "1"
        os.environ["TN_NO_LOWDIN_LQ"] = "1"
        try:
            house = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, off, max_batch=3)
        finally:
            del os.environ["TN_NO_CHOLQR"], os.environ["TN_NO_LOWDIN_LQ"]
        fast = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, off, max_batch=3)
        sc0, g0 = house.environments(G)
        sc1, g1 = fast.environments(G)
        H0, H1 = house.apply(V), fast.apply(V)
        assert abs(sc0[0].item() - sc1[0].item()) <= 1e-11 * abs(sc0[0].item())
        assert rel(g1.cpu().numpy(), g0.cpu().numpy()) < 1e-11
        assert rel(H1.cpu().numpy(), H0.cpu().numpy()) < 1e-11
        house.close()
        fast.close()


def test_point_free_graph_follows_the_point():
    """The point-free apply graph is captured at the first point and replayed
    at later points: it must read everything point-specific (store, frozen
    truncation factors) at run time -- bitwise equal to an eager apply at
    each point (the GEMM probe forces the eager path)."""
    from paper_2604_20384_b200 import _native as N
    from paper_2604_20384_b200.api import HVPEngine
    from tn_inputs.reference import reference_mpo
    cfg = C.small_case(83, 8, 5, 8, batch=3)
    ref = reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)
    K = C.num_gates(cfg.n, cfg.depth)
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=3)
    for point in (83, 84, 85):
        G = C.haar_gates(point, K)
        V = torch.tensor(C.tangent_directions(point, G, 3), device=dev)
        eng.environments(torch.tensor(G, device=dev))
        H_graph = eng.apply(V).clone()                 # first apply at the point: point-free graph
        N.tn_gemm_profile(1)
        H_eager = eng.apply(V).clone()                 # profiling forces the eager path
        N.tn_gemm_profile(0)
        assert torch.equal(H_graph, H_eager), point
    eng.close()
