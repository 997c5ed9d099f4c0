"""GPU checks of the boundary's contracts (include/tn_hvp.h): the argument
flags, fault isolation of tn_hvp_cost, the primal-import
check, caller-owned primal store, graph replay with changing directions."""
import numpy as np
import pytest
import torch

from tn_inputs import configs as C
from tn_inputs.reference import reference_mpo

pytestmark = pytest.mark.gpu


def _setup(cid, n=6, depth=4, chi=8, batch=2, flags=0, max_batch=2):
    from paper_2604_20384_b200.api import HVPEngine
    cfg = C.small_case(cid, n, depth, chi, batch=batch)
    ref = reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)
    K = C.num_gates(cfg.n, cfg.depth)
    G = C.haar_gates(cid, K)
    V = C.tangent_directions(cid, G, batch)
    dev = torch.device("cuda")
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to(dev) for a in ref], max_batch=max_batch, flags=flags)
    return eng, torch.tensor(G, device=dev), torch.tensor(V, device=dev)


def test_check_unitary_flag():
    from paper_2604_20384_b200 import _native as N
    eng, G, V = _setup(301, flags=N.TN_CHECK_UNITARY)
    bad = G.clone()
    bad[5] *= 1.0 + 1e-8                       # ||G^dag G - I|| ~ 4e-8 > 1e-10
    for call in (lambda: eng.environments(bad), lambda: eng.cost(bad), lambda: eng.step(bad, V)):
        with pytest.raises(N.TNError) as e:
            call()
        assert e.value.status == N.TN_EINVAL and "gate 5" in str(e.value)
    eng.environments(G)                        # unitary gates pass
    assert torch.isfinite(eng.apply(V)).all()


def test_check_tangent_flag():
    from paper_2604_20384_b200 import _native as N
    eng, G, V = _setup(302, flags=N.TN_CHECK_TANGENT)
    eng.environments(G)
    H = eng.apply(V)
    bad = V.clone()
    bad[1] += 1e-6 * G                         # P_G(G) = 0: a purely normal component on direction 1
    for call in (lambda: eng.apply(bad), lambda: eng.step(G, bad)):
        with pytest.raises(N.TNError) as e:
            call()
        assert e.value.status == N.TN_EINVAL and "direction 1" in str(e.value)
    eng.environments(G)
    assert torch.equal(eng.apply(V), H)


def test_apply_after_failed_cost_is_unchanged():
    """tn_hvp_cost never writes the stored point: a cost call that fails
    (non-finite trial gates -> TN_ENUMERIC) or succeeds at other gates leaves
    later applies bitwise unchanged (no arena swap)."""
    from paper_2604_20384_b200 import _native as N
    eng, G, V = _setup(303)
    eng.environments(G)
    H0 = eng.apply(V).clone()
    bad = G.clone()
    bad[2, 1, 3] = float("nan")
    with pytest.raises(N.TNError) as e:
        eng.cost(bad)
    assert e.value.status == N.TN_ENUMERIC
    assert torch.equal(eng.apply(V), H0)
    G2 = torch.tensor(C.haar_gates(304, G.shape[0]), device=G.device)
    sc = eng.cost(G2)
    assert torch.isfinite(sc).all()
    for _ in range(3):                         # eager, capture, replay
        assert torch.equal(eng.apply(V), H0)


def test_primal_import_checks_the_point():
    from paper_2604_20384_b200 import _native as N
    from paper_2604_20384_b200.api import primal_export, primal_import
    eng, G, V = _setup(305)
    eng.environments(G)
    H0 = eng.apply(V).clone()
    blob = primal_export(eng).clone()
    G2 = torch.tensor(C.haar_gates(306, G.shape[0]), device=G.device)
    eng.environments(G2)
    with pytest.raises(N.TNError) as e:        # the blob was built at G, not G2
        primal_import(eng, blob, G2)
    assert e.value.status == N.TN_EINVAL
    with pytest.raises(N.TNError) as e:        # store invalid after the failed import
        eng.apply(V)
    assert e.value.status == N.TN_ESTATE
    primal_import(eng, blob, G)
    assert torch.equal(eng.apply(V), H0)


def test_caller_owned_store_and_trim():
    """The primal store is the engine's caller-owned torch buffer of
    tn_hvp_query's size; trimming drops caches/graphs and keeps results."""
    eng, G, V = _setup(307)
    assert eng.primal.numel() >= eng.primal_bytes > 0
    eng.environments(G)
    H0 = eng.apply(V).clone()
    eng.apply(V)
    eng.trim_memory()
    assert torch.equal(eng.apply(V), H0)
    assert torch.equal(eng.apply(V), H0)


def test_graph_replay_follows_new_directions():
    """Repeated same-batch applies are replayed from a CUDA graph: the replay
    must read each call's directions, i.e. equal a cold apply of
    the same direction in another batch shape (no graph for that key yet)."""
    eng, G, V = _setup(308, batch=4, max_batch=4)
    eng.environments(G)
    outs = [eng.apply(V[j:j + 1]).clone() for j in range(4)]   # calls 2..4 replay the batch-1 graph
    full = eng.apply(V)                                         # batch 4: eager
    for j in range(4):
        rel = (outs[j] - full[j:j + 1]).norm() / full[j].norm()
        assert rel < 1e-13, (j, float(rel))
    assert not torch.equal(outs[2], outs[3])


def test_split_primal_two_contexts_equal_full_pass():
    """The split primal of parallel.split_primal emulated with two contexts on
    one GPU (no rank waits on another): context A sweeps the bottom side,
    context B the top side, each copies the other's store region, both finish
    -- f, grad_R and the HVPs equal one full tn_hvp_environments pass."""
    eng, G, V = _setup(309, n=8, depth=5, chi=8, batch=2)
    engB, _, _ = _setup(309, n=8, depth=5, chi=8, batch=2)
    sc, gR = eng.environments(G)
    sc, gR = sc.clone(), gR.clone()
    H = eng.apply(V).clone()
    A, Bc = _setup(309, n=8, depth=5, chi=8, batch=2)[0], engB
    A.environments_part(G, 0)
    Bc.environments_part(G, 1)
    for src, dst, part in ((A, Bc, 0), (Bc, A, 1)):
        off, nb = src.primal_region(part)
        dst.primal_store()[off:off + nb].copy_(src.primal_store()[off:off + nb])
    for e in (A, Bc):
        s2, g2 = e.environments_finish(G)
        assert torch.equal(s2[:6], sc[:6]) and torch.equal(g2, gR)
        assert torch.equal(e.apply(V), H)
