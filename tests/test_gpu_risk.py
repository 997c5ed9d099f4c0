"""GPU parity of N1, the sampled-state empirical risk (PAPER.md:525-554,
eq:costHS): the state-mode CUDA path (site_dim = 2) against the pinned oracle
oracle/risk.py (state-mode O3) on the same seeded product states and labels.
Bar: 1e-10 relative (north_star), whole output and per gate."""
import numpy as np
import pytest
import torch

from oracle import risk as R
from tests.helpers import gatewise, rel
from tn_inputs import configs as C
from tn_inputs import samples as SMP
from tn_inputs.reference import reference_mpo

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _case(cid, n, D, chi, S, nb, offset=0, model_cfg=None):
    cfg = model_cfg or C.small_case(cid, n, D, chi, batch=nb, first_offset=offset)
    ref = [a.numpy() for a in reference_mpo(C.reference_layers(cfg), cfg.n, max(cfg.chi, 64))]
    psis = SMP.haar_product_states(cid, S, cfg.n)
    labels = [SMP.label_mps(ref, p) for p in psis]
    K = C.num_gates(cfg.n, cfg.depth, cfg.first_offset)
    G = C.haar_gates(cid, K)
    V = C.tangent_directions(cid, G, nb)
    return cfg, psis, labels, G, V


CASES = [(501, 5, 4, 64, 2, 2, 0),     # untruncated
         (502, 6, 4, 4, 3, 2, 0),      # truncation active
         (503, 7, 5, 4, 2, 2, 1),      # odd n, offset 1, odd depth
         (504, 8, 6, 8, 3, 3, 0)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"n{c[1]}-D{c[2]}-chi{c[3]}-S{c[4]}")
def test_risk_parity_small(case):
    from paper_2604_20384_b200.risk import EmpiricalRisk
    cid, n, D, chi, S, nb, off = case
    cfg, psis, labels, G, V = _case(cid, n, D, chi, S, nb, off)
    o = R.empirical_risk(n, D, chi, G, labels, psis, V, off)
    dev = torch.device("cuda")
    er = EmpiricalRisk(n, D, chi, [[torch.tensor(a, device=dev) for a in lab] for lab in labels], psis, off,
                       max_batch=2)
    risk, gR = er.environments(torch.tensor(G, device=dev))
    H = er.apply(torch.tensor(V, device=dev))
    torch.cuda.synchronize()
    assert abs(risk.item() - o["risk"]) <= TOL * abs(o["risk"])
    assert rel(gR.cpu().numpy(), o["grad_R"]) < TOL
    gatewise(gR.cpu().numpy(), o["grad_R"], TOL)
    Hn = H.cpu().numpy()
    for b in range(nb):
        assert rel(Hn[b], o["HR"][b]) < TOL, b
        gatewise(Hn[b], o["HR"][b], TOL)
    # per-sample overlaps and E of the state-mode engines against O3 state mode
    for s, eng in enumerate(er.engines):
        sc, _ = eng.environments(torch.tensor(G, device=dev))
        T = complex(sc[1].item(), sc[2].item())
        assert abs(T - o["T"][s]) <= TOL * abs(o["T"][s])
        E = eng.gradient_T().cpu().numpy()
        assert rel(E, o["oracles"][s].gradient_T()) < TOL
    er.close()


def test_risk_parity_config2_width():
    """C2's width and reference (n = 16 XXX, chi = 64, depth 8) with 4 samples."""
    from paper_2604_20384_b200.risk import EmpiricalRisk
    c2 = C.CONFIGS[2]
    cfg, psis, labels, G, V = _case(511, 0, 0, 0, 4, 2, model_cfg=c2)
    o = R.empirical_risk(c2.n, c2.depth, c2.chi, G, labels, psis, V)
    dev = torch.device("cuda")
    er = EmpiricalRisk(c2.n, c2.depth, c2.chi, [[torch.tensor(a, device=dev) for a in lab] for lab in labels],
                       psis, max_batch=2)
    risk, gR = er.environments(torch.tensor(G, device=dev))
    H = er.apply(torch.tensor(V, device=dev)).cpu().numpy()
    assert abs(risk.item() - o["risk"]) <= TOL * abs(o["risk"])
    gatewise(gR.cpu().numpy(), o["grad_R"], TOL)
    for b in range(2):
        assert rel(H[b], o["HR"][b]) < TOL
        gatewise(H[b], o["HR"][b], TOL)
    er.close()


def test_state_mode_rejects_operator_calls():
    from paper_2604_20384_b200 import _native as N
    from paper_2604_20384_b200.api import HVPEngine
    cfg = C.small_case(521, 4, 2, 8, batch=1)
    ref = [a.to("cuda") for a in reference_mpo(C.reference_layers(cfg), 4, 8)]
    eng = HVPEngine(4, 2, 8, ref, max_batch=1)                 # operator mode
    with pytest.raises(N.TNError) as e:
        eng.set_product_state(torch.zeros(4, 2, dtype=torch.complex128, device="cuda"))
    assert e.value.status == N.TN_EINVAL
    eng.close()


def test_trust_region_on_the_empirical_risk():
    """The paper's training loop: Riemannian trust
    region with truncated CG on the sampled-state risk, every f, gradient and
    HVP from the state-mode engines.  The risk's cost() equals its primal pass
    at the same gates, accepted steps decrease the risk, iterates stay unitary."""
    from paper_2604_20384_b200.risk import EmpiricalRisk
    from paper_2604_20384_b200.trust_region import TRParams, TrustRegion
    cid, n, D, chi, S = 541, 8, 4, 8, 3
    cfg = C.small_case(cid, n, D, chi, batch=1)
    ref = [a.numpy() for a in reference_mpo(C.reference_layers(cfg), n, 64)]
    psis = SMP.haar_product_states(cid, S, n)
    dev = torch.device("cuda")
    labels = [[torch.tensor(a, device=dev) for a in SMP.label_mps(ref, p)] for p in psis]
    er = EmpiricalRisk(n, D, chi, labels, psis, max_batch=1)
    x0 = torch.tensor(C.trotter_init_gates(cfg, 0), device=dev)
    r0, _ = er.environments(x0)
    assert abs(er.cost(x0).item() - r0.item()) <= 1e-12 * abs(r0.item())
    x, f, tr = TrustRegion(er, TRParams(outer=6, max_hvp=10)).run(x0)
    acc = [r for r in tr.records if r.get("accepted")]
    assert acc and f < r0.item()
    fs = [tr.records[0]["f"]] + [r["f_trial"] for r in acc]
    assert all(b <= a + 1e-14 for a, b in zip(fs, fs[1:]))
    Xn = x.cpu().numpy()
    assert np.abs(np.einsum("kba,kbc->kac", Xn.conj(), Xn) - np.eye(4)).max() < 1e-12
    er.close()
