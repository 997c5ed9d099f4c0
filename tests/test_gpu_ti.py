"""N2 on the GPU (reading X20): tn_hvp_ti_environments /
tn_hvp_ti_apply against oracle/ti.py over the O3 (truncated) and O1 (exact)
oracles on the same seeded inputs (1e-10)."""
import numpy as np
import pytest
import torch

from oracle import common as cm
from oracle import dense as O
from oracle import mpo as M
from oracle import ti
from tests.helpers import rel, workload
from tests.test_oracle_exact import problem
from tn_inputs import configs as C

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _gpu(cfg, ref, g, v):
    from paper_2604_20384_b200.api import HVPEngine
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [torch.as_tensor(a).to("cuda") for a in ref], cfg.first_offset,
                    max_batch=2)
    sc, gR = eng.ti_environments(torch.tensor(g, device="cuda"))
    HR = eng.ti_apply(torch.tensor(v, device="cuda"))
    out = (sc[0].item(), gR.cpu().numpy(), HR.cpu().numpy())
    eng.close()
    return out


@pytest.mark.parametrize("cfg", [C.small_case(51, 6, 4, 6, batch=3),
                                 C.small_case(52, 7, 5, 8, batch=3, first_offset=1)], ids=lambda c: c.name)
def test_ti_truncated_matches_oracle(cfg):
    ref, _, _ = workload(cfg, nb=0)
    lay = ti.layer_of_gates(cfg.n, cfg.depth, cfg.first_offset)
    g = C.haar_gates(cfg.cid + 1000, cfg.depth)
    v = C.tangent_directions(cfg.cid + 1000, g, cfg.batch)
    G, V = ti.expand(g, lay), ti.expand(v, lay)
    refs = [a.detach().resolve_conj().cpu().numpy() for a in ref]
    o3 = M.MPOOracle(cfg.n, cfg.depth, cfg.chi, G, refs, V, cfg.first_offset)
    E = o3.gradient_T()
    f, _, gR, _ = ti.gradient(o3.T, E, g, lay)
    HR = np.stack([ti.hvp(o3.T, E, o3.hvp_T(b), g, v[b], lay)[0] for b in range(cfg.batch)])
    fg, gRg, HRg = _gpu(cfg, ref, g, v)              # 3 directions, max_batch 2: ragged sub-batch
    assert abs(fg - f) <= TOL * abs(f)
    assert rel(gRg, gR) < TOL
    assert max(rel(HRg[b], HR[b]) for b in range(cfg.batch)) < TOL


def test_ti_exact_matches_dense_oracle():
    n, sites, _, U, _ = problem(n=4, D=3)
    cfg = C.small_case(11, 4, 3, 64, batch=2)
    from tn_inputs.reference import reference_mpo
    ref = reference_mpo(C.reference_layers(cfg), 4, 4096)
    lay = ti.layer_of_gates(4, 3)
    g = C.haar_gates(1011, 3)
    v = C.tangent_directions(1011, g, 2)
    T, E, _ = O.alg1(n, sites, ti.expand(g, lay), U)
    f, _, gR, _ = ti.gradient(T, E, g, lay)
    HR = []
    for b in range(2):
        _, _, H = O.alg1(n, sites, ti.expand(g, lay), U, ti.expand(v[b], lay))
        HR.append(ti.hvp(T, E, H, g, v[b], lay)[0])
    fg, gRg, HRg = _gpu(cfg, ref, g, v)
    assert abs(fg - f) <= TOL * abs(f)
    assert rel(gRg, gR) < TOL
    assert max(rel(HRg[b], HR[b]) for b in range(2)) < TOL
    assert abs(cm.inner(v[0], HRg[1]) - cm.inner(HRg[0], v[1])) < 1e-12   # exact: self-adjoint


def test_ti_state_errors():
    from paper_2604_20384_b200 import _native as N
    from paper_2604_20384_b200.api import HVPEngine
    cfg = C.small_case(53, 4, 2, 8, batch=1)
    ref, G, V = workload(cfg, nb=1)
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, [a.to("cuda") for a in ref], max_batch=1)
    g = torch.tensor(C.haar_gates(53, 2), device="cuda")
    v = torch.tensor(C.tangent_directions(53, g.cpu().numpy(), 1), device="cuda")
    with pytest.raises(N.TNError) as e:
        eng.ti_apply(v)
    assert e.value.status == N.TN_ESTATE
    eng.ti_environments(g)
    eng.ti_apply(v)
    eng.environments(torch.tensor(G, device="cuda"))     # per-gate pass invalidates the TI view
    with pytest.raises(N.TNError) as e:
        eng.ti_apply(v)
    assert e.value.status == N.TN_ESTATE
    eng.close()
