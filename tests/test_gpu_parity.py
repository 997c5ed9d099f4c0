"""GPU parity: f, T, gradient and Riemannian HVPs of libtn_hvp.so vs the oracle.

Bar (BASELINE.json north_star): relative error <= 1e-10 in complex128 on the
same seeded inputs (X18: rel = ||x_gpu - x_ref|| / ||x_ref|| per output; for
Hess_R the max over directions)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from tests.helpers import oracle_outputs, rel, workload  # noqa: E402
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


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
def test_parity_small(cfg):
    ref, G, V = workload(cfg, ref_chi=max(cfg.chi, 4))
    o = oracle_outputs(cfg, ref, G, V)
    g = gpu_outputs(cfg, ref, G, V)
    assert abs(g["T"] - o["T"]) <= TOL * abs(o["T"])
    assert abs(g["f"] - o["f"]) <= TOL * abs(o["f"])
    assert rel(g["E"], o["E"]) < TOL
    assert rel(g["grad_R"], o["grad_R"]) < TOL
    for b in range(V.shape[0]):
        assert rel(g["HT"][b], o["HT"][b]) < TOL, b
        assert rel(g["HR"][b], o["HR"][b]) < TOL, b
        assert abs(g["OM"][b] - o["OM"][b]) <= TOL * abs(o["OM"][b])


def test_parity_config1():
    cfg = C.CONFIGS[1]
    ref, G, V = workload(cfg)
    o = oracle_outputs(cfg, ref, G, V)
    g = gpu_outputs(cfg, ref, G, V)
    assert abs(g["f"] - o["f"]) <= TOL * abs(o["f"])
    assert rel(g["grad_R"], o["grad_R"]) < TOL
    assert rel(g["HR"][0], o["HR"][0]) < TOL


def test_parity_config2():
    cfg = C.CONFIGS[2]
    ref, G, V = workload(cfg)
    o = oracle_outputs(cfg, ref, G, V, dirs=[0, 7, 15])
    g = gpu_outputs(cfg, ref, G, V, max_batch=6)   # ragged sub-batches
    assert abs(g["f"] - o["f"]) <= TOL * abs(o["f"])
    assert rel(g["grad_R"], o["grad_R"]) < TOL
    for b in (0, 7, 15):
        assert rel(g["HR"][b], o["HR"][b]) < TOL, b


def test_apply_is_linear_and_batch_independent():
    cfg = C.small_case(205, 8, 6, 8, batch=3)
    ref, G, V = workload(cfg)
    a, b = 0.6, -1.7                    # Hess_R is real-linear (H_f has conj(H_T))
    Vc = np.concatenate([V[:2], (a * V[0] + b * V[1])[None]], 0)
    g = gpu_outputs(cfg, ref, G, Vc, max_batch=2)
    assert rel(g["HR"][2], a * g["HR"][0] + b * g["HR"][1]) < 1e-12
    g1 = gpu_outputs(cfg, ref, G, Vc[1:2])
    assert rel(g1["HR"][0], g["HR"][1]) < 1e-13
