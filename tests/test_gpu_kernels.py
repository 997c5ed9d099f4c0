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
@pytest.mark.parametrize("M,N,K,batch", [(64, 64, 16, 1), (70, 33, 29, 3), (1, 1, 1, 2), (130, 257, 200, 2)])
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
