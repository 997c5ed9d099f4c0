"""N3 on the GPU: Pauli basis and coordinate kernels,
the symmetric-part eigensolver, the assembled Hessian matrix, its spectrum and
the CG probe, against oracle/spectrum.py on the same seeded inputs (1e-10)."""
import numpy as np
import pytest
import torch

from oracle import common as cm
from oracle import mpo as M
from oracle import spectrum as S
from tests.helpers import rel, workload
from tests.test_oracle_exact import dense_riemannian_hessian, problem
from tn_inputs import configs as C

pytestmark = pytest.mark.gpu
TOL = 1e-10


def test_basis_and_coordinate_kernels():
    from paper_2604_20384_b200.api import pauli_basis, pauli_coords
    G = C.haar_gates(31, 7)
    Gt = torch.tensor(G, device="cuda")
    B = S.pauli_basis(G)
    assert np.abs(pauli_basis(Gt, 0, 112).cpu().numpy() - B).max() < 1e-15
    assert np.abs(pauli_basis(Gt, 37, 20).cpu().numpy() - B[37:57]).max() < 1e-15   # ragged window
    assert pauli_basis(Gt, 112, 0).shape == (0, 7, 4, 4)
    X = C.tangent_directions(31, G, 5) + 0.3 * np.stack([G] * 5)     # not tangent: coordinates still defined
    c = pauli_coords(Gt, torch.tensor(X, device="cuda")).cpu().numpy()
    want = np.stack([S.coordinates(B, x) for x in X])
    assert np.abs(c - want).max() < 1e-14 * np.abs(want).max()


@pytest.mark.parametrize("n", [1, 7, 160, 517])
def test_sym_eig(n):
    from paper_2604_20384_b200.api import sym_eig
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    A = A + A.T + 1e-3 * rng.standard_normal((n, n))
    want, asym = S.spectrum(A)
    w, a, Vt = sym_eig(torch.tensor(A, device="cuda"), vectors=True)
    w, a, Vt = w.cpu().numpy(), a.cpu().numpy(), Vt.cpu().numpy()
    assert np.abs(w - want).max() < 1e-12 * np.abs(want).max()
    assert abs(a[0] / a[1] - asym) < 1e-12
    Sm = 0.5 * (A + A.T)
    assert np.abs(Vt @ Vt.T - np.eye(n)).max() < 1e-12
    assert np.abs(Vt @ Sm - w[:, None] * Vt).max() < 1e-11 * np.abs(want).max()


def _engine(n, D, chi, ref, G, max_batch):
    from paper_2604_20384_b200.api import HVPEngine
    eng = HVPEngine(n, D, chi, [torch.as_tensor(a).to("cuda") for a in ref], max_batch=max_batch)
    Gt = torch.tensor(G, device="cuda")
    sc, gR = eng.environments(Gt)
    return eng, Gt, gR


def test_exact_hessian_matrix_and_spectrum():
    """Untruncated (chi = 4^n/2): the GPU matrix equals the dense O1 Hessian,
    phase columns vanish, the spectrum matches."""
    from paper_2604_20384_b200.spectrum import hessian_matrix, hessian_spectrum
    n, sites, G, U, _ = problem(n=4, D=3)
    Mo = dense_riemannian_hessian(n, sites, G, U)
    from tn_inputs.reference import reference_mpo
    cfg = C.small_case(11, 4, 3, 4096)
    ref = reference_mpo(C.reference_layers(cfg), 4, 4096)
    eng, Gt, _ = _engine(4, 3, 64, ref, G, 48)
    Mt = hessian_matrix(eng, Gt, chunk=48).cpu().numpy()       # 16K = 80: ragged last chunk
    assert rel(Mt.T, Mo) < TOL
    assert np.abs(Mt[::16]).max() < 1e-12 * np.abs(Mo).max()  # phase directions
    w, asym = hessian_spectrum(eng, Gt, chunk=80)
    wo, asym_o = S.spectrum(Mo)
    assert np.abs(w.cpu().numpy() - wo).max() < TOL * np.abs(wo).max()
    assert asym < 1e-12 and asym_o < 1e-12
    eng.close()


def test_truncated_hessian_matrix_and_cg_probe():
    """Truncation active (n=6, D=4, chi=6): matrix vs O3 column by column,
    asymmetry reported identically, CG residual history vs the oracle's CG."""
    from paper_2604_20384_b200.spectrum import cg_probe, hessian_matrix, hessian_spectrum
    cfg = C.small_case(41, 6, 4, 6, batch=1)
    ref, G, _ = workload(cfg, nb=0)
    B = S.pauli_basis(G)
    refs = [a.detach().resolve_conj().cpu().numpy() for a in ref]
    o3 = M.MPOOracle(cfg.n, cfg.depth, cfg.chi, G, refs, B, cfg.first_offset)
    E = o3.gradient_T()
    _, grad_f, _ = cm.postprocess_gradient(o3.T, E)
    gR = cm.riemannian_gradient(G, grad_f)

    def hvp_col(j):
        Hf, _ = cm.postprocess_hvp(o3.T, E, o3.hvp_T(j), B[j])
        return cm.riemannian_hvp(G, grad_f, Hf, B[j])
    cols = [hvp_col(j) for j in range(len(B))]
    Mo = np.array([S.coordinates(B, c) for c in cols]).T
    eng, Gt, gR_gpu = _engine(cfg.n, cfg.depth, cfg.chi, ref, G, 64)
    Mt = hessian_matrix(eng, Gt).cpu().numpy()
    assert rel(Mt.T, Mo) < TOL
    w, asym = hessian_spectrum(eng, Gt)
    wo, asym_o = S.spectrum(Mo)
    assert asym_o > 1e-8                        # truncation: not exactly self-adjoint (X19)
    assert abs(asym - asym_o) < 1e-8 * asym_o
    assert np.abs(w.cpu().numpy() - wo).max() < TOL * np.abs(wo).max()
    # CG on H x = -grad_R, matrix-free: the oracle's CG on the oracle matrix in coordinates
    iters = 6
    _, res = cg_probe(eng, -gR_gpu, iters)
    _, res_o = S.cg_probe(lambda v: Mo @ v, lambda a, c: float(a @ c), -S.coordinates(B, gR), iters)
    assert len(res) == len(res_o)
    assert np.max(np.abs(np.array(res) - res_o) / res_o[0]) < 1e-8
    eng.close()
