"""GPU parity of N4: the reference MPO built by the library (tn_mpo_tebd, the
primal pass's kernels) against the oracle (oracle/trotter.py): the dense
Trotter product when untruncated, the numpy TEBD of reading X11 when
truncated (bonds equal; gauge-invariant operator Schmidt values at every cut
and the normalised overlap agree)."""
import numpy as np
import pytest
import torch

from oracle import trotter as TR
from tn_inputs import configs as C
from tn_inputs.models import Model, trotter_layers
from tn_inputs.reference import mpo_to_dense_operator

pytestmark = pytest.mark.gpu


def _seq(layers):
    return [(i, g) for ly in layers for i, g in ly]


def _overlap(a, b):
    L = np.ones((1, 1), dtype=np.complex128)
    for x, y in zip(a, b):
        L = np.einsum("tb,tpu,bpv->uv", L, np.conj(x), y)
    return complex(L[0, 0])


@pytest.mark.parametrize("n,order", [(5, 1), (6, 2), (7, 4)])
def test_tebd_without_bond_cap(n, order):
    """No chi cap: the GPU keeps every sigma above its resolution floor
    1e-7 sigma_1 (X23); the oracle TEBD at the same threshold gives the same
    operator to that floor (the Gram split resolves the kept vectors next to a
    1e-7 cut only to ~1e-8), and both are the dense Trotter product to the size
    of the discarded tail (1e-6)."""
    from paper_2604_20384_b200.api import mpo_tebd
    m = Model("tfim", {"J": 1.0, "h": 0.9, "g": 0.4})
    layers = trotter_layers(m, n, 1.0, 3, order)
    sites = [a.cpu().numpy() for a in mpo_tebd(n, layers, 4096, 1e-14)]
    o = TR.tebd(n, _seq(layers), 4096, 1e-7)
    assert [x.shape for x in sites] == [x.shape for x in o]
    U = mpo_to_dense_operator(sites) * 2 ** (n / 2)
    assert np.abs(U - mpo_to_dense_operator(o) * 2 ** (n / 2)).max() <= 1e-7 * np.abs(U).max()
    assert np.abs(U - TR.dense_product(n, _seq(layers))).max() < 1e-6
    for a in sites[1:]:
        mm = a.reshape(a.shape[0], -1)
        assert np.abs(mm @ mm.conj().T - np.eye(mm.shape[0])).max() < 1e-12


@pytest.mark.parametrize("cid", [2, 3])
def test_tebd_truncated_matches_oracle(cid):
    """C2 / C3 references (chi = 64 / 128) at tol 1e-7, the threshold the Gram
    split resolves: same bonds, same operator (Schmidt values at every cut to
    1e-7 of the cut's largest -- the split's resolution, X23 -- and normalised
    overlap 1 - O(1e-12), the difference entering it only at second order)."""
    from paper_2604_20384_b200.api import mpo_tebd
    cfg = C.CONFIGS[cid]
    layers = C.reference_layers(cfg)
    g = [a.cpu().numpy() for a in mpo_tebd(cfg.n, layers, cfg.chi, 1e-7)]
    o = TR.tebd(cfg.n, _seq(layers), cfg.chi, 1e-7)
    assert [x.shape for x in g] == [x.shape for x in o]
    for sg, so in zip(C.ref_schmidt_spectra(g), C.ref_schmidt_spectra(o)):
        assert np.abs(sg - so).max() <= 1e-7 * so[0]
    assert abs(_overlap(g, o)) > 1 - 1e-12
    assert abs(_overlap(g, g) - 1) < 1e-12
