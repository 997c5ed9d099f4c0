"""Pins for the N4 oracle (oracle/trotter.py): the reference construction of
reading X11.  Against mathematics: the dense Trotter product converges to
exp(-i H t) at the order's rate (textbook Trotter/Suzuki error: ratio 2^order
when the step count doubles), and the untruncated TEBD is that dense product."""
import numpy as np
import pytest

from oracle import trotter as TR
from tn_inputs.models import Model, dense_hamiltonian, expm_herm, trotter_layers
from tn_inputs.reference import mpo_to_dense_operator


def _seq(m, n, t, steps, order):
    return [(i, g) for ly in trotter_layers(m, n, t, steps, order) for i, g in ly]


@pytest.mark.parametrize("order", [1, 2, 4])
def test_dense_product_converges_at_the_trotter_order(order):
    n, t = 5, 0.6
    m = Model("xxz", {"Delta": 0.5, "hz": 0.2})
    ex = expm_herm(dense_hamiltonian(m, n), t)
    e = [np.linalg.norm(TR.dense_product(n, _seq(m, n, t, s, order)) - ex, 2) for s in (3, 6)]
    assert abs(e[0] / e[1] - 2 ** order) < 0.3 * 2 ** order


@pytest.mark.parametrize("n,order", [(5, 1), (6, 2), (6, 4)])
def test_untruncated_tebd_is_the_dense_product(n, order):
    m = Model("tfim", {"J": 1.0, "h": 0.9, "g": 0.4})
    seq = _seq(m, n, 1.0, 3, order)
    sites = TR.tebd(n, seq, 4096, 1e-14)
    U = mpo_to_dense_operator(sites) * 2 ** (n / 2)
    assert np.abs(U - TR.dense_product(n, seq)).max() < 1e-12
    for a in sites[1:]:                                   # right-canonical, centre at 0
        mm = a.reshape(a.shape[0], -1)
        assert np.abs(mm @ mm.conj().T - np.eye(mm.shape[0])).max() < 1e-12
    assert abs(np.linalg.norm(sites[0]) - 1.0) < 1e-14


def test_truncated_tebd_keeps_chi_and_norm():
    n, chi = 8, 8
    m = Model("xxx", {"J": 1.0})
    sites = TR.tebd(n, _seq(m, n, 1.0, 4, 2), chi, 1e-14)
    assert max(a.shape[2] for a in sites) == chi
    assert abs(np.linalg.norm(mpo_to_dense_operator(sites)) - 1.0) < 1e-12
