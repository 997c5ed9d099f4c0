"""CPU-side checks of the boundary: the library loads, exports every symbol
include/tn_hvp.h declares, and rejects bad arguments before any launch."""
import ctypes
import os
import re

import pytest

import paper_2604_20384_b200._native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "tn_hvp.h")).read()
    return sorted(set(re.findall(r"\b(tn_[a-z_A-Z0-9]+)\s*\(", src)))


def test_header_and_library_exports_match():
    names = declared()
    assert set(names) == set(N.EXPORTS)
    lib = ctypes.CDLL(N.LIB_PATH)
    for nm in names:
        assert hasattr(lib, nm), nm


def test_num_gates():
    assert [N.tn_hvp_num_gates(n, d) for n, d in [(6, 4), (16, 8), (32, 12), (50, 16), (128, 24)]] == \
        [10, 60, 186, 392, 1524]
    assert N.tn_hvp_num_gates(1, 4, 0) == -1


def test_invalid_arguments_rejected_without_gpu():
    cfg = N.make_config(1, 4, 8, max_batch=4)         # n < 2
    with pytest.raises(N.TNError) as e:
        N.tn_hvp_setup(cfg, [1, 1], 1, 0)
    assert e.value.status == N.TN_EINVAL
    cfg = N.make_config(4, 4, 8, max_batch=4)
    with pytest.raises(N.TNError) as e:
        N.tn_hvp_setup(cfg, [2, 1, 1, 1, 1], 1, 0)  # boundary bond != 1
    assert e.value.status == N.TN_EINVAL
    with pytest.raises(N.TNError) as e:
        N.tn_zgemm("X", "N", 4, 4, 4, 1.0, 1, 4, 0, 1, 4, 0, 0.0, 1, 4, 0, 1, 0)
    assert e.value.status == N.TN_EINVAL
    with pytest.raises(N.TNError) as e:
        N.tn_riemannian_project(-1, 1, 1, 1, 1, 0)
    assert e.value.status == N.TN_EINVAL
    for call in (lambda: N.tn_pauli_basis(3, 40, 9, 1, 1, 0),     # first + count > 16 K
                 lambda: N.tn_pauli_basis(3, -1, 1, 1, 1, 0),
                 lambda: N.tn_pauli_coords(3, 2, 0, 1, 1, 0),     # null gates
                 lambda: N.tn_sym_eig(4, 1, 1, 1, 2, 0)):         # vectors not in {0, 1}
        with pytest.raises(N.TNError) as e:
            call()
        assert e.value.status == N.TN_EINVAL


def test_product_path_has_no_oracle_import():
    pkg = os.path.join(ROOT, "paper_2604_20384_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith(".py"):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f


def test_query_sizes_without_gpu():
    """tn_hvp_query plans the sweeps on the host: no CUDA call, sizes grow with chi."""
    bonds = [1] + [4] * 7 + [1]
    sizes = []
    for chi in (4, 8, 16):
        cfg = N.make_config(8, 6, chi, max_batch=2)
        p, w, d = N.tn_hvp_query(cfg, bonds)
        assert p > 0 and w > 0 and d > 0 and p % 256 == 0
        sizes.append((p, w, d))
    assert sizes[0][0] < sizes[1][0] < sizes[2][0]
    assert sizes[0][2] < sizes[1][2] <= sizes[2][2]
    # C4-sized plan (host only): the primal store is GiB-scale, a direction ~1 GiB
    c4 = N.make_config(50, 16, 256, max_batch=32)
    p, w, d = N.tn_hvp_query(c4, [1] + [min(4 ** min(s, 50 - s), 256) for s in range(1, 50)] + [1])
    assert 1 << 30 < p < 64 << 30 and 1 << 28 < d < 8 << 30


def test_config_checks_without_gpu():
    bonds = [1, 4, 4, 4, 1]
    for cfg, why in ((N.make_config(4, 4, 8, 2, dtype=N.TN_C64), "complex64 not built"),
                     (N.make_config(4, 4, 8, 2, flags=1 << 7), "unknown flag"),
                     (N.make_config(4, 4, 8, 2, first_offset=2), "offset"),
                     (N.make_config(4, 4, 8, 0), "max_batch"),
                     (N.make_config(4, 4, 8, 2, site_dim=3), "site_dim"),
                     (N.make_config(4, 4, 8, 2, site_dim=2), "state-mode bonds within a factor 2")):
        with pytest.raises(N.TNError) as e:
            N.tn_hvp_query(cfg, bonds)
        assert e.value.status == N.TN_EINVAL, why
    ok = N.make_config(4, 4, 8, 2, flags=N.TN_CHECK_UNITARY | N.TN_CHECK_TANGENT)
    p, _, _ = N.tn_hvp_query(ok, bonds)
    # a caller-owned primal store smaller than the query's size is rejected
    # before any CUDA call (fake, aligned device pointers: nothing is touched)
    with pytest.raises(N.TNError) as e:
        N.tn_hvp_setup(ok, bonds, 256, 0, primal_ptr=1 << 20, primal_bytes=p - 256)
    assert e.value.status == N.TN_EINVAL and "primal_buf" in str(e.value)
    with pytest.raises(N.TNError) as e:
        N.tn_hvp_setup(ok, bonds, 256, 0, primal_ptr=(1 << 20) + 8, primal_bytes=p)
    assert e.value.status == N.TN_EINVAL and "aligned" in str(e.value)
