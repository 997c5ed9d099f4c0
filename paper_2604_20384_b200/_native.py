"""ctypes binding of libtn_hvp.so (include/tn_hvp.h): argument marshalling only.

Same names as the C ABI.  Loading fails loudly if the in-tree library is
missing; there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtn_hvp.so")

TN_OK, TN_EINVAL, TN_ENOMEM, TN_ECUDA, TN_ENUMERIC, TN_ESTATE = range(6)
STATUS = {0: "TN_OK", 1: "TN_EINVAL", 2: "TN_ENOMEM", 3: "TN_ECUDA", 4: "TN_ENUMERIC", 5: "TN_ESTATE"}

EXPORTS = ["tn_hvp_num_gates", "tn_hvp_setup", "tn_hvp_environments", "tn_hvp_apply", "tn_hvp_gradient_T",
           "tn_hvp_cost", "tn_hvp_primal_blob", "tn_hvp_primal_imported", "tn_riemannian_project", "tn_zgemm",
           "tn_hvp_work", "tn_hvp_split_stats", "tn_retract", "tn_tangent_dot", "tn_tangent_axpby", "tn_hvp_primal_copy",
           "tn_hvp_launch_count", "tn_gemm_profile", "tn_pauli_basis", "tn_pauli_coords", "tn_sym_eig",
           "tn_hvp_ti_environments", "tn_hvp_ti_apply", "tn_hvp_step", "tn_hvp_query", "tn_hvp_trim_memory",
           "tn_hvp_set_product_state", "tn_hvp_set_reference", "tn_mpo_tebd",
           "tn_hvp_set_cache_budget", "tn_hvp_environments_part", "tn_hvp_environments_finish",
           "tn_hvp_primal_region",
           "tn_hvp_destroy", "tn_hvp_last_error"]
TN_C128, TN_C64 = 0, 1
TN_CHECK_UNITARY, TN_CHECK_TANGENT = 1, 2


class TNError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("n_sites", C.c_int32), ("depth", C.c_int32), ("first_offset", C.c_int32), ("chi", C.c_int32),
                ("site_dim", C.c_int32), ("dtype", C.c_int32), ("max_batch", C.c_int32), ("device", C.c_int32),
                ("flags", C.c_uint32)]


def make_config(n, depth, chi, max_batch=1, first_offset=0, site_dim=4, dtype=0, device=0, flags=0) -> Config:
    return Config(n, depth, first_offset, chi, site_dim, dtype, max_batch, device, flags)


class Sizes(C.Structure):
    _fields_ = [("primal_bytes", C.c_size_t), ("workspace_bytes", C.c_size_t), ("per_direction_bytes", C.c_size_t)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2604_20384_b200.build` (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.tn_hvp_num_gates.argtypes = [i32, i32, i32]
        L.tn_hvp_num_gates.restype = i32
        L.tn_hvp_setup.argtypes = [C.POINTER(Config), C.POINTER(i32), vp, vp, C.c_size_t, vp, C.POINTER(vp)]
        L.tn_hvp_query.argtypes = [C.POINTER(Config), C.POINTER(i32), C.POINTER(Sizes)]
        L.tn_hvp_trim_memory.argtypes = [vp, vp]
        L.tn_hvp_set_product_state.argtypes = [vp, vp, vp]
        L.tn_hvp_set_reference.argtypes = [vp, vp, vp]
        L.tn_hvp_set_cache_budget.argtypes = [vp, C.c_size_t]
        L.tn_hvp_environments_part.argtypes = [vp, vp, i32, vp]
        L.tn_hvp_environments_finish.argtypes = [vp, vp, vp, vp, vp]
        L.tn_hvp_primal_region.argtypes = [vp, i32, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        L.tn_mpo_tebd.argtypes = [i32, i32, C.POINTER(i32), vp, i32, C.c_double, i32, C.POINTER(i32), vp,
                                  C.c_size_t, vp]
        L.tn_hvp_environments.argtypes = [vp, vp, vp, vp, vp]
        L.tn_hvp_apply.argtypes = [vp, i32, vp, vp, vp, vp]
        L.tn_hvp_gradient_T.argtypes = [vp, vp, vp]
        L.tn_hvp_cost.argtypes = [vp, vp, vp, vp]
        L.tn_hvp_primal_blob.argtypes = [vp, C.POINTER(vp), C.POINTER(C.c_size_t)]
        L.tn_hvp_primal_imported.argtypes = [vp, vp, vp]
        L.tn_riemannian_project.argtypes = [i32, i32, vp, vp, vp, vp]
        L.tn_zgemm.argtypes = [C.c_char, C.c_char, i32, i32, i32, C.POINTER(C.c_double), vp, i64, i64, vp, i64, i64,
                               C.POINTER(C.c_double), vp, i64, i64, i32, vp]
        L.tn_hvp_work.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.tn_hvp_split_stats.argtypes = [vp, C.POINTER(C.c_int64)]
        L.tn_hvp_split_stats.restype = C.c_int
        L.tn_retract.argtypes = [i32, vp, vp, C.c_double, vp, vp]
        L.tn_tangent_dot.argtypes = [i64, i32, vp, vp, vp, vp]
        L.tn_tangent_axpby.argtypes = [i64, C.POINTER(C.c_double), vp, C.POINTER(C.c_double), vp, vp]
        L.tn_hvp_primal_copy.argtypes = [vp, vp, C.c_size_t, i32, vp]
        L.tn_hvp_step.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, vp]
        L.tn_hvp_ti_environments.argtypes = [vp, vp, vp, vp, vp]
        L.tn_hvp_ti_apply.argtypes = [vp, i32, vp, vp, vp]
        L.tn_pauli_basis.argtypes = [i32, i64, i32, vp, vp, vp]
        L.tn_pauli_coords.argtypes = [i32, i32, vp, vp, vp, vp]
        L.tn_sym_eig.argtypes = [i32, vp, vp, vp, i32, vp]
        for name in ("tn_retract", "tn_tangent_dot", "tn_tangent_axpby", "tn_hvp_primal_copy", "tn_pauli_basis",
                     "tn_pauli_coords", "tn_sym_eig", "tn_hvp_ti_environments", "tn_hvp_ti_apply",
                     "tn_hvp_step", "tn_hvp_query", "tn_hvp_trim_memory", "tn_hvp_set_product_state",
                     "tn_hvp_set_reference", "tn_mpo_tebd", "tn_hvp_set_cache_budget",
                     "tn_hvp_environments_part", "tn_hvp_environments_finish", "tn_hvp_primal_region"):
            getattr(L, name).restype = C.c_int
        L.tn_hvp_launch_count.argtypes = []
        L.tn_hvp_launch_count.restype = C.c_int64
        L.tn_gemm_profile.argtypes = [i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.tn_gemm_profile.restype = C.c_int
        L.tn_hvp_destroy.argtypes = [vp]
        L.tn_hvp_destroy.restype = None
        L.tn_hvp_last_error.argtypes = [vp]
        L.tn_hvp_last_error.restype = C.c_char_p
        for name in ("tn_hvp_setup", "tn_hvp_environments", "tn_hvp_apply", "tn_hvp_gradient_T", "tn_hvp_cost",
                     "tn_hvp_primal_blob", "tn_hvp_primal_imported", "tn_riemannian_project", "tn_zgemm",
                     "tn_hvp_work"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def check(status, ctx=None):
    if status != TN_OK:
        msg = lib().tn_hvp_last_error(ctx)
        raise TNError(status, msg.decode() if msg else "")


def tn_hvp_num_gates(n, depth, first_offset=0):
    return lib().tn_hvp_num_gates(n, depth, first_offset)


def tn_hvp_query(cfg: Config, ref_bonds):
    """-> (primal_bytes, workspace_bytes, per_direction_bytes)."""
    arr = (C.c_int32 * len(ref_bonds))(*ref_bonds)
    out = Sizes()
    check(lib().tn_hvp_query(C.byref(cfg), arr, C.byref(out)))
    return out.primal_bytes, out.workspace_bytes, out.per_direction_bytes


def tn_hvp_setup(cfg: Config, ref_bonds, ref_mpo_ptr, stream, primal_ptr=0, primal_bytes=0):
    arr = (C.c_int32 * len(ref_bonds))(*ref_bonds)
    out = C.c_void_p()
    check(lib().tn_hvp_setup(C.byref(cfg), arr, C.c_void_p(ref_mpo_ptr), C.c_void_p(primal_ptr or None),
                             C.c_size_t(primal_bytes), C.c_void_p(stream), C.byref(out)))
    return out


def tn_hvp_trim_memory(ctx, stream):
    check(lib().tn_hvp_trim_memory(ctx, C.c_void_p(stream)), ctx)


def tn_hvp_set_product_state(ctx, psi_ptr, stream):
    check(lib().tn_hvp_set_product_state(ctx, C.c_void_p(psi_ptr), C.c_void_p(stream)), ctx)


def tn_hvp_set_reference(ctx, ref_ptr, stream):
    check(lib().tn_hvp_set_reference(ctx, C.c_void_p(ref_ptr), C.c_void_p(stream)), ctx)


def tn_hvp_environments(ctx, gates_ptr, scalars_ptr, grad_R_ptr, stream):
    check(lib().tn_hvp_environments(ctx, C.c_void_p(gates_ptr), C.c_void_p(scalars_ptr),
                                    C.c_void_p(grad_R_ptr), C.c_void_p(stream)), ctx)


def tn_hvp_apply(ctx, batch, dirs_ptr, hess_ptr, aux_ptr, stream):
    check(lib().tn_hvp_apply(ctx, batch, C.c_void_p(dirs_ptr), C.c_void_p(hess_ptr), C.c_void_p(aux_ptr),
                             C.c_void_p(stream)), ctx)


def tn_hvp_gradient_T(ctx, E_ptr, stream):
    check(lib().tn_hvp_gradient_T(ctx, C.c_void_p(E_ptr), C.c_void_p(stream)), ctx)


def tn_hvp_cost(ctx, gates_ptr, scalars_ptr, stream):
    check(lib().tn_hvp_cost(ctx, C.c_void_p(gates_ptr), C.c_void_p(scalars_ptr), C.c_void_p(stream)), ctx)


def tn_hvp_primal_blob(ctx):
    p, n = C.c_void_p(), C.c_size_t()
    check(lib().tn_hvp_primal_blob(ctx, C.byref(p), C.byref(n)), ctx)
    return p.value, n.value


def tn_hvp_primal_imported(ctx, gates_ptr, stream):
    check(lib().tn_hvp_primal_imported(ctx, C.c_void_p(gates_ptr), C.c_void_p(stream)), ctx)


def tn_riemannian_project(K, batch, gates_ptr, in_ptr, out_ptr, stream):
    check(lib().tn_riemannian_project(K, batch, C.c_void_p(gates_ptr), C.c_void_p(in_ptr), C.c_void_p(out_ptr),
                                      C.c_void_p(stream)))


def tn_zgemm(opa, opb, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, Cp, ldc, sC, batch, stream):
    a = (C.c_double * 2)(alpha.real, alpha.imag)
    b = (C.c_double * 2)(beta.real, beta.imag)
    check(lib().tn_zgemm(opa.encode(), opb.encode(), M, N, K, a, C.c_void_p(A), lda, sA, C.c_void_p(B), ldb, sB, b,
                         C.c_void_p(Cp), ldc, sC, batch, C.c_void_p(stream)))


def tn_hvp_work(ctx):
    a, b = C.c_double(), C.c_double()
    check(lib().tn_hvp_work(ctx, C.byref(a), C.byref(b)), ctx)
    return a.value, b.value


def tn_hvp_split_stats(ctx):
    out = (C.c_int64 * 6)()
    check(lib().tn_hvp_split_stats(ctx, out), ctx)
    return list(out)


def tn_retract(K, gates_ptr, xi_ptr, alpha, out_ptr, stream):
    check(lib().tn_retract(K, C.c_void_p(gates_ptr), C.c_void_p(xi_ptr), alpha, C.c_void_p(out_ptr),
                           C.c_void_p(stream)))


def tn_tangent_dot(n, batch, A_ptr, B_ptr, out_ptr, stream):
    check(lib().tn_tangent_dot(n, batch, C.c_void_p(A_ptr), C.c_void_p(B_ptr), C.c_void_p(out_ptr),
                               C.c_void_p(stream)))


def tn_tangent_axpby(n, a, x_ptr, b, y_ptr, stream):
    av = (C.c_double * 2)(complex(a).real, complex(a).imag)
    bv = (C.c_double * 2)(complex(b).real, complex(b).imag)
    check(lib().tn_tangent_axpby(n, av, C.c_void_p(x_ptr), bv, C.c_void_p(y_ptr), C.c_void_p(stream)))


def tn_hvp_primal_copy(ctx, buf_ptr, nbytes, into_ctx, stream):
    check(lib().tn_hvp_primal_copy(ctx, C.c_void_p(buf_ptr), nbytes, into_ctx, C.c_void_p(stream)), ctx)


def tn_hvp_launch_count():
    return lib().tn_hvp_launch_count()


def tn_gemm_profile(mode):
    a, b = C.c_double(), C.c_double()
    check(lib().tn_gemm_profile(mode, C.byref(a), C.byref(b)))
    return a.value, b.value


def tn_hvp_destroy(ctx):
    lib().tn_hvp_destroy(ctx)


def tn_pauli_basis(K, first, count, gates_ptr, out_ptr, stream):
    check(lib().tn_pauli_basis(K, first, count, C.c_void_p(gates_ptr), C.c_void_p(out_ptr), C.c_void_p(stream)))


def tn_pauli_coords(K, count, gates_ptr, X_ptr, out_ptr, stream):
    check(lib().tn_pauli_coords(K, count, C.c_void_p(gates_ptr), C.c_void_p(X_ptr), C.c_void_p(out_ptr),
                                C.c_void_p(stream)))


def tn_sym_eig(n, A_ptr, w_ptr, asym_ptr, vectors, stream):
    check(lib().tn_sym_eig(n, C.c_void_p(A_ptr), C.c_void_p(w_ptr), C.c_void_p(asym_ptr), int(vectors),
                           C.c_void_p(stream)))


def tn_hvp_ti_environments(ctx, g_ptr, scalars_ptr, grad_R_ptr, stream):
    check(lib().tn_hvp_ti_environments(ctx, C.c_void_p(g_ptr), C.c_void_p(scalars_ptr), C.c_void_p(grad_R_ptr),
                                       C.c_void_p(stream)), ctx)


def tn_hvp_ti_apply(ctx, batch, v_ptr, hess_ptr, stream):
    check(lib().tn_hvp_ti_apply(ctx, batch, C.c_void_p(v_ptr), C.c_void_p(hess_ptr), C.c_void_p(stream)), ctx)


def tn_hvp_step(ctx, gates_ptr, scalars_ptr, grad_R_ptr, batch, dirs_ptr, hess_ptr, aux_ptr, stream):
    check(lib().tn_hvp_step(ctx, C.c_void_p(gates_ptr), C.c_void_p(scalars_ptr), C.c_void_p(grad_R_ptr), batch,
                            C.c_void_p(dirs_ptr), C.c_void_p(hess_ptr), C.c_void_p(aux_ptr), C.c_void_p(stream)), ctx)


def tn_mpo_tebd(n, sites, gates_ptr, chi, tol, device, out_ptr, capacity, stream):
    """-> bonds (list of n+1)."""
    sarr = (C.c_int32 * max(len(sites), 1))(*sites)
    barr = (C.c_int32 * (n + 1))()
    check(lib().tn_mpo_tebd(n, len(sites), sarr, C.c_void_p(gates_ptr), chi, tol, device, barr,
                            C.c_void_p(out_ptr), C.c_size_t(capacity), C.c_void_p(stream)))
    return list(barr)


def tn_hvp_set_cache_budget(ctx, nbytes):
    check(lib().tn_hvp_set_cache_budget(ctx, C.c_size_t(int(nbytes))), ctx)


def tn_hvp_environments_part(ctx, gates_ptr, part, stream):
    check(lib().tn_hvp_environments_part(ctx, C.c_void_p(gates_ptr), part, C.c_void_p(stream)), ctx)


def tn_hvp_environments_finish(ctx, gates_ptr, scalars_ptr, grad_R_ptr, stream):
    check(lib().tn_hvp_environments_finish(ctx, C.c_void_p(gates_ptr), C.c_void_p(scalars_ptr),
                                           C.c_void_p(grad_R_ptr), C.c_void_p(stream)), ctx)


def tn_hvp_primal_region(ctx, part):
    """-> (byte offset, bytes) of side `part` (0 bottom, 1 top) inside the primal store."""
    o, b = C.c_size_t(), C.c_size_t()
    check(lib().tn_hvp_primal_region(ctx, part, C.byref(o), C.byref(b)), ctx)
    return o.value, b.value
