// extern "C" boundary (include/tn_hvp.h).  Argument checking, status codes,
// last-error text; the work itself lives in engine.cu / zgemm.cu / kernels.cu.
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tn_hvp.h"
#include "common.cuh"
#include "engine.cuh"
#include "kernels.cuh"

namespace {
thread_local std::string g_last_error;

tn_status fail(tn_hvp_ctx* ctx, tn_status st, const std::string& msg) {
  g_last_error = msg;
  if (ctx) tn::engine_set_error(ctx, msg);
  return st;
}

template <class F>
tn_status guarded(tn_hvp_ctx* ctx, F&& f) {
  try {
    f();
    return TN_OK;
  } catch (const std::invalid_argument& e) {
    return fail(ctx, TN_EINVAL, e.what());
  } catch (const std::bad_alloc& e) {
    return fail(ctx, TN_ENOMEM, e.what());
  } catch (const tn::NumericError& e) {
    return fail(ctx, TN_ENUMERIC, e.what());
  } catch (const tn::StateError& e) {
    return fail(ctx, TN_ESTATE, e.what());
  } catch (const tn::CudaError& e) {
    return fail(ctx, TN_ECUDA, e.what());
  } catch (const std::exception& e) {
    return fail(ctx, TN_ECUDA, e.what());
  }
}

bool valid_op(char c) { return c == 'N' || c == 'T' || c == 'C'; }
}  // namespace

extern "C" {

int32_t tn_hvp_num_gates(int32_t n, int32_t depth, int32_t off) {
  if (n < 2 || depth < 1 || (off != 0 && off != 1)) return -1;
  int32_t K = 0;
  for (int32_t ell = 1; ell <= depth; ++ell) {
    const int32_t o = (off + ell - 1) % 2;
    for (int32_t s = o; s + 1 < n; s += 2) ++K;
  }
  return K;
}

tn_status tn_zgemm(char opa, char opb, int32_t M, int32_t N, int32_t K, const double* alpha, const void* A,
                   int64_t lda, int64_t sA, const void* B, int64_t ldb, int64_t sB, const double* beta, void* C,
                   int64_t ldc, int64_t sC, int32_t batch, void* stream) {
  if (!valid_op(opa) || !valid_op(opb) || M < 0 || N < 0 || K < 0 || batch < 0 || !alpha || !beta)
    return fail(nullptr, TN_EINVAL, "tn_zgemm: bad op/size/scalar argument");
  if ((M && N && batch) && (!C || (K && (!A || !B)))) return fail(nullptr, TN_EINVAL, "tn_zgemm: null pointer");
  return guarded(nullptr, [&] {
    tn::zgemm((cudaStream_t)stream, opa, opb, M, N, K, make_double2(alpha[0], alpha[1]), (const tn::cplx*)A, lda,
              sA, (const tn::cplx*)B, ldb, sB, make_double2(beta[0], beta[1]), (tn::cplx*)C, ldc, sC, batch);
  });
}

tn_status tn_riemannian_project(int32_t K, int32_t batch, const void* gates, const void* in, void* out,
                                void* stream) {
  if (K < 0 || batch < 0) return fail(nullptr, TN_EINVAL, "tn_riemannian_project: negative size");
  if ((K && batch) && (!gates || !in || !out)) return fail(nullptr, TN_EINVAL, "tn_riemannian_project: null pointer");
  return guarded(nullptr, [&] {
    tn::project((cudaStream_t)stream, K, batch, (const tn::cplx*)gates, (const tn::cplx*)in, (tn::cplx*)out);
  });
}

namespace {
tn_status check_config(const tn_hvp_config* cfg, const int32_t* ref_bonds, const char* who) {
  const std::string w(who);
  if (cfg->n_sites < 2 || cfg->depth < 1 || (cfg->first_offset != 0 && cfg->first_offset != 1) || cfg->chi < 1 ||
      cfg->max_batch < 1 || cfg->device < 0)
    return fail(nullptr, TN_EINVAL, w + ": n>=2, depth>=1, offset in {0,1}, chi>=1, max_batch>=1, device>=0");
  if (cfg->site_dim != 4 && cfg->site_dim != 2)
    return fail(nullptr, TN_EINVAL, w + ": site_dim must be 4 (operator mode) or 2 (state mode)");
  if (cfg->dtype != TN_C128)
    return fail(nullptr, TN_EINVAL, w + ": only dtype TN_C128 is built (the complex64 mode is not implemented)");
  if (cfg->flags & ~(TN_CHECK_UNITARY | TN_CHECK_TANGENT))
    return fail(nullptr, TN_EINVAL, w + ": unknown flag bits");
  if (ref_bonds[0] != 1 || ref_bonds[cfg->n_sites] != 1)
    return fail(nullptr, TN_EINVAL, w + ": boundary bonds must be 1");
  for (int s = 0; s < cfg->n_sites; ++s) {
    const int64_t bl = ref_bonds[s], br = ref_bonds[s + 1];
    const int64_t P = cfg->site_dim;
    if (bl < 1 || br < 1 || br > P * bl || bl > P * br)
      return fail(nullptr, TN_EINVAL, w + ": reference bonds must satisfy 1 <= b_{s+1} <= site_dim b_s and vice versa");
  }
  return TN_OK;
}
}  // namespace

tn_status tn_hvp_query(const tn_hvp_config* cfg, const int32_t* ref_bonds, tn_hvp_sizes* out) {
  if (!cfg || !ref_bonds || !out) return fail(nullptr, TN_EINVAL, "tn_hvp_query: null argument");
  if (tn_status st = check_config(cfg, ref_bonds, "tn_hvp_query")) return st;
  return guarded(nullptr, [&] {
    tn::engine_query(*cfg, ref_bonds, &out->primal_bytes, &out->workspace_bytes, &out->per_direction_bytes);
  });
}

tn_status tn_hvp_setup(const tn_hvp_config* cfg, const int32_t* ref_bonds, const void* ref_mpo, void* primal_buf,
                       size_t primal_bytes_avail, void* stream, tn_hvp_ctx** out) {
  if (!cfg || !ref_bonds || !ref_mpo || !out) return fail(nullptr, TN_EINVAL, "tn_hvp_setup: null argument");
  if (tn_status st = check_config(cfg, ref_bonds, "tn_hvp_setup")) return st;
  *out = nullptr;
  return guarded(nullptr, [&] {
    *out = tn::engine_create(*cfg, ref_bonds, ref_mpo, primal_buf, primal_bytes_avail, (cudaStream_t)stream);
  });
}

tn_status tn_hvp_set_product_state(tn_hvp_ctx* ctx, const void* psi, void* stream) {
  if (!ctx || !psi) return fail(ctx, TN_EINVAL, "tn_hvp_set_product_state: null argument");
  return guarded(ctx, [&] { tn::engine_set_product_state(ctx, (const tn::cplx*)psi, (cudaStream_t)stream); });
}

tn_status tn_hvp_set_reference(tn_hvp_ctx* ctx, const void* ref, void* stream) {
  if (!ctx || !ref) return fail(ctx, TN_EINVAL, "tn_hvp_set_reference: null argument");
  return guarded(ctx, [&] { tn::engine_set_reference(ctx, (const tn::cplx*)ref, (cudaStream_t)stream); });
}

tn_status tn_mpo_tebd(int32_t n, int32_t ngates, const int32_t* sites, const void* gates, int32_t chi, double tol,
                      int32_t device, int32_t* bonds_out, void* out, size_t cap, void* stream) {
  if (n < 2 || ngates < 0 || chi < 1 || device < 0 || !bonds_out || !out || (ngates && (!sites || !gates)) ||
      !(tol >= 0.0))
    return fail(nullptr, TN_EINVAL, "tn_mpo_tebd: bad argument");
  return guarded(nullptr, [&] {
    TN_CUDA(cudaSetDevice(device));
    tn::engine_tebd(n, ngates, sites, (const tn::cplx*)gates, chi, tol, device, bonds_out, (tn::cplx*)out, cap,
                    (cudaStream_t)stream);
  });
}

tn_status tn_hvp_set_cache_budget(tn_hvp_ctx* ctx, size_t bytes) {
  if (!ctx) return fail(nullptr, TN_EINVAL, "tn_hvp_set_cache_budget: null context");
  return guarded(ctx, [&] { tn::engine_set_cache_budget(ctx, bytes); });
}

tn_status tn_hvp_environments_part(tn_hvp_ctx* ctx, const void* gates, int32_t part, void* stream) {
  if (!ctx || !gates || (part != 0 && part != 1)) return fail(ctx, TN_EINVAL, "tn_hvp_environments_part: bad argument");
  return guarded(ctx, [&] { tn::engine_environments_part(ctx, (const tn::cplx*)gates, part, (cudaStream_t)stream); });
}

tn_status tn_hvp_environments_finish(tn_hvp_ctx* ctx, const void* gates, void* scalars_out, void* grad_R_out,
                                     void* stream) {
  if (!ctx || !gates || !scalars_out) return fail(ctx, TN_EINVAL, "tn_hvp_environments_finish: null argument");
  return guarded(ctx, [&] {
    tn::engine_environments_finish(ctx, (const tn::cplx*)gates, (double*)scalars_out, (tn::cplx*)grad_R_out,
                                   (cudaStream_t)stream);
  });
}

tn_status tn_hvp_primal_region(tn_hvp_ctx* ctx, int32_t part, size_t* offset, size_t* bytes) {
  if (!ctx || !offset || !bytes || (part != 0 && part != 1))
    return fail(ctx, TN_EINVAL, "tn_hvp_primal_region: bad argument");
  return guarded(ctx, [&] { tn::engine_primal_region(ctx, part, offset, bytes); });
}

tn_status tn_hvp_trim_memory(tn_hvp_ctx* ctx, void* stream) {
  if (!ctx) return fail(nullptr, TN_EINVAL, "tn_hvp_trim_memory: null context");
  return guarded(ctx, [&] { tn::engine_trim_memory(ctx, (cudaStream_t)stream); });
}

tn_status tn_hvp_environments(tn_hvp_ctx* ctx, const void* gates, void* scalars_out, void* grad_R_out, void* stream) {
  if (!ctx || !gates || !scalars_out) return fail(ctx, TN_EINVAL, "tn_hvp_environments: null argument");
  return guarded(ctx, [&] {
    tn::engine_environments(ctx, (const tn::cplx*)gates, (double*)scalars_out, (tn::cplx*)grad_R_out,
                            (cudaStream_t)stream);
  });
}

tn_status tn_hvp_apply(tn_hvp_ctx* ctx, int32_t batch, const void* dirs, void* hess_R_out, void* aux_out,
                       void* stream) {
  if (!ctx || batch < 0 || (batch && (!dirs || !hess_R_out)))
    return fail(ctx, TN_EINVAL, "tn_hvp_apply: null argument or negative batch");
  return guarded(ctx, [&] {
    tn::engine_apply(ctx, batch, (const tn::cplx*)dirs, (tn::cplx*)hess_R_out, (tn::cplx*)aux_out,
                     (cudaStream_t)stream);
  });
}

tn_status tn_hvp_ti_environments(tn_hvp_ctx* ctx, const void* layer_gates, void* scalars_out, void* grad_R_out,
                                 void* stream) {
  if (!ctx || !layer_gates || !scalars_out || !grad_R_out)
    return fail(ctx, TN_EINVAL, "tn_hvp_ti_environments: null argument");
  return guarded(ctx, [&] {
    tn::engine_ti_environments(ctx, (const tn::cplx*)layer_gates, (double*)scalars_out, (tn::cplx*)grad_R_out,
                               (cudaStream_t)stream);
  });
}

tn_status tn_hvp_ti_apply(tn_hvp_ctx* ctx, int32_t batch, const void* layer_dirs, void* hess_R_out, void* stream) {
  if (!ctx || batch < 0 || (batch && (!layer_dirs || !hess_R_out)))
    return fail(ctx, TN_EINVAL, "tn_hvp_ti_apply: null argument or negative batch");
  return guarded(ctx, [&] {
    tn::engine_ti_apply(ctx, batch, (const tn::cplx*)layer_dirs, (tn::cplx*)hess_R_out, (cudaStream_t)stream);
  });
}

tn_status tn_hvp_step(tn_hvp_ctx* ctx, const void* gates, void* scalars_out, void* grad_R_out, int32_t batch,
                      const void* dirs, void* hess_R_out, void* aux_out, void* stream) {
  if (!ctx || !gates || !scalars_out || !grad_R_out || batch < 0 || (batch && (!dirs || !hess_R_out)))
    return fail(ctx, TN_EINVAL, "tn_hvp_step: null argument or negative batch");
  return guarded(ctx, [&] {
    tn::engine_step(ctx, (const tn::cplx*)gates, (double*)scalars_out, (tn::cplx*)grad_R_out, batch,
                    (const tn::cplx*)dirs, (tn::cplx*)hess_R_out, (tn::cplx*)aux_out, (cudaStream_t)stream);
  });
}

tn_status tn_hvp_gradient_T(tn_hvp_ctx* ctx, void* E_out, void* stream) {
  if (!ctx || !E_out) return fail(ctx, TN_EINVAL, "tn_hvp_gradient_T: null argument");
  return guarded(ctx, [&] { tn::engine_gradient_T(ctx, (tn::cplx*)E_out, (cudaStream_t)stream); });
}

tn_status tn_hvp_cost(tn_hvp_ctx* ctx, const void* gates, void* scalars_out, void* stream) {
  if (!ctx || !gates || !scalars_out) return fail(ctx, TN_EINVAL, "tn_hvp_cost: null argument");
  return guarded(ctx, [&] {
    tn::engine_cost(ctx, (const tn::cplx*)gates, (double*)scalars_out, (cudaStream_t)stream);
  });
}

tn_status tn_hvp_primal_blob(tn_hvp_ctx* ctx, void** ptr, size_t* bytes) {
  if (!ctx || !ptr || !bytes) return fail(ctx, TN_EINVAL, "tn_hvp_primal_blob: null argument");
  return guarded(ctx, [&] { tn::engine_primal_blob(ctx, ptr, bytes); });
}

tn_status tn_hvp_primal_imported(tn_hvp_ctx* ctx, const void* gates, void* stream) {
  if (!ctx || !gates) return fail(ctx, TN_EINVAL, "tn_hvp_primal_imported: null argument");
  return guarded(ctx, [&] { tn::engine_primal_imported(ctx, (const tn::cplx*)gates, (cudaStream_t)stream); });
}

tn_status tn_hvp_work(tn_hvp_ctx* ctx, double* per_dir, double* primal) {
  if (!ctx || !per_dir || !primal) return fail(ctx, TN_EINVAL, "tn_hvp_work: null argument");
  return guarded(ctx, [&] { tn::engine_work(ctx, per_dir, primal); });
}

tn_status tn_hvp_split_stats(tn_hvp_ctx* ctx, int64_t* out6) {
  if (!ctx || !out6) return fail(ctx, TN_EINVAL, "tn_hvp_split_stats: null argument");
  return guarded(ctx, [&] { tn::engine_split_stats(ctx, out6); });
}

tn_status tn_retract(int32_t K, const void* gates, const void* xi, double alpha, void* out, void* stream) {
  if (K < 0 || (K && (!gates || !xi || !out))) return fail(nullptr, TN_EINVAL, "tn_retract: bad argument");
  return guarded(nullptr, [&] {
    if (!K) return;
    int* st = (int*)tn::dalloc(sizeof(int), (cudaStream_t)stream);
    TN_CUDA(cudaMemsetAsync(st, 0, sizeof(int), (cudaStream_t)stream));
    tn::retract((cudaStream_t)stream, K, (const tn::cplx*)gates, (const tn::cplx*)xi, alpha, (tn::cplx*)out, st);
    int h = 0;
    TN_CUDA(cudaMemcpyAsync(&h, st, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    tn::dfree(st, (cudaStream_t)stream);
    TN_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (h) throw tn::NumericError("tn_retract: singular iterate");
  });
}

tn_status tn_tangent_dot(int64_t n, int32_t batch, const void* A, const void* B, void* out, void* stream) {
  if (n < 0 || batch < 0 || (n && batch && (!A || !B || !out))) return fail(nullptr, TN_EINVAL, "tn_tangent_dot: bad argument");
  return guarded(nullptr, [&] {
    tn::tangent_dot((cudaStream_t)stream, n, batch, (const tn::cplx*)A, (const tn::cplx*)B, (double*)out);
  });
}

tn_status tn_tangent_axpby(int64_t n, const double* a, const void* x, const double* b, void* y, void* stream) {
  if (n < 0 || !a || !b || (n && (!x || !y))) return fail(nullptr, TN_EINVAL, "tn_tangent_axpby: bad argument");
  return guarded(nullptr, [&] {
    tn::axpby((cudaStream_t)stream, (tn::cplx*)y, (const tn::cplx*)x, make_double2(a[0], a[1]),
              make_double2(b[0], b[1]), n);
  });
}

tn_status tn_pauli_basis(int32_t K, int64_t first, int32_t count, const void* gates, void* out, void* stream) {
  if (K < 0 || count < 0 || first < 0 || first + count > (int64_t)16 * K)
    return fail(nullptr, TN_EINVAL, "tn_pauli_basis: need 0 <= first, 0 <= count, first + count <= 16 K");
  if (K && count && (!gates || !out)) return fail(nullptr, TN_EINVAL, "tn_pauli_basis: null pointer");
  return guarded(nullptr, [&] {
    tn::pauli_basis((cudaStream_t)stream, K, first, count, (const tn::cplx*)gates, (tn::cplx*)out);
  });
}

tn_status tn_pauli_coords(int32_t K, int32_t count, const void* gates, const void* X, void* out, void* stream) {
  if (K < 0 || count < 0) return fail(nullptr, TN_EINVAL, "tn_pauli_coords: negative size");
  if (K && count && (!gates || !X || !out)) return fail(nullptr, TN_EINVAL, "tn_pauli_coords: null pointer");
  return guarded(nullptr, [&] {
    tn::pauli_coords((cudaStream_t)stream, K, count, (const tn::cplx*)gates, (const tn::cplx*)X, (double*)out);
  });
}

tn_status tn_sym_eig(int32_t n, void* A, void* w, void* asym, int32_t vectors, void* stream) {
  if (n < 0 || (vectors != 0 && vectors != 1)) return fail(nullptr, TN_EINVAL, "tn_sym_eig: n >= 0, vectors in {0,1}");
  if (n && (!A || !w || !asym)) return fail(nullptr, TN_EINVAL, "tn_sym_eig: null pointer");
  return guarded(nullptr, [&] {
    tn::sym_eig((cudaStream_t)stream, n, (double*)A, (double*)w, (double*)asym, vectors == 1);
  });
}

tn_status tn_hvp_primal_copy(tn_hvp_ctx* ctx, void* buf, size_t bytes, int32_t into_ctx, void* stream) {
  if (!ctx || !buf || (into_ctx != 0 && into_ctx != 1)) return fail(ctx, TN_EINVAL, "tn_hvp_primal_copy: bad argument");
  return guarded(ctx, [&] { tn::engine_primal_copy(ctx, buf, bytes, into_ctx, (cudaStream_t)stream); });
}

int64_t tn_hvp_launch_count(void) { return tn::launch_count(); }

tn_status tn_gemm_profile(int32_t mode, double* ms, double* cmac) {
  if (mode != 0 && mode != 1) return fail(nullptr, TN_EINVAL, "tn_gemm_profile: mode must be 0 or 1");
  return guarded(nullptr, [&] {
    if (mode == 1) {
      tn::gemm_profile_begin();
    } else {
      double a = 0, b = 0;
      tn::gemm_profile_end(&a, &b);
      if (ms) *ms = a;
      if (cmac) *cmac = b;
    }
  });
}

void tn_hvp_destroy(tn_hvp_ctx* ctx) {
  if (ctx) tn::engine_destroy(ctx);
}

const char* tn_hvp_last_error(const tn_hvp_ctx* ctx) {
  if (ctx) return tn::engine_error(ctx);
  return g_last_error.c_str();
}

}  // extern "C"
