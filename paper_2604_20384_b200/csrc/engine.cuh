// Engine entry points used by the C ABI (abi.cu).  Not part of the public ABI.
#pragma once
#include <stdexcept>
#include <string>

#include "../../include/tn_hvp.h"
#include "common.cuh"

namespace tn {
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

tn_hvp_ctx* engine_create(const tn_hvp_config& cfg, const int32_t* ref_bonds, const void* ref_mpo, void* primal_buf,
                          size_t primal_bytes, cudaStream_t st);
void engine_environments(tn_hvp_ctx* ctx, const cplx* gates, double* scalars, cplx* grad_R, cudaStream_t st);
void engine_apply(tn_hvp_ctx* ctx, int batch, const cplx* dirs, cplx* hess_R, cplx* aux, cudaStream_t st);
void engine_step(tn_hvp_ctx* ctx, const cplx* gates, double* scalars, cplx* grad_R, int batch, const cplx* dirs,
                 cplx* hess_R, cplx* aux, cudaStream_t st);
void engine_gradient_T(tn_hvp_ctx* ctx, cplx* E, cudaStream_t st);
void engine_ti_environments(tn_hvp_ctx* ctx, const cplx* g, double* scalars, cplx* grad_R, cudaStream_t st);
void engine_ti_apply(tn_hvp_ctx* ctx, int batch, const cplx* v, cplx* hess_R, cudaStream_t st);
void engine_cost(tn_hvp_ctx* ctx, const cplx* gates, double* scalars, cudaStream_t st);
void engine_primal_blob(tn_hvp_ctx* ctx, void** ptr, size_t* bytes);
void engine_primal_imported(tn_hvp_ctx* ctx, const cplx* gates, cudaStream_t st);
void engine_primal_copy(tn_hvp_ctx* ctx, void* buf, size_t bytes, int into_ctx, cudaStream_t st);
void engine_trim_memory(tn_hvp_ctx* ctx, cudaStream_t st);
void engine_set_cache_budget(tn_hvp_ctx* ctx, size_t bytes);
void engine_environments_part(tn_hvp_ctx* ctx, const cplx* gates, int part, cudaStream_t st);
void engine_environments_finish(tn_hvp_ctx* ctx, const cplx* gates, double* scalars, cplx* grad_R, cudaStream_t st);
void engine_primal_region(tn_hvp_ctx* ctx, int part, size_t* offset, size_t* bytes);
void engine_tebd(int n, int ngates, const int32_t* sites, const cplx* gates, int chi, double tol, int device,
                 int32_t* bonds_out, cplx* out, size_t cap, cudaStream_t st);
void engine_set_product_state(tn_hvp_ctx* ctx, const cplx* psi, cudaStream_t st);
void engine_set_reference(tn_hvp_ctx* ctx, const cplx* ref, cudaStream_t st);
void engine_work(tn_hvp_ctx* ctx, double* per_dir, double* primal);
void engine_split_stats(tn_hvp_ctx* ctx, int64_t* out6);
void engine_query(const tn_hvp_config& cfg, const int32_t* ref_bonds, size_t* primal_bytes, size_t* work_bytes,
                  size_t* per_dir_bytes);
void engine_destroy(tn_hvp_ctx* ctx);
void engine_set_error(tn_hvp_ctx* ctx, const std::string& msg);
const char* engine_error(const tn_hvp_ctx* ctx);
}  // namespace tn
