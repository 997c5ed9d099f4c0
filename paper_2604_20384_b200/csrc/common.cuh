// Shared device/host helpers of the sm_100a HVP library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace tn {

using cplx = double2;  // interleaved complex128 (re, im)

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define TN_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      throw ::tn::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " @" +       \
                            __FILE__ + ":" + std::to_string(__LINE__));                     \
  } while (0)

__host__ __device__ inline cplx cmul(cplx a, cplx b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ inline cplx cmulc(cplx a, cplx b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ inline cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ inline cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ inline cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
__host__ __device__ inline cplx cconj(cplx a) { return make_double2(a.x, -a.y); }

// Kernel-launch counter of this library (all wrappers bump it) and the
// optional per-launch GEMM timing used by bench.py's roofline.
void count_launch(int64_t n = 1);
int64_t launch_count();
void gemm_profile_begin();                      // enable + reset (host side)
void gemm_profile_end(double* ms, double* cmac);  // sync, disable, read totals
bool gemm_profile_active();

// Library-private stream-ordered device memory (zgemm.cu): a cudaMemPool per
// device owned by this library (the device's default pool is left untouched).
// pool_trim returns the pool's unused blocks to the device.
void* dalloc(size_t bytes, cudaStream_t st);
void dfree(void* p, cudaStream_t st);
void pool_trim(int device);

// Batched row-major complex GEMM on DMMA (zgemm.cu).
// C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b]; op(A): M x K, op(B): K x N.
// opa/opb in {'N','T','C'}; strides in elements, 0 = operand shared.
// dscale (nullable, DEVICE): alpha and beta are multiplied by *dscale in the
// epilogue (a scalar known only on the device, e.g. a frozen truncation factor).
void zgemm(cudaStream_t st, char opa, char opb, int M, int N, int K, cplx alpha, const cplx* A, int64_t lda,
           int64_t sA, const cplx* B, int64_t ldb, int64_t sB, cplx beta, cplx* C, int64_t ldc, int64_t sC,
           int batch, const double* dscale = nullptr);

}  // namespace tn
