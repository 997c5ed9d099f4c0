// N3: the Riemannian Hessian in the Pauli tangent basis
// (App. "Spectral analysis").
//
//  * pauli_basis: B_{16k+4a+b} = (0, .., i G_k (P_a (x) P_b)/2, .., 0)
//    (PAPER.md:1179), a window [first, first+count) of the 16K vectors.
//  * pauli_coords: c_i(X) = <B_i, X> = Re Tr(B_i^dag X_k) = 1/2 Im Tr(P G_k^dag X_k)
//    for every i (with an orthonormal basis the HVP of
//    B_j is column j of H_R).
//  * sym_eig: eigenvalues of the symmetric part of the assembled matrix
//    (reading X19), cuSOLVER syevd.
#include <cusolverDn.h>

#include <string>

#include "kernels.cuh"

namespace tn {
namespace {

// Pauli P_a[r][c] (a = I, X, Y, Z)
__device__ __forceinline__ cplx pauli(int a, int r, int c) {
  switch (a) {
    case 0: return make_double2(r == c ? 1.0 : 0.0, 0.0);
    case 1: return make_double2(r != c ? 1.0 : 0.0, 0.0);
    case 2: return r == c ? make_double2(0.0, 0.0) : make_double2(0.0, r == 0 ? -1.0 : 1.0);
    default: return make_double2(r == c ? (r == 0 ? 1.0 : -1.0) : 0.0, 0.0);
  }
}
// (P_a (x) P_b)[m][c], 4x4 index 2 q_i + q_{i+1} (X6)
__device__ __forceinline__ cplx pauli_pair(int p, int m, int c) {
  return cmul(pauli(p >> 2, m >> 1, c >> 1), pauli(p & 3, m & 1, c & 1));
}

// out[j][k][r][c], one thread per complex element
__global__ void pauli_basis_kernel(int K, int64_t first, int count, const cplx* __restrict__ G,
                                   cplx* __restrict__ out) {
  const int64_t total = (int64_t)count * K * 16;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(idx & 15);
    const int64_t jk = idx >> 4;
    const int k = (int)(jk % K);
    const int64_t i = first + jk / K;
    cplx v = make_double2(0.0, 0.0);
    if (i / 16 == k) {
      const int p = (int)(i & 15), r = e >> 2, c = e & 3;
      cplx acc = make_double2(0.0, 0.0);
      for (int m = 0; m < 4; ++m) acc = cadd(acc, cmul(G[(int64_t)k * 16 + r * 4 + m], pauli_pair(p, m, c)));
      v = make_double2(-0.5 * acc.y, 0.5 * acc.x);  // i/2 * acc
    }
    out[idx] = v;
  }
}

// out[j][16k + p] = 1/2 Im sum_{m,c,r} P[m][c] conj(G_k[r][c]) X_jk[r][m]
__global__ void pauli_coords_kernel(int K, int count, const cplx* __restrict__ G, const cplx* __restrict__ X,
                                    double* __restrict__ out) {
  const int64_t total = (int64_t)count * K * 16;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(idx & 15);
    const int64_t jk = idx >> 4;
    const int k = (int)(jk % K);
    const cplx* g = G + (int64_t)k * 16;
    const cplx* x = X + jk * 16;
    cplx tr = make_double2(0.0, 0.0);
    for (int m = 0; m < 4; ++m)
      for (int c = 0; c < 4; ++c) {
        const cplx pmc = pauli_pair(p, m, c);
        if (pmc.x == 0.0 && pmc.y == 0.0) continue;
        cplx y = make_double2(0.0, 0.0);  // (G^dag X)[c][m]
        for (int r = 0; r < 4; ++r) y = cadd(y, cmulc(g[r * 4 + c], x[r * 4 + m]));
        tr = cadd(tr, cmul(pmc, y));
      }
    out[idx] = 0.5 * tr.y;
  }
}

// part[blk] = (sum (A_ij - A_ji)^2, sum A_ij^2) over this block's entries; then A <- (A + A^T)/2
__global__ void asym_norms_kernel(int n, const double* __restrict__ A, double* __restrict__ part) {
  double d = 0, a = 0;
  const int64_t total = (int64_t)n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    const double x = A[idx], t = A[(int64_t)j * n + i];
    d += (x - t) * (x - t);
    a += x * x;
  }
  __shared__ double rd[32], ra[32];
  for (int off = 16; off > 0; off >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, off);
    a += __shfl_xor_sync(0xffffffffu, a, off);
  }
  if ((threadIdx.x & 31) == 0) {
    rd[threadIdx.x >> 5] = d;
    ra[threadIdx.x >> 5] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double td = 0, ta = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      td += rd[w];
      ta += ra[w];
    }
    part[2 * blockIdx.x] = td;
    part[2 * blockIdx.x + 1] = ta;
  }
}

__global__ void asym_finish_kernel(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double d = 0, a = 0;
    for (int b = 0; b < nblk; ++b) {
      d += part[2 * b];
      a += part[2 * b + 1];
    }
    out[0] = sqrt(d);
    out[1] = sqrt(a);
  }
}

// upper-triangle threads write both (i,j) and (j,i)
__global__ void symmetrize_kernel(int n, double* __restrict__ A) {
  const int64_t total = (int64_t)n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    if (j <= i) continue;
    const double s = 0.5 * (A[idx] + A[(int64_t)j * n + i]);
    A[idx] = s;
    A[(int64_t)j * n + i] = s;
  }
}

int grid_for(int64_t total, int threads) {
  const int64_t g = (total + threads - 1) / threads;
  return (int)std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 16);
}

}  // namespace

void pauli_basis(cudaStream_t st, int K, int64_t first, int count, const cplx* G, cplx* out) {
  if ((int64_t)count * K == 0) return;
  pauli_basis_kernel<<<grid_for((int64_t)count * K * 16, 256), 256, 0, st>>>(K, first, count, G, out);
  TN_CUDA(cudaGetLastError());
  count_launch();
}

void pauli_coords(cudaStream_t st, int K, int count, const cplx* G, const cplx* X, double* out) {
  if ((int64_t)count * K == 0) return;
  pauli_coords_kernel<<<grid_for((int64_t)count * K * 16, 256), 256, 0, st>>>(K, count, G, X, out);
  TN_CUDA(cudaGetLastError());
  count_launch();
}

void sym_eig(cudaStream_t st, int n, double* A, double* w, double* asym, bool vectors) {
  if (n == 0) return;
  const int64_t total = (int64_t)n * n;
  const int nblk = std::min(grid_for(total, 256), 1024);
  double* part = nullptr;
  part = (double*)dalloc(sizeof(double) * 2 * nblk, st);
  asym_norms_kernel<<<nblk, 256, 0, st>>>(n, A, part);
  TN_CUDA(cudaGetLastError());
  asym_finish_kernel<<<1, 32, 0, st>>>(part, nblk, asym);
  TN_CUDA(cudaGetLastError());
  symmetrize_kernel<<<grid_for(total, 256), 256, 0, st>>>(n, A);
  TN_CUDA(cudaGetLastError());
  count_launch(3);
  dfree(part, st);
  cusolverDnHandle_t h = nullptr;
  auto chk = [](cusolverStatus_t s, const char* what) {
    if (s != CUSOLVER_STATUS_SUCCESS) throw CudaError(std::string(what) + ": cuSOLVER status " + std::to_string((int)s));
  };
  chk(cusolverDnCreate(&h), "cusolverDnCreate");
  try {
    chk(cusolverDnSetStream(h, st), "cusolverDnSetStream");
    const cusolverEigMode_t jobz = vectors ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
    int lwork = 0;
    chk(cusolverDnDsyevd_bufferSize(h, jobz, CUBLAS_FILL_MODE_LOWER, n, A, n, w, &lwork), "Dsyevd_bufferSize");
    double* work = nullptr;
    int* info = nullptr;
    work = (double*)dalloc(sizeof(double) * std::max(lwork, 1), st);
    info = (int*)dalloc(sizeof(int), st);
    chk(cusolverDnDsyevd(h, jobz, CUBLAS_FILL_MODE_LOWER, n, A, n, w, work, lwork, info), "Dsyevd");
    int hinfo = 0;
    TN_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    dfree(work, st);
    dfree(info, st);
    TN_CUDA(cudaStreamSynchronize(st));
    if (hinfo != 0) throw NumericError("tn_sym_eig: syevd info " + std::to_string(hinfo));
  } catch (...) {
    cusolverDnDestroy(h);
    throw;
  }
  cusolverDnDestroy(h);
}

}  // namespace tn
