// cuSOLVER SVD variants on an n x n complex128 matrix: time + accuracy.
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cuComplex.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cstring>

#define CK(x) do { auto e = (x); if ((int)e != 0) { printf("{\"error\": \"%s -> %d line %d\"}\n", #x, (int)e, __LINE__); exit(1);} } while (0)

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 1024;
  cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
  std::vector<cuDoubleComplex> A(n * (size_t)n);
  srand(1);
  for (auto& a : A) a = make_cuDoubleComplex(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
  // give it a decaying spectrum: scale columns
  for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) { double f = exp(-8.0 * j / n); A[i + (size_t)j * n].x *= f; A[i + (size_t)j * n].y *= f; }
  cuDoubleComplex *dA, *dW, *dU, *dV; double* dS; int* info;
  size_t bytes = sizeof(cuDoubleComplex) * n * (size_t)n;
  CK(cudaMalloc(&dA, bytes)); CK(cudaMalloc(&dW, bytes)); CK(cudaMalloc(&dU, bytes)); CK(cudaMalloc(&dV, bytes));
  CK(cudaMalloc(&dS, sizeof(double) * n)); CK(cudaMalloc(&info, sizeof(int)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  printf("{\"n\": %d", n);
  // gesvdj
  {
    gesvdjInfo_t p; CK(cusolverDnCreateGesvdjInfo(&p)); CK(cusolverDnXgesvdjSetTolerance(p, 1e-15)); CK(cusolverDnXgesvdjSetMaxSweeps(p, 100));
    int lw; CK(cusolverDnZgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, dA, n, dS, dU, n, dV, n, &lw, p));
    cuDoubleComplex* work; CK(cudaMalloc(&work, sizeof(cuDoubleComplex) * lw));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemcpy(dA, A.data(), bytes, cudaMemcpyHostToDevice));
      cudaEventRecord(e0);
      CK(cusolverDnZgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, dA, n, dS, dU, n, dV, n, work, lw, info, p));
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double res; int sw; CK(cusolverDnXgesvdjGetResidual(h, p, &res)); CK(cusolverDnXgesvdjGetSweeps(h, p, &sw));
    printf(", \"gesvdj_ms\": %.2f, \"gesvdj_sweeps\": %d, \"gesvdj_residual\": %.3e", ms, sw, res);
    cudaFree(work);
  }
  // gesvd (QR iteration), 64-bit API
  {
    cusolverDnParams_t prm; CK(cusolverDnCreateParams(&prm));
    size_t dws, hws;
    CK(cusolverDnXgesvd_bufferSize(h, prm, 'S', 'S', n, n, CUDA_C_64F, dA, n, CUDA_R_64F, dS, CUDA_C_64F, dU, n, CUDA_C_64F, dV, n, CUDA_C_64F, &dws, &hws));
    void* dw; CK(cudaMalloc(&dw, dws)); std::vector<char> hw(hws + 1);
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemcpy(dA, A.data(), bytes, cudaMemcpyHostToDevice));
      cudaEventRecord(e0);
      CK(cusolverDnXgesvd(h, prm, 'S', 'S', n, n, CUDA_C_64F, dA, n, CUDA_R_64F, dS, CUDA_C_64F, dU, n, CUDA_C_64F, dV, n, CUDA_C_64F, dw, dws, hw.data(), hws, info));
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"xgesvd_ms\": %.2f", ms);
    cudaFree(dw);
  }
  // gesvdp (polar decomposition)
  {
    cusolverDnParams_t prm; CK(cusolverDnCreateParams(&prm));
    size_t dws, hws;
    CK(cusolverDnXgesvdp_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, CUDA_C_64F, dA, n, CUDA_R_64F, dS, CUDA_C_64F, dU, n, CUDA_C_64F, dV, n, CUDA_C_64F, &dws, &hws));
    void* dw; CK(cudaMalloc(&dw, dws)); std::vector<char> hw(hws + 1);
    double herr;
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemcpy(dA, A.data(), bytes, cudaMemcpyHostToDevice));
      cudaEventRecord(e0);
      CK(cusolverDnXgesvdp(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, CUDA_C_64F, dA, n, CUDA_R_64F, dS, CUDA_C_64F, dU, n, CUDA_C_64F, dV, n, CUDA_C_64F, dw, dws, hw.data(), hws, info, &herr));
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"xgesvdp_ms\": %.2f, \"xgesvdp_err\": %.3e", ms, herr);
    cudaFree(dw);
  }
  // heevd on the Gram matrix (speed reference only)
  {
    int lw; CK(cusolverDnZheevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dS, &lw));
    cuDoubleComplex* work; CK(cudaMalloc(&work, sizeof(cuDoubleComplex) * lw));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemcpy(dA, A.data(), bytes, cudaMemcpyHostToDevice));
      cudaEventRecord(e0);
      CK(cusolverDnZheevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dS, work, lw, info));
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"heevd_ms\": %.2f", ms);
  }
  // geqrf + ungqr
  {
    int lw, lw2; cuDoubleComplex* tau; CK(cudaMalloc(&tau, sizeof(cuDoubleComplex) * n));
    CK(cusolverDnZgeqrf_bufferSize(h, n, n / 4, dA, n, &lw));
    CK(cusolverDnZungqr_bufferSize(h, n, n / 4, n / 4, dA, n, tau, &lw2));
    cuDoubleComplex* work; CK(cudaMalloc(&work, sizeof(cuDoubleComplex) * (lw > lw2 ? lw : lw2)));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemcpy(dA, A.data(), bytes / 4, cudaMemcpyHostToDevice));
      cudaEventRecord(e0);
      CK(cusolverDnZgeqrf(h, n, n / 4, dA, n, tau, work, lw, info));
      CK(cusolverDnZungqr(h, n, n / 4, n / 4, dA, n, tau, work, lw2, info));
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"qr_%dx%d_ms\": %.2f", n, n / 4, ms);
  }
  printf("}\n");
  return 0;
}
