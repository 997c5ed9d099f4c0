// Latency probe for the split's library steps on an n x n complex128 Hermitian matrix:
// Zheevd alone / two at once on two streams, Zheevdx (top n/4), XsyevBatched (batch 1, 2), Zpotrf, Zgeqrf+Zungqr (n x n/4).
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cuComplex.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#define CK(x) do { auto e = (x); if ((int)e != 0) { printf("{\"error\": \"%s -> %d line %d\"}\n", #x, (int)e, __LINE__); exit(1);} } while (0)
typedef cuDoubleComplex Z;
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 1024;
  int r = n / 4;
  cusolverDnHandle_t h[2]; cudaStream_t st[2];
  for (int i = 0; i < 2; ++i) { CK(cusolverDnCreate(&h[i])); CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking)); CK(cusolverDnSetStream(h[i], st[i])); }
  size_t nn = (size_t)n * n;
  std::vector<Z> A(nn), H(nn);
  srand(1);
  for (auto& a : A) a = make_cuDoubleComplex(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
  for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) {  // H = A A^H + I (HPD)
    double re = 0, im = 0;
    for (int k = 0; k < 64; ++k) { Z a = A[i + (size_t)k * n], b = A[j + (size_t)k * n]; re += a.x * b.x + a.y * b.y; im += a.y * b.x - a.x * b.y; }
    if (i == j) { re += 1.0; im = 0; }
    H[i + (size_t)j * n] = make_cuDoubleComplex(re, im); H[j + (size_t)i * n] = make_cuDoubleComplex(re, -im);
  }
  Z *dH[2], *dW[2]; double* dL[2]; int* info[2];
  for (int i = 0; i < 2; ++i) { CK(cudaMalloc(&dH[i], 2 * nn * sizeof(Z))); CK(cudaMalloc(&dL[i], 2 * n * sizeof(double))); CK(cudaMalloc(&info[i], 8 * sizeof(int))); }
  int lw; CK(cusolverDnZheevd_bufferSize(h[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, dL[0], &lw));
  for (int i = 0; i < 2; ++i) CK(cudaMalloc(&dW[i], (size_t)lw * sizeof(Z)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  auto load = [&](int i) { CK(cudaMemcpy(dH[i], H.data(), nn * sizeof(Z), cudaMemcpyHostToDevice)); CK(cudaMemcpy(dH[i] + nn, H.data(), nn * sizeof(Z), cudaMemcpyHostToDevice)); };
  printf("{\"n\": %d", n);
  for (int rep = 0; rep < 3; ++rep) {  // one heevd
    load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, st[0]);
    CK(cusolverDnZheevd(h[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, dL[0], dW[0], lw, info[0]));
    cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf(", \"heevd_ms\": %.3f", ms);
  for (int rep = 0; rep < 3; ++rep) {  // eigenvalues only
    load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, st[0]);
    CK(cusolverDnZheevd(h[0], CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, dL[0], dW[0], lw, info[0]));
    cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf(", \"heevd_novec_ms\": %.3f", ms);
  for (int rep = 0; rep < 3; ++rep) {  // two heevd at once
    load(0); load(1); cudaDeviceSynchronize();
    cudaEventRecord(e0, st[0]); cudaStreamWaitEvent(st[1], e0, 0);
    CK(cusolverDnZheevd(h[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, dL[0], dW[0], lw, info[0]));
    CK(cusolverDnZheevd(h[1], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[1], n, dL[1], dW[1], lw, info[1]));
    cudaEventRecord(e1, st[1]); cudaStreamWaitEvent(st[0], e1, 0); cudaEventRecord(e1, st[0]);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf(", \"heevd_two_streams_ms\": %.3f", ms);
  {  // heevdx, top r
    int lx, found; CK(cusolverDnZheevdx_bufferSize(h[0], CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, 0, 0, n - r + 1, n, &found, dL[0], &lx));
    Z* w; CK(cudaMalloc(&w, (size_t)lx * sizeof(Z)));
    for (int rep = 0; rep < 3; ++rep) {
      load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, st[0]);
      CK(cusolverDnZheevdx(h[0], CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, 0, 0, n - r + 1, n, &found, dL[0], w, lx, info[0]));
      cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"heevdx_top_quarter_ms\": %.3f", ms);
    cudaFree(w);
  }
#if CUSOLVER_VERSION >= 11700
  for (int batch = 1; batch <= 2; ++batch) {  // batched syev (64-bit API)
    cusolverDnParams_t prm; CK(cusolverDnCreateParams(&prm));
    size_t dws = 0, hws = 0;
    cusolverStatus_t s = cusolverDnXsyevBatched_bufferSize(h[0], prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, dH[0], n, CUDA_R_64F, dL[0], CUDA_C_64F, &dws, &hws, batch);
    if (s != CUSOLVER_STATUS_SUCCESS) { printf(", \"syev_batched_%d\": \"buffersize status %d\"", batch, (int)s); continue; }
    void* dw; CK(cudaMalloc(&dw, dws + 16)); std::vector<char> hw(hws + 16);
    for (int rep = 0; rep < 3; ++rep) {
      load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, st[0]);
      s = cusolverDnXsyevBatched(h[0], prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, dH[0], n, CUDA_R_64F, dL[0], CUDA_C_64F, dw, dws, hw.data(), hws, info[0], batch);
      cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"syev_batched_%d_ms\": %.3f, \"syev_batched_%d_status\": %d", batch, ms, batch, (int)s);
    cudaFree(dw);
  }
#endif
  {  // potrf n and r
    int lp; CK(cusolverDnZpotrf_bufferSize(h[0], CUBLAS_FILL_MODE_LOWER, n, dH[0], n, &lp));
    Z* w; CK(cudaMalloc(&w, (size_t)lp * sizeof(Z)));
    for (int rep = 0; rep < 3; ++rep) {
      load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, st[0]);
      CK(cusolverDnZpotrf(h[0], CUBLAS_FILL_MODE_LOWER, n, dH[0], n, w, lp, info[0]));
      cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"potrf_n_ms\": %.3f", ms);
    for (int rep = 0; rep < 3; ++rep) {
      load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, st[0]);
      CK(cusolverDnZpotrf(h[0], CUBLAS_FILL_MODE_LOWER, r, dH[0], n, w, lp, info[0]));
      cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"potrf_quarter_ms\": %.3f", ms);
    cudaFree(w);
  }
  {  // geqrf + ungqr of n x r
    int l1, l2; Z* tau; CK(cudaMalloc(&tau, n * sizeof(Z)));
    CK(cusolverDnZgeqrf_bufferSize(h[0], n, r, dH[0], n, &l1)); CK(cusolverDnZungqr_bufferSize(h[0], n, r, r, dH[0], n, tau, &l2));
    int l = l1 > l2 ? l1 : l2; Z* w; CK(cudaMalloc(&w, (size_t)l * sizeof(Z)));
    float msq = 0;
    for (int rep = 0; rep < 3; ++rep) {
      load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, st[0]);
      CK(cusolverDnZgeqrf(h[0], n, r, dH[0], n, tau, w, l, info[0]));
      cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&msq, e0, e1);
      cudaEventRecord(e0, st[0]);
      CK(cusolverDnZungqr(h[0], n, r, r, dH[0], n, tau, w, l, info[0]));
      cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"geqrf_n_by_quarter_ms\": %.3f, \"ungqr_ms\": %.3f", msq, ms);
  }
  printf("}\n");
  return 0;
}
