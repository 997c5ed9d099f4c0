// Does cuSOLVER's Zheevd run inside green contexts (SM partitions), and do two solves on disjoint
// partitions overlap?  Times Zheevd(n) on the whole GPU, on one partition of `sms` SMs, and two at
// once on two disjoint partitions.  Run under `timeout`: a library kernel that assumes the whole
// GPU could deadlock inside a partition.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cuComplex.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { auto e = (x); if ((int)e != 0) { printf("{\"error\": \"%s -> %d line %d\"}\n", #x, (int)e, __LINE__); fflush(stdout); exit(1);} } while (0)
typedef cuDoubleComplex Z;
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 1024;
  unsigned sms = argc > 2 ? atoi(argv[2]) : 72;
  CK(cudaFree(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource parts[2], rem; unsigned ng = 2;
  CK(cuDevSmResourceSplitByCount(parts, &ng, &all, &rem, 0, sms));
  printf("{\"n\": %d, \"sm_total\": %u, \"groups\": %u, \"sm_per_group\": %u, \"sm_remaining\": %u", n, all.sm.smCount, ng, parts[0].sm.smCount, rem.sm.smCount);
  fflush(stdout);
  if (ng < 2) { printf(", \"error\": \"fewer than 2 groups\"}\n"); return 1; }
  CUgreenCtx g[2]; CUstream gs[2]; cusolverDnHandle_t h[3]; cudaStream_t full;
  for (int i = 0; i < 2; ++i) {
    CUdevResourceDesc d; CK(cuDevResourceGenerateDesc(&d, &parts[i], 1));
    CK(cuGreenCtxCreate(&g[i], d, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxStreamCreate(&gs[i], g[i], CU_STREAM_NON_BLOCKING, 0));
    CK(cusolverDnCreate(&h[i])); CK(cusolverDnSetStream(h[i], (cudaStream_t)gs[i]));
  }
  CK(cudaStreamCreateWithFlags(&full, cudaStreamNonBlocking));
  CK(cusolverDnCreate(&h[2])); CK(cusolverDnSetStream(h[2], full));
  size_t nn = (size_t)n * n;
  std::vector<Z> H(nn);
  srand(1);
  for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) {
    double re = rand() / (double)RAND_MAX - 0.5, im = (i == j) ? 0.0 : rand() / (double)RAND_MAX - 0.5;
    H[i + (size_t)j * n] = make_cuDoubleComplex(re, im); H[j + (size_t)i * n] = make_cuDoubleComplex(re, -im);
  }
  Z *dH[2], *dW[2]; double* dL[2]; int* info[2];
  int lw; CK(cusolverDnZheevd_bufferSize(h[2], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, nullptr, n, nullptr, &lw));
  for (int i = 0; i < 2; ++i) { CK(cudaMalloc(&dH[i], nn * sizeof(Z))); CK(cudaMalloc(&dL[i], n * sizeof(double))); CK(cudaMalloc(&info[i], sizeof(int))); CK(cudaMalloc(&dW[i], (size_t)lw * sizeof(Z))); }
  cudaEvent_t e0, e1, e2; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  float ms;
  auto load = [&](int i) { CK(cudaMemcpy(dH[i], H.data(), nn * sizeof(Z), cudaMemcpyHostToDevice)); };
  for (int rep = 0; rep < 3; ++rep) {
    load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, full);
    CK(cusolverDnZheevd(h[2], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, dL[0], dW[0], lw, info[0]));
    cudaEventRecord(e1, full); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf(", \"heevd_full_gpu_ms\": %.3f", ms); fflush(stdout);
  for (int rep = 0; rep < 3; ++rep) {
    load(0); cudaDeviceSynchronize(); cudaEventRecord(e0, (cudaStream_t)gs[0]);
    CK(cusolverDnZheevd(h[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, dL[0], dW[0], lw, info[0]));
    cudaEventRecord(e1, (cudaStream_t)gs[0]); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  int hi = -1; CK(cudaMemcpy(&hi, info[0], sizeof(int), cudaMemcpyDeviceToHost));
  printf(", \"heevd_one_partition_ms\": %.3f, \"info\": %d", ms, hi); fflush(stdout);
  for (int rep = 0; rep < 3; ++rep) {
    load(0); load(1); cudaDeviceSynchronize();
    cudaEventRecord(e0, (cudaStream_t)gs[0]); cudaStreamWaitEvent((cudaStream_t)gs[1], e0, 0);
    CK(cusolverDnZheevd(h[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[0], n, dL[0], dW[0], lw, info[0]));
    CK(cusolverDnZheevd(h[1], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dH[1], n, dL[1], dW[1], lw, info[1]));
    cudaEventRecord(e2, (cudaStream_t)gs[1]); cudaStreamWaitEvent((cudaStream_t)gs[0], e2, 0); cudaEventRecord(e1, (cudaStream_t)gs[0]);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf(", \"heevd_two_partitions_ms\": %.3f}\n", ms);
  return 0;
}
