// FP64 roofline denominators on the box: DMMA (mma.sync m8n8k4 f64) and DFMA
// throughput loops.  Prints one JSON line.  Standalone measurement tool.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void dmma_loop(double* out, int iters) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  for (int t = 0; t < 8; ++t) x[t] = threadIdx.x + t;
  const double a = 1.0000001, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = fma(x[t], a, b);
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += x[t];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  double best_mma = 0, best_fma = 0;
  for (int blocks_per_sm : {1, 2, 4}) {
    int grid = sms * blocks_per_sm, threads = 256;
    dmma_loop<<<grid, threads>>>(d, 100);
    cudaEventRecord(e0);
    dmma_loop<<<grid, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256.0 * 8 * iters * (double)grid * (threads / 32);
    double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best_mma) best_mma = tf;
    dfma_loop<<<grid, threads>>>(d, 100);
    cudaEventRecord(e0);
    dfma_loop<<<grid, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * iters * (double)grid * threads;
    tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best_fma) best_fma = tf;
  }
  printf("{\"dmma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"sms\": %d, \"clock_khz\": %d}\n", best_mma, best_fma, sms, clk);
  return 0;
}
