// Batched complex128 GEMM on the FP64 tensor cores of sm_100a.
//
// tcgen05.mma has no f64 kind (ptxas rejects .kind::f64), so the FP64 tensor
// path on B200 is the warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  The
// complex product uses the 3M (Gauss) form -- three real DMMAs per complex
// k-step on planar fragments (zgemm3m_kernel below).  CTA tile 64x64 (complex)
// x BK=16; operands staged global->shared with cp.async (16 B per complex
// element, zero-filled outside the matrix), double-buffered, two CTAs per SM;
// shared strides padded so every fragment load (one LDS.128 = one complex) is
// bank-conflict free.  op(A), op(B) in {N, T, C}; conjugation is folded into
// the fragment sign.  Row-major everywhere; batch strides may be 0 (shared).
#include <algorithm>
#include <array>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace tn {
namespace {

std::atomic<int64_t> g_launches{0};
struct Prof {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::vector<double> cm;
  std::vector<std::array<int, 9>> shape;  // M, N, K, batch, opa, opb, A batched, B batched, has beta
};
Prof g_prof;
std::mutex g_prof_mu;
constexpr int BM = 64, BN = 64, BK = 16;
constexpr int LDN = BK + 4;    // [rows][BK] tiles: row stride = 20 complex (= 4 mod 8 slots)
constexpr int LDT = BM + 2;    // [BK][cols] tiles: row stride = 66 complex (= 2 mod 8 slots)
constexpr int TILE = BM * LDN; // 1280 >= BK * LDT = 1056
constexpr int STAGE = 2 * TILE;

struct Params {
  int M, N, K;
  int ksplit;          // > 1: blockIdx.z = batch * ksplit + split, partial sums to `part`
  double* part;        // [batch][ksplit][M][N] complex partials (split-K only)
  cplx alpha, beta;
  int has_beta;
  const double* dscale;  // nullable DEVICE scalar: alpha and beta are multiplied by *dscale
  const cplx* A;
  const cplx* B;
  cplx* C;
  int64_t lda, ldb, ldc, sA, sB, sC;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// 3M (Gauss) variant: (a + ib)(c + id) = ac - bd + i[(a + b)(c + d) - ac - bd],
// three real DMMAs per complex k-step: P1 += Ar Br, P2 += Ai Bi,
// P3 += (Ar + Ai)(Br + Bi); C_re = P1 - P2, C_im = P3 - P1 - P2.  CTA 64x64,
// 8 warps (4 x 2), warp tile 16 x 32 (2 x 4 DMMA tiles), NSTAGE-deep cp.async
// pipeline, one CTA per SM (<= 255 registers).
constexpr int NT3 = 256;

template <char OPA, char OPB, int NSTAGE3, int MINB>
__global__ void __launch_bounds__(NT3, MINB) zgemm3m_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* smem = reinterpret_cast<cplx*>(smem_raw);
  const int ks = p.ksplit > 1 ? p.ksplit : 1;
  const int64_t bz = blockIdx.z / ks;
  const int split = blockIdx.z % ks;
  const cplx* __restrict__ A = p.A + bz * p.sA;
  const cplx* __restrict__ B = p.B + bz * p.sB;
  cplx* __restrict__ C = p.C + bz * p.sC;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // 4 x 2 warps: warp rows of 16, columns of 32
  const int nk_all = (p.K + BK - 1) / BK;
  const int kt0 = (int)((int64_t)nk_all * split / ks), kt1 = (int)((int64_t)nk_all * (split + 1) / ks);
  const int g = lane >> 2, q = lane & 3;

  auto load_stage = [&](int stage, int k0) {
    cplx* sA = smem + stage * STAGE;
    cplx* sB = sA + TILE;
#pragma unroll
    for (int j = 0; j < (BM * BK) / NT3; ++j) {
      const int e = tid + j * NT3;
      if (OPA == 'N') {
        const int m = e / BK, k = e % BK, gm = m0 + m, gk = k0 + k;
        const bool ok = gm < p.M && gk < p.K;
        cp_async16(sA + m * LDN + k, ok ? (const void*)(A + (int64_t)gm * p.lda + gk) : (const void*)A, ok);
      } else {
        const int k = e / BM, m = e % BM, gm = m0 + m, gk = k0 + k;
        const bool ok = gm < p.M && gk < p.K;
        cp_async16(sA + k * LDT + m, ok ? (const void*)(A + (int64_t)gk * p.lda + gm) : (const void*)A, ok);
      }
    }
#pragma unroll
    for (int j = 0; j < (BN * BK) / NT3; ++j) {
      const int e = tid + j * NT3;
      if (OPB == 'N') {
        const int k = e / BN, n = e % BN, gn = n0 + n, gk = k0 + k;
        const bool ok = gn < p.N && gk < p.K;
        cp_async16(sB + k * LDT + n, ok ? (const void*)(B + (int64_t)gk * p.ldb + gn) : (const void*)B, ok);
      } else {
        const int n = e / BK, k = e % BK, gn = n0 + n, gk = k0 + k;
        const bool ok = gn < p.N && gk < p.K;
        cp_async16(sB + n * LDN + k, ok ? (const void*)(B + (int64_t)gn * p.ldb + gk) : (const void*)B, ok);
      }
    }
  };

  double p1[2][4][2], p2[2][4][2], p3[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int t = 0; t < 2; ++t) p1[i][j][t] = p2[i][j][t] = p3[i][j][t] = 0.0;

  const int nk = kt1 - kt0;
#pragma unroll
  for (int s = 0; s < NSTAGE3 - 1; ++s) {
    if (s < nk) load_stage(s, (kt0 + s) * BK);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<NSTAGE3 - 2>();
    __syncthreads();
    {
      const int nx = kt + NSTAGE3 - 1;
      if (nx < nk) load_stage(nx % NSTAGE3, (kt0 + nx) * BK);
      cp_commit();
    }
    const cplx* sA = smem + (kt % NSTAGE3) * STAGE;
    const cplx* sB = sA + TILE;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double ar[2], ai[2], as[2], br[4], bi[4], bs[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int row = wm * 16 + mi * 8 + g, col = kk * 4 + q;
        const cplx a = (OPA == 'N') ? sA[row * LDN + col] : sA[col * LDT + row];
        ar[mi] = a.x;
        ai[mi] = (OPA == 'C') ? -a.y : a.y;
        as[mi] = ar[mi] + ai[mi];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int krow = kk * 4 + q, ncol = wn * 32 + ni * 8 + g;
        const cplx b = (OPB == 'N') ? sB[krow * LDT + ncol] : sB[ncol * LDN + krow];
        br[ni] = b.x;
        bi[ni] = (OPB == 'C') ? -b.y : b.y;
        bs[ni] = br[ni] + bi[ni];
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          dmma(p1[mi][ni], ar[mi], br[ni]);
          dmma(p2[mi][ni], ai[mi], bi[ni]);
          dmma(p3[mi][ni], as[mi], bs[ni]);
        }
    }
  }
  cp_wait<0>();

#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const int row = m0 + wm * 16 + mi * 8 + g;
    if (row >= p.M) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = n0 + wn * 32 + ni * 8 + 2 * q + j;
        if (col < p.N) {
          const double re = p1[mi][ni][j] - p2[mi][ni][j];
          const double im = p3[mi][ni][j] - p1[mi][ni][j] - p2[mi][ni][j];
          if (ks > 1) {  // partial of this K slice (reduced in split order by zreduce_kernel)
            reinterpret_cast<cplx*>(p.part)[((bz * ks + split) * (int64_t)p.M + row) * p.N + col] = make_double2(re, im);
          } else {
            const double f = p.dscale ? *p.dscale : 1.0;
            cplx v = cmul(cscale(p.alpha, f), make_double2(re, im));
            cplx* dst = C + (int64_t)row * p.ldc + col;
            if (p.has_beta) v = cadd(v, cmul(cscale(p.beta, f), *dst));
            *dst = v;
          }
        }
      }
    }
  }
}

// C = alpha * sum_split part + beta * C, splits summed in fixed order (deterministic)
__global__ void zreduce_kernel(Params p, int batch) {
  const int64_t mn = (int64_t)p.M * p.N, total = mn * batch;
  const cplx* part = reinterpret_cast<const cplx*>(p.part);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / mn, e = idx % mn;
    cplx acc = make_double2(0, 0);
    for (int sp = 0; sp < p.ksplit; ++sp) acc = cadd(acc, part[(b * p.ksplit + sp) * mn + e]);
    const int row = (int)(e / p.N), col = (int)(e % p.N);
    const double f = p.dscale ? *p.dscale : 1.0;
    cplx v = cmul(cscale(p.alpha, f), acc);
    cplx* dst = p.C + b * p.sC + (int64_t)row * p.ldc + col;
    if (p.has_beta) v = cadd(v, cmul(cscale(p.beta, f), *dst));
    *dst = v;
  }
}

constexpr int SMEM3_2 = 2 * STAGE * (int)sizeof(cplx);

template <char OPA, char OPB>
void launch(const Params& p, int batch, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    TN_CUDA(cudaFuncSetAttribute(zgemm3m_kernel<OPA, OPB, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM3_2));
    attr = true;
  }
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, batch);
  Params q = p;
  q.ksplit = 1;
  q.part = nullptr;
  const int64_t ctas = (int64_t)grid.x * grid.y * batch;
  const int nk = (p.K + BK - 1) / BK;
  if (ctas < 148 && nk >= 16) {  // split K to fill the SMs (>= 8 k-tiles per split)
    int ks = (int)std::min<int64_t>((296 + ctas - 1) / ctas, nk / 8);
    if (ks > 1) {
      q.ksplit = ks;
      q.part = (double*)dalloc(sizeof(cplx) * (size_t)ks * p.M * p.N * batch, st);
      if (std::getenv("TN_POISON")) TN_CUDA(cudaMemsetAsync(q.part, 0xFF, sizeof(cplx) * (size_t)ks * p.M * p.N * batch, st));
      grid.z = batch * ks;
    }
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_prof.on) {
    TN_CUDA(cudaEventCreate(&e0));
    TN_CUDA(cudaEventCreate(&e1));
    TN_CUDA(cudaEventRecord(e0, st));
  }
  zgemm3m_kernel<OPA, OPB, 2, 2><<<grid, NT3, SMEM3_2, st>>>(q);
  TN_CUDA(cudaGetLastError());
  count_launch();
  if (q.ksplit > 1) {
    const int64_t tot = (int64_t)p.M * p.N * batch;
    zreduce_kernel<<<(int)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, st>>>(q, batch);
    TN_CUDA(cudaGetLastError());
    count_launch();
    dfree(q.part, st);
  }
  if (g_prof.on) {
    TN_CUDA(cudaEventRecord(e1, st));
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.ev.push_back({e0, e1});
    g_prof.cm.push_back((double)p.M * p.N * p.K * batch);
    g_prof.shape.push_back({p.M, p.N, p.K, batch, (int)OPA, (int)OPB, p.sA != 0, p.sB != 0, p.has_beta});
  }
}

template <char OPA>
void dispatch_b(char opb, const Params& p, int batch, cudaStream_t st) {
  switch (opb) {
    case 'N': launch<OPA, 'N'>(p, batch, st); break;
    case 'T': launch<OPA, 'T'>(p, batch, st); break;
    case 'C': launch<OPA, 'C'>(p, batch, st); break;
    default: throw std::invalid_argument("opb");
  }
}


}  // namespace

void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Library-private stream-ordered memory: one cudaMemPool per device, created on
// first use, never the device's default pool (so torch's and other libraries'
// allocations are not affected by its policies).  Cached blocks are kept
// (release threshold max); the pool never inserts a dependency to reuse a
// block across streams (the two primal sweeps run on two streams and must not
// be serialised through recycled blocks).  Inside a stream capture the
// allocation becomes a graph memory node (cudaMallocAsync).
namespace {
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};
cudaMemPool_t device_pool(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (dev < 0 || dev >= 64) throw std::invalid_argument("device ordinal");
  if (!g_pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    TN_CUDA(cudaMemPoolCreate(&p, &props));
    uint64_t thr = UINT64_MAX;
    int off = 0;
    TN_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr));
    // a block freed on one stream may serve another stream only when that
    // costs no new dependency (already ordered, or the free has completed)
    int on = 1;  // measured at C3: 3.08 s per step with these two on, 3.20 s with them off
    TN_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolReuseFollowEventDependencies, &on));
    TN_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolReuseAllowOpportunistic, &on));
    TN_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolReuseAllowInternalDependencies, &off));
    g_pools[dev] = p;
  }
  return g_pools[dev];
}
}  // namespace

void* dalloc(size_t bytes, cudaStream_t st) {
  void* p = nullptr;
  bytes = std::max<size_t>(bytes, 16);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  TN_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone) {
    TN_CUDA(cudaMallocAsync(&p, bytes, st));
    return p;
  }
  int dev = 0;
  TN_CUDA(cudaGetDevice(&dev));
  TN_CUDA(cudaMallocFromPoolAsync(&p, bytes, device_pool(dev), st));
  return p;
}

void dfree(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

void pool_trim(int dev) {
  cudaMemPool_t p = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev >= 0 && dev < 64) p = g_pools[dev];
  }
  if (p) cudaMemPoolTrimTo(p, 0);
}
int64_t launch_count() { return g_launches.load(); }

bool gemm_profile_active() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  return g_prof.on;
}

void gemm_profile_begin() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& e : g_prof.ev) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  g_prof.ev.clear();
  g_prof.cm.clear();
  g_prof.shape.clear();
  g_prof.on = true;
}

void gemm_profile_end(double* ms, double* cmac) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.on = false;
  double t = 0, c = 0;
  FILE* log = nullptr;
  if (const char* path = std::getenv("TN_GEMM_LOG")) log = std::fopen(path, "w");
  for (size_t i = 0; i < g_prof.ev.size(); ++i) {
    TN_CUDA(cudaEventSynchronize(g_prof.ev[i].second));
    float m = 0;
    TN_CUDA(cudaEventElapsedTime(&m, g_prof.ev[i].first, g_prof.ev[i].second));
    t += m;
    c += g_prof.cm[i];
    if (log) {
      const auto& sh = g_prof.shape[i];
      std::fprintf(log, "%d %d %d %d %c %c %.6f %d %d %d\n", sh[0], sh[1], sh[2], sh[3], (char)sh[4], (char)sh[5], m,
                   sh[6], sh[7], sh[8]);
    }
    cudaEventDestroy(g_prof.ev[i].first);
    cudaEventDestroy(g_prof.ev[i].second);
  }
  if (log) std::fclose(log);
  g_prof.ev.clear();
  g_prof.cm.clear();
  g_prof.shape.clear();
  *ms = t;
  *cmac = c;
}

void zgemm(cudaStream_t st, char opa, char opb, int M, int N, int K, cplx alpha, const cplx* A, int64_t lda,
           int64_t sA, const cplx* B, int64_t ldb, int64_t sB, cplx beta, cplx* C, int64_t ldc, int64_t sC,
           int batch, const double* dscale) {
  if (M <= 0 || N <= 0 || batch <= 0) return;
  Params p;
  p.ksplit = 1;
  p.part = nullptr;
  p.alpha = alpha;
  p.beta = beta;
  p.has_beta = (beta.x != 0.0 || beta.y != 0.0);
  p.dscale = dscale;
  p.A = A; p.B = B; p.C = C;
  p.lda = lda; p.ldb = ldb; p.ldc = ldc; p.sA = sA; p.sB = sB; p.sC = sC;
  p.M = M; p.N = N; p.K = K;
  if (K <= 0) {  // C = beta C (alpha * empty product)
    p.K = 0;
  }
  // Stack a batch with a shared B into one tall GEMM when rows are contiguous.
  if (batch > 1 && sB == 0 && opa == 'N' && sA == (int64_t)M * lda && sC == (int64_t)M * ldc) {
    p.M = M * batch;
    batch = 1;
  }
  while (batch > 0) {  // grid.z <= 65535
    const int b = batch < 65535 ? batch : 65535;
    switch (opa) {
      case 'N': dispatch_b<'N'>(opb, p, b, st); break;
      case 'T': dispatch_b<'T'>(opb, p, b, st); break;
      case 'C': dispatch_b<'C'>(opb, p, b, st); break;
      default: throw std::invalid_argument("opa");
    }
    batch -= b;
    p.A += (int64_t)b * p.sA;
    p.B += (int64_t)b * p.sB;
    p.C += (int64_t)b * p.sC;
  }
}

}  // namespace tn
