// The HVP engine: static plan of the sweeps, primal pass (tn_hvp_environments)
// and batched tangent pass (tn_hvp_apply).  Every contraction is a call of the
// DMMA complex GEMM (zgemm.cu) or a small kernel (kernels.cu); SVD / QR of the
// two-site primal blocks use cuSOLVER (library primitives).
//
// Method (readings X7-X9):
//  * bottom sweep B_0 = I/2^{n/2} -> B_D applying G_k on the out legs, top sweep
//    T_D = U_ref/2^{n/2} -> T_0 applying G_k^dag (eq:fis, eq:bis),
//    each gate followed by a truncated two-site SVD (keep r = min(chi,4m,4bl,4br),
//    frozen renormalisation s);
//  * tangents in channel form sum_j Ab..B_j..Aa (App. D) with
//    the primal's isometries as fixed projectors;
//  * E_k and H_T[V]_k layer-wise from left/right environments (eq:environment,
//    eq:overlap-hvp) -- Algorithm 1's two passes
//     at layer granularity, forward tangent cached, backward
//    tangent on the fly.
#include <cublas_v2.h>
#include <cuda.h>
#include <cusolverDn.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <numeric>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <thread>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "engine.cuh"
#include "kernels.cuh"

struct tn_hvp_ctx;

namespace tn {
namespace {

#define TN_SOLVER(x)                                                                                   \
  do {                                                                                                 \
    cusolverStatus_t s_ = (x);                                                                         \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                                 \
      throw CudaError(std::string(#x) + ": cusolver status " + std::to_string((int)s_) + " @" + __FILE__ + \
                      ":" + std::to_string(__LINE__));                                                 \
  } while (0)

const cplx ONE = {1.0, 0.0}, ZERO = {0.0, 0.0}, MONE = {-1.0, 0.0};

enum StepType { MOVE_R = 0, MOVE_L = 1, PAIR = 2 };

struct Step {
  StepType type;
  int site = 0;  // MOVE: centre c before the move; PAIR: left site i
  int k = -1;
  bool lr = true;
  int bl = 0, m = 0, br = 0, r = 0, mn = 0;  // PAIR primal shapes
  int b = 0, bp = 0, kq = 0, nb2 = 0;        // MOVE primal shapes; nb2 = neighbour's other bond
  // chain bonds before the step (cuts site-1 .. site+2)
  int abm = 0, ab0 = 0, ab1 = 0, ab2 = 0;
  int aam = 0, aa0 = 0, aa1 = 0, aa2 = 0;
  size_t o_theta = 0, o_uh = 0, o_vh = 0, o_S = 0, o_s = 0, o_q = 0;  // primal-arena offsets (bytes)
  int s_index = -1;                                                  // ordinal of the pair step
};

struct Bonds {
  std::vector<int> p, ab, aa;
};

struct SidePlan {
  std::vector<int> ell;                     // processing order of layers
  std::vector<std::vector<Step>> steps;     // per processed layer
  std::vector<Bonds> snap;                  // bonds at each snapshot (before processing; + final)
  std::vector<std::vector<size_t>> o_snap;  // primal-arena offsets of snapshot sites
  Bonds init;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// TN_POISON=1 (diagnostic): every new device buffer is filled with NaN bytes,
// so a read of uninitialised memory that reaches an output shows up as NaN.
const bool g_poison = std::getenv("TN_POISON") != nullptr;
void poison(void* p, size_t bytes, cudaStream_t st) {
  if (g_poison) TN_CUDA(cudaMemsetAsync(p, 0xFF, bytes, st));
}

cplx* dnew(int64_t n, cudaStream_t st) {
  const size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(cplx);
  void* p = dalloc(bytes, st);
  poison(p, bytes, st);
  return (cplx*)p;
}
void ddel(cplx*& p, cudaStream_t st) {
  dfree(p, st);
  p = nullptr;
}
void dset(cplx*& slot, cplx* nw, cudaStream_t st) {
  ddel(slot, st);
  slot = nw;
}

struct Pool {  // stream-ordered transient device buffers
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Pool(cudaStream_t s) : st(s) {}
  cplx* c(int64_t n) {
    if (n <= 0) n = 1;
    void* p = dalloc((size_t)n * sizeof(cplx), st);
    poison(p, (size_t)n * sizeof(cplx), st);
    ptrs.push_back(p);
    return (cplx*)p;
  }
  void* raw(size_t bytes) {
    void* p = dalloc(std::max<size_t>(bytes, 16), st);
    poison(p, std::max<size_t>(bytes, 16), st);
    ptrs.push_back(p);
    return p;
  }
  ~Pool() {
    for (void* p : ptrs) dfree(p, st);
  }
};

}  // namespace

// set on the fused step's forward-tangent thread: its GEMMs count as apply work
thread_local bool g_fwd_thread = false;

struct Engine {
  tn_hvp_config cfg{};
  int n = 0, D = 0, off = 0, chi = 0, K = 0;
  // Site physical dimension P = 2 NI (index p = out * NI + in): operator mode
  // P = 4 (MPO sites, bottom start I/2^{n/2}); state mode P = 2 (MPS sites,
  // bottom start a product state).  PP = P^2, NI2 = NI^2.
  int P = 4, PP = 16, NI = 2, NI2 = 4;
  cplx* d_init = nullptr;  // [n][P] bond-1 bottom start (identity/sqrt 2 per site, or the product state)
  std::vector<std::vector<std::pair<int, int>>> layers;  // per layer (k, s)
  std::vector<int> ref_bonds;
  SidePlan bot, top;
  int n_pair_steps = 0;
  // primal arena
  char* arena = nullptr;
  size_t arena_bytes = 0;
  bool own_arena = true;  // false: caller-owned primal_buf (tn_hvp_setup)
  size_t o_gates = 0, o_gdag = 0, o_E = 0, o_gradf = 0, o_scal = 0, o_diag = 0;
  // side regions of the store (split primal over two ranks): [o_side[0], o_side[1])
  // = bottom sweep (its diagnostics, snapshots, replay data), [o_side[1], o_side[2]) = top
  size_t o_side[3] = {0, 0, 0}, o_sdiag[2] = {0, 0};
  std::vector<std::vector<size_t>> o_L, o_R;  // per layer, per cut
  cplx* ref = nullptr;                        // reference MPO copy (device)
  std::vector<size_t> ref_off;
  // solvers: one per concurrent primal sweep (bottom on the caller's stream,
  // top on an internal stream driven by a second host thread)
  struct Solver {
    cusolverDnHandle_t h = nullptr;
    cusolverDnParams_t prm = nullptr;
    cublasHandle_t bl = nullptr;  // triangular solves of CholeskyQR2 (created on first use)
    int lwork_potrf = 0;
    std::vector<char> host_ws;
  };
  Solver sol[2];
  int lwork_heevd = 0;
  std::atomic<int> n_fallback{0}, n_deflate{0}, n_noise{0};
  const bool lowdin_lq = std::getenv("TN_NO_LOWDIN_LQ") == nullptr;
  const bool cholqr = std::getenv("TN_NO_CHOLQR") == nullptr;
  // rows above deflate_step x (the level's top sigma) count as resolved by that level's Gram matrix
  const double deflate_step = std::getenv("TN_DEFLATE_STEP") ? std::atof(std::getenv("TN_DEFLATE_STEP")) : 1e-4;
  static constexpr int kCholMin = 32;  // below: the Householder panel is as fast
  std::atomic<int> n_cholqr_fallback{0}, n_lowrank{0};
  const bool lowrank_on = std::getenv("TN_NO_LOWRANK") == nullptr;
  FILE* split_log = std::getenv("TN_SPLIT_LOG") ? fopen(std::getenv("TN_SPLIT_LOG"), "a") : nullptr;
  std::mutex split_log_mu;
  std::vector<char> lowrank_hint;  // per pair step (s_index): 1 = try the range probe at the next pass, 0 = not now, 2 = it failed here
  cplx* d_omega = nullptr;         // fixed test matrix of the range probe (om_rows x om_cols)
  int om_rows = 0, om_cols = 0;
  size_t svd_dws = 0, svd_hws = 0;
  int lwork_geqrf = 0, lwork_ungqr = 0;
  cudaStream_t st2 = nullptr, st1 = nullptr;  // top / bottom sweep streams (non-blocking)
  cudaStream_t stg = nullptr;                 // layer gradients, overlapped with the sweeps
  cudaStream_t stf = nullptr, sth = nullptr;  // fused step: forward tangents; spare side stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join1 = nullptr, ev_joing = nullptr, ev_joinf = nullptr;
  std::vector<cudaEvent_t> ev_snap[2];        // per side: layer snapshot idx is in the arena
  bool primal_valid = false;
  // N2: translation-invariant mode (layer gates), valid after ti_environments
  int* d_layer_of = nullptr;   // [K] layer index of each gate
  int* d_layer_start = nullptr;  // [D+1] first gate of each layer
  cplx* ti_buf = nullptr;      // [3][D][16]: layer gates g, dT/dg, grad_f
  bool ti_valid = false;
  // Direction-independent tangent chains of one side at the current point:
  // every chain tensor the replay creates (and the move factors X), recorded
  // by the first apply after a primal pass and borrowed by later ones.
  struct ChainCache {
    bool built = false;
    std::vector<cplx*> init_Ab, init_Aa;
    std::vector<std::array<cplx*, 4>> step;  // per replayed step, in order
    std::vector<cplx*> owned;                // everything to free on drop
  };
  enum ChainMode { CHAIN_OWN = 0, CHAIN_RECORD = 1, CHAIN_REPLAY = 2 };
  struct Tangent {  // channel-form tangents for nb directions
    std::vector<cplx*> Ab, Aa, B;  // B[s]: nb blocks, direction stride = size(B[s])
    Bonds bd;                      // bonds: ab / aa used (p = primal)
    ChainMode mode = CHAIN_OWN;    // RECORD / REPLAY: chains belong to `cache`
    ChainCache* cache = nullptr;
    size_t step_no = 0;
  };
  struct TanSnap {
    std::vector<cplx*> Ab, Aa, B;
    Bonds bd;
    bool chains_owned = true;
  };
  ChainCache chain_cache[2];  // 0 bottom (forward tangents), 1 top (backward)
  const bool chain_cache_enabled = std::getenv("TN_NO_CHAIN_CACHE") == nullptr;
  // Per-point memo of the direction-independent tensors of layer_hvp (block
  // pairs, shared chain environments, shared products), keyed (layer, site,
  // tag); recorded by the first apply after a primal pass within a memory
  // budget (a third of the free memory then), borrowed afterwards.
  std::unordered_map<uint64_t, cplx*> memo_map;
  std::vector<cplx*> memo_owned;
  size_t memo_bytes = 0, memo_budget = 0;
  bool memo_budget_set = false;
  // tn_hvp_set_cache_budget: 0 = automatic (chain caches within half, memo
  // within a third of the free memory at the first apply); else a cap in bytes
  // on chain caches + memo together (several contexts sharing a device).
  size_t cache_budget = 0;
  // CUDA-graph replay of tn_hvp_apply: a (batch, aux) key seen a second time
  // since the last primal pass is captured once (engine-owned I/O buffers) and
  // replayed; host scalars baked into the graph (frozen s) are per point, so
  // every primal pass drops the graphs.  TN_NO_GRAPH=1 disables.
  struct ApplyGraph {
    int batch = 0;
    bool aux = false;
    bool point_free = false;  // captured without per-point caches: valid across primal passes
    int calls = 0;
    bool failed = false;
    cudaGraphExec_t exec = nullptr;
    cplx *in = nullptr, *out = nullptr, *auxb = nullptr;
    int64_t launches = 0;
    double work = 0, work_apply = 0;
  };
  std::vector<ApplyGraph> graphs;
  cudaStream_t stc = nullptr;  // capture stream
  const bool graphs_enabled = std::getenv("TN_NO_GRAPH") == nullptr;
  int applies_at_point = 0;     // tn_hvp_apply calls since the last primal pass
  bool no_cache = false;        // a point-free capture is running: no chain cache, no memo
  static constexpr int kGraphMaxBatch = 8;
  double work_primal = 0, work_apply = 0, work_fwd_first = 0;
  std::atomic<double> work_counter{0.0};
  std::atomic<double> work_counter_fwd{0.0};  // GEMMs issued by the fused step's forward-tangent thread
  std::string err;
  int device = 0;

  template <class T = cplx>
  T* at(size_t o) const {
    return reinterpret_cast<T*>(arena + o);
  }

  // ------------------------------------------------------------ GEMMs --
  // ds (nullable, DEVICE): a and b are scaled by *ds in the GEMM epilogue
  void mm(cudaStream_t st, char oa, char ob, int M, int N, int Kd, cplx a, const cplx* A, int64_t lda, int64_t sA,
          const cplx* B, int64_t ldb, int64_t sB, cplx b, cplx* C, int64_t ldc, int64_t sC, int batch,
          const double* ds = nullptr) {
    if (M <= 0 || N <= 0 || batch <= 0) return;
    (g_fwd_thread ? work_counter_fwd : work_counter)
        .fetch_add((double)M * N * std::max(Kd, 0) * batch, std::memory_order_relaxed);
    zgemm(st, oa, ob, M, N, Kd, a, A, lda, sA, B, ldb, sB, b, C, ldc, sC, batch, ds);
  }
  // C(MxN) = a A(MxK) B(KxN) + b C
  void nn(cudaStream_t st, int M, int N, int Kd, const cplx* A, int64_t sA, const cplx* B, int64_t sB, cplx* C,
          int64_t sC, int batch, cplx a = ONE, cplx b = ZERO, const double* ds = nullptr) {
    mm(st, 'N', 'N', M, N, Kd, a, A, Kd, sA, B, N, sB, b, C, N, sC, batch, ds);
  }
  // C(MxN) = a A^H B, A stored (K x M), B (K x N)
  void cn(cudaStream_t st, int M, int N, int Kd, const cplx* A, int64_t sA, const cplx* B, int64_t sB, cplx* C,
          int64_t sC, int batch, cplx a = ONE, cplx b = ZERO, const double* ds = nullptr) {
    mm(st, 'C', 'N', M, N, Kd, a, A, M, sA, B, N, sB, b, C, N, sC, batch, ds);
  }
  // C(MxN) = a A B^H, A (M x K), B stored (N x K)
  void nc(cudaStream_t st, int M, int N, int Kd, const cplx* A, int64_t sA, const cplx* B, int64_t sB, cplx* C,
          int64_t sC, int batch, cplx a = ONE, cplx b = ZERO, const double* ds = nullptr) {
    mm(st, 'N', 'C', M, N, Kd, a, A, Kd, sA, B, Kd, sB, b, C, N, sC, batch, ds);
  }

  // ------------------------------------------------------------- plan --
  void build_layers() {
    layers.assign(D, {});
    int k = 0;
    for (int ell = 1; ell <= D; ++ell) {
      const int o = (off + ell - 1) % 2;
      for (int s = o; s + 1 < n; s += 2) layers[ell - 1].push_back({k++, s});
    }
    K = k;
  }

  void plan_side(SidePlan& sp, const std::vector<int>& init, bool is_top) {
    sp = SidePlan();
    Bonds b;
    b.p = init;
    b.ab = init;
    b.aa = init;
    sp.init = b;
    int c = 0;
    if (is_top)
      for (int ell = D; ell >= 1; --ell) sp.ell.push_back(ell);
    else
      for (int ell = 1; ell <= D; ++ell) sp.ell.push_back(ell);
    for (int ell : sp.ell) {
      sp.snap.push_back(b);
      const bool lr = is_top ? ((D - ell) % 2 == 0) : (ell % 2 == 1);
      std::vector<std::pair<int, int>> ly = layers[ell - 1];
      if (!lr) std::reverse(ly.begin(), ly.end());
      std::vector<Step> steps;
      for (auto [k, i] : ly) {
        const int target = lr ? i : i + 1;
        while (c != target) {
          Step st;
          const bool right = c < target;
          st.type = right ? MOVE_R : MOVE_L;
          st.site = c;
          st.b = b.p[c];
          st.bp = b.p[c + 1];
          st.abm = c > 0 ? b.ab[c - 1] : 0;
          st.ab0 = b.ab[c];
          st.ab1 = b.ab[c + 1];
          st.ab2 = c + 2 <= n ? b.ab[c + 2] : 0;
          st.aam = c > 0 ? b.aa[c - 1] : 0;
          st.aa0 = b.aa[c];
          st.aa1 = b.aa[c + 1];
          st.aa2 = c + 2 <= n ? b.aa[c + 2] : 0;
          if (right) {
            st.kq = std::min(P * st.b, st.bp);
            st.nb2 = b.p[c + 2];
            if (b.ab[c] != b.p[c]) throw std::logic_error("plan: before-chain bond != primal bond (move right)");
            b.p[c + 1] = st.kq;
            b.ab[c + 1] = st.kq;
            ++c;
          } else {
            st.kq = std::min(st.b, P * st.bp);
            st.nb2 = b.p[c - 1];
            if (b.aa[c + 1] != b.p[c + 1]) throw std::logic_error("plan: after-chain bond != primal bond (move left)");
            b.p[c] = st.kq;
            b.aa[c] = st.kq;
            --c;
          }
          steps.push_back(st);
        }
        Step st;
        st.type = PAIR;
        st.site = i;
        st.k = k;
        st.lr = lr;
        st.bl = b.p[i];
        st.m = b.p[i + 1];
        st.br = b.p[i + 2];
        st.mn = std::min(P * st.bl, P * st.br);
        st.r = std::min({chi, 4 * st.m, P * st.bl, P * st.br});  // gate operator-Schmidt rank <= 4
        st.abm = i > 0 ? b.ab[i - 1] : 0;
        st.ab0 = b.ab[i];
        st.ab1 = b.ab[i + 1];
        st.ab2 = b.ab[i + 2];
        st.aam = i > 0 ? b.aa[i - 1] : 0;
        st.aa0 = b.aa[i];
        st.aa1 = b.aa[i + 1];
        st.aa2 = b.aa[i + 2];
        if (b.ab[i] != st.bl || b.aa[i + 2] != st.br) throw std::logic_error("plan: chain/primal bond mismatch at pair");
        b.p[i + 1] = st.r;
        b.ab[i + 1] = st.r;
        b.aa[i + 1] = st.r;
        c = lr ? i + 1 : i;
        steps.push_back(st);
        ++n_pair_steps;
      }
      sp.steps.push_back(steps);
    }
    sp.snap.push_back(b);
  }

  size_t mpo_elems(const std::vector<int>& p) const {
    size_t e = 0;
    for (int s = 0; s < n; ++s) e += (size_t)p[s] * P * p[s + 1];
    return e;
  }

  void layout_arena() {
    size_t o = 0;
    auto take = [&](size_t bytes) {
      const size_t r = o;
      o = align256(o + bytes);
      return r;
    };
    const size_t C = sizeof(cplx);
    o_gates = take(K * 16 * C);
    o_gdag = take(K * 16 * C);
    o_E = take(K * 16 * C);
    o_gradf = take(K * 16 * C);
    o_scal = take(8 * sizeof(double));
    o_diag = take(8 * sizeof(double));
    int s_index = 0;
    for (SidePlan* sp : {&bot, &top}) {
      const int side = sp == &top;
      o_side[side] = o;
      o_sdiag[side] = take(8 * sizeof(double));
      sp->o_snap.clear();
      for (const Bonds& b : sp->snap) {
        std::vector<size_t> offs(n);
        for (int s = 0; s < n; ++s) offs[s] = take((size_t)b.p[s] * P * b.p[s + 1] * C);
        sp->o_snap.push_back(offs);
      }
      for (auto& ls : sp->steps)
        for (Step& st : ls) {
          if (st.type == PAIR) {
            st.o_theta = take((size_t)PP * st.bl * st.br * C);
            st.o_uh = take((size_t)st.r * P * st.bl * C);
            st.o_vh = take((size_t)st.r * P * st.br * C);
            st.o_S = take((size_t)st.mn * sizeof(double));
            st.o_s = take(sizeof(double));
            st.s_index = s_index++;
          } else {
            st.o_q = take((size_t)P * std::max(st.b, st.bp) * st.kq * C);
          }
        }
    }
    o_side[2] = o;
    // layer environments L0/R0: layer ell uses T_ell (top snapshot index D-ell) and B_{ell-1} (bottom index ell-1)
    o_L.assign(D + 1, std::vector<size_t>(n + 1, 0));
    o_R.assign(D + 1, std::vector<size_t>(n + 1, 0));
    for (int ell = 1; ell <= D; ++ell) {
      const Bonds& tb = top.snap[D - ell];
      const Bonds& bb = bot.snap[ell - 1];
      for (int c = 0; c <= n; ++c) {
        o_L[ell][c] = take((size_t)tb.p[c] * bb.p[c] * C);
        o_R[ell][c] = take((size_t)tb.p[c] * bb.p[c] * C);
      }
    }
    arena_bytes = o;
  }

  // Fresh device status word for one cuSOLVER call; fold it into `acc` afterwards.
  int* call_info(Pool& pool, cudaStream_t st) {
    int* p = (int*)pool.raw(sizeof(int));
    TN_CUDA(cudaMemsetAsync(p, 0, sizeof(int), st));
    return p;
  }

  CUgreenCtx green_ctx[2] = {nullptr, nullptr};
  // Driver entry points through the runtime (the library does not link libcuda:
  // it must load on a machine without a driver for the ABI tests).
  template <class F>
  static F driver_fn(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &qr) != cudaSuccess || qr != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return reinterpret_cast<F>(fn);
  }
  void destroy_green() {
    auto destroy = driver_fn<CUresult (*)(CUgreenCtx)>("cuGreenCtxDestroy");
    for (CUgreenCtx& g : green_ctx) {
      if (g && destroy) destroy(g);
      g = nullptr;
    }
  }
  // st1 / st2 in two disjoint SM partitions of half the device each.
  bool make_green_streams(int prio) {
    auto dev_get = driver_fn<CUresult (*)(CUdevice*, int)>("cuDeviceGet");
    auto get_res = driver_fn<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>("cuDeviceGetDevResource");
    auto split = driver_fn<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned,
                                        unsigned)>("cuDevSmResourceSplitByCount");
    auto gen_desc = driver_fn<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>("cuDevResourceGenerateDesc");
    auto ctx_create = driver_fn<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>("cuGreenCtxCreate");
    auto stream_create = driver_fn<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>("cuGreenCtxStreamCreate");
    if (!dev_get || !get_res || !split || !gen_desc || !ctx_create || !stream_create) return false;
    CUdevice dev;
    CUdevResource all, parts[2], rem;
    unsigned ng = 2;
    if (dev_get(&dev, device) != CUDA_SUCCESS) return false;
    if (get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return false;
    const unsigned half = (all.sm.smCount / 2) / 8 * 8;  // sm_90+: partitions are multiples of 8 SMs
    if (half < 8) return false;
    if (split(parts, &ng, &all, &rem, 0, half) != CUDA_SUCCESS || ng < 2) return false;
    cudaStream_t out[2] = {nullptr, nullptr};
    for (int i = 0; i < 2; ++i) {
      CUdevResourceDesc d;
      CUstream s = nullptr;
      if (gen_desc(&d, &parts[i], 1) != CUDA_SUCCESS ||
          ctx_create(&green_ctx[i], d, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
          stream_create(&s, green_ctx[i], CU_STREAM_NON_BLOCKING, prio) != CUDA_SUCCESS) {
        for (cudaStream_t x : out)
          if (x) cudaStreamDestroy(x);
        destroy_green();
        return false;
      }
      out[i] = (cudaStream_t)s;
    }
    st1 = out[0];
    st2 = out[1];
    return true;
  }

  // ------------------------------------------------------------ setup --
  // Host-only plan: layers, both sides' step lists with their static bond
  // profiles (a2/a3 keep rule, X7), and the primal-arena layout.
  void plan(const tn_hvp_config& c, const int32_t* rb) {
    cfg = c;
    P = c.site_dim == 2 ? 2 : 4;
    NI = P / 2;
    PP = P * P;
    NI2 = NI * NI;
    n = c.n_sites;
    D = c.depth;
    off = c.first_offset;
    chi = c.chi;
    device = c.device;
    build_layers();
    ref_bonds.assign(rb, rb + n + 1);
    std::vector<int> ones(n + 1, 1);
    n_pair_steps = 0;
    plan_side(bot, ones, false);
    plan_side(top, ref_bonds, true);
    layout_arena();
  }

  // Bytes of one direction's tangent state: the cached forward tangent blocks
  // of every bottom snapshot plus the live backward tangent's blocks.
  size_t per_direction_bytes() const {
    size_t e = 0;
    for (size_t li = 0; li + 1 < bot.snap.size(); ++li)
      for (int s = 0; s < n; ++s) e += (size_t)bsize(bot.snap[li], s);
    size_t mx = 0;
    for (const Bonds& b : top.snap) {
      size_t t = 0;
      for (int s = 0; s < n; ++s) t += (size_t)bsize(b, s);
      mx = std::max(mx, t);
    }
    return (e + mx) * sizeof(cplx);
  }

  size_t chain_cache_bytes() const {
    return sizeof(cplx) * (size_t)(chain_cache_elems(bot) + chain_cache_elems(top));
  }

  // primal_buf: caller-owned DEVICE buffer of at least arena_bytes (nullptr:
  // the context allocates and owns it).
  void setup(const tn_hvp_config& c, const int32_t* rb, const void* ref_mpo, void* primal_buf, size_t primal_bytes,
             cudaStream_t st) {
    plan(c, rb);
    if (primal_buf && primal_bytes < arena_bytes)
      throw std::invalid_argument("tn_hvp_setup: primal_buf smaller than tn_hvp_query's primal_bytes (" +
                                  std::to_string(primal_bytes) + " < " + std::to_string(arena_bytes) + ")");
    if (reinterpret_cast<uintptr_t>(primal_buf) % 256 != 0)
      throw std::invalid_argument("tn_hvp_setup: primal_buf must be 256-byte aligned");
    TN_CUDA(cudaSetDevice(device));
    {
      std::vector<int> lo, ls(1, 0);
      for (int ell = 1; ell <= D; ++ell) {
        for (size_t j = 0; j < layers[ell - 1].size(); ++j) lo.push_back(ell - 1);
        ls.push_back((int)lo.size());
      }
      TN_CUDA(cudaMalloc(&d_layer_of, sizeof(int) * std::max<size_t>(lo.size(), 1)));
      TN_CUDA(cudaMalloc(&d_layer_start, sizeof(int) * ls.size()));
      TN_CUDA(cudaMalloc(&ti_buf, sizeof(cplx) * 3 * 16 * std::max(D, 1)));
      if (!lo.empty()) TN_CUDA(cudaMemcpy(d_layer_of, lo.data(), sizeof(int) * lo.size(), cudaMemcpyHostToDevice));
      TN_CUDA(cudaMemcpy(d_layer_start, ls.data(), sizeof(int) * ls.size(), cudaMemcpyHostToDevice));
    }
    {  // bottom start: operator mode delta_{oi}/sqrt 2 per site; state mode |0> (tn_hvp_set_product_state)
      std::vector<cplx> h((size_t)n * P, ZERO);
      const double r2 = 1.0 / std::sqrt(2.0);
      for (int s = 0; s < n; ++s) {
        if (P == 4) {
          h[(size_t)s * 4] = {r2, 0.0};
          h[(size_t)s * 4 + 3] = {r2, 0.0};
        } else {
          h[(size_t)s * 2] = ONE;
        }
      }
      TN_CUDA(cudaMalloc(&d_init, sizeof(cplx) * h.size()));
      TN_CUDA(cudaMemcpy(d_init, h.data(), sizeof(cplx) * h.size(), cudaMemcpyHostToDevice));
    }
    if (primal_buf) {
      arena = static_cast<char*>(primal_buf);
      own_arena = false;
    } else {
      TN_CUDA(cudaMalloc(&arena, std::max<size_t>(arena_bytes, 256)));
      own_arena = true;
    }
    if (g_poison) TN_CUDA(cudaMemsetAsync(arena, 0xFF, std::max<size_t>(arena_bytes, 256), st));
    // reference copy
    ref_off.assign(n, 0);
    size_t e = 0;
    for (int s = 0; s < n; ++s) {
      ref_off[s] = e;
      e += (size_t)ref_bonds[s] * P * ref_bonds[s + 1];
    }
    TN_CUDA(cudaMalloc(&ref, e * sizeof(cplx)));
    TN_CUDA(cudaMemcpyAsync(ref, ref_mpo, e * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    {  // range-probe test matrix and per-step hints (lowrank_split)
      int np = 0;
      for (SidePlan* sp : {&bot, &top})
        for (auto& ls : sp->steps)
          for (Step& x : ls)
            if (x.type == PAIR) {
              om_rows = std::max(om_rows, P * x.br);
              om_cols = std::max(om_cols, x.r);
              np = std::max(np, x.s_index + 1);
            }
      lowrank_hint.assign(np, 1);
      if (lowrank_on && om_rows > 0) {
        TN_CUDA(cudaMalloc(&d_omega, (size_t)om_rows * om_cols * sizeof(cplx)));
        fill_test_matrix(st, d_omega, (int64_t)om_rows * om_cols, 0x7AD5B200ULL);
      }
    }
    // Stream priorities: the two primal sweeps are latency-bound chains (the
    // critical path of a step), the layer environments and the fused step's
    // forward tangents are throughput work that fills in behind them.
    int prio_lo = 0, prio_hi = 0;
    TN_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    const bool use_prio = std::getenv("TN_NO_STREAM_PRIO") == nullptr;
    auto mkstream = [&](cudaStream_t* s, int level) {  // level 0 = highest
      const int pr = use_prio ? (int)std::min<int64_t>(prio_lo, (int64_t)prio_hi + level) : prio_lo;
      TN_CUDA(cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, pr));
    };
    // SM partitions for the two sweeps (CUDA green contexts): cuSOLVER's
    // tridiagonalisation kernels take the whole GPU, so two eigensolves on
    // plain streams run one after the other (Zheevd 512: 10.4 ms for two vs
    // 5.9 ms for one); on disjoint halves of the SMs two n <= 512 solves
    // overlap (7.9 ms for two, 6.7 ms for one: tools/green_probe.cu).  The
    // n = 1024 solves of chi = 256 serialise in any case (30.5 ms for two), so
    // partitions are used only when every Gram matrix is <= 512 wide.  Any
    // failure here falls back to plain streams.
    bool green = false;
    {
      int max_gram = 0;
      for (SidePlan* sp : {&bot, &top})
        for (auto& ls : sp->steps)
          for (Step& x : ls)
            if (x.type == PAIR) max_gram = std::max(max_gram, P * x.bl);
      if (std::getenv("TN_NO_GREEN_CTX") == nullptr && max_gram > 64 && max_gram <= 512) green = make_green_streams(prio_hi);
    }
    if (!green) {
      mkstream(&st2, 0);
      mkstream(&st1, 0);
    }
    TN_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    TN_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    TN_CUDA(cudaEventCreateWithFlags(&ev_join1, cudaEventDisableTiming));
    mkstream(&stg, 1);
    mkstream(&stf, 1 << 20);  // lowest (the default priority, like the caller's stream)
    mkstream(&stc, 1 << 20);
    mkstream(&sth, 1 << 20);
    TN_CUDA(cudaEventCreateWithFlags(&ev_joinf, cudaEventDisableTiming));
    TN_CUDA(cudaEventCreateWithFlags(&ev_joing, cudaEventDisableTiming));
    for (auto& v : ev_snap) {
      v.assign(D + 1, nullptr);
      for (auto& e : v) TN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (Solver& so : sol) {
      TN_SOLVER(cusolverDnCreate(&so.h));
      TN_SOLVER(cusolverDnCreateParams(&so.prm));
    }
    Solver& so = sol[0];
    TN_SOLVER(cusolverDnSetStream(so.h, st));
    for (SidePlan* sp : {&bot, &top})
      for (auto& ls : sp->steps)
        for (Step& s : ls) {
          if (s.type == PAIR) {
            const int mr = std::max(P * s.bl, P * s.br), nc_ = std::min(P * s.bl, P * s.br);
            {
              int lw = 0;
              TN_SOLVER(cusolverDnZheevd_bufferSize(so.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, P * s.bl,
                                                    nullptr, P * s.bl, nullptr, &lw));
              lwork_heevd = std::max(lwork_heevd, lw);
            }
            {  // QR-iteration SVD workspace (fallback of the Gram split)
              size_t d2 = 0, h2 = 0;
              TN_SOLVER(cusolverDnXgesvd_bufferSize(so.h, so.prm, 'S', 'S', mr, nc_, CUDA_C_64F, nullptr, mr,
                                                    CUDA_R_64F, nullptr, CUDA_C_64F, nullptr, mr, CUDA_C_64F, nullptr,
                                                    nc_, CUDA_C_64F, &d2, &h2));
              svd_dws = std::max(svd_dws, d2);
              svd_hws = std::max(svd_hws, h2);
            }
            int lw = 0;  // LQ of Y (r x 4br): geqrf on the column-major (4br x r) view
            TN_SOLVER(cusolverDnZgeqrf_bufferSize(so.h, P * s.br, s.r, nullptr, P * s.br, &lw));
            lwork_geqrf = std::max(lwork_geqrf, lw);
            TN_SOLVER(cusolverDnZungqr_bufferSize(so.h, P * s.br, s.r, s.r, nullptr, P * s.br, nullptr, &lw));
            lwork_ungqr = std::max(lwork_ungqr, lw);
          } else {
            const int mr = s.type == MOVE_R ? P * s.b : P * s.bp;
            const int nc_ = s.type == MOVE_R ? s.bp : s.b;
            int lw = 0;
            TN_SOLVER(cusolverDnZgeqrf_bufferSize(so.h, mr, nc_, nullptr, mr, &lw));
            lwork_geqrf = std::max(lwork_geqrf, lw);
            TN_SOLVER(cusolverDnZungqr_bufferSize(so.h, mr, s.kq, s.kq, nullptr, mr, nullptr, &lw));
            lwork_ungqr = std::max(lwork_ungqr, lw);
          }
        }
    for (Solver& x : sol) x.host_ws.assign(svd_hws + 64, 0);
  }

  // The caller has synchronised the streams it used with this context
  // (tn_hvp_destroy contract); the engine drains its own streams.
  ~Engine() {
    if (!st1) {  // never set up (tn_hvp_query, or setup failed early)
      if (d_init) cudaFree(d_init);
      if (d_layer_of) cudaFree(d_layer_of);
      if (d_layer_start) cudaFree(d_layer_start);
      if (ti_buf) cudaFree(ti_buf);
      if (arena && own_arena) cudaFree(arena);
      if (ref) cudaFree(ref);
      if (d_omega) cudaFree(d_omega);
      return;
    }
    for (cudaStream_t x : {st1, st2, stg, stf, sth, stc})
      if (x) cudaStreamSynchronize(x);
    drop_graphs(stc, true);
    drop_chain_cache(stc);
    cudaStreamSynchronize(stc);
    if (d_init) cudaFree(d_init);
    if (d_layer_of) cudaFree(d_layer_of);
    if (d_layer_start) cudaFree(d_layer_start);
    if (ti_buf) cudaFree(ti_buf);
    for (Solver& so : sol) {
      if (so.prm) cusolverDnDestroyParams(so.prm);
      if (so.h) cusolverDnDestroy(so.h);
      if (so.bl) cublasDestroy(so.bl);
    }
    for (cudaEvent_t e : {ev_fork, ev_join, ev_join1, ev_joing, ev_joinf})
      if (e) cudaEventDestroy(e);
    for (auto& v : ev_snap)
      for (auto& e : v)
        if (e) cudaEventDestroy(e);
    for (cudaStream_t x : {st1, st2, stg, stf, sth, stc})
      if (x) cudaStreamDestroy(x);
    destroy_green();
    if (arena && own_arena) cudaFree(arena);
    if (ref) cudaFree(ref);
    if (d_omega) cudaFree(d_omega);
    pool_trim(device);
    cudaDeviceGraphMemTrim(device);
  }

  // ------------------------------------------- N4: reference construction --
  // TEBD of a gate sequence on the operator I/2^{n/2} with the primal pass's
  // own kernels (reading X11): gates on the OUT legs, the
  // centre moved by QR / LQ, every two-site split through the Gram
  // eigendecomposition (DMMA GEMM + heevd), keep r = min(chi, #{sigma_j >
  // tol sigma_1}) (tol >= 1e-7: the Gram split resolves sigma to ~1e-8 sigma_1),
  // U_r^H A rescaled to the pre-truncation norm; finally right-canonical with
  // the centre at site 0 and unit Frobenius norm.  Data-dependent shapes: the
  // split sizes are read on the host (one stream synchronisation per gate).
  // out: DEVICE, capacity cap complex elements; bonds: n+1 on return.
  void tebd(cudaStream_t st, int nn_, int ngates, const int32_t* gsite, const cplx* G, int chi_, double tol,
            std::vector<int>& bonds, cplx* out, size_t cap) {
    n = nn_;
    chi = chi_;
    TN_CUDA(cudaSetDevice(device));
    Solver& so = sol[0];
    TN_SOLVER(cusolverDnCreate(&so.h));
    TN_SOLVER(cusolverDnSetStream(so.h, st));
    {
      const int R = 4 * chi;  // largest two-site row / column count
      TN_SOLVER(cusolverDnZheevd_bufferSize(so.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, R, nullptr, R,
                                            nullptr, &lwork_heevd));
      TN_SOLVER(cusolverDnZgeqrf_bufferSize(so.h, R, R, nullptr, R, &lwork_geqrf));
      TN_SOLVER(cusolverDnZungqr_bufferSize(so.h, R, R, R, nullptr, R, nullptr, &lwork_ungqr));
    }
    const double tolg = std::max(tol, 1e-7);
    std::vector<cplx*> a(n, nullptr);
    bonds.assign(n + 1, 1);
    const double h = 1.0 / std::sqrt(2.0);
    for (int s = 0; s < n; ++s) {
      a[s] = dnew(4, st);
      set_small(st, a[s], 4, {h, 0.0}, ZERO, ZERO, {h, 0.0});
    }
    Pool keep_alive(st);
    int* info = (int*)keep_alive.raw(sizeof(int));
    TN_CUDA(cudaMemsetAsync(info, 0, sizeof(int), st));
    int c = 0;
    auto move_right = [&]() {
      Pool tmp(st);
      const int b = bonds[c], bp = bonds[c + 1], kq = std::min(4 * b, bp), nb2 = bonds[c + 2];
      cplx* Q = dnew((int64_t)4 * b * kq, st);
      cplx* Rm = tmp.c((int64_t)kq * bp);
      qr_right(st, so, tmp, a[c], 4 * b, bp, kq, Q, Rm, info);
      cplx* nx = dnew((int64_t)kq * 4 * nb2, st);
      nn(st, kq, 4 * nb2, bp, Rm, 0, a[c + 1], 0, nx, 0, 1);
      dset(a[c], Q, st);
      dset(a[c + 1], nx, st);
      bonds[c + 1] = kq;
      ++c;
    };
    auto move_left = [&]() {
      Pool tmp(st);
      const int b = bonds[c], bp = bonds[c + 1], kq = std::min(b, 4 * bp), nb2 = bonds[c - 1];
      cplx* Q = dnew((int64_t)kq * 4 * bp, st);
      cplx* L = tmp.c((int64_t)b * kq);
      lq_left(st, so, tmp, a[c], b, 4 * bp, kq, Q, L, info);
      cplx* nx = dnew((int64_t)nb2 * 4 * kq, st);
      nn(st, nb2 * 4, kq, b, a[c - 1], 0, L, 0, nx, 0, 1);
      dset(a[c], Q, st);
      dset(a[c - 1], nx, st);
      bonds[c] = kq;
      --c;
    };
    for (int g = 0; g < ngates; ++g) {
      const int i = gsite[g];
      if (i < 0 || i + 1 >= n) throw std::invalid_argument("tn_mpo_tebd: gate site out of range");
      while (c < i) move_right();
      while (c > i) move_left();
      Pool tmp(st);
      const int bl = bonds[i], m = bonds[i + 1], br = bonds[i + 2], R = 4 * bl, Cc = 4 * br;
      cplx* th = tmp.c((int64_t)R * Cc);
      nn(st, R, Cc, m, a[i], 0, a[i + 1], 0, th, 0, 1);
      cplx* A = tmp.c((int64_t)R * Cc);
      apply_gate(st, A, 0, th, 0, G + (int64_t)g * 16, 0, bl, br, 1, ONE, false, 2);
      double* nrm = (double*)tmp.raw(2 * sizeof(double));
      tangent_dot(st, (int64_t)R * Cc, 1, A, A, nrm);
      cplx* uhf = tmp.c((int64_t)R * R);
      double* S = (double*)tmp.raw((size_t)R * sizeof(double));
      cplx* Acp = tmp.c((int64_t)R * Cc);
      TN_CUDA(cudaMemcpyAsync(Acp, A, (size_t)R * Cc * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      svd_rowmajor(st, so, tmp, Acp, R, Cc, S, uhf, info, kGram);
      std::vector<double> hS(R);
      TN_CUDA(cudaMemcpyAsync(hS.data(), S, R * sizeof(double), cudaMemcpyDeviceToHost, st));
      TN_CUDA(cudaStreamSynchronize(st));
      int r = 0;
      while (r < R && hS[r] > tolg * hS[0]) ++r;
      r = std::max(1, std::min(chi, r));
      // kept-subspace refinement across the cut (as in the primal pass): the
      // Gram basis mixes kept and discarded directions by ~eps s_1^2 / gap
      refine_kept(st, tmp, uhf, S, A, R, Cc, R, r, 2);
      cplx* ni = dnew((int64_t)R * r, st);
      conjT_scale_cols(st, ni, uhf, r, R, nullptr, nullptr);       // U_r (4bl x r)
      cplx* nj = dnew((int64_t)r * Cc, st);
      nn(st, r, Cc, R, uhf, 0, A, 0, nj, 0, 1);                     // U_r^H A
      tangent_dot(st, (int64_t)r * Cc, 1, nj, nj, nrm + 1);
      scale_by_norm_ratio(st, nj, nrm, (int64_t)r * Cc);            // x sqrt(nrm[0] / nrm[1])
      dset(a[i], ni, st);
      dset(a[i + 1], nj, st);
      bonds[i + 1] = r;
      c = i + 1;
    }
    while (c > 0) move_left();
    {  // unit Frobenius norm (site 0 is the centre)
      Pool tmp(st);
      double* nrm = (double*)tmp.raw(2 * sizeof(double));
      const int64_t e0 = (int64_t)4 * bonds[1];
      set_small(st, reinterpret_cast<cplx*>(nrm), 1, ONE);   // nrm[0] = 1
      tangent_dot(st, e0, 1, a[0], a[0], nrm + 1);
      scale_by_norm_ratio(st, a[0], nrm, e0);
      TN_CUDA(cudaStreamSynchronize(st));
    }
    size_t tot = 0;
    for (int s = 0; s < n; ++s) tot += (size_t)bonds[s] * 4 * bonds[s + 1];
    if (tot > cap) throw std::invalid_argument("tn_mpo_tebd: output capacity " + std::to_string(cap) +
                                               " < " + std::to_string(tot) + " elements");
    size_t o = 0;
    for (int s = 0; s < n; ++s) {
      const size_t e = (size_t)bonds[s] * 4 * bonds[s + 1];
      TN_CUDA(cudaMemcpyAsync(out + o, a[s], e * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      o += e;
      ddel(a[s], st);
    }
    int hinfo = 0;
    TN_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    if (hinfo) throw NumericError("tn_mpo_tebd: cuSOLVER info nonzero");
  }

  // ------------------------------------------------------ primal pass --
  struct Mps {  // current site tensors (pool-owned)
    std::vector<cplx*> a;
    std::vector<int> b;  // bonds
  };

  // CholeskyQR2 of a row-major P (rows x cols): two passes of Gram matrix (DMMA
  // GEMM) -> potrf -> triangular solve instead of a Householder panel
  // factorisation (geqr2 is one latency-bound CTA: 1.5 ms for 1024 x 256).
  //   right: rows >= cols, P = Q R, Q (rows x cols) column-orthonormal, T = R (cols x cols) upper;
  //   left : rows <= cols, P = L Q, Q (rows x cols) row-orthonormal,    T = L (rows x rows) lower.
  // Orthonormal to rounding when cond(P)^2 eps << 1.  Returns false when a Gram
  // matrix is not numerically positive definite or the second pass is not a
  // small correction (|T_2 - I| > 0.1): the caller falls back to Householder.
  // One host read of the flag per call (the sweeps already return to the host per split).
  bool cholqr2(cudaStream_t st, Solver& so, Pool& pool, const cplx* Pm, int rows, int cols, bool right, cplx* Q,
               cplx* T) {
    const int n = right ? cols : rows;
    if (!so.bl) {
      if (cublasCreate(&so.bl) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasCreate failed");
    }
    if (cublasSetStream(so.bl, st) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream failed");
    TN_SOLVER(cusolverDnSetStream(so.h, st));
    const cublasFillMode_t uplo = right ? CUBLAS_FILL_MODE_LOWER : CUBLAS_FILL_MODE_UPPER;  // of the column-major view
    int lw = 0;
    TN_SOLVER(cusolverDnZpotrf_bufferSize(so.h, uplo, n, nullptr, n, &lw));
    cplx* work = pool.c(std::max(lw, 1));
    cplx* Gm[2] = {pool.c((int64_t)n * n), pool.c((int64_t)n * n)};
    int* flag = (int*)pool.raw(sizeof(int));
    TN_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    TN_CUDA(cudaMemcpyAsync(Q, Pm, (size_t)rows * cols * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
    for (int pass = 0; pass < 2; ++pass) {
      cplx* G = Gm[pass];
      if (right)
        cn(st, n, n, rows, Q, 0, Q, 0, G, 0, 1);  // Q^H Q
      else
        nc(st, n, n, cols, Q, 0, Q, 0, G, 0, 1);  // Q Q^H
      int* ci = call_info(pool, st);
      // the row-major Hermitian G read column-major is conj(G): its Cholesky factor
      // read back row-major is the upper R with G = R^H R (right) / the lower L with G = L L^H (left)
      TN_SOLVER(cusolverDnZpotrf(so.h, uplo, n, (cuDoubleComplex*)G, n, (cuDoubleComplex*)work, lw, ci));
      // Q <- Q R^{-1} (right) / L^{-1} Q (left), on the column-major view Q^T (cols x rows)
      const cublasStatus_t bs =
          right ? cublasZtrsm(so.bl, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, cols,
                              rows, &one, (const cuDoubleComplex*)G, n, (cuDoubleComplex*)Q, cols)
                : cublasZtrsm(so.bl, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, cols,
                              rows, &one, (const cuDoubleComplex*)G, n, (cuDoubleComplex*)Q, cols);
      if (bs != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasZtrsm status " + std::to_string((int)bs));
      tri_keep(st, G, n, right);
      chol_flag(st, G, n, right, ci, pass == 1, 0.1, flag);
    }
    if (right)
      nn(st, n, n, n, Gm[1], 0, Gm[0], 0, T, 0, 1);  // R = R2 R1
    else
      nn(st, n, n, n, Gm[0], 0, Gm[1], 0, T, 0, 1);  // L = L1 L2
    int hflag = 0;
    TN_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    if (hflag) ++n_cholqr_fallback;
    return hflag == 0;
  }

  void qr_right(cudaStream_t st, Solver& so, Pool& pool, const cplx* P, int rows, int cols, int kq, cplx* Q, cplx* R,
                int* info, bool allow_chol = true) {
    // P row-major rows x cols -> Q (rows x kq) row-major, R (kq x cols) row-major
    if (cholqr && allow_chol && kq == cols && rows >= cols && cols >= kCholMin &&
        cholqr2(st, so, pool, P, rows, cols, true, Q, R))
      return;
    cplx* cm = pool.c((int64_t)rows * cols);
    transpose(st, cm, P, rows, cols, false);  // column-major rows x cols
    cplx* tau = pool.c(std::min(rows, cols));
    cplx* work = pool.c(std::max(lwork_geqrf, lwork_ungqr));
    TN_SOLVER(cusolverDnSetStream(so.h, st));
    int* ci = call_info(pool, st);
    TN_SOLVER(cusolverDnZgeqrf(so.h, rows, cols, (cuDoubleComplex*)cm, rows, (cuDoubleComplex*)tau,
                               (cuDoubleComplex*)work, lwork_geqrf, ci));
    info_accum(st, info, ci);
    tri_extract(st, R, cm, kq, cols, rows, true);
    TN_SOLVER(cusolverDnZungqr(so.h, rows, kq, kq, (cuDoubleComplex*)cm, rows, (cuDoubleComplex*)tau,
                               (cuDoubleComplex*)work, lwork_ungqr, ci));
    info_accum(st, info, ci);
    transpose(st, Q, cm, kq, rows, false);  // cm is (kq x rows) row-major -> Q rows x kq
  }

  void lq_left(cudaStream_t st, Solver& so, Pool& pool, const cplx* P, int rows, int cols, int kq, cplx* Q, cplx* L,
               int* info, bool allow_chol = true) {
    // P row-major rows x cols = L (rows x kq) Q (kq x cols), Q row-orthonormal
    if (cholqr && allow_chol && kq == rows && cols >= rows && rows >= kCholMin &&
        cholqr2(st, so, pool, P, rows, cols, false, Q, L))
      return;
    cplx* cm = pool.c((int64_t)rows * cols);
    TN_CUDA(cudaMemcpyAsync(cm, P, (size_t)rows * cols * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    cplx* tau = pool.c(std::min(rows, cols));
    cplx* work = pool.c(std::max(lwork_geqrf, lwork_ungqr));
    TN_SOLVER(cusolverDnSetStream(so.h, st));
    int* ci = call_info(pool, st);
    // column-major view: cols x rows matrix P^T
    TN_SOLVER(cusolverDnZgeqrf(so.h, cols, rows, (cuDoubleComplex*)cm, cols, (cuDoubleComplex*)tau,
                               (cuDoubleComplex*)work, lwork_geqrf, ci));
    info_accum(st, info, ci);
    tri_extract(st, L, cm, rows, kq, cols, false);
    TN_SOLVER(cusolverDnZungqr(so.h, cols, kq, kq, (cuDoubleComplex*)cm, cols, (cuDoubleComplex*)tau,
                               (cuDoubleComplex*)work, lwork_ungqr, ci));
    info_accum(st, info, ci);
    TN_CUDA(cudaMemcpyAsync(Q, cm, (size_t)kq * cols * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
  }

  // SVD of a row-major (R x Cc) matrix A (destroyed): singular values S (mn =
  // min(R, Cc), descending) and the full left basis uhf = U^H (mn x R row-major).
  // method kGram: eigendecomposition of A A^H (R x R, all R left vectors);
  // kQRIter: QR-iteration SVD (the fallback for unresolved cuts).
  static constexpr int kQRIter = 2, kGram = 3;
  void svd_rowmajor(cudaStream_t st, Solver& so, Pool& pool, cplx* A, int R, int Cc, double* S, cplx* uhf,
                    int* info, int method) {
    if (method == kGram) {
      // Gram split: G = A A^H (R x R), heevd -> all R left vectors (zeros beyond min(R, Cc))
      cplx* Gm = pool.c((int64_t)R * R);
      nc(st, R, R, Cc, A, 0, A, 0, Gm, 0, 1);
      double* lam = (double*)pool.raw((size_t)R * sizeof(double));
      cplx* work = pool.c(std::max(lwork_heevd, 1));
      TN_SOLVER(cusolverDnSetStream(so.h, st));
      int* ci = call_info(pool, st);
      TN_SOLVER(cusolverDnZheevd(so.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, R, (cuDoubleComplex*)Gm, R,
                                 lam, (cuDoubleComplex*)work, lwork_heevd, ci));
      info_accum(st, info, ci);
      eig_to_svd(st, uhf, S, Gm, lam, R);
      return;
    }
    const bool tr = Cc >= R;  // column-major view of A is A^T (Cc x R): use it directly when Cc >= R
    cplx* M = A;
    int m = Cc, nn_ = R;
    if (!tr) {
      M = pool.c((int64_t)R * Cc);
      transpose(st, M, A, R, Cc, false);  // column-major R x Cc = A
      m = R;
      nn_ = Cc;
    }
    const int mn = nn_;
    cplx* Up = pool.c((int64_t)m * mn);
    cplx* Vp = pool.c((int64_t)nn_ * mn);
    void* dws = pool.raw(svd_dws + 64);
    TN_SOLVER(cusolverDnSetStream(so.h, st));
    int* ci = call_info(pool, st);
    {  // QR-iteration SVD (LAPACK-like accuracy); Xgesvd returns V^H (mn x nn_, ldvt = mn) in Vp
      TN_SOLVER(cusolverDnXgesvd(so.h, so.prm, 'S', 'S', m, nn_, CUDA_C_64F, M, m, CUDA_R_64F, S, CUDA_C_64F, Up, m,
                                 CUDA_C_64F, Vp, mn, CUDA_C_64F, dws, svd_dws, so.host_ws.data(), svd_hws, ci));
      cplx* V = pool.c((int64_t)nn_ * mn);
      transpose(st, V, Vp, nn_, mn, true);
      Vp = V;
    }
    info_accum(st, info, ci);
    // column-major M = Up S Vp^H
    if (tr)  // M = A^T -> A = conj(Vp) S Up^T: U_A^H = Vp^T (row-major view of Vp)
      TN_CUDA(cudaMemcpyAsync(uhf, Vp, (size_t)mn * R * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    else     // M = A -> U_A^H = conj(Up)^T
      conj_copy(st, uhf, Up, (int64_t)mn * R);
  }

  // Range probe for a two-site block A (R x Cc) whose numerical rank does not
  // exceed the kept rank r (low-entanglement states: Trotter-initialised
  // circuits, the trust-region regime of config 5): Q = orth(A Omega) with a
  // fixed Cc x r test matrix (Householder QR; A Omega is ill-conditioned) and
  // the residual ||A - Q Q^H A||_F measured explicitly.  If it is below
  // kLowRankTol ||A||_F the truncation to ANY r-dimensional subspace containing
  // range(Q) discards nothing above the noise floor -- the oracle's top-r
  // singular subspace is range(A) plus noise-floor directions to which the
  // outputs are insensitive (reading X10) -- so U_r^H = Q^H without an
  // eigendecomposition (one 1.7 ms panel QR instead of 1 + up to 3 Gram levels of
  // 13 ms each).  Returns false (uh untouched) when the residual test fails.
  static constexpr double kLowRankTol = 1e-13;
  bool lowrank_split(cudaStream_t st, Solver& so, Pool& pool, const cplx* A, int R, int Cc, int r, cplx* uh, int* info) {
    cplx* Yr = pool.c((int64_t)R * r);
    mm(st, 'N', 'N', R, r, Cc, ONE, A, Cc, 0, d_omega, om_cols, 0, ZERO, Yr, r, 0, 1);
    cplx* Qm = pool.c((int64_t)R * r);
    cplx* Rq = pool.c((int64_t)r * r);
    qr_right(st, so, pool, Yr, R, r, r, Qm, Rq, info, /*allow_chol=*/false);
    cplx* uht = pool.c((int64_t)r * R);
    transpose(st, uht, Qm, R, r, true);  // Q^H (r x R)
    cplx* Bq = pool.c((int64_t)r * Cc);
    nn(st, r, Cc, R, uht, 0, A, 0, Bq, 0, 1);
    cplx* Res = pool.c((int64_t)R * Cc);
    TN_CUDA(cudaMemcpyAsync(Res, A, (size_t)R * Cc * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    nn(st, R, Cc, r, Qm, 0, Bq, 0, Res, 0, 1, MONE, ONE);
    double* nrm = (double*)pool.raw(2 * sizeof(double));
    tangent_dot(st, (int64_t)R * Cc, 1, A, A, nrm);
    tangent_dot(st, (int64_t)R * Cc, 1, Res, Res, nrm + 1);
    double h[2] = {0, 0};
    TN_CUDA(cudaMemcpyAsync(h, nrm, sizeof(h), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    if (!(h[1] <= kLowRankTol * kLowRankTol * h[0])) return false;
    TN_CUDA(cudaMemcpyAsync(uh, uht, (size_t)r * R * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    return true;
  }

  // Kept left subspace refinement (SVD-method independent, relative accuracy):
  // with B = U^H A, make the kept rows orthogonal to the discarded rows by the
  // first-order rotation c_ij = (B_i B_j^H) / (s_j^2 - s_i^2) (one-sided Jacobi
  // across the cut), twice, then Loewdin re-orthonormalisation of the kept rows.
  void refine_kept(cudaStream_t st, Pool& pool, cplx* uhf, const double* S, const cplx* A, int R, int Cc, int mn,
                   int r, int iters, bool kept_only = false) {
    const int nd = mn - r;
    if (nd <= 0 || iters <= 0) return;
    cplx* B = pool.c((int64_t)mn * Cc);
    cplx* Md = pool.c((int64_t)nd * r);
    cplx* Cm = pool.c((int64_t)nd * r);
    cplx* old = pool.c((int64_t)mn * R);
    for (int it = 0; it < iters; ++it) {
      nn(st, mn, Cc, R, uhf, 0, A, 0, B, 0, 1);
      nc(st, nd, r, Cc, B + (int64_t)r * Cc, 0, B, 0, Md, 0, 1);
      kept_rotation(st, Cm, Md, S, nd, r);
      TN_CUDA(cudaMemcpyAsync(old, uhf, (size_t)r * R * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      cn(st, r, R, nd, Cm, 0, uhf + (int64_t)r * R, 0, uhf, 0, 1, ONE, ONE);      // kept += C^H disc
      nn(st, nd, R, r, Cm, 0, old, 0, uhf + (int64_t)r * R, 0, 1, MONE, ONE);    // disc -= C kept_old
    }
    // Loewdin re-orthonormalisation U <- (3/2 - 1/2 U U^H) U of the whole basis, or
    // (kept_only: the caller uses nothing but the kept rows afterwards) of the
    // kept rows among themselves
    const int no = kept_only ? r : mn;
    cplx* F = pool.c((int64_t)no * no);
    nc(st, no, no, R, uhf, 0, uhf, 0, F, 0, 1);
    TN_CUDA(cudaMemcpyAsync(old, uhf, (size_t)no * R * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    nn(st, no, R, no, F, 0, old, 0, uhf, 0, 1, {-0.5, 0.0}, {1.5, 0.0});
  }

  // W^H = row-orthonormal basis of the rows of Y (r x Cc), L = Y W (r x r), for
  // Y = U_r^H A whose rows are mutually orthogonal up to the eigensolver's
  // residual, <y_i, y_j> ~ eps sigma_1^2, with norms sigma_i (S, device): the
  // row-scaled Yt = diag(1/sigma) Y has Yt Yt^H = I + O(eps (sigma_1/sigma_r)^2),
  // so `steps` Newton-Schulz (Loewdin) steps Yt <- (3/2 - 1/2 Yt Yt^H) Yt (error e
  // -> 3/2 e^2) orthonormalise it with GEMMs only -- no panel factorisation.
  // Same row space as the LQ factor, another r x r gauge (outputs are invariant).
  void lq_rows_lowdin(cudaStream_t st, Pool& pool, const cplx* Y, const double* S, int r, int Cc, int steps, cplx* Wh,
                      cplx* L) {
    rows_over_s(st, Wh, Y, S, r, Cc);
    cplx* F = pool.c((int64_t)r * r);
    cplx* old = pool.c((int64_t)r * Cc);
    for (int it = 0; it < steps; ++it) {
      nc(st, r, r, Cc, Wh, 0, Wh, 0, F, 0, 1);
      TN_CUDA(cudaMemcpyAsync(old, Wh, (size_t)r * Cc * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      nn(st, r, Cc, r, F, 0, old, 0, Wh, 0, 1, {-0.5, 0.0}, {1.5, 0.0});
    }
    nc(st, r, r, Cc, Y, 0, Wh, 0, L, 0, 1);
  }

  // Second Gram level for the low part of the spectrum: rows n_hi.. of uhf
  // (already split from the high part by refine_kept) span a block whose
  // singular values are small; A_lo = U_lo^H A, heevd of A_lo A_lo^H resolves
  // them relative to their own scale.  Rotates those rows and rewrites S.
  void deflate_low(cudaStream_t st, Solver& so, Pool& pool, cplx* uhf, double* S, const cplx* A, int R, int Cc,
                   int n_hi, int* info) {
    const int nl = R - n_hi;
    if (nl <= 0) return;
    cplx* lo = uhf + (int64_t)n_hi * R;
    cplx* Alo = pool.c((int64_t)nl * Cc);
    nn(st, nl, Cc, R, lo, 0, A, 0, Alo, 0, 1);
    cplx* G2 = pool.c((int64_t)nl * nl);
    nc(st, nl, nl, Cc, Alo, 0, Alo, 0, G2, 0, 1);
    double* lam = (double*)pool.raw((size_t)nl * sizeof(double));
    cplx* work = pool.c(std::max(lwork_heevd, 1));
    TN_SOLVER(cusolverDnSetStream(so.h, st));
    int* ci = call_info(pool, st);
    TN_SOLVER(cusolverDnZheevd(so.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, nl, (cuDoubleComplex*)G2, nl,
                               lam, (cuDoubleComplex*)work, lwork_heevd, ci));
    info_accum(st, info, ci);
    cplx* rot = pool.c((int64_t)nl * nl);
    eig_to_svd(st, rot, S + n_hi, G2, lam, nl);
    cplx* old = pool.c((int64_t)nl * R);
    TN_CUDA(cudaMemcpyAsync(old, lo, (size_t)nl * R * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    nn(st, nl, R, nl, rot, 0, old, 0, lo, 0, 1);
  }

  // Runs one side's primal sweep.  store: write snapshots / replay data to the arena.
  // Returns the final MPS (pool-owned) -- the top side's T_0.
  // on_snap(idx): called after layer snapshot idx has been enqueued on st
  // gmat (optional): the side's gate array (G, or G^dag for the top side) to
  // use instead of the stored point's (tn_hvp_cost: trial gates, arena untouched).
  Mps primal_side(cudaStream_t st, Solver& so, Pool& pool, bool is_top, bool store, int* info, double* diag,
                  const std::function<void(int)>& on_snap = nullptr, const cplx* gmat = nullptr) {
    SidePlan& sp = is_top ? top : bot;
    const cplx* G = gmat ? gmat : is_top ? at(o_gdag) : at(o_gates);
    Mps ps;
    ps.a.assign(n, nullptr);
    ps.b = sp.init.p;
    for (int s = 0; s < n; ++s) {
      const int64_t e = (int64_t)ps.b[s] * P * ps.b[s + 1];
      ps.a[s] = dnew(e, st);
      const cplx* src = is_top ? ref + ref_off[s] : d_init + (int64_t)s * P;  // bottom: bond-1 start
      TN_CUDA(cudaMemcpyAsync(ps.a[s], src, e * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    }
    for (size_t li = 0; li < sp.steps.size(); ++li) {
      if (store) snapshot(st, ps, sp.o_snap[li]);
      if (on_snap) on_snap((int)li);
      for (const Step& s : sp.steps[li]) {
        Pool tmp(st);  // step temporaries
        if (s.type == MOVE_R) {
          const int c = s.site;
          cplx* Q = store ? at(s.o_q) : tmp.c((int64_t)P * s.b * s.kq);
          cplx* R = tmp.c((int64_t)s.kq * s.bp);
          qr_right(st, so, tmp, ps.a[c], P * s.b, s.bp, s.kq, Q, R, info);
          cplx* nc_ = dnew((int64_t)P * s.b * s.kq, st);
          TN_CUDA(cudaMemcpyAsync(nc_, Q, (size_t)P * s.b * s.kq * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
          cplx* nx = dnew((int64_t)s.kq * P * s.nb2, st);
          nn(st, s.kq, P * s.nb2, s.bp, R, 0, ps.a[c + 1], 0, nx, 0, 1);
          dset(ps.a[c], nc_, st);
          dset(ps.a[c + 1], nx, st);
          ps.b[c + 1] = s.kq;
        } else if (s.type == MOVE_L) {
          const int c = s.site;
          cplx* Q = store ? at(s.o_q) : tmp.c((int64_t)s.kq * P * s.bp);
          cplx* L = tmp.c((int64_t)s.b * s.kq);
          lq_left(st, so, tmp, ps.a[c], s.b, P * s.bp, s.kq, Q, L, info);
          cplx* nc_ = dnew((int64_t)s.kq * P * s.bp, st);
          TN_CUDA(cudaMemcpyAsync(nc_, Q, (size_t)s.kq * P * s.bp * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
          cplx* nx = dnew((int64_t)s.nb2 * P * s.kq, st);
          nn(st, s.nb2 * P, s.kq, s.b, ps.a[c - 1], 0, L, 0, nx, 0, 1);
          dset(ps.a[c], nc_, st);
          dset(ps.a[c - 1], nx, st);
          ps.b[c] = s.kq;
        } else {
          const int i = s.site;
          const int64_t nth = (int64_t)PP * s.bl * s.br;
          cplx* theta = store ? at(s.o_theta) : tmp.c(nth);
          nn(st, P * s.bl, P * s.br, s.m, ps.a[i], 0, ps.a[i + 1], 0, theta, 0, 1);
          cplx* A = tmp.c(nth);
          apply_gate(st, A, 0, theta, 0, G + (int64_t)s.k * 16, 0, s.bl, s.br, 1, ONE, false, NI);
          double* S = store ? at<double>(s.o_S) : (double*)tmp.raw((size_t)s.mn * sizeof(double));
          cplx* uh = store ? at(s.o_uh) : tmp.c((int64_t)s.r * P * s.bl);
          cplx* vh = store ? at(s.o_vh) : tmp.c((int64_t)s.r * P * s.br);
          // Split: Gram heevd (fast) when the cut lies where it resolves the
          // spectrum (smallest kept sigma >= 1e-6 sigma_1 and a boundary gap in
          // sigma^2 >= 1e-12 sigma_1^2), else one-sided Jacobi (relative accuracy).
          int method = kGram;
          int nbas = P * s.bl;
          double* Sf = (double*)tmp.raw((size_t)P * s.bl * sizeof(double));
          int iters = 0;
          int lq_steps = 0;  // > 0: W_r^H by Newton-Schulz steps on the sigma-scaled rows (lq_rows_lowdin)
          bool y_ill = false;  // Y = U_r^H A known to be ill-conditioned (cut in the unresolved tail): Householder LQ
          // Low-rank blocks (numerical rank <= r): range probe instead of an
          // eigendecomposition.  Tried where the last pass at this step found it
          // (or a cut inside the noise floor); a failed probe switches it off.
          char* hint = (d_omega && s.s_index >= 0 && s.s_index < (int)lowrank_hint.size() && s.r < P * s.bl)
                           ? &lowrank_hint[s.s_index]
                           : nullptr;
          bool lowrank = false;
          if (hint && *hint == 1) {
            lowrank = lowrank_split(st, so, tmp, A, P * s.bl, P * s.br, s.r, uh, info);
            if (lowrank) {
              ++n_lowrank;
              static const double one_d = 1.0;  // diagnostics only: S = (1, 0, ...), gap 0
              TN_CUDA(cudaMemsetAsync(S, 0, (size_t)s.mn * sizeof(double), st));
              TN_CUDA(cudaMemcpyAsync(S, &one_d, sizeof(double), cudaMemcpyHostToDevice, st));
            } else {
              *hint = 2;  // failed here: off for good (a noise-floor cut must not switch it back on every pass)
            }
          }
          if (!lowrank) {
          cplx* Acp = tmp.c(nth);
          TN_CUDA(cudaMemcpyAsync(Acp, A, nth * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
          cplx* uhf = tmp.c((int64_t)P * s.bl * P * s.bl);
          svd_rowmajor(st, so, tmp, Acp, P * s.bl, P * s.br, Sf, uhf, info + 1, method);
          if (s.r < P * s.bl) {  // something (discarded or null) is excluded
            // kept/excluded mixing of a Gram basis ~ eps sigma_top^2 / (sigma_{r-1}^2 - sigma_r^2)
            // (sigma_r = 0 for a null direction); first-order refinement converges
            // quadratically from delta <~ 1e-2.  Otherwise a second Gram level on the
            // low block (resolves relative to its own scale), else QR-iteration SVD.
            const int R = P * s.bl;
            std::vector<double> hS(R);
            TN_CUDA(cudaMemcpyAsync(hS.data(), Sf, R * sizeof(double), cudaMemcpyDeviceToHost, st));
            TN_CUDA(cudaStreamSynchronize(st));
            auto mixing = [&](double top) {
              const double low = s.r < s.mn ? hS[s.r] : 0.0;
              const double gap2 = (hS[s.r - 1] * hS[s.r - 1] - low * low) / (top * top);
              return gap2 > 0 ? 2.2e-16 / gap2 : 1.0;
            };
            double delta = mixing(hS[0]);
            // Deflation levels: while the cut is unresolved relative to the
            // current level's top, refine the rows above 1e-4 of that top and
            // re-solve the block below them with its own Gram matrix (each
            // level resolves ~1e-4 further down the spectrum).
            int top_i = 0;
            for (int level = 0; level < 3 && delta > 1e-2; ++level) {
              int n_hi = top_i;
              while (n_hi < R && hS[n_hi] >= deflate_step * hS[top_i]) ++n_hi;
              if (!(n_hi > top_i && n_hi < s.r)) break;
              refine_kept(st, tmp, uhf, Sf, A, R, P * s.br, R, n_hi, 2);
              deflate_low(st, so, tmp, uhf, Sf, A, R, P * s.br, n_hi, info + 1);
              TN_CUDA(cudaMemcpyAsync(hS.data(), Sf, R * sizeof(double), cudaMemcpyDeviceToHost, st));
              TN_CUDA(cudaStreamSynchronize(st));
              delta = mixing(hS[n_hi]);
              top_i = n_hi;
              ++n_deflate;
            }
            // A boundary inside the double-precision noise floor (after the second
            // level: sigma_{r-1} < 1e-12 sigma_1) is not determined by the data for
            // any SVD algorithm; outputs are insensitive to it (reading X10).
            const bool in_noise = hS[s.r - 1] < 1e-12 * hS[0];
            if (delta > 1e-2 && in_noise) {
              delta = 1e-3;
              ++n_noise;
            }
            if (hint && in_noise && *hint == 0) *hint = 1;  // rank <= r to ~1e-12: probe the range at the next pass
            if (split_log) {  // diagnostic: spectrum profile of this split
              int c4 = 0, c7 = 0, c10 = 0, c13 = 0;
              for (int q = 0; q < R; ++q) {
                c4 += hS[q] > 1e-4 * hS[0];
                c7 += hS[q] > 1e-7 * hS[0];
                c10 += hS[q] > 1e-10 * hS[0];
                c13 += hS[q] > 1e-13 * hS[0];
              }
              std::lock_guard<std::mutex> g(split_log_mu);
              fprintf(split_log, "%d %d %d %d %d %d %d %d %d %.3e %d\n", (int)is_top, s.s_index, R, P * s.br, s.r, c4, c7, c10,
                      c13, delta, top_i);
            }
            if (delta > 1e-2) {
              method = kQRIter;
              nbas = s.mn;
              iters = 2;
              TN_CUDA(cudaMemcpyAsync(Acp, A, nth * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
              svd_rowmajor(st, so, tmp, Acp, P * s.bl, P * s.br, Sf, uhf, info + 1, method);
              ++n_fallback;
            } else {
              iters = delta < 1e-8 ? 1 : delta < 1e-4 ? 2 : 4;
              // row-orthogonality defect of the scaled Y ~ eps (sigma_1/sigma_{r-1})^2 (x100 margin);
              // only plain Gram splits (no deflation level rewrote the low rows' scale)
              if (lowdin_lq && top_i == 0 && hS[s.r - 1] > 0) {
                const double e0 = 2.2e-14 * (hS[0] / hS[s.r - 1]) * (hS[0] / hS[s.r - 1]);
                lq_steps = e0 < 1e-9 ? 1 : e0 < 1e-5 ? 2 : e0 < 1e-3 ? 3 : 0;
              }
              y_ill = top_i > 0 || !(hS[s.r - 1] > 1e-6 * hS[0]);
            }
          }
          TN_CUDA(cudaMemcpyAsync(S, Sf, (size_t)s.mn * sizeof(double), cudaMemcpyDeviceToDevice, st));
          refine_kept(st, tmp, uhf, Sf, A, P * s.bl, P * s.br, nbas, s.r, iters, /*kept_only=*/true);
          TN_CUDA(cudaMemcpyAsync(uh, uhf, (size_t)s.r * P * s.bl * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
          }  // !lowrank
          double* sc = store ? at<double>(s.o_s) : (double*)tmp.raw(sizeof(double));
          // Y = U_r^H A (= S_r W_r^H up to a kept-space rotation); LQ gives W_r^H
          cplx* Y = tmp.c((int64_t)s.r * P * s.br);
          nn(st, s.r, P * s.br, P * s.bl, uh, 0, A, 0, Y, 0, 1);
          {  // frozen s = ||A|| / ||U_r^H A|| and diagnostics
            double* nrm = (double*)tmp.raw(2 * sizeof(double));
            tangent_dot(st, nth, 1, A, A, nrm);
            tangent_dot(st, (int64_t)s.r * P * s.br, 1, Y, Y, nrm + 1);
            s_from_norms(st, nrm, S, s.mn, s.r, sc, diag);
          }
          cplx* Lq = tmp.c((int64_t)s.r * s.r);
          if (lq_steps > 0)
            lq_rows_lowdin(st, tmp, Y, Sf, s.r, P * s.br, lq_steps, vh, Lq);
          else  // (a low-rank Y is rank deficient: Householder only)
            lq_left(st, so, tmp, Y, s.r, P * s.br, s.r, vh, Lq, info, /*allow_chol=*/!lowrank && !y_ill);
          cplx* ni = dnew((int64_t)P * s.bl * s.r, st);
          cplx* nj = dnew((int64_t)s.r * P * s.br, st);
          if (s.lr) {  // (U_r, s U_r^H A), centre -> i+1
            conjT_scale_cols(st, ni, uh, s.r, P * s.bl, nullptr, nullptr);
            TN_CUDA(cudaMemcpyAsync(nj, Y, (size_t)s.r * P * s.br * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
            scale_by(st, nj, sc, 1.0, (int64_t)s.r * P * s.br);
          } else {     // (s U_r L, W_r^H), centre -> i
            cn(st, P * s.bl, s.r, s.r, uh, 0, Lq, 0, ni, 0, 1);
            scale_by(st, ni, sc, 1.0, (int64_t)P * s.bl * s.r);
            TN_CUDA(cudaMemcpyAsync(nj, vh, (size_t)s.r * P * s.br * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
          }
          dset(ps.a[i], ni, st);
          dset(ps.a[i + 1], nj, st);
          ps.b[i + 1] = s.r;
        }
      }
    }
    if (store) snapshot(st, ps, sp.o_snap.back());
    if (on_snap) on_snap((int)sp.steps.size());
    return ps;
  }

  void snapshot(cudaStream_t st, const Mps& ps, const std::vector<size_t>& offs) {
    for (int s = 0; s < n; ++s)
      TN_CUDA(cudaMemcpyAsync(at(offs[s]), ps.a[s], (size_t)ps.b[s] * P * ps.b[s + 1] * sizeof(cplx),
                              cudaMemcpyDeviceToDevice, st));
  }

  // overlap <<top|bot>> as a 1x1 complex on device
  cplx* overlap(cudaStream_t st, Pool& pool, const std::vector<const cplx*>& tp, const std::vector<int>& tb,
                const std::vector<const cplx*>& bp, const std::vector<int>& bb) {
    cplx* L = pool.c(1);
    TN_CUDA(cudaMemcpyAsync(L, &ONE, sizeof(cplx), cudaMemcpyHostToDevice, st));
    for (int s = 0; s < n; ++s) {
      cplx* Y = pool.c((int64_t)tb[s] * P * bb[s + 1]);
      nn(st, tb[s], P * bb[s + 1], bb[s], L, 0, bp[s], 0, Y, 0, 1);
      cplx* L2 = pool.c((int64_t)tb[s + 1] * bb[s + 1]);
      cn(st, tb[s + 1], bb[s + 1], P * tb[s], tp[s], 0, Y, 0, L2, 0, 1);
      L = L2;
    }
    return L;
  }

  std::vector<const cplx*> snap_ptrs(const SidePlan& sp, int idx) const {
    std::vector<const cplx*> v(n);
    for (int s = 0; s < n; ++s) v[s] = at(sp.o_snap[idx][s]);
    return v;
  }

  // Blocks of layer ell: (s, k) with k = -1 for an idle single site.
  std::vector<std::pair<int, int>> blocks(int ell) const {
    std::vector<std::pair<int, int>> out;
    const auto& ly = layers[ell - 1];
    size_t j = 0;
    for (int s = 0; s < n;) {
      if (j < ly.size() && ly[j].second == s) {
        out.push_back({s, ly[j].first});
        s += 2;
        ++j;
      } else {
        out.push_back({s, -1});
        s += 1;
      }
    }
    return out;
  }

  // N2 (reading X20): the per-gate pass at G_k = g_ell,
  // then dT/dg_ell = sum_{k in I_ell} E_k and Alg. 2 + App. E on U(4)^D.
  void ti_environments(cudaStream_t st, const cplx* g, double* scalars, cplx* grad_R) {
    Pool pool(st);
    cplx* G = pool.c((int64_t)K * 16);
    cplx* gR = pool.c((int64_t)K * 16);
    ti_expand(st, D, K, 1, d_layer_of, g, G);
    environments(st, G, scalars, gR);
    cplx *tg = ti_buf, *tE = ti_buf + 16 * D, *tf = ti_buf + 32 * D;
    TN_CUDA(cudaMemcpyAsync(tg, g, (size_t)D * 16 * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    ti_reduce(st, D, K, 1, d_layer_start, at(o_E), tE);
    gradient_post(st, D, tg, tE, at<double>(o_scal), tf, grad_R);
    TN_CUDA(cudaStreamSynchronize(st));
    ti_valid = true;
  }

  // H_T[v]_ell = sum_{k in I_ell} H_T[expand(v)]_k, then Alg. 2 + App. E on U(4)^D
  void ti_apply(cudaStream_t st, int batch, const cplx* v, cplx* hess) {
    if (!ti_valid || !primal_valid) throw StateError("tn_hvp_ti_apply before tn_hvp_ti_environments");
    if (batch == 0) return;
    Pool pool(st);
    const int64_t KK = (int64_t)K * 16;
    cplx* V = pool.c(KK * batch);
    cplx* H = pool.c(KK * batch);
    cplx* aux = pool.c(KK * batch + batch);
    cplx* HT = pool.c((int64_t)D * 16 * batch);
    cplx* om = pool.c(batch);
    ti_expand(st, D, K, batch, d_layer_of, v, V);
    apply_call(st, batch, V, H, aux);
    ti_reduce(st, D, K, batch, d_layer_start, aux, HT);
    hessian_post(st, D, batch, ti_buf, ti_buf + 16 * D, ti_buf + 32 * D, at<double>(o_scal), HT, v, om, hess);
    TN_CUDA(cudaStreamSynchronize(st));  // pool temporaries are freed on return
  }

  // ABI flag checks, before any work of the call: each gate
  // ||G^dag G - I||_F <= 1e-10 (TN_CHECK_UNITARY); each direction
  // ||V - P_G V|| <= 1e-8 ||V|| (TN_CHECK_TANGENT).  TN_EINVAL otherwise.
  void check_gates(cudaStream_t st, const cplx* G, int Kg) {
    if (!(cfg.flags & TN_CHECK_UNITARY) || Kg <= 0) return;
    Pool pool(st);
    double* res = (double*)pool.raw(sizeof(double) * Kg);
    check_unitary(st, Kg, G, res);
    std::vector<double> h(Kg);
    TN_CUDA(cudaMemcpyAsync(h.data(), res, sizeof(double) * Kg, cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < Kg; ++k)
      if (!(h[k] <= 1e-10))
        throw std::invalid_argument("gate " + std::to_string(k) + " is not unitary: ||G^dag G - I||_F = " +
                                    std::to_string(h[k]) + " > 1e-10 (TN_CHECK_UNITARY)");
  }
  void check_dirs(cudaStream_t st, const cplx* G, const cplx* V, int batch) {
    if (!(cfg.flags & TN_CHECK_TANGENT) || batch <= 0) return;
    Pool pool(st);
    const int64_t m = (int64_t)K * batch;
    double* res = (double*)pool.raw(sizeof(double) * 2 * m);
    check_tangent(st, K, batch, G, V, res);
    std::vector<double> h(2 * m);
    TN_CUDA(cudaMemcpyAsync(h.data(), res, sizeof(double) * 2 * m, cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    for (int b = 0; b < batch; ++b) {
      double r2 = 0, n2 = 0;
      for (int k = 0; k < K; ++k) {
        r2 += h[2 * ((int64_t)b * K + k)];
        n2 += h[2 * ((int64_t)b * K + k) + 1];
      }
      if (!(std::sqrt(r2) <= 1e-8 * std::sqrt(n2)))
        throw std::invalid_argument("direction " + std::to_string(b) + " is not tangent at G: ||V - P_G V|| = " +
                                    std::to_string(std::sqrt(r2)) + " > 1e-8 ||V|| = " +
                                    std::to_string(1e-8 * std::sqrt(n2)) + " (TN_CHECK_TANGENT)");
    }
  }

  // fwd_out (fused step): also replay the forward tangents of fwd_nb directions
  // fwd_V on stream stf while the sweeps run (see step()).
  void environments(cudaStream_t st, const cplx* gates, double* scalars, cplx* grad_R, int fwd_nb = 0,
                    const cplx* fwd_V = nullptr, std::vector<TanSnap>* fwd_out = nullptr) {
    TN_CUDA(cudaSetDevice(device));
    check_gates(st, gates, K);
    if (fwd_out) check_dirs(st, gates, fwd_V, fwd_nb);
    primal_valid = false;
    ti_valid = false;
    applies_at_point = 0;
    drop_graphs(st);
    drop_chain_cache(st);
    n_fallback = 0;
    n_deflate = 0;
    n_noise = 0;
    n_lowrank = 0;
    n_cholqr_fallback = 0;
    const double wc0 = work_counter.load();
    Pool pool(st);
    TN_CUDA(cudaMemcpyAsync(at(o_gates), gates, (size_t)K * 16 * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    dagger4(st, at(o_gdag), at(o_gates), K);
    // info[0..1]: bottom (qr, svd); info[2..3]: top.  diag: bottom [0..2], top [8..10]
    const int n_info = 4;
    int* info = (int*)pool.raw(n_info * sizeof(int));
    TN_CUDA(cudaMemsetAsync(info, 0, n_info * sizeof(int), st));
    double* dg = (double*)pool.raw(16 * sizeof(double));
    double hdiag[16] = {0, 1.0, 0, 0, 0, 0, 0, 0, 0, 1.0, 0, 0, 0, 0, 0, 0};
    TN_CUDA(cudaMemcpyAsync(dg, hdiag, sizeof(hdiag), cudaMemcpyHostToDevice, st));
    // fork: the top sweep runs on st2 from a second host thread (the split
    // decisions return to the host per step, so two threads keep both in
    // flight), the bottom sweep on st1 from this thread, and a third thread
    // issues the layer gradients of layer ell on stg as soon as both of its
    // snapshots (B_{ell-1}, T_ell) are enqueued: layers near the middle are
    // ready halfway through the sweeps, so their GEMMs overlap the eigensolves.
    TN_CUDA(cudaEventRecord(ev_fork, st));
    TN_CUDA(cudaStreamWaitEvent(st2, ev_fork, 0));
    TN_CUDA(cudaStreamWaitEvent(st1, ev_fork, 0));
    TN_CUDA(cudaStreamWaitEvent(stg, ev_fork, 0));
    const bool serial = std::getenv("TN_SERIAL_PRIMAL") != nullptr;
    if (serial) {  // diagnostic: bottom, top, then gradients on the caller's stream
      Mps BD = primal_side(st, sol[0], pool, false, true, info, dg);
      for (cplx*& p : BD.a) ddel(p, st);
      Mps T0 = primal_side(st, sol[0], pool, true, true, info + 2, dg + 8);
      for (cplx*& p : T0.a) ddel(p, st);
      layer_gradients(st);
    } else {
      std::mutex mu;
      std::condition_variable cv;
      int ready[2] = {0, 0};  // snapshots enqueued per side (0 bottom, 1 top)
      bool abort = false;
      auto publisher = [&](int side, cudaStream_t s) {
        return std::function<void(int)>([&, side, s](int idx) {
          TN_CUDA(cudaEventRecord(ev_snap[side][idx], s));
          {
            std::lock_guard<std::mutex> g(mu);
            ready[side] = idx + 1;
          }
          cv.notify_all();
        });
      };
      auto fail = [&] {
        {
          std::lock_guard<std::mutex> g(mu);
          abort = true;
        }
        cv.notify_all();
      };
      std::exception_ptr top_err, grad_err;
      std::thread th([&] {
        try {
          TN_CUDA(cudaSetDevice(device));
          Pool pool2(st2);
          Mps T0 = primal_side(st2, sol[1], pool2, true, true, info + 2, dg + 8, publisher(1, st2));
          for (cplx*& p : T0.a) ddel(p, st2);
        } catch (...) {
          top_err = std::current_exception();
          fail();
        }
      });
      std::thread tg([&] {
        try {
          TN_CUDA(cudaSetDevice(device));
          TN_CUDA(cudaMemsetAsync(at(o_E), 0, (size_t)K * 16 * sizeof(cplx), stg));
          std::vector<int> order(D);
          std::iota(order.begin(), order.end(), 1);
          std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
            return std::max(a - 1, D - a) < std::max(b - 1, D - b);
          });
          for (int ell : order) {
            {
              std::unique_lock<std::mutex> lk(mu);
              cv.wait(lk, [&] { return abort || (ready[0] > ell - 1 && ready[1] > D - ell); });
              if (abort) return;
            }
            TN_CUDA(cudaStreamWaitEvent(stg, ev_snap[0][ell - 1], 0));
            TN_CUDA(cudaStreamWaitEvent(stg, ev_snap[1][D - ell], 0));
            layer_gradient(stg, ell);
          }
        } catch (...) {
          grad_err = std::current_exception();
          fail();
        }
      });
      std::exception_ptr fwd_err;
      const double wf0 = work_counter_fwd.load();
      std::thread tf;
      if (fwd_out) {
        TN_CUDA(cudaStreamWaitEvent(stf, ev_fork, 0));
        tf = std::thread([&] {
          try {
            TN_CUDA(cudaSetDevice(device));
            g_fwd_thread = true;
            *fwd_out = forward_tangents(stf, fwd_nb, fwd_V, [&](int li) {
              {  // bottom layer li fully enqueued (its end snapshot published)
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return abort || ready[0] > li + 1; });
                if (abort) throw std::runtime_error("fused step: primal pass failed");
              }
              TN_CUDA(cudaStreamWaitEvent(stf, ev_snap[0][li + 1], 0));
            });
          } catch (...) {
            fwd_err = std::current_exception();
            fail();
          }
          g_fwd_thread = false;
        });
      }
      auto join_all = [&] {
        th.join();
        tg.join();
        if (tf.joinable()) tf.join();
      };
      // failure: let every side stream drain before the caller's stream frees
      // this call's buffers (info, diagnostics, pools) during unwinding
      auto drain = [&] {
        for (cudaStream_t x : {st1, st2, stg, stf, sth}) cudaStreamSynchronize(x);
      };
      try {
        Pool pool1(st1);
        Mps BD = primal_side(st1, sol[0], pool1, false, true, info, dg, publisher(0, st1));
        for (cplx*& p : BD.a) ddel(p, st1);
      } catch (...) {
        fail();
        join_all();
        drain();
        throw;
      }
      join_all();
      if (top_err || grad_err || fwd_err) drain();
      if (top_err) std::rethrow_exception(top_err);
      if (grad_err) std::rethrow_exception(grad_err);
      if (fwd_err) std::rethrow_exception(fwd_err);
      if (fwd_out) {
        work_fwd_first = work_counter_fwd.load() - wf0;
        TN_CUDA(cudaEventRecord(ev_joinf, stf));
        TN_CUDA(cudaStreamWaitEvent(st, ev_joinf, 0));
      }
      TN_CUDA(cudaEventRecord(ev_join, st2));
      TN_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
      TN_CUDA(cudaEventRecord(ev_join1, st1));
      TN_CUDA(cudaStreamWaitEvent(st, ev_join1, 0));
      TN_CUDA(cudaEventRecord(ev_joing, stg));
      TN_CUDA(cudaStreamWaitEvent(st, ev_joing, 0));
    }
    combine_diag(st, at<double>(o_diag), dg);
    TN_CUDA(cudaMemcpyAsync(at<double>(o_sdiag[0]), dg, 8 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    TN_CUDA(cudaMemcpyAsync(at<double>(o_sdiag[1]), dg + 8, 8 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    // T = <<T_0|B_0>>  (Alg. 1)
    cplx* T11 = overlap(st, pool, snap_ptrs(top, D), top.snap[D].p, snap_ptrs(bot, 0), bot.snap[0].p);
    finish_cost(st, at<double>(o_scal), T11);
    gradient_post(st, K, at(o_gates), at(o_E), at<double>(o_scal), at(o_gradf), grad_R);
    // host copies: scalars/diag, solver info
    int hinfo[n_info];
    TN_CUDA(cudaMemcpyAsync(hinfo, info, sizeof(hinfo), cudaMemcpyDeviceToHost, st));
    double sc[8];
    TN_CUDA(cudaMemcpyAsync(sc, at<double>(o_scal), 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaMemcpyAsync(sc + 3, at<double>(o_diag), 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    for (int j = 0; j < n_info; ++j)
      if (hinfo[j] != 0)
        throw NumericError("cuSOLVER info nonzero (slot " + std::to_string(j) + ": " + std::to_string(hinfo[j]) + ")");
    for (int j = 0; j < 6; ++j)
      if (!std::isfinite(sc[j]))
        throw NumericError("non-finite primal scalar: f=" + std::to_string(sc[0]) + " T=(" + std::to_string(sc[1]) +
                           "," + std::to_string(sc[2]) + ") discarded=" + std::to_string(sc[3]) +
                           " gap=" + std::to_string(sc[4]) + " log10s=" + std::to_string(sc[5]));
    sc[6] = (double)n_fallback.load();
    sc[7] = (double)n_deflate.load();
    TN_CUDA(cudaMemcpyAsync(scalars, sc, 8 * sizeof(double), cudaMemcpyHostToDevice, st));
    TN_CUDA(cudaMemcpyAsync(at<double>(o_scal), sc, 8 * sizeof(double), cudaMemcpyHostToDevice, st));
    TN_CUDA(cudaStreamSynchronize(st));
    work_primal = work_counter.load() - wc0;
    primal_valid = true;
  }

  // ---- split primal (multi-GPU): one side's sweep per rank, then finish ----
  // part 0: bottom sweep (a2), part 1: top sweep (a3), each on the caller's
  // stream, writing only that side's region of the store and its diagnostics.
  void environments_part(cudaStream_t st, const cplx* gates, int part) {
    TN_CUDA(cudaSetDevice(device));
    check_gates(st, gates, K);
    invalidate(st);
    TN_CUDA(cudaMemcpyAsync(at(o_gates), gates, (size_t)K * 16 * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    dagger4(st, at(o_gdag), at(o_gates), K);
    Pool pool(st);
    int* info = (int*)pool.raw(2 * sizeof(int));
    TN_CUDA(cudaMemsetAsync(info, 0, 2 * sizeof(int), st));
    double* dg = at<double>(o_sdiag[part]);
    double hdiag[8] = {0, 1.0, 0, 0, 0, 0, 0, 0};
    TN_CUDA(cudaMemcpyAsync(dg, hdiag, sizeof(hdiag), cudaMemcpyHostToDevice, st));
    Mps last = primal_side(st, sol[0], pool, part == 1, true, info, dg);
    for (cplx*& p : last.a) ddel(p, st);
    int hinfo[2];
    TN_CUDA(cudaMemcpyAsync(hinfo, info, sizeof(hinfo), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    if (hinfo[0] || hinfo[1]) throw NumericError("cuSOLVER info nonzero in the split primal sweep");
  }

  // After both side regions hold this point's sweeps (local or received):
  // layer environments, E, T, f, grad_R -- the rest of tn_hvp_environments.
  void environments_finish(cudaStream_t st, const cplx* gates, double* scalars, cplx* grad_R) {
    TN_CUDA(cudaSetDevice(device));
    invalidate(st);
    TN_CUDA(cudaMemcpyAsync(at(o_gates), gates, (size_t)K * 16 * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    dagger4(st, at(o_gdag), at(o_gates), K);
    Pool pool(st);
    layer_gradients(st);
    double* dg = (double*)pool.raw(16 * sizeof(double));
    TN_CUDA(cudaMemcpyAsync(dg, at<double>(o_sdiag[0]), 8 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    TN_CUDA(cudaMemcpyAsync(dg + 8, at<double>(o_sdiag[1]), 8 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    combine_diag(st, at<double>(o_diag), dg);
    cplx* T11 = overlap(st, pool, snap_ptrs(top, D), top.snap[D].p, snap_ptrs(bot, 0), bot.snap[0].p);
    finish_cost(st, at<double>(o_scal), T11);
    gradient_post(st, K, at(o_gates), at(o_E), at<double>(o_scal), at(o_gradf), grad_R);
    double sc[8];
    TN_CUDA(cudaMemcpyAsync(sc, at<double>(o_scal), 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaMemcpyAsync(sc + 3, at<double>(o_diag), 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    for (int j = 0; j < 6; ++j)
      if (!std::isfinite(sc[j])) throw NumericError("non-finite primal scalar after the split primal");
    sc[6] = sc[7] = 0.0;  // fallback / deflation counts stay with the ranks that swept
    TN_CUDA(cudaMemcpyAsync(scalars, sc, 8 * sizeof(double), cudaMemcpyHostToDevice, st));
    TN_CUDA(cudaMemcpyAsync(at<double>(o_scal), sc, 8 * sizeof(double), cudaMemcpyHostToDevice, st));
    TN_CUDA(cudaStreamSynchronize(st));
    primal_valid = true;
  }

  // Two-site block of site tensors a (x,4,m), b (m,4,y): out (x,4,4,y)
  void pair(cudaStream_t st, cplx* out, const cplx* a, int64_t sa, const cplx* b, int64_t sb, int x, int m, int y,
            int batch) {
    nn(st, P * x, P * y, m, a, sa, b, sb, out, (int64_t)PP * x * y, batch);
  }

  // a4: per layer right sweep, left sweep with E_k (primal envs stored for apply)
  void layer_gradients(cudaStream_t st) {
    TN_CUDA(cudaMemsetAsync(at(o_E), 0, (size_t)K * 16 * sizeof(cplx), st));
    for (int ell = 1; ell <= D; ++ell) layer_gradient(st, ell);
  }

  // layer ell's environments o_L/o_R and its gates' E_k (disjoint per layer)
  void layer_gradient(cudaStream_t st, int ell) {
    const auto tp = snap_ptrs(top, D - ell);
    const auto bp = snap_ptrs(bot, ell - 1);
    const auto& tb = top.snap[D - ell].p;
    const auto& bb = bot.snap[ell - 1].p;
    const auto blks = blocks(ell);
    TN_CUDA(cudaMemcpyAsync(at(o_L[ell][0]), &ONE, sizeof(cplx), cudaMemcpyHostToDevice, st));
    TN_CUDA(cudaMemcpyAsync(at(o_R[ell][n]), &ONE, sizeof(cplx), cudaMemcpyHostToDevice, st));
    // two-site blocks of the gate pairs, formed once for both sweeps:
    // TB[s] = B_s B_{s+1}, TT[s] = T_s T_{s+1} (ungated)
    Pool lp(st);
    std::vector<cplx*> TBs(n, nullptr), TTs(n, nullptr);
    // right sweep
    for (int j = (int)blks.size() - 1; j >= 0; --j) {
      const int s = blks[j].first, k = blks[j].second;
      Pool pool(st);  // block temporaries
      if (k < 0) {
        cplx* Y = pool.c((int64_t)bb[s] * P * tb[s + 1]);
        nn(st, P * bb[s], tb[s + 1], bb[s + 1], bp[s], 0, at(o_R[ell][s + 1]), 0, Y, 0, 1);
        nc(st, bb[s], tb[s], P * tb[s + 1], Y, 0, tp[s], 0, at(o_R[ell][s]), 0, 1);
      } else {
        cplx* TB = TBs[s] = lp.c((int64_t)PP * bb[s] * bb[s + 2]);
        pair(st, TB, bp[s], 0, bp[s + 1], 0, bb[s], bb[s + 1], bb[s + 2], 1);
        cplx* TT = TTs[s] = lp.c((int64_t)PP * tb[s] * tb[s + 2]);
        pair(st, TT, tp[s], 0, tp[s + 1], 0, tb[s], tb[s + 1], tb[s + 2], 1);
        cplx* TTg = pool.c((int64_t)PP * tb[s] * tb[s + 2]);
        apply_gate(st, TTg, 0, TT, 0, at(o_gdag) + (int64_t)k * 16, 0, tb[s], tb[s + 2], 1, ONE, false, NI);
        cplx* Y = pool.c((int64_t)PP * bb[s] * tb[s + 2]);
        nn(st, PP * bb[s], tb[s + 2], bb[s + 2], TB, 0, at(o_R[ell][s + 2]), 0, Y, 0, 1);
        nc(st, bb[s], tb[s], PP * tb[s + 2], Y, 0, TTg, 0, at(o_R[ell][s]), 0, 1);
      }
    }
    // left sweep + extraction
    for (size_t j = 0; j < blks.size(); ++j) {
      const int s = blks[j].first, k = blks[j].second;
      Pool pool(st);  // block temporaries
      if (k < 0) {
        cplx* Y = pool.c((int64_t)tb[s] * P * bb[s + 1]);
        nn(st, tb[s], P * bb[s + 1], bb[s], at(o_L[ell][s]), 0, bp[s], 0, Y, 0, 1);
        cn(st, tb[s + 1], bb[s + 1], P * tb[s], tp[s], 0, Y, 0, at(o_L[ell][s + 1]), 0, 1);
      } else {
        cplx* TB = TBs[s];
        cplx* TT = TTs[s];
        cplx* Y = pool.c((int64_t)PP * tb[s] * bb[s + 2]);
        nn(st, tb[s], PP * bb[s + 2], bb[s], at(o_L[ell][s]), 0, TB, 0, Y, 0, 1);
        cplx* Z = pool.c((int64_t)PP * tb[s] * tb[s + 2]);
        nn(st, PP * tb[s], tb[s + 2], bb[s + 2], Y, 0, at(o_R[ell][s + 2]), 0, Z, 0, 1);
        extract_env(st, at(o_E) + (int64_t)k * 16, 0, TT, 0, Z, 0, tb[s], tb[s + 2], 1, ONE, NI);
        apply_gate(st, TT, 0, TT, 0, at(o_gdag) + (int64_t)k * 16, 0, tb[s], tb[s + 2], 1, ONE, false, NI);
        cn(st, tb[s + 2], bb[s + 2], PP * tb[s], TT, 0, Y, 0, at(o_L[ell][s + 2]), 0, 1);
      }
    }
  }

  // T and f at trial gates (a3 top sweep only, the TR rho test).  The stored
  // point (arena, caches, graphs) is never touched, so a failure here leaves
  // the primal store valid for later applies.
  void cost(cudaStream_t st, const cplx* gates, double* scalars) {
    TN_CUDA(cudaSetDevice(device));
    check_gates(st, gates, K);
    Pool pool(st);
    cplx* Gd = pool.c((int64_t)K * 16);
    dagger4(st, Gd, gates, K);
    int* info = (int*)pool.raw(2 * sizeof(int));
    TN_CUDA(cudaMemsetAsync(info, 0, 2 * sizeof(int), st));
    Mps T0 = primal_side(st, sol[0], pool, true, false, info, nullptr, nullptr, Gd);
    std::vector<const cplx*> tp(T0.a.begin(), T0.a.end());
    std::vector<int> ones(n + 1, 1);
    std::vector<const cplx*> bp(n);
    for (int s = 0; s < n; ++s) bp[s] = d_init + (int64_t)s * P;  // B_0: the bond-1 bottom start
    cplx* T11 = overlap(st, pool, tp, T0.b, bp, ones);
    for (cplx*& p : T0.a) ddel(p, st);
    double* sc = (double*)pool.raw(8 * sizeof(double));
    TN_CUDA(cudaMemsetAsync(sc, 0, 8 * sizeof(double), st));
    finish_cost(st, sc, T11);
    TN_CUDA(cudaMemcpyAsync(scalars, sc, 8 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    int hinfo[2];
    double hsc[3];
    TN_CUDA(cudaMemcpyAsync(hinfo, info, sizeof(hinfo), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaMemcpyAsync(hsc, sc, sizeof(hsc), cudaMemcpyDeviceToHost, st));
    TN_CUDA(cudaStreamSynchronize(st));
    if (hinfo[0] != 0 || hinfo[1] != 0) throw NumericError("cuSOLVER info nonzero in tn_hvp_cost");
    if (!std::isfinite(hsc[0]) || !std::isfinite(hsc[1]) || !std::isfinite(hsc[2]))
      throw NumericError("tn_hvp_cost: non-finite T");
  }

  // ---------------------------------------------------- tangent pass --

  int64_t bsize(const Bonds& b, int s) const { return (int64_t)b.ab[s] * P * b.aa[s + 1]; }

  void tangent_init(cudaStream_t st, Tangent& t, const SidePlan& sp, bool is_top, int nb,
                    ChainCache* cache = nullptr) {
    t.bd = sp.init;
    t.Ab.assign(n, nullptr);
    t.Aa.assign(n, nullptr);
    t.B.assign(n, nullptr);
    t.cache = cache;
    t.step_no = 0;
    t.mode = !cache ? CHAIN_OWN : cache->built ? CHAIN_REPLAY : CHAIN_RECORD;
    if (t.mode == CHAIN_RECORD) {
      cache->step.clear();
      cache->init_Ab.assign(n, nullptr);
      cache->init_Aa.assign(n, nullptr);
    }
    for (int s = 0; s < n; ++s) {
      const int64_t e = (int64_t)t.bd.p[s] * P * t.bd.p[s + 1];
      t.B[s] = dnew(e * nb, st);
      TN_CUDA(cudaMemsetAsync(t.B[s], 0, (size_t)e * nb * sizeof(cplx), st));
      if (t.mode == CHAIN_REPLAY) {
        t.Ab[s] = cache->init_Ab[s];
        t.Aa[s] = cache->init_Aa[s];
        continue;
      }
      t.Ab[s] = dnew(e, st);
      t.Aa[s] = dnew(e, st);
      const cplx* src = is_top ? ref + ref_off[s] : d_init + (int64_t)s * P;
      TN_CUDA(cudaMemcpyAsync(t.Ab[s], src, e * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      TN_CUDA(cudaMemcpyAsync(t.Aa[s], src, e * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      if (t.mode == CHAIN_RECORD) {
        cache->init_Ab[s] = t.Ab[s];
        cache->init_Aa[s] = t.Aa[s];
        cache->owned.push_back(t.Ab[s]);
        cache->owned.push_back(t.Aa[s]);
      }
    }
  }

  // end of a side's replay: free what the tangent owns (recorded chains stay
  // in the cache, which is complete from now on)
  void release(Tangent& t, cudaStream_t st) {
    for (cplx*& p : t.B) ddel(p, st);
    if (t.mode == CHAIN_OWN) {
      for (auto* v : {&t.Ab, &t.Aa})
        for (cplx*& p : *v) ddel(p, st);
    } else if (t.mode == CHAIN_RECORD) {
      t.cache->built = true;
    }
  }
  void release(TanSnap& t, cudaStream_t st) {
    for (cplx*& p : t.B) ddel(p, st);
    if (t.chains_owned)
      for (auto* v : {&t.Ab, &t.Aa})
        for (cplx*& p : *v) ddel(p, st);
  }
  // a chain slot takes a new tensor: freed if the tangent owns its chains
  void chain_set(Tangent& t, cplx*& slot, cplx* nw, cudaStream_t st) {
    if (t.mode == CHAIN_OWN) dset(slot, nw, st);
    else slot = nw;
  }
  void record(Tangent& t, std::array<cplx*, 4> c) {
    t.cache->step.push_back(c);
    for (cplx* p : c)
      if (p) t.cache->owned.push_back(p);
  }

  int64_t chain_cache_elems(const SidePlan& sp) const {
    int64_t e = 0;
    for (int s = 0; s < n; ++s) e += 2LL * sp.init.p[s] * P * sp.init.p[s + 1];
    for (auto& ls : sp.steps)
      for (const Step& x : ls) {
        if (x.type == MOVE_R) e += (int64_t)x.kq * x.ab1 + (int64_t)P * x.b * x.kq + (int64_t)x.kq * P * x.ab2;
        else if (x.type == MOVE_L) e += (int64_t)x.aa0 * x.kq + (int64_t)x.kq * P * x.bp + (int64_t)x.aam * P * x.kq;
        else e += (int64_t)P * x.aa0 * x.r + (int64_t)x.r * P * x.br + (int64_t)P * x.bl * x.r + (int64_t)x.r * P * x.ab2;
      }
    return e;
  }
  // The side's cache if enabled and it fits (keeping half the free memory).
  // Inside a stream capture only an already-built cache is used: recording
  // there would store graph-owned allocations in it.
  ChainCache* chain_cache_for(int side, cudaStream_t st) {
    if (!chain_cache_enabled || no_cache) return nullptr;
    ChainCache& c = chain_cache[side];
    if (c.built) return &c;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TN_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    size_t fr = 0, tot = 0;
    TN_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t need = sizeof(cplx) * (size_t)chain_cache_elems(side ? top : bot);
    if (cache_budget) {
      const size_t used = sizeof(cplx) * (size_t)((chain_cache[0].built ? chain_cache_elems(bot) : 0) +
                                                  (chain_cache[1].built ? chain_cache_elems(top) : 0));
      return used + need <= cache_budget && need < fr / 2 ? &c : nullptr;
    }
    return need < fr / 2 ? &c : nullptr;
  }
  // Release the per-point caches, stream-ordered on st: every use of them was
  // enqueued on st or joined into it (calls on one context are stream-ordered,
  // tn_hvp.h), so no host or device-wide synchronisation is needed.  Blocks go
  // back to the library pool (not trimmed: the next pass reuses them).
  void drop_chain_cache(cudaStream_t st) {
    memo_budget_set = false;
    for (ChainCache& c : chain_cache) {
      for (cplx* p : c.owned) dfree(p, st);
      c = ChainCache{};
    }
    for (cplx* p : memo_owned) dfree(p, st);
    memo_owned.clear();
    memo_map.clear();
    memo_bytes = 0;
  }

  template <class F>
  cplx* memo(cudaStream_t st, Pool& tmp, int ell, int s, int tag, int64_t elems, F&& fill) {
    const uint64_t key = ((uint64_t)ell << 40) | ((uint64_t)(s + 1) << 16) | (uint64_t)tag;
    if (chain_cache_enabled && !no_cache) {
      auto it = memo_map.find(key);
      if (it != memo_map.end()) return it->second;
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      TN_CUDA(cudaStreamIsCapturing(st, &cs));
      if (cs == cudaStreamCaptureStatusNone) {
        if (!memo_budget_set) {
          size_t fr = 0, tot = 0;
          TN_CUDA(cudaMemGetInfo(&fr, &tot));
          memo_budget = fr / 3;
          if (cache_budget) {
            const size_t chains =
                sizeof(cplx) * (size_t)((chain_cache[0].built ? chain_cache_elems(bot) : 0) +
                                        (chain_cache[1].built ? chain_cache_elems(top) : 0));
            memo_budget = std::min(memo_budget, cache_budget > chains ? cache_budget - chains : 0);
          }
          memo_budget_set = true;
        }
        const size_t bytes = (size_t)std::max<int64_t>(elems, 1) * sizeof(cplx);
        if (memo_bytes + bytes <= memo_budget) {
          cplx* p = dnew(elems, st);
          fill(p);
          memo_map.emplace(key, p);
          memo_owned.push_back(p);
          memo_bytes += bytes;
          return p;
        }
      }
    }
    cplx* p = tmp.c(elems);
    fill(p);
    return p;
  }

  // One replayed step on a batch of tangents.  M: gate array (G or G^dag),
  // VM: per-direction gate variations [nb][K][16] (V or V^dag).
  void tangent_step(cudaStream_t st, Tangent& t, const Step& s, const cplx* M, const cplx* VM, int nb) {
    const int64_t KK = (int64_t)K * 16;
    const size_t sn = t.step_no++;  // index of this step in the side's chain cache
    Pool pool(st);  // step temporaries
    if (s.type == MOVE_R) {
      const int c = s.site, b = s.b, kq = s.kq;
      const int ab1 = s.ab1, ab2 = s.ab2, aa1 = s.aa1, aa2 = s.aa2;
      const cplx* Q = at(s.o_q);                        // (4b x kq)
      cplx *X, *nAbc, *nAb1;                            // X = Q^H Ab_c; chains
      if (t.mode == CHAIN_REPLAY) {
        const auto& cc = t.cache->step.at(sn);
        X = cc[0], nAbc = cc[1], nAb1 = cc[2];
      } else {
        X = t.mode == CHAIN_RECORD ? dnew((int64_t)kq * ab1, st) : pool.c((int64_t)kq * ab1);
        cn(st, kq, ab1, P * b, Q, 0, t.Ab[c], 0, X, 0, 1);
        nAbc = dnew((int64_t)P * b * kq, st);
        TN_CUDA(cudaMemcpyAsync(nAbc, Q, (size_t)P * b * kq * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        nAb1 = dnew((int64_t)kq * P * ab2, st);
        nn(st, kq, P * ab2, ab1, X, 0, t.Ab[c + 1], 0, nAb1, 0, 1);
        if (t.mode == CHAIN_RECORD) record(t, {X, nAbc, nAb1, nullptr});
      }
      // blocks: B_c (b,4,aa1), B_{c+1} (ab1,4,aa2)
      const int64_t sc0 = (int64_t)P * b * aa1, sc1o = (int64_t)ab1 * P * aa2, sc1n = (int64_t)kq * P * aa2;
      cplx* Y = pool.c((int64_t)kq * aa1 * nb);
      cn(st, kq, aa1, P * b, Q, 0, t.B[c], sc0, Y, (int64_t)kq * aa1, nb);
      nn(st, P * b, aa1, kq, Q, 0, Y, (int64_t)kq * aa1, t.B[c], sc0, nb, MONE, ONE);
      cplx* nB1 = dnew(sc1n * nb, st);
      nn(st, kq, P * aa2, ab1, X, 0, t.B[c + 1], sc1o, nB1, sc1n, nb);
      nn(st, kq, P * aa2, aa1, Y, (int64_t)kq * aa1, t.Aa[c + 1], 0, nB1, sc1n, nb, ONE, ONE);
      chain_set(t, t.Ab[c], nAbc, st);
      chain_set(t, t.Ab[c + 1], nAb1, st);
      dset(t.B[c + 1], nB1, st);
      t.bd.p[c + 1] = kq;
      t.bd.ab[c + 1] = kq;
    } else if (s.type == MOVE_L) {
      const int c = s.site, bp = s.bp, kq = s.kq;
      const int aa0 = s.aa0, aam = s.aam, ab0 = s.ab0, abm = s.abm;
      const cplx* Q = at(s.o_q);                        // (kq x 4bp)
      cplx *X, *nAac, *nAam;                            // X = Aa_c Q^H; chains
      if (t.mode == CHAIN_REPLAY) {
        const auto& cc = t.cache->step.at(sn);
        X = cc[0], nAac = cc[1], nAam = cc[2];
      } else {
        X = t.mode == CHAIN_RECORD ? dnew((int64_t)aa0 * kq, st) : pool.c((int64_t)aa0 * kq);
        nc(st, aa0, kq, P * bp, t.Aa[c], 0, Q, 0, X, 0, 1);
        nAac = dnew((int64_t)kq * P * bp, st);
        TN_CUDA(cudaMemcpyAsync(nAac, Q, (size_t)kq * P * bp * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        nAam = dnew((int64_t)aam * P * kq, st);
        nn(st, aam * P, kq, aa0, t.Aa[c - 1], 0, X, 0, nAam, 0, 1);
        if (t.mode == CHAIN_RECORD) record(t, {X, nAac, nAam, nullptr});
      }
      // blocks: B_c (ab0,4,bp), B_{c-1} (abm,4,aa0)
      const int64_t sc0 = (int64_t)ab0 * P * bp, sm_o = (int64_t)abm * P * aa0, sm_n = (int64_t)abm * P * kq;
      cplx* Y = pool.c((int64_t)ab0 * kq * nb);
      nc(st, ab0, kq, P * bp, t.B[c], sc0, Q, 0, Y, (int64_t)ab0 * kq, nb);
      nn(st, ab0, P * bp, kq, Y, (int64_t)ab0 * kq, Q, 0, t.B[c], sc0, nb, MONE, ONE);
      cplx* nBm = dnew(sm_n * nb, st);
      nn(st, abm * P, kq, aa0, t.B[c - 1], sm_o, X, 0, nBm, sm_n, nb);
      nn(st, abm * P, kq, ab0, t.Ab[c - 1], 0, Y, (int64_t)ab0 * kq, nBm, sm_n, nb, ONE, ONE);
      chain_set(t, t.Aa[c], nAac, st);
      chain_set(t, t.Aa[c - 1], nAam, st);
      dset(t.B[c - 1], nBm, st);
      t.bd.p[c] = kq;
      t.bd.aa[c] = kq;
    } else {
      const int i = s.site, bl = s.bl, br = s.br, r = s.r;
      const int ab1 = s.ab1, ab2 = s.ab2, aa0 = s.aa0, aa1 = s.aa1;
      const double* sc = at<double>(s.o_s);  // frozen s, read on the device (no host constant)
      const cplx* theta = at(s.o_theta);
      const cplx* uh = at(s.o_uh);  // (r x 4bl)
      const cplx* vh = at(s.o_vh);  // (r x 4br)
      const cplx* Mk = M + (int64_t)s.k * 16;
      const int64_t nD = (int64_t)PP * bl * br;
      // DTheta = M (B_i Aa_{i+1} + Ab_i B_{i+1}) + V_M Theta
      cplx* Dt = pool.c(nD * nb);
      nn(st, P * bl, P * br, aa1, t.B[i], (int64_t)P * bl * aa1, t.Aa[i + 1], 0, Dt, nD, nb);
      nn(st, P * bl, P * br, ab1, t.Ab[i], 0, t.B[i + 1], (int64_t)ab1 * P * br, Dt, nD, nb, ONE, ONE);
      apply_gate2(st, Dt, nD, Dt, nD, Mk, 0, theta, 0, VM + (int64_t)s.k * 16, KK, bl, br, nb, NI);
      const int64_t sUD = (int64_t)r * P * br, sZ = (int64_t)P * bl * r, sRR = (int64_t)r * r;
      cplx* UD = pool.c(sUD * nb);
      nn(st, r, P * br, P * bl, uh, 0, Dt, nD, UD, sUD, nb);  // U^H D (uh is U^H, r x 4bl)
      cplx* Z = pool.c(sZ * nb);
      nc(st, P * bl, r, P * br, Dt, nD, vh, 0, Z, sZ, nb);  // D W = D vh^H
      cplx* nBi = dnew(sZ * nb, st);
      cplx* nBj = dnew(sUD * nb, st);
      if (s.lr) {
        // B_{i+1} = s U^H D ; B_i = s (D W - U (U^H D W))
        cplx* UDW = pool.c(sRR * nb);
        nc(st, r, r, P * br, UD, sUD, vh, 0, UDW, sRR, nb);
        TN_CUDA(cudaMemcpyAsync(nBi, Z, (size_t)sZ * nb * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        cn(st, P * bl, r, r, uh, 0, UDW, sRR, nBi, sZ, nb, MONE, ONE, sc);
        TN_CUDA(cudaMemcpyAsync(nBj, UD, (size_t)sUD * nb * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        scale_by(st, nBj, sc, 1.0, sUD * nb);
      } else {
        // B_i = s D W ; B_{i+1} = s (U^H D - (U^H D W) W^H)
        cplx* UDW = pool.c(sRR * nb);
        nn(st, r, r, P * bl, uh, 0, Z, sZ, UDW, sRR, nb);
        TN_CUDA(cudaMemcpyAsync(nBj, UD, (size_t)sUD * nb * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        nn(st, r, P * br, r, UDW, sRR, vh, 0, nBj, sUD, nb, MONE, ONE, sc);
        TN_CUDA(cudaMemcpyAsync(nBi, Z, (size_t)sZ * nb * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        scale_by(st, nBi, sc, 1.0, sZ * nb);
      }
      // chains (direction-independent; recorded / replayed per point)
      cplx *nAai, *nAaj, *nAbi, *nAbj;
      if (t.mode == CHAIN_REPLAY) {
        const auto& cc = t.cache->step.at(sn);
        nAai = cc[0], nAaj = cc[1], nAbi = cc[2], nAbj = cc[3];
      } else {
        cplx* aa2t = pool.c((int64_t)PP * aa0 * br);
        nn(st, P * aa0, P * br, aa1, t.Aa[i], 0, t.Aa[i + 1], 0, aa2t, 0, 1);
        apply_gate(st, aa2t, 0, aa2t, 0, Mk, 0, aa0, br, 1, ONE, false, NI);
        nAai = dnew((int64_t)P * aa0 * r, st);
        nc(st, P * aa0, r, P * br, aa2t, 0, vh, 0, nAai, 0, 1, ONE, ZERO, sc);
        nAaj = dnew((int64_t)r * P * br, st);
        TN_CUDA(cudaMemcpyAsync(nAaj, vh, (size_t)r * P * br * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        cplx* ab2t = pool.c((int64_t)PP * bl * ab2);
        nn(st, P * bl, P * ab2, ab1, t.Ab[i], 0, t.Ab[i + 1], 0, ab2t, 0, 1);
        apply_gate(st, ab2t, 0, ab2t, 0, Mk, 0, bl, ab2, 1, ONE, false, NI);
        nAbj = dnew((int64_t)r * P * ab2, st);
        nn(st, r, P * ab2, P * bl, uh, 0, ab2t, 0, nAbj, 0, 1, ONE, ZERO, sc);
        nAbi = dnew((int64_t)P * bl * r, st);
        conjT_scale_cols(st, nAbi, uh, r, P * bl, nullptr, nullptr);
        if (t.mode == CHAIN_RECORD) record(t, {nAai, nAaj, nAbi, nAbj});
      }
      chain_set(t, t.Aa[i], nAai, st);
      chain_set(t, t.Aa[i + 1], nAaj, st);
      chain_set(t, t.Ab[i], nAbi, st);
      chain_set(t, t.Ab[i + 1], nAbj, st);
      dset(t.B[i], nBi, st);
      dset(t.B[i + 1], nBj, st);
      t.bd.p[i + 1] = r;
      t.bd.ab[i + 1] = r;
      t.bd.aa[i + 1] = r;
    }
  }


  TanSnap take_snapshot(cudaStream_t st, const Tangent& t, int nb) {
    TanSnap sn;
    sn.bd = t.bd;
    sn.Ab.resize(n);
    sn.Aa.resize(n);
    sn.B.resize(n);
    if (t.mode != CHAIN_OWN) {  // chains live in the cache: borrow them
      sn.chains_owned = false;
      sn.Ab = t.Ab;
      sn.Aa = t.Aa;
      for (int s = 0; s < n; ++s) {
        const int64_t e = bsize(t.bd, s) * nb;
        sn.B[s] = dnew(e, st);
        TN_CUDA(cudaMemcpyAsync(sn.B[s], t.B[s], e * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      }
      return sn;
    }
    for (int s = 0; s < n; ++s) {
      const int64_t eb = (int64_t)t.bd.ab[s] * P * t.bd.ab[s + 1];
      const int64_t ea = (int64_t)t.bd.aa[s] * P * t.bd.aa[s + 1];
      const int64_t e = bsize(t.bd, s) * nb;
      sn.Ab[s] = dnew(eb, st);
      sn.Aa[s] = dnew(ea, st);
      sn.B[s] = dnew(e, st);
      TN_CUDA(cudaMemcpyAsync(sn.Ab[s], t.Ab[s], eb * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      TN_CUDA(cudaMemcpyAsync(sn.Aa[s], t.Aa[s], ea * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      TN_CUDA(cudaMemcpyAsync(sn.B[s], t.B[s], e * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    }
    return sn;
  }

  // Shared (direction-independent) environment sweeps of layer ell over its
  // blocks: TT[s] / TB[s] = top (already gated with G^dag) / bottom block
  // tensor starting at site s (two-site pair for a gate block, the site
  // tensor for an idle site), taken from layer_hvp's block cache.
  // Left: L[0] = 1, L[e] = TT^H (L[s] TB); right: R[n] = 1, R[s] = (TB R[e]) TT^H.
  void shared_left(cudaStream_t st, Pool& pool, int ell, int tag, std::vector<cplx*>& L,
                   const std::vector<const cplx*>& TT, const std::vector<int>& tb, const std::vector<const cplx*>& TB,
                   const std::vector<int>& bb) {
    L.assign(n + 1, nullptr);
    L[0] = memo(st, pool, ell, 0, tag, 1, [&](cplx* o) { set_small(st, o, 1, ONE); });
    for (auto [s, k] : blocks(ell)) {
      const int w = k < 0 ? P : PP, e = k < 0 ? s + 1 : s + 2;
      L[e] = memo(st, pool, ell, e, tag, (int64_t)tb[e] * bb[e], [&](cplx* o) {
        Pool tmp(st);
        cplx* Y = tmp.c((int64_t)tb[s] * w * bb[e]);
        nn(st, tb[s], w * bb[e], bb[s], L[s], 0, TB[s], 0, Y, 0, 1);
        cn(st, tb[e], bb[e], w * tb[s], TT[s], 0, Y, 0, o, 0, 1);
      });
    }
  }

  void shared_right(cudaStream_t st, Pool& pool, int ell, int tag, std::vector<cplx*>& R,
                    const std::vector<const cplx*>& TT, const std::vector<int>& tb, const std::vector<const cplx*>& TB,
                    const std::vector<int>& bb) {
    R.assign(n + 1, nullptr);
    R[n] = memo(st, pool, ell, n, tag, 1, [&](cplx* o) { set_small(st, o, 1, ONE); });
    auto blks = blocks(ell);
    for (int j = (int)blks.size() - 1; j >= 0; --j) {
      const int s = blks[j].first, k = blks[j].second;
      const int w = k < 0 ? P : PP, e = k < 0 ? s + 1 : s + 2;
      R[s] = memo(st, pool, ell, s, tag, (int64_t)bb[s] * tb[s], [&](cplx* o) {
        Pool tmp(st);
        cplx* Y = tmp.c((int64_t)bb[s] * w * tb[e]);
        nn(st, w * bb[s], tb[e], bb[e], TB[s], 0, R[e], 0, Y, 0, 1);
        nc(st, bb[s], tb[s], w * tb[e], Y, 0, TT[s], 0, o, 0, 1);
      });
    }
  }

  // H_T contributions of layer ell (all three channels) for nb directions.
  void layer_hvp(cudaStream_t st, int ell, const TanSnap& DBs, const Tangent& DT, const cplx* V, cplx* HT, int nb,
                 bool skipB, bool skipT) {
    Pool pool(st);  // layer-lifetime buffers
    const auto tpv = snap_ptrs(top, D - ell);
    const auto bpv = snap_ptrs(bot, ell - 1);
    const auto& tb = top.snap[D - ell].p;
    const auto& bb = bot.snap[ell - 1].p;
    const auto& xb = DBs.bd.ab;  // bottom before-chain bonds
    const auto& ya = DBs.bd.aa;  // bottom after-chain bonds
    const auto& ub = DT.bd.ab;   // top before-chain bonds
    const auto& va = DT.bd.aa;   // top after-chain bonds
    std::vector<const cplx*> BAb(DBs.Ab.begin(), DBs.Ab.end()), BAa(DBs.Aa.begin(), DBs.Aa.end());
    std::vector<const cplx*> TAb(DT.Ab.begin(), DT.Ab.end()), TAa(DT.Aa.begin(), DT.Aa.end());
    const int64_t KK = (int64_t)K * 16;
    auto blks = blocks(ell);
    // per-direction right environments at every block boundary
    std::vector<cplx*> dRB(n + 1, nullptr), dRT(n + 1, nullptr), dRV(n + 1, nullptr);
    auto zero1 = [&](int64_t e) {
      cplx* p = pool.c(e * nb);
      TN_CUDA(cudaMemsetAsync(p, 0, (size_t)e * nb * sizeof(cplx), st));
      return p;
    };
    dRV[n] = zero1(1);
    if (!skipB) dRB[n] = zero1(1);
    if (!skipT) dRT[n] = zero1(1);
    // block tensors cache (per block start site)
    struct Blk {
      cplx *TT = nullptr, *TTg = nullptr, *BB = nullptr;          // primal blocks (TTg gated with G^dag)
      cplx* TTp = nullptr;                                          // TT with out legs split off
      cplx *BAaB = nullptr, *BAbB = nullptr, *BBd = nullptr;       // bottom chains + per-dir block
      cplx *TAaB = nullptr, *TAaG = nullptr, *TAbB = nullptr, *TAbG = nullptr, *TBd = nullptr, *TBdG = nullptr;
    };
    std::vector<Blk> bk(n);
    for (auto [s, k] : blks) {
      Blk& q = bk[s];
      const int e = k < 0 ? s + 1 : s + 2;
      const int w = k < 0 ? P : PP;
      auto mk2 = [&](int tag, const std::vector<const cplx*>& a, const std::vector<int>& bd) -> cplx* {
        if (k < 0) return const_cast<cplx*>(a[s]);
        return memo(st, pool, ell, s, tag, (int64_t)PP * bd[s] * bd[e],
                    [&](cplx* o) { pair(st, o, a[s], 0, a[s + 1], 0, bd[s], bd[s + 1], bd[e], 1); });
      };
      auto gated = [&](int tag, const cplx* x, int X, int Y) -> cplx* {
        if (k < 0) return const_cast<cplx*>(x);
        return memo(st, pool, ell, s, tag, (int64_t)PP * X * Y, [&](cplx* o) {
          apply_gate(st, o, 0, x, 0, at(o_gdag) + (int64_t)k * 16, 0, X, Y, 1, ONE, false, NI);
        });
      };
      q.TT = mk2(1, tpv, tb);
      q.TTg = gated(2, q.TT, tb[s], tb[e]);
      if (k >= 0)
        q.TTp = memo(st, pool, ell, s, 3, (int64_t)PP * tb[s] * tb[e],
                     [&](cplx* o) { out_leg_split(st, o, q.TT, tb[s], tb[e], NI); });
      q.BB = mk2(4, bpv, bb);
      if (!skipB) {
        q.BAaB = mk2(5, BAa, ya);
        q.BAbB = mk2(6, BAb, xb);
        const int64_t sz = (int64_t)w * xb[s] * ya[e];
        q.BBd = pool.c(sz * nb);
        if (k < 0) {
          TN_CUDA(cudaMemcpyAsync(q.BBd, DBs.B[s], sz * nb * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        } else {
          nn(st, P * xb[s], P * ya[e], ya[s + 1], DBs.B[s], bsize(DBs.bd, s), BAa[s + 1], 0, q.BBd, sz, nb);
          nn(st, P * xb[s], P * ya[e], xb[s + 1], BAb[s], 0, DBs.B[s + 1], bsize(DBs.bd, s + 1), q.BBd, sz, nb,
             ONE, ONE);
        }
      }
      if (!skipT) {
        q.TAaB = mk2(7, TAa, va);
        q.TAaG = gated(8, q.TAaB, va[s], va[e]);
        q.TAbB = mk2(9, TAb, ub);
        q.TAbG = gated(10, q.TAbB, ub[s], ub[e]);
        const int64_t sz = (int64_t)w * ub[s] * va[e];
        q.TBd = pool.c(sz * nb);
        if (k < 0) {
          TN_CUDA(cudaMemcpyAsync(q.TBd, DT.B[s], sz * nb * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
          q.TBdG = q.TBd;
        } else {
          nn(st, P * ub[s], P * va[e], va[s + 1], DT.B[s], bsize(DT.bd, s), TAa[s + 1], 0, q.TBd, sz, nb);
          nn(st, P * ub[s], P * va[e], ub[s + 1], TAb[s], 0, DT.B[s + 1], bsize(DT.bd, s + 1), q.TBd, sz, nb, ONE,
             ONE);
          q.TBdG = pool.c(sz * nb);
          apply_gate(st, q.TBdG, sz, q.TBd, sz, at(o_gdag) + (int64_t)k * 16, 0, ub[s], va[e], nb, ONE, false, NI);
        }
      }
    }
    // shared chain environments from the cached block tensors
    std::vector<cplx*> LBb, RBa, LTb, RTa;
    {
      std::vector<const cplx*> TTg(n), BAbB(n), BAaB(n), BBs(n), TAbG(n), TAaG(n);
      for (auto [s, k] : blks) {
        TTg[s] = bk[s].TTg;
        BAbB[s] = bk[s].BAbB;
        BAaB[s] = bk[s].BAaB;
        BBs[s] = bk[s].BB;
        TAbG[s] = bk[s].TAbG;
        TAaG[s] = bk[s].TAaG;
      }
      if (!skipB) {
        shared_left(st, pool, ell, 20, LBb, TTg, tb, BAbB, xb);
        shared_right(st, pool, ell, 21, RBa, TTg, tb, BAaB, ya);
      }
      if (!skipT) {
        shared_left(st, pool, ell, 22, LTb, TAbG, ub, BBs, bb);
        shared_right(st, pool, ell, 23, RTa, TAaG, va, BBs, bb);
      }
    }
    const cplx* Vd = V;  // [nb][K][16]
    // ---------------- right sweep (per direction)
    for (int j = (int)blks.size() - 1; j >= 0; --j) {
      const int s = blks[j].first, k = blks[j].second;
      const int w = k < 0 ? P : PP, e = k < 0 ? s + 1 : s + 2;
      Blk& q = bk[s];
      const cplx* R0e = at(o_R[ell][e]);
      Pool rp(st);  // block temporaries
      // V channel: dRV[s] = (BB dRV[e] + [V] BB R0[e]) TTg^H   (V replaces G: top ungated)
      {
        const int64_t sY = (int64_t)bb[s] * w * tb[e];
        cplx* Y = rp.c(sY * nb);
        nn(st, w * bb[s], tb[e], bb[e], q.BB, 0, dRV[e], (int64_t)bb[e] * tb[e], Y, sY, nb);
        dRV[s] = pool.c((int64_t)bb[s] * tb[s] * nb);
        nc(st, bb[s], tb[s], w * tb[e], Y, sY, q.TTg, 0, dRV[s], (int64_t)bb[s] * tb[s], nb);
        if (k >= 0) {  // (V Y0) TT^H = sum_ac V[a,c] Y0_c TT_a^H: 16 shared products, one K=16 GEMM
          const int64_t sq = (int64_t)bb[s] * tb[s], sy = (int64_t)bb[s] * NI2 * tb[e], stt = (int64_t)tb[s] * NI2 * tb[e];
          cplx* Q = memo(st, rp, ell, s, 60, 16 * sq, [&](cplx* o) {
            Pool tmp(st);
            cplx* Y0 = tmp.c(sY);
            nn(st, w * bb[s], tb[e], bb[e], q.BB, 0, R0e, 0, Y0, 0, 1);
            cplx* Y0p = tmp.c(sY);
            out_leg_split(st, Y0p, Y0, bb[s], tb[e], NI);
            for (int a = 0; a < 4; ++a)  // Q[a*4+c] = Y0p[c] TTp[a]^H
              nc(st, bb[s], tb[s], NI2 * tb[e], Y0p, sy, q.TTp + a * stt, 0, o + (int64_t)a * 4 * sq, sq, 4);
          });
          mm(st, 'N', 'N', nb, (int)sq, 16, ONE, Vd + (int64_t)k * 16, KK, 0, Q, sq, 0, ONE, dRV[s], sq, 0, 1);
        }
      }
      if (!skipB) {  // dRB[s] = (BAbB dRB[e] + BBd RBa[e]) TTg^H
        const int64_t sY = (int64_t)xb[s] * w * tb[e];
        cplx* Y = rp.c(sY * nb);
        nn(st, w * xb[s], tb[e], xb[e], q.BAbB, 0, dRB[e], (int64_t)xb[e] * tb[e], Y, sY, nb);
        nn(st, w * xb[s], tb[e], ya[e], q.BBd, (int64_t)w * xb[s] * ya[e], RBa[e], 0, Y, sY, nb, ONE, ONE);
        dRB[s] = pool.c((int64_t)xb[s] * tb[s] * nb);
        nc(st, xb[s], tb[s], w * tb[e], Y, sY, q.TTg, 0, dRB[s], (int64_t)xb[s] * tb[s], nb);
      }
      if (!skipT) {  // dRT[s] = (BB dRT[e]) TAbG^H + (BB RTa[e]) TBdG^H
        const int64_t sY = (int64_t)bb[s] * w * ub[e];
        cplx* Y = rp.c(sY * nb);
        nn(st, w * bb[s], ub[e], bb[e], q.BB, 0, dRT[e], (int64_t)bb[e] * ub[e], Y, sY, nb);
        dRT[s] = pool.c((int64_t)bb[s] * ub[s] * nb);
        nc(st, bb[s], ub[s], w * ub[e], Y, sY, q.TAbG, 0, dRT[s], (int64_t)bb[s] * ub[s], nb);
        const int64_t sY2 = (int64_t)bb[s] * w * va[e];
        cplx* Y2 = memo(st, rp, ell, s, 61, sY2,
                        [&](cplx* o) { nn(st, w * bb[s], va[e], bb[e], q.BB, 0, RTa[e], 0, o, 0, 1); });
        nc(st, bb[s], ub[s], w * va[e], Y2, 0, q.TBdG, (int64_t)w * ub[s] * va[e], dRT[s], (int64_t)bb[s] * ub[s],
           nb, ONE, ONE);
      }
    }
    // ---------------- left sweep with extraction
    auto zero_owned = [&](int64_t e) {
      cplx* p = dnew(e * nb, st);
      TN_CUDA(cudaMemsetAsync(p, 0, (size_t)e * nb * sizeof(cplx), st));
      return p;
    };
    cplx* dLV = zero_owned(1);
    cplx* dLB = skipB ? nullptr : zero_owned(1);
    cplx* dLT = skipT ? nullptr : zero_owned(1);
    for (auto [s, k] : blks) {
      const int w = k < 0 ? P : PP, e = k < 0 ? s + 1 : s + 2;
      Blk& q = bk[s];
      Pool bpool(st);  // block temporaries
      const cplx* L0s = at(o_L[ell][s]);
      const cplx* R0e = at(o_R[ell][e]);
      // Y tensors (open gate, bottom side), per direction, top-index rows: (t x w x b')
      const int64_t sYV = (int64_t)tb[s] * w * bb[e];
      cplx* YV = bpool.c(sYV * nb);  // dLV BB
      nn(st, tb[s], w * bb[e], bb[s], dLV, (int64_t)tb[s] * bb[s], q.BB, 0, YV, sYV, nb);
      cplx* Y0 = nullptr;  // L0 BB (shared)
      if (k >= 0)
        Y0 = memo(st, bpool, ell, s, 70, sYV, [&](cplx* o) { nn(st, tb[s], w * bb[e], bb[s], L0s, 0, q.BB, 0, o, 0, 1); });
      cplx* YB = nullptr;
      int64_t sYB = 0;
      if (!skipB) {  // dLB BAaB + LBb BBd : (t x w x ya')
        sYB = (int64_t)tb[s] * w * ya[e];
        YB = bpool.c(sYB * nb);
        nn(st, tb[s], w * ya[e], ya[s], dLB, (int64_t)tb[s] * ya[s], q.BAaB, 0, YB, sYB, nb);
        nn(st, tb[s], w * ya[e], xb[s], LBb[s], 0, q.BBd, (int64_t)w * xb[s] * ya[e], YB, sYB, nb, ONE, ONE);
      }
      cplx* YT = nullptr;
      cplx* YT0 = nullptr;
      int64_t sYT = 0;
      if (!skipT) {  // dLT BB : (va x w x b') ; LTb BB (shared) : (ub x w x b')
        sYT = (int64_t)va[s] * w * bb[e];
        YT = bpool.c(sYT * nb);
        nn(st, va[s], w * bb[e], bb[s], dLT, (int64_t)va[s] * bb[s], q.BB, 0, YT, sYT, nb);
        YT0 = memo(st, bpool, ell, s, 71, (int64_t)ub[s] * w * bb[e],
                   [&](cplx* o) { nn(st, ub[s], w * bb[e], bb[s], LTb[s], 0, q.BB, 0, o, 0, 1); });
      }
      if (k >= 0) {
        // ---- extraction.  Terms whose right environment R is shared across
        // directions use Wt = Theta_top R^H (once per block) so that
        // sum conj(top) (Y R) = sum conj(Wt) Y  -- no per-direction Y R product.
        {
          cplx* Wt = memo(st, bpool, ell, s, 72, (int64_t)PP * tb[s] * bb[e],   // TT R0^H
                          [&](cplx* o) { nc(st, PP * tb[s], bb[e], tb[e], q.TT, 0, R0e, 0, o, 0, 1); });
          extract_env(st, HT + (int64_t)k * 16, KK, Wt, 0, YV, sYV, tb[s], bb[e], nb, ONE, NI);
        }
        {  // per-direction right environments: Z = Y0 dRV (+ LBb BAbB dRB)
          const int64_t sZ = (int64_t)PP * tb[s] * tb[e];
          cplx* Z = bpool.c(sZ * nb);
          nn(st, PP * tb[s], tb[e], bb[e], Y0, 0, dRV[e], (int64_t)bb[e] * tb[e], Z, sZ, nb);
          if (!skipB) {
            cplx* LBA = memo(st, bpool, ell, s, 73, (int64_t)PP * tb[s] * xb[e],
                             [&](cplx* o) { nn(st, tb[s], PP * xb[e], xb[s], LBb[s], 0, q.BAbB, 0, o, 0, 1); });
            nn(st, PP * tb[s], tb[e], xb[e], LBA, 0, dRB[e], (int64_t)xb[e] * tb[e], Z, sZ, nb, ONE, ONE);
          }
          extract_env(st, HT + (int64_t)k * 16, KK, q.TT, 0, Z, sZ, tb[s], tb[e], nb, ONE, NI);
        }
        if (!skipB) {  // (dLB BAaB + LBb BBd) RBa  ->  Wt = TT RBa^H
          cplx* Wt = memo(st, bpool, ell, s, 74, (int64_t)PP * tb[s] * ya[e],
                          [&](cplx* o) { nc(st, PP * tb[s], ya[e], tb[e], q.TT, 0, RBa[e], 0, o, 0, 1); });
          extract_env(st, HT + (int64_t)k * 16, KK, Wt, 0, YB, sYB, tb[s], ya[e], nb, ONE, NI);
        }
        if (!skipT) {
          {  // top TAaB with (dLT BB) RTa  ->  Wt = TAaB RTa^H
            cplx* Wt = memo(st, bpool, ell, s, 75, (int64_t)PP * va[s] * bb[e],
                            [&](cplx* o) { nc(st, PP * va[s], bb[e], va[e], q.TAaB, 0, RTa[e], 0, o, 0, 1); });
            extract_env(st, HT + (int64_t)k * 16, KK, Wt, 0, YT, sYT, va[s], bb[e], nb, ONE, NI);
          }
          // per-dir top TBd with shared (LTb BB) RTa
          const int64_t sZ3 = (int64_t)PP * ub[s] * va[e];
          cplx* Z3 = memo(st, bpool, ell, s, 76, sZ3,
                          [&](cplx* o) { nn(st, PP * ub[s], va[e], bb[e], YT0, 0, RTa[e], 0, o, 0, 1); });
          extract_env(st, HT + (int64_t)k * 16, KK, q.TBd, sZ3, Z3, 0, ub[s], va[e], nb, ONE, NI);
          // top TAbB with (LTb BB) dRT
          const int64_t sZ4 = (int64_t)PP * ub[s] * ub[e];
          cplx* Z4 = bpool.c(sZ4 * nb);
          nn(st, PP * ub[s], ub[e], bb[e], YT0, 0, dRT[e], (int64_t)bb[e] * ub[e], Z4, sZ4, nb);
          extract_env(st, HT + (int64_t)k * 16, KK, q.TAbB, 0, Z4, sZ4, ub[s], ub[e], nb, ONE, NI);
        }
      }
      // ---- left updates
      {  // dLV' = TT^H (G YV + V Y0)  ==  TTg^H YV + TT^H (V Y0)
        cplx* nL = dnew((int64_t)tb[e] * bb[e] * nb, st);
        cn(st, tb[e], bb[e], w * tb[s], q.TTg, 0, YV, sYV, nL, (int64_t)tb[e] * bb[e], nb);
        if (k >= 0) {  // TT^H (V Y0) = sum_ac V[a,c] TT_a^H Y0_c: 16 shared products, one K=16 GEMM
          const int64_t sp = (int64_t)tb[e] * bb[e], sy = (int64_t)tb[s] * NI2 * bb[e], stt = (int64_t)tb[s] * NI2 * tb[e];
          cplx* Pm = memo(st, bpool, ell, s, 77, 16 * sp, [&](cplx* o) {
            Pool tmp(st);
            cplx* Y0p = tmp.c(sYV);
            out_leg_split(st, Y0p, Y0, tb[s], bb[e], NI);
            for (int a = 0; a < 4; ++a)  // P[a*4+c] = TTp[a]^H Y0p[c]
              cn(st, tb[e], bb[e], NI2 * tb[s], q.TTp + a * stt, 0, Y0p, sy, o + (int64_t)a * 4 * sp, sp, 4);
          });
          mm(st, 'N', 'N', nb, (int)sp, 16, ONE, Vd + (int64_t)k * 16, KK, 0, Pm, sp, 0, ONE, nL, sp, 0, 1);
        }
        dset(dLV, nL, st);
      }
      if (!skipB) {
        cplx* nL = dnew((int64_t)tb[e] * ya[e] * nb, st);
        cn(st, tb[e], ya[e], w * tb[s], q.TTg, 0, YB, sYB, nL, (int64_t)tb[e] * ya[e], nb);
        dset(dLB, nL, st);
      }
      if (!skipT) {
        cplx* nL = dnew((int64_t)va[e] * bb[e] * nb, st);
        cn(st, va[e], bb[e], w * va[s], q.TAaG, 0, YT, sYT, nL, (int64_t)va[e] * bb[e], nb);
        cn(st, va[e], bb[e], w * ub[s], q.TBdG, (int64_t)w * ub[s] * va[e], YT0, 0, nL, (int64_t)va[e] * bb[e], nb,
           ONE, ONE);
        dset(dLT, nL, st);
      }
    }
    ddel(dLV, st);
    ddel(dLB, st);
    ddel(dLT, st);
  }

  // a6: forward (bottom) tangents of nb directions, cached per layer: DB[ell-1]
  // holds DB_{ell-1}.  before_layer(li), when given, runs on the host before
  // the steps of bottom layer li are issued (fused step: waits for the sweep).
  std::vector<TanSnap> forward_tangents(cudaStream_t st, int nb, const cplx* V,
                                        const std::function<void(int)>& before_layer = nullptr) {
    std::vector<TanSnap> DB(D);
    Tangent t;
    tangent_init(st, t, bot, false, nb, chain_cache_for(0, st));
    for (size_t li = 0; li < bot.steps.size(); ++li) {
      DB[li] = take_snapshot(st, t, nb);
      if (before_layer) before_layer((int)li);
      for (const Step& s : bot.steps[li]) tangent_step(st, t, s, at(o_gates), V, nb);
    }
    release(t, st);
    return DB;
  }

  void apply(cudaStream_t st, int batch, const cplx* dirs, cplx* hess, cplx* aux,
             std::vector<TanSnap>* first_fwd = nullptr) {
    TN_CUDA(cudaSetDevice(device));
    if (!primal_valid) throw StateError("tn_hvp_apply before tn_hvp_environments");
    const double wc0 = work_counter.load();
    const int64_t KK = (int64_t)K * 16;
    for (int b0 = 0; b0 < batch; b0 += cfg.max_batch) {
      const int nb = std::min(cfg.max_batch, batch - b0);
      Pool pool(st);
      const cplx* V = dirs + (int64_t)b0 * KK;
      cplx* Vd = pool.c(KK * nb);
      dagger4(st, Vd, V, (int64_t)K * nb);
      cplx* HT = pool.c(KK * nb);
      TN_CUDA(cudaMemsetAsync(HT, 0, (size_t)KK * nb * sizeof(cplx), st));
      const bool phases = std::getenv("TN_PHASES") != nullptr;
      cudaEvent_t pe[4];
      if (phases)
        for (auto& e : pe) TN_CUDA(cudaEventCreate(&e));
      float t_fwd = 0, t_bwd = 0, t_hvp = 0;
      if (phases) TN_CUDA(cudaEventRecord(pe[0], st));
      // forward (bottom) tangent, cached per layer: DB_{ell-1} (precomputed
      // for the first sub-batch by the fused step)
      std::vector<TanSnap> DB = (b0 == 0 && first_fwd && !first_fwd->empty()) ? std::move(*first_fwd)
                                                                               : forward_tangents(st, nb, V);
      if (phases) {
        TN_CUDA(cudaEventRecord(pe[1], st));
        TN_CUDA(cudaEventSynchronize(pe[1]));
        TN_CUDA(cudaEventElapsedTime(&t_fwd, pe[0], pe[1]));
      }
      // backward (top) tangent on the fly + layer HVP extraction
      Tangent t;
      tangent_init(st, t, top, true, nb, chain_cache_for(1, st));
      for (size_t li = 0; li < top.steps.size(); ++li) {
        const int ell = top.ell[li];
        if (phases) TN_CUDA(cudaEventRecord(pe[2], st));
        layer_hvp(st, ell, DB[ell - 1], t, V, HT, nb, ell == 1, li == 0);
        release(DB[ell - 1], st);
        if (phases) {
          TN_CUDA(cudaEventRecord(pe[3], st));
          TN_CUDA(cudaEventSynchronize(pe[3]));
          float a = 0;
          TN_CUDA(cudaEventElapsedTime(&a, pe[2], pe[3]));
          t_hvp += a;
          TN_CUDA(cudaEventRecord(pe[2], st));
        }
        for (const Step& s : top.steps[li]) tangent_step(st, t, s, at(o_gdag), Vd, nb);
        if (phases) {
          TN_CUDA(cudaEventRecord(pe[3], st));
          TN_CUDA(cudaEventSynchronize(pe[3]));
          float a = 0;
          TN_CUDA(cudaEventElapsedTime(&a, pe[2], pe[3]));
          t_bwd += a;
        }
      }
      release(t, st);
      if (phases) {
        fprintf(stderr, "[tn phases] sub-batch %d: forward tangent %.1f ms, backward tangent %.1f ms, layer HVP %.1f ms\n",
                nb, t_fwd, t_bwd, t_hvp);
        for (auto& e : pe) cudaEventDestroy(e);
      }
      cplx* om = pool.c(nb);
      hessian_post(st, K, nb, at(o_gates), at(o_E), at(o_gradf), at<double>(o_scal), HT, V, om,
                   hess + (int64_t)b0 * KK);
      if (aux) {
        TN_CUDA(cudaMemcpyAsync(aux + (int64_t)b0 * KK, HT, (size_t)KK * nb * sizeof(cplx), cudaMemcpyDeviceToDevice,
                                st));
        TN_CUDA(cudaMemcpyAsync(aux + (int64_t)batch * KK + b0, om, (size_t)nb * sizeof(cplx),
                                cudaMemcpyDeviceToDevice, st));
      }
    }
    work_apply = (work_counter.load() - wc0 + work_fwd_first) / std::max(batch, 1);
    work_fwd_first = 0;
  }

  // Replays run on the caller's stream: wait for that stream only (not the
  // device) before the executable graphs and their I/O buffers go.
  // all = false (every primal pass): only the point-specific graphs go (they
  // replay per-point caches); point-free graphs read everything point-specific
  // from the store at run time and stay.
  void drop_graphs(cudaStream_t st, bool all = false) {
    bool any = false;
    for (ApplyGraph& g : graphs) any = any || all || !g.point_free;
    if (!any) return;
    TN_CUDA(cudaStreamSynchronize(st));
    std::vector<ApplyGraph> keep;
    for (ApplyGraph& g : graphs) {
      if (!all && g.point_free) {
        keep.push_back(g);
        continue;
      }
      if (g.exec) cudaGraphExecDestroy(g.exec);
      for (cplx* p : {g.in, g.out, g.auxb}) dfree(p, st);
    }
    graphs.swap(keep);
    cudaDeviceGraphMemTrim(device);
  }

  // The inputs of the stored point change: nothing of it may be reused.
  void invalidate(cudaStream_t st) {
    primal_valid = false;
    ti_valid = false;
    applies_at_point = 0;
    drop_graphs(st);
    drop_chain_cache(st);
  }

  // tn_hvp_trim_memory: drop the per-point caches and graphs (rebuilt by the
  // next apply) and return the library pool's unused blocks to the device.
  void trim_memory(cudaStream_t st) {
    drop_graphs(st, true);
    drop_chain_cache(st);
    TN_CUDA(cudaStreamSynchronize(st));
    pool_trim(device);
  }

  bool capture(ApplyGraph& g, cudaStream_t st) {
    const int64_t n = (int64_t)g.batch * K * 16;
    g.in = (cplx*)dalloc(sizeof(cplx) * n, st);
    g.out = (cplx*)dalloc(sizeof(cplx) * n, st);
    if (g.aux) g.auxb = (cplx*)dalloc(sizeof(cplx) * (n + g.batch), st);
    TN_CUDA(cudaMemsetAsync(g.in, 0, sizeof(cplx) * n, st));
    // the capture stream starts after the caller's stream (buffers ready)
    TN_CUDA(cudaEventRecord(ev_fork, st));
    TN_CUDA(cudaStreamWaitEvent(stc, ev_fork, 0));
    const int64_t l0 = launch_count();
    const double w0 = work_counter.load();
    cudaGraph_t graph = nullptr;
    TN_CUDA(cudaStreamBeginCapture(stc, cudaStreamCaptureModeThreadLocal));
    bool ok = true;
    no_cache = g.point_free;
    try {
      apply(stc, g.batch, g.in, g.out, g.aux ? g.auxb : nullptr);
    } catch (...) {
      ok = false;
    }
    no_cache = false;
    const cudaError_t e = cudaStreamEndCapture(stc, &graph);
    g.launches = launch_count() - l0;
    g.work = work_counter.load() - w0;
    g.work_apply = work_apply;
    count_launch(-g.launches);  // captured, not executed: credited per replay
    work_counter.fetch_add(-g.work, std::memory_order_relaxed);
    if (!ok || e != cudaSuccess || !graph) {
      cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      return false;
    }
    const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
      cudaGetLastError();
      g.exec = nullptr;
      return false;
    }
    return true;
  }

  // A point-free graph owns its working memory for its lifetime: only when one
  // apply's tangent state plus the uncached chains fit in 1/16 of the device.
  bool point_free_ok(int batch) {
    size_t fr = 0, tot = 0;
    TN_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t need = per_direction_bytes() * (size_t)std::min(batch, cfg.max_batch) + chain_cache_bytes();
    return need < tot / 16 && need < fr / 4;
  }

  // tn_hvp_apply entry: eager, or graph replay for a repeated (batch, aux)
  void apply_call(cudaStream_t st, int batch, const cplx* dirs, cplx* hess, cplx* aux) {
    TN_CUDA(cudaSetDevice(device));
    if (!primal_valid) throw StateError("tn_hvp_apply before tn_hvp_environments");
    check_dirs(st, at(o_gates), dirs, batch);
    // graphs pay off for launch-bound small batches (truncated CG: batch 1);
    // large batches are GEMM-bound and would double the memory footprint
    const bool first = ++applies_at_point == 1;
    if (!graphs_enabled || batch <= 0 || gemm_profile_active() || std::getenv("TN_PHASES")) {
      apply(st, batch, dirs, hess, aux);
      return;
    }
    // First apply at a point: a point-free graph (no per-point caches, the
    // frozen factors read from the store on the device) captured once per
    // (batch, aux) and replayed at every later point -- launch-bound small
    // configurations -- when its graph-owned working memory is small.
    // Repeated applies at one point (truncated CG): per-point caches recorded
    // by an eager call, then a point-specific graph that replays them.
    const bool pf = first && point_free_ok(batch);
    if (!pf && batch > kGraphMaxBatch) {
      apply(st, batch, dirs, hess, aux);
      return;
    }
    ApplyGraph* g = nullptr;
    for (ApplyGraph& x : graphs)
      if (x.batch == batch && x.aux == (aux != nullptr) && x.point_free == pf) g = &x;
    if (!g) {
      graphs.push_back(ApplyGraph{});
      g = &graphs.back();
      g->batch = batch;
      g->aux = aux != nullptr;
      g->point_free = pf;
      if (pf) g->calls = 1;  // captured at once: the capture costs about one eager call
    }
    if (++g->calls == 1 || g->failed) {
      apply(st, batch, dirs, hess, aux);
      return;
    }
    if (!g->exec && !capture(*g, st)) {
      g->failed = true;
      apply(st, batch, dirs, hess, aux);
      return;
    }
    const int64_t n = (int64_t)batch * K * 16;
    TN_CUDA(cudaMemcpyAsync(g->in, dirs, sizeof(cplx) * n, cudaMemcpyDeviceToDevice, st));
    if (cudaGraphLaunch(g->exec, st) != cudaSuccess) {  // e.g. graph memory: run eagerly from now on
      cudaGetLastError();
      cudaGraphExecDestroy(g->exec);
      g->exec = nullptr;
      g->failed = true;
      cudaDeviceGraphMemTrim(device);
      apply(st, batch, dirs, hess, aux);
      return;
    }
    TN_CUDA(cudaMemcpyAsync(hess, g->out, sizeof(cplx) * n, cudaMemcpyDeviceToDevice, st));
    if (aux) TN_CUDA(cudaMemcpyAsync(aux, g->auxb, sizeof(cplx) * (n + batch), cudaMemcpyDeviceToDevice, st));
    count_launch(g->launches);
    work_counter.fetch_add(g->work, std::memory_order_relaxed);
    work_apply = g->work_apply;
  }

  // Fused step (tn_hvp_step): environments + HVPs of `batch` directions, with
  // the first sub-batch's forward tangents replayed on a fourth stream while
  // the top sweep and the layer gradients still run (the forward tangent of
  // bottom layer li needs only the bottom sweep's replay data up to li).
  void step(cudaStream_t st, const cplx* gates, double* scalars, cplx* grad_R, int batch, const cplx* dirs,
            cplx* hess, cplx* aux) {
    if (batch == 0) {
      environments(st, gates, scalars, grad_R);
      return;
    }
    check_gates(st, gates, K);
    check_dirs(st, gates, dirs, batch);
    // (measured: at C2 / C3 the point-free apply graph alone gains what the
    // forward-tangent overlap of the fused step gains -- 307 vs 298 ms per C2
    // step, 3.08 s either way at C3 -- so the step stays fused)
    std::vector<TanSnap> DB0;
    environments(st, gates, scalars, grad_R, std::min(batch, cfg.max_batch), dirs, &DB0);
    apply(st, batch, dirs, hess, aux, &DB0);
  }
};

}  // namespace tn

struct tn_hvp_ctx {
  tn::Engine e;
};

namespace tn {

tn_hvp_ctx* engine_create(const tn_hvp_config& cfg, const int32_t* ref_bonds, const void* ref_mpo, void* primal_buf,
                          size_t primal_bytes, cudaStream_t st) {
  auto ctx = std::make_unique<tn_hvp_ctx>();
  ctx->e.setup(cfg, ref_bonds, ref_mpo, primal_buf, primal_bytes, st);
  TN_CUDA(cudaStreamSynchronize(st));
  return ctx.release();
}
void engine_environments(tn_hvp_ctx* ctx, const cplx* gates, double* scalars, cplx* grad_R, cudaStream_t st) {
  ctx->e.environments(st, gates, scalars, grad_R);
}
void engine_apply(tn_hvp_ctx* ctx, int batch, const cplx* dirs, cplx* hess_R, cplx* aux, cudaStream_t st) {
  ctx->e.apply_call(st, batch, dirs, hess_R, aux);
}
void engine_step(tn_hvp_ctx* ctx, const cplx* gates, double* scalars, cplx* grad_R, int batch, const cplx* dirs,
                 cplx* hess_R, cplx* aux, cudaStream_t st) {
  ctx->e.step(st, gates, scalars, grad_R, batch, dirs, hess_R, aux);
}
void engine_ti_environments(tn_hvp_ctx* ctx, const cplx* g, double* scalars, cplx* grad_R, cudaStream_t st) {
  ctx->e.ti_environments(st, g, scalars, grad_R);
}
void engine_ti_apply(tn_hvp_ctx* ctx, int batch, const cplx* v, cplx* hess_R, cudaStream_t st) {
  ctx->e.ti_apply(st, batch, v, hess_R);
}
void engine_gradient_T(tn_hvp_ctx* ctx, cplx* E, cudaStream_t st) {
  if (!ctx->e.primal_valid) throw StateError("no primal pass");
  TN_CUDA(cudaMemcpyAsync(E, ctx->e.at(ctx->e.o_E), (size_t)ctx->e.K * 16 * sizeof(cplx), cudaMemcpyDeviceToDevice,
                          st));
}
void engine_cost(tn_hvp_ctx* ctx, const cplx* gates, double* scalars, cudaStream_t st) {
  ctx->e.cost(st, gates, scalars);
}
void engine_primal_blob(tn_hvp_ctx* ctx, void** ptr, size_t* bytes) {
  *ptr = ctx->e.arena;
  *bytes = ctx->e.arena_bytes;
}
// After a collective filled the primal store (tn_hvp_primal_copy into the
// context): the blob carries the point's gates (o_gates); they must be the
// caller's `gates` bit for bit, else TN_EINVAL and the store stays invalid.
void engine_primal_imported(tn_hvp_ctx* ctx, const cplx* gates, cudaStream_t st) {
  Engine& e = ctx->e;
  TN_CUDA(cudaSetDevice(e.device));
  e.primal_valid = false;
  e.ti_valid = false;
  e.drop_graphs(st);
  e.drop_chain_cache(st);
  std::vector<cplx> hg((size_t)e.K * 16), hb((size_t)e.K * 16);
  TN_CUDA(cudaMemcpyAsync(hg.data(), gates, sizeof(cplx) * hg.size(), cudaMemcpyDeviceToHost, st));
  TN_CUDA(cudaMemcpyAsync(hb.data(), e.at(e.o_gates), sizeof(cplx) * hb.size(), cudaMemcpyDeviceToHost, st));
  TN_CUDA(cudaStreamSynchronize(st));
  if (std::memcmp(hg.data(), hb.data(), sizeof(cplx) * hg.size()) != 0)
    throw std::invalid_argument("tn_hvp_primal_imported: gates differ from the imported primal store's point");
  e.primal_valid = true;
}
// tn_hvp_primal_copy: into_ctx = 1 overwrites the store, so everything that
// describes the old point is invalidated first (valid again after
// tn_hvp_primal_imported).
void engine_primal_copy(tn_hvp_ctx* ctx, void* buf, size_t bytes, int into_ctx, cudaStream_t st) {
  Engine& e = ctx->e;
  TN_CUDA(cudaSetDevice(e.device));
  if (bytes != e.arena_bytes) throw std::invalid_argument("tn_hvp_primal_copy: size mismatch");
  if (into_ctx) {
    e.primal_valid = false;
    e.ti_valid = false;
    e.drop_graphs(st);
    e.drop_chain_cache(st);
    if (buf != e.arena)  // buf == the store: the caller fills it in place (invalidate only)
      TN_CUDA(cudaMemcpyAsync(e.arena, buf, bytes, cudaMemcpyDeviceToDevice, st));
  } else {
    if (!e.primal_valid) throw StateError("tn_hvp_primal_copy: no valid primal pass to export");
    TN_CUDA(cudaMemcpyAsync(buf, e.arena, bytes, cudaMemcpyDeviceToDevice, st));
  }
}
void engine_set_product_state(tn_hvp_ctx* ctx, const cplx* psi, cudaStream_t st) {
  Engine& e = ctx->e;
  if (e.P != 2) throw std::invalid_argument("tn_hvp_set_product_state: the context is in operator mode (site_dim 4)");
  TN_CUDA(cudaSetDevice(e.device));
  e.invalidate(st);
  TN_CUDA(cudaMemcpyAsync(e.d_init, psi, sizeof(cplx) * 2 * e.n, cudaMemcpyDeviceToDevice, st));
}
void engine_set_reference(tn_hvp_ctx* ctx, const cplx* ref, cudaStream_t st) {
  Engine& e = ctx->e;
  TN_CUDA(cudaSetDevice(e.device));
  e.invalidate(st);
  size_t el = 0;
  for (int s = 0; s < e.n; ++s) el += (size_t)e.ref_bonds[s] * e.P * e.ref_bonds[s + 1];
  TN_CUDA(cudaMemcpyAsync(e.ref, ref, sizeof(cplx) * el, cudaMemcpyDeviceToDevice, st));
}
void engine_set_cache_budget(tn_hvp_ctx* ctx, size_t bytes) { ctx->e.cache_budget = bytes; }
void engine_environments_part(tn_hvp_ctx* ctx, const cplx* gates, int part, cudaStream_t st) {
  ctx->e.environments_part(st, gates, part);
}
void engine_environments_finish(tn_hvp_ctx* ctx, const cplx* gates, double* scalars, cplx* grad_R,
                                cudaStream_t st) {
  ctx->e.environments_finish(st, gates, scalars, grad_R);
}
void engine_primal_region(tn_hvp_ctx* ctx, int part, size_t* offset, size_t* bytes) {
  *offset = ctx->e.o_side[part];
  *bytes = ctx->e.o_side[part + 1] - ctx->e.o_side[part];
}
void engine_trim_memory(tn_hvp_ctx* ctx, cudaStream_t st) {
  TN_CUDA(cudaSetDevice(ctx->e.device));
  ctx->e.trim_memory(st);
}
void engine_tebd(int n, int ngates, const int32_t* sites, const cplx* gates, int chi, double tol, int device,
                 int32_t* bonds_out, cplx* out, size_t cap, cudaStream_t st) {
  Engine e;
  e.device = device;
  std::vector<int> b;
  e.tebd(st, n, ngates, sites, gates, chi, tol, b, out, cap);
  for (int s = 0; s <= n; ++s) bonds_out[s] = b[s];
  if (e.sol[0].h) {
    cusolverDnDestroy(e.sol[0].h);
    e.sol[0].h = nullptr;
  }
}
void engine_query(const tn_hvp_config& cfg, const int32_t* ref_bonds, size_t* primal_bytes, size_t* work_bytes,
                  size_t* per_dir_bytes) {
  Engine e;
  e.plan(cfg, ref_bonds);
  *primal_bytes = e.arena_bytes;
  *work_bytes = e.chain_cache_bytes();
  *per_dir_bytes = e.per_direction_bytes();
}
void engine_work(tn_hvp_ctx* ctx, double* per_dir, double* primal) {
  *per_dir = ctx->e.work_apply;
  *primal = ctx->e.work_primal;
}
void engine_split_stats(tn_hvp_ctx* ctx, int64_t* out6) {
  Engine& e = ctx->e;
  out6[0] = e.n_fallback.load();
  out6[1] = e.n_deflate.load();
  out6[2] = e.n_noise.load();
  out6[3] = e.n_lowrank.load();
  out6[4] = e.n_cholqr_fallback.load();
  out6[5] = e.n_pair_steps;
}
void engine_destroy(tn_hvp_ctx* ctx) { delete ctx; }
void engine_set_error(tn_hvp_ctx* ctx, const std::string& msg) { ctx->e.err = msg; }
const char* engine_error(const tn_hvp_ctx* ctx) { return ctx->e.err.c_str(); }

}  // namespace tn
