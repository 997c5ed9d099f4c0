/*
 * tn_hvp.h -- C ABI of the B200 (sm_100a) Hessian-vector-product kernel for
 * brickwall circuits compressed against an MPO reference
 * (arXiv:2604.20384, "Hessian-vector products for tensor networks via
 * recursive tangent-state propagation").
 *
 * Problem:
 *   W = L_D ... L_1, layer L_ell = tensor product of two-qubit gates G_k on the
 *   pairs (off, off+1), (off+2, off+3), ... with off = (first_offset+ell-1)%2;
 *   gate index k layer-major, left->right (reading X5).
 *   T = Tr(U_ref^dag W) / 2^n,  f = -|T|^2  (BASELINE.json config 1).
 *   The reference U_ref/2^{n/2} is an MPO (site tensors [b_s][4][b_{s+1}],
 *   p = 2*out + in, right-canonical, centre at site 0).
 *   Bond cap chi: every two-site split keeps r = min(chi, 4 m, 4 b_l, 4 b_r)
 *   singular values and rescales to the pre-truncation norm; tangents are
 *   propagated with the primal's frozen Schmidt projectors (App. D,
 *   PAPER.md:1019-1023; readings X7-X9).
 *
 * Numbers: complex128 interleaved (re, im) = 16 bytes, row-major.
 *   gates [K][4][4]: row index = 2 q_i + q_{i+1} of the gate OUTPUT.
 *   directions [B][K][4][4], outputs likewise.
 *
 * Ownership: every pointer argument is CALLER-owned.  Device pointers must
 * stay valid for the duration of the call (stream-ordered).  The primal store
 * (tn_hvp_query's primal_bytes) is either caller-owned (primal_buf of
 * tn_hvp_setup, kept until tn_hvp_destroy) or allocated by the context.  The
 * context owns its cuSOLVER handles, internal streams and the transient
 * buffers of a call; those come from a stream-ordered cudaMemPool private to
 * this library (never the device's default pool), whose cached blocks are
 * returned by tn_hvp_trim_memory and tn_hvp_destroy.  The primal store is one
 * flat byte range (tn_hvp_primal_blob) so a collective can move it.
 *
 * Streams: `stream` is a cudaStream_t passed as void*; all device work is
 * enqueued on it (the primal pass forks internal streams and joins them back
 * into it).  Calls on one context must be stream-ordered: the same stream, or
 * the caller orders them.  No call synchronises the device; calls that must
 * read a device value on the host synchronise `stream` and say so.
 *
 * Errors: every call returns tn_status and never throws across the ABI.
 *   TN_EINVAL  argument error, detected before any launch;
 *   TN_ENOMEM  arena allocation failed;
 *   TN_ECUDA   CUDA / cuSOLVER error (text via tn_hvp_last_error);
 *   TN_ENUMERIC SVD non-convergence or non-finite output;
 *   TN_ESTATE  tn_hvp_apply before tn_hvp_environments for the current gates.
 * There is no CPU fallback: without a CUDA device every compute call returns
 * TN_ECUDA.
 */
#ifndef TN_HVP_H
#define TN_HVP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { TN_OK = 0, TN_EINVAL = 1, TN_ENOMEM = 2, TN_ECUDA = 3, TN_ENUMERIC = 4, TN_ESTATE = 5 } tn_status;

/* Arithmetic type.  Only complex128 is built (north_star's complex64 mode is
 * optional and not implemented: TN_C64 returns TN_EINVAL). */
typedef enum { TN_C128 = 0, TN_C64 = 1 } tn_dtype;

/* Argument checks, each costs one small kernel and a
 * stream synchronisation per call:
 *   TN_CHECK_UNITARY: every gate of environments / step / cost has
 *     ||G^dag G - I||_F <= 1e-10, else TN_EINVAL before any other work;
 *   TN_CHECK_TANGENT: every direction of apply / step has
 *     ||V - P_G V|| <= 1e-8 ||V|| (norms over all K gates), else TN_EINVAL. */
#define TN_CHECK_UNITARY 1u
#define TN_CHECK_TANGENT 2u

typedef struct tn_hvp_ctx tn_hvp_ctx;

typedef struct {
  int32_t n_sites;      /* n >= 2                                               */
  int32_t depth;        /* D >= 1 brickwall layers                              */
  int32_t first_offset; /* 0 | 1: first layer on (0,1),(2,3).. or (1,2),(3,4).. */
  int32_t chi;          /* primal bond cap; tangent bonds <= 2*chi              */
  int32_t site_dim;     /* 4: operator mode (MPO reference, bottom start        */
                        /*    I/2^{n/2}); 2: state mode (MPS label, bottom      */
                        /*    start a product state)         */
  int32_t dtype;        /* tn_dtype; TN_C128                                    */
  int32_t max_batch;    /* directions per internal sub-batch of tn_hvp_apply    */
  int32_t device;       /* CUDA device ordinal                                  */
  uint32_t flags;       /* TN_CHECK_UNITARY | TN_CHECK_TANGENT, or 0            */
} tn_hvp_config;

typedef struct {
  size_t primal_bytes;        /* the primal store (tn_hvp_primal_blob's size)          */
  size_t workspace_bytes;     /* direction-independent tangent chains, recorded by the */
                              /* first apply at a point (from the library pool)        */
  size_t per_direction_bytes; /* one direction's tangent state (cached forward tangent */
                              /* + live backward tangent); x max_batch per sub-batch   */
} tn_hvp_sizes;

/* Number of gates K implied by (n_sites, depth, first_offset). */
int32_t tn_hvp_num_gates(int32_t n_sites, int32_t depth, int32_t first_offset);

/* Sizes of a context for (cfg, ref_bonds) without creating it (host only, no
 * CUDA call).  ref_bonds: HOST int32[n+1].  TN_EINVAL as tn_hvp_setup. */
tn_status tn_hvp_query(const tn_hvp_config* cfg, const int32_t* ref_bonds, tn_hvp_sizes* out);

/* Create a context.  ref_bonds: HOST int32[n+1] (b_0 = b_n = 1, neighbouring
 * bonds within a factor site_dim); ref_mpo: DEVICE, the n site tensors packed back to
 * back in site order, sum_s b_s*4*b_{s+1} complex128 (copied into the context).
 * primal_buf: DEVICE, 256-byte aligned, >= tn_hvp_query's primal_bytes
 * (primal_bytes_avail), caller-owned and kept until tn_hvp_destroy; or NULL:
 * the context allocates the store itself.  Synchronises the stream. */
tn_status tn_hvp_setup(const tn_hvp_config* cfg, const int32_t* ref_bonds, const void* ref_mpo, void* primal_buf,
                       size_t primal_bytes_avail, void* stream, tn_hvp_ctx** out);

/* Primal pass (a2-a5): bottom and top sweeps with truncation, per-layer
 * left/right environments, E_k = dT/dG_k (eq:environment),
 * f and the Riemannian gradient.
 * gates: DEVICE [K][4][4].
 * scalars_out: DEVICE double[8] = {f, Re T, Im T, max discarded weight,
 *   min relative gap at a cut, max |log10 s|, #QR-iteration SVD fallbacks,
 *   #second-level Gram deflations}.
 * grad_R_out: DEVICE [K][4][4] (may be NULL).
 * Synchronises the stream once at the end (SVD convergence flags). */
tn_status tn_hvp_environments(tn_hvp_ctx* ctx, const void* gates, void* scalars_out, void* grad_R_out,
                              void* stream);

/* Riemannian HVP (a6-a9) for a batch of directions at the gates of the last
 * tn_hvp_environments call: forward tangent propagation (eq:dfis), backward
 * tangent propagation fused with the layer environments (eq:dbis,
 * eq:overlap-hvp), then Omega, H_f and the Riemannian Hessian
 * (PAPER.md:501-505, :1152-1157).
 * dirs: DEVICE [batch][K][4][4] tangent at G (checked with TN_CHECK_TANGENT).
 * hess_R_out: DEVICE [batch][K][4][4].
 * aux_out: DEVICE, nullable: [batch][K][4][4] H_T (Wirtinger HVP of T)
 *   followed by [batch] complex Omega.
 * Graphs and per-point reuse (results are bitwise those of a cold eager
 * call): the first call at a point replays a point-free CUDA graph of the
 * whole apply (captured once per (batch, aux) for the context's lifetime; the
 * frozen truncation factors are read from the store on the device) when its
 * graph-owned working memory is small (launch-bound configurations); the
 * second call records the direction-independent tensors (tangent chains;
 * layer-HVP block tensors within a third of the then-free memory, or the cap
 * of tn_hvp_set_cache_budget) and later calls borrow them; a third call with
 * the same (batch <= 8, aux) is captured into a point-specific graph that
 * replays the cached tensors.  Point-specific state is released by the next
 * primal pass; point-free graphs by tn_hvp_trim_memory and tn_hvp_destroy.
 * Environment switches read at setup / load: TN_NO_CHAIN_CACHE=1,
 * TN_NO_GRAPH=1. */
tn_status tn_hvp_apply(tn_hvp_ctx* ctx, int32_t batch, const void* dirs, void* hess_R_out, void* aux_out,
                       void* stream);

/* One whole step of the hot path: tn_hvp_environments(gates) followed by
 * tn_hvp_apply(batch, dirs) with the same arguments, outputs and state
 * afterwards, bitwise identical results.  Fused: the forward tangents of the
 * first sub-batch (min(batch, max_batch) directions) are replayed on their own
 * stream while the top sweep and the layer environments are still running
 * (the forward tangent of bottom layer l needs only the bottom sweep up to l,
 * Alg. 1), so their GEMMs fill the SMs during the
 * latency-bound eigensolves.  batch = 0 is tn_hvp_environments. */
tn_status tn_hvp_step(tn_hvp_ctx* ctx, const void* gates, void* scalars_out, void* grad_R_out, int32_t batch,
                      const void* dirs, void* hess_R_out, void* aux_out, void* stream);

/* Euclidean pieces of the last environments call: E [K][4][4] (DEVICE out). */
tn_status tn_hvp_gradient_T(tn_hvp_ctx* ctx, void* E_out, void* stream);

/* ---- N2: translation-invariant circuits ----
 * Every gate of layer ell is the layer gate g_ell and directions are
 * layer-wise constant.  Reading X20 (chain rule,
 * the equations before Alg. 3): dT/dg_ell = sum_{k in I_ell} dT/dG_k (:1040),
 * H_T[v]_ell = sum_{k in I_ell} D_v(dT/dG_k) (:1063-1066); f, gradient and HVP
 * then follow Alg. 2 and App. E on U(4)^D.
 * tn_hvp_ti_environments: layer_gates DEVICE complex128 [D][4][4] (unitary);
 *   runs the per-gate primal pass at G_k = g_ell; scalars_out as
 *   tn_hvp_environments (f, T are the circuit's); grad_R_out DEVICE [D][4][4].
 *   A layer without gates (n = 2, even layer) gets a zero gradient.
 *   Invalidates the per-gate state's TI view on the next tn_hvp_environments.
 * tn_hvp_ti_apply: layer_dirs DEVICE [B][D][4][4] tangent at g; hess_R_out
 *   DEVICE [B][D][4][4].  TN_ESTATE before tn_hvp_ti_environments (or after a
 *   later per-gate tn_hvp_environments).  Synchronises the stream. */
tn_status tn_hvp_ti_environments(tn_hvp_ctx* ctx, const void* layer_gates, void* scalars_out, void* grad_R_out,
                                 void* stream);
tn_status tn_hvp_ti_apply(tn_hvp_ctx* ctx, int32_t batch, const void* layer_dirs, void* hess_R_out, void* stream);

/* Cost only (a3, top sweep): T and f at the given gates without touching the
 * stored primal (for the trust-region rho test).  scalars_out as above.  The
 * stored point's primal store, caches and graphs are never written, so later
 * tn_hvp_apply calls are unaffected even when this call fails.  TN_ENUMERIC on
 * a solver failure or a non-finite T.  Synchronises the stream. */
tn_status tn_hvp_cost(tn_hvp_ctx* ctx, const void* gates, void* scalars_out, void* stream);

/* Primal store as one flat device byte range (for an NCCL broadcast). */
tn_status tn_hvp_primal_blob(tn_hvp_ctx* ctx, void** ptr, size_t* bytes);

/* Mark the primal store as valid after a collective filled it (through
 * tn_hvp_primal_copy into the context, or the blob pointer) instead of
 * tn_hvp_environments.  gates: DEVICE [K][4][4], the point the store was built
 * at; the store carries its own copy and the two must agree bit for bit, else
 * TN_EINVAL and the store stays invalid.  Drops the per-point caches and the
 * translation-invariant state.  Synchronises the stream. */
tn_status tn_hvp_primal_imported(tn_hvp_ctx* ctx, const void* gates, void* stream);

/* ---- N1: sampled-state empirical risk (PAPER.md:525-554,
 * eq:costHS) ------------------------------------------------------------------
 * State mode (site_dim = 2): site tensors [b][2][b'] (p = out), the bottom
 * start is a product state |psi> = (x)_s psi_s and the top start the label MPS
 * phi = U_ref |psi>, so T = <phi| W |psi> and f = -|T|^2 is
 * minus the sample's L_HS; every other call behaves as in operator mode (the
 * empirical risk 1 - mean_s |T_s|^2 and its derivatives are sample means).
 * tn_hvp_set_product_state: psi DEVICE complex128 [n][2] (each site normalised
 *   by the caller); default |0...0>.  TN_EINVAL in operator mode.  Invalidates
 *   the stored point.
 * tn_hvp_set_reference: new reference / label tensors, same bonds as at setup,
 *   packed as in tn_hvp_setup (DEVICE).  Invalidates the stored point.
 * The label MPS phi = U_ref |psi> is input data (tn_inputs/samples.py builds it,
 * right-canonical with structural bonds, as the reference MPO is). */
tn_status tn_hvp_set_product_state(tn_hvp_ctx* ctx, const void* psi, void* stream);
tn_status tn_hvp_set_reference(tn_hvp_ctx* ctx, const void* ref, void* stream);

/* ---- N4: GPU-side reference construction (PAPER.md:589,
 * :601; reading X11) ------------------------------------------------------------
 * TEBD of a gate sequence (e.g. a 1st/2nd/4th-order Trotter circuit) on the
 * operator I/2^{n/2} with the library's primal kernels: gate g (DEVICE
 * complex128 gates[g][4][4]) acts on the OUT legs of sites (sites[g],
 * sites[g]+1) (HOST int32), each split keeps r = min(chi, #{sigma_j >
 * max(tol, 1e-7) sigma_1}) singular values rescaled to the pre-truncation norm;
 * the result is right-canonical, centre at site 0, unit Frobenius norm -- the
 * reference MPO U_ref / 2^{n/2} that tn_hvp_setup takes.  bonds_out: HOST
 * int32[n+1]; out: DEVICE, capacity out_capacity complex128 elements (n 16 chi^2
 * always suffices), site tensors [b][4][b'] packed.  Synchronises the stream
 * once per gate (data-dependent split sizes).  TN_EINVAL on a bad site or too
 * small a capacity. */
tn_status tn_mpo_tebd(int32_t n_sites, int32_t n_gates, const int32_t* sites, const void* gates, int32_t chi,
                      double tol, int32_t device, int32_t* bonds_out, void* out, size_t out_capacity, void* stream);

/* Cap, in bytes, on the per-point caches (tangent chains + layer-HVP memo)
 * of this context; 0 (default) = automatic (chains within half, memo within a
 * third of the free memory at the first apply).  For several contexts sharing
 * one device (N1 samples).  Takes effect at the next primal pass. */
tn_status tn_hvp_set_cache_budget(tn_hvp_ctx* ctx, size_t bytes);

/* ---- split primal pass (a10, multi-GPU) ------------------------
 * The two primal sweeps are independent (a2 bottom, a3 top), so two ranks can
 * run one each and exchange their halves of the store:
 * tn_hvp_environments_part(part 0 | 1): the bottom (0) or top (1) sweep at
 *   gates (DEVICE [K][4][4]) on `stream`, writing only that side's region of the
 *   store (tn_hvp_primal_region) and its diagnostics; invalidates the point;
 *   synchronises (solver status).
 * tn_hvp_primal_region(part): byte offset and size of that side's region inside
 *   the primal store (for a collective on a slice of the caller-owned buffer).
 * tn_hvp_environments_finish: once both regions hold the sweeps at `gates`
 *   (computed here or received), the layer environments, E_k, T, f and grad_R
 *   as tn_hvp_environments would produce them (scalars_out as there, with the
 *   fallback / deflation counts left 0); the point is then valid for apply.
 *   Synchronises. */
tn_status tn_hvp_environments_part(tn_hvp_ctx* ctx, const void* gates, int32_t part, void* stream);
tn_status tn_hvp_primal_region(tn_hvp_ctx* ctx, int32_t part, size_t* offset, size_t* bytes);
tn_status tn_hvp_environments_finish(tn_hvp_ctx* ctx, const void* gates, void* scalars_out, void* grad_R_out,
                                     void* stream);

/* Release the per-point caches and CUDA graphs (the next apply rebuilds them)
 * and return the library pool's unused device memory to the device, e.g.
 * before the caller allocates large buffers of its own.  Synchronises. */
tn_status tn_hvp_trim_memory(tn_hvp_ctx* ctx, void* stream);

/* out = P_G(in) = 1/2 (in - G in^dag G), gate-wise, batched (eq:projec,
 * PAPER.md:1113-1115).  gates [K][4][4], in/out [batch][K][4][4], DEVICE. */
tn_status tn_riemannian_project(int32_t K, int32_t batch, const void* gates, const void* in, void* out,
                                void* stream);

/* Retraction for the trust region: out_k = polar factor of (G_k + alpha xi_k)
 * (unitary to machine precision).  DEVICE gates, xi, out
 * [K][4][4]; returns TN_ENUMERIC if an iterate is singular (synchronises). */
tn_status tn_retract(int32_t K, const void* gates, const void* xi, double alpha, void* out, void* stream);

/* Tangent-vector algebra for tCG on U(4)^K (metric Re sum Tr(A^dag B), X15):
 * out[b] = Re <A_b, B_b> over n complex entries each (DEVICE double[batch]);
 * y = a x + b y over n complex entries (a, b complex, HOST double[2]). */
tn_status tn_tangent_dot(int64_t n, int32_t batch, const void* A, const void* B, void* out, void* stream);
tn_status tn_tangent_axpby(int64_t n, const double* a, const void* x, const double* b, void* y, void* stream);

/* ---- N3: Hessian spectrum in the Pauli tangent basis (
 * PAPER.md:1161-1190, App. "Spectral analysis") --------------------------------
 * Basis: B_{16k+4a+b} = (0, .., i G_k (P_a (x) P_b)/2, .., 0),
 * 16K vectors, orthonormal under <A,B> = Re sum_k Tr(A_k^dag B_k); P_a in
 * {I, X, Y, Z}, 4x4 index 2 q_i + q_{i+1}.  With it, column j of the matrix
 * (H_R)_ij = <B_i, H_R[B_j]> is pauli_coords(tn_hvp_apply(B_j)).
 *
 * tn_pauli_basis: writes basis vectors first .. first+count-1 to out
 *   (DEVICE complex128 [count][K][4][4]); gates DEVICE [K][4][4].
 *   TN_EINVAL if first < 0, count < 0 or first + count > 16 K.
 * tn_pauli_coords: out[j][i] = <B_i, X_j> for i < 16K (DEVICE double
 *   [count][16K]); X DEVICE complex128 [count][K][4][4].  Filling the rows j of
 *   a [16K][16K] buffer with the coordinates of H_R[B_j] stores H_R^T
 *   row-major (= H_R column-major).
 * tn_sym_eig: A (DEVICE double [n][n], overwritten) -> w (DEVICE double [n]),
 *   the eigenvalues of the symmetric part (A + A^T)/2 in ascending order
 *   (reading X19: the truncated HVP is only approximately self-adjoint);
 *   asym (DEVICE double [2]) = (||A - A^T||_F, ||A||_F) of the input.  With
 *   vectors = 1 the orthonormal eigenvectors overwrite A (row i = vector i);
 *   else A holds workspace garbage.  cuSOLVER syevd; synchronises the stream
 *   (host-visible info); TN_ENUMERIC if it does not converge. */
tn_status tn_pauli_basis(int32_t K, int64_t first, int32_t count, const void* gates, void* out, void* stream);
tn_status tn_pauli_coords(int32_t K, int32_t count, const void* gates, const void* X, void* out, void* stream);
tn_status tn_sym_eig(int32_t n, void* A, void* w, void* asym, int32_t vectors, void* stream);

/* Copy the primal store to (into_ctx = 0; TN_ESTATE without a valid primal
 * pass) or from (into_ctx = 1) a caller DEVICE buffer of exactly
 * tn_hvp_primal_blob's size (broadcast support).  into_ctx = 1 invalidates the
 * context's point until tn_hvp_primal_imported. */
tn_status tn_hvp_primal_copy(tn_hvp_ctx* ctx, void* buf, size_t bytes, int32_t into_ctx, void* stream);

/* Building block exposed for tests: batched complex128 GEMM on the FP64
 * tensor cores (DMMA), C[b] = alpha op(A[b]) op(B[b]) + beta C[b], row-major,
 * op in {'N','T','C'}; op(A) is M x K.  Strides in elements (0 = shared).
 * alpha, beta: HOST double[2]. */
tn_status tn_zgemm(char opa, char opb, int32_t M, int32_t N, int32_t K, const double* alpha,
                   const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb, int64_t strideB,
                   const double* beta, void* C, int64_t ldc, int64_t strideC, int32_t batch, void* stream);

/* Work model of one tn_hvp_apply direction (complex MACs of the schedule the
 * context runs), and the bytes of the dominant kernel class; for rooflines. */
tn_status tn_hvp_work(tn_hvp_ctx* ctx, double* cmac_per_direction, double* cmac_primal);

/* Split statistics of the context's last primal pass (both sweeps), HOST
 * int64[6]: [0] splits that fell back to the QR-iteration SVD, [1] extra Gram
 * (deflation) levels, [2] cuts accepted inside the double-precision noise
 * floor (reading X10), [3] low-rank blocks split by the range probe (numerical
 * rank <= kept rank: no eigendecomposition), [4] centre
 * moves whose CholeskyQR2 was rejected (Householder used), [5] pair steps.
 * Diagnostics only; TN_EINVAL on a null argument. */
tn_status tn_hvp_split_stats(tn_hvp_ctx* ctx, int64_t* out6);

/* Number of kernels this library has launched since it was loaded (all
 * contexts, all streams) -- the bench's gpu_launches evidence. */
int64_t tn_hvp_launch_count(void);

/* GEMM timing probe for the roofline: mode 1 = reset and start recording a
 * CUDA-event pair around every DMMA GEMM launch; mode 0 = stop, synchronise
 * the recorded events and return the summed kernel milliseconds and complex
 * MACs (HOST outputs, may be NULL when mode = 1). */
tn_status tn_gemm_profile(int32_t mode, double* ms, double* cmac);

/* Destroy a context.  The caller has synchronised the streams it used with it. */
void tn_hvp_destroy(tn_hvp_ctx* ctx);

/* Last error text of ctx (or of the calling thread when ctx is NULL). */
const char* tn_hvp_last_error(const tn_hvp_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TN_HVP_H */
