// Declarations of the small kernels (kernels.cu).
#pragma once
#include "common.cuh"

namespace tn {
// Site physical index p = out * ni + in: ni = 2 for operator (MPO) sites,
// ni = 1 for state (MPS) sites.
// out[b] = alpha * gate[b] (x) I_in applied to the out legs of x[b] viewed as
// [X][2ni][2ni][Y]; accumulate adds to out.  In-place allowed.
void apply_gate(cudaStream_t st, cplx* out, int64_t sout, const cplx* x, int64_t sx, const cplx* gate, int64_t sg,
                int X, int Y, int batch, cplx alpha, bool accumulate, int ni = 2);
// out[b] = g1[b] x[b] + g2[b] y[b] on the out legs in one pass (strides in elements, 0 = shared); out may alias x.
void apply_gate2(cudaStream_t st, cplx* out, int64_t sout, const cplx* x, int64_t sx, const cplx* g1, int64_t sg1,
                 const cplx* y, int64_t sy, const cplx* g2, int64_t sg2, int X, int Y, int batch, int ni = 2);
void axpby(cudaStream_t st, cplx* y, const cplx* x, cplx a, cplx b, int64_t n);   // y = a x + b y
void scale_by(cudaStream_t st, cplx* y, const double* s, double pw, int64_t n);    // y *= s^pw (device s)
// dst[i][j] = src[i][j] / S[i] (device S[rows]; rows x cols row-major)
void rows_over_s(cudaStream_t st, cplx* dst, const cplx* src, const double* S, int rows, int64_t cols);
// E[b] += alpha * sum conj(top[t,(o1 i1),(o2 i2),u]) z[b][t,(c1 i1),(c2 i2),u]
void extract_env(cudaStream_t st, cplx* E, int64_t sE, const cplx* top, int64_t stop, const cplx* z, int64_t sz,
                 int T, int U, int batch, cplx alpha, int ni = 2);
void project(cudaStream_t st, int K, int batch, const cplx* G, const cplx* in, cplx* out);
void gradient_post(cudaStream_t st, int K, const cplx* G, const cplx* E, const double* scal, cplx* grad_f,
                   cplx* grad_R);
void hessian_post(cudaStream_t st, int K, int batch, const cplx* G, const cplx* E, const cplx* grad_f,
                  const double* scal, const cplx* HT, const cplx* V, cplx* om, cplx* out);
}  // namespace tn

namespace tn {
// dst[c][r] = (conj?) src[r][c]; src rows x cols row-major (ld = cols).
void transpose(cudaStream_t st, cplx* dst, const cplx* src, int rows, int cols, bool conj);
// dst[a][j] = conj(uh[j][a]) * (S ? s*S[j] : 1)  for uh (r x m) row-major -> dst (m x r).
void conjT_scale_cols(cudaStream_t st, cplx* dst, const cplx* uh, int r, int m, const double* S, const double* s);
// Row-major (rows x cols) from the upper triangle of a column-major buffer
// (lda): dst[i][j] = (j >= i) ? buf[i + j*lda] : 0          (upper = true)
// Lower variant for LQ: dst[i][j] = (j <= i) ? buf[j + i*lda] : 0 (rows x cols = b x kq).
void tri_extract(cudaStream_t st, cplx* dst, const cplx* buf, int rows, int cols, int64_t lda, bool upper);
// In place on a row-major n x n matrix: zero the strictly lower (upper = true) or strictly upper triangle.
void tri_keep(cudaStream_t st, cplx* M, int n, bool upper);
// CholeskyQR bookkeeping: *flag |= 1 if *info != 0 (potrf), if the kept triangle of the
// row-major n x n factor M has a non-finite entry, or (near_identity) if max |M - I| > tol.
void chol_flag(cudaStream_t st, const cplx* M, int n, bool upper, const int* info, bool near_identity, double tol,
               int* flag);
// p[i] = uniform in (-1, 1)^2 from a counter-based hash of (seed, i): the fixed
// test matrix of the low-rank range probe (not an input of the method).
void fill_test_matrix(cudaStream_t st, cplx* p, int64_t n, uint64_t seed);
// Vd[b][k] = V[b][k]^dag (4x4 each), n = batch*K matrices.
void dagger4(cudaStream_t st, cplx* dst, const cplx* src, int64_t n);
// out[0..2] = (max, min, max) of the two sides' diagnostics d[0..2], d[8..10]
void combine_diag(cudaStream_t st, double* out, const double* d);
// C[i][j] = M[i][j] / (S[j]^2 - S[r+i]^2) for i < nd (discarded), j < r (kept);
// the first-order rotation that makes the kept rows of B = U^H A orthogonal to
// the discarded ones (one-sided Jacobi step across the cut).
void kept_rotation(cudaStream_t st, cplx* Cm, const cplx* M, const double* S, int nd, int r);
// heevd output (column-major W, ascending lam) -> uhf = U^H rows (descending), S = sqrt(lam)
void eig_to_svd(cudaStream_t st, cplx* uhf, double* S, const cplx* W, const double* lam, int R);
// s = sqrt(nrm[0]/nrm[1]) into s_out; diag[0] = max(diag[0], discarded weight),
// diag[1] = min(diag[1], relative gap (S[r-1]-S[r])/S[0]), diag[2] = max(diag[2], |log10 s|)
void s_from_norms(cudaStream_t st, const double* nrm, const double* S, int mn, int r, double* s_out, double* diag);
// dst[(o1 o2)][x][i1 i2][y] = src[x][(o1 i1)][(o2 i2)][y]
void out_leg_split(cudaStream_t st, cplx* dst, const cplx* src, int X, int Y, int ni = 2);
// *acc = max(*acc, |*info|)  (cuSOLVER status accumulation)
void info_accum(cudaStream_t st, int* acc, const int* info);
// dst = conj(src), n elements
void conj_copy(cudaStream_t st, cplx* dst, const cplx* src, int64_t n);
// out_k = polar(G_k + alpha xi_k) (unitary retraction); status[0] = 1 on a singular iterate
void retract(cudaStream_t st, int K, const cplx* G, const cplx* xi, double alpha, cplx* out, int* status);
// out[b] = Re <A_b, B_b> over n complex entries per batch item
void tangent_dot(cudaStream_t st, int64_t n, int batch, const cplx* A, const cplx* B, double* out);
// scalars[0] = -|T|^2, [1..2] = T from a 1x1 complex env; keeps [3..] untouched.
void finish_cost(cudaStream_t st, double* scalars, const cplx* T11);
}  // namespace tn

namespace tn {
// N3 (spectrum.cu): Pauli tangent basis window, Pauli coordinates of tangent
// vectors, eigenvalues of the symmetric part of a real n x n matrix.
void pauli_basis(cudaStream_t st, int K, int64_t first, int count, const cplx* G, cplx* out);
void pauli_coords(cudaStream_t st, int K, int count, const cplx* G, const cplx* X, double* out);
void sym_eig(cudaStream_t st, int n, double* A, double* w, double* asym, bool vectors);
}  // namespace tn

namespace tn {
// N2 (kernels.cu): tied layer gates.  ti_expand: dst[b][k] = src[b][layer_of[k]]
// ([batch][L][4][4] -> [batch][K][4][4]); ti_reduce: dst[b][l] = sum of
// src[b][k] over the layer's contiguous gates start[l] <= k < start[l+1].
void ti_expand(cudaStream_t st, int L, int K, int batch, const int* layer_of, const cplx* src, cplx* dst);
void ti_reduce(cudaStream_t st, int L, int K, int batch, const int* start, const cplx* src, cplx* dst);
}  // namespace tn

namespace tn {
// p[0..n) = (v0, v1, v2, v3)[0..n), n <= 4: device-side constants (no pageable
// host copies, so the apply path can be captured into a CUDA graph)
void set_small(cudaStream_t st, cplx* p, int n, cplx v0, cplx v1 = {0.0, 0.0}, cplx v2 = {0.0, 0.0},
               cplx v3 = {0.0, 0.0});
}  // namespace tn

namespace tn {
// ABI flag checks.  res[k] = ||G_k^dag G_k - I||_F (DEVICE
// double[K]); res[2 (b K + k) + {0,1}] = (||V - P_G V||^2, ||V||^2) of gate k of
// direction b (DEVICE double[2 batch K]).
void check_unitary(cudaStream_t st, int K, const cplx* G, double* res);
void check_tangent(cudaStream_t st, int K, int batch, const cplx* G, const cplx* V, double* res);
}  // namespace tn


namespace tn {
// y *= sqrt(nrm[0] / nrm[1]) (device scalars; norm-restoring rescale)
void scale_by_norm_ratio(cudaStream_t st, cplx* y, const double* nrm, int64_t n);
}  // namespace tn
