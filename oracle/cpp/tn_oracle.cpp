// Plain C++17 complex128 oracle of the HVP kernel (north_star subsystem (1)).
//
// TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): nothing of the CUDA path
// is used or shared -- no BLAS, no LAPACK, no headers of the library; only
// std::complex<double> loops and a one-sided Jacobi SVD written out here.
// Built by oracle/cpp/build.py (g++ -O2), loaded by oracle/cpp_oracle.py.
//
//  * tno_alg1: Algorithm 1 of the paper literally, on dense
//    2^n x m matrices (m = 2^n: operators psi0 = I/2^{n/2}, phi0 = U/2^{n/2};
//    m = 1: states psi0 = |psi>, phi0 = U|psi>): the forward pass caches
//    psi^(k), Dpsi^(k) (eq:fis, eq:dfis); the backward pass accumulates
//    E_k = sum conj(phi^(K-k)) psi^(k-1) and H_T[V]_k (eq:overlap-hvp) with the
//    PRE-update Dphi, phi (reading X3), then updates them; T = <phi^(K)|psi^(0)>.
//  * tno_dense_truncated: the truncated definition of SURVEY.md §8(c.2)
//    (readings X7-X9) written out on p^n vectors (p = 4 operator sites
//    p = 2 out + in, p = 2 state sites): per gate a Schmidt decomposition at its
//    cut (one-sided Jacobi SVD), keep r = min(chi, 4 m_c, p b_{c-1}, p b_{c+1}),
//    frozen renormalisation s = ||X|| / ||P^L X||, tangent
//    s (P^L(x)I + I(x)P^R - P^L(x)P^R)(M DX + V_M X); layer-wise E and H_T with
//    the layer's own gates exact; T = <<T_0|B_0>>.
//  * tno_postprocess: Alg. 2 (reading X2: f = -|T|^2,
//    grad f = -2 T conj(E), H_f = -2 [Omega conj(E) + T conj(H_T)]) and the
//    Riemannian maps of App. E.
// Complex arrays are interleaved (re, im) doubles, row-major, as numpy stores
// complex128.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <vector>

using cd = std::complex<double>;
using Vec = std::vector<cd>;

namespace {

inline const cd* C(const double* p) { return reinterpret_cast<const cd*>(p); }
inline cd* C(double* p) { return reinterpret_cast<cd*>(p); }

// ------------------------------------------------------------------ O1 --
// Y = (G on qubits s, s+1) X for X: 2^n x m.
Vec apply_op(const Vec& X, int n, int s, const cd* G, int m) {
  const int64_t a = int64_t(1) << s, b = int64_t(1) << (n - s - 2);
  Vec Y(X.size(), cd(0, 0));
  for (int64_t x = 0; x < a; ++x)
    for (int64_t y = 0; y < b; ++y)
      for (int o = 0; o < 4; ++o)
        for (int i = 0; i < 4; ++i) {
          const cd g = G[o * 4 + i];
          if (g == cd(0, 0)) continue;
          const int64_t ro = ((x * 4 + o) * b + y) * m, ri = ((x * 4 + i) * b + y) * m;
          for (int z = 0; z < m; ++z) Y[ro + z] += g * X[ri + z];
        }
  return Y;
}

// E[a][b] = sum conj(phi[x,a,y,z]) psi[x,b,y,z] (eq:environment; X4: a = gate output)
void env_op(const Vec& phi, const Vec& psi, int n, int s, int m, cd* E) {
  const int64_t a = int64_t(1) << s, b = int64_t(1) << (n - s - 2);
  for (int i = 0; i < 16; ++i) E[i] = 0;
  for (int64_t x = 0; x < a; ++x)
    for (int64_t y = 0; y < b; ++y)
      for (int o = 0; o < 4; ++o)
        for (int i = 0; i < 4; ++i) {
          cd acc = 0;
          const int64_t ro = ((x * 4 + o) * b + y) * m, ri = ((x * 4 + i) * b + y) * m;
          for (int z = 0; z < m; ++z) acc += std::conj(phi[ro + z]) * psi[ri + z];
          E[o * 4 + i] += acc;
        }
}

void dagger4(const cd* G, cd* D) {
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) D[a * 4 + b] = std::conj(G[b * 4 + a]);
}

// ------------------------------------------------------------------ O2 --
// One-sided (Hestenes) Jacobi SVD of A (rows x cols, row-major): A = U S V^H with
// U: rows x k, V: cols x k (k = min(rows, cols)), S descending.  Columns whose
// singular value vanishes get an orthonormal completion (their weight is zero).
void svd(const Vec& A, int rows, int cols, Vec& U, std::vector<double>& S, Vec& V) {
  const bool tr = cols > rows;  // work on the tall orientation
  const int m = tr ? cols : rows, nn = tr ? rows : cols;
  Vec W((size_t)m * nn), Q((size_t)nn * nn, cd(0, 0));
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < nn; ++j) W[(size_t)i * nn + j] = tr ? std::conj(A[(size_t)j * cols + i]) : A[(size_t)i * cols + j];
  for (int j = 0; j < nn; ++j) Q[(size_t)j * nn + j] = 1;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0;
    for (int i = 0; i < nn - 1; ++i)
      for (int j = i + 1; j < nn; ++j) {
        double al = 0, be = 0;
        cd ga = 0;
        for (int r = 0; r < m; ++r) {
          const cd wi = W[(size_t)r * nn + i], wj = W[(size_t)r * nn + j];
          al += std::norm(wi);
          be += std::norm(wj);
          ga += std::conj(wi) * wj;
        }
        const double ag = std::abs(ga);
        if (ag == 0.0 || ag <= 1e-17 * std::sqrt(al * be)) continue;
        off = std::max(off, ag / std::sqrt(al * be));
        const cd e = ga / ag;  // phase making the inner product real
        const double zeta = (be - al) / (2 * ag);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
        const double c = 1 / std::sqrt(1 + t * t), s = c * t;
        for (int r = 0; r < m; ++r) {
          const cd wi = W[(size_t)r * nn + i], wj = W[(size_t)r * nn + j] * std::conj(e);
          W[(size_t)r * nn + i] = c * wi - s * wj;
          W[(size_t)r * nn + j] = s * wi + c * wj;
        }
        for (int r = 0; r < nn; ++r) {
          const cd qi = Q[(size_t)r * nn + i], qj = Q[(size_t)r * nn + j] * std::conj(e);
          Q[(size_t)r * nn + i] = c * qi - s * qj;
          Q[(size_t)r * nn + j] = s * qi + c * qj;
        }
      }
    if (off < 1e-15) break;
  }
  std::vector<double> sv(nn);
  for (int j = 0; j < nn; ++j) {
    double a = 0;
    for (int r = 0; r < m; ++r) a += std::norm(W[(size_t)r * nn + j]);
    sv[j] = std::sqrt(a);
  }
  std::vector<int> ord(nn);
  for (int j = 0; j < nn; ++j) ord[j] = j;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return sv[a] > sv[b]; });
  // left vectors of the working orientation (m x nn), completed where sigma ~ 0
  Vec L((size_t)m * nn, cd(0, 0)), R((size_t)nn * nn);
  S.assign(nn, 0.0);
  const double floor = 1e-300 + 1e-15 * (nn ? sv[ord[0]] : 0.0);
  for (int jj = 0; jj < nn; ++jj) {
    const int j = ord[jj];
    S[jj] = sv[j];
    for (int r = 0; r < nn; ++r) R[(size_t)r * nn + jj] = Q[(size_t)r * nn + j];
    if (sv[j] > floor) {
      for (int r = 0; r < m; ++r) L[(size_t)r * nn + jj] = W[(size_t)r * nn + j] / sv[j];
    } else {  // orthonormal completion by Gram-Schmidt against the earlier columns
      for (int e = 0; e < m; ++e) {
        Vec v(m, cd(0, 0));
        v[e] = 1;
        for (int pass = 0; pass < 2; ++pass)
          for (int q = 0; q < jj; ++q) {
            cd d = 0;
            for (int r = 0; r < m; ++r) d += std::conj(L[(size_t)r * nn + q]) * v[r];
            for (int r = 0; r < m; ++r) v[r] -= d * L[(size_t)r * nn + q];
          }
        double nv = 0;
        for (int r = 0; r < m; ++r) nv += std::norm(v[r]);
        nv = std::sqrt(nv);
        if (nv > 1e-8) {
          for (int r = 0; r < m; ++r) L[(size_t)r * nn + jj] = v[r] / nv;
          break;
        }
      }
    }
  }
  // back to A's orientation: A = L S R^H (not transposed) or A = conj(R) S L^T (transposed)
  const int k = nn;
  U.assign((size_t)rows * k, 0);
  V.assign((size_t)cols * k, 0);
  if (!tr) {
    U = L;
    V = R;
  } else {  // A^H = W-space: A^H = L S R^H  =>  A = R S L^H
    U = R;    // rows x k (rows = nn)
    V = L;    // cols x k (cols = m)
  }
}

struct Dense {  // one truncated dense sweep state: x and the directions' tangents
  int n, p, chi;
  int64_t dim;
};

// x viewed [p^s][p][p][rest]; gate on the OUT legs of sites (s, s+1)
Vec vec_apply(const Vec& x, int n, int p, int s, const cd* M) {
  const int ni = p / 2;
  int64_t a = 1, b = 1;
  for (int i = 0; i < s; ++i) a *= p;
  for (int i = s + 2; i < n; ++i) b *= p;
  Vec y(x.size(), cd(0, 0));
  for (int64_t xa = 0; xa < a; ++xa)
    for (int64_t yb = 0; yb < b; ++yb)
      for (int i1 = 0; i1 < ni; ++i1)
        for (int i2 = 0; i2 < ni; ++i2)
          for (int o = 0; o < 4; ++o) {
            const int o1 = o >> 1, o2 = o & 1;
            cd acc = 0;
            for (int c = 0; c < 4; ++c) {
              const int c1 = c >> 1, c2 = c & 1;
              acc += M[o * 4 + c] * x[((xa * p + (c1 * ni + i1)) * p + (c2 * ni + i2)) * b + yb];
            }
            y[((xa * p + (o1 * ni + i1)) * p + (o2 * ni + i2)) * b + yb] = acc;
          }
  return y;
}

void vec_env(const Vec& top, const Vec& bot, int n, int p, int s, cd* E) {
  const int ni = p / 2;
  int64_t a = 1, b = 1;
  for (int i = 0; i < s; ++i) a *= p;
  for (int i = s + 2; i < n; ++i) b *= p;
  for (int i = 0; i < 16; ++i) E[i] = 0;
  for (int64_t xa = 0; xa < a; ++xa)
    for (int64_t yb = 0; yb < b; ++yb)
      for (int i1 = 0; i1 < ni; ++i1)
        for (int i2 = 0; i2 < ni; ++i2)
          for (int o = 0; o < 4; ++o)
            for (int c = 0; c < 4; ++c) {
              const int o1 = o >> 1, o2 = o & 1, c1 = c >> 1, c2 = c & 1;
              E[o * 4 + c] += std::conj(top[((xa * p + (o1 * ni + i1)) * p + (o2 * ni + i2)) * b + yb]) *
                              bot[((xa * p + (c1 * ni + i1)) * p + (c2 * ni + i2)) * b + yb];
            }
}

double norm2(const Vec& v) {
  double a = 0;
  for (const cd& z : v) a += std::norm(z);
  return a;
}

struct Truncated {
  int n, D, chi, off, p, nb, K;
  const cd* G;
  const cd* V;
  std::vector<std::vector<std::pair<int, int>>> layers;  // (k, s)
  std::vector<Vec> B, Tt;                                // B_{l-1}, T_l
  std::vector<std::vector<Vec>> DB, DT;

  void step(Vec& x, std::vector<Vec>& dx, int s, const cd* M, const std::vector<const cd*>& VM, std::vector<int>& bonds) {
    const int c = s + 1;
    Vec xp = vec_apply(x, n, p, s, M);
    std::vector<Vec> dxp(dx.size());
    for (size_t b = 0; b < dx.size(); ++b) {
      dxp[b] = vec_apply(dx[b], n, p, s, M);
      Vec t = vec_apply(x, n, p, s, VM[b]);
      for (size_t i = 0; i < t.size(); ++i) dxp[b][i] += t[i];
    }
    int64_t rows = 1, cols = 1;
    for (int i = 0; i < c; ++i) rows *= p;
    for (int i = c; i < n; ++i) cols *= p;
    Vec U, Vv;
    std::vector<double> S;
    svd(xp, (int)rows, (int)cols, U, S, Vv);
    const int k = (int)S.size();
    const int r = std::min({chi, 4 * bonds[c], p * bonds[c - 1], p * bonds[c + 1], k});
    // y = Ur Ur^H X ; frozen s = ||X|| / ||y||
    auto PL = [&](const Vec& X) {  // Ur (Ur^H X)
      Vec t((size_t)r * cols, 0), out(X.size(), 0);
      for (int a = 0; a < r; ++a)
        for (int64_t i = 0; i < rows; ++i) {
          const cd u = std::conj(U[(size_t)i * k + a]);
          if (u == cd(0, 0)) continue;
          for (int64_t j = 0; j < cols; ++j) t[(size_t)a * cols + j] += u * X[(size_t)i * cols + j];
        }
      for (int64_t i = 0; i < rows; ++i)
        for (int a = 0; a < r; ++a) {
          const cd u = U[(size_t)i * k + a];
          if (u == cd(0, 0)) continue;
          for (int64_t j = 0; j < cols; ++j) out[(size_t)i * cols + j] += u * t[(size_t)a * cols + j];
        }
      return out;
    };
    auto PR = [&](const Vec& X) {  // (X Vr) Vr^H
      Vec t((size_t)rows * r, 0), out(X.size(), 0);
      for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) {
          const cd xv = X[(size_t)i * cols + j];
          if (xv == cd(0, 0)) continue;
          for (int a = 0; a < r; ++a) t[(size_t)i * r + a] += xv * Vv[(size_t)j * k + a];
        }
      for (int64_t i = 0; i < rows; ++i)
        for (int a = 0; a < r; ++a) {
          const cd tv = t[(size_t)i * r + a];
          if (tv == cd(0, 0)) continue;
          for (int64_t j = 0; j < cols; ++j) out[(size_t)i * cols + j] += tv * std::conj(Vv[(size_t)j * k + a]);
        }
      return out;
    };
    Vec y = PL(xp);
    const double sc = std::sqrt(norm2(xp) / norm2(y));
    for (size_t b = 0; b < dx.size(); ++b) {
      Vec a = PL(dxp[b]), bb = PR(dxp[b]), ab = PR(a);
      for (size_t i = 0; i < a.size(); ++i) dxp[b][i] = sc * (a[i] + bb[i] - ab[i]);
      dx[b] = dxp[b];
    }
    for (auto& z : y) z *= sc;
    x = y;
    bonds[c] = r;
  }

  // E_k of layer l for <<top| L_l |bot>>, gate kp replaced by Msub when kp >= 0
  void layer_env(int l, const Vec& top, const Vec& bot, int kp, const cd* Msub, std::vector<cd>& Eout,
                 bool skip_kp) {
    const auto& ly = layers[l - 1];
    for (auto [k, s] : ly) {
      if (skip_kp && k == kp) continue;
      Vec z = bot;
      for (auto [kk, ss] : ly)
        if (kk != k) z = vec_apply(z, n, p, ss, kk == kp ? Msub : G + (int64_t)kk * 16);
      cd E[16];
      vec_env(top, z, n, p, s, E);
      for (int i = 0; i < 16; ++i) Eout[(size_t)k * 16 + i] += E[i];
    }
  }
};

}  // namespace

extern "C" {

int tno_alg1(int n, int K, const int* sites, const double* Gd, int m, const double* psi0, const double* phi0, int nb,
             const double* Vd, double* T, double* Ed, double* Hd) {
  const int64_t d = int64_t(1) << n;
  const cd* G = C(Gd);
  const cd* V = C(Vd);
  std::vector<Vec> psi(K + 1);
  std::vector<std::vector<Vec>> dpsi(nb, std::vector<Vec>(K + 1));
  psi[0] = Vec(C(psi0), C(psi0) + d * m);
  for (int b = 0; b < nb; ++b) dpsi[b][0] = Vec(d * m, cd(0, 0));
  for (int k = 0; k < K; ++k) {  // forward pass (Alg. 1)
    for (int b = 0; b < nb; ++b) {
      Vec a = apply_op(dpsi[b][k], n, sites[k], G + (int64_t)k * 16, m);
      Vec c = apply_op(psi[k], n, sites[k], V + ((int64_t)b * K + k) * 16, m);
      for (size_t i = 0; i < a.size(); ++i) a[i] += c[i];
      dpsi[b][k + 1] = a;
    }
    psi[k + 1] = apply_op(psi[k], n, sites[k], G + (int64_t)k * 16, m);
  }
  Vec phi(C(phi0), C(phi0) + d * m);
  std::vector<Vec> dphi(nb, Vec(d * m, cd(0, 0)));
  cd* E = C(Ed);
  cd* H = C(Hd);
  for (int k = K - 1; k >= 0; --k) {  // backward pass (lines 286-291), reading X3
    cd Gd_[16];
    dagger4(G + (int64_t)k * 16, Gd_);
    env_op(phi, psi[k], n, sites[k], m, E + (int64_t)k * 16);
    for (int b = 0; b < nb; ++b) {
      cd h1[16], h2[16], Vd_[16];
      env_op(dphi[b], psi[k], n, sites[k], m, h1);
      env_op(phi, dpsi[b][k], n, sites[k], m, h2);
      for (int i = 0; i < 16; ++i) H[((int64_t)b * K + k) * 16 + i] = h1[i] + h2[i];
      dagger4(V + ((int64_t)b * K + k) * 16, Vd_);
      Vec a = apply_op(dphi[b], n, sites[k], Gd_, m);
      Vec c = apply_op(phi, n, sites[k], Vd_, m);
      for (size_t i = 0; i < a.size(); ++i) a[i] += c[i];
      dphi[b] = a;
    }
    phi = apply_op(phi, n, sites[k], Gd_, m);
  }
  cd t = 0;
  for (int64_t i = 0; i < d * m; ++i) t += std::conj(phi[i]) * psi[0][i];
  T[0] = t.real();
  T[1] = t.imag();
  return 0;
}

int tno_dense_truncated(int n, int depth, int chi, int first_offset, int p, const double* Gd, const double* x0,
                        const double* top0, const int* ref_bonds, int nb, const double* Vd, double* T, double* Ed,
                        double* Hd) {
  Truncated tr;
  tr.n = n;
  tr.D = depth;
  tr.chi = chi;
  tr.off = first_offset;
  tr.p = p;
  tr.nb = nb;
  tr.G = C(Gd);
  tr.V = C(Vd);
  int k = 0;
  tr.layers.assign(depth, {});
  for (int l = 1; l <= depth; ++l) {
    const int o = (first_offset + l - 1) % 2;
    for (int s = o; s + 1 < n; s += 2) tr.layers[l - 1].push_back({k++, s});
  }
  tr.K = k;
  int64_t dim = 1;
  for (int i = 0; i < n; ++i) dim *= p;
  // bottom sweep: layers 1..D, odd layers left->right (X7)
  Vec x(C(x0), C(x0) + dim);
  std::vector<Vec> dx(nb, Vec(dim, cd(0, 0)));
  std::vector<int> bonds(n + 1, 1);
  tr.B.resize(depth);
  tr.DB.resize(depth);
  for (int l = 1; l <= depth; ++l) {
    tr.B[l - 1] = x;
    tr.DB[l - 1] = dx;
    auto ly = tr.layers[l - 1];
    if (l % 2 == 0) std::reverse(ly.begin(), ly.end());
    for (auto [kk, s] : ly) {
      std::vector<const cd*> vm(nb);
      for (int b = 0; b < nb; ++b) vm[b] = tr.V + ((int64_t)b * tr.K + kk) * 16;
      tr.step(x, dx, s, tr.G + (int64_t)kk * 16, vm, bonds);
    }
  }
  // top sweep: layers D..1 with G^dag, layer D left->right then alternating
  x = Vec(C(top0), C(top0) + dim);
  dx.assign(nb, Vec(dim, cd(0, 0)));
  bonds.assign(ref_bonds, ref_bonds + n + 1);
  tr.Tt.resize(depth + 1);
  tr.DT.resize(depth + 1);
  std::vector<cd> Gdag((size_t)tr.K * 16), Vdag((size_t)std::max(nb, 1) * tr.K * 16);
  for (int q = 0; q < tr.K; ++q) dagger4(tr.G + (int64_t)q * 16, &Gdag[(size_t)q * 16]);
  for (int b = 0; b < nb; ++b)
    for (int q = 0; q < tr.K; ++q) dagger4(tr.V + ((int64_t)b * tr.K + q) * 16, &Vdag[((size_t)b * tr.K + q) * 16]);
  for (int l = depth; l >= 1; --l) {
    tr.Tt[l] = x;
    tr.DT[l] = dx;
    auto ly = tr.layers[l - 1];
    if ((depth - l) % 2 != 0) std::reverse(ly.begin(), ly.end());
    for (auto [kk, s] : ly) {
      std::vector<const cd*> vm(nb);
      for (int b = 0; b < nb; ++b) vm[b] = &Vdag[((size_t)b * tr.K + kk) * 16];
      tr.step(x, dx, s, &Gdag[(size_t)kk * 16], vm, bonds);
    }
  }
  cd t = 0;
  for (int64_t i = 0; i < dim; ++i) t += std::conj(x[i]) * tr.B[0][i];
  T[0] = t.real();
  T[1] = t.imag();
  // layer-wise E (X9) and H_T: future (DT), past (DB), in-layer (k' != k) channels
  std::vector<cd> E((size_t)tr.K * 16, 0);
  for (int l = 1; l <= depth; ++l) tr.layer_env(l, tr.Tt[l], tr.B[l - 1], -1, nullptr, E, false);
  for (size_t i = 0; i < E.size(); ++i) C(Ed)[i] = E[i];
  for (int b = 0; b < nb; ++b) {
    std::vector<cd> H((size_t)tr.K * 16, 0);
    for (int l = 1; l <= depth; ++l) {
      tr.layer_env(l, tr.DT[l][b], tr.B[l - 1], -1, nullptr, H, false);
      tr.layer_env(l, tr.Tt[l], tr.DB[l - 1][b], -1, nullptr, H, false);
      for (auto [kp, s] : tr.layers[l - 1])
        tr.layer_env(l, tr.Tt[l], tr.B[l - 1], kp, tr.V + ((int64_t)b * tr.K + kp) * 16, H, true);
    }
    for (size_t i = 0; i < H.size(); ++i) C(Hd)[(size_t)b * tr.K * 16 + i] = H[i];
  }
  return 0;
}

// Alg. 2 (X2) + App. E.  T: 2 doubles; E, HT: [K][16], [nb][K][16]; V: [nb][K][16].
// out: f (1 double), grad_R [K][16], hess_R [nb][K][16].
int tno_postprocess(int K, int nb, const double* Gd, const double* T2, const double* Ed, const double* HTd,
                    const double* Vd, double* f, double* gRd, double* hRd) {
  const cd* G = C(Gd);
  const cd* E = C(Ed);
  const cd T(T2[0], T2[1]);
  f[0] = -std::norm(T);
  auto proj = [](const cd* g, const cd* z, cd* out) {  // P_G(Z) = (Z - G Z^dag G) / 2
    cd w[16];
    for (int a = 0; a < 4; ++a)
      for (int c = 0; c < 4; ++c) {
        cd s = 0;
        for (int m = 0; m < 4; ++m) s += std::conj(z[m * 4 + a]) * g[m * 4 + c];
        w[a * 4 + c] = s;
      }
    for (int a = 0; a < 4; ++a)
      for (int c = 0; c < 4; ++c) {
        cd s = 0;
        for (int m = 0; m < 4; ++m) s += g[a * 4 + m] * w[m * 4 + c];
        out[a * 4 + c] = 0.5 * (z[a * 4 + c] - s);
      }
  };
  std::vector<cd> gf((size_t)K * 16);
  for (int i = 0; i < K * 16; ++i) gf[i] = -2.0 * T * std::conj(E[i]);
  for (int k = 0; k < K; ++k) proj(G + k * 16, &gf[(size_t)k * 16], C(gRd) + k * 16);
  for (int b = 0; b < nb; ++b) {
    const cd* V = C(Vd) + (size_t)b * K * 16;
    const cd* HT = C(HTd) + (size_t)b * K * 16;
    cd om = 0;
    for (int i = 0; i < K * 16; ++i) om += E[i] * V[i];
    for (int k = 0; k < K; ++k) {
      cd hf[16], gh[16], t1[16], t2[16], z[16];
      for (int i = 0; i < 16; ++i) hf[i] = -2.0 * (om * std::conj(E[k * 16 + i]) + T * std::conj(HT[k * 16 + i]));
      for (int a = 0; a < 4; ++a)
        for (int c = 0; c < 4; ++c) gh[a * 4 + c] = std::conj(gf[(size_t)k * 16 + c * 4 + a]);  // grad f^dag
      // t1 = V gh G, t2 = G gh V
      for (int a = 0; a < 4; ++a)
        for (int c = 0; c < 4; ++c) {
          cd s1 = 0, s2 = 0;
          for (int m = 0; m < 4; ++m)
            for (int q = 0; q < 4; ++q) {
              s1 += V[k * 16 + a * 4 + m] * gh[m * 4 + q] * G[k * 16 + q * 4 + c];
              s2 += G[k * 16 + a * 4 + m] * gh[m * 4 + q] * V[k * 16 + q * 4 + c];
            }
          t1[a * 4 + c] = s1;
          t2[a * 4 + c] = s2;
        }
      for (int i = 0; i < 16; ++i) z[i] = hf[i] - 0.5 * t1[i] - 0.5 * t2[i];
      proj(G + k * 16, z, C(hRd) + ((size_t)b * K + k) * 16);
    }
  }
  return 0;
}

}  // extern "C"
