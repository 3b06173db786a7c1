// TFPS alpha-space problem setup (NEXT-3; §2.2, readings R37-R39 in DESIGN.md §3),
// host fp64: per material the two local eigenproblems of eq:discretization_2D_eigenfunc_constraint,
//   x-modes: (gamma S - I) l = xi C l,   y-modes: (gamma S - I) l = xi S_y l,   gamma = sigma_s / sigma_t,
// then the basis values at the four face midpoints and the centre of a cell (eq:2D_eigenfunc).
//
// Eigen solver (our own; no LAPACK): S = K~ W is row-stochastic with positive entries, and the
// diagonal Delta_m = S_0m / S_m0 (Delta_0 = 1) symmetrises it (Delta S = W kappa W up to a factor, since
// K~ = D^-1 kappa with kappa symmetric).  Multiplying by Delta,
//   P l = lambda E l,   P = Delta (I - gamma S) (symmetric, strictly diagonally dominant with a positive
//   diagonal for gamma < 1, hence SPD),   E = Delta D (diagonal, D = C or S_y),   lambda = -xi.
// With P = R R^T (Cholesky) and y = R^T l:  R^-1 E R^-T y = (1/lambda) y, a symmetric eigenproblem,
// solved by cyclic Jacobi rotations.  So xi = -1/mu, l = R^-T y: every eigenvalue is real, as the
// paper's ordering presumes.  Eigenvectors are scaled to ||l||_inf = 1 with the largest-|.| entry
// positive (first index on ties).
#include <math.h>

#include <algorithm>
#include <map>
#include <numeric>
#include <tuple>
#include <vector>

#include "common.h"

namespace rte {

namespace {

// Cholesky P = R R^T (R lower, row-major n x n); fails if P is not SPD.
void cholesky(std::vector<double>& P, int n) {
  for (int j = 0; j < n; ++j) {
    double d = P[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= P[(size_t)j * n + k] * P[(size_t)j * n + k];
    RTE_REQUIRE(d > 0.0, "rte_setup_tfps: local operator not positive definite (sigma_t <= sigma_s?)");
    const double r = sqrt(d);
    P[(size_t)j * n + j] = r;
    for (int i = j + 1; i < n; ++i) {
      double s = P[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= P[(size_t)i * n + k] * P[(size_t)j * n + k];
      P[(size_t)i * n + j] = s / r;
    }
    for (int k = j + 1; k < n; ++k) P[(size_t)j * n + k] = 0.0;
  }
}

// Cyclic Jacobi eigen-decomposition of the symmetric A (destroyed): eigenvalues in ev, eigenvectors
// as the columns of V (row-major).
void jacobi_eig(std::vector<double>& A, int n, std::vector<double>& ev, std::vector<double>& V) {
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[(size_t)i * n + j]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += a(i, j) * a(i, j);
        if (i != j) off += a(i, j) * a(i, j);
      }
    if (off <= 1e-30 * tot) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (fabs(apq) < 1e-300) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // columns p, q
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // rows p, q
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
          V[(size_t)k * n + p] = c * vkp - s * vkq;
          V[(size_t)k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  ev.resize(n);
  for (int i = 0; i < n; ++i) ev[i] = a(i, i);
}

}  // namespace

// Modes of one material: xi [2M] (x-modes ascending, then y-modes ascending), L [M][2M] row-major
// (column k = eigenvector k).
void tfps_local_modes(const double* S, const std::vector<double>& c, const std::vector<double>& s, double gamma,
                      std::vector<double>& xi, std::vector<double>& L) {
  const int M = (int)c.size();
  RTE_REQUIRE(gamma >= 0.0 && gamma < 1.0, "rte_setup_tfps: need 0 <= sigma_s / sigma_t < 1");
  std::vector<double> delta(M);
  for (int m = 0; m < M; ++m) delta[m] = S[m] / S[(size_t)m * M];  // S_0m / S_m0
  xi.assign(2 * M, 0.0);
  L.assign((size_t)M * 2 * M, 0.0);
  for (int axis = 0; axis < 2; ++axis) {
    const std::vector<double>& d = axis == 0 ? c : s;
    std::vector<double> P((size_t)M * M);
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < M; ++j) {
        // symmetric part of Delta (I - gamma S) (exactly symmetric in exact arithmetic)
        const double a = delta[i] * ((i == j ? 1.0 : 0.0) - gamma * S[(size_t)i * M + j]);
        const double b = delta[j] * ((i == j ? 1.0 : 0.0) - gamma * S[(size_t)j * M + i]);
        P[(size_t)i * M + j] = 0.5 * (a + b);
      }
    cholesky(P, M);  // P = R R^T, R lower
    // T = R^-1 E R^-T with E = diag(delta d): first X = R^-1 diag(e) (forward substitution per column),
    // then T = X R^-T = (R^-1 X^T)^T
    std::vector<double> X((size_t)M * M, 0.0), Tm((size_t)M * M, 0.0);
    for (int col = 0; col < M; ++col) {  // solve R x = e_col * E_col
      std::vector<double> x(M, 0.0);
      for (int i = 0; i < M; ++i) {
        double r = (i == col ? delta[col] * d[col] : 0.0);
        for (int k = 0; k < i; ++k) r -= P[(size_t)i * M + k] * x[k];
        x[i] = r / P[(size_t)i * M + i];
      }
      for (int i = 0; i < M; ++i) X[(size_t)i * M + col] = x[i];
    }
    for (int row = 0; row < M; ++row) {  // solve R t = X[row, :]^T  ->  T[:, row] ... T symmetric
      std::vector<double> t(M, 0.0);
      for (int i = 0; i < M; ++i) {
        double r = X[(size_t)row * M + i];
        for (int k = 0; k < i; ++k) r -= P[(size_t)i * M + k] * t[k];
        t[i] = r / P[(size_t)i * M + i];
      }
      for (int i = 0; i < M; ++i) Tm[(size_t)row * M + i] = t[i];
    }
    for (int i = 0; i < M; ++i)  // symmetrise the rounding
      for (int j = i + 1; j < M; ++j) {
        const double v = 0.5 * (Tm[(size_t)i * M + j] + Tm[(size_t)j * M + i]);
        Tm[(size_t)i * M + j] = Tm[(size_t)j * M + i] = v;
      }
    std::vector<double> mu, Y;
    jacobi_eig(Tm, M, mu, Y);
    // xi = -1/mu, l = R^-T y (back substitution with R^T)
    std::vector<std::pair<double, std::vector<double>>> pairs;
    for (int k = 0; k < M; ++k) {
      RTE_REQUIRE(fabs(mu[k]) > 1e-300, "rte_setup_tfps: zero eigenvalue");
      std::vector<double> l(M);
      for (int i = M - 1; i >= 0; --i) {
        double r = Y[(size_t)i * M + k];
        for (int j = i + 1; j < M; ++j) r -= P[(size_t)j * M + i] * l[j];
        l[i] = r / P[(size_t)i * M + i];
      }
      double amax = 0.0;
      for (int i = 0; i < M; ++i) amax = std::max(amax, fabs(l[i]));
      int big = 0;  // the lowest index within 1e-9 of the largest magnitude (ties: the +-1 pairs)
      while (fabs(l[big]) < amax * (1.0 - 1e-9)) ++big;
      const double sc = l[big];
      for (double& v : l) v /= sc;
      pairs.emplace_back(-1.0 / mu[k], l);
    }
    std::sort(pairs.begin(), pairs.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (int k = 0; k < M; ++k) {
      xi[axis * M + k] = pairs[k].first;
      for (int i = 0; i < M; ++i) L[(size_t)i * 2 * M + axis * M + k] = pairs[k].second[i];
    }
  }
}

// Basis values of one material at the face midpoints f = L, R, B, T and the centre C of a cell of side
// h (eq:2D_eigenfunc with the R38 reference points): fac[f][k] = exp(sigma_t xi_k (z_f - z_ref,k)) along
// the mode's axis; chi^k(z_f) = fac[f][k] l^k.
void tfps_face_factors(const std::vector<double>& xi, int M, double sigma_t, double h, double* fac /*[5][2M]*/) {
  for (int k = 0; k < 2 * M; ++k) {
    const bool xmode = k < M;
    const double x = xi[k];
    // offset of each face midpoint from the reference face along the mode's axis
    // (reference: the low face for xi < 0, the high face for xi > 0)
    const double lo = x < 0 ? 0.0 : -h, hi = x < 0 ? h : 0.0, mid = x < 0 ? 0.5 * h : -0.5 * h;
    double off[5];
    if (xmode) {  // faces L, R along x; B, T, C at the centre in x
      off[0] = lo; off[1] = hi; off[2] = mid; off[3] = mid; off[4] = mid;
    } else {
      off[0] = mid; off[1] = mid; off[2] = lo; off[3] = hi; off[4] = mid;
    }
    for (int f = 0; f < 5; ++f) fac[(size_t)f * 2 * M + k] = exp(sigma_t * x * off[f]);
  }
}

// ---- ATFPS interface bases (NEXT-3b, readings R40-R42) ------------------------
namespace {

// Orthonormalise the columns of S (d x n, row-major) in order by Gram-Schmidt applied twice (CGS2, fp64;
// the same Q as a QR with positive diagonal); then each column gets its largest-|.| entry +1 (lowest
// index on ties within 1e-9) and ||.||_inf = 1 (R40).
void qr_eta(std::vector<double>& S, int d, int n) {
  for (int j = 0; j < n; ++j) {
    for (int pass = 0; pass < 2; ++pass)
      for (int q = 0; q < j; ++q) {
        double dot = 0.0, nq = 0.0;
        for (int i = 0; i < d; ++i) {
          dot += S[(size_t)i * n + q] * S[(size_t)i * n + j];
          nq += S[(size_t)i * n + q] * S[(size_t)i * n + q];
        }
        const double c = dot / nq;
        for (int i = 0; i < d; ++i) S[(size_t)i * n + j] -= c * S[(size_t)i * n + q];
      }
    double nr = 0.0;
    for (int i = 0; i < d; ++i) nr += S[(size_t)i * n + j] * S[(size_t)i * n + j];
    RTE_REQUIRE(nr > 0.0, "rte_setup_atfps: linearly dependent selected modes at an interface");
  }
  for (int j = 0; j < n; ++j) {  // (the scaling leaves the span and the orthogonality intact)
    double amax = 0.0;
    for (int i = 0; i < d; ++i) amax = std::max(amax, fabs(S[(size_t)i * n + j]));
    int big = 0;
    while (fabs(S[(size_t)big * n + j]) < amax * (1.0 - 1e-9)) ++big;
    const double sc = S[(size_t)big * n + j];
    for (int i = 0; i < d; ++i) S[(size_t)i * n + j] /= sc;
  }
}

// In-place inverse of the d x d row-major A by Gauss-Jordan with partial pivoting (fp64).
void invert(std::vector<double>& A, int d) {
  std::vector<double> I((size_t)d * d, 0.0);
  for (int i = 0; i < d; ++i) I[(size_t)i * d + i] = 1.0;
  for (int c = 0; c < d; ++c) {
    int piv = c;
    for (int r = c + 1; r < d; ++r)
      if (fabs(A[(size_t)r * d + c]) > fabs(A[(size_t)piv * d + c])) piv = r;
    RTE_REQUIRE(fabs(A[(size_t)piv * d + c]) > 0.0, "rte_setup_atfps: singular interface basis");
    if (piv != c)
      for (int k = 0; k < d; ++k) {
        std::swap(A[(size_t)c * d + k], A[(size_t)piv * d + k]);
        std::swap(I[(size_t)c * d + k], I[(size_t)piv * d + k]);
      }
    const double inv = 1.0 / A[(size_t)c * d + c];
    for (int k = 0; k < d; ++k) {
      A[(size_t)c * d + k] *= inv;
      I[(size_t)c * d + k] *= inv;
    }
    for (int r = 0; r < d; ++r) {
      if (r == c) continue;
      const double f = A[(size_t)r * d + c];
      if (f == 0.0) continue;
      for (int k = 0; k < d; ++k) {
        A[(size_t)r * d + k] -= f * A[(size_t)c * d + k];
        I[(size_t)r * d + k] -= f * I[(size_t)c * d + k];
      }
    }
  }
  A.swap(I);
}

}  // namespace

// One interface type: the centred modes of C- (`fm`, material a) and of C+ (`fp`, material b; fp < 0 for a
// boundary face of material a), restricted to the direction list `dirs`.  Modes are ordered
// [x-modes ascending | y-modes ascending], so the face a mode is centred at is k / (M/2) in L, R, B, T.
// Outputs P (d x d, row-major) and rowmap[2][2M] (the P-row of each centred mode of each side, -1 else).
void atfps_interface(const std::vector<double>& Lh /*[nmat][M][2M]*/, const std::vector<uint8_t>& sel /*[nmat][2M]*/,
                     int M, int a, int b, int fm, int fp, const std::vector<int>& dirs, std::vector<double>& P,
                     int* rowmap) {
  const int K = 2 * M, d = (int)dirs.size();
  std::vector<std::pair<int, int>> cols_s, cols_u;  // (side, k)
  for (int side = 0; side < 2; ++side) {
    const int f = side == 0 ? fm : fp;
    if (f < 0) continue;
    const int mt = side == 0 ? a : b;
    for (int k = f * (M / 2); k < (f + 1) * (M / 2); ++k)
      (sel[(size_t)mt * K + k] ? cols_s : cols_u).push_back({side, k});
  }
  const int ns = (int)cols_s.size(), n = ns + (int)cols_u.size();
  RTE_REQUIRE(n == d, "rte_setup_atfps: interface basis is not square");
  auto vecv = [&](int side, int k, int i) {
    const int mt = side == 0 ? a : b;
    return Lh[((size_t)mt * M + dirs[i]) * K + k];
  };
  std::vector<double> Sq((size_t)d * std::max(ns, 1), 0.0);
  for (int j = 0; j < ns; ++j)
    for (int i = 0; i < d; ++i) Sq[(size_t)i * ns + j] = vecv(cols_s[j].first, cols_s[j].second, i);
  if (ns > 0) qr_eta(Sq, d, ns);
  std::vector<double> E((size_t)d * d);
  for (int i = 0; i < d; ++i) {
    for (int j = 0; j < ns; ++j) E[(size_t)i * d + j] = Sq[(size_t)i * ns + j];
    for (int j = ns; j < d; ++j) E[(size_t)i * d + j] = vecv(cols_u[j - ns].first, cols_u[j - ns].second, i);
  }
  invert(E, d);
  P.swap(E);
  for (int t = 0; t < 2 * K; ++t) rowmap[t] = -1;
  for (int j = 0; j < n; ++j) {
    const auto& c = j < ns ? cols_s[j] : cols_u[j - ns];
    rowmap[c.first * K + c.second] = j;
  }
}

}  // namespace rte

namespace rte {

// The D_delta fit of the filtered loss (NEXT-4; reading R43): for one material, the
// minimum-norm least-squares solution operator of the collocation fit over the selected modes,
// Dp [2M][5M] row-major (rows of dropped modes 0; columns point-major C, L, R, B, T x direction), so that
// alpha = Dp (samples - chi^s).  G[p M + i][k] = L[i][k] fac[p][k] (the basis value chi^k_i at point p;
// fac order L, R, B, T, C) over the selected k.  Dp = V diag(1/lambda) V^T G^T from the Jacobi
// eigen-decomposition of G^T G; eigenvalues at or below 1e-13 lambda_max are dropped (the numerical null
// space of the fit: the minimum-norm solution).
void atfps_fit_pinv(const double* L, const double* fac, const uint8_t* sel, int M, double* Dp) {
  const int K = 2 * M, R = 5 * M;
  static const int fpos[5] = {4, 0, 1, 2, 3};  // point C, L, R, B, T -> fac row
  std::vector<int> ks;
  for (int k = 0; k < K; ++k)
    if (sel[k]) ks.push_back(k);
  const int n = (int)ks.size();
  std::fill(Dp, Dp + (size_t)K * R, 0.0);
  if (n == 0) return;
  std::vector<double> G((size_t)R * n);
  for (int p = 0; p < 5; ++p)
    for (int i = 0; i < M; ++i)
      for (int c = 0; c < n; ++c) G[((size_t)p * M + i) * n + c] = L[(size_t)i * K + ks[c]] * fac[(size_t)fpos[p] * K + ks[c]];
  std::vector<double> GtG((size_t)n * n, 0.0);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      double s = 0.0;
      for (int r = 0; r < R; ++r) s += G[(size_t)r * n + a] * G[(size_t)r * n + b];
      GtG[(size_t)a * n + b] = s;
    }
  std::vector<double> ev, V;
  jacobi_eig(GtG, n, ev, V);
  double lmax = 0.0;
  for (double l : ev) lmax = std::max(lmax, l);
  // X = V diag(1/lambda) V^T  (n x n), then Dp rows = X G^T
  std::vector<double> X((size_t)n * n, 0.0);
  for (int e = 0; e < n; ++e) {
    if (!(ev[e] > 1e-13 * lmax)) continue;
    const double inv = 1.0 / ev[e];
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) X[(size_t)a * n + b] += V[(size_t)a * n + e] * inv * V[(size_t)b * n + e];
  }
  for (int a = 0; a < n; ++a)
    for (int r = 0; r < R; ++r) {
      double s = 0.0;
      for (int b = 0; b < n; ++b) s += X[(size_t)a * n + b] * G[(size_t)r * n + b];
      Dp[(size_t)ks[a] * R + r] = s;
    }
}

}  // namespace rte
