// Host-side setup (layer L0) for libiga2l.  See host_setup.h.  Every formula cites the paper
// (arXiv 2009.01499, PAPER.md line P:<n>) or the DESIGN.md reading (A<n>) it implements.
#include "host_setup.h"

#include <algorithm>
#include <cmath>
#include <map>

namespace iga2l {

std::vector<double> knot_vector(int p, int64_t m) {
  // Ξ_{p,h} = {0 (p+1 times), 1/m, ..., (m-1)/m, 1 (p+1 times)}, ξ_{p+i+1} = i/m.
  std::vector<double> U(2 * p + m + 1);
  for (int i = 0; i <= p; ++i) U[i] = 0.0;
  for (int64_t i = 1; i < m; ++i) U[p + i] = double(i) / double(m);
  for (int i = 0; i <= p; ++i) U[p + m + i] = 1.0;
  return U;
}

void gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(pi * (i + 0.75) / (n + 0.5)), pp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {  // Legendre three-term recurrence
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      double z1 = z;
      z = z1 - p1 / pp;
      if (std::fabs(z - z1) < 1e-16) break;
    }
    x[i] = -z;
    x[n - 1 - i] = z;
    w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

void basis_on_span(const std::vector<double> &U, int p, int k, double x, double *N, double *dN) {
  // Triangular evaluation of the Cox–de Boor recursion on span [U[k], U[k+1]):
  // after step j, ndu[0..j] = N^j_{k-j..k}(x).  Fractions 0/0 never arise for non-zero terms.
  double left[17], right[17], ndu[17], prev[17];
  ndu[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = x - U[k + 1 - j];
    right[j] = U[k + j] - x;
    if (j == p)
      for (int r = 0; r < p; ++r) prev[r] = ndu[r];  // degree p-1 values of N_{k-p+1..k}
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      double temp = ndu[r] / (right[r + 1] + left[j - r]);
      ndu[r] = saved + right[r + 1] * temp;
      saved = left[j - r] * temp;
    }
    ndu[j] = saved;
  }
  for (int r = 0; r <= p; ++r) N[r] = ndu[r];
  if (!dN) return;
  // N_i^p' = p/(ξ_{i+p}-ξ_i) N_i^{p-1} - p/(ξ_{i+p+1}-ξ_{i+1}) N_{i+1}^{p-1}, i = k-p+r.
  for (int r = 0; r <= p; ++r) {
    if (p == 0) { dN[r] = 0.0; continue; }
    int i = k - p + r;
    double a = (r >= 1) ? prev[r - 1] / (U[i + p] - U[i]) : 0.0;
    double b = (r <= p - 1) ? prev[r] / (U[i + p + 1] - U[i + 1]) : 0.0;
    dN[r] = p * (a - b);
  }
}

void band_tables(int p, int64_t m, std::vector<double> &K, std::vector<double> &M) {
  // Element-by-element Gauss quadrature with p+1 points per span (exact for the degree-2p
  // integrands of a(u,v) = ∫u'v' and the mass) over the full basis, then the Dirichlet
  // functions N_1, N_{m+p} are dropped.
  const std::vector<double> U = knot_vector(p, m);
  const int64_t nf = m + p, n1 = nf - 2;
  const int W = 2 * p + 1;
  std::vector<double> Kf(nf * W, 0.0), Mf(nf * W, 0.0), gx, gw;
  gauss_legendre(p + 1, gx, gw);
  double N[17], dN[17];
  for (int64_t e = 0; e < m; ++e) {
    const int k = int(p + e);
    const double a = U[k], b = U[k + 1], mid = 0.5 * (a + b), half = 0.5 * (b - a);
    for (size_t g = 0; g < gx.size(); ++g) {
      const double x = mid + half * gx[g], wq = half * gw[g];
      basis_on_span(U, p, k, x, N, dN);
      for (int r1 = 0; r1 <= p; ++r1)
        for (int r2 = 0; r2 <= p; ++r2) {
          const int64_t f1 = e + r1;
          const int t = r2 - r1;
          Kf[f1 * W + t + p] += wq * dN[r1] * dN[r2];
          Mf[f1 * W + t + p] += wq * N[r1] * N[r2];
        }
    }
  }
  K.assign(std::max<int64_t>(n1, 0) * W, 0.0);
  M.assign(std::max<int64_t>(n1, 0) * W, 0.0);
  for (int64_t i = 0; i < n1; ++i)
    for (int t = -p; t <= p; ++t) {
      if (i + t < 0 || i + t >= n1) continue;
      K[i * W + t + p] = Kf[(i + 1) * W + t + p];
      M[i * W + t + p] = Mf[(i + 1) * W + t + p];
    }
  // Interior rows: every basis function they couple is a uniform (translated) B-spline, so the rows
  // are mathematically identical (cardinal B-spline values, SURVEY §8(c) pins); the quadrature
  // above reproduces them only up to rounding.  Make them bitwise identical (one representative
  // row) so that kernels may hold them in registers (Toeplitz) and every interior block has the same
  // local matrix.  Changes entries by a few ulp.
  int64_t lo, hi;
  toeplitz_rows(p, m, &lo, &hi);
  if (lo <= hi) {
    const int64_t ref = (lo + hi) / 2;
    for (int64_t i = lo; i <= hi; ++i)
      for (int t = 0; t < W; ++t) {
        K[i * W + t] = K[ref * W + t];
        M[i * W + t] = M[ref * W + t];
      }
  }
}

void toeplitz_rows(int p, int64_t m, int64_t *lo, int64_t *hi) {
  // constrained row i = full function f = i + 1; f and its neighbours f-p..f+p are uniform B-splines
  // (support inside [ξ_{p+1}, ξ_{m+p+1}] with simple knots) iff 2p <= f <= m - 1 - p.
  *lo = 2 * int64_t(p) - 1;
  *hi = m - 2 - int64_t(p);
}

std::vector<double> load_1d_sine(int p, int64_t m) {
  const std::vector<double> U = knot_vector(p, m);
  const int64_t nf = m + p;
  std::vector<double> gf(nf, 0.0), gx, gw;
  gauss_legendre(p + 3, gx, gw);
  const double pi = 3.14159265358979323846;
  double N[17];
  for (int64_t e = 0; e < m; ++e) {
    const int k = int(p + e);
    const double a = U[k], b = U[k + 1], mid = 0.5 * (a + b), half = 0.5 * (b - a);
    for (size_t g = 0; g < gx.size(); ++g) {
      const double x = mid + half * gx[g], wq = half * gw[g];
      basis_on_span(U, p, k, x, N, nullptr);
      const double f = std::sin(pi * x);
      for (int r = 0; r <= p; ++r) gf[e + r] += wq * f * N[r];
    }
  }
  return std::vector<double>(gf.begin() + 1, gf.end() - 1);
}

BandOp degree_restriction(int p, int q, int64_t m) {
  // (M_p^q)_{ij} = ∫ φ_i^q φ_j^p, lumped (M_q^q) -> D (reading A6).
  const std::vector<double> Up = knot_vector(p, m), Uq = knot_vector(q, m);
  const int64_t nfq = m + q, n1q = nfq - 2, n1p = m + p - 2;
  const int W = p + q + 1;
  std::vector<double> Mf(nfq * W, 0.0), gx, gw;  // row fi: cols fj = fi - q + k
  gauss_legendre(std::max(p, q) + 1, gx, gw);
  double Np[17], Nq[17];
  for (int64_t e = 0; e < m; ++e) {
    const double a = Up[p + e], b = Up[p + e + 1], mid = 0.5 * (a + b), half = 0.5 * (b - a);
    for (size_t g = 0; g < gx.size(); ++g) {
      const double x = mid + half * gx[g], wq = half * gw[g];
      basis_on_span(Up, p, int(p + e), x, Np, nullptr);
      basis_on_span(Uq, q, int(q + e), x, Nq, nullptr);
      for (int rq = 0; rq <= q; ++rq)
        for (int rp = 0; rp <= p; ++rp) {
          const int64_t fi = e + rq, fj = e + rp;
          Mf[fi * W + (fj - (fi - q))] += wq * Nq[rq] * Np[rp];
        }
    }
  }
  BandOp R;
  R.rows = int(n1q);
  R.cols = int(n1p);
  R.W = W;
  R.lo.resize(n1q);
  R.c.assign(n1q * W, 0.0);
  for (int64_t ic = 0; ic < n1q; ++ic) {
    const int64_t fi = ic + 1;
    const double D = (Uq[fi + q + 1] - Uq[fi]) / (q + 1);  // ∫ N_i^q (reading A6)
    R.lo[ic] = int(ic - q);                                // constrained col = fj - 1
    for (int k = 0; k < W; ++k) {
      const int64_t jc = ic - q + k;
      if (jc < 0 || jc >= n1p) continue;
      R.c[ic * W + k] = Mf[fi * W + k] / D;
    }
  }
  return R;
}

static BandOp band_from_dense(const std::vector<std::vector<double>> &rows, int cols) {
  BandOp B;
  B.rows = int(rows.size());
  B.cols = cols;
  B.lo.assign(B.rows, 0);
  int W = 1;
  std::vector<int> hi(B.rows, 0);
  for (int r = 0; r < B.rows; ++r) {
    int lo = -1, h = -1;
    for (int c = 0; c < cols; ++c)
      if (rows[r][c] != 0.0) {
        if (lo < 0) lo = c;
        h = c;
      }
    if (lo < 0) lo = h = std::min(r, cols - 1);
    B.lo[r] = lo;
    hi[r] = h;
    W = std::max(W, h - lo + 1);
  }
  B.W = W;
  B.c.assign((size_t)B.rows * W, 0.0);
  for (int r = 0; r < B.rows; ++r)
    for (int c = B.lo[r]; c <= hi[r]; ++c) B.c[(size_t)r * W + (c - B.lo[r])] = rows[r][c];
  return B;
}

BandOp mesh_prolongation(int q, int64_t mc) {
  // Boehm knot insertion of every midpoint (2j+1)/(2mc) into Ξ_{q,2h}: the coefficients of each
  // coarse B-spline in the fine basis (exact embedding of nested spaces, reading A8).
  std::vector<double> U = knot_vector(q, mc);
  const int ncf = int(mc + q);
  std::vector<std::vector<double>> P(ncf, std::vector<double>(ncf, 0.0));
  for (int i = 0; i < ncf; ++i) P[i][i] = 1.0;
  for (int64_t j = 0; j < mc; ++j) {
    const double xn = double(2 * j + 1) / double(2 * mc);
    int k = 0;
    while (!(U[k] <= xn && xn < U[k + 1])) ++k;
    std::vector<std::vector<double>> Q(P.size() + 1, std::vector<double>(ncf, 0.0));
    for (int i = 0; i < (int)Q.size(); ++i) {
      if (i <= k - q) Q[i] = P[i];
      else if (i >= k + 1) Q[i] = P[i - 1];
      else {
        const double al = (xn - U[i]) / (U[i + q] - U[i]);
        for (int c = 0; c < ncf; ++c) Q[i][c] = al * P[i][c] + (1.0 - al) * P[i - 1][c];
      }
    }
    U.insert(U.begin() + k + 1, xn);
    P.swap(Q);
  }
  // constrained: drop first/last fine rows and coarse columns (Dirichlet functions)
  std::vector<std::vector<double>> Pc;
  for (size_t i = 1; i + 1 < P.size(); ++i)
    Pc.emplace_back(P[i].begin() + 1, P[i].end() - 1);
  return band_from_dense(Pc, ncf - 2);
}

BandOp transpose(const BandOp &A) {
  std::vector<std::vector<double>> T(A.cols, std::vector<double>(A.rows, 0.0));
  for (int r = 0; r < A.rows; ++r)
    for (int k = 0; k < A.W; ++k) {
      const int c = A.lo[r] + k;
      if (c >= 0 && c < A.cols) T[c][r] = A.c[(size_t)r * A.W + k];
    }
  return band_from_dense(T, A.rows);
}

BandOp multiply(const BandOp &A, const BandOp &B) {
  std::vector<std::vector<double>> C(A.rows, std::vector<double>(B.cols, 0.0));
  for (int r = 0; r < A.rows; ++r)
    for (int k = 0; k < A.W; ++k) {
      const int mid = A.lo[r] + k;
      if (mid < 0 || mid >= A.cols) continue;
      const double a = A.c[(size_t)r * A.W + k];
      if (a == 0.0) continue;
      for (int k2 = 0; k2 < B.W; ++k2) {
        const int c = B.lo[mid] + k2;
        if (c >= 0 && c < B.cols) C[r][c] += a * B.c[(size_t)mid * B.W + k2];
      }
    }
  return band_from_dense(C, B.cols);
}

// ---- small dense SPD helpers (k <= 7 for FD, N <= 2048 for the coarse inverse) ----
static bool cholesky(std::vector<double> &A, int n) {  // lower, in place, row-major
  for (int j = 0; j < n; ++j) {
    double d = A[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    A[(size_t)j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = A[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
      A[(size_t)i * n + j] = s / d;
    }
    for (int i = 0; i < j; ++i) A[(size_t)i * n + j] = 0.0;
  }
  return true;
}

static void jacobi_eigen(std::vector<double> &C, int n, std::vector<double> &Q, std::vector<double> &lam) {
  // cyclic Jacobi for a symmetric n x n matrix: C = Q diag(lam) Q^T
  Q.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) Q[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += C[(size_t)i * n + j] * C[(size_t)i * n + j];
    if (off < 1e-34) break;
    for (int pi = 0; pi < n; ++pi)
      for (int qi = pi + 1; qi < n; ++qi) {
        const double apq = C[(size_t)pi * n + qi];
        if (apq == 0.0) continue;
        const double app = C[(size_t)pi * n + pi], aqq = C[(size_t)qi * n + qi];
        const double theta = 0.5 * (aqq - app) / apq;
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // rotate columns p, q
          const double ckp = C[(size_t)k * n + pi], ckq = C[(size_t)k * n + qi];
          C[(size_t)k * n + pi] = c * ckp - s * ckq;
          C[(size_t)k * n + qi] = s * ckp + c * ckq;
        }
        for (int k = 0; k < n; ++k) {  // rotate rows p, q
          const double cpk = C[(size_t)pi * n + k], cqk = C[(size_t)qi * n + k];
          C[(size_t)pi * n + k] = c * cpk - s * cqk;
          C[(size_t)qi * n + k] = s * cpk + c * cqk;
        }
        for (int k = 0; k < n; ++k) {
          const double qkp = Q[(size_t)k * n + pi], qkq = Q[(size_t)k * n + qi];
          Q[(size_t)k * n + pi] = c * qkp - s * qkq;
          Q[(size_t)k * n + qi] = s * qkp + c * qkq;
        }
      }
  }
  lam.resize(n);
  for (int i = 0; i < n; ++i) lam[i] = C[(size_t)i * n + i];
}

bool fd_tables(int p, int s, int64_t n1, const std::vector<double> &K, const std::vector<double> &M,
               std::vector<double> &V, std::vector<double> &lam) {
  const int w = (s - 1) / 2, W = 2 * p + 1;
  V.assign((size_t)n1 * s * s, 0.0);
  lam.assign((size_t)n1 * s, 1.0);
  for (int64_t c = 0; c < n1; ++c) {
    const int64_t lo = std::max<int64_t>(0, c - w), hi = std::min<int64_t>(n1 - 1, c + w);
    const int L = int(hi - lo + 1), off = int(lo - (c - w));  // local row of global lo
    std::vector<double> KI((size_t)L * L, 0.0), MI((size_t)L * L, 0.0);
    for (int a = 0; a < L; ++a)
      for (int b = 0; b < L; ++b) {
        const int t = b - a;
        if (t < -p || t > p) continue;
        KI[(size_t)a * L + b] = K[(lo + a) * W + t + p];
        MI[(size_t)a * L + b] = M[(lo + a) * W + t + p];
      }
    // generalized symmetric eigenproblem via M = L L^T: C = L^{-1} K L^{-T}, V = L^{-T} Q
    std::vector<double> Lc = MI;
    if (!cholesky(Lc, L)) return false;
    std::vector<double> X((size_t)L * L);  // X = L^{-1} K
    for (int col = 0; col < L; ++col)
      for (int i = 0; i < L; ++i) {
        double sacc = KI[(size_t)i * L + col];
        for (int k = 0; k < i; ++k) sacc -= Lc[(size_t)i * L + k] * X[(size_t)k * L + col];
        X[(size_t)i * L + col] = sacc / Lc[(size_t)i * L + i];
      }
    std::vector<double> C((size_t)L * L);  // C = X L^{-T}  <=>  C^T = L^{-1} X^T
    for (int row = 0; row < L; ++row)
      for (int i = 0; i < L; ++i) {
        double sacc = X[(size_t)row * L + i];
        for (int k = 0; k < i; ++k) sacc -= Lc[(size_t)i * L + k] * C[(size_t)row * L + k];
        C[(size_t)row * L + i] = sacc / Lc[(size_t)i * L + i];
      }
    for (int i = 0; i < L; ++i)  // symmetrise rounding
      for (int j = i + 1; j < L; ++j) {
        const double avg = 0.5 * (C[(size_t)i * L + j] + C[(size_t)j * L + i]);
        C[(size_t)i * L + j] = C[(size_t)j * L + i] = avg;
      }
    std::vector<double> Q, ev;
    jacobi_eigen(C, L, Q, ev);
    for (int j = 0; j < L; ++j) {
      if (!(ev[j] > 0.0)) return false;
      // v = L^{-T} q_j (back substitution with L^T)
      std::vector<double> v(L);
      for (int i = L - 1; i >= 0; --i) {
        double sacc = Q[(size_t)i * L + j];
        for (int k = i + 1; k < L; ++k) sacc -= Lc[(size_t)k * L + i] * v[k];
        v[i] = sacc / Lc[(size_t)i * L + i];
      }
      for (int i = 0; i < L; ++i) V[((size_t)c * s + (off + i)) * s + j] = v[i];
      lam[(size_t)c * s + j] = ev[j];
    }
  }
  return true;
}

bool dense_kron_inverse(int dim, int q, int n, const std::vector<double> &K, const std::vector<double> &M,
                        std::vector<double> &inv, int64_t ays) {
  const int W = 2 * q + 1;
  int N = 1;
  for (int a = 0; a < dim; ++a) N *= n;
  std::vector<double> A((size_t)N * N, 0.0);
  auto band = [&](const std::vector<double> &T, int a, int i, int j) -> double {   // axis a's table
    const int t = j - i;
    return (t < -q || t > q) ? 0.0 : T[(size_t)(a * ays) + (size_t)i * W + t + q];
  };
  for (int g = 0; g < N; ++g)
    for (int h = 0; h < N; ++h) {
      int ig[3] = {g % n, (g / n) % n, g / (n * n)}, ih[3] = {h % n, (h / n) % n, h / (n * n)};
      bool near = true;
      for (int a = 0; a < dim; ++a) near &= std::abs(ig[a] - ih[a]) <= q;
      if (!near) continue;
      double v = 0.0;  // Σ_a ⊗(K on axis a, M elsewhere) (tensor-product basis)
      for (int a = 0; a < dim; ++a) {
        double t = 1.0;
        for (int b = 0; b < dim; ++b) t *= (a == b) ? band(K, b, ig[b], ih[b]) : band(M, b, ig[b], ih[b]);
        v += t;
      }
      A[(size_t)g * N + h] = v;
    }
  if (!cholesky(A, N)) return false;
  inv.assign((size_t)N * N, 0.0);
  std::vector<double> y(N);
  for (int col = 0; col < N; ++col) {
    for (int i = 0; i < N; ++i) {  // L y = e_col
      double sacc = (i == col) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) sacc -= A[(size_t)i * N + k] * y[k];
      y[i] = sacc / A[(size_t)i * N + i];
    }
    for (int i = N - 1; i >= 0; --i) {  // L^T x = y
      double sacc = y[i];
      for (int k = i + 1; k < N; ++k) sacc -= A[(size_t)k * N + i] * inv[(size_t)k * N + col];
      inv[(size_t)i * N + col] = sacc / A[(size_t)i * N + i];
    }
  }
  return true;
}


// ---- symmetric eigen-decomposition for larger n (coarse-level fast diagonalisation) ----------
// Householder tridiagonalisation, then implicit symmetric QR steps with the Wilkinson shift and
// Givens rotations accumulated into Q (Golub & Van Loan, Matrix Computations, Alg. 8.3.1 / 8.3.2).
// A: n x n symmetric, row-major (destroyed).  On return A = Q diag(lam) Q^T, Q row-major.
static void sym_eigen(std::vector<double> &A, int n, std::vector<double> &Q, std::vector<double> &lam) {
  auto a = [&](int i, int j) -> double & { return A[(size_t)i * n + j]; };
  std::vector<double> vs((size_t)n * n, 0.0), betas(n, 0.0), v(n), pv(n), wv(n);
  for (int k = 0; k + 2 < n; ++k) {                  // Householder: zero A[k+2:, k]
    double sig = 0.0;
    for (int i = k + 2; i < n; ++i) sig += a(i, k) * a(i, k);
    const double x0 = a(k + 1, k);
    if (sig == 0.0) { betas[k] = 0.0; continue; }
    const double mu = std::sqrt(x0 * x0 + sig);
    const double v0 = x0 <= 0.0 ? x0 - mu : -sig / (x0 + mu);
    const double beta = 2.0 * v0 * v0 / (sig + v0 * v0);
    for (int i = k + 1; i < n; ++i) v[i] = (i == k + 1) ? 1.0 : a(i, k) / v0;
    betas[k] = beta;
    for (int i = k + 1; i < n; ++i) vs[(size_t)k * n + i] = v[i];
    for (int i = k + 1; i < n; ++i) {                // p = beta A v (trailing block)
      double t = 0.0;
      for (int j = k + 1; j < n; ++j) t += a(i, j) * v[j];
      pv[i] = beta * t;
    }
    double pvv = 0.0;
    for (int i = k + 1; i < n; ++i) pvv += pv[i] * v[i];
    for (int i = k + 1; i < n; ++i) wv[i] = pv[i] - 0.5 * beta * pvv * v[i];
    for (int i = k + 1; i < n; ++i)
      for (int j = k + 1; j < n; ++j) a(i, j) -= v[i] * wv[j] + wv[i] * v[j];
    a(k + 1, k) = a(k, k + 1) = mu;                    // P x = ||x|| e_1 (GVL house)
    for (int i = k + 2; i < n; ++i) a(i, k) = a(k, i) = 0.0;
  }
  std::vector<double> d(n), e(n, 0.0);
  for (int i = 0; i < n; ++i) d[i] = a(i, i);
  for (int i = 0; i + 1 < n; ++i) e[i] = a(i + 1, i);
  Q.assign((size_t)n * n, 0.0);                        // Q = H_0 H_1 ... H_{n-3}
  for (int i = 0; i < n; ++i) Q[(size_t)i * n + i] = 1.0;
  for (int k = n - 3; k >= 0; --k) {
    if (betas[k] == 0.0) continue;
    const double *vk = &vs[(size_t)k * n];
    for (int j = k + 1; j < n; ++j) {
      double t = 0.0;
      for (int i = k + 1; i < n; ++i) t += vk[i] * Q[(size_t)i * n + j];
      t *= betas[k];
      for (int i = k + 1; i < n; ++i) Q[(size_t)i * n + j] -= t * vk[i];
    }
  }
  // implicit symmetric QR on (d, e); rotations applied to the columns of Q
  int hi = n - 1;
  int guard = 0;
  while (hi > 0 && guard < 100 * n) {
    ++guard;
    for (int i = 0; i < hi; ++i)
      if (std::fabs(e[i]) <= 1e-16 * (std::fabs(d[i]) + std::fabs(d[i + 1]))) e[i] = 0.0;
    if (e[hi - 1] == 0.0) { --hi; continue; }
    int lo = hi - 1;
    while (lo > 0 && e[lo - 1] != 0.0) --lo;
    const double dd = 0.5 * (d[hi - 1] - d[hi]), eh = e[hi - 1];
    const double mu = d[hi] - eh * eh / (dd + (dd >= 0 ? 1.0 : -1.0) * std::sqrt(dd * dd + eh * eh));
    double x = d[lo] - mu, z = e[lo];
    for (int k = lo; k < hi; ++k) {
      double c, s_;
      if (z == 0.0) { c = 1.0; s_ = 0.0; }
      else if (std::fabs(z) > std::fabs(x)) { const double t = -x / z; s_ = 1.0 / std::sqrt(1.0 + t * t); c = s_ * t; }
      else { const double t = -z / x; c = 1.0 / std::sqrt(1.0 + t * t); s_ = c * t; }
      // rotation G = [c s; -s c] on rows/cols k, k+1 of T
      if (k > lo) e[k - 1] = c * e[k - 1] - s_ * z;
      const double dk = d[k], dk1 = d[k + 1], ek = e[k];
      d[k] = c * c * dk - 2.0 * c * s_ * ek + s_ * s_ * dk1;
      d[k + 1] = s_ * s_ * dk + 2.0 * c * s_ * ek + c * c * dk1;
      e[k] = c * s_ * (dk - dk1) + (c * c - s_ * s_) * ek;
      if (k + 1 < hi) { x = e[k]; z = -s_ * e[k + 1]; e[k + 1] = c * e[k + 1]; }
      for (int i = 0; i < n; ++i) {
        const double qk = Q[(size_t)i * n + k], qk1 = Q[(size_t)i * n + k + 1];
        Q[(size_t)i * n + k] = c * qk - s_ * qk1;
        Q[(size_t)i * n + k + 1] = s_ * qk + c * qk1;
      }
    }
  }
  lam = d;
}

bool coarse_fd_tables(int q, int64_t m, std::vector<double> &V, std::vector<double> &lam) {
  std::vector<double> Kb, Mb;
  band_tables(q, m, Kb, Mb);
  return band_fd_tables(q, int(m + q - 2), Kb.data(), Mb.data(), V, lam);
}

bool band_fd_tables(int q, int n, const double *Kb, const double *Mb, std::vector<double> &V, std::vector<double> &lam) {
  // generalized problem K V = M V Λ with V^T M V = I for constrained degree-q band tables:
  // M = L L^T, C = L^{-1} K L^{-T} = Q Λ Q^T, V = L^{-T} Q  (then A_q^{-1} = (⊗V)(Σ_a λ)^{-1}(⊗V)^T)
  const int W = 2 * q + 1;
  if (n < 1) return false;
  std::vector<double> Kd((size_t)n * n, 0.0), L((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int t = 0; t < W; ++t) {
      const int j = i + t - q;
      if (j < 0 || j >= n) continue;
      Kd[(size_t)i * n + j] = Kb[(size_t)i * W + t];
      L[(size_t)i * n + j] = Mb[(size_t)i * W + t];
    }
  if (!cholesky(L, n)) return false;
  // C = L^{-1} K L^{-T}: X = L^{-1} K (forward substitution per column), C = L^{-1} X^T
  auto fwd = [&](std::vector<double> &B) {            // B <- L^{-1} B (all columns)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double sacc = B[(size_t)i * n + j];
        for (int k = std::max(0, i - q); k < i; ++k) sacc -= L[(size_t)i * n + k] * B[(size_t)k * n + j];
        B[(size_t)i * n + j] = sacc / L[(size_t)i * n + i];
      }
  };
  fwd(Kd);                                             // L^{-1} K
  std::vector<double> C((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) C[(size_t)i * n + j] = Kd[(size_t)j * n + i];   // (L^{-1} K)^T = K L^{-T}
  fwd(C);                                              // L^{-1} K L^{-T}
  for (int i = 0; i < n; ++i)                          // symmetrise
    for (int j = i + 1; j < n; ++j) {
      const double av = 0.5 * (C[(size_t)i * n + j] + C[(size_t)j * n + i]);
      C[(size_t)i * n + j] = C[(size_t)j * n + i] = av;
    }
  std::vector<double> Q;
  sym_eigen(C, n, Q, lam);
  for (double l : lam)
    if (!(l > 0.0)) return false;
  // V = L^{-T} Q: back substitution with L^T (upper, bandwidth q)
  V = Q;
  for (int j = 0; j < n; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double sacc = V[(size_t)i * n + j];
      for (int k = i + 1; k <= std::min(n - 1, i + q); ++k) sacc -= L[(size_t)k * n + i] * V[(size_t)k * n + j];
      V[(size_t)i * n + j] = sacc / L[(size_t)i * n + i];
    }
  return true;
}

bool periodic_fd_tables(int q, int n, const double *krow, const double *mrow, std::vector<double> &V,
                        std::vector<double> &lam) {
  // circulant K, M (row i: column (i + t - q) mod n holds krow[t], mrow[t]); M = L L^T (dense Cholesky:
  // the periodic factor fills in), C = L^{-1} K L^{-T} = Q Λ Q^T, V = L^{-T} Q.  K annihilates constants,
  // so one λ vanishes: it is returned as exactly 0 (the caller's solve uses the pseudo-inverse).
  const int W = 2 * q + 1;
  if (n < W) return false;
  std::vector<double> Kd((size_t)n * n, 0.0), L((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int t = 0; t < W; ++t) {
      const int j = ((i + t - q) % n + n) % n;
      Kd[(size_t)i * n + j] += krow[t];
      L[(size_t)i * n + j] += mrow[t];
    }
  if (!cholesky(L, n)) return false;
  auto fwd = [&](std::vector<double> &B) {            // B <- L^{-1} B (dense lower L)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double sacc = B[(size_t)i * n + j];
        for (int k = 0; k < i; ++k) sacc -= L[(size_t)i * n + k] * B[(size_t)k * n + j];
        B[(size_t)i * n + j] = sacc / L[(size_t)i * n + i];
      }
  };
  fwd(Kd);
  std::vector<double> C((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) C[(size_t)i * n + j] = Kd[(size_t)j * n + i];
  fwd(C);
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double av = 0.5 * (C[(size_t)i * n + j] + C[(size_t)j * n + i]);
      C[(size_t)i * n + j] = C[(size_t)j * n + i] = av;
    }
  std::vector<double> Q;
  sym_eigen(C, n, Q, lam);
  double mx = 0.0;
  for (double l : lam) mx = std::max(mx, std::fabs(l));
  int nz = 0;
  for (double &l : lam)
    if (std::fabs(l) <= 1e-10 * mx) {
      l = 0.0;
      ++nz;
    } else if (l < 0.0) {
      return false;
    }
  if (nz != 1) return false;
  V = Q;
  for (int j = 0; j < n; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double sacc = V[(size_t)i * n + j];
      for (int k = i + 1; k < n; ++k) sacc -= L[(size_t)k * n + i] * V[(size_t)k * n + j];
      V[(size_t)i * n + j] = sacc / L[(size_t)i * n + i];
    }
  return true;
}

}  // namespace iga2l
