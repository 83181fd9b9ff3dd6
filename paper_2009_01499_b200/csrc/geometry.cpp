// Host-side setup for the quarter-annulus NURBS workload (geometry P:132-151; SURVEY §8(f)
// row 3).  Independent of oracle/ (shares no code).  See host_setup.h for the contracts.
//
// Geometry: F(ξ, η) = ρ(η) c(ξ), c the exact quarter circle as the rational quadratic Bézier arc with
// control points (1,0), (1,1), (0,1) and weights 1, √2/2, 1; ρ(η) = r + (R - r) η,
// r = 0.3, R = 0.5.  |c| = 1, so the Jacobian columns ρ c' and ρ' c are orthogonal and
// |det J| = ρ ρ' s with s = |c'|.  Hence, for φ_ik = R_i(ξ) N_k(η),
//     a(φ_ik, φ_jl) = ∫ R_i' R_j' / s dξ ∫ N_k N_l ρ'/ρ dη + ∫ R_i R_j s dξ ∫ N_k' N_l' ρ/ρ' dη,
// i.e. A = My ⊗ Kx + Ky ⊗ Mx: the SAME Kronecker-sum form as on the square with one pair of
// weighted 1D band tables per axis -- every device kernel of the 2D path runs it with per-axis tables.
// The L2 mass (transfers, load vector) has the separable weight |det J| = (s)(ρ ρ').
//
// NURBS space: R_i = w_i N_i / W, W(ξ) = Σ ω_k B_k^2(ξ) the arc's weight function and w its
// coefficients in the degree-p basis.  W is a quadratic polynomial, so for p >= 2 the coefficients follow
// from the blossom (Marsden's identity): for f(ξ) = a0 + a1 ξ + a2 ξ²,
//     w_i = a0 + a1 σ1/p + a2 σ2 / C(p, 2),   σ1 = Σ u_k, σ2 = Σ_{j<k} u_j u_k over u = ξ_{i+1..i+p}.
// Quadrature: (deg + 3) Gauss points per span for the 1D tables, cross mass and load (the integrands
// are rational; reading A29: the same rule as the oracle, not exact).
#include <cmath>

#include "host_setup.h"

namespace iga2l {
namespace {

constexpr double kRin = 0.3, kRout = 0.5;
const double kW1 = std::sqrt(2.0) / 2.0;

// c(ξ), c'(ξ) of the rational quadratic arc
void arc(double xi, double c[2], double dc[2]) {
  const double b0 = (1 - xi) * (1 - xi), b1 = 2 * xi * (1 - xi), b2 = xi * xi;
  const double d0 = -2 * (1 - xi), d1 = 2 - 4 * xi, d2 = 2 * xi;
  const double W = b0 + kW1 * b1 + b2, dW = d0 + kW1 * d1 + d2;
  const double nx = b0 + kW1 * b1, ny = kW1 * b1 + b2;      // Σ ω_k B_k P_k, P = (1,0), (1,1), (0,1)
  const double dnx = d0 + kW1 * d1, dny = kW1 * d1 + d2;
  c[0] = nx / W;
  c[1] = ny / W;
  dc[0] = (dnx * W - nx * dW) / (W * W);
  dc[1] = (dny * W - ny * dW) / (W * W);
}

double arc_speed(double xi) {
  double c[2], dc[2];
  arc(xi, c, dc);
  return std::hypot(dc[0], dc[1]);
}

}  // namespace

std::vector<double> nurbs_weights(int p, int64_t m) {
  // W(ξ) = (1-ξ)² + √2 ξ(1-ξ) + ξ² = 1 + (√2 - 2) ξ + (2 - √2) ξ²
  const double a0 = 1.0, a1 = std::sqrt(2.0) - 2.0, a2 = 2.0 - std::sqrt(2.0);
  const std::vector<double> U = knot_vector(p, m);
  const int64_t nf = m + p;
  std::vector<double> w(nf);
  for (int64_t i = 0; i < nf; ++i) {
    double s1 = 0.0, s2 = 0.0;
    for (int j = 1; j <= p; ++j) {
      s2 += s1 * U[i + j];          // Σ_{j' < j} u_j' u_j
      s1 += U[i + j];
    }
    w[i] = a0 + a1 * s1 / p + a2 * s2 / (0.5 * p * (p - 1));
  }
  return w;
}

void nurbs_on_span(const std::vector<double> &U, const std::vector<double> &w, int p, int64_t e, double x, double *R,
                   double *dR) {
  double N[17], dN[17];
  const int k = int(p + e);
  basis_on_span(U, p, k, x, N, dN);
  double W = 0.0, dW = 0.0;
  for (int r = 0; r <= p; ++r) {
    W += w[e + r] * N[r];
    dW += w[e + r] * dN[r];
  }
  for (int r = 0; r <= p; ++r) {
    R[r] = w[e + r] * N[r] / W;
    if (dR) dR[r] = w[e + r] * (dN[r] * W - N[r] * dW) / (W * W);
  }
}

void annulus_band_tables(int p, int64_t m, std::vector<double> &K, std::vector<double> &M) {
  const std::vector<double> U = knot_vector(p, m), w = nurbs_weights(p, m);
  const int64_t nf = m + p, n1 = nf - 2;
  const int W = 2 * p + 1;
  const double dr = kRout - kRin;
  // full tables, per axis: a = 0 (ξ, NURBS): K = ∫ R'R'/s, M = ∫ R R s; a = 1 (η): K = ∫ N'N' ρ/ρ', M = ∫ N N ρ'/ρ
  std::vector<double> Kf(2 * nf * W, 0.0), Mf(2 * nf * W, 0.0), gx, gw;
  gauss_legendre(p + 3, gx, gw);
  double R[17], dR[17], N[17], dN[17];
  for (int64_t e = 0; e < m; ++e) {
    const int k = int(p + e);
    const double a = U[k], b = U[k + 1], mid = 0.5 * (a + b), half = 0.5 * (b - a);
    for (size_t g = 0; g < gx.size(); ++g) {
      const double x = mid + half * gx[g], wq = half * gw[g];
      nurbs_on_span(U, w, p, e, x, R, dR);
      basis_on_span(U, p, k, x, N, dN);
      const double s = arc_speed(x), rho = kRin + dr * x;
      for (int r1 = 0; r1 <= p; ++r1)
        for (int r2 = 0; r2 <= p; ++r2) {
          const int64_t o = (e + r1) * W + (r2 - r1) + p;
          Kf[o] += wq / s * dR[r1] * dR[r2];
          Mf[o] += wq * s * R[r1] * R[r2];
          Kf[nf * W + o] += wq * rho / dr * dN[r1] * dN[r2];
          Mf[nf * W + o] += wq * dr / rho * N[r1] * N[r2];
        }
    }
  }
  K.assign(2 * n1 * W, 0.0);
  M.assign(2 * n1 * W, 0.0);
  for (int ax = 0; ax < 2; ++ax)
    for (int64_t i = 0; i < n1; ++i)
      for (int t = -p; t <= p; ++t) {
        if (i + t < 0 || i + t >= n1) continue;
        K[(ax * n1 + i) * W + t + p] = Kf[(ax * nf + i + 1) * W + t + p];
        M[(ax * n1 + i) * W + t + p] = Mf[(ax * nf + i + 1) * W + t + p];
      }
}

BandOp annulus_degree_restriction(int axis, int p, int q, int64_t m) {
  // One axis of R = D^{-1} C (P:217-220 with the map's mass): C = ∫ φ^q φ^p |det J|, D_ii = ∫ φ^q_i |det J|
  // (row-sum lumping of the unconstrained q-mass: partition of unity, reading A6); |det J| = s(ξ) · ρρ'(η).
  // Rules as the oracle: p+3 points for C, q+3 for D.
  const std::vector<double> Up = knot_vector(p, m), Uq = knot_vector(q, m);
  const std::vector<double> wp = nurbs_weights(p, m), wq_ = nurbs_weights(q, m);
  const int64_t nfq = m + q, n1q = nfq - 2, n1p = m + p - 2;
  const int W = p + q + 1;
  const double dr = kRout - kRin;
  auto basis = [&](const std::vector<double> &U, const std::vector<double> &w, int deg, int64_t e, double x, double *B) {
    if (axis == 0) nurbs_on_span(U, w, deg, e, x, B, nullptr);
    else basis_on_span(U, deg, int(deg + e), x, B, nullptr);
  };
  auto weight = [&](double x) { return axis == 0 ? arc_speed(x) : (kRin + dr * x) * dr; };
  std::vector<double> Cf(nfq * W, 0.0), D(nfq, 0.0), gx, gw;
  double Bp[17], Bq[17];
  gauss_legendre(p + 3, gx, gw);
  for (int64_t e = 0; e < m; ++e) {
    const double a = Up[p + e], b = Up[p + e + 1], mid = 0.5 * (a + b), half = 0.5 * (b - a);
    for (size_t g = 0; g < gx.size(); ++g) {
      const double x = mid + half * gx[g], wt = half * gw[g] * weight(x);
      basis(Up, wp, p, e, x, Bp);
      basis(Uq, wq_, q, e, x, Bq);
      for (int rq = 0; rq <= q; ++rq)
        for (int rp = 0; rp <= p; ++rp) Cf[(e + rq) * W + (rp - rq + q)] += wt * Bq[rq] * Bp[rp];
    }
  }
  gauss_legendre(q + 3, gx, gw);
  for (int64_t e = 0; e < m; ++e) {
    const double a = Uq[q + e], b = Uq[q + e + 1], mid = 0.5 * (a + b), half = 0.5 * (b - a);
    for (size_t g = 0; g < gx.size(); ++g) {
      const double x = mid + half * gx[g], wt = half * gw[g] * weight(x);
      basis(Uq, wq_, q, e, x, Bq);
      for (int rq = 0; rq <= q; ++rq) D[e + rq] += wt * Bq[rq];
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
    R.lo[ic] = int(ic - q);
    for (int k = 0; k < W; ++k) {
      const int64_t jc = ic - q + k;
      if (jc < 0 || jc >= n1p) continue;
      R.c[ic * W + k] = Cf[fi * W + k] / D[fi];
    }
  }
  return R;
}

BandOp annulus_embedding(int axis, int q, int64_t mc) {
  // Exact embedding of the degree-q space on mc spans into the one on 2 mc spans (reading A8).  η: plain
  // B-splines (knot insertion T).  ξ: NURBS with the same W, Σ a_c w^c_c N^c_c / W = Σ a'_f w^f_f N^f_f / W,
  // so a'_f = Σ_c T_fc (w^c_c / w^f_f) a_c (indices of the full bases: constrained + 1).
  BandOp P = mesh_prolongation(q, mc);
  if (axis == 0) {
    const std::vector<double> wc = nurbs_weights(q, mc), wf = nurbs_weights(q, 2 * mc);
    for (int r = 0; r < P.rows; ++r)
      for (int k = 0; k < P.W; ++k) {
        const int col = P.lo[r] + k;
        if (col >= 0 && col < P.cols) P.c[(size_t)r * P.W + k] *= wc[col + 1] / wf[r + 1];
      }
  }
  return P;
}

std::vector<double> annulus_load(int p, int64_t m) {
  // b_ik = ∫_Ω f φ_ik dx: f = -Δu for u = sin(πx) sin(πy)(t - r²)(t - R²), t = x² + y²;
  // (p+3)² Gauss points per element, |det J| = s ρ ρ'.
  const std::vector<double> U = knot_vector(p, m), w = nurbs_weights(p, m);
  const int64_t n1 = m + p - 2;
  const double dr = kRout - kRin, pi = 3.14159265358979323846, r2 = kRin * kRin, R2 = kRout * kRout;
  auto f = [&](double x, double y) {
    const double t = x * x + y * y, s = std::sin(pi * x) * std::sin(pi * y);
    const double g = (t - r2) * (t - R2), g1 = 2 * t - r2 - R2;
    const double sx = pi * std::cos(pi * x) * std::sin(pi * y), sy = pi * std::sin(pi * x) * std::cos(pi * y);
    // Δ(s g) = g Δs + 2 ∇s·∇g + s Δg,  Δs = -2π² s,  ∇g = g'(t) (2x, 2y),  Δg = 8t + 4 g'(t)
    return -(-2 * pi * pi * s * g + 4 * g1 * (x * sx + y * sy) + s * (8 * t + 4 * g1));
  };
  std::vector<double> gx, gw;
  gauss_legendre(p + 3, gx, gw);
  const int ng = int(gx.size());
  std::vector<double> b(n1 * n1, 0.0);
  std::vector<double> Rx(ng * (p + 1)), Ny(ng * (p + 1)), xs(ng), wxs(ng), ys(ng), wys(ng);
  double tmp[17];
  for (int64_t ey = 0; ey < m; ++ey) {
    const double ay = U[p + ey], by = U[p + ey + 1], my = 0.5 * (ay + by), hy = 0.5 * (by - ay);
    for (int g = 0; g < ng; ++g) {
      ys[g] = my + hy * gx[g];
      wys[g] = hy * gw[g] * (kRin + dr * ys[g]) * dr;
      basis_on_span(U, p, int(p + ey), ys[g], tmp, nullptr);
      for (int r = 0; r <= p; ++r) Ny[g * (p + 1) + r] = tmp[r];
    }
    for (int64_t ex = 0; ex < m; ++ex) {
      const double ax = U[p + ex], bx = U[p + ex + 1], mx = 0.5 * (ax + bx), hx = 0.5 * (bx - ax);
      for (int g = 0; g < ng; ++g) {
        xs[g] = mx + hx * gx[g];
        wxs[g] = hx * gw[g] * arc_speed(xs[g]);
        nurbs_on_span(U, w, p, ex, xs[g], tmp, nullptr);
        for (int r = 0; r <= p; ++r) Rx[g * (p + 1) + r] = tmp[r];
      }
      for (int gy = 0; gy < ng; ++gy)
        for (int gxi = 0; gxi < ng; ++gxi) {
          double c[2], dc[2];
          arc(xs[gxi], c, dc);
          const double rho = kRin + dr * ys[gy];
          const double v = wxs[gxi] * wys[gy] * f(rho * c[0], rho * c[1]);
          for (int jy = 0; jy <= p; ++jy) {
            const int64_t iy = ey + jy - 1;
            if (iy < 0 || iy >= n1) continue;
            const double vy = v * Ny[gy * (p + 1) + jy];
            for (int jx = 0; jx <= p; ++jx) {
              const int64_t ix = ex + jx - 1;
              if (ix < 0 || ix >= n1) continue;
              b[iy * n1 + ix] += vy * Rx[gxi * (p + 1) + jx];
            }
          }
        }
    }
  }
  return b;
}

}  // namespace iga2l
