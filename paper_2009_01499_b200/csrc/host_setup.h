// Host-side setup (layer L0): everything computed once per context on the CPU and uploaded.
// Independent of oracle/ (shares no code); cites the paper (P:<line>) for every formula.
#pragma once
#include <cstdint>
#include <vector>

namespace iga2l {

// Banded 1D operator: row r holds W coefficients for columns lo[r] .. lo[r]+W-1 (zeros padded,
// columns outside [0, cols) carry a zero coefficient).
struct BandOp {
  int rows = 0, cols = 0, W = 0;
  std::vector<int> lo;
  std::vector<double> c;  // rows * W
  double at(int r, int col) const {
    int k = col - lo[r];
    return (k >= 0 && k < W) ? c[(size_t)r * W + k] : 0.0;
  }
};

// Open uniform knot vector Ξ_{p,h}, 0-based array of 2p+m+1 knots.
std::vector<double> knot_vector(int p, int64_t m);

// n-point Gauss–Legendre nodes/weights on [-1, 1] (Newton on the Legendre recurrence).
void gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w);

// Values N[0..p] and derivatives dN[0..p] of the p+1 B-splines that are non-zero on span
// [U[k], U[k+1]) (full 0-based indices k-p .. k), at x (triangular Cox–de Boor scheme).
void basis_on_span(const std::vector<double> &U, int p, int k, double x, double *N, double *dN);

// Constrained 1D band tables (P:83 in 1D): K[i*(2p+1) + t+p] = ∫ N'_{i+2} N'_{i+2+t},
// M[...] = ∫ N_{i+2} N_{i+2+t}, i in [0, n1), zero where i+t is outside [0, n1).
void band_tables(int p, int64_t m, std::vector<double> &K, std::vector<double> &M);
// constrained rows [lo, hi] whose band rows are translation invariant (bitwise equal after band_tables)
void toeplitz_rows(int p, int64_t m, int64_t *lo, int64_t *hi);

// g_i = ∫ sin(π x) N_{i+2}(x) dx, p+3 Gauss points per span (reading A17); n1 values.
std::vector<double> load_1d_sine(int p, int64_t m);

// Degree restriction R1 = D^{-1} M_c on the same mesh, D_ii = ∫ φ_i^q (row-sum
// lumping, reading A6) = (ξ_{i+q+1} - ξ_i)/(q+1).  Rows: constrained q-functions; cols: p.
BandOp degree_restriction(int p, int q, int64_t m);

// Exact embedding S^q_{2h} ⊂ S^q_h by knot insertion (Boehm) at every coarse span midpoint
// (reading A8).  Constrained: rows = fine (2 mc + q - 2), cols = coarse (mc + q - 2).
BandOp mesh_prolongation(int q, int64_t mc);

BandOp transpose(const BandOp &A);
BandOp multiply(const BandOp &A, const BandOp &B);  // A (r x k) * B (k x c), banded result

// Fast-diagonalisation tables for the Schwarz block of every centre c along one axis
// (A_B = K_I ⊗ M_I + M_I ⊗ K_I is a Kronecker sum on the clipped window I = [c-w, c+w] ∩ [0,n1)):
// K_I V = M_I V Λ, V^T M_I V = I.  V[(c*s + l)*s + j]: local row l (global c-w+l; zero if outside I),
// eigen-column j (zero if j >= |I|); lam[c*s + j] (1.0 padding).  Returns false if not SPD.
bool fd_tables(int p, int s, int64_t n1, const std::vector<double> &K, const std::vector<double> &M,
               std::vector<double> &V, std::vector<double> &lam);

// Fast diagonalisation of the degree-q level on m spans (exact coarse solve at any size, SURVEY
// §8(f) row 1): K V = M V Λ, V^T M V = I; V row-major n x n (row = 1D index, column = eigen index).
bool coarse_fd_tables(int q, int64_t m, std::vector<double> &V, std::vector<double> &lam);
// The same from given band tables (bandwidth 2q+1, n rows): K V = M V Λ, V^T M V = I.
bool band_fd_tables(int q, int n, const double *K, const double *M, std::vector<double> &V, std::vector<double> &lam);

// The same on the n-point TORUS (circulant K, M from one interior band row each, bandwidth 2q+1): the one
// vanishing eigenvalue (constants) is returned as exactly 0.  False unless M is SPD and exactly one λ vanishes.
bool periodic_fd_tables(int q, int n, const double *krow, const double *mrow, std::vector<double> &V,
                        std::vector<double> &lam);

// Dense inverse of the d-dim operator Σ_a ⊗ (K on axis a, M elsewhere) from band tables of
// degree q (bandwidth 2q+1) on n points per axis.  Returns false if not SPD.  Row-major N x N.
// ays > 0: per-axis tables, axis a's rows at K[a * ays ...] (the quarter annulus, A = My ⊗ Kx + Ky ⊗ Mx).
bool dense_kron_inverse(int dim, int q, int n, const std::vector<double> &K, const std::vector<double> &M,
                        std::vector<double> &inv, int64_t ays = 0);

// ---- quarter annulus (geometry.cpp) ----
// Coefficients w of the arc's weight function W(ξ) in the degree-p (p >= 2) basis on m spans (nf = m+p).
std::vector<double> nurbs_weights(int p, int64_t m);
// NURBS R_r = w_{e+r} N_{e+r} / W and dR_r/dξ (r = 0..p) on span e at x.
void nurbs_on_span(const std::vector<double> &U, const std::vector<double> &w, int p, int64_t e, double x, double *R,
                   double *dR);
// Per-axis constrained band tables [2][n1][2p+1]: axis 0 (ξ): Kx = ∫R'R'/s, Mx = ∫R R s; axis 1 (η):
// Ky = ∫N'N'ρ/ρ', My = ∫N N ρ'/ρ, so that A = My ⊗ Kx + Ky ⊗ Mx (x = ξ fastest).
void annulus_band_tables(int p, int64_t m, std::vector<double> &K, std::vector<double> &M);
// One axis (0: ξ, 1: η) of the lumped L2 degree restriction on the map (weights s and ρρ').
BandOp annulus_degree_restriction(int axis, int p, int q, int64_t m);
// One axis of the exact embedding of the degree-q space on mc spans into the one on 2 mc spans.
BandOp annulus_embedding(int axis, int q, int64_t mc);
// Load vector (f, φ_ik) of the manufactured solution, n1*n1 (x = ξ fastest).
std::vector<double> annulus_load(int p, int64_t m);

}  // namespace iga2l
