// Device kernels of libiga2l (layer L1), sm_100a.  All arithmetic is IEEE fp64.
// Sources: apply.cu (operator, norms), schwarz2d.cu (2D DMMA colour kernel, generic fallback, dispatch),
// schwarz3d.cu (3D colour kernel), transfer.cu (band transfers), vcycle.cu (second level),
// coarse_fd.cu (exact second level by fast diagonalisation).
//
// Operator: the degree-p stiffness on the tensor basis is
//     A = Σ_a ⊗_b X_b,  X_b = K (1D stiffness) if b == a else M (1D mass),
// applied matrix-free from per-row 1D band tables K[i*(2p+1) + t+p] (row i, column i+t; zero
// outside the domain), by sum factorisation: one 1D pass per axis over a tile staged in shared
// memory (2D: 4(2p+1) FMAs/DOF; 3D: 7(2p+1) FMAs/DOF).
#pragma once
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

namespace iga2l {

struct Band1D {          // banded 1D transfer: row r uses columns lo[r] .. lo[r]+W-1
  int rows, cols, W;
  const int *lo;
  const double *c;
  int lo_max_span;       // max over 32-row tiles of lo[last] - lo[first] (0: unknown)
  int lo_max_span16;     // the same over 16-row tiles
};

// Window of the LAST axis (y in 2D, z in 3D) of a vector held by a context: local plane 0 is the
// global plane zoff; kernels compute/output the global planes [zlo, zhi).  {0, 0, -1} = whole grid.
struct SlabView {
  int zoff, zlo, zhi;
};
constexpr SlabView kFull{0, 0, -1};
void centre_range(int c, int D, int lo, int hi, int *first, int *count);

// Interior (translation-invariant) 1D data of the fine level (reading A27), passed BY VALUE as a
// kernel parameter: with compile-time indices the FMAs read it as constant-bank operands.
constexpr int kToeMaxW = 17, kToeMaxS = 7;
struct ToeP {
  double k[kToeMaxW], m[kToeMaxW];           // interior band row of K and M (t = 0 .. 2p)
  double v[kToeMaxS * kToeMaxS], lam[kToeMaxS];   // FD tables of an interior block (V[l][j], λ_j)
  int valid;                                 // 0: no interior rows (small grids)
};

// ---- fine operator: apply / residual -------------------------------------------------------
// mode 0: y = A x;  mode 1: y = b - A x.  If partial != nullptr, partial[cta] = Σ y^2 over the tile.
// ys: offset (doubles) of the y-axis tables from the x-axis ones (2D; 0 = the same tables; the quarter
// annulus stores [2][n1][2p+1] per-axis tables, A = My ⊗ Kx + Ky ⊗ Mx, and passes ys = n1 (2p+1)).
void launch_apply(int dim, int p, int64_t n1, const double *K, const double *M, const double *x,
                  const double *b, double *y, double *partial, int mode, cudaStream_t st, int *nparts,
                  SlabView sv = kFull, const ToeP *tp = nullptr, int64_t ys = 0);
int apply_num_partials(int dim, int p, int64_t n1);
// The TMA streaming apply (stream.cu), used by launch_apply for 1 <= p <= 8 unless IGA2L_APPLY_STREAM=0.
// count_only: only report *nparts.  False if not launched (p unsupported, tensor map encode failed).
bool launch_apply_stream(int dim, int p, int64_t n1, const double *K, const double *M, const double *x, const double *b,
                         double *y, double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv,
                         const ToeP *tp, bool count_only);

// ---- multicolour Schwarz: one colour ---------------------------------------------------------
// Blocks centred at c = col + D*j (per axis) are solved in parallel (A-decoupled, reading A4):
// r_B = b_B - (A x)_B; δ = A_B^{-1} r_B by fast diagonalisation with per-centre 1D tables V, lam;
// x_B += δ.
// (slab: blocks with last-axis centre in [sv.zlo, sv.zhi); x, b stored from plane sv.zoff)
void launch_schwarz_colour(int dim, int p, int s, int64_t n1, const double *K, const double *M,
                           const double *V, const double *lam, const double *b, double *x,
                           int colour, int D, cudaStream_t st, SlabView sv = kFull, int ax = 0);

// ---- tensor-product band transform along one axis ------------------------------------------
// in: [outer][nin][inner]  ->  out: [outer][B.rows][inner],  out (+)= Σ_k B.c[r,k] in[.., lo[r]+k, ..]
// (optional: only input columns in [clo, chi) stored from coff; only output rows [rlo, rhi))
void launch_band_axis(const double *in, double *out, int64_t outer, int nin, int64_t inner,
                      const Band1D &B, int accumulate, cudaStream_t st, int clo = 0, int chi = -1,
                      int coff = 0, int rlo = 0, int rhi = -1);

// ---- q-level (V-cycle) kernels, direct (2q+1)^d stencil --------------------------------------
// ays: offset of axis a's band tables = a * ays (0: shared tables; per-axis for the quarter annulus).
void launch_q_gs_colour(int dim, int q, int n, const double *K, const double *M, const double *b,
                        double *x, int colour, cudaStream_t st, int64_t ays = 0);
void launch_q_residual(int dim, int q, int n, const double *K, const double *M, const double *b,
                       const double *x, double *r, cudaStream_t st, int64_t ays = 0);

// x = Ainv b (dense, N <= 4096), one warp per row.
void launch_dense_mv(int N, const double *Ainv, const double *b, double *x, cudaStream_t st);

// out[0] = Σ partial[0..n) (deterministic, single CTA); if hist/count given and *count < cap,
// also hist[*count] = sqrt(out[0]), ++*count.
void launch_sum_partials(const double *partial, int n, double *out, double *hist, int *count, int cap,
                         cudaStream_t st);

// ---- optimised paths ------------------------------------------------------------------------
// Colour `colour` by the specialised kernels (2D: DMMA warp-per-block for the paper's (p, s) pairs;
// 3D: pencil kernel for s = 3 (p <= 4), s = 5 (p = 5, 6)); false = not specialised (use the generic kernel).
// fb: interior-block DMMA operand fragments (export_interior_frags) or nullptr.
bool launch_schwarz_colour_fast(int dim, int p, int s, int64_t n1, const double *K, const double *M,
                                const double *V, const double *lam, const double *b, double *x, int colour,
                                int D, cudaStream_t st, SlabView sv = kFull, const double *fb = nullptr,
                                const ToeP *tp = nullptr, int ax = 0);
// ax = 1 (2D): per-axis tables -- K, M [2][n1][2p+1], V [2][n1][s*s], lam [2][n1][s], y after x
// (the quarter annulus, A = My ⊗ Kx + Ky ⊗ Mx); fb must be nullptr then.
bool launch_schwarz3d_colour(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                             const double *lam, const double *b, double *x, int c0, int c1, int f2, int D, int nb0,
                             int nb1, int nb2, int zoff, int tlo, int thi, cudaStream_t st, const ToeP *tp);
// Interior-block operand fragments of the 2D DMMA kernel (lane-major, A27) into out (device); with
// out == nullptr returns the number of doubles needed; -1 if no interior block or (p, s) not specialised.
int export_interior_frags(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                          const double *lam, double *out, cudaStream_t st);
// Operand fragments of every x-centre ([n1][NX][32]) then every y-centre ([n1][NY][32]) for k_schwarz2d_mmg,
// written to out (device) right after the interior fragments; out == nullptr: count only; -1 if not specialised.
int export_centre_frags(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                        const double *lam, double *out, cudaStream_t st);
// 2D tensor transfer out (+)= (By ⊗ B) in in one launch (in: B.cols^2, out: B.rows^2).
// (optional: input rows valid in [iylo, iyhi) stored from iyoff; output rows [rylo, ryhi) stored from ryoff)
// By: the y-axis band if it differs from the x-axis one (per-axis transfers of the quarter annulus).
void launch_tensor2d(const double *in, double *out, const Band1D &B, int accumulate, cudaStream_t st,
                     int iylo = 0, int iyhi = -1, int iyoff = 0, int rylo = 0, int ryhi = -1, int ryoff = 0,
                     const Band1D *By = nullptr);

// One q-level of the V-cycle hierarchy, as seen by the single-CTA tail kernel (device array).
struct QLevelDev {
  int n;
  int64_t N;
  const double *K, *M;
  double *x, *b, *r, *t1, *t2;
  Band1D P, PT;          // to the next coarser level (unused at the coarsest)
  const double *inv;     // dense inverse at the coarsest level
};
// Shared-memory V-cycle tail (levels [l0, nlev)), one thread-block cluster of cs CTAs:
//  * levels [l0, l0 + nsp) are SPREAD over the CTAs by rows of the last axis (CTA r owns rows
//    [z0[l][r], z0[l][r+1]) and keeps H halo rows each side, refreshed by the writing thread with
//    DSMEM stores to the neighbour); phases are separated by cluster barriers;
//  * levels [l0 + nsp, nlev) live in CTA 0's shared memory (phases: __syncthreads).
// Offsets are in doubles (ints for the transfer column starts, in the int area after the doubles).
constexpr int kVcMaxLev = 12, kVcMaxCS = 16, kVcMaxCopy = 64;
struct VcCopy {
  const void *src;
  int dst, count, is_int, pad;
};
struct VcLayout {
  const double *gb0;                   // level l0 right-hand side (global, written by the caller)
  double *gx0;                         // level l0 solution (global, read by the caller)
  const double *ginv;                  // coarsest dense inverse (global)
  int l0, nlev, nsp, cs, dim3, H;
  int n[kVcMaxLev], WP[kVcMaxLev], WPT[kVcMaxLev];
  int x[kVcMaxLev], b[kVcMaxLev], r[kVcMaxLev];
  int K[kVcMaxLev], M[kVcMaxLev], Pc[kVcMaxLev], PTc[kVcMaxLev], Plo[kVcMaxLev], PTlo[kVcMaxLev];
  short z0[kVcMaxLev][kVcMaxCS + 1];   // spread levels: row partition
  short rc0[kVcMaxCS + 1];             // restriction into the first CTA-0 level: coarse rows of CTA r
  short pc0[kVcMaxCS];                 // prolongation from it: coarse rows [pc0[r], pc0[r] + pcn) pulled
  int pcn, pbuf, cbuf, inv_sm, xend;   // pull buffers, staged coarsest inverse (-1: global), x area end
  int ncopy, copy_start[kVcMaxCopy + 1];
  VcCopy copy[kVcMaxCopy];
  int ndouble, nint;
};
// Build the layout for tail levels [l0, nlev) on a cluster of cs CTAs (cs = 1: CTA-0 levels only).
// tab: HOST copy of the level table (device pointers inside).  False if it does not fit / partition
// constraints fail.
bool vcycle_smem_layout(int dim, int q, const QLevelDev *tab, int nlev, int l0, int cs, size_t max_bytes,
                        VcLayout *out);
size_t vcycle_smem_bytes(const VcLayout &L);
bool vcycle_smem_probe(int dim, int q, const VcLayout &L);   // call outside stream capture
cudaError_t launch_vcycle_smem(int dim, int q, const VcLayout &L, cudaStream_t st);

// Strided batched FP64 GEMM on the tensor pipe: C[b](m,n) = Σ_k A[b](m,k) B[b](k,n).
void launch_dgemm(const double *A, const double *B, double *C, int M, int N, int K, int batch, int64_t sAb,
                  int64_t sAm, int64_t sAk, int64_t sBb, int64_t sBk, int64_t sBn, int64_t sCb, int64_t sCm,
                  int64_t sCn, cudaStream_t st);
// Exact second-level solve by Kronecker fast diagonalisation: e = (⊗V)(Σ_a λ)^{-1}(⊗V)^T d
// (V: n x n row-major, K V = M V Λ, V^T M V = I).  t1, t2: n^dim scratch.  Returns the launch count.
// ax = 1 (2D): per-axis decompositions, V [2][n][n], lam [2][n] (x then y; the quarter annulus).
int launch_coarse_fd(int dim, int n, const double *V, const double *lam, const double *d, double *e, double *t1,
                     double *t2, cudaStream_t st, int ax = 0);

// Torus LFA run (torus.cu): spectral radius of the 2D two-grid error operator on the n x n torus by power
// iteration with the hot-path kernels.  Returns an IGA2L code; *err set on failure.
int lfa_torus_run(int dim, int p, int q, int n, int s, int hf, int iters, unsigned long long seed, double *rho,
                  double *ratios, std::string *err);

// y += x (fixed-order sums of the slab partial coarse vectors in local multi-slab mode)
void launch_axpy(double *y, const double *x, int64_t n, cudaStream_t st);

// b[idx] = scale * ∏_a g[i_a]
void launch_tensor_rhs(int dim, int64_t n1, const double *g, double scale, double *b, cudaStream_t st);

}  // namespace iga2l
