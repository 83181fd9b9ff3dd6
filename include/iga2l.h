/*
 * iga2l — B200-native two-level solver for maximally smooth B-spline (IGA) Galerkin
 * discretizations of the Poisson problem on the unit square / cube.
 *
 * This header is the C-ABI boundary of libiga2l.so.  It follows the paper's problem statement
 * (arXiv 2009.01499, /root/reference/PAPER.md, cited P:<line>):
 *   -Δu = f in Ω = (0,1)^d, u = 0 on ∂Ω; Galerkin system A_p u_p = b_p with
 *   A_p = (a(φ_j, φ_i)), b_p = ((f, φ_i)); φ = tensor-product B-splines of degree p with
 *   maximal smoothness C^{p-1} on a uniform open knot vector with m spans per axis, Dirichlet
 *   functions removed: n1 = m + p - 2 unknowns per axis.
 * and it runs the paper's Algorithm 1: one overlapping multiplicative Schwarz sweep,
 * defect, L2-projection restriction to degree q (lumped mass), second-level solve
 * (exact, or one V(1,1) h-multigrid cycle; optionally on H = 2h),
 * prolongation.  Readings of the paper where it is silent are listed in DESIGN.md (A1..A26).
 *
 * Data layout of every vector (x, b, y): N = n1^d fp64 values, x-fastest:
 *     index(i_0, i_1[, i_2]) = i_0 + n1 * (i_1 + n1 * i_2),   0 <= i_a < n1,
 * constrained index i_a is the paper's basis function N_{i_a + 2}.
 *
 * Pointers.  Every vector argument may be a DEVICE pointer (cudaMalloc / PyTorch CUDA tensor on
 * the context's device) or a HOST pointer (pageable or pinned).  Device pointers are used in place,
 * stream-ordered on the context stream.  Host pointers are staged through context-owned device
 * buffers (H2D before, D2H after for outputs) and the call returns after the D2H copy completed.
 * The caller owns all vectors; the library never retains a caller pointer after a call returns.
 * Device-pointer calls are asynchronous w.r.t. the host unless stated otherwise.
 *
 * Errors.  Every int-returning function returns an iga2l_status.  On a non-OK return
 * iga2l_last_error() gives a thread-local one-line message naming the offending field / call.
 * Calls never abort the process.  A context serves one stream at a time (not thread-safe).
 */
#ifndef IGA2L_H
#define IGA2L_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct iga2l_ctx iga2l_ctx;

typedef enum {
  IGA2L_OK = 0,
  IGA2L_EPARAM = 1,    /* invalid argument; message names the field                         */
  IGA2L_ENUMERIC = 2,  /* NaN/Inf residual, or a non-SPD local/coarse matrix during setup   */
  IGA2L_NOTCONV = 3,   /* iga2l_solve hit maxit; outputs are valid (non-fatal)  */
  IGA2L_ECUDA = 4,     /* CUDA runtime error (no device, launch failure, ...)               */
  IGA2L_ENCCL = 5,     /* NCCL error (multi-GPU)                                            */
  IGA2L_ENOMEM = 6     /* device or host allocation failed                                  */
} iga2l_status;

typedef enum {
  IGA2L_COARSE_EXACT = 0,  /* A_q e = d_q solved exactly: dense inverse (Nc <= 1024) or, above,  */
                           /* Kronecker fast diagonalisation (⊗V)(Σλ)^{-1}(⊗V)^T, n <= 2048/axis */
                           /* (IGA2L_COARSE_FD=0/1 forces dense (Nc <= 4096) / FD)              */
  IGA2L_COARSE_VCYCLE = 1  /* one V(1,1) h-multigrid cycle, zero initial guess     */
} iga2l_coarse_mode;

typedef enum {
  IGA2L_GEOM_SQUARE = 0,            /* Ω = (0,1)^d, B-splines (the benchmark workloads)      */
  IGA2L_GEOM_QUARTER_ANNULUS = 1    /* Ω = {0.3² <= x²+y² <= 0.5², x,y >= 0}: F = ρ(η)c(ξ), */
                                    /*   NURBS in ξ (exact arc), B-splines in η.  2D only,  */
                                    /*   q = 2, p >= 2, nranks 1.  Orthogonal map, so          */
                                    /*   A = My ⊗ Kx + Ky ⊗ Mx with weighted 1D tables per axis       */
} iga2l_geometry;

typedef struct {
  int coarse_mode;       /* iga2l_coarse_mode; default VCYCLE                                    */
  int coarse_h_factor;   /* 1: q-level on the same mesh h (Algorithm 1); 2: aggressive   */
                         /*    H = 2h.  Default 2.                                       */
  int vcycle_coarsest_m; /* V-cycle coarsens while m > this (must be >= 1); default 8    */
  void *stream;          /* cudaStream_t for all work; NULL = the context creates its own       */
                         /*    blocking stream (ordered w.r.t. the legacy default stream)      */
  int use_graph;         /* 1 (default): iterations are replayed from a captured CUDA graph      */
  int nranks, rank;      /* slab partition along the last axis:                  */
                         /*   nranks == 1: one domain (rank 0);                                 */
                         /*   nranks  > 1, rank in [0, nranks): this process owns slab `rank`;  */
                         /*     vectors are its owned planes [z0, z1) (iga2l_sizes); halos and  */
                         /*     reductions over NCCL (nccl_id required);                         */
                         /*   nranks  > 1, rank == -1: all slabs in this process on this device */
                         /*     (global vectors; halo exchange by device copies; nccl_id NULL)   */
  const void *nccl_id;   /* 128-byte ncclUniqueId from iga2l_nccl_unique_id() on one rank,       */
                         /*   broadcast by the caller (NULL unless rank >= 0 and nranks > 1)     */
  int geometry;          /* iga2l_geometry; default SQUARE                                        */
} iga2l_opts;

/* Fill *o with the defaults above. */
void iga2l_default_opts(iga2l_opts *o);

/*
 * Build a context (host setup + upload), P:90-113 and P:186-220:
 *   dim     2 or 3 (the paper is 2D; 3D is the tensor generalisation, reading A25)
 *   p       fine degree, 1..8
 *   q       second-level degree, 1 <= q <= min(p, 2) ("linear/quadratic")
 *   n       m = number of uniform spans per axis (h = 1/m), n >= 1, n1 = n + p - 2 >= 1
 *   block   Schwarz block side s in {1,3,5,7} (s^d unknowns per block; paper: 3 for p<=4,
 *           5 for p=5,6, 7 for p=7,8), s <= n1
 *   overlap must be s - 1 (maximal overlap: one block per grid point)
 * Aggressive coarsening / V-cycle need m divisible by 2 as required; violations -> EPARAM.
 * On success *out owns all device memory it allocated; free with iga2l_destroy.
 */
int iga2l_setup(int dim, int p, int q, int64_t n, int block, int overlap, iga2l_ctx **out);
int iga2l_setup_ex(int dim, int p, int q, int64_t n, int block, int overlap,
                   const iga2l_opts *opts, iga2l_ctx **out);

/* Sizes: n_local = N (unknowns held by this rank), slab [z0, z1) along the last axis, n1. */
int iga2l_sizes(const iga2l_ctx *ctx, int64_t *n_local, int64_t *z0, int64_t *z1, int64_t *n1);

/* b_i = (f, φ_i) for f = d π² ∏ sin(π x_a) (exact solution u = ∏ sin(π x_a); P:397-405 for d=2),
 * Gauss quadrature with p+3 points per span (reading A17).  b: N fp64 (output). */
int iga2l_rhs_sine(iga2l_ctx *ctx, double *b);
/* The paper's right-hand side for the context's geometry: square -> iga2l_rhs_sine; quarter annulus ->
 * b_ik = (f, φ_ik), f = -Δu for u = sin(πx) sin(πy)(x²+y²-r²)(x²+y²-R²), (p+3)² Gauss points
 * per element (host quadrature, then copied).  b: N fp64, host or device. */
int iga2l_rhs(iga2l_ctx *ctx, double *b);

/* y = A_p x, matrix-free ((2p+1)^d-point operator).  x, y: N fp64, must not alias. */
int iga2l_apply(iga2l_ctx *ctx, const double *x, double *y);

/* *out = ||b - A_p x||_2 (reading A15).  Synchronises the context stream. */
int iga2l_residual_norm(iga2l_ctx *ctx, const double *b, const double *x, double *out);

/*
 * `iters` two-level iterations of Algorithm 1 (ν1 = 1, ν2 = 0; reading A14) on x in place.
 * Schwarz order: multicolour, colour(c) = Σ_a (c_a mod D) D^a, D = s + p, ascending (reading A4).
 * res_hist: NULL, or a HOST array of iters+1 doubles receiving ||b - A x_k||_2 for k = 0..iters
 * (then the call synchronises).  iters >= 0.
 */
int iga2l_iterate(iga2l_ctx *ctx, const double *b, double *x, int iters, double *res_hist);

/*
 * Torus LFA run: the spectral radius of the two-grid error operator
 * E = (I - P A_q^+ R A_p) S_p of the multicolour method (reading A4) on the n^dim (dim 2 or 3)
 * PERIODIC grid, by `iters` power iterations with the library's kernels from a seeded mean-zero start
 * (the constant, E 1 = 1, projected out: LFA excludes it).  h_factor 1: exact degree-q level on the
 * same mesh (Table 1's ρ_2g); 2: aggressive, degree q on H = 2h (Table 3's ρ_2g^ag); 3: three-grid, the
 * degree-q level by one two-grid cycle ((q+1)^2-colour GS, exact 2h solve; Table 2's ρ_3g; 2D).  With n = nk (s + p),
 * nk even, the torus frequencies are the Bloch quasi-momenta of an nk^2 LFA grid.  Synchronous; allocates
 * and frees its own device memory on the current device.
 * rho (host): geometric mean of the last quarter of the norm ratios; ratios (host, NULL or `iters`
 * doubles): every ratio.  Errors: IGA2L_EPARAM (dim not 2/3, n not a multiple of s + p or < 2(s + p), n /
 * h_factor < 2q + 1, iters outside 4..100000, ...), IGA2L_ENUMERIC, IGA2L_ECUDA, IGA2L_ENOMEM.
 */
int iga2l_lfa_torus(int dim, int p, int q, int n, int block, int h_factor, int iters, unsigned long long seed,
                    double *rho, double *ratios);

/*
 * Iterate until ||b - A x_k|| <= rtol ||b - A x_0|| or maxit iterations.
 * iters_out / relres_out (host, may be NULL) receive the count and ||r_k||/||r_0||.
 * Returns IGA2L_NOTCONV (outputs valid) if maxit was reached, IGA2L_ENUMERIC on NaN/Inf.
 */
int iga2l_solve(iga2l_ctx *ctx, const double *b, double *x, double rtol, int maxit,
                int *iters_out, double *relres_out);

/* ---- single phases of Algorithm 1 (same layouts; used by parity tests and the bench) ---- */

/* Schwarz colours [colour_begin, colour_end) of the multicolour sweep on x in place
 * (0 <= begin <= end <= D^d).  One full sweep = [0, D^d). */
int iga2l_sweep(iga2l_ctx *ctx, const double *b, double *x, int colour_begin, int colour_end);

/* dq = I_p^q (b - A_p x): defect + restriction.  dq: Nc = n1c^d fp64. */
int iga2l_defect_restrict(iga2l_ctx *ctx, const double *b, const double *x, double *dq);

/* e = second-level solve of A_q e = dq (exact or one V(1,1), per opts).  dq, e: Nc fp64. */
int iga2l_coarse_solve(iga2l_ctx *ctx, const double *dq, double *e);

/* x += I_q^p e (prolongation = adjoint of the restriction). */
int iga2l_prolong_add(iga2l_ctx *ctx, const double *e, double *x);

/* ---- introspection ---- */
typedef struct {
  int64_t n1, N, n1c, Nc;       /* fine / second-level sizes                                    */
  int colours;                  /* D^d                                                          */
  int levels;                   /* second-level V-cycle depth (1 = direct)                      */
  int launches_per_iter;        /* kernel launches in one iteration (graph nodes of ours)      */
  double sweep_flops;           /* algorithmic FP64 flops of one sweep           */
  double iter_hbm_bytes;        /* algorithmic HBM bytes of one iteration outside the sweep    */
  int vc_smem_level;            /* first second-level level run by the shared-memory cluster   */
                                /*   V-cycle kernel (-1: none)                                  */
  int vc_smem_cs;               /* its cluster size (CTAs); 0 if none                           */
} iga2l_info;
int iga2l_get_info(const iga2l_ctx *ctx, iga2l_info *out);

/* Host-only helper (no GPU needed): the 1D constrained band tables of degree p on m spans as
 * used by the device path: K[i*(2p+1) + t+p] = ∫ N_{i+2}' N_{i+2+t}', M likewise (0 outside).
 * K, M: host arrays of (m+p-2)*(2p+1) doubles. */
int iga2l_host_band_tables(int p, int64_t m, double *K, double *M);

/* 128-byte NCCL unique id (call on one rank, broadcast to all, pass as opts.nccl_id). */
int iga2l_nccl_unique_id(void *out128);

/* Host-only helper: the slab plan of `rank` among `nranks` for the last axis of n1 = m+p-2 points:
 * out8 = {z0, z1 (owned planes), za, zb (stored planes incl. halo), first / end block centre handled,
 *         halo H = block-1+p, feasible (z1-z0 >= H)}. */
int iga2l_host_slab_plan(int dim, int p, int block, int64_t m, int nranks, int rank, int64_t *out8);

/* Host-only helper: 1D transfer operator used for the restriction, as a dense row-major
 * (n1c x n1) host matrix (h_factor 1: D^{-1} M_c; 2: P_mesh^T D^{-1} M_c). */
int iga2l_host_restriction_1d(int p, int q, int64_t m, int h_factor, double *R);

/* Host-only helper: the exact second-level solve's 1D generalised eigen-decomposition for degree q on
 * m spans (n = m+q-2): K V = M V diag(lam), V^T M V = I.  V: host n*n doubles, row-major (row = 1D
 * index, column = eigen index); lam: host n doubles.  Then A_q^{-1} = (⊗V) (Σ_a lam)^{-1} (⊗V)^T
 * (SURVEY §8(f) row 1).  ENUMERIC if M or K is not SPD. */
int iga2l_host_coarse_fd(int q, int64_t m, double *V, double *lam);

/* The same for the degree-q level on the n-point TORUS (the torus LFA run's exact second level, 1 <= q <= 2,
 * 2q+1 <= n <= 4096): circulant K, M from the interior band rows; the constant's eigenvalue is exactly 0
 * (the run applies the pseudo-inverse).  V: host n*n, lam: host n.  ENUMERIC unless exactly one λ vanishes. */
int iga2l_host_periodic_fd(int q, int n, double *V, double *lam);

/* Host-only helpers of the quarter annulus (no GPU needed):
 *  tables: per-axis constrained band tables, K and M each [2][n1][2p+1] (axis 0 = ξ: ∫R'R'/s, ∫R R s;
 *          axis 1 = η: ∫N'N' ρ/ρ', ∫N N ρ'/ρ), so that A = My ⊗ Kx + Ky ⊗ Mx;
 *  restriction_1d: one axis of the restriction (lumped L2 on the map, composed with the exact NURBS /
 *          B-spline embedding for h_factor 2), dense row-major (n1c x n1), q = 2;
 *  load: the load vector of iga2l_rhs, n1*n1 (x = ξ fastest). */
int iga2l_host_annulus_tables(int p, int64_t m, double *K, double *M);
int iga2l_host_annulus_restriction_1d(int axis, int p, int q, int64_t m, int h_factor, double *R);
int iga2l_host_annulus_load(int p, int64_t m, double *b);

int iga2l_destroy(iga2l_ctx *ctx);
const char *iga2l_last_error(void);
const char *iga2l_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IGA2L_H */
