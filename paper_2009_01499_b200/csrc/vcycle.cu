// Second level: the q-level V(1,1) cycle -- level-by-level kernels for the large
// levels and the shared-memory cluster kernel for the tail -- and the dense coarsest solve.
#include <cooperative_groups.h>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
namespace cg = cooperative_groups;

namespace iga2l {
namespace {

__global__ void k_dense_mv(int N, const double *__restrict__ A, const double *__restrict__ b, double *__restrict__ x) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= N) return;
  double s = 0.0;
  for (int j = lane; j < N; j += 32) s = fma(A[(int64_t)warp * N + j], b[j], s);
  s = warp_sum(s);
  if (lane == 0) x[warp] = s;
}

}  // namespace

void launch_dense_mv(int N, const double *Ainv, const double *b, double *x, cudaStream_t st) {
  const int warps_per_block = 8;
  k_dense_mv<<<(N + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(N, Ainv, b, x);
}

}  // namespace iga2l

// ============================================================================================
// V-cycle tail with its levels resident in SHARED memory of one thread-block cluster (v3).
// One V(1,1) with the arithmetic and order of the level-by-level kernels: (q+1)^d-colour
// Gauss-Seidel (A11), residual, P^T restriction (A8), dense coarsest solve (A12), P prolongation,
// zero initial guess (A13).  See VcLayout (kernels.cuh) for the data placement.
// ============================================================================================
namespace iga2l {
namespace {

template <int DIM>
struct XOff {               // level values in shared memory; last-axis row j stored at row j - zoff
  const double *x;
  int n, zoff;
  __device__ __forceinline__ double operator()(int jx, int jy, int jz) const {
    return DIM == 3 ? x[((jz - zoff) * n + jy) * n + jx] : x[(jy - zoff) * n + jx];
  }
};

// Σ_j a_ij x_j over the (2Q+1)^d stencil of point (ix, iy, iz) and a_ii.  ays: offset of axis a's
// tables = a * ays (0: one table pair for all axes; per-axis tables of the quarter annulus otherwise)
template <int DIM, int Q, class XA>
__device__ __forceinline__ double q_point_acc(int n, const double *sK, const double *sM, const XA &xa, int ix,
                                              int iy, int iz, double *diag, int64_t ays = 0) {
  constexpr int W = 2 * Q + 1;
  const unsigned un = unsigned(n);
  double kx[W], mx[W], ky[W], my[W];
#pragma unroll
  for (int t = 0; t < W; ++t) {
    kx[t] = sK[ix * W + t]; mx[t] = sM[ix * W + t];
    ky[t] = sK[ays + iy * W + t]; my[t] = sM[ays + iy * W + t];
  }
  double acc0 = 0.0, acc1 = 0.0;
  if (DIM == 2) {
    double xv[W][W];
#pragma unroll
    for (int u = 0; u < W; ++u)
#pragma unroll
      for (int t = 0; t < W; ++t) {
        const int jy = iy + u - Q, jx = ix + t - Q;
        xv[u][t] = (unsigned(jy) < un && unsigned(jx) < un) ? xa(jx, jy, 0) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < W; ++u)
#pragma unroll
      for (int t = 0; t < W; ++t) {
        if (t & 1) acc1 = fma(kx[t] * my[u] + mx[t] * ky[u], xv[u][t], acc1);
        else acc0 = fma(kx[t] * my[u] + mx[t] * ky[u], xv[u][t], acc0);
      }
    *diag = kx[Q] * my[Q] + mx[Q] * ky[Q];
  } else {
    double kz[W], mz[W];
#pragma unroll
    for (int t = 0; t < W; ++t) { kz[t] = sK[2 * ays + iz * W + t]; mz[t] = sM[2 * ays + iz * W + t]; }
#pragma unroll
    for (int v = 0; v < W; ++v) {
      const int jz = iz + v - Q;
      const bool okz = unsigned(jz) < un;
      double xv[W][W];
#pragma unroll
      for (int u = 0; u < W; ++u)
#pragma unroll
        for (int t = 0; t < W; ++t) {
          const int jy = iy + u - Q, jx = ix + t - Q;
          xv[u][t] = (okz && unsigned(jy) < un && unsigned(jx) < un) ? xa(jx, jy, jz) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < W; ++u) {
        const double cyz_k = my[u] * mz[v], cyz_m = ky[u] * mz[v] + my[u] * kz[v];
#pragma unroll
        for (int t = 0; t < W; ++t) {
          if (t & 1) acc1 = fma(kx[t] * cyz_k + mx[t] * cyz_m, xv[u][t], acc1);
          else acc0 = fma(kx[t] * cyz_k + mx[t] * cyz_m, xv[u][t], acc0);
        }
      }
    }
    *diag = kx[Q] * my[Q] * mz[Q] + mx[Q] * ky[Q] * mz[Q] + mx[Q] * my[Q] * kz[Q];
  }
  return acc0 + acc1;
}

// out point (rx, ry[, rz]) of the tensor transfer (⊗B) in (band W <= 4; input via accessor)
template <int DIM, class XA>
__device__ __forceinline__ double tensor_point_acc(const XA &xa, int nin, int W, const int *lo, const double *c,
                                                   int rx, int ry, int rz) {
  constexpr int WM = 4;
  const int lx = lo[rx], ly = lo[ry], lz = DIM == 3 ? lo[rz] : 0;
  double cx[WM], cy[WM], cz[WM];
#pragma unroll
  for (int k = 0; k < WM; ++k) {
    cx[k] = (k < W && unsigned(lx + k) < unsigned(nin)) ? c[rx * W + k] : 0.0;
    cy[k] = (k < W && unsigned(ly + k) < unsigned(nin)) ? c[ry * W + k] : 0.0;
    cz[k] = (DIM == 3 && k < W && unsigned(lz + k) < unsigned(nin)) ? c[rz * W + k] : 0.0;
  }
  if (DIM == 2) {
    double v[WM][WM];
#pragma unroll
    for (int ky = 0; ky < WM; ++ky)
#pragma unroll
      for (int kx = 0; kx < WM; ++kx) v[ky][kx] = (cy[ky] != 0.0 && cx[kx] != 0.0) ? xa(lx + kx, ly + ky, 0) : 0.0;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int ky = 0; ky < WM; ++ky) {
      double t = 0.0;
#pragma unroll
      for (int kx = 0; kx < WM; ++kx) t = fma(cx[kx], v[ky][kx], t);
      if (ky & 1) s1 = fma(cy[ky], t, s1); else s0 = fma(cy[ky], t, s0);
    }
    return s0 + s1;
  }
  double s = 0.0;
#pragma unroll
  for (int kz = 0; kz < WM; ++kz) {
    double v[WM][WM];
#pragma unroll
    for (int ky = 0; ky < WM; ++ky)
#pragma unroll
      for (int kx = 0; kx < WM; ++kx)
        v[ky][kx] = (cz[kz] != 0.0 && cy[ky] != 0.0 && cx[kx] != 0.0) ? xa(lx + kx, ly + ky, lz + kz) : 0.0;
    double u = 0.0;
#pragma unroll
    for (int ky = 0; ky < WM; ++ky) {
      double t = 0.0;
#pragma unroll
      for (int kx = 0; kx < WM; ++kx) t = fma(cx[kx], v[ky][kx], t);
      u = fma(cy[ky], t, u);
    }
    s = fma(cz[kz], u, s);
  }
  return s;
}

// ---- level-by-level kernels for the q-levels above the shared-memory tail (same point arithmetic as the
// tail kernel: q_point_acc, compile-time q, unrolled stencil) ----
// one (q+1)^d Gauss-Seidel colour (A11): every point of the colour, x_i += (b_i - (A x)_i) / a_ii
template <int DIM, int Q>
__global__ void __launch_bounds__(128) k_q_gs(int n, const double *__restrict__ K, const double *__restrict__ M,
                                              const double *__restrict__ b, double *__restrict__ x, int c0, int c1,
                                              int c2, int na0, int na1, int64_t total, int64_t ays) {
  constexpr int st = Q + 1;
  const XOff<DIM> xa{x, n, 0};
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int ix = c0 + st * int(idx % na0);
    const int iy = c1 + st * int((idx / na0) % na1);
    const int iz = (DIM == 3) ? c2 + st * int(idx / ((int64_t)na0 * na1)) : 0;
    double dg;
    const double ax = q_point_acc<DIM, Q>(n, K, M, xa, ix, iy, iz, &dg, ays);
    const int64_t g = ((int64_t)iz * n + iy) * n + ix;
    x[g] += (b[g] - ax) / dg;
  }
}

// r = b - A x on a whole level
template <int DIM, int Q>
__global__ void __launch_bounds__(128) k_q_resid(int n, const double *__restrict__ K, const double *__restrict__ M,
                                                 const double *__restrict__ b, const double *__restrict__ x,
                                                 double *__restrict__ r, int64_t total, int64_t ays) {
  const XOff<DIM> xa{x, n, 0};
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int ix = int(idx % n), iy = int((idx / n) % n), iz = (DIM == 3) ? int(idx / ((int64_t)n * n)) : 0;
    double dg;
    r[idx] = b[idx] - q_point_acc<DIM, Q>(n, K, M, xa, ix, iy, iz, &dg, ays);
  }
}

// Thread-level work distribution over the points of a box of rows [zlo, zhi) of the last axis;
// decode flat index -> (ix, iy, iz).
template <int DIM>
__device__ __forceinline__ void decode(int idx, int n, int zlo, int *ix, int *iy, int *iz) {
  *ix = idx % n;
  if (DIM == 2) {
    *iy = zlo + idx / n;
    *iz = 0;
  } else {
    *iy = (idx / n) % n;
    *iz = zlo + idx / (n * n);
  }
}

struct VcLev {              // one tail level as a kernel sees it
  int l, n, plane, zlo, zhi, zoff;   // own rows [zlo, zhi), stored from row zoff
  double *x, *b, *r;
  const double *K, *M;
};

template <int DIM>
__device__ __forceinline__ VcLev vc_level(const VcLayout &L, int l, int rank, double *sm) {
  VcLev v;
  v.l = l;
  v.n = L.n[l];
  v.plane = DIM == 3 ? v.n * v.n : v.n;
  if (l < L.l0 + L.nsp) {
    v.zlo = L.z0[l][rank];
    v.zhi = L.z0[l][rank + 1];
    v.zoff = v.zlo - L.H;
  } else {
    v.zlo = 0; v.zhi = v.n; v.zoff = 0;
  }
  v.x = sm + L.x[l]; v.b = sm + L.b[l]; v.r = sm + L.r[l];
  v.K = sm + L.K[l]; v.M = sm + L.M[l];
  return v;
}

// write val at own point (gz = last-axis row, inner offset) of a spread level array; refresh the
// neighbours' halo copies (DSMEM stores) when the row is within H of the slab edge
template <int DIM>
__device__ __forceinline__ void put_spread(const VcLayout &L, const VcLev &v, double *arr, int rank, int gz,
                                           int inner, double val) {
  arr[(gz - v.zoff) * v.plane + inner] = val;
  if (rank > 0 && gz < v.zlo + L.H) {
    double *rem = cg::this_cluster().map_shared_rank(arr, rank - 1);
    rem[(gz - L.z0[v.l][rank - 1] + L.H) * v.plane + inner] = val;
  }
  if (rank + 1 < L.cs && gz >= v.zhi - L.H) {
    double *rem = cg::this_cluster().map_shared_rank(arr, rank + 1);
    rem[(gz - L.z0[v.l][rank + 1] + L.H) * v.plane + inner] = val;
  }
}

// one GS colour on own rows; spread = push halos
template <int DIM, int Q>
__device__ __forceinline__ void vc_gs_colour(const VcLayout &L, const VcLev &v, int col, int rank, bool spread) {
  constexpr int st = Q + 1;
  const int n = v.n;
  const int c0 = col % st, c1 = (col / st) % st, c2 = DIM == 3 ? col / (st * st) : 0;
  const int cl = DIM == 3 ? c2 : c1;
  int fl = cl;
  if (fl < v.zlo) fl += ((v.zlo - fl + st - 1) / st) * st;
  const int nl = fl < v.zhi ? (v.zhi - 1 - fl) / st + 1 : 0;
  const int na0 = (n - c0 + Q) / st;
  const int na1 = DIM == 3 ? (n - c1 + Q) / st : nl;
  const int na2 = DIM == 3 ? nl : 1;
  const int tot = (c0 < n && (DIM == 2 || c1 < n)) ? na0 * na1 * na2 : 0;
  const XOff<DIM> xa{v.x, n, v.zoff};
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int ix = c0 + st * (idx % na0);
    int iy, iz = 0;
    if (DIM == 2) {
      iy = fl + st * (idx / na0);
    } else {
      iy = c1 + st * ((idx / na0) % na1);
      iz = fl + st * (idx / (na0 * na1));
    }
    double dg;
    const double ax = q_point_acc<DIM, Q>(n, v.K, v.M, xa, ix, iy, iz, &dg);
    const int gz = DIM == 3 ? iz : iy;
    const int inner = DIM == 3 ? iy * n + ix : ix;
    const int il = (gz - v.zoff) * v.plane + inner;
    const double nv = v.x[il] + (v.b[il] - ax) / dg;
    if (spread) put_spread<DIM>(L, v, v.x, rank, gz, inner, nv);
    else v.x[il] = nv;
  }
}

template <int DIM, int Q>
__device__ __forceinline__ void vc_residual(const VcLayout &L, const VcLev &v, int rank, bool spread) {
  const XOff<DIM> xa{v.x, v.n, v.zoff};
  const int tot = (v.zhi - v.zlo) * v.plane;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    int ix, iy, iz;
    decode<DIM>(idx, v.n, v.zlo, &ix, &iy, &iz);
    double dg;
    const double ax = q_point_acc<DIM, Q>(v.n, v.K, v.M, xa, ix, iy, iz, &dg);
    const int gz = DIM == 3 ? iz : iy;
    const int inner = DIM == 3 ? iy * v.n + ix : ix;
    const double val = v.b[(gz - v.zoff) * v.plane + inner] - ax;
    if (spread) put_spread<DIM>(L, v, v.r, rank, gz, inner, val);
    else v.r[(gz - v.zoff) * v.plane + inner] = val;
  }
}

// b_c (own rows [rlo, rhi) of level w, written to dst with row offset doff) = P^T r_v
template <int DIM>
__device__ __forceinline__ void vc_restrict(const VcLayout &L, const VcLev &v, const VcLev &w, int rlo, int rhi,
                                            double *dst, int doff, const double *sm, const int *si) {
  const XOff<DIM> ra{v.r, v.n, v.zoff};
  const int tot = (rhi - rlo) * w.plane;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    int rx, ry, rz;
    decode<DIM>(idx, w.n, rlo, &rx, &ry, &rz);
    const int gz = DIM == 3 ? rz : ry;
    const int inner = DIM == 3 ? ry * w.n + rx : rx;
    dst[(gz - doff) * w.plane + inner] =
        tensor_point_acc<DIM>(ra, v.n, L.WPT[v.l], si + L.PTlo[v.l], sm + L.PTc[v.l], rx, ry, rz);
  }
}

// x_v (own rows) += P e, e = level w values through accessor ea; spread = push halos
template <int DIM, class XA>
__device__ __forceinline__ void vc_prolong(const VcLayout &L, const VcLev &v, const VcLev &w, const XA &ea, int rank,
                                           bool spread, const double *sm, const int *si) {
  const int tot = (v.zhi - v.zlo) * v.plane;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    int rx, ry, rz;
    decode<DIM>(idx, v.n, v.zlo, &rx, &ry, &rz);
    const int gz = DIM == 3 ? rz : ry;
    const int inner = DIM == 3 ? ry * v.n + rx : rx;
    const double val = v.x[(gz - v.zoff) * v.plane + inner] +
                       tensor_point_acc<DIM>(ea, w.n, L.WP[v.l], si + L.Plo[v.l], sm + L.Pc[v.l], rx, ry, rz);
    if (spread) put_spread<DIM>(L, v, v.x, rank, gz, inner, val);
    else v.x[(gz - v.zoff) * v.plane + inner] = val;
  }
}

// coarsest level: x = A^{-1} b, rows [r0, r1): one thread per row when they fit the CTA (4 partial sums),
// else by warps; b from bsrc, x to xdst (may be remote)
__device__ __forceinline__ void vc_dense(const double *inv, int Nc, const double *bsrc, double *xdst, int r0, int r1) {
  if (r1 - r0 <= int(blockDim.x) && Nc <= 128) {
    const int row = r0 + int(threadIdx.x);
    if (row < r1) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int j = 0;
      for (; j + 3 < Nc; j += 4) {
        s0 = fma(inv[(int64_t)row * Nc + j], bsrc[j], s0);
        s1 = fma(inv[(int64_t)row * Nc + j + 1], bsrc[j + 1], s1);
        s2 = fma(inv[(int64_t)row * Nc + j + 2], bsrc[j + 2], s2);
        s3 = fma(inv[(int64_t)row * Nc + j + 3], bsrc[j + 3], s3);
      }
      for (; j < Nc; ++j) s0 = fma(inv[(int64_t)row * Nc + j], bsrc[j], s0);
      xdst[row] = (s0 + s1) + (s2 + s3);
    }
    return;
  }
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int row = r0 + int(threadIdx.x >> 5); row < r1; row += nw) {
    double s = 0.0;
    for (int j = lane; j < Nc; j += 32) s = fma(inv[(int64_t)row * Nc + j], bsrc[j], s);
    s = warp_sum(s);
    if (lane == 0) xdst[row] = s;
  }
}

template <int DIM, int Q>
__device__ void vc_local_down(const VcLayout &L, int lf, double *sm, const int *si) {
  constexpr int ncol = DIM == 3 ? (Q + 1) * (Q + 1) * (Q + 1) : (Q + 1) * (Q + 1);
  for (int l = lf; l < L.nlev - 1; ++l) {
    const VcLev v = vc_level<DIM>(L, l, 0, sm), w = vc_level<DIM>(L, l + 1, 0, sm);
    for (int col = 0; col < ncol; ++col) {
      vc_gs_colour<DIM, Q>(L, v, col, 0, false);
      __syncthreads();
    }
    vc_residual<DIM, Q>(L, v, 0, false);
    __syncthreads();
    vc_restrict<DIM>(L, v, w, 0, w.n, w.b, 0, sm, si);
    __syncthreads();
  }
}

template <int DIM, int Q>
__device__ void vc_local_up(const VcLayout &L, int lf, double *sm, const int *si) {
  constexpr int ncol = DIM == 3 ? (Q + 1) * (Q + 1) * (Q + 1) : (Q + 1) * (Q + 1);
  for (int l = L.nlev - 2; l >= lf; --l) {
    const VcLev v = vc_level<DIM>(L, l, 0, sm), w = vc_level<DIM>(L, l + 1, 0, sm);
    vc_prolong<DIM>(L, v, w, XOff<DIM>{w.x, w.n, 0}, 0, false, sm, si);
    __syncthreads();
    for (int col = 0; col < ncol; ++col) {
      vc_gs_colour<DIM, Q>(L, v, col, 0, false);
      __syncthreads();
    }
  }
}

template <int DIM, int Q>
__global__ void __launch_bounds__(512, 1) k_vcycle_smem(const VcLayout L) {
  extern __shared__ double sm[];
  int *si = reinterpret_cast<int *>(sm + L.ndouble);
  constexpr int ncol = DIM == 3 ? (Q + 1) * (Q + 1) * (Q + 1) : (Q + 1) * (Q + 1);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank());
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int l0 = L.l0, nlev = L.nlev, lf = l0 + L.nsp;   // lf: first CTA-0 level
  const bool spread = L.nsp > 0;
  if (!spread && rank != 0) return;
  // ---- staging: zero x (with halos); tables by a flat copy list (4 independent loads in flight per
  // thread); level l0's right-hand side (own rows) ----
  for (int i = tid; i < L.xend; i += nthr) sm[i] = 0.0;
  {                                                  // tables: one copy-list entry per warp, lanes strided,
    const int warp = tid >> 5, lane = tid & 31, nw = nthr >> 5;   // asynchronous (LDGSTS)
    const int ninv = L.inv_sm >= 0 ? 1 : 0;        // the staged coarsest inverse is the last entry: own group
    for (int e = warp; e < L.ncopy - ninv; e += nw) {
      const VcCopy &c = L.copy[e];
      if (c.is_int) {
        const int *src = static_cast<const int *>(c.src);
        for (int j = lane; j < c.count; j += 32) si[c.dst + j] = src[j];
      } else {
        const double *src = static_cast<const double *>(c.src);
        for (int j = lane; j < c.count; j += 32) cp_async8(sm + c.dst + j, src + j, true);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (ninv) {                                      // needed only at the coarsest solve: overlaps the down-sweep
      const VcCopy &c = L.copy[L.ncopy - 1];
      const double *src = static_cast<const double *>(c.src);
      for (int j = tid; j < c.count; j += nthr) cp_async8(sm + c.dst + j, src + j, true);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  {
    const VcLev v = vc_level<DIM>(L, l0, rank, sm);
    const int tot = (v.zhi - v.zlo) * v.plane;
    for (int i0 = tid; i0 < tot; i0 += 4 * nthr) {
      double t[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = i0 + k * nthr;
        t[k] = i < tot ? L.gb0[(int64_t)v.zlo * v.plane + i] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = i0 + k * nthr;
        if (i < tot) v.b[(v.zlo - v.zoff) * v.plane + i] = t[k];
      }
    }
  }
  asm volatile("cp.async.wait_group 1;" ::: "memory");   // tables landed (the inverse may still be in flight)
  if (spread) cl.sync(); else __syncthreads();
  // ---- down-sweep on the spread levels ----
  for (int l = l0; l < lf; ++l) {
    const VcLev v = vc_level<DIM>(L, l, rank, sm), w = vc_level<DIM>(L, l + 1, rank, sm);
    for (int col = 0; col < ncol; ++col) {
      vc_gs_colour<DIM, Q>(L, v, col, rank, true);
      cl.sync();
    }
    vc_residual<DIM, Q>(L, v, rank, true);
    cl.sync();
    if (l + 1 < lf) {                                             // into the next spread level (own rows)
      vc_restrict<DIM>(L, v, w, w.zlo, w.zhi, w.b, w.zoff, sm, si);
    } else {                                                      // into CTA 0's first level
      double *dst = cl.map_shared_rank(sm + L.b[l + 1], 0);
      vc_restrict<DIM>(L, v, w, L.rc0[rank], L.rc0[rank + 1], dst, 0, sm, si);
    }
    cl.sync();
  }
  // ---- CTA-0 levels and the coarsest solve ----
  const int NC = DIM == 3 ? L.n[nlev - 1] * L.n[nlev - 1] * L.n[nlev - 1] : L.n[nlev - 1] * L.n[nlev - 1];
  const double *inv = L.inv_sm >= 0 ? sm + L.inv_sm : L.ginv;
  if (rank == 0) vc_local_down<DIM, Q>(L, lf, sm, si);
  cp_async_wait_all();                                      // the staged inverse (own copies) ...
  __syncthreads();                                          // ... visible to the whole CTA
  if (spread && L.cbuf >= 0) {                                   // coarsest by the whole cluster
    cl.sync();
    const double *bc0 = cl.map_shared_rank(sm + L.b[nlev - 1], 0);
    for (int i = tid; i < NC; i += nthr) sm[L.cbuf + i] = bc0[i];
    __syncthreads();
    const int cs = L.cs;
    vc_dense(inv, NC, sm + L.cbuf, cl.map_shared_rank(sm + L.x[nlev - 1], 0), NC * rank / cs, NC * (rank + 1) / cs);
    cl.sync();
  } else if (rank == 0) {
    vc_dense(inv, NC, sm + L.b[nlev - 1], sm + L.x[nlev - 1], 0, NC);
    __syncthreads();
  }
  if (rank == 0) vc_local_up<DIM, Q>(L, lf, sm, si);
  // ---- up-sweep on the spread levels ----
  if (spread) {
    cl.sync();
  }
  for (int l = lf - 1; l >= l0; --l) {
    const VcLev v = vc_level<DIM>(L, l, rank, sm), w = vc_level<DIM>(L, l + 1, rank, sm);
    if (l + 1 < lf) {
      vc_prolong<DIM>(L, v, w, XOff<DIM>{w.x, w.n, w.zoff}, rank, true, sm, si);
    } else {                                                      // pull CTA 0's rows, then prolong
      const double *e0 = cl.map_shared_rank(sm + L.x[l + 1], 0);
      const int cnt = L.pcn * w.plane, off = L.pc0[rank] * w.plane;
      for (int i = tid; i < cnt; i += nthr) sm[L.pbuf + i] = (off + i < w.n * w.plane) ? e0[off + i] : 0.0;
      __syncthreads();
      vc_prolong<DIM>(L, v, w, XOff<DIM>{sm + L.pbuf, w.n, L.pc0[rank]}, rank, true, sm, si);
    }
    cl.sync();
    for (int col = 0; col < ncol; ++col) {
      vc_gs_colour<DIM, Q>(L, v, col, rank, true);
      cl.sync();
    }
  }
  {
    const VcLev v = vc_level<DIM>(L, l0, rank, sm);
    const int tot = (v.zhi - v.zlo) * v.plane;
    for (int i = tid; i < tot; i += nthr) L.gx0[(int64_t)v.zlo * v.plane + i] = v.x[(v.zlo - v.zoff) * v.plane + i];
  }
}

}  // namespace

void launch_q_gs_colour(int dim, int q, int n, const double *K, const double *M, const double *b, double *x,
                        int colour, cudaStream_t st, int64_t ays) {
  const int st_ = q + 1;
  const int c0 = colour % st_, c1 = (colour / st_) % st_, c2 = (dim == 3) ? colour / (st_ * st_) : 0;
  if (c0 >= n || c1 >= n || c2 >= n) return;
  const int na0 = (n - c0 + q) / st_, na1 = (n - c1 + q) / st_, na2 = (dim == 3) ? (n - c2 + q) / st_ : 1;
  const int64_t total = (int64_t)na0 * na1 * na2;
  const int g = grid_for(total, 128);
  if (dim == 2 && q == 1) k_q_gs<2, 1><<<g, 128, 0, st>>>(n, K, M, b, x, c0, c1, c2, na0, na1, total, ays);
  else if (dim == 2) k_q_gs<2, 2><<<g, 128, 0, st>>>(n, K, M, b, x, c0, c1, c2, na0, na1, total, ays);
  else if (q == 1) k_q_gs<3, 1><<<g, 128, 0, st>>>(n, K, M, b, x, c0, c1, c2, na0, na1, total, ays);
  else k_q_gs<3, 2><<<g, 128, 0, st>>>(n, K, M, b, x, c0, c1, c2, na0, na1, total, ays);
}

void launch_q_residual(int dim, int q, int n, const double *K, const double *M, const double *b, const double *x,
                       double *r, cudaStream_t st, int64_t ays) {
  int64_t total = (int64_t)n * n;
  if (dim == 3) total *= n;
  const int g = grid_for(total, 128);
  if (dim == 2 && q == 1) k_q_resid<2, 1><<<g, 128, 0, st>>>(n, K, M, b, x, r, total, ays);
  else if (dim == 2) k_q_resid<2, 2><<<g, 128, 0, st>>>(n, K, M, b, x, r, total, ays);
  else if (q == 1) k_q_resid<3, 1><<<g, 128, 0, st>>>(n, K, M, b, x, r, total, ays);
  else k_q_resid<3, 2><<<g, 128, 0, st>>>(n, K, M, b, x, r, total, ays);
}

bool vcycle_smem_layout(int dim, int q, const QLevelDev *tab, int nlev, int l0, int cs, size_t max_bytes,
                        VcLayout *out) {
  if (nlev > kVcMaxLev || l0 < 0 || l0 >= nlev || cs < 1 || cs > kVcMaxCS) return false;
  VcLayout L{};
  L.gb0 = tab[l0].b;
  L.gx0 = tab[l0].x;
  L.ginv = tab[nlev - 1].inv;
  L.l0 = l0; L.nlev = nlev; L.cs = cs; L.dim3 = dim == 3;
  const int W = 2 * q + 1;
  auto plane = [&](int l) { return dim == 3 ? tab[l].n * tab[l].n : tab[l].n; };
  for (int l = l0; l < nlev; ++l) {
    L.n[l] = tab[l].n;
    L.WP[l] = tab[l].P.W;
    L.WPT[l] = tab[l].PT.W;
    if (l + 1 < nlev && (tab[l].P.W > 4 || tab[l].PT.W > 4)) return false;
  }
  // host copies of the transfer bands (device pointers in tab): fetch lo arrays for the checks
  auto host_lo = [](const Band1D &B) {
    std::vector<int> h(B.rows);
    cudaMemcpy(h.data(), B.lo, B.rows * sizeof(int), cudaMemcpyDeviceToHost);
    return h;
  };
  // spread levels: every level (from l0 on) with >= 2 rows per CTA, never the coarsest
  int nsp = 0;
  if (cs > 1)
    while (l0 + nsp < nlev - 1 && tab[l0 + nsp].n >= 2 * cs) ++nsp;
  if (cs > 1 && nsp == 0) return false;
  L.nsp = nsp;
  const int lf = l0 + nsp;
  int H = 0;
  if (nsp > 0) {
    // partition: balanced on the coarsest spread level, doubled towards the finer ones
    const int lc = lf - 1;
    for (int r = 0; r <= cs; ++r) L.z0[lc][r] = short(int64_t(tab[lc].n) * r / cs);
    for (int l = lc - 1; l >= l0; --l) {
      L.z0[l][0] = 0;
      for (int r = 1; r < cs; ++r) L.z0[l][r] = short(std::min(2 * int(L.z0[l + 1][r]), tab[l].n));
      L.z0[l][cs] = short(tab[l].n);
    }
    H = q;   // GS / residual stencil reach
    for (int l = l0; l < lf; ++l)
      for (int r = 0; r < cs; ++r)
        if (L.z0[l][r + 1] - L.z0[l][r] < 1) return false;
    // halo needed by the transfers between spread levels
    for (int l = l0; l + 1 < lf; ++l) {
      const std::vector<int> plo = host_lo(tab[l].P), ptlo = host_lo(tab[l].PT);
      for (int r = 0; r < cs; ++r) {
        for (int j = L.z0[l + 1][r]; j < L.z0[l + 1][r + 1]; ++j) {   // restriction reads fine rows
          const int a = std::max(0, ptlo[j]), b = std::min(tab[l].n, ptlo[j] + tab[l].PT.W);
          H = std::max({H, L.z0[l][r] - a, b - L.z0[l][r + 1]});
        }
        for (int i = L.z0[l][r]; i < L.z0[l][r + 1]; ++i) {           // prolongation reads coarse rows
          const int a = std::max(0, plo[i]), b = std::min(tab[l + 1].n, plo[i] + tab[l].P.W);
          H = std::max({H, L.z0[l + 1][r] - a, b - L.z0[l + 1][r + 1]});
        }
      }
    }
    for (int l = l0; l < lf; ++l)
      for (int r = 0; r < cs; ++r)
        if (L.z0[l][r + 1] - L.z0[l][r] < H) return false;   // halos come from the next CTA only
    // restriction into CTA 0's level lf: coarse row j by the CTA owning the centre of its support
    {
      const int l = lf - 1;
      const std::vector<int> ptlo = host_lo(tab[l].PT);
      const int nc = tab[lf].n;
      int rr = 0;
      L.rc0[0] = 0;
      for (int j = 0; j < nc; ++j) {
        const int cen = std::min(tab[l].n - 1, std::max(0, ptlo[j] + (tab[l].PT.W - 1) / 2));
        while (rr < cs - 1 && cen >= L.z0[l][rr + 1]) L.rc0[++rr] = short(j);
        const int a = std::max(0, ptlo[j]), b = std::min(tab[l].n, ptlo[j] + tab[l].PT.W);
        if (a < L.z0[l][rr] - H || b > L.z0[l][rr + 1] + H) return false;
      }
      while (rr < cs) L.rc0[++rr] = short(nc);
      // prolongation from level lf: coarse rows each CTA pulls
      const std::vector<int> plo = host_lo(tab[l].P);
      int pcn = 0;
      for (int r = 0; r < cs; ++r) {
        int a = 1 << 30, b = -1;
        for (int i = L.z0[l][r]; i < L.z0[l][r + 1]; ++i) {
          a = std::min(a, std::max(0, plo[i]));
          b = std::max(b, std::min(tab[lf].n, plo[i] + tab[l].P.W));
        }
        L.pc0[r] = short(a);
        pcn = std::max(pcn, b - a);
      }
      L.pcn = pcn;
    }
  }
  L.H = H;
  // ---- shared-memory layout: x arrays first (zeroed at start), then b, r, buffers, tables ----
  int nd = 0, ni = 0;
  auto cnt = [&](int l) {
    if (l < lf) {
      int ny = 0;
      for (int r = 0; r < cs; ++r) ny = std::max(ny, int(L.z0[l][r + 1] - L.z0[l][r]));
      return (ny + 2 * H) * plane(l);
    }
    return int(tab[l].N);
  };
  for (int l = l0; l < nlev; ++l) { L.x[l] = nd; nd += cnt(l); }
  L.xend = nd;
  for (int l = l0; l < nlev; ++l) { L.b[l] = nd; nd += cnt(l); }
  for (int l = l0; l < nlev; ++l) { L.r[l] = nd; nd += (l == nlev - 1) ? 0 : cnt(l); }
  L.pbuf = -1;
  if (nsp > 0) { L.pbuf = nd; nd += L.pcn * plane(lf); }
  const int NC = int(tab[nlev - 1].N);
  L.cbuf = -1;
  if (nsp > 0 && NC > 64) { L.cbuf = nd; nd += NC; }
  int nc = 0;
  auto add = [&](const void *src, int dst, int count, int is_int) {
    if (count <= 0) return true;
    if (nc >= kVcMaxCopy) return false;
    L.copy[nc] = VcCopy{src, dst, count, is_int, 0};
    L.copy_start[nc + 1] = L.copy_start[nc] + count;
    ++nc;
    return true;
  };
  L.copy_start[0] = 0;
  bool ok = true;
  for (int l = l0; l < nlev; ++l) {
    const int n = tab[l].n;
    L.K[l] = nd; nd += n * W;
    L.M[l] = nd; nd += n * W;
    ok = ok && add(tab[l].K, L.K[l], n * W, 0) && add(tab[l].M, L.M[l], n * W, 0);
    if (l + 1 < nlev) {
      L.Pc[l] = nd; nd += tab[l].P.rows * tab[l].P.W;
      L.PTc[l] = nd; nd += tab[l].PT.rows * tab[l].PT.W;
      L.Plo[l] = ni; ni += tab[l].P.rows;
      L.PTlo[l] = ni; ni += tab[l].PT.rows;
      ok = ok && add(tab[l].P.c, L.Pc[l], tab[l].P.rows * tab[l].P.W, 0) &&
           add(tab[l].PT.c, L.PTc[l], tab[l].PT.rows * tab[l].PT.W, 0) && add(tab[l].P.lo, L.Plo[l], tab[l].P.rows, 1) &&
           add(tab[l].PT.lo, L.PTlo[l], tab[l].PT.rows, 1);
    }
  }
  L.inv_sm = -1;
  if (size_t(NC) * NC <= 4096 && (size_t(nd) + size_t(NC) * NC) * 8 + size_t(ni) * 4 <= max_bytes) {
    L.inv_sm = nd;
    nd += NC * NC;
    ok = ok && add(tab[nlev - 1].inv, L.inv_sm, NC * NC, 0);
  }
  if (!ok) return false;
  L.ncopy = nc;
  L.ndouble = nd;
  L.nint = ni;
  if (size_t(nd) * 8 + size_t(ni) * 4 > max_bytes) return false;
  *out = L;
  return true;
}

size_t vcycle_smem_bytes(const VcLayout &L) { return size_t(L.ndouble) * 8 + size_t(L.nint) * 4; }

namespace {
template <int DIM, int Q>
void *vc_kernel() { return reinterpret_cast<void *>(k_vcycle_smem<DIM, Q>); }
void *vc_kernel_for(int dim, int q) {
  return dim == 2 ? (q == 1 ? vc_kernel<2, 1>() : vc_kernel<2, 2>()) : (q == 1 ? vc_kernel<3, 1>() : vc_kernel<3, 2>());
}
cudaLaunchConfig_t vc_config(const VcLayout &L, cudaStream_t st, cudaLaunchAttribute *at) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.cs, 1, 1);
  cfg.blockDim = dim3(512, 1, 1);
  cfg.dynamicSmemBytes = vcycle_smem_bytes(L);
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = L.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}
}  // namespace

bool vcycle_smem_probe(int dim, int q, const VcLayout &L) {
  const void *kern = vc_kernel_for(dim, q);
  const size_t sm = vcycle_smem_bytes(L);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)) != cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = vc_config(L, nullptr, at);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    return false;
  }
  return true;
}

cudaError_t launch_vcycle_smem(int dim, int q, const VcLayout &L, cudaStream_t st) {
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = vc_config(L, st, at);
  void *args[] = {const_cast<VcLayout *>(&L)};
  return cudaLaunchKernelExC(&cfg, vc_kernel_for(dim, q), args);
}

}  // namespace iga2l
