// Tensor-product band transfers: restriction d_q = (⊗R1) d and
// prolongation x += (⊗R1)^T e on the fine level, the h<->2h transfers of the V-cycle.  See kernels.cuh.
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace iga2l {
namespace {

// =============================== band transform along one axis ===========================
// Columns valid in [clo, chi), stored from column coff on (nin stored columns per outer slice);
// output rows r in [rlo, rhi), stored from row rlo on (rhi - rlo rows per outer slice).
// One thread per output, no index divisions: inner > 1 -> threads along the contiguous inner index,
// blockIdx.y = output row, blockIdx.z = outer slice; inner == 1 -> threads along the output rows,
// blockIdx.y + gridDim.y * blockIdx.z = outer slice.
__global__ void __launch_bounds__(256) k_band_axis(const double *__restrict__ in, double *__restrict__ out,
                                                   int64_t outer, int nin, int64_t inner, int W,
                                                   const int *__restrict__ lo, const double *__restrict__ c, int acc,
                                                   int clo, int chi, int coff, int rlo, int rhi) {
  const int nr = rhi - rlo;
  int64_t i, o;
  int r;
  if (inner == 1) {
    r = rlo + int(blockIdx.x * blockDim.x + threadIdx.x);
    o = blockIdx.y + int64_t(gridDim.y) * blockIdx.z;
    i = 0;
    if (r >= rhi || o >= outer) return;
  } else {
    i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    r = rlo + int(blockIdx.y);
    o = blockIdx.z;
    if (i >= inner) return;
  }
  const int l0 = lo[r];
  const double *src = in + (o * nin - coff) * inner + i;
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {              // all gathers independent (W <= 16 checked at setup)
    const int col = l0 + k;
    const bool ok = k < W && col >= clo && col < chi;
    const double v = ok ? c[int64_t(r) * W + k] * src[int64_t(col) * inner] : 0.0;
    if (k & 1) s1 += v; else s0 += v;
  }
  const double s = s0 + s1;
  const int64_t idx = (o * nr + (r - rlo)) * inner + i;
  out[idx] = acc ? out[idx] + s : s;
}

// The same transform with a compile-time band width (v2: the generic kernel above was issue-bound at ~87%
// of issue slots on C5's transfers): coefficients of the CTA's output row in registers, valid-column range
// decided once per CTA (uniform branch), pointer increments instead of 64-bit products, and V = 2
// consecutive inner outputs per thread by 16-byte loads when the inner extent is even.
template <int W, int V>
__global__ void __launch_bounds__(256) k_band_inner(const double *__restrict__ in, double *__restrict__ out, int nin,
                                                    int64_t inner, const int *__restrict__ lo,
                                                    const double *__restrict__ c, int acc, int clo, int chi, int coff,
                                                    int rlo, int nr) {
  const int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * V;
  if (i >= inner) return;
  const int r = rlo + int(blockIdx.y);
  const int64_t o = blockIdx.z;
  const int l0 = lo[r];
  const int kb = max(0, clo - l0), ke = min(W, chi - l0);     // valid band columns (uniform per CTA)
  double cf[W];
#pragma unroll
  for (int k = 0; k < W; ++k) cf[k] = __ldg(c + int64_t(r) * W + k);
  const double *src = in + (o * nin - coff + l0) * inner + i;
  double s0[V], s1[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s0[v] = s1[v] = 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k >= kb && k < ke) {
      if constexpr (V == 2) {
        const double2 t = __ldg(reinterpret_cast<const double2 *>(src + k * inner));
        if (k & 1) { s1[0] = fma(cf[k], t.x, s1[0]); s1[1] = fma(cf[k], t.y, s1[1]); }
        else { s0[0] = fma(cf[k], t.x, s0[0]); s0[1] = fma(cf[k], t.y, s0[1]); }
      } else {
        const double t = __ldg(src + k * inner);
        if (k & 1) s1[0] = fma(cf[k], t, s1[0]); else s0[0] = fma(cf[k], t, s0[0]);
      }
    }
  }
  double *dst = out + (o * nr + (r - rlo)) * inner + i;
  if constexpr (V == 2) {
    double2 res = make_double2(s0[0] + s1[0], s0[1] + s1[1]);
    if (acc) {
      const double2 prev = *reinterpret_cast<const double2 *>(dst);
      res.x += prev.x;
      res.y += prev.y;
    }
    *reinterpret_cast<double2 *>(dst) = res;
  } else {
    const double s = s0[0] + s1[0];
    *dst = acc ? *dst + s : s;
  }
}

// inner == 1 (the contiguous axis): one thread per output row r of one outer slice.
template <int W>
__global__ void __launch_bounds__(128) k_band_rows(const double *__restrict__ in, double *__restrict__ out,
                                                   int64_t outer, int nin, const int *__restrict__ lo,
                                                   const double *__restrict__ c, int acc, int clo, int chi, int coff,
                                                   int rlo, int rhi) {
  const int r = rlo + int(blockIdx.x * blockDim.x + threadIdx.x);
  const int64_t o = blockIdx.y + int64_t(gridDim.y) * blockIdx.z;
  if (r >= rhi || o >= outer) return;
  const int l0 = lo[r];
  const double *src = in + o * nin - coff + l0;
  const double *cr = c + int64_t(r) * W;
  double s0 = 0.0, s1 = 0.0;
  if (l0 >= clo && l0 + W <= chi) {                          // interior row: no column checks
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const double t = __ldg(cr + k) * __ldg(src + k);
      if (k & 1) s1 += t; else s0 += t;
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int col = l0 + k;
      if (col >= clo && col < chi) {
        const double t = __ldg(cr + k) * __ldg(src + k);
        if (k & 1) s1 += t; else s0 += t;
      }
    }
  }
  const double s = s0 + s1;
  const int64_t idx = (o * (rhi - rlo) + (r - rlo));
  out[idx] = acc ? out[idx] + s : s;
}

// 2D tensor transfer, direct: out[ry][rx] (+)= Σ_{ky,kx} c[ry][ky] c[rx][kx] in[lo[ry]+ky][lo[rx]+kx].
// The band loops are unrolled to a compile-time bound so that all W^2 gathers of an output are
// independent loads (one L2 round trip instead of W^2 dependent ones).
// Input rows (last axis) are valid in [iylo, iyhi) and stored from row iyoff on; columns in [0, nin).
template <int WMAX>
__device__ __forceinline__ double tensor2d_point(const double *__restrict__ in, int nin, int iylo, int iyhi, int iyoff,
                                                 int W, const int *__restrict__ lo, const double *__restrict__ c,
                                                 int Wy, const int *__restrict__ loy, const double *__restrict__ cyt,
                                                 int ry, int rx) {
  const int ly = loy[ry], lx = lo[rx];
  double cy[WMAX], cx[WMAX];
#pragma unroll
  for (int k = 0; k < WMAX; ++k) {
    const bool oky = k < Wy && ly + k >= iylo && ly + k < iyhi, okx = k < W && unsigned(lx + k) < unsigned(nin);
    cy[k] = oky ? cyt[(int64_t)ry * Wy + k] : 0.0;
    cx[k] = okx ? c[(int64_t)rx * W + k] : 0.0;
  }
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int ky = 0; ky < WMAX; ++ky) {
    double t = 0.0;
#pragma unroll
    for (int kx = 0; kx < WMAX; ++kx) {
      const bool ok = cy[ky] != 0.0 && cx[kx] != 0.0;
      const double v = ok ? in[(int64_t)(ly + ky - iyoff) * nin + (lx + kx)] : 0.0;
      t = fma(cx[kx], v, t);
    }
    if (ky & 1) s1 = fma(cy[ky], t, s1); else s0 = fma(cy[ky], t, s0);
  }
  return s0 + s1;
}

// Output rows ry in [rylo, ryhi) are stored from row ryoff on (all rows.x columns).
template <int WMAX>
__global__ void k_tensor2d(const double *__restrict__ in, double *__restrict__ out, int nin, int rows, int W,
                           const int *__restrict__ lo, const double *__restrict__ c, int Wy,
                           const int *__restrict__ loy, const double *__restrict__ cyt, int acc, int iylo, int iyhi,
                           int iyoff, int rylo, int ryhi, int ryoff) {
  const int64_t total = (int64_t)(ryhi - rylo) * rows;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int ry = rylo + int(idx / rows), rx = int(idx % rows);
    const double s = tensor2d_point<WMAX>(in, nin, iylo, iyhi, iyoff, W, lo, c, Wy, loy, cyt, ry, rx);
    const int64_t o = (int64_t)(ry - ryoff) * rows + rx;
    out[o] = acc ? out[o] + s : s;
  }
}

// ---------------- separable 2D tensor transfer (v2): out (+)= (B ⊗ B) in, two passes ----------
// CTA = TO x TO outputs.  Pass 1 (x): T[iy][rx] = Σ_k c[rx][k] in[iy][lo[rx]+k] for the input rows the
// tile needs; pass 2 (y): out[ry][rx] = Σ_k c[ry][k] T[lo[ry]+k][rx].  2W FMAs per output (plus the
// input-row halo of pass 1) instead of W^2 gathers.  Input rows valid in [iylo, iyhi) stored from
// iyoff; output rows [rylo, ryhi) stored from ryoff (slab views).
template <int TO>
__global__ void __launch_bounds__(256) k_transfer2d_sep(const double *__restrict__ in, double *__restrict__ out, int nin,
                                                        int rows, int W, const int *__restrict__ lo,
                                                        const double *__restrict__ c, int Wy,
                                                        const int *__restrict__ loy, const double *__restrict__ cyt,
                                                        int acc, int iylo, int iyhi, int iyoff, int rylo, int ryhi,
                                                        int ryoff, int LI) {
  extern __shared__ double sm[];
  const int rx0 = blockIdx.x * TO, ry0 = rylo + blockIdx.y * TO;
  const int nrx = min(TO, rows - rx0), nry = min(TO, ryhi - ry0);
  if (nrx <= 0 || nry <= 0) return;
  const int ix0 = lo[rx0], iy0 = loy[ry0];                 // first input column / row of the tile
  double *X = sm;                                           // [LI][LI] input window
  double *T = X + LI * LI;                                  // [LI][TO]
  double *cx = T + LI * TO, *cy = cx + TO * W;              // coefficient rows of the tile
  int *lx = reinterpret_cast<int *>(cy + TO * Wy), *ly = lx + TO;
  const int tid = threadIdx.x;
  for (int i = tid; i < LI * LI; i += 256) {
    const int wy = i / LI, wx = i - wy * LI, gx = ix0 + wx, gy = iy0 + wy;
    const bool ok = unsigned(gx) < unsigned(nin) && gy >= iylo && gy < iyhi;
    cp_async8(X + i, in + (ok ? (int64_t)(gy - iyoff) * nin + gx : 0), ok);
  }
  for (int i = tid; i < TO * W; i += 256) {
    const int r = i / W;
    const bool okx = r < nrx;
    cp_async8(cx + i, c + (okx ? (int64_t)(rx0 + r) * W + i % W : 0), okx);
  }
  for (int i = tid; i < TO * Wy; i += 256) {
    const int r = i / Wy;
    const bool oky = r < nry;
    cp_async8(cy + i, cyt + (oky ? (int64_t)(ry0 + r) * Wy + i % Wy : 0), oky);
  }
  if (tid < TO) {
    lx[tid] = tid < nrx ? lo[rx0 + tid] - ix0 : 0;
    ly[tid] = tid < nry ? loy[ry0 + tid] - iy0 : 0;
  }
  cp_async_wait_all();
  __syncthreads();
  // pass 1: rows of the window that pass 2 reads: [0, ly[nry-1] + W)
  const int nrow = min(LI, ly[nry - 1] + Wy);
  for (int i = tid; i < nrow * TO; i += 256) {
    const int wy = i / TO, r = i - wy * TO;
    double s0 = 0.0, s1 = 0.0;
    if (r < nrx) {
      const double *xr = X + wy * LI + lx[r], *cr = cx + r * W;
      for (int k = 0; k < W; ++k) {
        if (k & 1) s1 = fma(cr[k], xr[k], s1); else s0 = fma(cr[k], xr[k], s0);
      }
    }
    T[i] = s0 + s1;
  }
  __syncthreads();
  for (int i = tid; i < TO * TO; i += 256) {
    const int ry = i / TO, r = i - ry * TO;
    if (ry >= nry || r >= nrx) continue;
    const double *tc = T + ly[ry] * TO + r, *cr = cy + ry * Wy;
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < Wy; ++k) {
      if (k & 1) s1 = fma(cr[k], tc[k * TO], s1); else s0 = fma(cr[k], tc[k * TO], s0);
    }
    const int64_t o = (int64_t)(ry0 + ry - ryoff) * rows + rx0 + r;
    out[o] = acc ? out[o] + (s0 + s1) : (s0 + s1);
  }
}

}  // namespace

void launch_band_axis(const double *in, double *out, int64_t outer, int nin, int64_t inner, const Band1D &B,
                      int accumulate, cudaStream_t st, int clo, int chi, int coff, int rlo, int rhi) {
  if (chi < 0) { clo = 0; chi = nin; coff = 0; }
  if (rhi < 0) { rlo = 0; rhi = B.rows; }
  const int64_t total = outer * (rhi - rlo) * inner;
  if (total <= 0) return;
  const int nr = rhi - rlo;
  const unsigned gy = unsigned(std::min<int64_t>(outer, 32768)), gz = unsigned((outer + gy - 1) / gy);
  const bool v2 = inner % 2 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  bool done = false;
  auto go = [&](auto wtag) {
    constexpr int Wc = decltype(wtag)::value;
    if (inner == 1) {
      k_band_rows<Wc><<<dim3((nr + 127) / 128, gy, gz), 128, 0, st>>>(in, out, outer, nin, B.lo, B.c, accumulate, clo,
                                                                        chi, coff, rlo, rhi);
    } else if (v2) {
      k_band_inner<Wc, 2><<<dim3(unsigned((inner / 2 + 255) / 256), unsigned(nr), unsigned(outer)), 256, 0, st>>>(
          in, out, nin, inner, B.lo, B.c, accumulate, clo, chi, coff, rlo, nr);
    } else {
      k_band_inner<Wc, 1><<<dim3(unsigned((inner + 255) / 256), unsigned(nr), unsigned(outer)), 256, 0, st>>>(
          in, out, nin, inner, B.lo, B.c, accumulate, clo, chi, coff, rlo, nr);
    }
    done = true;
  };
  switch (B.W) {
#define IGA2L_BW(w_) case w_: go(std::integral_constant<int, w_>{}); break;
    IGA2L_BW(1) IGA2L_BW(2) IGA2L_BW(3) IGA2L_BW(4) IGA2L_BW(5) IGA2L_BW(6) IGA2L_BW(7) IGA2L_BW(8)
    IGA2L_BW(9) IGA2L_BW(10) IGA2L_BW(11) IGA2L_BW(12) IGA2L_BW(13) IGA2L_BW(14) IGA2L_BW(15) IGA2L_BW(16)
#undef IGA2L_BW
    default: break;
  }
  if (done) return;
  if (inner == 1) {
    k_band_axis<<<dim3((nr + 127) / 128, gy, gz), 128, 0, st>>>(in, out, outer, nin, inner, B.W, B.lo, B.c,
                                                                accumulate, clo, chi, coff, rlo, rhi);
  } else {
    k_band_axis<<<dim3(unsigned((inner + 255) / 256), unsigned(nr), unsigned(outer)), 256, 0, st>>>(
        in, out, outer, nin, inner, B.W, B.lo, B.c, accumulate, clo, chi, coff, rlo, rhi);
  }
}

void launch_tensor2d(const double *in, double *out, const Band1D &B, int accumulate, cudaStream_t st,
                     int iylo, int iyhi, int iyoff, int rylo, int ryhi, int ryoff, const Band1D *Byp) {
  const Band1D &By = Byp ? *Byp : B;        // y-axis band (per-axis transfers: the quarter annulus)
  if (iyhi < 0) { iylo = 0; iyhi = By.cols; iyoff = 0; }
  if (ryhi < 0) { rylo = 0; ryhi = By.rows; ryoff = 0; }
  const int64_t total = (int64_t)(ryhi - rylo) * B.rows;
  if (total <= 0) return;
  const int Wm = std::max(B.W, By.W);
  // test knob: IGA2L_TRANSFER_SEP=32|16 forces that separable tile at any size (the C3 path at PAR sizes)
  const char *fs = std::getenv("IGA2L_TRANSFER_SEP");
  const int force = fs ? std::atoi(fs) : 0;
  auto go = [&](auto kern, int TO, int span) {
    const int LI = span + Wm;
    const size_t sm = sizeof(double) * (size_t(LI) * LI + size_t(LI) * TO + TO * size_t(B.W + By.W)) + 2 * TO * sizeof(int);
    if (sm > 200 * 1024) return false;
    ensure_smem(kern, sm);
    dim3 grid((unsigned)((B.rows + TO - 1) / TO), (unsigned)((ryhi - rylo + TO - 1) / TO));
    kern<<<grid, 256, sm, st>>>(in, out, B.cols, B.rows, B.W, B.lo, B.c, By.W, By.lo, By.c, accumulate, iylo, iyhi,
                                iyoff, rylo, ryhi, ryoff, LI);
    return true;
  };
  const int span32 = (B.lo_max_span > 0 && By.lo_max_span > 0) ? std::max(B.lo_max_span, By.lo_max_span) : 0;
  const int span16 = (B.lo_max_span16 > 0 && By.lo_max_span16 > 0) ? std::max(B.lo_max_span16, By.lo_max_span16) : 0;
  if (force == 32 && span32 > 0 && go(k_transfer2d_sep<32>, 32, span32)) return;
  if (span32 > 0) {   // separable two-pass
    if (total >= 200000) {
      if (go(k_transfer2d_sep<32>, 32, span32)) return;
    } else if (span16 > 0 && go(k_transfer2d_sep<16>, 16, span16)) {
      return;
    }
  }
  const int g = grid_for(total, 128);
  if (Wm <= 4)
    k_tensor2d<4><<<g, 128, 0, st>>>(in, out, B.cols, B.rows, B.W, B.lo, B.c, By.W, By.lo, By.c, accumulate, iylo, iyhi,
                                     iyoff, rylo, ryhi, ryoff);
  else if (Wm <= 8)
    k_tensor2d<8><<<g, 128, 0, st>>>(in, out, B.cols, B.rows, B.W, B.lo, B.c, By.W, By.lo, By.c, accumulate, iylo, iyhi,
                                     iyoff, rylo, ryhi, ryoff);
  else
    k_tensor2d<16><<<g, 128, 0, st>>>(in, out, B.cols, B.rows, B.W, B.lo, B.c, By.W, By.lo, By.c, accumulate, iylo,
                                      iyhi, iyoff, rylo, ryhi, ryoff);
}

}  // namespace iga2l
