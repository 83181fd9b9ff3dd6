// 3D multicolour Schwarz colour kernel (reading A4, A25): one CTA per block, register-blocked
// pencil passes for the sum-factorised block residual, then fast diagonalisation.  See kernels.cuh.
#include <cuda.h>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace iga2l {
namespace {

// ---------------- v4: one block per CTA, per-thread roles fixed up front ----------------------------
// Sum-factorised block residual (pencil passes x, y, z) and fast diagonalisation; per block:
// the window is staged by rows (one division per row, Wn 8-byte cp.async with a per-block column range),
// band rows / FD tables of Toeplitz axes (reading A27) come from the kernel parameter (constant bank) and
// are only loaded for boundary axes, and every index is decoded once per thread.
template <int P, int S>
struct B4 {
  static constexpr int W = 2 * P + 1, Wn = S + 2 * P, w = (S - 1) / 2, S2 = S * S, S3 = S2 * S, Wn2 = Wn * Wn;
  static constexpr int OPa = Wn2 * Wn, OPb = OPa + Wn2 * S, OXc = OPb + Wn2 * S, OR = OXc + S3, OQ = OR + S3,
                       OBb = OQ + S3, OTk = OBb + S3, OTm = OTk + 3 * S * W, OVs = OTm + 3 * S * W, OLs = OVs + 3 * S2;
  static constexpr int PER = OLs + 3 * S;
  // TMA window.  Grid rows J (the n1-element x-rows, counted from the stored base) of one parity are
  // 2 n1 elements apart -- a 16-byte multiple even for odd n1 -- so the even rows and the odd rows each form
  // a 2D tensor (two maps; the odd one based one element early so that its base stays 16-byte aligned).
  // A window plane is then TWO box loads of BR rows x BOX columns into consecutive 128-byte shared rows
  // with 128B swizzle (chunk c of shared row R lands at chunk c ^ (R & 7): conflict-free pencil reads).  Boxes start at the
  // even column at or below the first needed one; rows are read with that parity shift.
  static constexpr int BOX = ((Wn + 2) / 2) * 2, RW = 16, BR = (Wn + 1) / 2, XT = Wn * 2 * BR * RW;
  static constexpr bool TMA_OK = BOX * 8 <= 128 && BR <= 8;
  static constexpr int OFF = TMA_OK ? (XT > OPa ? XT - OPa : 0) : 0;   // window area grows to Wn x 2 tiles
  static constexpr int PERT = PER + OFF;
  static constexpr int NT0 = ((Wn2 + 31) / 32) * 32 > 512 ? 512 : ((Wn2 + 31) / 32) * 32;
  static constexpr int NT = (S >= 5 && NT0 >= 128) ? NT0 / 2 : NT0;
  static_assert(2 * Wn * S2 <= Wn2 * Wn, "Pc/Pe must fit in the window");
  static_assert(S3 <= NT || S == 3, "one FD point per thread");
};

template <int S, int W, int Wn, bool TOE>
__device__ __forceinline__ void pencil_x(const double *xr, const double *ck, const double *cm, const ToeP &tp,
                                         double *oa, double *ob, int ostride) {
  double v[Wn];
#pragma unroll
  for (int k = 0; k < Wn; ++k) v[k] = xr[k];
#pragma unroll
  for (int l = 0; l < S; ++l) {
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int t = 0; t < W; ++t) {
      const double kc = TOE ? tp.k[t] : ck[l * W + t], mc = TOE ? tp.m[t] : cm[l * W + t];
      if (t & 1) { a1 = fma(kc, v[l + t], a1); b1 = fma(mc, v[l + t], b1); }
      else { a0 = fma(kc, v[l + t], a0); b0 = fma(mc, v[l + t], b0); }
    }
    oa[l * ostride] = a0 + a1;
    ob[l * ostride] = b0 + b1;
  }
}

template <int S, int W, int Wn, bool TOE>
__device__ __forceinline__ void pencil_yz(const double *pa_, const double *pb_, int stride, const double *ck,
                                          const double *cm, const ToeP &tp, double (&oc)[S], double (&oe)[S]) {
  double pa[Wn], pb[Wn];
#pragma unroll
  for (int k = 0; k < Wn; ++k) { pa[k] = pa_[k * stride]; pb[k] = pb_[k * stride]; }
#pragma unroll
  for (int l = 0; l < S; ++l) {
    double c0 = 0.0, c1 = 0.0, e0 = 0.0;
#pragma unroll
    for (int t = 0; t < W; ++t) {
      const double kc = TOE ? tp.k[t] : ck[l * W + t], mc = TOE ? tp.m[t] : cm[l * W + t];
      c0 = fma(mc, pa[l + t], c0);
      c1 = fma(kc, pb[l + t], c1);
      e0 = fma(mc, pb[l + t], e0);
    }
    oc[l] = c0 + c1;
    oe[l] = e0;
  }
}

template <int P, int S, bool TMA>
__global__ void __launch_bounds__(B4<P, S>::NT) k_schwarz3d_v4(const __grid_constant__ CUtensorMap xmap_e,
                                                                const __grid_constant__ CUtensorMap xmap_o, int n1,
                                                                const double *__restrict__ K,
                                                                const double *__restrict__ M,
                                                                const double *__restrict__ Vt,
                                                                const double *__restrict__ lamt,
                                                                const double *__restrict__ b, double *__restrict__ x,
                                                                int c0, int c1, int c2, int D, int nb0, int nb1,
                                                                int zoff, int tlo, int thi, const ToeP tp) {
  using B = B4<P, S>;
  constexpr int W = B::W, Wn = B::Wn, w = B::w, S2 = B::S2, S3 = B::S3, Wn2 = B::Wn2, NT = B::NT;
  constexpr int O = TMA ? B::OFF : 0;
  extern __shared__ __align__(1024) double sm[];
  double *X = sm, *Pa = sm + O + B::OPa, *Pb = sm + O + B::OPb, *Pc = sm, *Pe = sm + Wn * S2, *Xc = sm + O + B::OXc;
  double *R = sm + O + B::OR, *Q = sm + O + B::OQ, *Bb = sm + O + B::OBb, *Tk = sm + O + B::OTk, *Tm = sm + O + B::OTm;
  double *Vs = sm + O + B::OVs, *Ls = sm + O + B::OLs;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + O + B::PER);
  const int tid = threadIdx.x;
  const unsigned un = unsigned(n1);
  const int g = blockIdx.x;
  const int cc[3] = {c0 + D * (g % nb0), c1 + D * ((g / nb0) % nb1), c2 + D * (g / (nb0 * nb1))};
  const bool tv = tp.valid != 0;
  bool toe[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) toe[a] = tv && cc[a] - w >= tlo && cc[a] + w <= thi;
  const int ox = cc[0] - w - P, oy = cc[1] - w - P, oz = cc[2] - w - P;
  // ---- window rows r = (wz, wy) ----
  if constexpr (TMA) {                                            // two box loads per plane (see B4)
    if (tid == 0) {
      mbar_init(bar, 1);
      mbar_fence_init();
      mbar_expect_tx(bar, Wn * 2 * B::BR * B::BOX * 8);
    }
    __syncthreads();
    if (tid < 2 * Wn) {
      const int wz = tid >> 1, par = tid & 1;                   // plane, row parity (of J)
      const int J0 = (oz + wz - zoff) * n1 + oy;                // first window row of the plane
      const int Jf = J0 + ((J0 ^ par) & 1);                     // first window row of parity par
      double *dst = X + (wz * 2 + par) * B::BR * B::RW;
      if (par == 0) tma_load_2d(dst, &xmap_e, ox & ~1, Jf >> 1, bar);
      else tma_load_2d(dst, &xmap_o, (ox + 1) & ~1, Jf >> 1, bar);
    }
  } else {                                                        // LG lanes per row: coalesced row copies
    // (zero outside the domain)                                                               // LG lanes per row: coalesced row copies
    constexpr int LG = Wn <= 16 ? 16 : 32, RPI = NT / LG;           // rows per iteration of the CTA
    const int col = tid % LG, r0 = tid / LG;
    const bool colok = col < Wn && unsigned(ox + col) < un;
    for (int r = r0; r < Wn2; r += RPI) {
      const int wz = r / Wn, wy = r - wz * Wn, gy = oy + wy, gz = oz + wz;
      const bool ok = colok && unsigned(gy) < un && unsigned(gz) < un;
      if (col < Wn) cp_async8(X + r * Wn + col, ok ? x + (int64_t(gz - zoff) * n1 + gy) * n1 + ox + col : x, ok);
    }
  }
  // ---- b_B, and band rows / FD tables of the boundary axes ----
  int lx = 0, ly = 0, lz = 0;                                     // this thread's FD / update point
  if (tid < S3) {
    lz = tid / S2;
    ly = (tid - lz * S2) / S;
    lx = tid - lz * S2 - ly * S;
    const int gx = cc[0] - w + lx, gy = cc[1] - w + ly, gz = cc[2] - w + lz;
    const bool ok = unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un;
    cp_async8(Bb + tid, b + (ok ? (int64_t(gz - zoff) * n1 + gy) * n1 + gx : 0), ok);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (toe[a]) continue;
    for (int i = tid; i < S * W; i += NT) {
      const int l = i / W, t = i - l * W, gr = cc[a] - w + l;
      const bool ok = unsigned(gr) < un;
      cp_async8(Tk + a * S * W + i, K + (ok ? int64_t(gr) * W + t : 0), ok);
      cp_async8(Tm + a * S * W + i, M + (ok ? int64_t(gr) * W + t : 0), ok);
    }
    for (int i = tid; i < S2; i += NT) cp_async8(Vs + a * S2 + i, Vt + int64_t(cc[a]) * S2 + i, true);
    if (tid < S) cp_async8(Ls + a * S + tid, lamt + int64_t(cc[a]) * S + tid, true);
  }
  cp_async_wait_all();
  if constexpr (TMA) mbar_wait(bar, 0);
  __syncthreads();
  // ---- pass x: pencils (wy, wz) along x -> Pa = Kx X, Pb = Mx X ----
  // window row (wz, wy) -> tile row: parity of J = J0 + wy, index among the plane's rows of that parity
  auto trow = [&](int wz, int wy, int *k, int *sh) {
    const int J0 = (oz + wz - zoff) * n1 + oy, par = (J0 + wy) & 1, d0 = J0 & 1;
    *k = par == 0 ? ((wy + d0) >> 1) - d0 : (wy - 1 + d0) >> 1;
    *sh = par == 0 ? (ox & 1) : ((ox + 1) & 1);
    return (wz * 2 + par) * B::BR;
  };
  if constexpr (TMA) {
    for (int pi = tid; pi < Wn2; pi += NT) {
      const int wz = pi / Wn, wy = pi - wz * Wn;
      int k, sh;
      const int t0 = trow(wz, wy, &k, &sh);
      const double2 *row = reinterpret_cast<const double2 *>(X + (t0 + k) * B::RW);
      const int sw = (t0 + k) & 7;
      double v[B::BOX];
#pragma unroll
      for (int c = 0; c < B::BOX / 2; ++c) {
        const double2 t = row[c ^ sw];
        v[2 * c] = t.x;
        v[2 * c + 1] = t.y;
      }
      double u[Wn];
#pragma unroll
      for (int k = 0; k < Wn; ++k) u[k] = sh ? v[k + 1] : v[k];
      if (toe[0]) pencil_x<S, W, Wn, true>(u, Tk, Tm, tp, Pa + pi * S, Pb + pi * S, 1);
      else pencil_x<S, W, Wn, false>(u, Tk, Tm, tp, Pa + pi * S, Pb + pi * S, 1);
    }
    if (tid < S3) {
      int k, sh;
      const int t0 = trow(lz + P, ly + P, &k, &sh);
      const int e = lx + P + sh;
      Xc[tid] = X[(t0 + k) * B::RW + (((e >> 1) ^ ((t0 + k) & 7)) << 1) + (e & 1)];
    }
  } else {
    for (int pi = tid; pi < Wn2; pi += NT) {
      if (toe[0]) pencil_x<S, W, Wn, true>(X + pi * Wn, Tk, Tm, tp, Pa + pi * S, Pb + pi * S, 1);
      else pencil_x<S, W, Wn, false>(X + pi * Wn, Tk, Tm, tp, Pa + pi * S, Pb + pi * S, 1);
    }
    if (tid < S3) Xc[tid] = X[((lz + P) * Wn + ly + P) * Wn + lx + P];   // before Pc/Pe overwrite X
  }
  __syncthreads();
  // ---- pass y: pencils (wz, lx) along y -> Pc = My Pa + Ky Pb, Pe = My Pb ----
  for (int pi = tid; pi < Wn * S; pi += NT) {
    const int wz = pi / S, px = pi - wz * S;
    double oc[S], oe[S];
    if (toe[1]) pencil_yz<S, W, Wn, true>(Pa + wz * Wn * S + px, Pb + wz * Wn * S + px, S, Tk + S * W, Tm + S * W, tp, oc, oe);
    else pencil_yz<S, W, Wn, false>(Pa + wz * Wn * S + px, Pb + wz * Wn * S + px, S, Tk + S * W, Tm + S * W, tp, oc, oe);
#pragma unroll
    for (int l = 0; l < S; ++l) { Pc[(wz * S + l) * S + px] = oc[l]; Pe[(wz * S + l) * S + px] = oe[l]; }
  }
  __syncthreads();
  // ---- pass z: pencils (ly, lx) along z -> r_B = b_B - (Mz Pc + Kz Pe) ----
  if (tid < S2) {
    double oc[S], oe[S];
    if (toe[2]) pencil_yz<S, W, Wn, true>(Pc + tid, Pe + tid, S2, Tk + 2 * S * W, Tm + 2 * S * W, tp, oc, oe);
    else pencil_yz<S, W, Wn, false>(Pc + tid, Pe + tid, S2, Tk + 2 * S * W, Tm + 2 * S * W, tp, oc, oe);
#pragma unroll
    for (int l = 0; l < S; ++l) R[l * S2 + tid] = Bb[l * S2 + tid] - oc[l];
  }
  __syncthreads();
  // ---- δ = (⊗V) Λ^{-1} (⊗V)^T r_B (fast diagonalisation), x_B = X_c + δ ----
  auto Vax = [&](int a, int l, int j) { return toe[a] ? tp.v[l * S + j] : Vs[a * S2 + l * S + j]; };
  auto Lax = [&](int a, int j) { return toe[a] ? tp.lam[j] : Ls[a * S + j]; };
  if constexpr (S == 3) {                                         // 27 values: one warp, shuffles
    if (tid < 32) {
      const int li = tid < 27 ? tid : 0;
      const int fx = li % 3, fy = (li / 3) % 3, fz = li / 9;
      double v = tid < 27 ? R[li] : 0.0;
      auto src = [&](int ax, int l) { return ax == 0 ? fz * 9 + fy * 3 + l : (ax == 1 ? fz * 9 + l * 3 + fx : l * 9 + fy * 3 + fx); };
      auto step = [&](int ax, bool trans) {
        const int j = ax == 0 ? fx : (ax == 1 ? fy : fz);
        double o = 0.0;
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          const double in = __shfl_sync(0xffffffffu, v, src(ax, l));
          o = fma(trans ? Vax(ax, l, j) : Vax(ax, j, l), in, o);
        }
        v = o;
      };
      step(0, true);
      step(1, true);
      step(2, true);
      v /= (Lax(0, fx) + Lax(1, fy) + Lax(2, fz));
      step(2, false);
      step(1, false);
      step(0, false);
      const int gx = cc[0] - w + fx, gy = cc[1] - w + fy, gz = cc[2] - w + fz;
      if (tid < 27 && unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un)
        x[(int64_t(gz - zoff) * n1 + gy) * n1 + gx] = Xc[(fz * S + fy) * S + fx] + v;
    }
  } else {
    const int r = tid;
    const bool act = tid < S3;
    if (act) {                                                    // along x (transposed)
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(Vax(0, l, lx), R[r - lx + l], a0);
      Q[r] = a0;
    }
    __syncthreads();
    if (act) {                                                    // along y (transposed)
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(Vax(1, l, ly), Q[(lz * S + l) * S + lx], a0);
      R[r] = a0;
    }
    __syncthreads();
    if (act) {                                                    // along z (transposed), / (λx + λy + λz)
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(Vax(2, l, lz), R[(l * S + ly) * S + lx], a0);
      Q[r] = a0 / (Lax(0, lx) + Lax(1, ly) + Lax(2, lz));
    }
    __syncthreads();
    if (act) {                                                    // along z
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(Vax(2, lz, l), Q[(l * S + ly) * S + lx], a0);
      R[r] = a0;
    }
    __syncthreads();
    if (act) {                                                    // along y
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(Vax(1, ly, l), R[(lz * S + l) * S + lx], a0);
      Q[r] = a0;
    }
    __syncthreads();
    if (act) {                                                    // along x, and x_B += δ
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(Vax(0, lx, l), Q[r - lx + l], a0);
      const int gx = cc[0] - w + lx, gy = cc[1] - w + ly, gz = cc[2] - w + lz;
      if (unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un)
        x[(int64_t(gz - zoff) * n1 + gy) * n1 + gx] = Xc[r] + a0;
    }
  }
}

// ---------------- v5: one WARP per block, window planes streamed in groups of G -----------------------
// The same block step as v4 (r_B = b_B - (A x)_B by pencil passes x, y, z; δ by fast diagonalisation;
// x_B += δ), reorganised so that a block needs ~10 KB of shared memory and no CTA barrier:
//  * the window is read plane group by plane group straight from global memory (L2) into registers,
//    one x-row per lane ((plane, row) tasks), never staged whole;
//  * pass x -> Pa/Pb [S][G*Wn] (l-major: conflict-free stores), pass y per (plane, lx) pencil -> Pc/Pe
//    [G][S][S] (aliasing Pa/Pb), pass z ACCUMULATES the group's planes into r[lz] held by lane (lx, ly);
//  * on Toeplitz axes (A27) the symmetric band (k[t] = k[2p-t]) is applied to pair sums
//    v[l+t] + v[l+2p-t] shared by K and M: 5 adds + 12 FMAs per output instead of 22 FMAs (p = 5);
//  * the fast diagonalisation keeps (lx, ly) lanes with their S values of z in registers (the z
//    transforms are register-local; x and y exchange through two 125-value buffers).
// Smem offsets: conflict-free strides for the pass-y reads (TXP) and writes (PS); see the search below.
template <int P, int S, int G>
struct BW {
  static constexpr int W = 2 * P + 1, Wn = S + 2 * P, w = (S - 1) / 2, S2 = S * S, S3 = S2 * S;
  static constexpr int NG = Wn / G, TX = G * Wn, RX = (TX + 31) / 32, TY = G * S;
  static_assert(Wn % G == 0 && TY <= 32 && S2 <= 32, "group shape");
  static constexpr bool ok_txp(int t) {
    for (int h = 0; h < 2; ++h)
      for (int i = 16 * h; i < 16 * h + 16 && i < TY; ++i)
        for (int k = i + 1; k < 16 * h + 16 && k < TY; ++k)
          if (((i % S) * t + (i / S) * Wn) % 16 == ((k % S) * t + (k / S) * Wn) % 16) return false;
    return true;
  }
  static constexpr int find_txp() {
    for (int t = TX; t < TX + 64; ++t)
      if (ok_txp(t)) return t;
    return TX;
  }
  static constexpr int TXP = find_txp();
  static constexpr int PS = S2 + ((S - S2 % 16) % 16 + 16) % 16;           // PS = S (mod 16), >= S2
  static constexpr int AREA = (2 * S * TXP > 2 * G * PS ? 2 * S * TXP : 2 * G * PS);
  static constexpr int TAB = (6 * S * W > 2 * S3 ? 6 * S * W : 2 * S3);   // Tk, Tm | F0, F1
  static constexpr int OPA = 0, OPB = S * TXP, OPC = 0, OPE = G * PS, OT = AREA, OF = AREA,
                       OVS = AREA + TAB, OLS = OVS + 3 * S2;
  static constexpr int PERW = ((OLS + 3 * S + 1) / 2) * 2;                 // doubles per warp (16-byte multiple)
};

template <int P, int S, bool TOE>
__device__ __forceinline__ void w_pass_x(const double (&v)[S + 2 * P], const double *Tk, const double *Tm,
                                         const ToeP &tp, double *a, double *bo, int ostride) {
  constexpr int W = 2 * P + 1;
#pragma unroll
  for (int l = 0; l < S; ++l) {
    if constexpr (TOE) {
      double ka = tp.k[P] * v[l + P], ma = tp.m[P] * v[l + P];
#pragma unroll
      for (int t = 0; t < P; ++t) {
        const double s2 = v[l + t] + v[l + 2 * P - t];
        ka = fma(tp.k[t], s2, ka);
        ma = fma(tp.m[t], s2, ma);
      }
      a[l * ostride] = ka;
      bo[l * ostride] = ma;
    } else {
      double ka = 0.0, ma = 0.0;
#pragma unroll
      for (int t = 0; t < W; ++t) {
        ka = fma(Tk[l * W + t], v[l + t], ka);
        ma = fma(Tm[l * W + t], v[l + t], ma);
      }
      a[l * ostride] = ka;
      bo[l * ostride] = ma;
    }
  }
}

// pass y of one (plane, lx) pencil: Pc = My Pa + Ky Pb, Pe = My Pb
template <int P, int S, bool TOE>
__device__ __forceinline__ void w_pass_y(const double (&pa)[S + 2 * P], const double (&pb)[S + 2 * P], const double *Tk,
                                         const double *Tm, const ToeP &tp, double *oc, double *oe) {
  constexpr int W = 2 * P + 1;
#pragma unroll
  for (int l = 0; l < S; ++l) {
    if constexpr (TOE) {
      double c = tp.m[P] * pa[l + P], e = tp.m[P] * pb[l + P];
      c = fma(tp.k[P], pb[l + P], c);
#pragma unroll
      for (int t = 0; t < P; ++t) {
        const double sa = pa[l + t] + pa[l + 2 * P - t], sb = pb[l + t] + pb[l + 2 * P - t];
        c = fma(tp.m[t], sa, c);
        c = fma(tp.k[t], sb, c);
        e = fma(tp.m[t], sb, e);
      }
      oc[l * S] = c;
      oe[l * S] = e;
    } else {
      double c = 0.0, e = 0.0;
#pragma unroll
      for (int t = 0; t < W; ++t) {
        c = fma(Tm[l * W + t], pa[l + t], c);
        c = fma(Tk[l * W + t], pb[l + t], c);
        e = fma(Tm[l * W + t], pb[l + t], e);
      }
      oc[l * S] = c;
      oe[l * S] = e;
    }
  }
}

template <int P, int S, int G, int NW, int MINB, int LV>
__global__ void __launch_bounds__(32 * NW, MINB) k_schwarz3d_w(int n1, const double *__restrict__ K, const double *__restrict__ M,
                                                        const double *__restrict__ Vt, const double *__restrict__ lamt,
                                                        const double *__restrict__ b, double *__restrict__ x, int c0,
                                                        int c1, int c2, int D, int nb0, int nb1, int nblk, int zoff,
                                                        int tlo, int thi, const ToeP tp) {
  using B = BW<P, S, G>;
  constexpr int W = B::W, Wn = B::Wn, w = B::w, S2 = B::S2, TXP = B::TXP, PS = B::PS;
  extern __shared__ __align__(16) double smw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j0 = blockIdx.x * NW + wid;                           // grid (ceil(nb0 / NW), nb1, nb2)
  if (j0 >= nb0) return;                                          // the whole warp: no CTA barrier is used
  double *sw = smw + wid * B::PERW;
  double *Pa = sw + B::OPA, *Pb = sw + B::OPB, *Pc = sw + B::OPC, *Pe = sw + B::OPE;
  double *Tk = sw + B::OT, *Tm = sw + B::OT + 3 * S * W, *F0 = sw + B::OF, *F1 = sw + B::OF + B::S3;
  double *Vs = sw + B::OVS, *Ls = sw + B::OLS;
  const unsigned un = unsigned(n1);
  const int cc[3] = {c0 + D * j0, c1 + D * int(blockIdx.y), c2 + D * int(blockIdx.z)};
  const bool tv = tp.valid != 0;
  bool toe[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) toe[a] = tv && cc[a] - w >= tlo && cc[a] + w <= thi;
  const int ox = cc[0] - w - P, oy = cc[1] - w - P, oz = cc[2] - w - P;
  const bool xin = ox >= 0 && ox + Wn <= n1;
  // ---- band rows / FD tables of the boundary axes (zero rows outside the domain) ----
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (toe[a]) continue;
    for (int i = lane; i < S * W; i += 32) {
      const int l = i / W, t = i - l * W, gr = cc[a] - w + l;
      const bool ok = unsigned(gr) < un;
      Tk[a * S * W + i] = ok ? K[int64_t(gr) * W + t] : 0.0;
      Tm[a * S * W + i] = ok ? M[int64_t(gr) * W + t] : 0.0;
    }
    for (int i = lane; i < S2; i += 32) Vs[a * S2 + i] = Vt[int64_t(cc[a]) * S2 + i];
    if (lane < S) Ls[a * S + lane] = lamt[int64_t(cc[a]) * S + lane];
  }
  // ---- this lane's FD / update points (lx, ly, 0..S-1) and b_B there ----
  const bool vl = lane < S2;
  const int lx = vl ? lane % S : 0, ly = vl ? lane / S : 0;
  const int gx = cc[0] - w + lx, gy = cc[1] - w + ly;
  const bool xyok = vl && unsigned(gx) < un && unsigned(gy) < un;
  __syncwarp();
  double r[S];
#pragma unroll
  for (int lz = 0; lz < S; ++lz) r[lz] = 0.0;
  asm volatile("griddepcontrol.wait;" ::: "memory");              // PDL: the previous colour's x (no-op otherwise)
  // x-row of pass-x task t of group gi (zero outside the domain)
  // pass-x task t of group gi: window row (plane gi G + t / Wn, row t % Wn) -> Pa, Pb.  Rows inside the
  // domain in y and z, with the whole window inside in x (every interior block): LV-double vector loads and
  // the parity shift; rows outside the domain give zero rows (no loads).
  auto task_x = [&](int gi, int t) {
    const int jj = t / Wn, yy = t - jj * Wn;
    const int gz = oz + gi * G + jj, gyy = oy + yy;
    const bool rok = unsigned(gz) < un && unsigned(gyy) < un;
    const int64_t e0 = (int64_t(gz - zoff) * n1 + gyy) * n1 + ox;
    double v[Wn];
    if (rok && xin && LV > 1) {
      constexpr int NV = (Wn + 2 * LV - 2) / LV;                  // vectors covering [e0 & ~(LV-1), e0 + Wn)
      double u[NV * LV];
      const double *ap = x + (e0 & ~int64_t(LV - 1));
      const int sh = int(e0 & (LV - 1));
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        if constexpr (LV == 4) {
          asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                       : "=d"(u[4 * c]), "=d"(u[4 * c + 1]), "=d"(u[4 * c + 2]), "=d"(u[4 * c + 3])
                       : "l"(ap + 4 * c));
        } else {
          const double2 q = __ldg(reinterpret_cast<const double2 *>(ap) + c);
          u[2 * c] = q.x;
          u[2 * c + 1] = q.y;
        }
      }
      if constexpr (LV == 4) {
        double u2[Wn + 1];
#pragma unroll
        for (int k = 0; k < Wn + 1; ++k) u2[k] = (sh & 2) ? u[k + 2] : u[k];
#pragma unroll
        for (int k = 0; k < Wn; ++k) v[k] = (sh & 1) ? u2[k + 1] : u2[k];
      } else {
#pragma unroll
        for (int k = 0; k < Wn; ++k) v[k] = sh ? u[k + 1] : u[k];
      }
    } else if (rok) {
      const double *rp = x + e0;
#pragma unroll
      for (int k = 0; k < Wn; ++k) v[k] = (xin || unsigned(ox + k) < un) ? rp[k] : 0.0;
    } else {
#pragma unroll
      for (int l = 0; l < S; ++l) Pa[l * TXP + t] = Pb[l * TXP + t] = 0.0;
      return;
    }
    if (toe[0]) w_pass_x<P, S, true>(v, Tk, Tm, tp, Pa + t, Pb + t, TXP);
    else w_pass_x<P, S, false>(v, Tk, Tm, tp, Pa + t, Pb + t, TXP);
  };
#pragma unroll
  for (int gi = 0; gi < B::NG; ++gi) {
    // ---- pass x over the group's (plane, row) tasks: Pa = Kx X, Pb = Mx X ----
#pragma unroll 1
    for (int rr = 0; rr < B::RX; ++rr) {
      const int t = rr * 32 + lane;
      if (t < B::TX) task_x(gi, t);
    }
    __syncwarp();
    if (gi == 0) asm volatile("griddepcontrol.launch_dependents;");   // PDL: the next colour may launch
    // ---- pass y over the group's (plane, lx) pencils: Pc = My Pa + Ky Pb, Pe = My Pb (into Pa's area) ----
    {
      const bool act = lane < B::TY;
      const int jj = act ? lane / S : 0, px = act ? lane - jj * S : 0;   // idle lanes read pencil 0 (unused)
      const double *pap = Pa + px * TXP + jj * Wn, *pbp = Pb + px * TXP + jj * Wn;
      double pa[Wn], pb[Wn];
#pragma unroll
      for (int k = 0; k < Wn; ++k) {
        pa[k] = pap[k];
        pb[k] = pbp[k];
      }
      __syncwarp();
      if (act) {
        if (toe[1]) w_pass_y<P, S, true>(pa, pb, Tk + S * W, Tm + S * W, tp, Pc + jj * PS + px, Pe + jj * PS + px);
        else w_pass_y<P, S, false>(pa, pb, Tk + S * W, Tm + S * W, tp, Pc + jj * PS + px, Pe + jj * PS + px);
      }
    }
    __syncwarp();
    // ---- pass z: r[lz] += Mz[lz][j-lz] Pc_j + Kz[lz][j-lz] Pe_j over the group's planes j ----
    if (vl) {
      if (toe[2]) {
#pragma unroll
        for (int jj = 0; jj < G; ++jj) {
          const double pc = Pc[jj * PS + lane], pe = Pe[jj * PS + lane];
#pragma unroll
          for (int lz = 0; lz < S; ++lz) {
            const int t = gi * G + jj - lz;
            if (t >= 0 && t < W) r[lz] = fma(tp.k[t], pe, fma(tp.m[t], pc, r[lz]));
          }
        }
      } else {
        const double *tk = Tk + 2 * S * W, *tm = Tm + 2 * S * W;
#pragma unroll
        for (int jj = 0; jj < G; ++jj) {
          const double pc = Pc[jj * PS + lane], pe = Pe[jj * PS + lane];
#pragma unroll
          for (int lz = 0; lz < S; ++lz) {
            const int t = gi * G + jj - lz;
            if (t >= 0 && t < W) r[lz] = fma(tk[lz * W + t], pe, fma(tm[lz * W + t], pc, r[lz]));
          }
        }
      }
    }
    __syncwarp();
  }
  // ---- δ = (⊗V) Λ^{-1} (⊗V)^T (b_B - r), x_B += δ ----
  // this lane's FD operands (x, y), loaded once: Toeplitz axes from the kernel parameter (A27), others from Vs, Ls
  double vxt[S], vxn[S], vyt[S], vyn[S], lxy = 0.0;
  if (toe[0]) {
#pragma unroll
    for (int l = 0; l < S; ++l) { vxt[l] = tp.v[l * S + lx]; vxn[l] = tp.v[lx * S + l]; }
    lxy = tp.lam[lx];
  } else {
#pragma unroll
    for (int l = 0; l < S; ++l) { vxt[l] = Vs[l * S + lx]; vxn[l] = Vs[lx * S + l]; }
    lxy = Ls[lx];
  }
  if (toe[1]) {
#pragma unroll
    for (int l = 0; l < S; ++l) { vyt[l] = tp.v[l * S + ly]; vyn[l] = tp.v[ly * S + l]; }
    lxy += tp.lam[ly];
  } else {
#pragma unroll
    for (int l = 0; l < S; ++l) { vyt[l] = Vs[S2 + l * S + ly]; vyn[l] = Vs[S2 + ly * S + l]; }
    lxy += Ls[S + ly];
  }
  // z: the lane's S values are register-local; V_z, λ_z are uniform (constant bank when Toeplitz)
  auto zfd = [&](auto vz, auto lz_, const double (&qi)[S], double (&qo)[S]) {
    double q3[S];
#pragma unroll
    for (int j = 0; j < S; ++j) {
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(vz(l, j), qi[l], a0);
      q3[j] = a0 / (lxy + lz_(j));
    }
#pragma unroll
    for (int lz = 0; lz < S; ++lz) {
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(vz(lz, l), q3[l], a0);
      qo[lz] = a0;
    }
  };
  // the block's points of this lane: column (gx, gy), planes cc[2] - w + lz
  const int64_t col0 = (int64_t(cc[2] - w - zoff) * n1 + gy) * n1 + gx, pl = int64_t(n1) * n1;
  double q[S];
  if (vl) {
#pragma unroll
    for (int lz = 0; lz < S; ++lz) {
      const int gz = cc[2] - w + lz;
      const double bz = (xyok && unsigned(gz) < un) ? b[col0 + lz * pl] : 0.0;
      F0[lz * S2 + lane] = bz - r[lz];
    }
  }
  __syncwarp();
  if (vl) {                                                       // along x (transposed)
#pragma unroll
    for (int lz = 0; lz < S; ++lz) {
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(vxt[l], F0[lz * S2 + ly * S + l], a0);
      F1[lz * S2 + lane] = a0;
    }
  }
  __syncwarp();
  if (vl) {                                                       // along y (transposed), z (transposed), Λ^{-1}, z
#pragma unroll
    for (int lz = 0; lz < S; ++lz) {
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(vyt[l], F1[lz * S2 + l * S + lx], a0);
      q[lz] = a0;
    }
    double qo[S];
    if (toe[2]) zfd([&](int l, int j) { return tp.v[l * S + j]; }, [&](int j) { return tp.lam[j]; }, q, qo);
    else zfd([&](int l, int j) { return Vs[2 * S2 + l * S + j]; }, [&](int j) { return Ls[2 * S + j]; }, q, qo);
#pragma unroll
    for (int lz = 0; lz < S; ++lz) F0[lz * S2 + lane] = qo[lz];   // F0's last reads were before the barrier above
  }
  __syncwarp();
  if (vl) {                                                       // along y
#pragma unroll
    for (int lz = 0; lz < S; ++lz) {
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(vyn[l], F0[lz * S2 + l * S + lx], a0);
      F1[lz * S2 + lane] = a0;                                    // F1's last reads: two barriers ago
    }
  }
  __syncwarp();
  if (xyok) {                                                     // along x, and x_B += δ
#pragma unroll
    for (int lz = 0; lz < S; ++lz) {
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(vxn[l], F1[lz * S2 + ly * S + l], a0);
      if (unsigned(cc[2] - w + lz) < un) {
        double *xp = x + col0 + lz * pl;
        *xp = *xp + a0;
      }
    }
  }
}

// ---- 3D Schwarz colour kernel, z-chain variant (IGA2L_S3D_CHAIN = L > 0) ----
// For s = p (both 3D configs) the window length Wn = s + 2p is 3G and the colour spacing D = s + p is 2G with
// G = (s + p) / 2: the windows of the same-colour blocks (cx, cy, c2 + D k) along z overlap by one plane group
// (planes oz_k + 2G .. oz_k + 3G are the first group of block k + 1).  One warp runs a segment of L such blocks
// in ascending z: every plane group passes x and y once and its pass z accumulates into the one or two blocks
// whose window holds it (2L + 1 groups per segment instead of 3L; the pass-x/y arithmetic and the per-point
// operation order are those of k_schwarz3d_w, so the result is bitwise equal).  A block's update is written as
// soon as its last group is accumulated: no later group of the segment reads its points (A4: a same-colour
// window never holds another block's points), so the segment order is free.  z band rows / FD tables of
// non-Toeplitz blocks sit in two slots (block parity); the solve buffers F0/F1 overlay the pass buffers, not the
// tables (the x/y tables serve every block of the segment).
template <int P, int S, int GP>
struct BZ {
  static constexpr int G = (S + P) / 2, W = 2 * P + 1, Wn = S + 2 * P, w = (S - 1) / 2, S2 = S * S, S3 = S2 * S;
  static_assert(Wn == 3 * G && (GP == G || GP == 2 * G), "z-chain needs s = p");
  static constexpr int TX = GP * Wn, TY = GP * S;
  static_assert(TY <= 32 && S2 <= 32, "group shape");
  static constexpr bool ok_txp(int t) {
    for (int h = 0; h < 2; ++h)
      for (int i = 16 * h; i < 16 * h + 16 && i < TY; ++i)
        for (int k = i + 1; k < 16 * h + 16 && k < TY; ++k)
          if (((i % S) * t + (i / S) * Wn) % 16 == ((k % S) * t + (k / S) * Wn) % 16) return false;
    return true;
  }
  static constexpr int find_txp() {
    for (int t = TX; t < TX + 64; ++t)
      if (ok_txp(t)) return t;
    return TX;
  }
  static constexpr int TXP = find_txp();
  static constexpr int PS = S2 + ((S - S2 % 16) % 16 + 16) % 16;
  static constexpr int A1 = (2 * S * TXP > 2 * GP * PS ? 2 * S * TXP : 2 * GP * PS);
  static constexpr int AREA = (A1 > 2 * S3 ? A1 : 2 * S3);   // Pa/Pb | Pc/Pe | F0/F1 (the solve's buffers)
  static constexpr int OPA = 0, OPB = S * TXP, OPC = 0, OPE = GP * PS, OF = 0;
  static constexpr int OT = AREA;                           // Tk[4 S W]: x, y, z slot 0, z slot 1; Tm after it
  static constexpr int OTM = OT + 4 * S * W, OVS = OTM + 4 * S * W, OLS = OVS + 4 * S2;
  static constexpr int PERW = ((OLS + 4 * S + 1) / 2) * 2;
};

template <int P, int S, int GP, int NW, int MINB, int LV>
__global__ void __launch_bounds__(32 * NW, MINB) k_schwarz3d_zc(int n1, const double *__restrict__ K, const double *__restrict__ M,
                                                         const double *__restrict__ Vt, const double *__restrict__ lamt,
                                                         const double *__restrict__ b, double *__restrict__ x, int c0,
                                                         int c1, int c2, int D, int nb0, int nb2, int L, int zoff,
                                                         int tlo, int thi, const ToeP tp) {
  using Z = BZ<P, S, GP>;
  constexpr int G = Z::G, W = Z::W, Wn = Z::Wn, w = Z::w, S2 = Z::S2, TXP = Z::TXP, PS = Z::PS;
  extern __shared__ __align__(16) double smw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j0 = blockIdx.x * NW + wid;
  if (j0 >= nb0) return;                                          // the whole warp: no CTA barrier is used
  double *sw = smw + wid * Z::PERW;
  double *Pa = sw + Z::OPA, *Pb = sw + Z::OPB, *Pc = sw + Z::OPC, *Pe = sw + Z::OPE;
  double *Tk = sw + Z::OT, *Tm = sw + Z::OTM, *F0 = sw + Z::OF, *F1 = sw + Z::OF + Z::S3;
  double *Vs = sw + Z::OVS, *Ls = sw + Z::OLS;
  const unsigned un = unsigned(n1);
  const int k0 = int(blockIdx.z) * L, k1 = min(nb2, k0 + L);       // segment blockIdx.z: L blocks (the last short)
  const int cx = c0 + D * j0, cy = c1 + D * int(blockIdx.y);
  const bool tv = tp.valid != 0;
  const bool toex = tv && cx - w >= tlo && cx + w <= thi, toey = tv && cy - w >= tlo && cy + w <= thi;
  const int ox = cx - w - P, oy = cy - w - P;
  const bool xin = ox >= 0 && ox + Wn <= n1;
  // band rows / FD tables of a boundary axis a (0, 1; z: 2 + slot) centred at c
  auto load_tab = [&](int a, int c) {
    for (int i = lane; i < S * W; i += 32) {
      const int l = i / W, t = i - l * W, gr = c - w + l;
      const bool ok = unsigned(gr) < un;
      Tk[a * S * W + i] = ok ? K[int64_t(gr) * W + t] : 0.0;
      Tm[a * S * W + i] = ok ? M[int64_t(gr) * W + t] : 0.0;
    }
    for (int i = lane; i < S2; i += 32) Vs[a * S2 + i] = Vt[int64_t(c) * S2 + i];
    if (lane < S) Ls[a * S + lane] = lamt[int64_t(c) * S + lane];
  };
  auto toe_z = [&](int k) { const int cz = c2 + D * k; return tv && cz - w >= tlo && cz + w <= thi; };
  if (!toex) load_tab(0, cx);
  if (!toey) load_tab(1, cy);
  if (!toe_z(k0)) load_tab(2, c2 + D * k0);
  const bool vl = lane < S2;
  const int lx = vl ? lane % S : 0, ly = vl ? lane / S : 0;
  const int gx = cx - w + lx, gy = cy - w + ly;
  const bool xyok = vl && unsigned(gx) < un && unsigned(gy) < un;
  __syncwarp();
  asm volatile("griddepcontrol.wait;" ::: "memory");              // PDL: the previous colour's x (no-op otherwise)
  // pass x and y of NP (compile time) planes from absolute plane gzb: Pc/Pe[jj][lane] for the column (lx, ly)
  auto group_xy = [&](auto NPc, int gzb) {
    constexpr int NP = decltype(NPc)::value, TX = NP * Wn, RX = (TX + 31) / 32, TY = NP * S;
    auto task_x = [&](int t) {
      const int jj = t / Wn, yy = t - jj * Wn;
      const int gz = gzb + jj, gyy = oy + yy;
      const bool rok = unsigned(gz) < un && unsigned(gyy) < un;
      const int64_t e0 = (int64_t(gz - zoff) * n1 + gyy) * n1 + ox;
      double v[Wn];
      if (rok && xin && LV > 1) {
        constexpr int NV = (Wn + 2 * LV - 2) / LV;
        double u[NV * LV];
        const double *ap = x + (e0 & ~int64_t(LV - 1));
        const int sh = int(e0 & (LV - 1));
#pragma unroll
        for (int c = 0; c < NV; ++c) {
          if constexpr (LV == 4) {
            asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(u[4 * c]), "=d"(u[4 * c + 1]), "=d"(u[4 * c + 2]), "=d"(u[4 * c + 3])
                         : "l"(ap + 4 * c));
          } else {
            const double2 q = __ldg(reinterpret_cast<const double2 *>(ap) + c);
            u[2 * c] = q.x;
            u[2 * c + 1] = q.y;
          }
        }
        if constexpr (LV == 4) {
          double u2[Wn + 1];
#pragma unroll
          for (int k = 0; k < Wn + 1; ++k) u2[k] = (sh & 2) ? u[k + 2] : u[k];
#pragma unroll
          for (int k = 0; k < Wn; ++k) v[k] = (sh & 1) ? u2[k + 1] : u2[k];
        } else {
#pragma unroll
          for (int k = 0; k < Wn; ++k) v[k] = sh ? u[k + 1] : u[k];
        }
      } else if (rok) {
        const double *rp = x + e0;
#pragma unroll
        for (int k = 0; k < Wn; ++k) v[k] = (xin || unsigned(ox + k) < un) ? rp[k] : 0.0;
      } else {
#pragma unroll
        for (int l = 0; l < S; ++l) Pa[l * TXP + t] = Pb[l * TXP + t] = 0.0;
        return;
      }
      if (toex) w_pass_x<P, S, true>(v, Tk, Tm, tp, Pa + t, Pb + t, TXP);
      else w_pass_x<P, S, false>(v, Tk, Tm, tp, Pa + t, Pb + t, TXP);
    };
#pragma unroll 1
    for (int rr = 0; rr < RX; ++rr) {
      const int t = rr * 32 + lane;
      if (t < TX) task_x(t);
    }
    __syncwarp();
    const bool act = lane < TY;
    const int jj = act ? lane / S : 0, px = act ? lane - jj * S : 0;
    const double *pap = Pa + px * TXP + jj * Wn, *pbp = Pb + px * TXP + jj * Wn;
    double pa[Wn], pb[Wn];
#pragma unroll
    for (int k = 0; k < Wn; ++k) {
      pa[k] = pap[k];
      pb[k] = pbp[k];
    }
    __syncwarp();
    if (act) {
      if (toey) w_pass_y<P, S, true>(pa, pb, Tk + S * W, Tm + S * W, tp, Pc + jj * PS + px, Pe + jj * PS + px);
      else w_pass_y<P, S, false>(pa, pb, Tk + S * W, Tm + S * W, tp, Pc + jj * PS + px, Pe + jj * PS + px);
    }
    __syncwarp();
  };
  // pass z of the NP planes just passed into r: plane jj is window plane R + jj of r's block (compile time)
  auto acc_z = [&](auto NPc, auto Rc, double (&r)[S], bool toe, int slot) {
    constexpr int NP = decltype(NPc)::value, R = decltype(Rc)::value;
    if (!vl) return;
    if (toe) {
#pragma unroll
      for (int jj = 0; jj < NP; ++jj) {
        if (R + jj < 0 || R + jj - (S - 1) >= W) continue;
        const double pc = Pc[jj * PS + lane], pe = Pe[jj * PS + lane];
#pragma unroll
        for (int lz = 0; lz < S; ++lz) {
          const int t = R + jj - lz;
          if (t >= 0 && t < W) r[lz] = fma(tp.k[t], pe, fma(tp.m[t], pc, r[lz]));
        }
      }
    } else {
      const double *tk = Tk + (2 + slot) * S * W, *tm = Tm + (2 + slot) * S * W;
#pragma unroll
      for (int jj = 0; jj < NP; ++jj) {
        if (R + jj < 0 || R + jj - (S - 1) >= W) continue;
        const double pc = Pc[jj * PS + lane], pe = Pe[jj * PS + lane];
#pragma unroll
        for (int lz = 0; lz < S; ++lz) {
          const int t = R + jj - lz;
          if (t >= 0 && t < W) r[lz] = fma(tk[lz * W + t], pe, fma(tm[lz * W + t], pc, r[lz]));
        }
      }
    }
  };
  // δ = (⊗V) Λ^{-1} (⊗V)^T (b_B - r), x_B += δ for block k (z tables in slot); F0/F1 overlay Pa..Pe
  auto solve = [&](int k, const double (&r)[S], bool toe, int slot) {
    const int cz = c2 + D * k;
    double vxt[S], vxn[S], vyt[S], vyn[S], lxy = 0.0;
    if (toex) {
#pragma unroll
      for (int l = 0; l < S; ++l) { vxt[l] = tp.v[l * S + lx]; vxn[l] = tp.v[lx * S + l]; }
      lxy = tp.lam[lx];
    } else {
#pragma unroll
      for (int l = 0; l < S; ++l) { vxt[l] = Vs[l * S + lx]; vxn[l] = Vs[lx * S + l]; }
      lxy = Ls[lx];
    }
    if (toey) {
#pragma unroll
      for (int l = 0; l < S; ++l) { vyt[l] = tp.v[l * S + ly]; vyn[l] = tp.v[ly * S + l]; }
      lxy += tp.lam[ly];
    } else {
#pragma unroll
      for (int l = 0; l < S; ++l) { vyt[l] = Vs[S2 + l * S + ly]; vyn[l] = Vs[S2 + ly * S + l]; }
      lxy += Ls[S + ly];
    }
    const int64_t col0 = (int64_t(cz - w - zoff) * n1 + gy) * n1 + gx, pl = int64_t(n1) * n1;
    if (vl) {
#pragma unroll
      for (int lz = 0; lz < S; ++lz) {
        const int gz = cz - w + lz;
        const double bz = (xyok && unsigned(gz) < un) ? b[col0 + lz * pl] : 0.0;
        F0[lz * S2 + lane] = bz - r[lz];
      }
    }
    __syncwarp();
    if (vl) {
#pragma unroll
      for (int lz = 0; lz < S; ++lz) {
        double a0 = 0.0;
#pragma unroll
        for (int l = 0; l < S; ++l) a0 = fma(vxt[l], F0[lz * S2 + ly * S + l], a0);
        F1[lz * S2 + lane] = a0;
      }
    }
    __syncwarp();
    auto zfd = [&](auto vz, auto lz_, const double (&qi)[S], double (&qo)[S]) {
      double q3[S];
#pragma unroll
      for (int j = 0; j < S; ++j) {
        double a0 = 0.0;
#pragma unroll
        for (int l = 0; l < S; ++l) a0 = fma(vz(l, j), qi[l], a0);
        q3[j] = a0 / (lxy + lz_(j));
      }
#pragma unroll
      for (int lz = 0; lz < S; ++lz) {
        double a0 = 0.0;
#pragma unroll
        for (int l = 0; l < S; ++l) a0 = fma(vz(lz, l), q3[l], a0);
        qo[lz] = a0;
      }
    };
    if (vl) {
      double q[S], qo[S];
#pragma unroll
      for (int lz = 0; lz < S; ++lz) {
        double a0 = 0.0;
#pragma unroll
        for (int l = 0; l < S; ++l) a0 = fma(vyt[l], F1[lz * S2 + l * S + lx], a0);
        q[lz] = a0;
      }
      if (toe) zfd([&](int l, int j) { return tp.v[l * S + j]; }, [&](int j) { return tp.lam[j]; }, q, qo);
      else {
        const double *vz = Vs + (2 + slot) * S2, *lzs = Ls + (2 + slot) * S;
        zfd([&](int l, int j) { return vz[l * S + j]; }, [&](int j) { return lzs[j]; }, q, qo);
      }
#pragma unroll
      for (int lz = 0; lz < S; ++lz) F0[lz * S2 + lane] = qo[lz];   // F0's last reads were before the barrier above
    }
    __syncwarp();
    if (vl) {
#pragma unroll
      for (int lz = 0; lz < S; ++lz) {
        double a0 = 0.0;
#pragma unroll
        for (int l = 0; l < S; ++l) a0 = fma(vyn[l], F0[lz * S2 + l * S + lx], a0);
        F1[lz * S2 + lane] = a0;
      }
    }
    __syncwarp();
    if (xyok) {
#pragma unroll
      for (int lz = 0; lz < S; ++lz) {
        double a0 = 0.0;
#pragma unroll
        for (int l = 0; l < S; ++l) a0 = fma(vxn[l], F1[lz * S2 + ly * S + l], a0);
        if (unsigned(cz - w + lz) < un) {
          double *xp = x + col0 + lz * pl;
          *xp = *xp + a0;
        }
      }
    }
    __syncwarp();                                                 // F1's reads are done before Pa/Pb are rewritten
  };
  using CG = std::integral_constant<int, G>;
  using CGP = std::integral_constant<int, GP>;
  double rc[S];
#pragma unroll
  for (int lz = 0; lz < S; ++lz) rc[lz] = 0.0;
  bool tc = toe_z(k0);
  if constexpr (GP == G) {
    // one loop over the segment's 2 (k1 - k0) + 1 plane groups (a single inlined copy of the passes): group g
    // is plane group g / 2 of block k0 + g / 2 - 1 (even g > 0: its last, R = 2G) and the first of block
    // k0 + g / 2 (even g, R = 0); odd g is the middle group (R = G) of block k0 + (g - 1) / 2
    const int ng = 2 * (k1 - k0) + 1, oz0 = c2 + D * k0 - w - P;
    bool tn = false;
#pragma unroll 1
    for (int g = 0; g < ng; ++g) {
      group_xy(CG{}, oz0 + g * G);
      if (g == 0) asm volatile("griddepcontrol.launch_dependents;");   // PDL: the next colour may launch
      const int j = (g - 1) >> 1, k = k0 + j, slot = j & 1;       // the block whose middle / last group this is
      if (g & 1) {
        acc_z(CG{}, CG{}, rc, tc, slot);
        tn = k + 1 < k1 && toe_z(k + 1);
        if (k + 1 < k1 && !tn) load_tab(2 + (slot ^ 1), c2 + D * (k + 1));   // its last reader was block k - 1
        __syncwarp();
      } else {
        double rn[S];
        if (g > 0) acc_z(CG{}, std::integral_constant<int, 2 * G>{}, rc, tc, slot);
#pragma unroll
        for (int lz = 0; lz < S; ++lz) rn[lz] = 0.0;
        if (g < ng - 1) acc_z(CG{}, std::integral_constant<int, 0>{}, rn, g > 0 ? tn : tc, g > 0 ? slot ^ 1 : 0);
        __syncwarp();
        if (g > 0) {
          solve(k, rc, tc, slot);
          tc = tn;
        }
#pragma unroll
        for (int lz = 0; lz < S; ++lz) rc[lz] = rn[lz];
      }
    }
    return;
  }
  // GP == 2G (p = 3 shape): the first group of G planes, then per block one group of 2G planes (oz + G .. oz + 3G)
  group_xy(CG{}, c2 + D * k0 - w - P);
  asm volatile("griddepcontrol.launch_dependents;");              // PDL: the next colour may launch
  acc_z(CG{}, std::integral_constant<int, 0>{}, rc, tc, 0);
  __syncwarp();
#pragma unroll 1
  for (int k = k0; k < k1; ++k) {
    const int slot = (k - k0) & 1, oz = c2 + D * k - w - P;
    const bool nx = k + 1 < k1;
    const bool tn = nx && toe_z(k + 1);
    double rn[S];
    if (nx && !tn) load_tab(2 + (slot ^ 1), c2 + D * (k + 1));   // the other slot: its last reader was block k-1
    group_xy(CGP{}, oz + G);
    acc_z(CGP{}, CG{}, rc, tc, slot);
#pragma unroll
    for (int lz = 0; lz < S; ++lz) rn[lz] = 0.0;
    if (nx) acc_z(CGP{}, std::integral_constant<int, -G>{}, rn, tn, slot ^ 1);
    __syncwarp();
    solve(k, rc, tc, slot);
#pragma unroll
    for (int lz = 0; lz < S; ++lz) rc[lz] = rn[lz];
    tc = tn;
  }
}

// IGA2L_S3D_TMA=0: window by cp.async rows.  Read per launch (tests switch it within one process).
inline bool env_on(const char *name) {
  const char *e = std::getenv(name);
  return !(e && e[0] == '0');
}
template <int P, int S>
bool try_schwarz3d(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                   const double *b, double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nb2, int zoff,
                   int tlo, int thi, cudaStream_t st, const ToeP *tpp) {
  if (p != P || s != S) return false;
  {
    using B = B4<P, S>;
    ToeP tp{};
    if (tpp) tp = *tpp;
    CUtensorMap me{}, mo{};
    const int w = (S - 1) / 2;
    const int64_t rows = (std::min<int64_t>(n1, c2 + int64_t(D) * (nb2 - 1) + w + P + 1) - zoff) * n1;   // stored rows
    if (B::TMA_OK && env_on("IGA2L_S3D_TMA") && rows >= 2 && make_tmap_rows_swz128(&me, x, n1, (rows + 1) / 2, 2 * n1, B::BOX, B::BR) &&
        make_tmap_rows_swz128(&mo, x + n1 - 1, n1 + 1, rows / 2, 2 * n1, B::BOX, B::BR)) {
      constexpr size_t sm = sizeof(double) * B::PERT + 16 + 1024;
      ensure_smem(k_schwarz3d_v4<P, S, true>, sm);
      k_schwarz3d_v4<P, S, true><<<nb0 * nb1 * nb2, B::NT, sm, st>>>(me, mo, int(n1), K, M, V, lam, b, x, c0, c1, c2,
                                                                     D, nb0, nb1, zoff, tlo, thi, tp);
    } else {
      constexpr size_t sm = sizeof(double) * B::PER + 16 + 1024;
      ensure_smem(k_schwarz3d_v4<P, S, false>, sm);
      k_schwarz3d_v4<P, S, false><<<nb0 * nb1 * nb2, B::NT, sm, st>>>(me, mo, int(n1), K, M, V, lam, b, x, c0, c1,
                                                                      c2, D, nb0, nb1, zoff, tlo, thi, tp);
    }
    return true;
  }
}

// launch of v5: NW warps (blocks) per CTA, at least MINB CTAs per SM, LV-double row loads
template <int P, int S, int G, int NW, int MINB, int LV>
void launch_w(int64_t n1, const double *K, const double *M, const double *V, const double *lam, const double *b,
              double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nblk, int zoff, int tlo, int thi,
              cudaStream_t st, const ToeP &tp) {
  constexpr size_t sm = sizeof(double) * BW<P, S, G>::PERW * NW;
  ensure_smem(k_schwarz3d_w<P, S, G, NW, MINB, LV>, sm);
  const char *e = std::getenv("IGA2L_PDL");
  if (!(e && e[0] == '0')) {                                   // programmatic dependent launch (as 2D)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((nb0 + NW - 1) / NW, nb1, nblk / (nb0 * nb1));
    cfg.blockDim = dim3(32 * NW);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_schwarz3d_w<P, S, G, NW, MINB, LV>, int(n1), K, M, V, lam, b, x, c0, c1, c2, D, nb0,
                           nb1, nblk, zoff, tlo, thi, tp) == cudaSuccess)
      return;
    cudaGetLastError();
  }
  k_schwarz3d_w<P, S, G, NW, MINB, LV><<<dim3((nb0 + NW - 1) / NW, nb1, nblk / (nb0 * nb1)), 32 * NW, sm, st>>>(
      int(n1), K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nblk, zoff, tlo, thi, tp);
}
// Segment length of the z-chain: a wave-quantised makespan model, ceil(warps / resident warp slots) waves of
// (2 L + 1) plane groups each.  C5 (nb = 26): L = 4, 7 segments, 4732 warps = two full waves (model 18 vs 24 for
// v5; measured 153.5 vs 162.7 us per colour, same box; L = 3 157.7, 2 161.6, 9 164.2, 5 170.2, 6 187.7).  Segments of
// near-equal length measured slower (169 us at 7 segments) and were dropped.
inline int zchain_length(int nb0, int nb1, int nb2) {
  static int slots = 0;
  if (!slots) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    slots = sms * 16;                                             // 4 CTAs x 4 warps per SM
  }
  const int64_t cols = int64_t(nb0) * nb1;
  int best = 1;
  int64_t bc = -1;
  for (int L = 1; L <= nb2; ++L) {
    const int64_t segs = (nb2 + L - 1) / L, c = ((cols * segs + slots - 1) / slots) * (2 * L + 1);
    if (bc < 0 || c < bc) { bc = c; best = L; }
  }
  return best;
}
// z-chain variant: NW warps per CTA, grid (ceil(nb0 / NW), nb1, ceil(nb2 / L)) for segments of L blocks, PDL as v5
template <int P, int S, int GP, int NW, int MINB, int LV>
void launch_zc(int64_t n1, const double *K, const double *M, const double *V, const double *lam, const double *b,
               double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nb2, int L, int zoff, int tlo, int thi,
               cudaStream_t st, const ToeP &tp) {
  constexpr size_t sm = sizeof(double) * BZ<P, S, GP>::PERW * NW;
  ensure_smem(k_schwarz3d_zc<P, S, GP, NW, MINB, LV>, sm);
  const dim3 grid((nb0 + NW - 1) / NW, nb1, (nb2 + L - 1) / L);
  const char *e = std::getenv("IGA2L_PDL");
  if (!(e && e[0] == '0')) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(32 * NW);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_schwarz3d_zc<P, S, GP, NW, MINB, LV>, int(n1), K, M, V, lam, b, x, c0, c1, c2, D, nb0,
                           nb2, L, zoff, tlo, thi, tp) == cudaSuccess)
      return;
    cudaGetLastError();
  }
  k_schwarz3d_zc<P, S, GP, NW, MINB, LV><<<grid, 32 * NW, sm, st>>>(int(n1), K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb2, L,
                                                                zoff, tlo, thi, tp);
}
// v5 (warp per block) for the shapes of the 3D configs; IGA2L_S3D_WARP=0 selects v4.  4 warps (blocks) per CTA,
// at most 128 registers (4 CTAs per SM).
template <int P, int S, int G>
bool try_schwarz3d_w(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                     const double *b, double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nb2, int zoff,
                     int tlo, int thi, cudaStream_t st, const ToeP *tpp) {
  if (p != P || s != S || !env_on("IGA2L_S3D_WARP")) return false;
  ToeP tp{};
  if (tpp) tp = *tpp;
  const int nblk = nb0 * nb1 * nb2;
  if constexpr (P == S) {
    // z-chain (IGA2L_S3D_CHAIN): "0" off, L > 0 segments of L blocks, unset / "auto": zchain_length's L at p = 5
    // (v5 measured faster at p = 3, C4: 25.6 vs 29.3 us per colour at the best L, same box)
    const char *ce = std::getenv("IGA2L_S3D_CHAIN");
    int L = 0;
    if (ce && ce[0] >= '0' && ce[0] <= '9') {
      L = std::atoi(ce);
    } else if (P == 5) {
      L = zchain_length(nb0, nb1, nb2);
      if (L <= 1) L = 0;                                          // one block per warp: v5 is that, faster
    }
    if (L > 0 && !(reinterpret_cast<uintptr_t>(x) & 31)) {
      constexpr int GZ = (S + P) / 2, GP = (2 * GZ * S <= 32 ? 2 * GZ : GZ);   // 2G-plane groups where they fit a warp
      const char *lv = std::getenv("IGA2L_S3D_CHAIN_LV");         // A/B: row load width (doubles)
      if (lv && lv[0] == '1')
        launch_zc<P, S, GP, 4, 4, 1>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, L, zoff, tlo, thi, st, tp);
      else if (lv && lv[0] == '4')
        launch_zc<P, S, GP, 4, 4, 4>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, L, zoff, tlo, thi, st, tp);
      else if (const char *nw = std::getenv("IGA2L_S3D_NW"); nw && nw[0] == '4')   // A/B: warps per CTA
        launch_zc<P, S, GP, 4, 4, (P == 5 ? 2 : 4)>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, L, zoff, tlo,
                                                   thi, st, tp);
      else if (nw && nw[0] == '1')
        launch_zc<P, S, GP, 1, 16, (P == 5 ? 2 : 4)>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, L, zoff, tlo,
                                                    thi, st, tp);
      else   // 2 warps per CTA: C5's 26 block columns fill 13 CTAs (4 per CTA leave 2 of 28 warp slots idle): 140.2 vs
             // 144.5 us per colour, same box (1 per CTA 143.2)
        launch_zc<P, S, GP, 2, 8, (P == 5 ? 2 : 4)>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, L, zoff, tlo,
                                                   thi, st, tp);
      return true;
    }
  }
  // 32-byte row loads need a 32-byte aligned x (every torch / cudaMalloc allocation is)
  // row loads: 16 bytes at p = 5 (170.5 vs 173.3 us per C5 colour with 32), 32 bytes at p = 3 (25.96 vs 26.20 us
  // per C4 colour); 8 bytes when x is not 32-byte aligned.  More CTAs per SM (96 / 80 registers) measured
  // slower (173.3 us).
  if (reinterpret_cast<uintptr_t>(x) & 31)
    launch_w<P, S, G, 4, 4, 1>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nblk, zoff, tlo, thi, st, tp);
  else
    launch_w<P, S, G, 4, 4, (P == 5 ? 2 : 4)>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nblk, zoff, tlo, thi,
                                               st, tp);
  return true;
}

}  // namespace

bool launch_schwarz3d_colour(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                             const double *lam, const double *b, double *x, int c0, int c1, int f2, int D, int nb0,
                             int nb1, int nb2, int zoff, int tlo, int thi, cudaStream_t st, const ToeP *tp) {
  if (try_schwarz3d_w<3, 3, 9>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st, tp) ||
      try_schwarz3d_w<5, 5, 5>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st, tp))
    return true;
  return try_schwarz3d<1, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st, tp) ||
         try_schwarz3d<2, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st, tp) ||
         try_schwarz3d<3, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st, tp) ||
         try_schwarz3d<4, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st, tp) ||
         try_schwarz3d<5, 5>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st, tp) ||
         try_schwarz3d<6, 5>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st, tp);
}

}  // namespace iga2l
