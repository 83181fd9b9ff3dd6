// 3D multicolour Schwarz colour kernel (reading A4, A25): one CTA per block, register-blocked
// pencil passes for the sum-factorised block residual, then fast diagonalisation.  See kernels.cuh.
#include "common.cuh"
#include "kernels.cuh"

namespace iga2l {
namespace {

// ---------------- 3D Schwarz colour kernel, compile-time (p, s): one CTA per block ------------
// Same arithmetic as k_schwarz<3> (sum-factorised block residual over the (s+2p)^3 window, then
// fast diagonalisation), register-blocked: every pass maps one thread to a PENCIL (a line of the
// window along the contracted axis), loads it once into registers and produces all s outputs of that
// line.  A pass along an axis whose s block rows are all translation-invariant rows (tlo..thi, made
// bitwise equal at setup) keeps the 2(2p+1) band coefficients in registers; otherwise they are read
// per row from shared memory.
template <int S, int W, int Wn, bool TOE>
__device__ __forceinline__ void band_pencil(const double *in, int stride, const double *ck, const double *cm,
                                            double (&oa)[S], double (&ob)[S]) {
  double v[Wn];
#pragma unroll
  for (int k = 0; k < Wn; ++k) v[k] = in[k * stride];
#pragma unroll
  for (int l = 0; l < S; ++l) {
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int t = 0; t < W; ++t) {
      const double kc = TOE ? ck[t] : ck[l * W + t], mc = TOE ? cm[t] : cm[l * W + t];
      if (t & 1) { a1 = fma(kc, v[l + t], a1); b1 = fma(mc, v[l + t], b1); }
      else { a0 = fma(kc, v[l + t], a0); b0 = fma(mc, v[l + t], b0); }
    }
    oa[l] = a0 + a1;
    ob[l] = b0 + b1;
  }
}

// pass y: from pencils pa, pb (stride) -> c = My pa + Ky pb, e = My pb
template <int S, int W, int Wn, bool TOE>
__device__ __forceinline__ void band_pencil2(const double *pa_, const double *pb_, int stride, const double *ck,
                                             const double *cm, double (&oc)[S], double (&oe)[S]) {
  double pa[Wn], pb[Wn];
#pragma unroll
  for (int k = 0; k < Wn; ++k) { pa[k] = pa_[k * stride]; pb[k] = pb_[k * stride]; }
#pragma unroll
  for (int l = 0; l < S; ++l) {
    double c0 = 0.0, c1 = 0.0, e0 = 0.0;
#pragma unroll
    for (int t = 0; t < W; ++t) {
      const double kc = TOE ? ck[t] : ck[l * W + t], mc = TOE ? cm[t] : cm[l * W + t];
      c0 = fma(mc, pa[l + t], c0);
      c1 = fma(kc, pb[l + t], c1);
      e0 = fma(mc, pb[l + t], e0);
    }
    oc[l] = c0 + c1;
    oe[l] = e0;
  }
}

template <int P, int S>
struct Blk3 {
  static constexpr int W = 2 * P + 1, Wn = S + 2 * P, w = (S - 1) / 2, S2 = S * S, S3 = S2 * S, Wn2 = Wn * Wn;
  // per-block layout; Pc/Pe alias the window X (dead after pass x once its s^3 centre values are in Xc)
  static constexpr int OPa = Wn2 * Wn, OPb = OPa + Wn2 * S, OXc = OPb + Wn2 * S, OR = OXc + S3, OQ = OR + S3,
                       OBb = OQ + S3, OTk = OBb + S3, OTm = OTk + 3 * S * W, OVs = OTm + 3 * S * W, OLs = OVs + 3 * S2;
  static constexpr int PER = OLs + 3 * S;
  static_assert(2 * Wn * S2 <= Wn2 * Wn, "Pc/Pe must fit in the window");
};

// NBK blocks per CTA (block g = blockIdx.x * NBK + k of the colour's nb0 x nb1 x nb2 grid); every phase
// runs over (block, pencil) pairs so that the short phases still occupy the CTA.
template <int P, int S, int NBK, int NT, bool ROW, bool REGW = false>
__global__ void __launch_bounds__(NT) k_schwarz3d_t(int n1, const double *__restrict__ K, const double *__restrict__ M,
                                                    const double *__restrict__ Vt, const double *__restrict__ lamt,
                                                    const double *__restrict__ b, double *__restrict__ x, int c0, int c1,
                                                    int c2, int D, int nb0, int nb1, int nblk, int zoff, int tlo,
                                                    int thi) {
  using B = Blk3<P, S>;
  constexpr int W = B::W, Wn = B::Wn, w = B::w, S2 = B::S2, S3 = B::S3, Wn2 = B::Wn2, PER = B::PER;
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  const unsigned un = unsigned(n1);
  // per-block regions: X [z][y][x] window, Pa/Pb [wz][wy][lx], Pc/Pe [wz][ly][lx], R, Q, Bb,
  // Tk/Tm [axis][row][t], Vs [axis][l][j], Ls [axis][j]
  auto X = [&](int k) { return sm + k * PER; };
  auto Pa = [&](int k) { return sm + k * PER + B::OPa; };
  auto Pb = [&](int k) { return sm + k * PER + B::OPb; };
  auto Pc = [&](int k) { return sm + k * PER; };                     // aliases X (see Blk3)
  auto Pe = [&](int k) { return sm + k * PER + Wn * S2; };
  auto Xc = [&](int k) { return sm + k * PER + B::OXc; };
  auto R = [&](int k) { return sm + k * PER + B::OR; };
  auto Q = [&](int k) { return sm + k * PER + B::OQ; };
  auto Bb = [&](int k) { return sm + k * PER + B::OBb; };
  auto Tk = [&](int k) { return sm + k * PER + B::OTk; };
  auto Tm = [&](int k) { return sm + k * PER + B::OTm; };
  auto Vs = [&](int k) { return sm + k * PER + B::OVs; };
  auto Ls = [&](int k) { return sm + k * PER + B::OLs; };
  __shared__ int sC[NBK][3];
  __shared__ bool sT[NBK][3];
  if (NBK > 1 && tid < NBK) {                               // block centres, Toeplitz flags per axis
    const int g = blockIdx.x * NBK + tid;
    const int cc[3] = {c0 + D * (g % nb0), c1 + D * ((g / nb0) % nb1), c2 + D * (g / (nb0 * nb1))};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      sC[tid][a] = cc[a];
      sT[tid][a] = (cc[a] - w >= tlo) && (cc[a] + w <= thi);
    }
  }
  __syncthreads();
  int cc1[3];                                               // NBK == 1: the centre in registers
  bool tt1[3];
  if (NBK == 1) {
    const int g = blockIdx.x;
    cc1[0] = c0 + D * (g % nb0);
    cc1[1] = c1 + D * ((g / nb0) % nb1);
    cc1[2] = c2 + D * (g / (nb0 * nb1));
#pragma unroll
    for (int a = 0; a < 3; ++a) tt1[a] = (cc1[a] - w >= tlo) && (cc1[a] + w <= thi);
  }
  auto centre = [&](int k, int a) { return NBK == 1 ? cc1[a] : sC[k][a]; };
  const int nk = min(NBK, nblk - int(blockIdx.x) * NBK);   // blocks of this CTA
  // ---- loads: band rows, FD tables, b_B (through registers when one block per CTA: the 8-byte cp.async
  // issue cost dominated this phase), x windows ----
  if (NBK == 1 && !ROW) {
    constexpr int NTAB = 2 * 3 * S * W + 3 * S2 + 3 * S + S3;   // Tk, Tm, Vs, Ls, Bb
    constexpr int IT = (NTAB + NT - 1) / NT;
    double v[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = tid + k * NT;
      double val = 0.0;
      if (i < 2 * 3 * S * W) {
        const int r = i % (3 * S * W), a = r / (S * W), l = (r / W) % S, t = r % W;
        const int g = centre(0, a) - w + l;
        if (unsigned(g) < un) val = (i < 3 * S * W ? K : M)[(int64_t)g * W + t];
      } else if (i < 2 * 3 * S * W + 3 * S2) {
        const int r = i - 2 * 3 * S * W;
        val = Vt[(int64_t)centre(0, r / S2) * S2 + r % S2];
      } else if (i < 2 * 3 * S * W + 3 * S2 + 3 * S) {
        const int r = i - 2 * 3 * S * W - 3 * S2;
        val = lamt[(int64_t)centre(0, r / S) * S + r % S];
      } else if (i < NTAB) {
        const int r = i - 2 * 3 * S * W - 3 * S2 - 3 * S;
        const int gx = centre(0, 0) - w + r % S, gy = centre(0, 1) - w + (r / S) % S, gz = centre(0, 2) - w + r / S2;
        if (unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un)
          val = b[((int64_t)(gz - zoff) * n1 + gy) * n1 + gx];
      }
      v[k] = val;
    }
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = tid + k * NT;
      if (i < 3 * S * W) Tk(0)[i] = v[k];
      else if (i < 2 * 3 * S * W) Tm(0)[i - 3 * S * W] = v[k];
      else if (i < 2 * 3 * S * W + 3 * S2) Vs(0)[i - 2 * 3 * S * W] = v[k];
      else if (i < 2 * 3 * S * W + 3 * S2 + 3 * S) Ls(0)[i - 2 * 3 * S * W - 3 * S2] = v[k];
      else if (i < NTAB) Bb(0)[i - 2 * 3 * S * W - 3 * S2 - 3 * S] = v[k];
    }
  } else {
  for (int i = tid; i < nk * 3 * S * W; i += NT) {
    const int k = NBK == 1 ? 0 : i / (3 * S * W), r = NBK == 1 ? i : i % (3 * S * W);
    const int a = r / (S * W), l = (r / W) % S, t = r % W;
    const int g = centre(k, a) - w + l;
    const bool ok = unsigned(g) < un;
    cp_async8(Tk(k) + r, K + (ok ? (int64_t)g * W + t : 0), ok);
    cp_async8(Tm(k) + r, M + (ok ? (int64_t)g * W + t : 0), ok);
  }
  for (int i = tid; i < nk * 3 * S2; i += NT) {
    const int k = NBK == 1 ? 0 : i / (3 * S2), r = NBK == 1 ? i : i % (3 * S2);
    cp_async8(Vs(k) + r, Vt + (int64_t)centre(k, r / S2) * S2 + r % S2, true);
  }
  for (int i = tid; i < nk * 3 * S; i += NT) {
    const int k = NBK == 1 ? 0 : i / (3 * S), r = NBK == 1 ? i : i % (3 * S);
    cp_async8(Ls(k) + r, lamt + (int64_t)centre(k, r / S) * S + r % S, true);
  }
  for (int i = tid; i < nk * S3; i += NT) {
    const int k = NBK == 1 ? 0 : i / S3, r = NBK == 1 ? i : i % S3;
    const int gx = centre(k, 0) - w + r % S, gy = centre(k, 1) - w + (r / S) % S, gz = centre(k, 2) - w + r / S2;
    const bool ok = unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un;
    cp_async8(Bb(k) + r, b + (ok ? ((int64_t)(gz - zoff) * n1 + gy) * n1 + gx : 0), ok);
  }
  }
  if (!ROW && NBK == 1 && (REGW || Wn2 * Wn <= 1024)) {   // x window through registers, batches of 16 loads
                                                   // (measured: C4 40.6 -> 36.6 us/colour; C5 slower)
    constexpr int TOT = Wn2 * Wn, BATCH = 16;      // (8-byte cp.async issue costs ~95 cycles each)
    const int ox = centre(0, 0) - w - P, oy = centre(0, 1) - w - P, oz = centre(0, 2) - w - P;
    for (int i0 = 0; i0 < TOT; i0 += NT * BATCH) {
      double v[BATCH];
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        const int r = i0 + tid + k * NT;
        const int gx = ox + r % Wn, gy = oy + (r / Wn) % Wn, gz = oz + r / Wn2;
        const bool ok = r < TOT && unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un;
        v[k] = ok ? x[((int64_t)(gz - zoff) * n1 + gy) * n1 + gx] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        const int r = i0 + tid + k * NT;
        if (r < TOT) X(0)[r] = v[k];
      }
    }
  } else if (!ROW) {                               // x windows, element by element
    for (int i = tid; i < nk * Wn2 * Wn; i += NT) {
      const int k = NBK == 1 ? 0 : i / (Wn2 * Wn), r = NBK == 1 ? i : i % (Wn2 * Wn);
      const int gx = centre(k, 0) - w - P + r % Wn, gy = centre(k, 1) - w - P + (r / Wn) % Wn,
                gz = centre(k, 2) - w - P + r / Wn2;
      const bool ok = unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un;
      cp_async8(X(k) + r, x + (ok ? ((int64_t)(gz - zoff) * n1 + gy) * n1 + gx : 0), ok);
    }
  } else {                                          // x windows: one window row per 16 lanes
    const int lane16 = tid & 15;
    for (int row = tid >> 4; row < nk * Wn2; row += NT / 16) {
      const int k = NBK == 1 ? 0 : row / Wn2, rr = row - k * Wn2, wz = rr / Wn, wy = rr - wz * Wn;
      const int ox = centre(k, 0) - w - P, gy = centre(k, 1) - w - P + wy, gz = centre(k, 2) - w - P + wz;
      const bool okyz = unsigned(gy) < un && unsigned(gz) < un;
      const double *src = x + (okyz ? ((int64_t)(gz - zoff) * n1 + gy) * n1 : 0);
      double *dst = X(k) + rr * Wn;
#pragma unroll
      for (int wx = lane16; wx < Wn; wx += 16) {
        const int gx = ox + wx;
        const bool ok = okyz && unsigned(gx) < un;
        cp_async8(dst + wx, ok ? src + gx : x, ok);
      }
    }
  }
  cp_async_wait_all();
  auto toe = [&](int k, int a) { return NBK == 1 ? tt1[a] : sT[k][a]; };
  __syncthreads();
  // ---- pass x: pencils (wy, wz) along x -> Pa = Kx X, Pb = Mx X ----
  for (int i = tid; i < nk * Wn2; i += NT) {
    const int k = NBK == 1 ? 0 : i / Wn2, pi = NBK == 1 ? i : i % Wn2;
    double oa[S], ob[S];
    if (toe(k, 0)) band_pencil<S, W, Wn, true>(X(k) + pi * Wn, 1, Tk(k), Tm(k), oa, ob);
    else band_pencil<S, W, Wn, false>(X(k) + pi * Wn, 1, Tk(k), Tm(k), oa, ob);
#pragma unroll
    for (int l = 0; l < S; ++l) { Pa(k)[pi * S + l] = oa[l]; Pb(k)[pi * S + l] = ob[l]; }
  }
  for (int i = tid; i < nk * S3; i += NT) {        // the block's centre values, before Pc/Pe overwrite X
    const int k = NBK == 1 ? 0 : i / S3, r = NBK == 1 ? i : i % S3;
    const int lx = r % S, ly = (r / S) % S, lz = r / S2;
    Xc(k)[r] = X(k)[((lz + P) * Wn + ly + P) * Wn + lx + P];
  }
  __syncthreads();
  // ---- pass y: pencils (wz, lx) along y -> Pc = My Pa + Ky Pb, Pe = My Pb ----
  for (int i = tid; i < nk * Wn * S; i += NT) {
    const int k = NBK == 1 ? 0 : i / (Wn * S), pi = NBK == 1 ? i : i % (Wn * S);
    const int wz = pi / S, lx = pi % S;
    double oc[S], oe[S];
    const double *pa = Pa(k) + wz * Wn * S + lx, *pb = Pb(k) + wz * Wn * S + lx;
    if (toe(k, 1)) band_pencil2<S, W, Wn, true>(pa, pb, S, Tk(k) + S * W, Tm(k) + S * W, oc, oe);
    else band_pencil2<S, W, Wn, false>(pa, pb, S, Tk(k) + S * W, Tm(k) + S * W, oc, oe);
#pragma unroll
    for (int l = 0; l < S; ++l) { Pc(k)[(wz * S + l) * S + lx] = oc[l]; Pe(k)[(wz * S + l) * S + lx] = oe[l]; }
  }
  __syncthreads();
  // ---- pass z: pencils (ly, lx) along z -> r_B = b_B - (Mz Pc + Kz Pe) ----
  for (int i = tid; i < nk * S2; i += NT) {
    const int k = NBK == 1 ? 0 : i / S2, pi = NBK == 1 ? i : i % S2;
    double oc[S], oe[S];
    if (toe(k, 2)) band_pencil2<S, W, Wn, true>(Pc(k) + pi, Pe(k) + pi, S2, Tk(k) + 2 * S * W, Tm(k) + 2 * S * W, oc, oe);
    else band_pencil2<S, W, Wn, false>(Pc(k) + pi, Pe(k) + pi, S2, Tk(k) + 2 * S * W, Tm(k) + 2 * S * W, oc, oe);
#pragma unroll
    for (int l = 0; l < S; ++l) R(k)[l * S2 + pi] = Bb(k)[l * S2 + pi] - oc[l];
  }
  __syncthreads();
  // ---- δ = (⊗V) Λ^{-1} (⊗V)^T r ----
  if constexpr (S == 3 && NBK == 1) {   // s^3 = 27 values: the whole FD in one warp's registers (shuffles)
    if (tid < 32) {
      const int lane = tid, li = lane < 27 ? lane : 0;
      const int lx = li % 3, ly = (li / 3) % 3, lz = li / 9;
      const double *Vx = Vs(0), *Vy = Vs(0) + 9, *Vz = Vs(0) + 18, *L = Ls(0);
      double v;
      {
      v = lane < 27 ? R(0)[li] : 0.0;
      auto src = [&](int ax, int l) { return ax == 0 ? lz * 9 + ly * 3 + l : (ax == 1 ? lz * 9 + l * 3 + lx : l * 9 + ly * 3 + lx); };
      auto step = [&](int ax, const double *V, bool trans) {   // trans: out[j] = Σ_l V[l][j] in[l]; else V[j][l]
        const int j = ax == 0 ? lx : (ax == 1 ? ly : lz);
        double o = 0.0;
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          const double in = __shfl_sync(0xffffffffu, v, src(ax, l));
          o = fma(trans ? V[l * 3 + j] : V[j * 3 + l], in, o);
        }
        v = o;
      };
      step(0, Vx, true);
      step(1, Vy, true);
      step(2, Vz, true);
      v /= (L[lx] + L[3 + ly] + L[6 + lz]);
      step(2, Vz, false);
      step(1, Vy, false);
      step(0, Vx, false);
      }
      const int gx = centre(0, 0) - w + lx, gy = centre(0, 1) - w + ly, gz = centre(0, 2) - w + lz;
      if (lane < 27 && unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un)
        x[((int64_t)(gz - zoff) * n1 + gy) * n1 + gx] = Xc(0)[(lz * S + ly) * S + lx] + v;
    }
    return;
  }
  if constexpr (!(S == 3 && NBK == 1)) {   // general FD (s >= 5 or several blocks per CTA)
  for (int i = tid; i < nk * S3; i += NT) {         // along x (transposed)
    const int k = NBK == 1 ? 0 : i / S3, r = NBK == 1 ? i : i % S3, j = r % S, rest = r - j;
    const double *Vx = Vs(k);
    double a0 = 0.0;
#pragma unroll
    for (int l = 0; l < S; ++l) a0 = fma(Vx[l * S + j], R(k)[rest + l], a0);
    Q(k)[r] = a0;
  }
  __syncthreads();
  for (int i = tid; i < nk * S3; i += NT) {         // along y (transposed)
    const int k = NBK == 1 ? 0 : i / S3, r = NBK == 1 ? i : i % S3, j = r % S, kk = (r / S) % S, lz = r / S2;
    const double *Vy = Vs(k) + S2;
    double a0 = 0.0;
#pragma unroll
    for (int l = 0; l < S; ++l) a0 = fma(Vy[l * S + kk], Q(k)[(lz * S + l) * S + j], a0);
    R(k)[r] = a0;
  }
  __syncthreads();
  for (int i = tid; i < nk * S3; i += NT) {         // along z (transposed), then / (λx + λy + λz)
    const int k = NBK == 1 ? 0 : i / S3, r = NBK == 1 ? i : i % S3, j = r % S, kk = (r / S) % S, l3 = r / S2;
    const double *Vz = Vs(k) + 2 * S2, *L = Ls(k);
    double a0 = 0.0;
#pragma unroll
    for (int l = 0; l < S; ++l) a0 = fma(Vz[l * S + l3], R(k)[(l * S + kk) * S + j], a0);
    Q(k)[r] = a0 / (L[j] + L[S + kk] + L[2 * S + l3]);
  }
  __syncthreads();
  for (int i = tid; i < nk * S3; i += NT) {         // along z
    const int k = NBK == 1 ? 0 : i / S3, r = NBK == 1 ? i : i % S3, j = r % S, kk = (r / S) % S, lz = r / S2;
    const double *Vz = Vs(k) + 2 * S2;
    double a0 = 0.0;
#pragma unroll
    for (int l = 0; l < S; ++l) a0 = fma(Vz[lz * S + l], Q(k)[(l * S + kk) * S + j], a0);
    R(k)[r] = a0;
  }
  __syncthreads();
  for (int i = tid; i < nk * S3; i += NT) {         // along y
    const int k = NBK == 1 ? 0 : i / S3, r = NBK == 1 ? i : i % S3, j = r % S, ly = (r / S) % S, lz = r / S2;
    const double *Vy = Vs(k) + S2;
    double a0 = 0.0;
#pragma unroll
    for (int l = 0; l < S; ++l) a0 = fma(Vy[ly * S + l], R(k)[(lz * S + l) * S + j], a0);
    Q(k)[r] = a0;
  }
  __syncthreads();
  for (int i = tid; i < nk * S3; i += NT) {         // along x, and x_B += δ
    const int k = NBK == 1 ? 0 : i / S3, r = NBK == 1 ? i : i % S3, lx = r % S, ly = (r / S) % S, lz = r / S2, rest = r - lx;
    const double *Vx = Vs(k);
    double a0 = 0.0;
#pragma unroll
    for (int l = 0; l < S; ++l) a0 = fma(Vx[lx * S + l], Q(k)[rest + l], a0);
    const int gx = centre(k, 0) - w + lx, gy = centre(k, 1) - w + ly, gz = centre(k, 2) - w + lz;
    if (unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un)
      x[((int64_t)(gz - zoff) * n1 + gy) * n1 + gx] = Xc(k)[r] + a0;
  }
  }
}

template <int P, int S, int NBK, int NT, bool ROW, bool REGW = false>
void launch3d(int64_t n1, const double *K, const double *M, const double *V, const double *lam, const double *b,
              double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nb2, int zoff, int tlo, int thi,
              cudaStream_t st) {
  constexpr size_t sm = sizeof(double) * NBK * Blk3<P, S>::PER;
  ensure_smem(k_schwarz3d_t<P, S, NBK, NT, ROW, REGW>, sm);
  const int nblk = nb0 * nb1 * nb2;
  k_schwarz3d_t<P, S, NBK, NT, ROW, REGW><<<(nblk + NBK - 1) / NBK, NT, sm, st>>>(int(n1), K, M, V, lam, b, x, c0, c1,
                                                                                  c2, D, nb0, nb1, nblk, zoff, tlo, thi);
}

template <int P, int S>
bool try_schwarz3d(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                   const double *b, double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nb2, int zoff,
                   int tlo, int thi, cudaStream_t st) {
  if (p != P || s != S) return false;
  constexpr int NT1 = ((Blk3<P, S>::Wn2 + 31) / 32) * 32 > 512 ? 512 : ((Blk3<P, S>::Wn2 + 31) / 32) * 32;
  // measured best (profiles/variants_s3d_r01.txt): one block per CTA; s >= 5: half the pass-x pencil count of threads
  launch3d<P, S, 1, (S >= 5 && NT1 >= 128 ? NT1 / 2 : NT1), false>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2,
                                                                  zoff, tlo, thi, st);
  return true;
}

}  // namespace

bool launch_schwarz3d_colour(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                             const double *lam, const double *b, double *x, int c0, int c1, int f2, int D, int nb0,
                             int nb1, int nb2, int zoff, int tlo, int thi, cudaStream_t st) {
  return try_schwarz3d<1, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st) ||
         try_schwarz3d<2, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st) ||
         try_schwarz3d<3, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st) ||
         try_schwarz3d<4, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st) ||
         try_schwarz3d<5, 5>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st) ||
         try_schwarz3d<6, 5>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, zoff, tlo, thi, st);
}

}  // namespace iga2l
