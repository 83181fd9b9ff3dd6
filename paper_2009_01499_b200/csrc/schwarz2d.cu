// Multicolour Schwarz colour kernels (reading A4): the 2D DMMA kernel (one warp per block),
// the generic fallback for any (p, s, d), and the per-colour dispatcher.  See kernels.cuh.
#include "common.cuh"
#include "kernels.cuh"

namespace iga2l {
namespace {

// =============================== Schwarz colour kernel ====================================
// contract one axis of a [s]^DIM array (first index fastest) with an s x s matrix V[l*s + j]:
//   transposed: out[.., j, ..] = Σ_l V[l][j] in[.., l, ..];  else out[.., l, ..] = Σ_j V[l][j] in[.., j, ..]
template <int DIM>
__device__ __forceinline__ void fd_contract(const double *in, double *out, const double *V, int s, int axis,
                                            bool transposed) {
  int tot = s * s;
  if (DIM == 3) tot *= s;
  const int stride = (axis == 0) ? 1 : (axis == 1 ? s : s * s);
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    const int o = (i / stride) % s;
    const int base = i - o * stride;
    double acc = 0.0;
    for (int l = 0; l < s; ++l) {
      const double v = transposed ? V[l * s + o] : V[o * s + l];
      acc = fma(v, in[base + l * stride], acc);
    }
    out[i] = acc;
  }
}

template <int DIM>
__global__ void __launch_bounds__(128) k_schwarz(int p, int s, int n1, const double *__restrict__ K,
                                                 const double *__restrict__ M, const double *__restrict__ Vt,
                                                 const double *__restrict__ lamt, const double *__restrict__ b,
                                                 double *__restrict__ x, int c0, int c1, int c2, int D, int nb0,
                                                 int nb1, int zoff, int ax) {
  extern __shared__ double sm[];
  // memory index of global point (gx, gy, gz); the last axis is stored from plane zoff on
#define SIDX(gx, gy, gz) ((DIM == 3) ? (((int64_t)((gz) - zoff) * n1 + (gy)) * n1 + (gx)) \
                                    : ((int64_t)((gy) - zoff) * n1 + (gx)))
  const int w = (s - 1) / 2, Wn = s + 2 * p, W = 2 * p + 1;
  const int bid = blockIdx.x;
  const int j0 = bid % nb0, j1 = (bid / nb0) % nb1, j2 = bid / (nb0 * nb1);
  const int cx = c0 + D * j0, cy = c1 + D * j1, cz = (DIM == 3) ? c2 + D * j2 : 0;
  const int ox = cx - w - p, oy = cy - w - p, oz = (DIM == 3) ? cz - w - p : 0;   // window origin
  const int bx = cx - w, by = cy - w, bz = (DIM == 3) ? cz - w : 0;                // block origin
  const int s2 = s * s, sd = (DIM == 3) ? s2 * s : s2;
  double *X = sm;
  const int nX = (DIM == 3) ? Wn * Wn * Wn : Wn * Wn;
  double *Pa = X + nX;
  const int nP = (DIM == 3) ? s * Wn * Wn : s * Wn;
  double *Pb = Pa + nP;
  double *Pc = Pb + nP;                   // 3D only: [Wn][s][s]
  const int nC = (DIM == 3) ? s2 * Wn : 0;
  double *Pe = Pc + nC;
  double *R = Pe + nC;                    // [s]^DIM
  double *Q0 = R + sd, *Q1 = Q0 + sd;
  double *Vx = Q1 + sd, *Vy = Vx + s2, *Vz = Vy + s2;
  double *Lx = Vz + s2, *Ly = Lx + s, *Lz = Ly + s;
  // 2D per-axis tables (ax = 1, quarter annulus): the y axis's band / FD tables follow the x axis's
  const int64_t ys = (DIM == 2 && ax) ? (int64_t)n1 * W : 0, vys = (DIM == 2 && ax) ? (int64_t)n1 * s2 : 0,
                lys = (DIM == 2 && ax) ? (int64_t)n1 * s : 0;

  for (int i = threadIdx.x; i < s2; i += blockDim.x) {
    Vx[i] = Vt[(int64_t)cx * s2 + i];
    Vy[i] = Vt[vys + (int64_t)cy * s2 + i];
    if (DIM == 3) Vz[i] = Vt[(int64_t)cz * s2 + i];
  }
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    Lx[i] = lamt[(int64_t)cx * s + i];
    Ly[i] = lamt[lys + (int64_t)cy * s + i];
    if (DIM == 3) Lz[i] = lamt[(int64_t)cz * s + i];
  }
  // window of x (zero outside the domain: the band tables vanish there too)
  for (int i = threadIdx.x; i < nX; i += blockDim.x) {
    const int wx = i % Wn, wy = (i / Wn) % Wn, wz = (DIM == 3) ? i / (Wn * Wn) : 0;
    const int gx = ox + wx, gy = oy + wy, gz = oz + wz;
    bool ok = gx >= 0 && gx < n1 && gy >= 0 && gy < n1;
    if (DIM == 3) ok = ok && gz >= 0 && gz < n1;
    X[i] = ok ? x[SIDX(gx, gy, gz)] : 0.0;
  }
  __syncthreads();
  // pass x over (lx in block) x (rest of window)
  for (int i = threadIdx.x; i < nP; i += blockDim.x) {
    const int lx = i % s, rest = i / s, gx = bx + lx;
    double sa = 0.0, sb = 0.0;
    if (gx >= 0 && gx < n1) {
      const double *kr = K + (int64_t)gx * W, *mr = M + (int64_t)gx * W, *xr = X + rest * Wn + lx;
      for (int t = 0; t < W; ++t) {
        sa = fma(kr[t], xr[t], sa);
        sb = fma(mr[t], xr[t], sb);
      }
    }
    Pa[i] = sa;   // [rest][lx], rest = wy (2D) or wz*Wn + wy (3D)
    Pb[i] = sb;
  }
  __syncthreads();
  if (DIM == 2) {
    for (int i = threadIdx.x; i < s2; i += blockDim.x) {
      const int lx = i % s, ly = i / s, gx = bx + lx, gy = by + ly;
      double r = 0.0;
      if (gx >= 0 && gx < n1 && gy >= 0 && gy < n1) {
        const double *kr = K + ys + (int64_t)gy * W, *mr = M + ys + (int64_t)gy * W;
        double acc = 0.0;
        for (int u = 0; u < W; ++u) {
          acc = fma(mr[u], Pa[(ly + u) * s + lx], acc);
          acc = fma(kr[u], Pb[(ly + u) * s + lx], acc);
        }
        r = b[SIDX(gx, gy, 0)] - acc;
      }
      R[i] = r;
    }
  } else {
    for (int i = threadIdx.x; i < nC; i += blockDim.x) {   // pass y over (lx, ly) x wz
      const int lx = i % s, ly = (i / s) % s, wz = i / s2, gy = by + ly;
      double sc = 0.0, se = 0.0;
      if (gy >= 0 && gy < n1) {
        const double *kr = K + (int64_t)gy * W, *mr = M + (int64_t)gy * W;
        for (int u = 0; u < W; ++u) {
          const int j = (wz * Wn + ly + u) * s + lx;
          sc = fma(mr[u], Pa[j], sc);
          sc = fma(kr[u], Pb[j], sc);
          se = fma(mr[u], Pb[j], se);
        }
      }
      Pc[i] = sc;
      Pe[i] = se;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < sd; i += blockDim.x) {   // pass z
      const int lx = i % s, ly = (i / s) % s, lz = i / s2;
      const int gx = bx + lx, gy = by + ly, gz = bz + lz;
      double r = 0.0;
      if (gx >= 0 && gx < n1 && gy >= 0 && gy < n1 && gz >= 0 && gz < n1) {
        const double *kr = K + (int64_t)gz * W, *mr = M + (int64_t)gz * W;
        double acc = 0.0;
        for (int v = 0; v < W; ++v) {
          const int j = ((lz + v) * s + ly) * s + lx;
          acc = fma(mr[v], Pc[j], acc);
          acc = fma(kr[v], Pe[j], acc);
        }
        r = b[SIDX(gx, gy, gz)] - acc;
      }
      R[i] = r;
    }
  }
  __syncthreads();
  // δ = (⊗V) Λ^{-1} (⊗V)^T r  (fast diagonalisation of the Kronecker-sum block matrix)
  fd_contract<DIM>(R, Q0, Vx, s, 0, true);
  __syncthreads();
  fd_contract<DIM>(Q0, Q1, Vy, s, 1, true);
  __syncthreads();
  double *cur = Q1, *oth = Q0;
  if (DIM == 3) {
    fd_contract<DIM>(Q1, Q0, Vz, s, 2, true);
    __syncthreads();
    cur = Q0;
    oth = Q1;
  }
  for (int i = threadIdx.x; i < sd; i += blockDim.x) {
    const int j = i % s, k = (i / s) % s, l = (DIM == 3) ? i / s2 : 0;
    double den = Lx[j] + Ly[k];
    if (DIM == 3) den += Lz[l];
    cur[i] /= den;
  }
  __syncthreads();
  if (DIM == 3) {
    fd_contract<DIM>(cur, oth, Vz, s, 2, false);
    __syncthreads();
    double *t = cur; cur = oth; oth = t;
  }
  fd_contract<DIM>(cur, oth, Vy, s, 1, false);
  __syncthreads();
  fd_contract<DIM>(oth, R, Vx, s, 0, false);
  __syncthreads();
  for (int i = threadIdx.x; i < sd; i += blockDim.x) {
    const int lx = i % s, ly = (i / s) % s, lz = (DIM == 3) ? i / s2 : 0;
    const int gx = bx + lx, gy = by + ly, gz = bz + lz;
    bool ok = gx >= 0 && gx < n1 && gy >= 0 && gy < n1;
    if (DIM == 3) ok = ok && gz >= 0 && gz < n1;
    if (ok) x[SIDX(gx, gy, gz)] += R[i];
  }
#undef SIDX
}
size_t schwarz_smem(int dim, int p, int s) {
  const size_t Wn = s + 2 * p, s2 = s * s, sd = dim == 3 ? s2 * s : s2;
  const size_t nX = dim == 3 ? Wn * Wn * Wn : Wn * Wn;
  const size_t nP = dim == 3 ? s * Wn * Wn : s * Wn;
  const size_t nC = dim == 3 ? s2 * Wn : 0;
  return sizeof(double) * (nX + 2 * nP + 2 * nC + 3 * sd + 3 * s2 + 3 * s);
}
// ---------------- 2D Schwarz colour kernel on the FP64 tensor pipe (DMMA), one warp per block -------
// mma.sync.m8n8k4.f64 (A 8x4 row-major, B 4x8 column-major, C 8x8): per lane a = A[l/4][l%4],
// b = B[l%4][l/4], c[i] = C[l/4][2(l%4)+i].  The block solve is five small GEMMs:
//   pass x  Pab[wy][j] = Σ_c X[wy][c] Bx[c][j],  Bx[c][lx] = K(bx+lx, c-lx), Bx[c][S+lx] = M(..)
//   pass y  R[ly][lx] = b_B - Σ_r Ay[ly][r] Pab'[r][lx],  Ay = [M_y band | K_y band], Pab' = [Pa; Pb]
//   FD      T = R Vx,  Z = (Vy^T T) ./ (λx_j + λy_k),  U = Z Vx^T,  δ = Vy U
// Band and FD operands are read through L1 (__ldg) straight into fragments; C fragments feed the next
// GEMM through warp shuffles.  Zero padding everywhere outside the s x s block / window.
// element (row, col) of an 8x8 C fragment held by the warp (c0, c1 of every lane)
__device__ __forceinline__ double c_elem(double c0, double c1, int row, int col) {
  const int src = (row << 2) | (col >> 1);
  const double v0 = __shfl_sync(0xffffffffu, c0, src), v1 = __shfl_sync(0xffffffffu, c1, src);
  return (col & 1) ? v1 : v0;
}

template <int P, int S>
struct Mma2 {
  static constexpr int W = 2 * P + 1, Wn = S + 2 * P, w = (S - 1) / 2;
  static constexpr int MT = (Wn + 7) / 8;            // pass-x m-tiles (window rows)
  static constexpr int KT = (Wn + 3) / 4;            // pass-x k-steps (window cols)
  static constexpr int NTX = (2 * S + 7) / 8;        // pass-x n-tiles (K and M columns)
  static constexpr int WN4 = KT * 4;                 // padded window width
  static constexpr int LDX = WN4 + 1;                // smem row stride of the window (odd: fewer conflicts)
  static constexpr int LDP = NTX * 8 + 1;            // smem row stride of Pab
  static constexpr int KY = (2 * WN4) / 4;           // pass-y k-steps
  static constexpr int KF = (S + 3) / 4;             // FD k-steps
  static constexpr int PER = MT * 8 * LDX + MT * 8 * LDP + S * S;   // doubles per warp
};

// Operand fragments of one block solve (per lane), split by axis so that translation-invariant axes
// (A27) can reuse a warp's cached copy: x-axis: pass-x band B operand, Vx (as B and as B^T), λx;
// y-axis: pass-y band A operand, Vy (as A^T and as A), λy.
template <int P, int S>
struct FragX {
  double bxf[Mma2<P, S>::KT][Mma2<P, S>::NTX], vxb[Mma2<P, S>::KF], vxtb[Mma2<P, S>::KF], lam[2];
};
template <int P, int S>
struct FragY {
  double ayf[Mma2<P, S>::KY], vyta[Mma2<P, S>::KF], vya[Mma2<P, S>::KF], lam;
};

template <int P, int S>
__device__ __forceinline__ void build_fragx(FragX<P, S> &f, int n1, int cx, const double *__restrict__ K,
                                            const double *__restrict__ M, const double *__restrict__ Vt,
                                            const double *__restrict__ lamt) {
  using G = Mma2<P, S>;
  constexpr int W = G::W, w = G::w, KT = G::KT, NTX = G::NTX, KF = G::KF;
  const int lane = threadIdx.x & 31, r4 = lane >> 2, q4 = lane & 3, bx = cx - w;
  const unsigned un = unsigned(n1);
#pragma unroll
  for (int kt = 0; kt < KT; ++kt)
#pragma unroll
    for (int nt = 0; nt < NTX; ++nt) {
      const int c = 4 * kt + q4, j = 8 * nt + r4;
      const int lx = j < S ? j : j - S, t = c - lx, g = bx + lx;
      const bool ok = j < 2 * S && t >= 0 && t < W && unsigned(g) < un;
      f.bxf[kt][nt] = ok ? __ldg((j < S ? K : M) + (int64_t)g * W + t) : 0.0;
    }
  const double *Vx = Vt + (int64_t)cx * S * S;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) {
    const int kk = 4 * kt + q4;
    const bool ok = kk < S && r4 < S;
    f.vxb[kt] = ok ? __ldg(Vx + kk * S + r4) : 0.0;
    f.vxtb[kt] = ok ? __ldg(Vx + r4 * S + kk) : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) f.lam[i] = (2 * q4 + i < S) ? __ldg(lamt + (int64_t)cx * S + 2 * q4 + i) : 1.0;
}

template <int P, int S>
__device__ __forceinline__ void build_fragy(FragY<P, S> &f, int n1, int cy, const double *__restrict__ K,
                                            const double *__restrict__ M, const double *__restrict__ Vt,
                                            const double *__restrict__ lamt) {
  using G = Mma2<P, S>;
  constexpr int W = G::W, w = G::w, KY = G::KY, KF = G::KF, WN4 = G::WN4;
  const int lane = threadIdx.x & 31, r4 = lane >> 2, q4 = lane & 3, by = cy - w;
  const unsigned un = unsigned(n1);
#pragma unroll
  for (int kt = 0; kt < KY; ++kt) {
    const int r = 4 * kt + q4, ly = r4;
    const bool second = r >= WN4;
    const int rr = second ? r - WN4 : r, t = rr - ly, g = by + ly;
    const bool ok = ly < S && t >= 0 && t < W && unsigned(g) < un;
    f.ayf[kt] = ok ? __ldg((second ? K : M) + (int64_t)g * W + t) : 0.0;
  }
  const double *Vy = Vt + (int64_t)cy * S * S;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) {
    const int kk = 4 * kt + q4;
    const bool ok = kk < S && r4 < S;
    f.vyta[kt] = ok ? __ldg(Vy + kk * S + r4) : 0.0;
    f.vya[kt] = ok ? __ldg(Vy + r4 * S + kk) : 0.0;
  }
  f.lam = r4 < S ? __ldg(lamt + (int64_t)cy * S + r4) : 1.0;
}

// Fragment accessors: operands held in registers (FragX/FragY) or read per use from memory in the
// lane-major export layout ([k][32], FragX/FragY member order) -- the latter keeps a block's ~70 operand
// registers free (k_schwarz2d_mmg).
template <int P, int S>
struct FxReg {
  const FragX<P, S> &f;
  __device__ double bx(int kt, int nt) const { return f.bxf[kt][nt]; }
  __device__ double vb(int k) const { return f.vxb[k]; }
  __device__ double vtb(int k) const { return f.vxtb[k]; }
  __device__ double lam(int i) const { return f.lam[i]; }
};
template <int P, int S>
struct FyReg {
  const FragY<P, S> &f;
  __device__ double ay(int k) const { return f.ayf[k]; }
  __device__ double vta(int k) const { return f.vyta[k]; }
  __device__ double va(int k) const { return f.vya[k]; }
  __device__ double lam() const { return f.lam; }
};
template <int P, int S>
struct FxMem {
  const double *p;
  int lane;
  static constexpr int NTX = Mma2<P, S>::NTX, KT = Mma2<P, S>::KT, KF = Mma2<P, S>::KF;
  __device__ double at(int k) const { return __ldg(p + k * 32 + lane); }
  __device__ double bx(int kt, int nt) const { return at(kt * NTX + nt); }
  __device__ double vb(int k) const { return at(KT * NTX + k); }
  __device__ double vtb(int k) const { return at(KT * NTX + KF + k); }
  __device__ double lam(int i) const { return at(KT * NTX + 2 * KF + i); }
};
template <int P, int S>
struct FyMem {
  const double *p;
  int lane;
  static constexpr int KY = Mma2<P, S>::KY, KF = Mma2<P, S>::KF;
  __device__ double at(int k) const { return __ldg(p + k * 32 + lane); }
  __device__ double ay(int k) const { return at(k); }
  __device__ double vta(int k) const { return at(KY + k); }
  __device__ double va(int k) const { return at(KY + KF + k); }
  __device__ double lam() const { return at(KY + 2 * KF); }
};

// ALIAS: Pab overlays the window X (rows of Pab trail the rows of X that pass x has consumed); the block's
// own x values are read before pass x.
template <int P, int S, bool ALIAS = false, class FXA, class FYA, class OUT>
__device__ __forceinline__ void mma_block_a(const double *Xw, int ldx, double *Pab, int n1, int cx, int cy,
                                            const FXA &fx, const FYA &fy, const double *__restrict__ b, int zoff,
                                            OUT out);

template <int P, int S, class OUT>
__device__ __forceinline__ void mma_block_f(const double *Xw, int ldx, double *Pab, int n1, int cx, int cy,
                                            const FragX<P, S> &fx, const FragY<P, S> &fy,
                                            const double *__restrict__ b, int zoff, OUT out) {
  mma_block_a<P, S, false>(Xw, ldx, Pab, n1, cx, cy, FxReg<P, S>{fx}, FyReg<P, S>{fy}, b, zoff, out);
}

template <int P, int S, bool ALIAS, class FXA, class FYA, class OUT>
__device__ __forceinline__ void mma_block_a(const double *Xw, int ldx, double *Pab, int n1, int cx, int cy,
                                            const FXA &fx, const FYA &fy, const double *__restrict__ b, int zoff,
                                            OUT out) {
  using G = Mma2<P, S>;
  constexpr int Wn = G::Wn, w = G::w, MT = G::MT, KT = G::KT, NTX = G::NTX, WN4 = G::WN4, LDP = G::LDP,
                KY = G::KY, KF = G::KF;
  const int lane = threadIdx.x & 31, r4 = lane >> 2, q4 = lane & 3;
  const int bx = cx - w, by = cy - w;
  const unsigned un = unsigned(n1);
  double rden[2], bb[2];                                     // 1/(λx_j + λy_k) and b_B at this lane's C elements
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int j = 2 * q4 + i;
    rden[i] = (r4 < S && j < S) ? 1.0 / (fx.lam(i) + fy.lam()) : 0.0;
    const int gx = bx + j, gy = by + r4;
    bb[i] = (r4 < S && j < S && unsigned(gx) < un && unsigned(gy) < un) ? __ldg(b + (int64_t)(gy - zoff) * n1 + gx) : 0.0;
  }
  double xc[2] = {0.0, 0.0};                                 // the block's own x (ALIAS: before Pab overlays X)
  if constexpr (ALIAS) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int lx = 2 * q4 + i;
      if (r4 < S && lx < S) xc[i] = Xw[(r4 + P) * ldx + lx + P];
    }
    __syncwarp();                                              // other lanes' Pab stores overwrite these rows
  }
  // ---- pass x ----
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    double acc[NTX][2];
#pragma unroll
    for (int nt = 0; nt < NTX; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const double a = Xw[(8 * mt + r4) * ldx + 4 * kt + q4];
#pragma unroll
      for (int nt = 0; nt < NTX; ++nt) dmma(acc[nt][0], acc[nt][1], a, fx.bx(kt, nt));
    }
#pragma unroll
    for (int nt = 0; nt < NTX; ++nt) {
      Pab[(8 * mt + r4) * LDP + 8 * nt + 2 * q4] = acc[nt][0];
      Pab[(8 * mt + r4) * LDP + 8 * nt + 2 * q4 + 1] = acc[nt][1];
    }
  }
  __syncwarp();
  // ---- pass y: R = b_B - Ay [Pa; Pb] ----
  double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0;      // two independent accumulation chains
#pragma unroll
  for (int kt = 0; kt < KY; ++kt) {
    const int r = 4 * kt + q4, lx = r4;
    const bool second = r >= WN4;
    const int rr = second ? r - WN4 : r;
    const double bv = (lx < S && rr < Wn) ? Pab[rr * LDP + (second ? S : 0) + lx] : 0.0;
    if (kt & 1) dmma(s0, s1, fy.ay(kt), bv);
    else dmma(r0, r1, fy.ay(kt), bv);
  }
  r0 = (r4 < S && 2 * q4 < S) ? bb[0] - (r0 + s0) : 0.0;
  r1 = (r4 < S && 2 * q4 + 1 < S) ? bb[1] - (r1 + s1) : 0.0;
  // ---- FD: T = R Vx;  Z = Vy^T T ./ den;  U = Z Vx^T;  δ = Vy U ----
  double t0 = 0.0, t1 = 0.0;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) dmma(t0, t1, c_elem(r0, r1, r4, 4 * kt + q4), fx.vb(kt));
  double z0 = 0.0, z1 = 0.0;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) dmma(z0, z1, fy.vta(kt), c_elem(t0, t1, 4 * kt + q4, r4));
  z0 *= rden[0];
  z1 *= rden[1];
  double u0 = 0.0, u1 = 0.0;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) dmma(u0, u1, c_elem(z0, z1, r4, 4 * kt + q4), fx.vtb(kt));
  double e0 = 0.0, e1 = 0.0;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) dmma(e0, e1, fy.va(kt), c_elem(u0, u1, 4 * kt + q4, r4));
  // ---- x_B += δ ----
  const int ly = r4, gy = by + ly;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int lx = 2 * q4 + i, gx = bx + lx;
    if (ly < S && lx < S && unsigned(gx) < un && unsigned(gy) < un)
      out(ly, lx, (ALIAS ? xc[i] : Xw[(ly + P) * ldx + lx + P]) + (i ? e1 : e0));
  }
}

template <int P, int S, class OUT>
__device__ __forceinline__ void mma_block(const double *Xw, int ldx, double *Pab, int n1, int cx, int cy,
                                          const double *__restrict__ K, const double *__restrict__ M,
                                          const double *__restrict__ Vt, const double *__restrict__ lamt,
                                          const double *__restrict__ b, int zoff, OUT out) {
  FragX<P, S> fx;
  FragY<P, S> fy;
  build_fragx<P, S>(fx, n1, cx, K, M, Vt, lamt);
  build_fragy<P, S>(fy, n1, cy, K, M, Vt, lamt);
  mma_block_f<P, S>(Xw, ldx, Pab, n1, cx, cy, fx, fy, b, zoff, out);
}

// Interior fragments (A27) of the per-colour DMMA kernel, lane-major: frag[k * 32 + lane], k over the
// FragX then FragY fields.  Built once per context by one warp; loaded coalesced by interior blocks.
template <int P, int S>
__host__ __device__ constexpr int frag_count() {
  return (sizeof(FragX<P, S>) + sizeof(FragY<P, S>)) / sizeof(double);
}
template <int P, int S>
__global__ void k_export_frags(int n1, int cref, const double *__restrict__ K, const double *__restrict__ M,
                               const double *__restrict__ Vt, const double *__restrict__ lamt, double *out) {
  FragX<P, S> fx;
  FragY<P, S> fy;
  build_fragx<P, S>(fx, n1, cref, K, M, Vt, lamt);
  build_fragy<P, S>(fy, n1, cref, K, M, Vt, lamt);
  const double *a = reinterpret_cast<const double *>(&fx), *c = reinterpret_cast<const double *>(&fy);
  constexpr int NX = sizeof(FragX<P, S>) / sizeof(double), NY = sizeof(FragY<P, S>) / sizeof(double);
#pragma unroll
  for (int k = 0; k < NX; ++k) out[k * 32 + threadIdx.x] = a[k];
#pragma unroll
  for (int k = 0; k < NY; ++k) out[(NX + k) * 32 + threadIdx.x] = c[k];
}

template <int P, int S>
__device__ __forceinline__ void load_frags(const double *__restrict__ fb, FragX<P, S> &fx, FragY<P, S> &fy) {
  constexpr int NX = sizeof(FragX<P, S>) / sizeof(double), NY = sizeof(FragY<P, S>) / sizeof(double);
  const int lane = threadIdx.x & 31;
  double *a = reinterpret_cast<double *>(&fx), *c = reinterpret_cast<double *>(&fy);
#pragma unroll
  for (int k = 0; k < NX; ++k) a[k] = __ldg(fb + k * 32 + lane);
#pragma unroll
  for (int k = 0; k < NY; ++k) c[k] = __ldg(fb + (NX + k) * 32 + lane);
}

// Body of one colour's block solve for block `bid` by the calling warp (per-warp shared memory X).
template <int P, int S>
__device__ __forceinline__ void mma_colour_block(double *__restrict__ X, int bid, int n1, const double *__restrict__ K,
                                                 const double *__restrict__ M, const double *__restrict__ Vt,
                                                 const double *__restrict__ lamt, const double *__restrict__ b,
                                                 double *__restrict__ x, int c0, int c1, int D, int nb0, int nblk,
                                                 int zoff, const double *__restrict__ fb, int tlo, int thi, int ax,
                                                 int trig = -1) {
  using G = Mma2<P, S>;
  constexpr int Wn = G::Wn, w = G::w, MT = G::MT, WN4 = G::WN4, LDX = G::LDX;
  const int lane = threadIdx.x & 31;
  double *Pab = X + MT * 8 * LDX;
  const int j1 = bid / nb0, j0 = bid - j1 * nb0;
  const int cx = c0 + D * j0, cy = c1 + D * j1;
  const int bx = cx - w, by = cy - w, ox = bx - P, oy = by - P;
  const unsigned un = unsigned(n1);
  // operand fragments first: they do not depend on x, so under programmatic dependent launch (PDL) they
  // load while the previous colour's grid is still running
  FragX<P, S> fx;
  FragY<P, S> fy;
  const bool interior = fb && cx - w >= tlo && cx + w <= thi && cy - w >= tlo && cy + w <= thi;
  if (interior) {
    load_frags<P, S>(fb, fx, fy);                            // interior block: shared fragments (A27)
  } else {
    build_fragx<P, S>(fx, n1, cx, K, M, Vt, lamt);
    if (ax) {                                                // per-axis tables (quarter annulus)
      const int64_t ys = (int64_t)n1 * G::W;
      build_fragy<P, S>(fy, n1, cy, K + ys, M + ys, Vt + (int64_t)n1 * S * S, lamt + (int64_t)n1 * S);
    } else {
      build_fragy<P, S>(fy, n1, cy, K, M, Vt, lamt);
    }
  }
  // x of the previous colour: wait for the prerequisite grid (no-op without PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (trig == 3) asm volatile("griddepcontrol.launch_dependents;");   // IGA2L_PDL=4
  // zero-padded window through registers: every lane issues all its loads back to back, then stores
  // (measured: 8-byte cp.async copies cost ~95 issue cycles per window row, 1.2-3k cycles per block)
  constexpr int WT = MT * 8 * WN4, WI = (WT + 31) / 32;
  double wv[WI];
#pragma unroll
  for (int k = 0; k < WI; ++k) {
    const int i = lane + 32 * k, row = i / WN4, cc = i - row * WN4;
    const int gx = ox + cc, gy = oy + row;
    const bool ok = i < WT && row < Wn && cc < Wn && unsigned(gx) < un && unsigned(gy) < un;
    wv[k] = ok ? x[(int64_t)(gy - zoff) * n1 + gx] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < WI; ++k) {
    const int i = lane + 32 * k, row = i / WN4, cc = i - row * WN4;
    if (i < WT) X[row * LDX + cc] = wv[k];
  }
  __syncwarp();
  if (trig == 1) asm volatile("griddepcontrol.launch_dependents;");
  mma_block_f<P, S>(X, LDX, Pab, n1, cx, cy, fx, fy, b, zoff, [&](int ly, int lx, double v) {
    x[(int64_t)(by + ly - zoff) * n1 + bx + lx] = v;
  });
}

template <int P, int S, int WPC>
__global__ void __launch_bounds__(WPC * 32) k_schwarz2d_mma(int n1, const double *__restrict__ K,
                                                            const double *__restrict__ M,
                                                            const double *__restrict__ Vt,
                                                            const double *__restrict__ lamt,
                                                            const double *__restrict__ b, double *__restrict__ x,
                                                            int c0, int c1, int D, int nb0, int nblk, int zoff,
                                                            const double *__restrict__ fb, int tlo, int thi, int ax,
                                                            int trig) {
  extern __shared__ double sm[];
  // PDL: the next colour's grid may launch once every CTA of this one triggered (trig 0: at entry, 1: after the
  // window is staged, else at exit); it waits (griddepcontrol.wait) for this grid's completion before it reads x
  if (trig == 0) asm volatile("griddepcontrol.launch_dependents;");
  const int warp = threadIdx.x >> 5;
  const int bid = blockIdx.x * WPC + warp;
  if (bid >= nblk) return;                                   // whole warp exits together
  mma_colour_block<P, S>(sm + warp * Mma2<P, S>::PER, bid, n1, K, M, Vt, lamt, b, x, c0, c1, D, nb0, nblk, zoff, fb,
                         tlo, thi, ax, trig);
}

// IGA2L_PDL (read per launch): 0 plain launches; else the colour kernels are launched with programmatic
// stream serialisation and trigger their dependents at entry (1), once the window is staged (2, default:
// C2 step 0.428 -> 0.365 ms, p = 5 chain 0.340 -> 0.282 ms), at exit (3: 0.392 ms) or right after their own
// griddepcontrol.wait (4: 0.370 ms).  Entry triggers let every colour's grid launch at once (0.409 ms).
// ---- k_schwarz2d_mmg: the same block solve with the operand fragments read per use from memory ----------
// (interior axes: the shared export, A27; boundary axes: the per-centre export) and Pab overlaying the
// window: ~60 instead of ~125 registers and 4.7 KB of shared memory per block at p = 8, so a colour of C3's
// 4692 blocks fits ONE wave (32 warps per SM) instead of two.  fb: [interior NX+NY][32] then
// [n1][NX][32] (FragX per x-centre) then [n1][NY][32] (FragY per y-centre), export_centre_frags.
template <int P, int S, int WPC, int MINB>
__global__ void __launch_bounds__(WPC * 32, MINB) k_schwarz2d_mmg(int n1, const double *__restrict__ b,
                                                                  double *__restrict__ x, int c0, int c1, int D,
                                                                  int nb0, int nblk, int zoff,
                                                                  const double *__restrict__ fb, int tlo, int thi,
                                                                  int trig) {
  using G = Mma2<P, S>;
  constexpr int Wn = G::Wn, w = G::w, MT = G::MT, WN4 = G::WN4, LDX = G::LDX;
  constexpr int NX = sizeof(FragX<P, S>) / sizeof(double), NY = sizeof(FragY<P, S>) / sizeof(double);
  extern __shared__ double sm[];
  if (trig == 0) asm volatile("griddepcontrol.launch_dependents;");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bid = blockIdx.x * WPC + warp;
  if (bid >= nblk) return;
  double *X = sm + warp * (MT * 8 * LDX);
  const int j1 = bid / nb0, j0 = bid - j1 * nb0;
  const int cx = c0 + D * j0, cy = c1 + D * j1;
  const int bx = cx - w, by = cy - w, ox = bx - P, oy = by - P;
  const unsigned un = unsigned(n1);
  const double *fxall = fb + (NX + NY) * 32, *fyall = fxall + int64_t(n1) * NX * 32;
  const bool ix = cx - w >= tlo && cx + w <= thi, iy = cy - w >= tlo && cy + w <= thi;
  const FxMem<P, S> fx{ix ? fb : fxall + int64_t(cx) * NX * 32, lane};
  const FyMem<P, S> fy{iy ? fb + NX * 32 : fyall + int64_t(cy) * NY * 32, lane};
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (trig == 3) asm volatile("griddepcontrol.launch_dependents;");
  constexpr int WT = MT * 8 * WN4, WI = (WT + 31) / 32;
  double wv[WI];
#pragma unroll
  for (int k = 0; k < WI; ++k) {
    const int i = lane + 32 * k, row = i / WN4, cc = i - row * WN4;
    const int gx = ox + cc, gy = oy + row;
    const bool ok = i < WT && row < Wn && cc < Wn && unsigned(gx) < un && unsigned(gy) < un;
    wv[k] = ok ? x[(int64_t)(gy - zoff) * n1 + gx] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < WI; ++k) {
    const int i = lane + 32 * k, row = i / WN4, cc = i - row * WN4;
    if (i < WT) X[row * LDX + cc] = wv[k];
  }
  __syncwarp();
  if (trig == 1) asm volatile("griddepcontrol.launch_dependents;");
  mma_block_a<P, S, true>(X, LDX, X, n1, cx, cy, fx, fy, b, zoff, [&](int ly, int lx, double v) {
    x[(int64_t)(by + ly - zoff) * n1 + bx + lx] = v;
  });
}

template <int P, int S>
__global__ void k_export_cfrags(int n1, const double *__restrict__ K, const double *__restrict__ M,
                                const double *__restrict__ Vt, const double *__restrict__ lamt, double *outx,
                                double *outy) {
  const int c = blockIdx.x, lane = threadIdx.x;
  FragX<P, S> fx;
  FragY<P, S> fy;
  build_fragx<P, S>(fx, n1, c, K, M, Vt, lamt);
  build_fragy<P, S>(fy, n1, c, K, M, Vt, lamt);
  const double *a = reinterpret_cast<const double *>(&fx), *d = reinterpret_cast<const double *>(&fy);
  constexpr int NX = sizeof(FragX<P, S>) / sizeof(double), NY = sizeof(FragY<P, S>) / sizeof(double);
#pragma unroll
  for (int k = 0; k < NX; ++k) outx[(int64_t(c) * NX + k) * 32 + lane] = a[k];
#pragma unroll
  for (int k = 0; k < NY; ++k) outy[(int64_t(c) * NY + k) * 32 + lane] = d[k];
}

// IGA2L_MMG (read per launch): 1 / 0 force / forbid k_schwarz2d_mmg; default: when the colour has more
// blocks than one wave of k_schwarz2d_mma (16 one-warp blocks per SM) and the centre fragments exist
inline int mmg_mode() {
  const char *e = std::getenv("IGA2L_MMG");
  return (e && *e) ? std::atoi(e) : -1;
}

inline int pdl_mode() {
  const char *e = std::getenv("IGA2L_PDL");
  return (e && *e) ? std::atoi(e) : 2;
}

template <int P, int S, int WPC>
void launch2d_mma(int64_t n1, const double *K, const double *M, const double *V, const double *lam, const double *b,
                  double *x, int c0, int c1, int D, int nb0, int nblk, int zoff, cudaStream_t st, const double *fb,
                  int ax) {
  const int m = int(n1) - P + 2;
  const int pm = pdl_mode();
  const int mg = mmg_mode();
  if (fb && !ax && (mg == 1 || (mg < 0 && nblk > 148 * 16))) {   // fragments from memory (k_schwarz2d_mmg)
    constexpr int MW = 8, MB = 4;
    constexpr size_t smg = sizeof(double) * MW * Mma2<P, S>::MT * 8 * Mma2<P, S>::LDX;
    ensure_smem(k_schwarz2d_mmg<P, S, MW, MB>, smg);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((nblk + MW - 1) / MW);
    cfg.blockDim = dim3(MW * 32);
    cfg.dynamicSmemBytes = smg;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pm > 0 ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, k_schwarz2d_mmg<P, S, MW, MB>, int(n1), b, x, c0, c1, D, nb0, nblk, zoff, fb, 2 * P - 1,
                           m - 2 - P, pm > 0 ? pm - 1 : -1) == cudaSuccess)
      return;
    cudaGetLastError();
  }
  constexpr size_t sm = sizeof(double) * WPC * Mma2<P, S>::PER;
  ensure_smem(k_schwarz2d_mma<P, S, WPC>, sm);
  if (pm > 0) {                                              // programmatic dependent launch (IGA2L_PDL)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((nblk + WPC - 1) / WPC);
    cfg.blockDim = dim3(WPC * 32);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_schwarz2d_mma<P, S, WPC>, int(n1), K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff,
                           fb, 2 * P - 1, m - 2 - P, ax, pm - 1) == cudaSuccess)
      return;
    cudaGetLastError();                                      // not launched: plain launch below
  }
  k_schwarz2d_mma<P, S, WPC><<<(nblk + WPC - 1) / WPC, WPC * 32, sm, st>>>(int(n1), K, M, V, lam, b, x, c0, c1, D,
                                                                           nb0, nblk, zoff, fb, 2 * P - 1, m - 2 - P, ax,
                                                                           -1);
}

template <int P, int S>
bool try_schwarz2d_mma(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                       const double *b, double *x, int c0, int c1, int D, int nb0, int nblk, int zoff, cudaStream_t st,
                       const double *fb, int ax) {
  if (p != P || s != S) return false;
  // warps (blocks) per CTA: 1 for s >= 5 (profiles/variants_wpc_r01.txt); 2 for s = 3 under programmatic
  // dependent launch (C2 step 0.3987 vs 0.4024 ms with 4, p = 3 alone 0.153 vs 0.160 ms; same box)
  constexpr int wpc = S >= 5 ? 1 : 2;
  launch2d_mma<P, S, wpc>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, fb, ax);
  return true;
}

}  // namespace

void centre_range(int c, int D, int lo, int hi, int *first, int *count) {
  int f = c;
  if (f < lo) f += ((lo - f + D - 1) / D) * D;
  *first = f;
  *count = (f < hi) ? (hi - 1 - f) / D + 1 : 0;
}

void launch_schwarz_colour(int dim, int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                           const double *lam, const double *b, double *x, int colour, int D, cudaStream_t st,
                           SlabView sv, int ax) {
  if (sv.zhi < 0) sv = SlabView{0, 0, int(n1)};
  const int c0 = colour % D, c1 = (colour / D) % D, c2 = (dim == 3) ? colour / (D * D) : 0;
  int fl, nl;   // last axis: first centre and count inside the slab's centre range
  centre_range(dim == 3 ? c2 : c1, D, sv.zlo, sv.zhi, &fl, &nl);
  if (c0 >= n1 || nl == 0) return;
  if (dim == 3 && c1 >= n1) return;
  const int nb0 = int((n1 - c0 + D - 1) / D);
  const int nb1 = (dim == 3) ? int((n1 - c1 + D - 1) / D) : nl;
  const int nb2 = (dim == 3) ? nl : 1;
  const size_t sm = schwarz_smem(dim, p, s);
  const unsigned nblk = unsigned(nb0) * unsigned(nb1) * unsigned(nb2);
  if (dim == 2) {
    ensure_smem(k_schwarz<2>, sm);
    k_schwarz<2><<<nblk, 128, sm, st>>>(p, s, int(n1), K, M, V, lam, b, x, c0, fl, 0, D, nb0, nb1, sv.zoff, ax);
  } else {
    ensure_smem(k_schwarz<3>, sm);
    k_schwarz<3><<<nblk, 128, sm, st>>>(p, s, int(n1), K, M, V, lam, b, x, c0, c1, fl, D, nb0, nb1, sv.zoff, 0);
  }
}

bool launch_schwarz_colour_fast(int dim, int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                                const double *lam, const double *b, double *x, int colour, int D, cudaStream_t st,
                                SlabView sv, const double *fb, const ToeP *tp, int ax) {
  if (sv.zhi < 0) sv = SlabView{0, 0, int(n1)};
  if (dim == 3) {
    const int c0 = colour % D, c1 = (colour / D) % D, c2 = colour / (D * D);
    int f2, nb2;
    centre_range(c2, D, sv.zlo, sv.zhi, &f2, &nb2);
    if (c0 >= n1 || c1 >= n1 || nb2 == 0) return true;   // empty colour
    const int nb0 = int((n1 - c0 + D - 1) / D), nb1 = int((n1 - c1 + D - 1) / D);
    const int m = int(n1) - p + 2;
    const int tlo = 2 * p - 1, thi = m - 2 - p;            // translation-invariant rows (toeplitz_rows)
    const int z = sv.zoff;
    return launch_schwarz3d_colour(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, tlo, thi, st, tp);
  }
  if (dim != 2) return false;
  const int c0 = colour % D, c1 = (colour / D) % D;
  int f1, nb1;
  centre_range(c1, D, sv.zlo, sv.zhi, &f1, &nb1);
  if (c0 >= n1 || nb1 == 0) return true;   // empty colour
  const int nb0 = int((n1 - c0 + D - 1) / D), nblk = nb0 * nb1;
  const int z = sv.zoff;
  return try_schwarz2d_mma<1, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb, ax) ||
         try_schwarz2d_mma<2, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb, ax) ||
         try_schwarz2d_mma<3, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb, ax) ||
         try_schwarz2d_mma<4, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb, ax) ||
         try_schwarz2d_mma<5, 5>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb, ax) ||
         try_schwarz2d_mma<6, 5>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb, ax) ||
         try_schwarz2d_mma<7, 7>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb, ax) ||
         try_schwarz2d_mma<8, 7>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb, ax);
}

int export_centre_frags(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                        const double *lam, double *out, cudaStream_t st) {
#define IGA2L_EXPC(P_, S_)                                                                                  \
  if (p == P_ && s == S_) {                                                                                 \
    constexpr int NX = sizeof(FragX<P_, S_>) / sizeof(double), NY = sizeof(FragY<P_, S_>) / sizeof(double); \
    if (out)                                                                                                \
      k_export_cfrags<P_, S_><<<int(n1), 32, 0, st>>>(int(n1), K, M, V, lam, out, out + n1 * NX * 32);    \
    return int(n1 * (NX + NY) * 32);                                                                        \
  }
  IGA2L_EXPC(1, 3) IGA2L_EXPC(2, 3) IGA2L_EXPC(3, 3) IGA2L_EXPC(4, 3) IGA2L_EXPC(5, 5) IGA2L_EXPC(6, 5)
  IGA2L_EXPC(7, 7) IGA2L_EXPC(8, 7)
#undef IGA2L_EXPC
  return -1;
}

int export_interior_frags(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                          const double *lam, double *out, cudaStream_t st) {
  const int m = int(n1) - p + 2, tlo = 2 * p - 1, thi = m - 2 - p, w = (s - 1) / 2;
  if (thi - tlo < 2 * w) return -1;
  const int cref = (tlo + thi) / 2;
#define IGA2L_EXP(P_, S_)                                                                                   \
  if (p == P_ && s == S_) {                                                                                 \
    if (!out) return frag_count<P_, S_>() * 32;                                        \
    k_export_frags<P_, S_><<<1, 32, 0, st>>>(int(n1), cref, K, M, V, lam, out);                            \
    return frag_count<P_, S_>() * 32;                                                  \
  }
  IGA2L_EXP(1, 3) IGA2L_EXP(2, 3) IGA2L_EXP(3, 3) IGA2L_EXP(4, 3) IGA2L_EXP(5, 5) IGA2L_EXP(6, 5) IGA2L_EXP(7, 7)
  IGA2L_EXP(8, 7)
#undef IGA2L_EXP
  return -1;
}

}  // namespace iga2l
