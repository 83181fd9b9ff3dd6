// Device kernels of libiga2l (layer L1), sm_100a.  See kernels.cuh for the contracts.
#include "kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace iga2l {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block reduction (fixed tree); result valid in thread 0
__device__ double block_sum(double v, double *scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = (lane < nw) ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// 8-byte asynchronous global->shared copy (LDGSTS); ok == false writes 0.0 (zero fill, no read)
__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool ok) {
  const unsigned d = unsigned(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ============================ fine operator: apply / residual ============================
// 2D tile TX x TY outputs; window (TX+2p) x (TY+2p) staged in shared memory.
template <int TX, int TY>
__global__ void __launch_bounds__(256) k_apply2d(int p, int n1, const double *__restrict__ K,
                                                 const double *__restrict__ M, const double *__restrict__ x,
                                                 const double *__restrict__ b, double *__restrict__ y,
                                                 double *__restrict__ partial, int mode, int zoff, int zlo, int zhi) {
  extern __shared__ double sm[];
  const int W = 2 * p + 1, WX = TX + 2 * p, WY = TY + 2 * p;
  double *X = sm;              // [WY][WX]
  double *Tk = X + WX * WY;    // [WY][TX]
  double *Tm = Tk + WY * TX;   // [WY][TX]
  __shared__ double red[32];
  const int x0 = blockIdx.x * TX, y0 = zlo + blockIdx.y * TY;
  for (int i = threadIdx.x; i < WX * WY; i += blockDim.x) {   // asynchronous staging (LDGSTS)
    const int wy = i / WX, wx = i - wy * WX;
    const int gx = x0 - p + wx, gy = y0 - p + wy;
    const bool ok = gx >= 0 && gx < n1 && gy >= 0 && gy < n1;
    cp_async8(X + i, x + (ok ? (int64_t)(gy - zoff) * n1 + gx : 0), ok);
  }
  cp_async_wait_all();
  __syncthreads();
  for (int i = threadIdx.x; i < WY * TX; i += blockDim.x) {   // pass along x: K_x X, M_x X
    const int wy = i / TX, lx = i - wy * TX, gx = x0 + lx;
    double sk = 0.0, sm_ = 0.0;
    if (gx < n1) {
      const double *kr = K + (int64_t)gx * W, *mr = M + (int64_t)gx * W, *xr = X + wy * WX + lx;
      for (int t = 0; t < W; ++t) {
        sk = fma(kr[t], xr[t], sk);
        sm_ = fma(mr[t], xr[t], sm_);
      }
    }
    Tk[i] = sk;
    Tm[i] = sm_;
  }
  __syncthreads();
  double sq = 0.0;
  for (int i = threadIdx.x; i < TY * TX; i += blockDim.x) {   // pass along y: M_y Tk + K_y Tm
    const int ly = i / TX, lx = i - ly * TX, gx = x0 + lx, gy = y0 + ly;
    if (gx >= n1 || gy >= zhi) continue;
    const double *kr = K + (int64_t)gy * W, *mr = M + (int64_t)gy * W;
    double acc = 0.0;
    for (int u = 0; u < W; ++u) {
      acc = fma(mr[u], Tk[(ly + u) * TX + lx], acc);
      acc = fma(kr[u], Tm[(ly + u) * TX + lx], acc);
    }
    const int64_t g = (int64_t)(gy - zoff) * n1 + gx;
    const double out = mode ? b[g] - acc : acc;
    y[g] = out;
    sq = fma(out, out, sq);
  }
  if (partial) {
    const double t = block_sum(sq, red);
    if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// 3D tile TX x TY x TZ outputs.
template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(256) k_apply3d(int p, int n1, const double *__restrict__ K,
                                                 const double *__restrict__ M, const double *__restrict__ x,
                                                 const double *__restrict__ b, double *__restrict__ y,
                                                 double *__restrict__ partial, int mode, int zoff, int zlo, int zhi) {
  extern __shared__ double sm[];
  const int W = 2 * p + 1, WX = TX + 2 * p, WY = TY + 2 * p, WZ = TZ + 2 * p;
  double *X = sm;                       // [WZ][WY][WX]
  double *Pa = X + WX * WY * WZ;        // [WZ][WY][TX]  K_x X
  double *Pb = Pa + TX * WY * WZ;       // [WZ][WY][TX]  M_x X
  double *Pc = Pb + TX * WY * WZ;       // [WZ][TY][TX]
  double *Pe = Pc + TX * TY * WZ;
  __shared__ double red[32];
  const int nbx = (n1 + TX - 1) / TX;
  const int x0 = (blockIdx.x % nbx) * TX, y0 = (blockIdx.x / nbx) * TY, z0 = zlo + blockIdx.y * TZ;
  for (int i = threadIdx.x; i < WX * WY * WZ; i += blockDim.x) {   // asynchronous staging (LDGSTS)
    const int wx = i % WX, wy = (i / WX) % WY, wz = i / (WX * WY);
    const int gx = x0 - p + wx, gy = y0 - p + wy, gz = z0 - p + wz;
    const bool ok = gx >= 0 && gx < n1 && gy >= 0 && gy < n1 && gz >= 0 && gz < n1;
    cp_async8(X + i, x + (ok ? ((int64_t)(gz - zoff) * n1 + gy) * n1 + gx : 0), ok);
  }
  cp_async_wait_all();
  __syncthreads();
  for (int i = threadIdx.x; i < TX * WY * WZ; i += blockDim.x) {
    const int lx = i % TX, wyz = i / TX, gx = x0 + lx;
    double sa = 0.0, sb = 0.0;
    if (gx < n1) {
      const double *kr = K + (int64_t)gx * W, *mr = M + (int64_t)gx * W, *xr = X + wyz * WX + lx;
      for (int t = 0; t < W; ++t) {
        sa = fma(kr[t], xr[t], sa);
        sb = fma(mr[t], xr[t], sb);
      }
    }
    Pa[i] = sa;
    Pb[i] = sb;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TX * TY * WZ; i += blockDim.x) {
    const int lx = i % TX, ly = (i / TX) % TY, wz = i / (TX * TY), gy = y0 + ly;
    double sc = 0.0, se = 0.0;
    if (gy < n1) {
      const double *kr = K + (int64_t)gy * W, *mr = M + (int64_t)gy * W;
      for (int u = 0; u < W; ++u) {
        const int j = (wz * WY + ly + u) * TX + lx;
        sc = fma(mr[u], Pa[j], sc);
        sc = fma(kr[u], Pb[j], sc);
        se = fma(mr[u], Pb[j], se);
      }
    }
    Pc[i] = sc;
    Pe[i] = se;
  }
  __syncthreads();
  double sq = 0.0;
  for (int i = threadIdx.x; i < TX * TY * TZ; i += blockDim.x) {
    const int lx = i % TX, ly = (i / TX) % TY, lz = i / (TX * TY);
    const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
    if (gx >= n1 || gy >= n1 || gz >= zhi) continue;
    const double *kr = K + (int64_t)gz * W, *mr = M + (int64_t)gz * W;
    double acc = 0.0;
    for (int v = 0; v < W; ++v) {
      const int j = ((lz + v) * TY + ly) * TX + lx;
      acc = fma(mr[v], Pc[j], acc);
      acc = fma(kr[v], Pe[j], acc);
    }
    const int64_t g = ((int64_t)(gz - zoff) * n1 + gy) * n1 + gx;
    const double out = mode ? b[g] - acc : acc;
    y[g] = out;
    sq = fma(out, out, sq);
  }
  if (partial) {
    const double t = block_sum(sq, red);
    if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

template <typename F>
void ensure_smem(F *kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

// 2D apply, compile-time p, register-blocked (v2).  Tile AT x AT outputs; the (AT+2p)^2 window of x
// is staged by cp.async; pass x: each task = one window row, RX consecutive outputs (loads RX+2p
// values, 2(2p+1)RX FMAs); pass y: each task = one column, RY consecutive outputs.  Axes whose tile
// rows are translation-invariant (A27) keep the 2(2p+1) band coefficients in registers.
constexpr int ARY = 4;
template <int P, int AT>
struct Apl2 {
  static constexpr int ARX = P >= 6 ? 4 : 8;
  static constexpr int W = 2 * P + 1, WN = AT + 2 * P;
  static constexpr int SM = WN * WN + 2 * WN * AT + 4 * AT * W;   // doubles
};

template <int P, int AT, bool TOE>
__device__ __forceinline__ void apl_row(const double *xr, const double *ck, const double *cm, double *ok_, double *om_,
                                        const ToeP &tp) {
  constexpr int W = 2 * P + 1, ARX = Apl2<P, AT>::ARX;
  double v[ARX + 2 * P];
#pragma unroll
  for (int k = 0; k < ARX + 2 * P; ++k) v[k] = xr[k];
#pragma unroll
  for (int i = 0; i < ARX; ++i) {
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int t = 0; t < W; ++t) {
      const double kc = TOE ? tp.k[t] : ck[i * W + t], mc = TOE ? tp.m[t] : cm[i * W + t];
      if (t & 1) { a1 = fma(kc, v[i + t], a1); b1 = fma(mc, v[i + t], b1); }
      else { a0 = fma(kc, v[i + t], a0); b0 = fma(mc, v[i + t], b0); }
    }
    ok_[i] = a0 + a1;
    om_[i] = b0 + b1;
  }
}

template <int P, int AT, bool TOE>
__device__ __forceinline__ void apl_col(const double *tk, const double *tm, const double *ck, const double *cm,
                                        double *out, const ToeP &tp) {
  constexpr int W = 2 * P + 1;
  double a[ARY + 2 * P], c[ARY + 2 * P];
#pragma unroll
  for (int k = 0; k < ARY + 2 * P; ++k) { a[k] = tk[k * AT]; c[k] = tm[k * AT]; }
#pragma unroll
  for (int i = 0; i < ARY; ++i) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const double kc = TOE ? tp.k[u] : ck[i * W + u], mc = TOE ? tp.m[u] : cm[i * W + u];
      s0 = fma(mc, a[i + u], s0);      // M_y (K_x X)
      s1 = fma(kc, c[i + u], s1);      // K_y (M_x X)
    }
    out[i] = s0 + s1;
  }
}

template <int P, int AT>
__global__ void __launch_bounds__(AT * AT / ARY, 2) k_apply2d_t(int n1, const double *__restrict__ K, const double *__restrict__ M,
                                                   const double *__restrict__ x, const double *__restrict__ b,
                                                   double *__restrict__ y, double *__restrict__ partial, int mode,
                                                   int zoff, int zlo, int zhi, int tlo, int thi, const ToeP tp) {
  using A = Apl2<P, AT>;
  constexpr int NT = AT * AT / ARY;
  constexpr int W = A::W, WN = A::WN, ARX = A::ARX;
  extern __shared__ double sm[];
  double *X = sm;                    // [WN][WN]
  double *Tk = X + WN * WN;          // [WN][AT]  K_x X
  double *Tm = Tk + WN * AT;         // [WN][AT]  M_x X
  double *Kx = Tm + WN * AT, *Mx = Kx + AT * W, *Ky = Mx + AT * W, *My = Ky + AT * W;
  __shared__ double red[32];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * AT, y0 = zlo + blockIdx.y * AT;
  const unsigned un = unsigned(n1);
  for (int i = tid; i < WN * WN; i += NT) {
    const int wy = i / WN, wx = i - wy * WN;
    const int gx = x0 - P + wx, gy = y0 - P + wy;
    const bool ok = unsigned(gx) < un && unsigned(gy) < un;
    cp_async8(X + i, x + (ok ? (int64_t)(gy - zoff) * n1 + gx : 0), ok);
  }
  const bool tx = tp.valid && x0 >= tlo && x0 + AT - 1 <= thi, ty = tp.valid && y0 >= tlo && y0 + AT - 1 <= thi;
  for (int i = tid; i < AT * W; i += NT) {   // band rows of boundary tiles only (interior: tp, A27)
    const int l = i / W, t = i - l * W;
    const int gx = x0 + l, gy = y0 + l;
    const bool okx = unsigned(gx) < un, oky = gy < zhi && unsigned(gy) < un;
    if (!tx) {
      cp_async8(Kx + i, K + (okx ? (int64_t)gx * W + t : 0), okx);
      cp_async8(Mx + i, M + (okx ? (int64_t)gx * W + t : 0), okx);
    }
    if (!ty) {
      cp_async8(Ky + i, K + (oky ? (int64_t)gy * W + t : 0), oky);
      cp_async8(My + i, M + (oky ? (int64_t)gy * W + t : 0), oky);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  // pass x: rows wy of the window, segments of ARX outputs
  for (int task = tid; task < WN * (AT / ARX); task += NT) {
    const int wy = task / (AT / ARX), sg = task - wy * (AT / ARX);
    double ok_[ARX], om_[ARX];
    if (tx) apl_row<P, AT, true>(X + wy * WN + sg * ARX, Kx, Mx, ok_, om_, tp);
    else apl_row<P, AT, false>(X + wy * WN + sg * ARX, Kx + sg * ARX * W, Mx + sg * ARX * W, ok_, om_, tp);
#pragma unroll
    for (int i = 0; i < ARX; ++i) {
      Tk[wy * AT + sg * ARX + i] = ok_[i];
      Tm[wy * AT + sg * ARX + i] = om_[i];
    }
  }
  __syncthreads();
  // pass y: columns lx, segments of ARY outputs; y = A x or b - A x
  double sq = 0.0;
  {
    const int lx = tid % AT, sg = tid / AT;   // NT tasks = AT columns x AT/ARY segments
    double out[ARY];
    if (ty) apl_col<P, AT, true>(Tk + sg * ARY * AT + lx, Tm + sg * ARY * AT + lx, Ky, My, out, tp);
    else apl_col<P, AT, false>(Tk + sg * ARY * AT + lx, Tm + sg * ARY * AT + lx, Ky + sg * ARY * W, My + sg * ARY * W, out, tp);
    const int gx = x0 + lx;
#pragma unroll
    for (int i = 0; i < ARY; ++i) {
      const int gy = y0 + sg * ARY + i;
      if (gx < n1 && gy < zhi) {
        const int64_t g = (int64_t)(gy - zoff) * n1 + gx;
        const double v = mode ? b[g] - out[i] : out[i];
        y[g] = v;
        sq = fma(v, v, sq);
      }
    }
  }
  if (partial) {
    const double t = block_sum(sq, red);
    if (tid == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

template <int P>
bool try_apply2d(int p, int64_t n1, const double *K, const double *M, const double *x, const double *b, double *y,
                 double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv, const ToeP *tpp) {
  if (p != P) return false;
  ToeP tp{};
  if (tpp) tp = *tpp;
  const int nz = sv.zhi - sv.zlo;
  const int m = int(n1) - P + 2;
  auto go = [&](auto kern, int at, size_t sm) {
    ensure_smem(kern, sm);
    dim3 grid((unsigned)((n1 + at - 1) / at), (unsigned)((nz + at - 1) / at));
    kern<<<grid, at * at / ARY, sm, st>>>(int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi, 2 * P - 1,
                                          m - 2 - P, tp);
    if (nparts) *nparts = int(grid.x * grid.y);
  };
  // 32x32 tiles; 16x16 when that would leave fewer than two CTAs per SM
  if (((n1 + 31) / 32) * ((nz + 31) / 32) >= 296) go(k_apply2d_t<P, 32>, 32, sizeof(double) * Apl2<P, 32>::SM);
  else go(k_apply2d_t<P, 16>, 16, sizeof(double) * Apl2<P, 16>::SM);
  return true;
}

// 3D apply, z-streaming (v2).  CTA = (x, y) tile of TX x TY outputs and a chunk [zlo, zhi) of
// output planes.  For every input plane gi in [zlo - p, zhi + p): stage its (TY+2p) x (TX+2p) window
// (cp.async, double-buffered), pass x (K_x, M_x) into shared memory, pass y into a RING of 2p+1
// planes holding c = M_y K_x X + K_y M_x X and e = M_y M_x X; output plane go = gi - p is then
// complete: y = [b -] Σ_v (M_z(go, v) c[go-p+v] + K_z(go, v) e[go-p+v]).  Sum-factorised,
// 2(2p+1)(TY+2p)/TY + 3(2p+1) + 2(2p+1) FMAs per output; each x value is read once per CTA.
constexpr int A3TX = 32, A3TY = 16, A3NT = 256;
template <int P>
struct Apl3 {
  static constexpr int W = 2 * P + 1, WX = A3TX + 2 * P, WY = A3TY + 2 * P, NR = 2 * P + 1;
  static constexpr int SM = 2 * WY * WX + 2 * WY * A3TX + 2 * NR * A3TY * A3TX;   // doubles
};

template <int P>
__global__ void __launch_bounds__(A3NT) k_apply3d_s(int n1, const double *__restrict__ K, const double *__restrict__ M,
                                                    const double *__restrict__ x, const double *__restrict__ b,
                                                    double *__restrict__ y, double *__restrict__ partial, int mode,
                                                    int zoff, int zlo0, int zhi0, int zchunk, int tlo, int thi) {
  using A = Apl3<P>;
  constexpr int W = A::W, WX = A::WX, WY = A::WY, NR = A::NR, TX = A3TX, TY = A3TY, NT = A3NT;
  extern __shared__ double sm[];
  double *Xb = sm;                          // [2][WY][WX]
  double *Pa = Xb + 2 * WY * WX;            // [WY][TX]  K_x X
  double *Pb = Pa + WY * TX;                // [WY][TX]  M_x X
  double *Rc = Pb + WY * TX;                // [NR][TY][TX]
  double *Re = Rc + NR * TY * TX;
  __shared__ double red[32];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int zlo = zlo0 + blockIdx.z * zchunk, zhi = min(zhi0, zlo + zchunk);
  const unsigned un = unsigned(n1);
  const bool tx = x0 >= tlo && x0 + TX - 1 <= thi, ty = y0 >= tlo && y0 + TY - 1 <= thi;
  // this thread's band coefficients for pass x rows (lx) and pass y rows (ly): rows of the tile are
  // fixed, so load them once (registers) -- Toeplitz tiles use one row for all
  auto stage = [&](int gi, int buf) {       // window of input plane gi into buffer buf (zero outside)
    double *dst = Xb + buf * WY * WX;
    const bool okz = unsigned(gi) < un;
    for (int i = tid; i < WY * WX; i += NT) {
      const int wy = i / WX, wx = i - wy * WX, gx = x0 - P + wx, gyy = y0 - P + wy;
      const bool ok = okz && unsigned(gx) < un && unsigned(gyy) < un;
      cp_async8(dst + i, x + (ok ? ((int64_t)(gi - zoff) * n1 + gyy) * n1 + gx : 0), ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double sq = 0.0;
  const int gs = zlo - P, ge = zhi + P;
  if (zlo >= zhi) return;
  stage(gs, 0);
  for (int gi = gs; gi < ge; ++gi) {
    const int buf = (gi - gs) & 1;
    if (gi + 1 < ge) {
      stage(gi + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int slot = ((gi % NR) + NR) % NR;
    const bool okz = unsigned(gi) < un;
    if (okz) {
      const double *X = Xb + buf * WY * WX;
      // pass x: tasks = (window row wy, 4 consecutive lx)
      for (int task = tid; task < WY * (TX / 4); task += NT) {
        const int wy = task / (TX / 4), lx0 = (task - wy * (TX / 4)) * 4;
        double v[4 + 2 * P];
#pragma unroll
        for (int k = 0; k < 4 + 2 * P; ++k) v[k] = X[wy * WX + lx0 + k];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int gx = x0 + lx0 + i;
          const bool okx = unsigned(gx) < un;
          const int row = tx ? tlo : (okx ? gx : 0);
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int t = 0; t < W; ++t) {
            const double kc = __ldg(K + (int64_t)row * W + t), mc = __ldg(M + (int64_t)row * W + t);
            a0 = fma(kc, v[i + t], a0);
            a1 = fma(mc, v[i + t], a1);
          }
          Pa[wy * TX + lx0 + i] = okx ? a0 : 0.0;
          Pb[wy * TX + lx0 + i] = okx ? a1 : 0.0;
        }
      }
    }
    __syncthreads();
    // pass y: each thread owns TX*TY/NT (= 2) output columns (lx, ly)
#pragma unroll
    for (int o = 0; o < TX * TY / NT; ++o) {
      const int pt = tid + o * NT, ly = pt / TX, lx = pt - ly * TX;
      double c = 0.0, e = 0.0;
      if (okz) {
        const int gyy = y0 + ly;
        const bool oky = unsigned(gyy) < un;
        const int row = ty ? tlo : (oky ? gyy : 0);
        double c1 = 0.0;
#pragma unroll
        for (int u = 0; u < W; ++u) {
          const double kc = __ldg(K + (int64_t)row * W + u), mc = __ldg(M + (int64_t)row * W + u);
          const double pa = Pa[(ly + u) * TX + lx], pb = Pb[(ly + u) * TX + lx];
          c = fma(mc, pa, c);
          c1 = fma(kc, pb, c1);
          e = fma(mc, pb, e);
        }
        c = oky ? c + c1 : 0.0;
        e = oky ? e : 0.0;
      }
      Rc[(slot * TY + ly) * TX + lx] = c;
      Re[(slot * TY + ly) * TX + lx] = e;
    }
    __syncthreads();
    // output plane go = gi - P complete
    const int go = gi - P;
    if (go >= zlo && go < zhi) {
      const bool tz = go >= tlo && go <= thi;
      const int row = tz ? tlo : go;
#pragma unroll
      for (int o = 0; o < TX * TY / NT; ++o) {
        const int pt = tid + o * NT, ly = pt / TX, lx = pt - ly * TX;
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int v = 0; v < W; ++v) {
          const int sl = ((go - P + v) % NR + NR) % NR;
          s0 = fma(__ldg(M + (int64_t)row * W + v), Rc[(sl * TY + ly) * TX + lx], s0);
          s1 = fma(__ldg(K + (int64_t)row * W + v), Re[(sl * TY + ly) * TX + lx], s1);
        }
        const int gx = x0 + lx, gyy = y0 + ly;
        if (gx < n1 && gyy < n1) {
          const int64_t g = ((int64_t)(go - zoff) * n1 + gyy) * n1 + gx;
          const double val = mode ? b[g] - (s0 + s1) : (s0 + s1);
          y[g] = val;
          sq = fma(val, val, sq);
        }
      }
    }
  }
  if (partial) {
    const double t = block_sum(sq, red);
    if (tid == 0) partial[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
  }
}

// 3D apply v3: z-streaming with the z pass in REGISTERS.  Each thread owns two output columns
// (lx, ly0), (lx, ly0+1); input plane gi's pass-y values c = M_y K_x X + K_y M_x X, e = M_y M_x X are
// added into a register ring of 2p+1 partial outputs (plane loop unrolled by 2p+1, so ring slots are
// compile-time); output plane gi - p is complete after plane gi.  Interior band rows (A27) come from
// the kernel parameter tp (constant-bank operands); boundary rows through L1.
template <int P>
__device__ __forceinline__ void apl3_coef(const ToeP &tp, bool toe, const double *__restrict__ K,
                                          const double *__restrict__ M, int row, int t, double &kc, double &mc) {
  if (toe) { kc = tp.k[t]; mc = tp.m[t]; }
  else { kc = __ldg(K + (int64_t)row * (2 * P + 1) + t); mc = __ldg(M + (int64_t)row * (2 * P + 1) + t); }
}

template <int P>
__global__ void __launch_bounds__(A3NT) k_apply3d_r(int n1, const double *__restrict__ K, const double *__restrict__ M,
                                                    const double *__restrict__ x, const double *__restrict__ b,
                                                    double *__restrict__ y, double *__restrict__ partial, int mode,
                                                    int zoff, int zlo0, int zhi0, int zchunk, int tlo, int thi,
                                                    const ToeP tp) {
  constexpr int W = 2 * P + 1, TX = A3TX, TY = A3TY, NT = A3NT, WX = TX + 2 * P, WY = TY + 2 * P, NR = W;
  constexpr int SEG = 8;                    // pass-x outputs per task
  extern __shared__ double sm[];
  double *Xb = sm;                          // [2][WY][WX]
  double *Pa = Xb + 2 * WY * WX;            // [WY][TX]  K_x X
  double *Pb = Pa + WY * TX;                // [WY][TX]  M_x X
  __shared__ double red[32];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int zlo = zlo0 + blockIdx.z * zchunk, zhi = min(zhi0, zlo + zchunk);
  if (zlo >= zhi) return;
  const unsigned un = unsigned(n1);
  const bool tv = tp.valid != 0;
  const bool tx = tv && x0 >= tlo && x0 + TX - 1 <= thi, ty = tv && y0 >= tlo && y0 + TY - 1 <= thi;
  const int lx = tid % TX, ly0 = 2 * (tid / TX);              // this thread's two output columns
  auto stage = [&](int gi, int buf) {
    double *dst = Xb + buf * WY * WX;
    const bool okz = unsigned(gi) < un;
    for (int i = tid; i < WY * WX; i += NT) {
      const int wy = i / WX, wx = i - wy * WX, gx = x0 - P + wx, gyy = y0 - P + wy;
      const bool ok = okz && unsigned(gx) < un && unsigned(gyy) < un;
      cp_async8(dst + i, x + (ok ? ((int64_t)(gi - zoff) * n1 + gyy) * n1 + gx : 0), ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[NR][2];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r][0] = acc[r][1] = 0.0;
  double sq = 0.0;
  const int gs = zlo - P, ge = zhi + P;
  stage(gs, 0);
  for (int g0 = gs; g0 < ge; g0 += NR) {
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const int gi = g0 + k;
      if (gi >= ge) break;
      const int buf = (gi - gs) & 1;
      if (gi + 1 < ge) {
        stage(gi + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const bool okz = unsigned(gi) < un;
      if (okz) {                                              // pass x: (row, SEG consecutive outputs)
        const double *X = Xb + buf * WY * WX;
        for (int task = tid; task < WY * (TX / SEG); task += NT) {
          const int wy = task / (TX / SEG), l0 = (task - wy * (TX / SEG)) * SEG;
          double v[SEG + 2 * P];
#pragma unroll
          for (int q = 0; q < SEG + 2 * P; ++q) v[q] = X[wy * WX + l0 + q];
#pragma unroll
          for (int i = 0; i < SEG; ++i) {
            const int gx = x0 + l0 + i;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int t = 0; t < W; ++t) {
              double kc, mc;
              apl3_coef<P>(tp, tx, K, M, min(gx, n1 - 1), t, kc, mc);
              a0 = fma(kc, v[i + t], a0);
              a1 = fma(mc, v[i + t], a1);
            }
            Pa[wy * TX + l0 + i] = gx < n1 ? a0 : 0.0;
            Pb[wy * TX + l0 + i] = gx < n1 ? a1 : 0.0;
          }
        }
      }
      __syncthreads();
      // pass y for the two columns, then scatter into the register ring (output go = gi + P - t)
      double c[2] = {0.0, 0.0}, e[2] = {0.0, 0.0};
      if (okz) {
        double pa[2 + 2 * P], pb[2 + 2 * P];
#pragma unroll
        for (int u = 0; u < 2 + 2 * P; ++u) { pa[u] = Pa[(ly0 + u) * TX + lx]; pb[u] = Pb[(ly0 + u) * TX + lx]; }
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int gyy = y0 + ly0 + o;
          double c1 = 0.0;
#pragma unroll
          for (int u = 0; u < W; ++u) {
            double kc, mc;
            apl3_coef<P>(tp, ty, K, M, min(gyy, n1 - 1), u, kc, mc);
            c[o] = fma(mc, pa[o + u], c[o]);
            c1 = fma(kc, pb[o + u], c1);
            e[o] = fma(mc, pb[o + u], e[o]);
          }
          c[o] = gyy < n1 ? c[o] + c1 : 0.0;
          e[o] = gyy < n1 ? e[o] : 0.0;
        }
      }
#pragma unroll
      for (int t = 0; t < W; ++t) {                           // output go = gi + P - t gets tap t
        const int go = gi + P - t;
        if (go < zlo || go >= zhi) continue;
        const bool tz = tv && go >= tlo && go <= thi;
        double kc, mc;
        apl3_coef<P>(tp, tz, K, M, go, t, kc, mc);
        const int slot = (k + P - t + 2 * NR) % NR;            // compile-time after unrolling
#pragma unroll
        for (int o = 0; o < 2; ++o) acc[slot][o] = fma(mc, c[o], fma(kc, e[o], acc[slot][o]));
      }
      const int go = gi - P;                                   // complete now
      if (go >= zlo && go < zhi) {
        const int slot = (k + P + 1) % NR;
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int gx = x0 + lx, gyy = y0 + ly0 + o;
          if (gx < n1 && gyy < n1) {
            const int64_t gg = ((int64_t)(go - zoff) * n1 + gyy) * n1 + gx;
            const double val = mode ? b[gg] - acc[slot][o] : acc[slot][o];
            y[gg] = val;
            sq = fma(val, val, sq);
          }
          acc[slot][o] = 0.0;
        }
      }
    }
  }
  if (partial) {
    const double t = block_sum(sq, red);
    if (tid == 0) partial[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
  }
}

int apply3d_zchunks(int64_t n1, int nz) {   // z chunks: about two CTAs per SM, chunks >= 8 planes
  const int64_t tiles = ((n1 + A3TX - 1) / A3TX) * ((n1 + A3TY - 1) / A3TY);
  int ch = int(std::max<int64_t>(1, (296 + tiles - 1) / tiles));
  ch = std::min(ch, std::max(1, nz / 8));
  return ch;
}

template <int P>
bool try_apply3d(int p, int64_t n1, const double *K, const double *M, const double *x, const double *b, double *y,
                 double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv, const ToeP *tpp) {
  if (p != P) return false;
  const int nz = sv.zhi - sv.zlo;
  const int ch = apply3d_zchunks(n1, nz), zchunk = (nz + ch - 1) / ch;
  const int m = int(n1) - P + 2;
  dim3 grid((unsigned)((n1 + A3TX - 1) / A3TX), (unsigned)((n1 + A3TY - 1) / A3TY), (unsigned)ch);
  const char *ev = std::getenv("IGA2L_APPLY3D");   // 2 (default): shared-memory ring; 3: register z ring
  if (ev && ev[0] == '3') {                        // (measured slower: C5 2.07 vs 1.33 ms)
    ToeP tp{};
    if (tpp) tp = *tpp;
    constexpr int WX = A3TX + 2 * P, WY = A3TY + 2 * P;
    constexpr size_t sm = sizeof(double) * (2 * WY * WX + 2 * WY * A3TX);
    ensure_smem(k_apply3d_r<P>, sm);
    k_apply3d_r<P><<<grid, A3NT, sm, st>>>(int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi, zchunk,
                                           2 * P - 1, m - 2 - P, tp);
    if (nparts) *nparts = int(grid.x * grid.y * grid.z);
    return true;
  }
  constexpr size_t sm = sizeof(double) * Apl3<P>::SM;
  ensure_smem(k_apply3d_s<P>, sm);
  k_apply3d_s<P><<<grid, A3NT, sm, st>>>(int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi, zchunk,
                                         2 * P - 1, m - 2 - P);
  if (nparts) *nparts = int(grid.x * grid.y * grid.z);
  return true;
}

constexpr int A2X = 32, A2Y = 8, A3X = 8, A3Y = 8, A3Z = 4;
static const bool g_transfer_v2 = [] {
  const char *e = std::getenv("IGA2L_TRANSFER_V2");
  return !(e && e[0] == '0');
}();
static const bool g_apply_v2 = [] {
  const char *e = std::getenv("IGA2L_APPLY_V2");
  return !(e && e[0] == '0');
}();

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
                                                 int nb1, int zoff) {
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

  for (int i = threadIdx.x; i < s2; i += blockDim.x) {
    Vx[i] = Vt[(int64_t)cx * s2 + i];
    Vy[i] = Vt[(int64_t)cy * s2 + i];
    if (DIM == 3) Vz[i] = Vt[(int64_t)cz * s2 + i];
  }
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    Lx[i] = lamt[(int64_t)cx * s + i];
    Ly[i] = lamt[(int64_t)cy * s + i];
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
        const double *kr = K + (int64_t)gy * W, *mr = M + (int64_t)gy * W;
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

// =============================== band transform along one axis ===========================
// Columns valid in [clo, chi), stored from column coff on (nin stored columns per outer slice);
// output rows r in [rlo, rhi), stored from row rlo on (rhi - rlo rows per outer slice).
__global__ void k_band_axis(const double *__restrict__ in, double *__restrict__ out, int64_t outer, int nin,
                            int64_t inner, int rows, int W, const int *__restrict__ lo,
                            const double *__restrict__ c, int acc, int clo, int chi, int coff, int rlo, int rhi) {
  const int nr = rhi - rlo;
  const int64_t total = outer * nr * inner;
  (void)rows;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % inner;
    const int r = rlo + int((idx / inner) % nr);
    const int64_t o = idx / (inner * nr);
    const int l0 = lo[r];
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {            // all gathers independent (W <= 16 checked at setup)
      const int col = l0 + k;
      const bool ok = k < W && col >= clo && col < chi;
      const double v = ok ? c[(int64_t)r * W + k] * in[(o * nin + (col - coff)) * inner + i] : 0.0;
      if (k & 1) s1 += v; else s0 += v;
    }
    const double s = s0 + s1;
    out[idx] = acc ? out[idx] + s : s;
  }
}

// =============================== q-level kernels ==========================================
template <int DIM>
__device__ __forceinline__ double q_apply_point(int q, int n, const double *K, const double *M, const double *x,
                                                int ix, int iy, int iz, double *diag) {
  const int W = 2 * q + 1;
  double acc = 0.0;
  const double *kx = K + (int64_t)ix * W, *mx = M + (int64_t)ix * W;
  const double *ky = K + (int64_t)iy * W, *my = M + (int64_t)iy * W;
  if (DIM == 2) {
    for (int u = 0; u < W; ++u) {
      const int jy = iy + u - q;
      if (jy < 0 || jy >= n) continue;
      for (int t = 0; t < W; ++t) {
        const int jx = ix + t - q;
        if (jx < 0 || jx >= n) continue;
        acc = fma(kx[t] * my[u] + mx[t] * ky[u], x[(int64_t)jy * n + jx], acc);
      }
    }
    *diag = kx[q] * my[q] + mx[q] * ky[q];
  } else {
    const double *kz = K + (int64_t)iz * W, *mz = M + (int64_t)iz * W;
    for (int v = 0; v < W; ++v) {
      const int jz = iz + v - q;
      if (jz < 0 || jz >= n) continue;
      for (int u = 0; u < W; ++u) {
        const int jy = iy + u - q;
        if (jy < 0 || jy >= n) continue;
        for (int t = 0; t < W; ++t) {
          const int jx = ix + t - q;
          if (jx < 0 || jx >= n) continue;
          const double a = kx[t] * my[u] * mz[v] + mx[t] * ky[u] * mz[v] + mx[t] * my[u] * kz[v];
          acc = fma(a, x[((int64_t)jz * n + jy) * n + jx], acc);
        }
      }
    }
    *diag = kx[q] * my[q] * mz[q] + mx[q] * ky[q] * mz[q] + mx[q] * my[q] * kz[q];
  }
  return acc;
}

template <int DIM>
__global__ void k_q_gs(int q, int n, const double *__restrict__ K, const double *__restrict__ M,
                       const double *__restrict__ b, double *__restrict__ x, int c0, int c1, int c2, int na0,
                       int na1, int64_t total) {
  const int st = q + 1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int ix = c0 + st * int(idx % na0);
    const int iy = c1 + st * int((idx / na0) % na1);
    const int iz = (DIM == 3) ? c2 + st * int(idx / ((int64_t)na0 * na1)) : 0;
    double dg;
    const double ax = q_apply_point<DIM>(q, n, K, M, x, ix, iy, iz, &dg);
    const int64_t g = ((int64_t)iz * n + iy) * n + ix;
    x[g] += (b[g] - ax) / dg;
  }
}

template <int DIM>
__global__ void k_q_resid(int q, int n, const double *__restrict__ K, const double *__restrict__ M,
                          const double *__restrict__ b, const double *__restrict__ x, double *__restrict__ r,
                          int64_t total) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int ix = int(idx % n), iy = int((idx / n) % n), iz = (DIM == 3) ? int(idx / ((int64_t)n * n)) : 0;
    double dg;
    r[idx] = b[idx] - q_apply_point<DIM>(q, n, K, M, x, ix, iy, iz, &dg);
  }
}

__global__ void k_dense_mv(int N, const double *__restrict__ A, const double *__restrict__ b, double *__restrict__ x) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= N) return;
  double s = 0.0;
  for (int j = lane; j < N; j += 32) s = fma(A[(int64_t)warp * N + j], b[j], s);
  s = warp_sum(s);
  if (lane == 0) x[warp] = s;
}

__global__ void k_sum_partials(const double *__restrict__ partial, int n, double *out, double *hist, int *count,
                               int cap) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    out[0] = s;
    if (hist && *count < cap) {
      hist[*count] = sqrt(s);
      *count += 1;
    }
  }
}

__global__ void k_tensor_rhs(int dim, int64_t n1, const double *__restrict__ g, double scale, double *__restrict__ b,
                             int64_t total) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double v = scale * g[idx % n1] * g[(idx / n1) % n1];
    if (dim == 3) v *= g[idx / (n1 * n1)];
    b[idx] = v;
  }
}

inline int grid_for(int64_t total, int bs) {
  int64_t g = (total + bs - 1) / bs;
  return int(std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 32));
}

size_t apply_smem(int dim, int p) {
  if (dim == 2) return sizeof(double) * ((A2X + 2 * p) * (A2Y + 2 * p) + 2 * (A2Y + 2 * p) * A2X);
  const size_t wx = A3X + 2 * p, wy = A3Y + 2 * p, wz = A3Z + 2 * p;
  return sizeof(double) * (wx * wy * wz + 2 * A3X * wy * wz + 2 * A3X * A3Y * wz);
}

size_t schwarz_smem(int dim, int p, int s) {
  const size_t Wn = s + 2 * p, s2 = s * s, sd = dim == 3 ? s2 * s : s2;
  const size_t nX = dim == 3 ? Wn * Wn * Wn : Wn * Wn;
  const size_t nP = dim == 3 ? s * Wn * Wn : s * Wn;
  const size_t nC = dim == 3 ? s2 * Wn : 0;
  return sizeof(double) * (nX + 2 * nP + 2 * nC + 3 * sd + 3 * s2 + 3 * s);
}


}  // namespace

// first centre >= lo with residue c (mod D) and the number of such centres below hi
void centre_range(int c, int D, int lo, int hi, int *first, int *count) {
  int f = c;
  if (f < lo) f += ((lo - f + D - 1) / D) * D;
  *first = f;
  *count = (f < hi) ? (hi - 1 - f) / D + 1 : 0;
}

int apply_num_partials(int dim, int p, int64_t n1) {
  (void)p;
  if (dim == 2) {   // the most tiles any 2D apply variant launches
    const int64_t v1 = ((n1 + A2X - 1) / A2X) * ((n1 + A2Y - 1) / A2Y), v2 = ((n1 + 15) / 16) * ((n1 + 15) / 16);
    return int(std::max(v1, v2));
  }
  const int64_t v1 = ((n1 + A3X - 1) / A3X) * ((n1 + A3Y - 1) / A3Y) * ((n1 + A3Z - 1) / A3Z);
  const int64_t v2 = ((n1 + A3TX - 1) / A3TX) * ((n1 + A3TY - 1) / A3TY) * apply3d_zchunks(n1, int(n1));
  return int(std::max(v1, v2));
}

void launch_apply(int dim, int p, int64_t n1, const double *K, const double *M, const double *x, const double *b,
                  double *y, double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv, const ToeP *tp) {
  if (sv.zhi < 0) sv = SlabView{0, 0, int(n1)};
  const int nz = sv.zhi - sv.zlo;
  const size_t sm = apply_smem(dim, p);
  if (nz <= 0) return;
  if (dim == 2 && g_apply_v2 &&
      (try_apply2d<1>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply2d<2>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply2d<3>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply2d<4>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply2d<5>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply2d<6>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply2d<7>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply2d<8>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp)))
    return;
  if (dim == 3 && g_apply_v2 &&
      (try_apply3d<1>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply3d<2>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply3d<3>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply3d<4>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply3d<5>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp) ||
       try_apply3d<6>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp)))
    return;
  if (dim == 2) {
    dim3 grid((unsigned)((n1 + A2X - 1) / A2X), (unsigned)((nz + A2Y - 1) / A2Y));
    ensure_smem(k_apply2d<A2X, A2Y>, sm);
    k_apply2d<A2X, A2Y><<<grid, 256, sm, st>>>(p, int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi);
    if (nparts) *nparts = int(grid.x * grid.y);
  } else {
    const unsigned nbx = unsigned((n1 + A3X - 1) / A3X), nby = unsigned((n1 + A3Y - 1) / A3Y);
    dim3 grid(nbx * nby, (unsigned)((nz + A3Z - 1) / A3Z));
    ensure_smem(k_apply3d<A3X, A3Y, A3Z>, sm);
    k_apply3d<A3X, A3Y, A3Z><<<grid, 256, sm, st>>>(p, int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi);
    if (nparts) *nparts = int(grid.x * grid.y);
  }
}

void launch_schwarz_colour(int dim, int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                           const double *lam, const double *b, double *x, int colour, int D, cudaStream_t st,
                           SlabView sv) {
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
    k_schwarz<2><<<nblk, 128, sm, st>>>(p, s, int(n1), K, M, V, lam, b, x, c0, fl, 0, D, nb0, nb1, sv.zoff);
  } else {
    ensure_smem(k_schwarz<3>, sm);
    k_schwarz<3><<<nblk, 128, sm, st>>>(p, s, int(n1), K, M, V, lam, b, x, c0, c1, fl, D, nb0, nb1, sv.zoff);
  }
}

void launch_band_axis(const double *in, double *out, int64_t outer, int nin, int64_t inner, const Band1D &B,
                      int accumulate, cudaStream_t st, int clo, int chi, int coff, int rlo, int rhi) {
  if (chi < 0) { clo = 0; chi = nin; coff = 0; }
  if (rhi < 0) { rlo = 0; rhi = B.rows; }
  const int64_t total = outer * (rhi - rlo) * inner;
  if (total <= 0) return;
  k_band_axis<<<grid_for(total, 256), 256, 0, st>>>(in, out, outer, nin, inner, B.rows, B.W, B.lo, B.c, accumulate,
                                                   clo, chi, coff, rlo, rhi);
}

void launch_q_gs_colour(int dim, int q, int n, const double *K, const double *M, const double *b, double *x,
                        int colour, cudaStream_t st) {
  const int st_ = q + 1;
  const int c0 = colour % st_, c1 = (colour / st_) % st_, c2 = (dim == 3) ? colour / (st_ * st_) : 0;
  if (c0 >= n || c1 >= n || c2 >= n) return;
  const int na0 = (n - c0 + q) / st_, na1 = (n - c1 + q) / st_, na2 = (dim == 3) ? (n - c2 + q) / st_ : 1;
  const int64_t total = (int64_t)na0 * na1 * na2;
  if (dim == 2)
    k_q_gs<2><<<grid_for(total, 128), 128, 0, st>>>(q, n, K, M, b, x, c0, c1, c2, na0, na1, total);
  else
    k_q_gs<3><<<grid_for(total, 128), 128, 0, st>>>(q, n, K, M, b, x, c0, c1, c2, na0, na1, total);
}

void launch_q_residual(int dim, int q, int n, const double *K, const double *M, const double *b, const double *x,
                       double *r, cudaStream_t st) {
  int64_t total = (int64_t)n * n;
  if (dim == 3) total *= n;
  if (dim == 2)
    k_q_resid<2><<<grid_for(total, 128), 128, 0, st>>>(q, n, K, M, b, x, r, total);
  else
    k_q_resid<3><<<grid_for(total, 128), 128, 0, st>>>(q, n, K, M, b, x, r, total);
}

void launch_dense_mv(int N, const double *Ainv, const double *b, double *x, cudaStream_t st) {
  const int warps_per_block = 8;
  k_dense_mv<<<(N + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(N, Ainv, b, x);
}

void launch_sum_partials(const double *partial, int n, double *out, double *hist, int *count, int cap,
                         cudaStream_t st) {
  k_sum_partials<<<1, 256, 0, st>>>(partial, n, out, hist, count, cap);
}

void launch_tensor_rhs(int dim, int64_t n1, const double *g, double scale, double *b, cudaStream_t st) {
  int64_t total = n1 * n1;
  if (dim == 3) total *= n1;
  k_tensor_rhs<<<grid_for(total, 256), 256, 0, st>>>(dim, n1, g, scale, b, total);
}

}  // namespace iga2l

// ============================================================================================
// Optimised paths (v2): warp-per-block 2D Schwarz colour kernel (compile-time p, s), single-CTA
// V-cycle tail, direct 2D tensor transfers.
// ============================================================================================
namespace iga2l {
namespace {

// barrier for the G warps of one Schwarz block (named barrier 1 + group; __syncwarp if G == 1)
// (barrier ids are compile-time constants for groups 0..3 so that ptxas reserves only the ids used)
template <int G>
__device__ __forceinline__ void group_sync(int group) {
  if (G == 1) {
    __syncwarp();
    return;
  }
  switch (group) {
    case 0: asm volatile("bar.sync 1, %0;" ::"n"(32 * G) : "memory"); break;
    case 1: asm volatile("bar.sync 2, %0;" ::"n"(32 * G) : "memory"); break;
    case 2: asm volatile("bar.sync 3, %0;" ::"n"(32 * G) : "memory"); break;
    case 3: asm volatile("bar.sync 4, %0;" ::"n"(32 * G) : "memory"); break;
    default: asm volatile("bar.sync %0, %1;" ::"r"(group + 1), "n"(32 * G) : "memory"); break;
  }
}

// One 2D Schwarz block solve by a group of G warps (GT = 32 G threads), compile-time p, s.
// Per-group shared memory (PER doubles): x window, two pass buffers, r_B, Z, b_B, the block's 1D band
// rows and FD tables.  Phases: load_const (band rows, FD tables, b_B: independent of the sweep state),
// load_x (the (s+2p)^2 window of x), compute (pass x: K_x X, M_x X; pass y: r_B = b_B - (A x)_B;
// Z = (Vx^T R Vy) ./ (λx + λy); δ = Vx Z Vy^T; x_B += δ).  FMA chains split over two accumulators.
template <int P, int S, int G>
struct Blk2 {
  static constexpr int W = 2 * P + 1, Wn = S + 2 * P, w = (S - 1) / 2, S2 = S * S, GT = 32 * G;
  static constexpr int PER = Wn * Wn + 2 * S * Wn + 3 * S2 + 4 * S * W + 2 * S2 + 2 * S;

  __device__ static __forceinline__ void load_const(double *X, int lane, int n1, int cx, int cy,
                                                    const double *__restrict__ K, const double *__restrict__ M,
                                                    const double *__restrict__ Vt, const double *__restrict__ lamt,
                                                    const double *__restrict__ b, int zoff) {
    double *Pa = X + Wn * Wn, *Pb = Pa + S * Wn, *R = Pb + S * Wn, *Q = R + S2, *Bb = Q + S2;
    double *Kx = Bb + S2, *Mx = Kx + S * W, *Ky = Mx + S * W, *My = Ky + S * W;
    double *Vx = My + S * W, *Vy = Vx + S2, *Lx = Vy + S2, *Ly = Lx + S;
    const int bx = cx - w, by = cy - w;
    const unsigned un = unsigned(n1);
    for (int i = lane; i < S * W; i += GT) {
      const int l = i / W, t = i - l * W;
      const int gx = bx + l, gy = by + l;
      const bool okx = unsigned(gx) < un, oky = unsigned(gy) < un;
      cp_async8(Kx + i, K + (okx ? (int64_t)gx * W + t : 0), okx);
      cp_async8(Mx + i, M + (okx ? (int64_t)gx * W + t : 0), okx);
      cp_async8(Ky + i, K + (oky ? (int64_t)gy * W + t : 0), oky);
      cp_async8(My + i, M + (oky ? (int64_t)gy * W + t : 0), oky);
    }
    for (int i = lane; i < S2; i += GT) {
      const int ly = i / S, lx = i - ly * S, gx = bx + lx, gy = by + ly;
      const bool ok = unsigned(gx) < un && unsigned(gy) < un;
      cp_async8(Bb + i, b + (ok ? (int64_t)(gy - zoff) * n1 + gx : 0), ok);
      cp_async8(Vx + i, Vt + (int64_t)cx * S2 + i, true);
      cp_async8(Vy + i, Vt + (int64_t)cy * S2 + i, true);
    }
    if (lane < S) {
      cp_async8(Lx + lane, lamt + (int64_t)cx * S + lane, true);
      cp_async8(Ly + lane, lamt + (int64_t)cy * S + lane, true);
    }
  }

  // CG: read x through L2 only (other SMs update it inside the same kernel)
  template <bool CG>
  __device__ static __forceinline__ void load_x(double *X, int lane, int n1, int cx, int cy,
                                                const double *x, int zoff) {
    const int ox = cx - w - P, oy = cy - w - P;
    const unsigned un = unsigned(n1);
    if (CG) {   // registers, L2 only (ld.global.cg); all loads issued before the stores
      constexpr int IT = (Wn * Wn + GT - 1) / GT;
      double v[IT];
#pragma unroll
      for (int k = 0; k < IT; ++k) {
        const int i = lane + k * GT, wy = i / Wn, wx = i - wy * Wn;
        const int gx = ox + wx, gy = oy + wy;
        v[k] = (i < Wn * Wn && unsigned(gx) < un && unsigned(gy) < un) ? __ldcg(x + (int64_t)(gy - zoff) * n1 + gx) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < IT; ++k)
        if (lane + k * GT < Wn * Wn) X[lane + k * GT] = v[k];
    } else {
      for (int i = lane; i < Wn * Wn; i += GT) {
        const int wy = i / Wn, wx = i - wy * Wn;
        const int gx = ox + wx, gy = oy + wy;
        const bool ok = unsigned(gx) < un && unsigned(gy) < un;
        cp_async8(X + i, x + (ok ? (int64_t)(gy - zoff) * n1 + gx : 0), ok);
      }
    }
    cp_async_wait_all();   // this thread's copies (const and x) landed; compute() syncs the group
  }

  __device__ static __forceinline__ void compute(double *X, int lane, int group, int n1, int cx, int cy, double *x,
                                                 int zoff) {
    double *Pa = X + Wn * Wn, *Pb = Pa + S * Wn, *R = Pb + S * Wn, *Q = R + S2, *Bb = Q + S2;
    double *Kx = Bb + S2, *Mx = Kx + S * W, *Ky = Mx + S * W, *My = Ky + S * W;
    double *Vx = My + S * W, *Vy = Vx + S2, *Lx = Vy + S2, *Ly = Lx + S;
    const int bx = cx - w, by = cy - w;
    const unsigned un = unsigned(n1);
    group_sync<G>(group);
#pragma unroll
    for (int i = lane; i < S * Wn; i += GT) {          // pass x: K_x X, M_x X on the block columns
      const int wy = i / S, lx = i - wy * S;
      const double *kr = Kx + lx * W, *mr = Mx + lx * W, *xr = X + wy * Wn + lx;
      double sa0 = 0.0, sb0 = 0.0, sa1 = 0.0, sb1 = 0.0;
#pragma unroll
      for (int t = 0; t + 1 < W; t += 2) {
        sa0 = fma(kr[t], xr[t], sa0);
        sb0 = fma(mr[t], xr[t], sb0);
        sa1 = fma(kr[t + 1], xr[t + 1], sa1);
        sb1 = fma(mr[t + 1], xr[t + 1], sb1);
      }
      sa0 = fma(kr[W - 1], xr[W - 1], sa0);            // W = 2P+1 is odd
      sb0 = fma(mr[W - 1], xr[W - 1], sb0);
      Pa[i] = sa0 + sa1;
      Pb[i] = sb0 + sb1;
    }
    group_sync<G>(group);
#pragma unroll
    for (int i = lane; i < S2; i += GT) {              // pass y, block residual r_B = b_B - (A x)_B
      const int ly = i / S, lx = i - ly * S;
      const double *kr = Ky + ly * W, *mr = My + ly * W;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int u = 0; u < W; ++u) {
        a0 = fma(mr[u], Pa[(ly + u) * S + lx], a0);
        a1 = fma(kr[u], Pb[(ly + u) * S + lx], a1);
      }
      R[i] = Bb[i] - (a0 + a1);                        // rows/cols outside the grid: band rows are 0
    }
    group_sync<G>(group);
#pragma unroll
    for (int i = lane; i < S2; i += GT) {              // Z[k][j] = Σ_{ly,lx} Vx[lx][j] R[ly][lx] Vy[ly][k] / (λx_j + λy_k)
      const int k = i / S, j = i - k * S;
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int ly = 0; ly < S; ++ly) {
        double t = 0.0;
#pragma unroll
        for (int lx = 0; lx < S; ++lx) t = fma(Vx[lx * S + j], R[ly * S + lx], t);
        if (ly & 1) z1 = fma(Vy[ly * S + k], t, z1); else z0 = fma(Vy[ly * S + k], t, z0);
      }
      Q[i] = (z0 + z1) / (Lx[j] + Ly[k]);
    }
    group_sync<G>(group);
#pragma unroll
    for (int i = lane; i < S2; i += GT) {              // δ[ly][lx] = Σ_{k,j} Vy[ly][k] Vx[lx][j] Z[k][j];  x_B += δ
      const int ly = i / S, lx = i - ly * S, gx = bx + lx, gy = by + ly;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int k = 0; k < S; ++k) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < S; ++j) t = fma(Vx[lx * S + j], Q[k * S + j], t);
        if (k & 1) d1 = fma(Vy[ly * S + k], t, d1); else d0 = fma(Vy[ly * S + k], t, d0);
      }
      if (unsigned(gx) < un && unsigned(gy) < un) x[(int64_t)(gy - zoff) * n1 + gx] = X[(ly + P) * Wn + lx + P] + (d0 + d1);
    }
  }
};

// One colour: WPB Schwarz blocks (groups of G warps) per CTA; only group barriers inside.
template <int P, int S, int WPB, int G>
__global__ void __launch_bounds__(WPB * G * 32) k_schwarz2d_w(int n1, const double *__restrict__ K,
                                                         const double *__restrict__ M, const double *__restrict__ Vt,
                                                         const double *__restrict__ lamt,
                                                         const double *__restrict__ b, double *__restrict__ x,
                                                         int c0, int c1, int D, int nb0, int nblk, int zoff) {
  using B = Blk2<P, S, G>;
  extern __shared__ double sm[];
  const int warp = threadIdx.x / B::GT, lane = threadIdx.x % B::GT;
  const int bid = blockIdx.x * WPB + warp;
  if (bid >= nblk) return;                              // whole group exits together
  double *X = sm + warp * B::PER;
  const int j1 = bid / nb0, j0 = bid - j1 * nb0;
  const int cx = c0 + D * j0, cy = c1 + D * j1;
  // Programmatic dependent launch: let the next colour's grid start now; everything that does not
  // depend on the previous colour is loaded before griddepcontrol.wait.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  B::load_const(X, lane, n1, cx, cy, K, M, Vt, lamt, b, zoff);
  asm volatile("griddepcontrol.wait;" ::: "memory");   // previous colour complete and visible
  B::template load_x<false>(X, lane, n1, cx, cy, x, zoff);
  B::compute(X, lane, warp, n1, cx, cy, x, zoff);
}

// programmatic dependent launch between colour kernels (IGA2L_PDL=1; off by default)
int g_use_pdl = [] {
  const char *e = std::getenv("IGA2L_PDL");
  return (e && e[0] == '1') ? 1 : 0;
}();

template <int P, int S, int WPB, int G>
bool try_schwarz2d(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                   const double *b, double *x, int c0, int c1, int D, int nb0, int nblk, int zoff, cudaStream_t st) {
  if (p != P || s != S) return false;
  constexpr size_t sm = sizeof(double) * WPB * Blk2<P, S, G>::PER;
  ensure_smem(k_schwarz2d_w<P, S, WPB, G>, sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((nblk + WPB - 1) / WPB);
  cfg.blockDim = dim3(WPB * G * 32);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_use_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_schwarz2d_w<P, S, WPB, G>, int(n1), K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff);
  return true;
}

// ---------------- persistent 2D sweep: all D^2 colours in ONE launch -------------------------
// CTA t owns tile t of block centres (D*AX x D*AY, aligned to D, so each colour has the same AX*AY
// block positions in every tile) for the whole sweep; groups of G warps solve its blocks of the
// current colour.  Colour c of tile T may start once T and its 8 neighbour tiles have finished colour
// c-1 (per-tile progress counters done[], release/acquire at GPU scope): only blocks within
// 2w + p < D of each other interact, so this reproduces the colour-major multiplicative sweep exactly
// (reading A4).  The grid is launched cooperatively (all tiles co-resident, so the waits cannot
// deadlock).  done[] counts colours monotonically across launches: the launch's base is ctl[0], and
// the last CTA to finish advances it by D^2.
constexpr int kFlagStride = 32;   // one progress counter per 128-byte line
template <int P, int S, int AX, int AY, int NB, int G>
__global__ void __launch_bounds__(NB * G * 32) k_sweep2d_persist(int n1, const double *__restrict__ K,
                                                                 const double *__restrict__ M,
                                                                 const double *__restrict__ Vt,
                                                                 const double *__restrict__ lamt,
                                                                 const double *__restrict__ b, double *x, int ntx,
                                                                 int nty, unsigned *ctl, unsigned *done) {
  using B = Blk2<P, S, G>;
  constexpr int D = S + P, TX = D * AX, TY = D * AY, NC = D * D, NBLK = AX * AY;
  extern __shared__ double sm[];
  __shared__ unsigned s_base;
  const int group = threadIdx.x / B::GT, lane = threadIdx.x % B::GT;
  double *X = sm + group * B::PER;
  const int T = blockIdx.x, tx = T % ntx, ty = T / ntx;
  if (threadIdx.x == 0) s_base = *reinterpret_cast<volatile unsigned *>(ctl);
  __syncthreads();
  const unsigned base = s_base;
  for (int c = 0; c < NC; ++c) {
    auto centre = [&](int blk, int *cx, int *cy) {
      *cx = tx * TX + (c % D) + D * (blk % AX);
      *cy = ty * TY + (c / D) + D * (blk / AX);
      return *cx < n1 && *cy < n1;
    };
    int cx, cy;
    if (group < NBLK && centre(group, &cx, &cy))       // first block's constants overlap the wait
      B::load_const(X, lane, n1, cx, cy, K, M, Vt, lamt, b, 0);
    if (c > 0 && threadIdx.x < 9) {                    // wait: this tile and its neighbours done with c-1
      const int ux = tx + int(threadIdx.x % 3) - 1, uy = ty + int(threadIdx.x / 3) - 1;
      if (ux >= 0 && ux < ntx && uy >= 0 && uy < nty) {
        const volatile unsigned *f = done + kFlagStride * (uy * ntx + ux);
        while (int(*f - (base + unsigned(c))) < 0) {
        }
        __threadfence();                               // acquire side of the flag handshake
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int blk = group; blk < NBLK; blk += NB) {     // this group's blocks of colour c in the tile
      if (!centre(blk, &cx, &cy)) continue;
      if (blk != group) B::load_const(X, lane, n1, cx, cy, K, M, Vt, lamt, b, 0);
      B::template load_x<true>(X, lane, n1, cx, cy, x, 0);
      B::compute(X, lane, group, n1, cx, cy, x, 0);
      group_sync<G>(group);                            // the group's smem is reused by its next block
    }
    __syncthreads();                                   // every warp's x stores precede ...
    if (threadIdx.x == 0) {                            // ... the release by thread 0 (grid-sync pattern)
      __threadfence();
      *reinterpret_cast<volatile unsigned *>(done + kFlagStride * T) = base + unsigned(c) + 1u;
    }
  }
  if (threadIdx.x == 0) {                              // last CTA out advances the base
    __threadfence();
    if (atomicAdd(ctl + 1, 1u) == gridDim.x - 1) {
      ctl[1] = 0;
      __threadfence();
      atomicAdd(ctl, unsigned(NC));
    }
  }
}

template <int P, int S, int AX, int AY, int NB, int G>
int try_sweep2d_persist(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                        const double *b, double *x, unsigned *ctl, unsigned *done, int max_tiles, cudaStream_t st,
                        bool launch) {
  if (p != P || s != S) return -1;
  constexpr int D = S + P;
  const int ntx = int((n1 + D * AX - 1) / (D * AX)), nty = int((n1 + D * AY - 1) / (D * AY));
  const int ntiles = ntx * nty;
  constexpr size_t sm = sizeof(double) * NB * Blk2<P, S, G>::PER;
  auto kern = k_sweep2d_persist<P, S, AX, AY, NB, G>;
  if (!launch) {   // feasibility: every tile co-resident
    ensure_smem(kern, sm);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NB * G * 32, sm) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return (ntiles <= per_sm * nsm && ntiles <= max_tiles) ? ntiles : 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ntiles);
  cfg.blockDim = dim3(NB * G * 32);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, int(n1), K, M, V, lam, b, x, ntx, nty, ctl, done);
  return ntiles;
}

// 2D tensor transfer, direct: out[ry][rx] (+)= Σ_{ky,kx} c[ry][ky] c[rx][kx] in[lo[ry]+ky][lo[rx]+kx].
// The band loops are unrolled to a compile-time bound so that all W^2 gathers of an output are
// independent loads (one L2 round trip instead of W^2 dependent ones).
// Input rows (last axis) are valid in [iylo, iyhi) and stored from row iyoff on; columns in [0, nin).
template <int WMAX>
__device__ __forceinline__ double tensor2d_point(const double *__restrict__ in, int nin, int iylo, int iyhi, int iyoff,
                                                 int W, const int *__restrict__ lo, const double *__restrict__ c,
                                                 int ry, int rx) {
  const int ly = lo[ry], lx = lo[rx];
  double cy[WMAX], cx[WMAX];
#pragma unroll
  for (int k = 0; k < WMAX; ++k) {
    const bool oky = k < W && ly + k >= iylo && ly + k < iyhi, okx = k < W && unsigned(lx + k) < unsigned(nin);
    cy[k] = oky ? c[(int64_t)ry * W + k] : 0.0;
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
                           const int *__restrict__ lo, const double *__restrict__ c, int acc, int iylo, int iyhi,
                           int iyoff, int rylo, int ryhi, int ryoff) {
  const int64_t total = (int64_t)(ryhi - rylo) * rows;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int ry = rylo + int(idx / rows), rx = int(idx % rows);
    const double s = tensor2d_point<WMAX>(in, nin, iylo, iyhi, iyoff, W, lo, c, ry, rx);
    const int64_t o = (int64_t)(ry - ryoff) * rows + rx;
    out[o] = acc ? out[o] + s : s;
  }
}

// ---------------- V-cycle over the small tail levels in ONE thread-block cluster -------------
// All CTAs of the cluster share the loops; phases are separated by barrier.cluster (release /
// acquire at cluster scope; it also invalidates L1, so plain loads see the other SMs' stores).
// Each CTA stages the current level's 1D band tables K_q, M_q in shared memory.
__device__ unsigned long long *g_vc_trace = nullptr;   // optional phase timestamps (debug builds)
__device__ long long g_s2d_trace[8];                     // DMMA colour kernel phase clocks (IGA2L_TRACE builds)
__device__ int g_vc_trace_n = 0;

struct Team {
  int64_t tid, nthr;
  __device__ void sync() const {
    cg::this_cluster().sync();
    if (g_vc_trace && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_vc_trace[g_vc_trace_n++ & 1023] = t;
    }
  }
};

constexpr int kVcMaxN = 160;   // tail levels have <= 20000 unknowns: n <= 141 (2D), 27 (3D)

template <int DIM, int Q>
__device__ __forceinline__ double q_point(int n, const double *sK, const double *sM, const double *x, int ix, int iy,
                                          int iz, double *diag) {
  constexpr int W = 2 * Q + 1;
  const unsigned un = unsigned(n);
  double kx[W], mx[W], ky[W], my[W];
#pragma unroll
  for (int t = 0; t < W; ++t) {
    kx[t] = sK[ix * W + t]; mx[t] = sM[ix * W + t];
    ky[t] = sK[iy * W + t]; my[t] = sM[iy * W + t];
  }
  double acc0 = 0.0, acc1 = 0.0;
  if (DIM == 2) {
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int jy = iy + u - Q;
      const bool oky = unsigned(jy) < un;
#pragma unroll
      for (int t = 0; t < W; ++t) {
        const int jx = ix + t - Q;
        const double xv = (oky && unsigned(jx) < un) ? x[(int64_t)jy * n + jx] : 0.0;
        if (t & 1) acc1 = fma(kx[t] * my[u] + mx[t] * ky[u], xv, acc1);
        else acc0 = fma(kx[t] * my[u] + mx[t] * ky[u], xv, acc0);
      }
    }
    *diag = kx[Q] * my[Q] + mx[Q] * ky[Q];
  } else {
    double kz[W], mz[W];
#pragma unroll
    for (int t = 0; t < W; ++t) { kz[t] = sK[iz * W + t]; mz[t] = sM[iz * W + t]; }
#pragma unroll
    for (int v = 0; v < W; ++v) {
      const int jz = iz + v - Q;
      const bool okz = unsigned(jz) < un;
#pragma unroll
      for (int u = 0; u < W; ++u) {
        const int jy = iy + u - Q;
        const bool oky = okz && unsigned(jy) < un;
        const double cyz_k = my[u] * mz[v], cyz_m = ky[u] * mz[v] + my[u] * kz[v];
#pragma unroll
        for (int t = 0; t < W; ++t) {
          const int jx = ix + t - Q;
          const double xv = (oky && unsigned(jx) < un) ? x[((int64_t)jz * n + jy) * n + jx] : 0.0;
          if (t & 1) acc1 = fma(kx[t] * cyz_k + mx[t] * cyz_m, xv, acc1);
          else acc0 = fma(kx[t] * cyz_k + mx[t] * cyz_m, xv, acc0);
        }
      }
    }
    *diag = kx[Q] * my[Q] * mz[Q] + mx[Q] * ky[Q] * mz[Q] + mx[Q] * my[Q] * kz[Q];
  }
  return acc0 + acc1;
}

__device__ __forceinline__ void team_band_axis(const Team tm, const double *in, double *out, int64_t outer, int nin,
                                               int64_t inner, const Band1D B, int acc) {
  const int64_t total = outer * B.rows * inner;
  for (int64_t idx = tm.tid; idx < total; idx += tm.nthr) {
    const int64_t i = idx % inner;
    const int r = int((idx / inner) % B.rows);
    const int64_t o = idx / (inner * B.rows);
    const int l0 = B.lo[r];
    double s = 0.0;
    for (int k = 0; k < B.W; ++k) {
      const int col = l0 + k;
      if (col >= 0 && col < nin) s = fma(B.c[(int64_t)r * B.W + k], in[(o * nin + col) * inner + i], s);
    }
    out[idx] = acc ? out[idx] + s : s;
  }
}

__device__ __forceinline__ void team_tensor2d(const Team tm, const Band1D B, const double *in, double *out, int acc) {
  const int64_t total = (int64_t)B.rows * B.rows;
  for (int64_t idx = tm.tid; idx < total; idx += tm.nthr) {
    const int ry = int(idx / B.rows), rx = int(idx - (int64_t)ry * B.rows);
    const double s = B.W <= 4 ? tensor2d_point<4>(in, B.cols, 0, B.cols, 0, B.W, B.lo, B.c, ry, rx)
                              : tensor2d_point<8>(in, B.cols, 0, B.cols, 0, B.W, B.lo, B.c, ry, rx);
    out[idx] = acc ? out[idx] + s : s;
  }
}

template <int DIM>
__device__ __forceinline__ void team_tensor(const Team tm, const Band1D B, const double *in, double *out, double *t1,
                                            double *t2, int acc) {
  if (DIM == 2) {
    team_tensor2d(tm, B, in, out, acc);
    tm.sync();
    return;
  }
  const double *src = in;
  int64_t inner = 1, outer = 1;
  for (int a = 1; a < DIM; ++a) outer *= B.cols;
  for (int a = 0; a < DIM; ++a) {
    const bool last = (a == DIM - 1);
    double *dst = last ? out : (a % 2 == 0 ? t1 : t2);
    team_band_axis(tm, src, dst, outer, B.cols, inner, B, last ? acc : 0);
    tm.sync();
    src = dst;
    inner *= B.rows;
    if (a + 1 < DIM) outer /= B.cols;
  }
}

template <int DIM, int Q>
__device__ __forceinline__ void team_gs(const Team tm, const int n, double *__restrict__ x,
                                        const double *__restrict__ bb, const double *sK, const double *sM) {
  constexpr int st = Q + 1;
  constexpr int ncol = (DIM == 3) ? st * st * st : st * st;
#pragma unroll 1
  for (int col = 0; col < ncol; ++col) {
    const int c0 = col % st, c1 = (col / st) % st, c2 = (DIM == 3) ? col / (st * st) : 0;
    const int na0 = (n - c0 + Q) / st, na1 = (n - c1 + Q) / st, na2 = (DIM == 3) ? (n - c2 + Q) / st : 1;
    const int tot = (c0 < n && c1 < n && c2 < n) ? na0 * na1 * na2 : 0;
    for (int idx = int(tm.tid); idx < tot; idx += int(tm.nthr)) {
      const int ix = c0 + st * (idx % na0), iy = c1 + st * ((idx / na0) % na1);
      const int iz = (DIM == 3) ? c2 + st * (idx / (na0 * na1)) : 0;
      double dg;
      const double ax = q_point<DIM, Q>(n, sK, sM, x, ix, iy, iz, &dg);
      const int g = (iz * n + iy) * n + ix;
      x[g] += (bb[g] - ax) / dg;
    }
    tm.sync();
  }
}

template <int Q>
__device__ __forceinline__ void stage_tables(const int n, const double *K, const double *M, double *sK, double *sM) {
  constexpr int W = 2 * Q + 1;
  __syncthreads();
  for (int i = threadIdx.x; i < n * W; i += blockDim.x) {
    sK[i] = K[i];
    sM[i] = M[i];
  }
  __syncthreads();
}

template <int DIM, int Q>
__global__ void __launch_bounds__(512) k_vcycle_cluster(const QLevelDev *__restrict__ levs, int l0, int nlev) {
  __shared__ double sK[kVcMaxN * (2 * Q + 1)], sM[kVcMaxN * (2 * Q + 1)];
  cg::cluster_group cl = cg::this_cluster();
  const Team tm{(int64_t)cl.block_rank() * blockDim.x + threadIdx.x, (int64_t)cl.num_blocks() * blockDim.x};
  for (int l = l0; l < nlev - 1; ++l) {
    const int n = levs[l].n, N = int(levs[l].N);
    double *x = levs[l].x, *r = levs[l].r, *t1 = levs[l].t1, *t2 = levs[l].t2;
    const double *bb = levs[l].b;
    const Band1D PT = levs[l].PT;
    double *bnext = levs[l + 1].b;
    stage_tables<Q>(n, levs[l].K, levs[l].M, sK, sM);
    for (int i = int(tm.tid); i < N; i += int(tm.nthr)) x[i] = 0.0;        // zero initial guess (A13)
    tm.sync();
    team_gs<DIM, Q>(tm, n, x, bb, sK, sM);                                   // pre-smoothing (A11)
    for (int idx = int(tm.tid); idx < N; idx += int(tm.nthr)) {              // residual
      const int ix = idx % n, iy = (idx / n) % n, iz = (DIM == 3) ? idx / (n * n) : 0;
      double dg;
      r[idx] = bb[idx] - q_point<DIM, Q>(n, sK, sM, x, ix, iy, iz, &dg);
    }
    tm.sync();
    team_tensor<DIM>(tm, PT, r, bnext, t1, t2, 0);                           // restriction P^T (A8)
  }
  {                                                                          // coarsest: x = A^{-1} b
    const int NC = int(levs[nlev - 1].N);
    const double *inv = levs[nlev - 1].inv, *bc = levs[nlev - 1].b;
    double *xc = levs[nlev - 1].x;
    const int lane = threadIdx.x & 31;
    const int gw = int(tm.tid >> 5), nw = int(tm.nthr >> 5);
    for (int row = gw; row < NC; row += nw) {
      double s = 0.0;
      for (int j = lane; j < NC; j += 32) s = fma(inv[(int64_t)row * NC + j], bc[j], s);
      s = warp_sum(s);
      if (lane == 0) xc[row] = s;
    }
    tm.sync();
  }
  for (int l = nlev - 2; l >= l0; --l) {
    const int n = levs[l].n;
    double *x = levs[l].x, *t1 = levs[l].t1, *t2 = levs[l].t2;
    const double *bb = levs[l].b, *xnext = levs[l + 1].x;
    const Band1D P = levs[l].P;
    stage_tables<Q>(n, levs[l].K, levs[l].M, sK, sM);
    team_tensor<DIM>(tm, P, xnext, x, t1, t2, 1);                            // x += P e
    team_gs<DIM, Q>(tm, n, x, bb, sK, sM);                                   // post-smoothing
  }
}

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
                                                    int thi, const double *__restrict__ ainv) {
  using B = Blk3<P, S>;
  constexpr int W = B::W, Wn = B::Wn, w = B::w, S2 = B::S2, S3 = B::S3, Wn2 = B::Wn2, PER = B::PER;
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  const unsigned un = unsigned(n1);
#ifdef IGA2L_TRACE
  if (blockIdx.x == 0 && tid == 0) g_s2d_trace[0] = clock64();
#endif
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
#ifdef IGA2L_TRACE
  if (blockIdx.x == 0 && tid == 0) g_s2d_trace[1] = clock64();
#endif
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
#ifdef IGA2L_TRACE
  if (blockIdx.x == 0 && tid == 0) g_s2d_trace[2] = clock64();
#endif
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
#ifdef IGA2L_TRACE
  if (blockIdx.x == 0 && tid == 0) g_s2d_trace[3] = clock64();
#endif
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
#ifdef IGA2L_TRACE
  if (blockIdx.x == 0 && tid == 0) g_s2d_trace[4] = clock64();
#endif
  // ---- δ = (⊗V) Λ^{-1} (⊗V)^T r ----
  if constexpr (S == 3 && NBK == 1) {   // s^3 = 27 values: the whole FD in one warp's registers (shuffles)
    if (tid < 32) {
      const int lane = tid, li = lane < 27 ? lane : 0;
      const int lx = li % 3, ly = (li / 3) % 3, lz = li / 9;
      const double *Vx = Vs(0), *Vy = Vs(0) + 9, *Vz = Vs(0) + 18, *L = Ls(0);
      double v;
      if (ainv && tt1[0] && tt1[1] && tt1[2]) {   // interior block (A27): δ = row `lane` of A_B^{-1} times r_B
        double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
        for (int j = 0; j < 27; j += 3) {
          d0 = fma(__ldg(ainv + j * 32 + lane), R(0)[j], d0);
          d1 = fma(__ldg(ainv + (j + 1) * 32 + lane), R(0)[j + 1], d1);
          d2 = fma(__ldg(ainv + (j + 2) * 32 + lane), R(0)[j + 2], d2);
        }
        v = (d0 + d1) + d2;
      } else {
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
#ifdef IGA2L_TRACE
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) g_s2d_trace[5] = clock64();
#endif
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
#ifdef IGA2L_TRACE
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) g_s2d_trace[5] = clock64();
#endif
}

// Launch variants per (p, s): <blocks per CTA, threads, row-wise window staging>.  The default is
// variant 0; IGA2L_S3D_VARIANT=<i> selects another (A/B timing on one box, tools/variants.py).
int g_s3d_variant = -1;
int s3d_variant() {
  if (g_s3d_variant < 0) {
    const char *e = std::getenv("IGA2L_S3D_VARIANT");
    g_s3d_variant = e ? std::atoi(e) : 0;
  }
  return g_s3d_variant;
}

template <int P, int S, int NBK, int NT, bool ROW, bool REGW = false>
void launch3d(int64_t n1, const double *K, const double *M, const double *V, const double *lam, const double *b,
              double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nb2, int zoff, int tlo, int thi,
              cudaStream_t st, const double *ainv = nullptr) {
  constexpr size_t sm = sizeof(double) * NBK * Blk3<P, S>::PER;
  ensure_smem(k_schwarz3d_t<P, S, NBK, NT, ROW, REGW>, sm);
  const int nblk = nb0 * nb1 * nb2;
  k_schwarz3d_t<P, S, NBK, NT, ROW, REGW><<<(nblk + NBK - 1) / NBK, NT, sm, st>>>(int(n1), K, M, V, lam, b, x, c0, c1,
                                                                                  c2, D, nb0, nb1, nblk, zoff, tlo, thi,
                                                                                  ainv);
}

template <int P, int S>
bool try_schwarz3d(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                   const double *b, double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nb2, int zoff,
                   int tlo, int thi, cudaStream_t st, const double *ainv) {
  if (p != P || s != S) return false;
  {                                                 // IGA2L_S3D_INV=1: A_B^{-1} rows on interior blocks (opt-in:
    const char *e = std::getenv("IGA2L_S3D_INV");   // measured equal at C4, profiles/variants_inv_r01.txt)
    if (!(e && e[0] == '1')) ainv = nullptr;
  }
  constexpr int NT1 = ((Blk3<P, S>::Wn2 + 31) / 32) * 32 > 512 ? 512 : ((Blk3<P, S>::Wn2 + 31) / 32) * 32;
  switch (s3d_variant()) {
    case 1: launch3d<P, S, 1, NT1, true>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, zoff, tlo, thi, st); break;
    case 2: launch3d<P, S, 2, (2 * NT1 > 512 ? 512 : 2 * NT1), false>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, zoff, tlo, thi, st); break;
    case 3: launch3d<P, S, 1, (NT1 >= 128 ? NT1 / 2 : NT1), false>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, zoff, tlo, thi, st); break;
    case 5: launch3d<P, S, 1, (S >= 5 && NT1 >= 128 ? NT1 / 2 : NT1), false, true>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, zoff, tlo, thi, st); break;
    case 6: launch3d<P, S, 1, NT1, false, true>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, nb2, zoff, tlo, thi, st); break;
    default:   // measured best (tools/variants.py): s >= 5 -> half the pass-x pencil count of threads
      launch3d<P, S, 1, (S >= 5 && NT1 >= 128 ? NT1 / 2 : NT1), false>(n1, K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1,
                                                                      nb2, zoff, tlo, thi, st, ainv);
      break;
  }
  return true;
}

// ---------------- separable 2D tensor transfer (v2): out (+)= (B ⊗ B) in, two passes ----------
// CTA = TO x TO outputs.  Pass 1 (x): T[iy][rx] = Σ_k c[rx][k] in[iy][lo[rx]+k] for the input rows the
// tile needs; pass 2 (y): out[ry][rx] = Σ_k c[ry][k] T[lo[ry]+k][rx].  2W FMAs per output (plus the
// input-row halo of pass 1) instead of W^2 gathers.  Input rows valid in [iylo, iyhi) stored from
// iyoff; output rows [rylo, ryhi) stored from ryoff (slab views).
template <int TO>
__global__ void __launch_bounds__(256) k_transfer2d_sep(const double *__restrict__ in, double *__restrict__ out, int nin,
                                                        int rows, int W, const int *__restrict__ lo,
                                                        const double *__restrict__ c, int acc, int iylo, int iyhi,
                                                        int iyoff, int rylo, int ryhi, int ryoff, int LI) {
  extern __shared__ double sm[];
  const int rx0 = blockIdx.x * TO, ry0 = rylo + blockIdx.y * TO;
  const int nrx = min(TO, rows - rx0), nry = min(TO, ryhi - ry0);
  if (nrx <= 0 || nry <= 0) return;
  const int ix0 = lo[rx0], iy0 = lo[ry0];                 // first input column / row of the tile
  double *X = sm;                                           // [LI][LI] input window
  double *T = X + LI * LI;                                  // [LI][TO]
  double *cx = T + LI * TO, *cy = cx + TO * W;              // coefficient rows of the tile
  int *lx = reinterpret_cast<int *>(cy + TO * W), *ly = lx + TO;
  const int tid = threadIdx.x;
  for (int i = tid; i < LI * LI; i += 256) {
    const int wy = i / LI, wx = i - wy * LI, gx = ix0 + wx, gy = iy0 + wy;
    const bool ok = unsigned(gx) < unsigned(nin) && gy >= iylo && gy < iyhi;
    cp_async8(X + i, in + (ok ? (int64_t)(gy - iyoff) * nin + gx : 0), ok);
  }
  for (int i = tid; i < TO * W; i += 256) {
    const int r = i / W;
    const bool okx = r < nrx, oky = r < nry;
    cp_async8(cx + i, c + (okx ? (int64_t)(rx0 + r) * W + i % W : 0), okx);
    cp_async8(cy + i, c + (oky ? (int64_t)(ry0 + r) * W + i % W : 0), oky);
  }
  if (tid < TO) {
    lx[tid] = tid < nrx ? lo[rx0 + tid] - ix0 : 0;
    ly[tid] = tid < nry ? lo[ry0 + tid] - iy0 : 0;
  }
  cp_async_wait_all();
  __syncthreads();
  // pass 1: rows of the window that pass 2 reads: [0, ly[nry-1] + W)
  const int nrow = min(LI, ly[nry - 1] + W);
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
    const double *tc = T + ly[ry] * TO + r, *cr = cy + ry * W;
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < W; ++k) {
      if (k & 1) s1 = fma(cr[k], tc[k * TO], s1); else s0 = fma(cr[k], tc[k * TO], s0);
    }
    const int64_t o = (int64_t)(ry0 + ry - ryoff) * rows + rx0 + r;
    out[o] = acc ? out[o] + (s0 + s1) : (s0 + s1);
  }
}

// ---------------- 2D Schwarz colour kernel, register-blocked (v3): NBK blocks per CTA ------------
// Same arithmetic as Blk2 (pass x, pass y, fast diagonalisation), organised for FP64 throughput:
// pass x: one task per window ROW (Wn loads, 2 s (2p+1) FMAs, coefficients in registers on Toeplitz
// axes, A27); pass y: one task per (column, half of the block rows); FD as four s x s contractions
// with one task per row/column.  All phases run over the CTA's (block, task) pairs.
template <int P, int S>
struct Blk2R {
  static constexpr int W = 2 * P + 1, Wn = S + 2 * P, w = (S - 1) / 2, S2 = S * S;
  static constexpr int PER = Wn * Wn + 2 * Wn * S + 3 * S2 + 4 * S * W + 2 * S2 + 2 * S;
  static constexpr int HY = (S + 1) / 2;   // rows per pass-y task (two tasks per column)
};

template <int P, int S, int NBK, int NT>
__global__ void __launch_bounds__(NT) k_schwarz2d_r(int n1, const double *__restrict__ K, const double *__restrict__ M,
                                                    const double *__restrict__ Vt, const double *__restrict__ lamt,
                                                    const double *__restrict__ b, double *__restrict__ x, int c0, int c1,
                                                    int D, int nb0, int nblk, int zoff, int tlo, int thi,
                                                    const ToeP tp) {
  using B = Blk2R<P, S>;
  constexpr int W = B::W, Wn = B::Wn, w = B::w, S2 = B::S2, PER = B::PER, HY = B::HY;
  extern __shared__ double sm[];
  __shared__ int sC[NBK][2];
  __shared__ bool sT[NBK][2];
  const int tid = threadIdx.x;
  const unsigned un = unsigned(n1);
  const int nk = min(NBK, nblk - int(blockIdx.x) * NBK);
  if (tid < NBK) {
    const int g = blockIdx.x * NBK + tid, j1 = g / nb0, j0 = g - j1 * nb0;
    const int cx = c0 + D * j0, cy = c1 + D * j1;
    sC[tid][0] = cx; sC[tid][1] = cy;
    sT[tid][0] = tp.valid && cx - w >= tlo && cx + w <= thi;   // interior axis: tables in tp
    sT[tid][1] = tp.valid && cy - w >= tlo && cy + w <= thi;
  }
  __syncthreads();
  // per-block regions
  auto X = [&](int k) { return sm + k * PER; };                       // [wy][wx]
  auto Pa = [&](int k) { return X(k) + Wn * Wn; };                    // [wy][lx]
  auto Pb = [&](int k) { return Pa(k) + Wn * S; };
  auto R = [&](int k) { return Pb(k) + Wn * S; };                     // [ly][lx]
  auto Q = [&](int k) { return R(k) + S2; };
  auto Bb = [&](int k) { return Q(k) + S2; };
  auto Kx = [&](int k) { return Bb(k) + S2; };                        // [l][t]   (boundary axes only)
  auto Mx = [&](int k) { return Kx(k) + S * W; };
  auto Ky = [&](int k) { return Mx(k) + S * W; };
  auto My = [&](int k) { return Ky(k) + S * W; };
  auto Vx = [&](int k) { return My(k) + S * W; };                     // [l][j]
  auto Vy = [&](int k) { return Vx(k) + S2; };
  auto Lx = [&](int k) { return Vy(k) + S2; };
  auto Ly = [&](int k) { return Lx(k) + S; };
  // ---- loads (cp.async): x windows row by row, b_B, and the tables of boundary axes only ----
  for (int row = tid >> 4; row < nk * Wn; row += NT >> 4) {
    const int k = row / Wn, wy = row - k * Wn;
    const int gy = sC[k][1] - w - P + wy, ox = sC[k][0] - w - P;
    const bool oky = unsigned(gy) < un;
    const double *src = x + (oky ? (int64_t)(gy - zoff) * n1 : 0);
    double *dst = X(k) + wy * Wn;
#pragma unroll
    for (int wx = tid & 15; wx < Wn; wx += 16) {
      const int gx = ox + wx;
      const bool ok = oky && unsigned(gx) < un;
      cp_async8(dst + wx, ok ? src + gx : x, ok);
    }
  }
  for (int i = tid; i < nk * S2; i += NT) {
    const int k = i / S2, r = i - k * S2, ly = r / S, lx = r - ly * S;
    const int gx = sC[k][0] - w + lx, gy = sC[k][1] - w + ly;
    const bool ok = unsigned(gx) < un && unsigned(gy) < un;
    cp_async8(Bb(k) + r, b + (ok ? (int64_t)(gy - zoff) * n1 + gx : 0), ok);
  }
  for (int i = tid; i < nk * 2 * (S * W + S2 + S); i += NT) {
    const int k = i / (2 * (S * W + S2 + S)), r = i - k * (2 * (S * W + S2 + S));
    const int a = r / (S * W + S2 + S), e = r - a * (S * W + S2 + S);
    if (sT[k][a]) continue;
    const int c = sC[k][a];
    if (e < S * W) {
      const int l = e / W, t = e - l * W, g = c - w + l;
      const bool ok = unsigned(g) < un;
      cp_async8((a ? Ky(k) : Kx(k)) + e, K + (ok ? (int64_t)g * W + t : 0), ok);
      cp_async8((a ? My(k) : Mx(k)) + e, M + (ok ? (int64_t)g * W + t : 0), ok);
    } else if (e < S * W + S2) {
      cp_async8((a ? Vy(k) : Vx(k)) + (e - S * W), Vt + (int64_t)c * S2 + (e - S * W), true);
    } else {
      cp_async8((a ? Ly(k) : Lx(k)) + (e - S * W - S2), lamt + (int64_t)c * S + (e - S * W - S2), true);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  // ---- pass x: task = (block, window row wy) -> Pa[wy][lx] = Σ_t K_x v, Pb = Σ_t M_x v ----
  for (int i = tid; i < nk * Wn; i += NT) {
    const int k = i / Wn, wy = i - k * Wn;
    double v[Wn];
#pragma unroll
    for (int q = 0; q < Wn; ++q) v[q] = X(k)[wy * Wn + q];
    const bool toe = sT[k][0];
    const double *ck = Kx(k), *cm = Mx(k);
#pragma unroll
    for (int l = 0; l < S; ++l) {
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int t = 0; t < W; ++t) {
        const double kc = toe ? tp.k[t] : ck[l * W + t], mc = toe ? tp.m[t] : cm[l * W + t];
        if (t & 1) { a1 = fma(kc, v[l + t], a1); b1 = fma(mc, v[l + t], b1); }
        else { a0 = fma(kc, v[l + t], a0); b0 = fma(mc, v[l + t], b0); }
      }
      Pa(k)[wy * S + l] = a0 + a1;
      Pb(k)[wy * S + l] = b0 + b1;
    }
  }
  __syncthreads();
  // ---- pass y: task = (block, column lx, half h) -> R[ly][lx] = b - Σ_u (M_y Pa + K_y Pb) ----
  for (int i = tid; i < nk * S * 2; i += NT) {
    const int k = i / (2 * S), r = i - k * (2 * S), lx = r >> 1, h = r & 1;
    const int ly0 = h * HY, nly = h ? S - HY : HY;
    const double *pa = Pa(k) + lx, *pb = Pb(k) + lx;
    double a[HY + 2 * P], c[HY + 2 * P];
#pragma unroll
    for (int u = 0; u < HY + 2 * P; ++u) {
      const bool ok = ly0 + u < Wn;
      a[u] = ok ? pa[(ly0 + u) * S] : 0.0;
      c[u] = ok ? pb[(ly0 + u) * S] : 0.0;
    }
    const bool toe = sT[k][1];
    const double *ky = Ky(k), *my = My(k);
#pragma unroll
    for (int l = 0; l < HY; ++l) {
      if (l >= nly) break;
      const int ly = ly0 + l;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int u = 0; u < W; ++u) {
        const double mc = toe ? tp.m[u] : my[ly * W + u], kc = toe ? tp.k[u] : ky[ly * W + u];
        s0 = fma(mc, a[l + u], s0);
        s1 = fma(kc, c[l + u], s1);
      }
      R(k)[ly * S + lx] = Bb(k)[ly * S + lx] - (s0 + s1);
    }
  }
  __syncthreads();
  // ---- FD: Q[ly][j] = Σ_lx R[ly][lx] Vx[lx][j] ----
  for (int i = tid; i < nk * S; i += NT) {
    const int k = i / S, ly = i - k * S;
    double rr[S];
#pragma unroll
    for (int l = 0; l < S; ++l) rr[l] = R(k)[ly * S + l];
    const bool toe = sT[k][0];
    const double *vx = Vx(k);
#pragma unroll
    for (int j = 0; j < S; ++j) {
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(toe ? tp.v[l * S + j] : vx[l * S + j], rr[l], a0);
      Q(k)[ly * S + j] = a0;
    }
  }
  __syncthreads();
  // Z[kk][j] = Σ_ly Vy[ly][kk] Q[ly][j] / (λx_j + λy_kk)   (stored in R as [kk][j])
  for (int i = tid; i < nk * S; i += NT) {
    const int k = i / S, j = i - k * S;
    double qq[S];
#pragma unroll
    for (int l = 0; l < S; ++l) qq[l] = Q(k)[l * S + j];
    const bool tx = sT[k][0], ty = sT[k][1];
    const double *vy = Vy(k), *ly_ = Ly(k);
    double lxj = Lx(k)[j];
    if (tx) {
#pragma unroll
      for (int l = 0; l < S; ++l) if (l == j) lxj = tp.lam[l];
    }
#pragma unroll
    for (int kk = 0; kk < S; ++kk) {
      double a0 = 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l) a0 = fma(ty ? tp.v[l * S + kk] : vy[l * S + kk], qq[l], a0);
      R(k)[kk * S + j] = a0 / (lxj + (ty ? tp.lam[kk] : ly_[kk]));
    }
  }
  __syncthreads();
  // U[kk][lx] = Σ_j Vx[lx][j] Z[kk][j]   (into Q)
  for (int i = tid; i < nk * S; i += NT) {
    const int k = i / S, kk = i - k * S;
    double zz[S];
#pragma unroll
    for (int l = 0; l < S; ++l) zz[l] = R(k)[kk * S + l];
    const bool toe = sT[k][0];
    const double *vx = Vx(k);
#pragma unroll
    for (int lx = 0; lx < S; ++lx) {
      double a0 = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) a0 = fma(toe ? tp.v[lx * S + j] : vx[lx * S + j], zz[j], a0);
      Q(k)[kk * S + lx] = a0;
    }
  }
  __syncthreads();
  // δ[ly][lx] = Σ_kk Vy[ly][kk] U[kk][lx];  x_B += δ
  for (int i = tid; i < nk * S; i += NT) {
    const int k = i / S, lx = i - k * S;
    double uu[S];
#pragma unroll
    for (int l = 0; l < S; ++l) uu[l] = Q(k)[l * S + lx];
    const bool toe = sT[k][1];
    const double *vy = Vy(k);
    const int gx = sC[k][0] - w + lx;
#pragma unroll
    for (int ly = 0; ly < S; ++ly) {
      double a0 = 0.0;
#pragma unroll
      for (int kk = 0; kk < S; ++kk) a0 = fma(toe ? tp.v[ly * S + kk] : vy[ly * S + kk], uu[kk], a0);
      const int gy = sC[k][1] - w + ly;
      if (unsigned(gx) < un && unsigned(gy) < un)
        x[(int64_t)(gy - zoff) * n1 + gx] = X(k)[(ly + P) * Wn + lx + P] + a0;
    }
  }
}

template <int P, int S, int NBK, int NT>
void launch2d_r(int64_t n1, const double *K, const double *M, const double *V, const double *lam, const double *b,
                double *x, int c0, int c1, int D, int nb0, int nblk, int zoff, cudaStream_t st, const ToeP &tp) {
  constexpr size_t sm = sizeof(double) * NBK * Blk2R<P, S>::PER;
  ensure_smem(k_schwarz2d_r<P, S, NBK, NT>, sm);
  const int m = int(n1) - P + 2;
  k_schwarz2d_r<P, S, NBK, NT><<<(nblk + NBK - 1) / NBK, NT, sm, st>>>(int(n1), K, M, V, lam, b, x, c0, c1, D, nb0,
                                                                       nblk, zoff, 2 * P - 1, m - 2 - P, tp);
}

int s2d_variant() {   // IGA2L_S2D_VARIANT: 0/9 = DMMA kernel, 1-4 = register-blocked variants, 10 = warp-group (Blk2)
  const char *e = std::getenv("IGA2L_S2D_VARIANT");   // read per launch (host side, cheap): tests switch it
  return e ? std::atoi(e) : 0;
}

template <int P, int S>
bool try_schwarz2d_r(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                     const double *b, double *x, int c0, int c1, int D, int nb0, int nblk, int zoff, cudaStream_t st,
                     int variant, const ToeP *tpp) {
  if (p != P || s != S) return false;
  constexpr int Wn = S + 2 * P;
  ToeP tp{};
  if (tpp) tp = *tpp;
  switch (variant) {
    case 1: launch2d_r<P, S, 8, ((8 * Wn + 31) / 32) * 32>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, tp); break;
    case 2: launch2d_r<P, S, 4, ((4 * Wn + 31) / 32) * 32>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, tp); break;
    case 3: launch2d_r<P, S, 16, (((16 * Wn + 31) / 32) * 32 > 512 ? 512 : ((16 * Wn + 31) / 32) * 32)>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, tp); break;
    default: launch2d_r<P, S, 2, ((2 * Wn + 31) / 32) * 32>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, tp); break;
  }
  return true;
}

// ---------------- 2D Schwarz colour kernel on the FP64 tensor pipe (DMMA), one warp per block -------
// mma.sync.m8n8k4.f64 (A 8x4 row-major, B 4x8 column-major, C 8x8): per lane a = A[l/4][l%4],
// b = B[l%4][l/4], c[i] = C[l/4][2(l%4)+i].  The block solve is five small GEMMs:
//   pass x  Pab[wy][j] = Σ_c X[wy][c] Bx[c][j],  Bx[c][lx] = K(bx+lx, c-lx), Bx[c][S+lx] = M(..)
//   pass y  R[ly][lx] = b_B - Σ_r Ay[ly][r] Pab'[r][lx],  Ay = [M_y band | K_y band], Pab' = [Pa; Pb]
//   FD      T = R Vx,  Z = (Vy^T T) ./ (λx_j + λy_k),  U = Z Vx^T,  δ = Vy U
// Band and FD operands are read through L1 (__ldg) straight into fragments; C fragments feed the next
// GEMM through warp shuffles.  Zero padding everywhere outside the s x s block / window.
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
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

// Row `lane` of the interior block inverse A_B^{-1} (s^2 <= 32 only; A27 makes it the same matrix for
// every interior block): δ_lane = Σ_j a[j] r_j replaces the four FD GEMMs (INV path).
template <int S>
struct InvRow {
  double a[S * S];
};
// IGA2L_MMA_INV=1: interior blocks multiply by A_B^{-1} instead of the FD GEMMs (read per launch, host side).
// Opt-in: measured equal (C2 p3-p5, C1: within ±0.03 us per colour, profiles/variants_inv_r01.txt), so
// the default keeps one arithmetic for every block.
int mma_inv_enabled() {
  const char *e = std::getenv("IGA2L_MMA_INV");
  return e ? std::atoi(e) != 0 : 0;
}

// One block solve by one warp.  Xw: the block's (s+2p)^2 window inside a zero-padded array with row
// stride ldx (rows/cols beyond the window up to the fragment padding must be finite); Pab: per-warp
// scratch (MT*8 x LDP, plus s^2 doubles behind it on the INV path); writes x_B = Xw-centre + δ through
// out(ly, lx, value) for in-domain cells.
template <int P, int S, bool INV, class OUT>
__device__ __forceinline__ void mma_block_impl(const double *Xw, int ldx, double *Pab, int n1, int cx, int cy,
                                               const FragX<P, S> &fx, const FragY<P, S> &fy, const InvRow<S> &ai,
                                               const double *__restrict__ b, int zoff, OUT out, bool trace) {
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
    rden[i] = (r4 < S && j < S) ? 1.0 / (fx.lam[i] + fy.lam) : 0.0;
    const int gx = bx + j, gy = by + r4;
    bb[i] = (r4 < S && j < S && unsigned(gx) < un && unsigned(gy) < un) ? __ldg(b + (int64_t)(gy - zoff) * n1 + gx) : 0.0;
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
      for (int nt = 0; nt < NTX; ++nt) dmma(acc[nt][0], acc[nt][1], a, fx.bxf[kt][nt]);
    }
#pragma unroll
    for (int nt = 0; nt < NTX; ++nt) {
      Pab[(8 * mt + r4) * LDP + 8 * nt + 2 * q4] = acc[nt][0];
      Pab[(8 * mt + r4) * LDP + 8 * nt + 2 * q4 + 1] = acc[nt][1];
    }
  }
  __syncwarp();
#ifdef IGA2L_TRACE
  if (trace) g_s2d_trace[3] = clock64();
#endif
  // ---- pass y: R = b_B - Ay [Pa; Pb] ----
  double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0;      // two independent accumulation chains
#pragma unroll
  for (int kt = 0; kt < KY; ++kt) {
    const int r = 4 * kt + q4, lx = r4;
    const bool second = r >= WN4;
    const int rr = second ? r - WN4 : r;
    const double bv = (lx < S && rr < Wn) ? Pab[rr * LDP + (second ? S : 0) + lx] : 0.0;
    if (kt & 1) dmma(s0, s1, fy.ayf[kt], bv);
    else dmma(r0, r1, fy.ayf[kt], bv);
  }
  r0 = (r4 < S && 2 * q4 < S) ? bb[0] - (r0 + s0) : 0.0;
  r1 = (r4 < S && 2 * q4 + 1 < S) ? bb[1] - (r1 + s1) : 0.0;
#ifdef IGA2L_TRACE
  if (trace) g_s2d_trace[4] = clock64() + (r0 == 1.2345e300 ? 1 : 0);
#endif
  if constexpr (INV) {                                       // δ = A_B^{-1} r_B, one row per lane
    double *Rs = Pab + MT * 8 * LDP;
    if (r4 < S) {
      if (2 * q4 < S) Rs[r4 * S + 2 * q4] = r0;
      if (2 * q4 + 1 < S) Rs[r4 * S + 2 * q4 + 1] = r1;
    }
    __syncwarp();
    double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < S * S; ++j) d[j & 3] = fma(ai.a[j], Rs[j], d[j & 3]);
    __syncwarp();
    const double dl = (d[0] + d[1]) + (d[2] + d[3]);
    const int ly = lane / S, lx = lane - (lane / S) * S, gx = bx + lx, gy = by + ly;
    if (lane < S * S && unsigned(gx) < un && unsigned(gy) < un) out(ly, lx, Xw[(ly + P) * ldx + lx + P] + dl);
    return;
  }
  // ---- FD: T = R Vx;  Z = Vy^T T ./ den;  U = Z Vx^T;  δ = Vy U ----
  double t0 = 0.0, t1 = 0.0;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) dmma(t0, t1, c_elem(r0, r1, r4, 4 * kt + q4), fx.vxb[kt]);
  double z0 = 0.0, z1 = 0.0;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) dmma(z0, z1, fy.vyta[kt], c_elem(t0, t1, 4 * kt + q4, r4));
  z0 *= rden[0];
  z1 *= rden[1];
  double u0 = 0.0, u1 = 0.0;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) dmma(u0, u1, c_elem(z0, z1, r4, 4 * kt + q4), fx.vxtb[kt]);
  double e0 = 0.0, e1 = 0.0;
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) dmma(e0, e1, fy.vya[kt], c_elem(u0, u1, 4 * kt + q4, r4));
#ifdef IGA2L_TRACE
  if (trace) g_s2d_trace[5] = clock64() + (e0 == 1.2345e300 ? 1 : 0);
#endif
  // ---- x_B += δ ----
  const int ly = r4, gy = by + ly;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int lx = 2 * q4 + i, gx = bx + lx;
    if (ly < S && lx < S && unsigned(gx) < un && unsigned(gy) < un)
      out(ly, lx, Xw[(ly + P) * ldx + lx + P] + (i ? e1 : e0));
  }
}

template <int P, int S, class OUT>
__device__ __forceinline__ void mma_block_f(const double *Xw, int ldx, double *Pab, int n1, int cx, int cy,
                                            const FragX<P, S> &fx, const FragY<P, S> &fy,
                                            const double *__restrict__ b, int zoff, OUT out, bool trace = false) {
  InvRow<S> none;                                            // unused on the FD path
  mma_block_impl<P, S, false>(Xw, ldx, Pab, n1, cx, cy, fx, fy, none, b, zoff, out, trace);
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
template <int S>
__host__ __device__ constexpr int inv_count() {   // lane-major rows of the interior block inverse behind the fragments
  return S * S <= 32 ? S * S : 0;
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
  if constexpr (inv_count<S>() > 0) {
    // A_B^{-1}[(ly,lx)][(ky,kx)] = Σ_{k,j} Vy[ly][k] Vx[lx][j] Vy[ky][k] Vx[kx][j] / (λx_j + λy_k), both axes at
    // the reference centre (A27: the FD pair of every interior block)
    const double *V = Vt + (int64_t)cref * S * S, *L = lamt + (int64_t)cref * S;
    const int l = threadIdx.x, ly = l / S, lx = l % S;
    for (int c2 = 0; c2 < S * S; ++c2) {
      const int ky = c2 / S, kx = c2 % S;
      double acc = 0.0;
      if (l < S * S)
        for (int k = 0; k < S; ++k)
          for (int j = 0; j < S; ++j)
            acc += V[ly * S + k] * V[lx * S + j] * V[ky * S + k] * V[kx * S + j] / (L[j] + L[k]);
      out[(NX + NY + c2) * 32 + l] = acc;
    }
  }
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
                                                 int zoff, const double *__restrict__ fb, int tlo, int thi, int inv) {
  using G = Mma2<P, S>;
  constexpr int Wn = G::Wn, w = G::w, MT = G::MT, WN4 = G::WN4, LDX = G::LDX;
  const int lane = threadIdx.x & 31;
  double *Pab = X + MT * 8 * LDX;
  const int j1 = bid / nb0, j0 = bid - j1 * nb0;
  const int cx = c0 + D * j0, cy = c1 + D * j1;
  const int bx = cx - w, by = cy - w, ox = bx - P, oy = by - P;
  const unsigned un = unsigned(n1);
#ifdef IGA2L_TRACE
  const bool tr = (bid == 0 && lane == 0);
  long long t0 = clock64();
#endif
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
#ifdef IGA2L_TRACE
  long long t1 = clock64();
#endif
  FragX<P, S> fx;
  FragY<P, S> fy;
  const bool interior = fb && cx - w >= tlo && cx + w <= thi && cy - w >= tlo && cy + w <= thi;
  if constexpr (inv_count<S>() > 0) {
    if (interior && inv) {                                   // interior block: shared fragments + A_B^{-1} row
      load_frags<P, S>(fb, fx, fy);
      InvRow<S> ai;
      constexpr int NF = frag_count<P, S>();
#pragma unroll
      for (int j = 0; j < S * S; ++j) ai.a[j] = __ldg(fb + (NF + j) * 32 + lane);
#pragma unroll
      for (int k = 0; k < WI; ++k) {
        const int i = lane + 32 * k, row = i / WN4, cc = i - row * WN4;
        if (i < WT) X[row * LDX + cc] = wv[k];
      }
      __syncwarp();
      mma_block_impl<P, S, true>(X, LDX, Pab, n1, cx, cy, fx, fy, ai, b, zoff, [&](int ly, int lx, double v) {
        x[(int64_t)(by + ly - zoff) * n1 + bx + lx] = v;
      }, false);
      return;
    }
  }
  if (interior) {
    load_frags<P, S>(fb, fx, fy);                            // interior block: shared fragments (A27)
  } else {
    build_fragx<P, S>(fx, n1, cx, K, M, Vt, lamt);
    build_fragy<P, S>(fy, n1, cy, K, M, Vt, lamt);
  }
#pragma unroll
  for (int k = 0; k < WI; ++k) {
    const int i = lane + 32 * k, row = i / WN4, cc = i - row * WN4;
    if (i < WT) X[row * LDX + cc] = wv[k];
  }
  __syncwarp();
#ifdef IGA2L_TRACE
  const double f0 = fx.bxf[0][0] + fy.ayf[0];   // force the fragment loads to complete here
  long long t2 = clock64() + (f0 == 1.2345e300 ? 1 : 0);
#endif
#ifdef IGA2L_TRACE
  const bool trs = tr;
#else
  const bool trs = false;
#endif
  mma_block_f<P, S>(X, LDX, Pab, n1, cx, cy, fx, fy, b, zoff, [&](int ly, int lx, double v) {
    x[(int64_t)(by + ly - zoff) * n1 + bx + lx] = v;
  }, trs);
#ifdef IGA2L_TRACE
  long long t3 = clock64();
  if (tr) {
    g_s2d_trace[0] = t1 - t0;                  // issue of the window loads
    g_s2d_trace[1] = t2 - t1;                  // window + fragment loads landed
    g_s2d_trace[2] = t3 - t2;                  // the DMMA block solve incl. the x store issue
    g_s2d_trace[6] = g_s2d_trace[3] - t2;      // pass x (+ Pab stores)
    g_s2d_trace[7] = g_s2d_trace[4] - g_s2d_trace[3];   // pass y
    g_s2d_trace[3] = g_s2d_trace[5] - g_s2d_trace[4];   // FD chain
    g_s2d_trace[4] = t3 - g_s2d_trace[5];               // x update
  }
#endif
}

// ---------------- temporal blocking: KC consecutive colours per launch (latency-bound sizes) ------
// CTA = core tile [X0, X0+T)^2 (T = 2D).  It loads x on core ± KC r (r = 2w + p, the reach of one
// block update on the next colour's residual) into shared memory, solves colour c+j's blocks with
// centres in core ± (w + (KC-1-j) r) from that copy (outer ones redundantly with the neighbours,
// same arithmetic), and writes back its core only.  Equals KC per-colour launches (reading A4).
template <int P, int S>
struct Tb2 {
  using G = Mma2<P, S>;
  static constexpr int D = S + P, T = 2 * D, r = S - 1 + P, w = (S - 1) / 2;
  static constexpr int PADX = (G::MT * 8 - G::Wn) > (G::WN4 - G::Wn) ? (G::MT * 8 - G::Wn) : (G::WN4 - G::Wn);
  __host__ __device__ static constexpr int side(int kc) { return T + 2 * kc * r + PADX; }
};

template <int P, int S, int KC, int WPC>
__global__ void __launch_bounds__(WPC * 32) k_schwarz2d_tb(int n1, const double *__restrict__ K,
                                                           const double *__restrict__ M,
                                                           const double *__restrict__ Vt,
                                                           const double *__restrict__ lamt,
                                                           const double *__restrict__ b, double *__restrict__ x,
                                                           int col0, int ncol, int ntx, int tlo, int thi, int cref) {
  using G = Mma2<P, S>;
  using TB = Tb2<P, S>;
  constexpr int D = TB::D, T = TB::T, r = TB::r, w = TB::w, L = TB::side(KC), LDR = L + 1, LDP = G::LDP;
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5;
  double *Rg = sm, *Pab = sm + L * LDR + warp * (G::MT * 8 * LDP);
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const int X0 = tx * T, Y0 = ty * T, H = ncol * r;
  const int rx0 = X0 - H, ry0 = Y0 - H;                      // region origin (global)
  const unsigned un = unsigned(n1);
  for (int i = threadIdx.x; i < L * L; i += WPC * 32) {      // region (zero outside the domain / region)
    const int ry = i / L, rx = i - ry * L, gx = rx0 + rx, gy = ry0 + ry;
    const bool ok = rx < T + 2 * H && ry < T + 2 * H && unsigned(gx) < un && unsigned(gy) < un;
    cp_async8(Rg + ry * LDR + rx, x + (ok ? (int64_t)gy * n1 + gx : 0), ok);
  }
  FragX<P, S> fxi;                                           // interior fragments (A27), built once per warp
  FragY<P, S> fyi;
  if (cref >= 0) {
    build_fragx<P, S>(fxi, n1, cref, K, M, Vt, lamt);
    build_fragy<P, S>(fyi, n1, cref, K, M, Vt, lamt);
  }
  cp_async_wait_all();
  __syncthreads();
  for (int j = 0; j < ncol; ++j) {
    const int c = col0 + j, cc0 = c % D, cc1 = c / D;
    const int rho = w + (ncol - 1 - j) * r;
    // centres with residue (cc0, cc1) in [X0 - rho, X0 + T + rho) x [Y0 - rho, Y0 + T + rho), inside the domain
    auto first = [&](int res, int lo) { int f = res; if (f < lo) f += ((lo - f + D - 1) / D) * D; return f; };
    const int lox = max(0, X0 - rho), hix = min(n1, X0 + T + rho), loy = max(0, Y0 - rho), hiy = min(n1, Y0 + T + rho);
    const int fx = first(cc0, lox), fy = first(cc1, loy);
    const int nx = fx < hix ? (hix - 1 - fx) / D + 1 : 0, ny = fy < hiy ? (hiy - 1 - fy) / D + 1 : 0;
    for (int blk = warp; blk < nx * ny; blk += WPC) {
      const int cx = fx + D * (blk % nx), cy = fy + D * (blk / nx);
      const int ox = cx - w - P - rx0, oy = cy - w - P - ry0;  // window origin in the region
      double *Xw = Rg + oy * LDR + ox;
      auto put = [&](int ly, int lx, double v) { Xw[(ly + P) * LDR + lx + P] = v; };
      if (cref >= 0 && cx - w >= tlo && cx + w <= thi && cy - w >= tlo && cy + w <= thi)
        mma_block_f<P, S>(Xw, LDR, Pab, n1, cx, cy, fxi, fyi, b, 0, put);
      else
        mma_block<P, S>(Xw, LDR, Pab, n1, cx, cy, K, M, Vt, lamt, b, 0, put);
      __syncwarp();
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < T * T; i += WPC * 32) {      // write back the core
    const int cy = i / T, cx = i - cy * T, gx = X0 + cx, gy = Y0 + cy;
    if (gx < n1 && gy < n1) x[(int64_t)gy * n1 + gx] = Rg[(cy + H) * LDR + cx + H];
  }
}


template <int P, int S, int WPC>
__global__ void __launch_bounds__(WPC * 32) k_schwarz2d_mma(int n1, const double *__restrict__ K,
                                                            const double *__restrict__ M,
                                                            const double *__restrict__ Vt,
                                                            const double *__restrict__ lamt,
                                                            const double *__restrict__ b, double *__restrict__ x,
                                                            int c0, int c1, int D, int nb0, int nblk, int zoff,
                                                            const double *__restrict__ fb, int tlo, int thi, int inv) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5;
  const int bid = blockIdx.x * WPC + warp;
  if (bid >= nblk) return;                                   // whole warp exits together
  mma_colour_block<P, S>(sm + warp * Mma2<P, S>::PER, bid, n1, K, M, Vt, lamt, b, x, c0, c1, D, nb0, nblk, zoff, fb,
                         tlo, thi, inv);
}

// ---------------- batched colour launch: one colour of up to kBatchMax independent problems ----------
// CTA = one warp = one block; CTAs [beg[j], beg[j+1]) belong to problem j, whose (p, s) selects the body.
// WPC warps per CTA, one block per warp (block index over the concatenated problems); MAXPS limits the
// (p, s) bodies compiled in (registers / shared memory are the maximum over them).
template <int WPC, int MAXPS>
__global__ void __launch_bounds__(WPC * 32) k_schwarz2d_mma_batch(const BatchDesc d, int per, int inv) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5;
  const int g = int(blockIdx.x) * WPC + warp;
  if (g >= d.beg[d.n]) return;
  int j = 0;
  while (j + 1 < d.n && g >= d.beg[j + 1]) ++j;
  const BatchProb &q = d.pr[j];
  const int bid = g - d.beg[j];
  double *X = sm + warp * per;
#define IGA2L_B(I, P_, S_)                                                                                    \
  case I:                                                                                                     \
    if (I <= MAXPS)                                                                                           \
      mma_colour_block<P_, S_>(X, bid, q.n1, q.K, q.M, q.V, q.lam, q.b, q.x, q.c0, q.c1, q.D, q.nb0, q.nblk, 0, \
                               q.fb, q.tlo, q.thi, inv);                                                      \
    break;
  switch (q.ps) {
    IGA2L_B(0, 1, 3) IGA2L_B(1, 2, 3) IGA2L_B(2, 3, 3) IGA2L_B(3, 4, 3)
    IGA2L_B(4, 5, 5) IGA2L_B(5, 6, 5) IGA2L_B(6, 7, 7) IGA2L_B(7, 8, 7)
    default: break;
  }
#undef IGA2L_B
}

// Several blocks per warp (BPW consecutive blocks of the colour): interior fragments (A27) built once
// per warp, the next block's window prefetched by cp.async into the second buffer while this one is
// solved.  Same arithmetic as k_schwarz2d_mma (bitwise equal).
template <int P, int S, int WPC, int BPW>
__global__ void __launch_bounds__(WPC * 32) k_schwarz2d_mma_m(int n1, const double *__restrict__ K,
                                                              const double *__restrict__ M,
                                                              const double *__restrict__ Vt,
                                                              const double *__restrict__ lamt,
                                                              const double *__restrict__ b, double *__restrict__ x,
                                                              int c0, int c1, int D, int nb0, int nblk, int zoff,
                                                              int tlo, int thi, int cref) {
  using G = Mma2<P, S>;
  constexpr int Wn = G::Wn, w = G::w, MT = G::MT, WN4 = G::WN4, LDX = G::LDX, LDP = G::LDP;
  constexpr int XSZ = MT * 8 * LDX;
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b0 = (blockIdx.x * WPC + warp) * BPW;
  if (b0 >= nblk) return;
  double *Xs = sm + warp * (2 * XSZ + MT * 8 * LDP), *Pab = Xs + 2 * XSZ;
  const unsigned un = unsigned(n1);
  auto centre = [&](int bid, int *cx, int *cy) {
    const int j1 = bid / nb0, j0 = bid - j1 * nb0;
    *cx = c0 + D * j0;
    *cy = c1 + D * j1;
  };
  auto stage = [&](int bid, double *X) {
    int cx, cy;
    centre(bid, &cx, &cy);
    const int ox = cx - w - P, oy = cy - w - P;
    for (int row = 0; row < MT * 8; ++row) {
      const int gy = oy + row;
      const bool oky = row < Wn && unsigned(gy) < un;
      const double *src = x + (oky ? (int64_t)(gy - zoff) * n1 : 0);
#pragma unroll
      for (int cc = lane; cc < WN4; cc += 32) {
        const int gx = ox + cc;
        const bool ok = oky && cc < Wn && unsigned(gx) < un;
        cp_async8(X + row * LDX + cc, ok ? src + gx : x, ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  FragX<P, S> fxi;
  FragY<P, S> fyi;
  if (cref >= 0) {
    build_fragx<P, S>(fxi, n1, cref, K, M, Vt, lamt);
    build_fragy<P, S>(fyi, n1, cref, K, M, Vt, lamt);
  }
  const int nb = min(BPW, nblk - b0);
  stage(b0, Xs);
  for (int j = 0; j < nb; ++j) {
    double *X = Xs + (j & 1) * XSZ;
    if (j + 1 < nb) {
      stage(b0 + j + 1, Xs + ((j + 1) & 1) * XSZ);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    int cx, cy;
    centre(b0 + j, &cx, &cy);
    const int bx = cx - w, by = cy - w;
    auto put = [&](int ly, int lx, double v) { x[(int64_t)(by + ly - zoff) * n1 + bx + lx] = v; };
    if (cref >= 0 && cx - w >= tlo && cx + w <= thi && cy - w >= tlo && cy + w <= thi)
      mma_block_f<P, S>(X, LDX, Pab, n1, cx, cy, fxi, fyi, b, zoff, put);
    else
      mma_block<P, S>(X, LDX, Pab, n1, cx, cy, K, M, Vt, lamt, b, zoff, put);
    __syncwarp();
  }
}

template <int P, int S, int WPC>
void launch2d_mma(int64_t n1, const double *K, const double *M, const double *V, const double *lam, const double *b,
                  double *x, int c0, int c1, int D, int nb0, int nblk, int zoff, cudaStream_t st, const double *fb) {
  constexpr size_t sm = sizeof(double) * WPC * Mma2<P, S>::PER;
  ensure_smem(k_schwarz2d_mma<P, S, WPC>, sm);
  const int m = int(n1) - P + 2;
  k_schwarz2d_mma<P, S, WPC><<<(nblk + WPC - 1) / WPC, WPC * 32, sm, st>>>(int(n1), K, M, V, lam, b, x, c0, c1, D,
                                                                           nb0, nblk, zoff, fb, 2 * P - 1, m - 2 - P,
                                                                           mma_inv_enabled());
}

template <int P, int S>
bool try_schwarz2d_mma(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                       const double *b, double *x, int c0, int c1, int D, int nb0, int nblk, int zoff, cudaStream_t st,
                       const double *fb) {
  if (p != P || s != S) return false;
  const char *eb = std::getenv("IGA2L_MMA_BPW");   // blocks per warp (> 1: prefetching multi-block warps)
  const int bpw = eb ? std::atoi(eb) : 1;
  if (bpw > 1) {
    const int m = int(n1) - P + 2, tlo = 2 * P - 1, thi = m - 2 - P, w = (S - 1) / 2;
    const int cref = (thi - tlo >= 2 * w) ? (tlo + thi) / 2 : -1;
    constexpr int WPCm = 4;
    constexpr size_t sm = sizeof(double) * WPCm * (2 * Mma2<P, S>::MT * 8 * Mma2<P, S>::LDX + Mma2<P, S>::MT * 8 * Mma2<P, S>::LDP);
    auto go = [&](auto kern, int B) {
      ensure_smem(kern, sm);
      const int nw = (nblk + B - 1) / B;
      kern<<<(nw + WPCm - 1) / WPCm, WPCm * 32, sm, st>>>(int(n1), K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, tlo,
                                                          thi, cref);
    };
    if (bpw == 2) go(k_schwarz2d_mma_m<P, S, WPCm, 2>, 2);
    else if (bpw == 4) go(k_schwarz2d_mma_m<P, S, WPCm, 4>, 4);
    else go(k_schwarz2d_mma_m<P, S, WPCm, 8>, 8);
    return true;
  }
  const char *e = std::getenv("IGA2L_MMA_WPC");   // warps (blocks) per CTA; measured best (variants_wpc_r01):
  const int wpc = e ? std::atoi(e) : (S >= 5 ? 1 : 4);   // 1 for s >= 5 (C2 p5, C3), 4 for s = 3
  if (wpc == 1) launch2d_mma<P, S, 1>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, fb);
  else if (wpc == 2) launch2d_mma<P, S, 2>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, fb);
  else if (wpc == 8) launch2d_mma<P, S, 8>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, fb);
  else launch2d_mma<P, S, 4>(n1, K, M, V, lam, b, x, c0, c1, D, nb0, nblk, zoff, st, fb);
  return true;
}

template <int P, int S, int KC>
bool try_schwarz2d_tb(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                      const double *b, double *x, int col0, int ncol, cudaStream_t st) {
  if (p != P || s != S) return false;
  using TB = Tb2<P, S>;
  constexpr int WPC = 8, L = TB::side(KC);
  constexpr size_t sm = sizeof(double) * (size_t(L) * (L + 1) + WPC * Mma2<P, S>::MT * 8 * Mma2<P, S>::LDP);
  ensure_smem(k_schwarz2d_tb<P, S, KC, WPC>, sm);
  const int ntx = int((n1 + TB::T - 1) / TB::T);
  const int m = int(n1) - P + 2, tlo = 2 * P - 1, thi = m - 2 - P, w = (S - 1) / 2;
  const int cref = (thi - tlo >= 2 * w) ? (tlo + thi) / 2 : -1;   // an interior centre (A27)
  k_schwarz2d_tb<P, S, KC, WPC><<<ntx * ntx, WPC * 32, sm, st>>>(int(n1), K, M, V, lam, b, x, col0, ncol, ntx, tlo,
                                                                 thi, cref);
  return true;
}

// ---------------- 3D Schwarz colour kernel on the FP64 tensor pipe (DMMA): one CTA (NW warps) per block ----
// pass x : Pab[pencil][j]   = X[pencil][c] · Bx[c][j]               (pencil = (wz, wy); j: K part, M part)
// pass y : PcPe[m][(wz,lx)] = [[M_y, K_y], [0, M_y]][m][r] · [Pa; Pb][r][(wz,lx)]
// pass z : R[lz][(ly,lx)]   = b_B - [M_z | K_z][lz][r] · [Pc; Pe][r][(ly,lx)]
// FD     : six S^2 x S x S contractions (x, y, z forward, / (λx+λy+λz), z, y, x back) through shared memory.
template <int P, int S>
struct Mma3 {
  static constexpr int W = 2 * P + 1, Wn = S + 2 * P, w = (S - 1) / 2, S2 = S * S, S3 = S2 * S;
  static constexpr int WN4 = ((Wn + 3) / 4) * 4, KT = WN4 / 4;          // window x (pass-x K)
  static constexpr int MX = (Wn * Wn + 7) / 8;                           // pencils (pass-x M tiles)
  static constexpr int NTX = (2 * S + 7) / 8;                            // pass-x N tiles
  static constexpr int LDX = WN4 + 1, LDP = NTX * 8 + 1;
  static constexpr int MTY = (2 * S + 7) / 8, KY = 2 * WN4 / 4, NTY = (Wn * S + 7) / 8, LDQ = NTY * 8 + 1;
  static constexpr int KZ = 2 * WN4 / 4, NTZ = (S2 + 7) / 8;
  static constexpr int MF = (S2 + 7) / 8, KF = (S + 3) / 4;
  static constexpr int OX = 0, OP = MX * 8 * LDX, OQ = OP + MX * 8 * LDP, OR = OQ + MTY * 8 * LDQ;
  static constexpr int OT = OR + S3, OB = OT + S3, SM = OB + S3;        // doubles
};

// One FD contraction of a 3D s^3 array (index [z][y][x], x fastest) on DMMA; STEP selects the axis and
// direction: 0/1/2 = x/y/z forward (Vᵀ; step 2 also divides by λx_j + λy_k + λz_m), 3/4/5 = z/y/x back.
template <int S, int KF, int MF, int NW, int STEP>
__device__ __forceinline__ void fd3_step(const double *in, double *out, const double (&bf)[KF], const double *lx_,
                                         const double *ly_, const double *lz_) {
  constexpr int S2 = S * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r4 = lane >> 2, q4 = lane & 3;
  auto addr = [](int i, int l) -> int {   // element (row i, contracted index l); i = pair of the other two
    if (STEP == 0 || STEP == 5) return i * S + l;                              // rows (z,y), axis x
    if (STEP == 1 || STEP == 4) return ((i / S) * S + l) * S + i % S;          // rows (z,x), axis y
    return l * S2 + i;                                                          // rows (y,x), axis z
  };
  for (int mt = warp; mt < MF; mt += NW) {
    double d0 = 0.0, d1 = 0.0;
    const int i = 8 * mt + r4;
#pragma unroll
    for (int kt = 0; kt < KF; ++kt) {
      const int l = 4 * kt + q4;
      const double a = (i < S2 && l < S) ? in[addr(i, l)] : 0.0;
      dmma(d0, d1, a, bf[kt]);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 2 * q4 + e;
      if (i < S2 && j < S) {
        double v = e ? d1 : d0;
        if (STEP == 2) v /= (__ldg(lx_ + i % S) + __ldg(ly_ + i / S) + __ldg(lz_ + j));
        out[addr(i, j)] = v;
      }
    }
  }
  __syncthreads();
}

template <int P, int S, int NW>
__global__ void __launch_bounds__(NW * 32) k_schwarz3d_mma(int n1, const double *__restrict__ K,
                                                           const double *__restrict__ M,
                                                           const double *__restrict__ Vt,
                                                           const double *__restrict__ lamt,
                                                           const double *__restrict__ b, double *__restrict__ x,
                                                           int c0, int c1, int c2, int D, int nb0, int nb1, int zoff) {
  using G = Mma3<P, S>;
  constexpr int W = G::W, Wn = G::Wn, w = G::w, S2 = G::S2, S3 = G::S3, WN4 = G::WN4, KT = G::KT, MX = G::MX,
                NTX = G::NTX, LDX = G::LDX, LDP = G::LDP, MTY = G::MTY, KY = G::KY, NTY = G::NTY, LDQ = G::LDQ,
                KZ = G::KZ, NTZ = G::NTZ, MF = G::MF, KF = G::KF;
  extern __shared__ double sm[];
  double *X = sm + G::OX, *Pab = sm + G::OP, *Q = sm + G::OQ, *R = sm + G::OR, *T = sm + G::OT, *Bb = sm + G::OB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r4 = lane >> 2, q4 = lane & 3;
  const int g = blockIdx.x;
  const int cx = c0 + D * (g % nb0), cy = c1 + D * ((g / nb0) % nb1), cz = c2 + D * (g / (nb0 * nb1));
  const int bx = cx - w, by = cy - w, bz = cz - w;
  const unsigned un = unsigned(n1);
  // ---- stage: window pencils [(wz, wy)][wx] (zero padded), b_B ----
  for (int row = warp; row < MX * 8; row += NW) {
    const int wz = row / Wn, wy = row - wz * Wn, gy = by - P + wy, gz = bz - P + wz;
    const bool okyz = row < Wn * Wn && unsigned(gy) < un && unsigned(gz) < un;
    const double *src = x + (okyz ? ((int64_t)(gz - zoff) * n1 + gy) * n1 : 0);
#pragma unroll
    for (int c = lane; c < WN4; c += 32) {
      const int gx = bx - P + c;
      const bool ok = okyz && c < Wn && unsigned(gx) < un;
      cp_async8(X + row * LDX + c, ok ? src + gx : x, ok);
    }
  }
  for (int i = threadIdx.x; i < S3; i += NW * 32) {
    const int gx = bx + i % S, gy = by + (i / S) % S, gz = bz + i / S2;
    const bool ok = unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un;
    cp_async8(Bb + i, b + (ok ? ((int64_t)(gz - zoff) * n1 + gy) * n1 + gx : 0), ok);
  }
  // ---- operand fragments (independent of x; overlap the copies) ----
  auto band = [&](const double *T_, int row0, int l, int t) {   // T_(row0 + l, t), 0 outside
    const int gr = row0 + l;
    return (t >= 0 && t < W && unsigned(gr) < un) ? __ldg(T_ + (int64_t)gr * W + t) : 0.0;
  };
  double bxf[KT][NTX];
#pragma unroll
  for (int kt = 0; kt < KT; ++kt)
#pragma unroll
    for (int nt = 0; nt < NTX; ++nt) {
      const int c = 4 * kt + q4, j = 8 * nt + r4;
      bxf[kt][nt] = j < S ? band(K, bx, j, c - j) : (j < 2 * S ? band(M, bx, j - S, c - (j - S)) : 0.0);
    }
  double ayf[MTY][KY];
#pragma unroll
  for (int mt = 0; mt < MTY; ++mt)
#pragma unroll
    for (int kt = 0; kt < KY; ++kt) {
      const int m = 8 * mt + r4, r = 4 * kt + q4;
      const bool second = r >= WN4;
      const int rr = second ? r - WN4 : r;
      double v = 0.0;
      if (m < S) v = second ? band(K, by, m, rr - m) : band(M, by, m, rr - m);
      else if (m < 2 * S) v = second ? band(M, by, m - S, rr - (m - S)) : 0.0;
      ayf[mt][kt] = v;
    }
  double azf[KZ];
#pragma unroll
  for (int kt = 0; kt < KZ; ++kt) {
    const int r = 4 * kt + q4;
    const bool second = r >= WN4;
    const int rr = second ? r - WN4 : r;
    azf[kt] = r4 < S ? (second ? band(K, bz, r4, rr - r4) : band(M, bz, r4, rr - r4)) : 0.0;
  }
  const double *Vx = Vt + (int64_t)cx * S2, *Vy = Vt + (int64_t)cy * S2, *Vz = Vt + (int64_t)cz * S2;
  double vf[6][KF];   // FD B operands: B[l][j], l = 4kt+q4, j = r4
#pragma unroll
  for (int kt = 0; kt < KF; ++kt) {
    const int l = 4 * kt + q4, j = r4;
    const bool ok = l < S && j < S;
    vf[0][kt] = ok ? __ldg(Vx + l * S + j) : 0.0;   // x forward:  Vx[l][j]
    vf[1][kt] = ok ? __ldg(Vy + l * S + j) : 0.0;   // y forward:  Vy[l][k]
    vf[2][kt] = ok ? __ldg(Vz + l * S + j) : 0.0;   // z forward:  Vz[l][m]
    vf[3][kt] = ok ? __ldg(Vz + j * S + l) : 0.0;   // z back:     Vz[z][m]  (B[m][z])
    vf[4][kt] = ok ? __ldg(Vy + j * S + l) : 0.0;   // y back:     Vy[y][k]  (B[k][y])
    vf[5][kt] = ok ? __ldg(Vx + j * S + l) : 0.0;   // x back:     Vx[x][j]  (B[j][x])
  }
  cp_async_wait_all();
  __syncthreads();
  // ---- pass x ----
  for (int mt = warp; mt < MX; mt += NW) {
    double acc[NTX][2];
#pragma unroll
    for (int nt = 0; nt < NTX; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const double a = X[(8 * mt + r4) * LDX + 4 * kt + q4];
#pragma unroll
      for (int nt = 0; nt < NTX; ++nt) dmma(acc[nt][0], acc[nt][1], a, bxf[kt][nt]);
    }
#pragma unroll
    for (int nt = 0; nt < NTX; ++nt) {
      Pab[(8 * mt + r4) * LDP + 8 * nt + 2 * q4] = acc[nt][0];
      Pab[(8 * mt + r4) * LDP + 8 * nt + 2 * q4 + 1] = acc[nt][1];
    }
  }
  __syncthreads();
  // ---- pass y: columns (wz, lx) ----
  for (int nt = warp; nt < NTY; nt += NW) {
    double acc[MTY][2];
#pragma unroll
    for (int mt = 0; mt < MTY; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    const int col = 8 * nt + r4, wz = col / S, lx = col - wz * S;
    const bool okc = col < Wn * S;
#pragma unroll
    for (int kt = 0; kt < KY; ++kt) {
      const int r = 4 * kt + q4;
      const bool second = r >= WN4;
      const int rr = second ? r - WN4 : r;
      const double bv = (okc && rr < Wn) ? Pab[(wz * Wn + rr) * LDP + (second ? S : 0) + lx] : 0.0;
#pragma unroll
      for (int mt = 0; mt < MTY; ++mt) dmma(acc[mt][0], acc[mt][1], ayf[mt][kt], bv);
    }
#pragma unroll
    for (int mt = 0; mt < MTY; ++mt) {
      Q[(8 * mt + r4) * LDQ + 8 * nt + 2 * q4] = acc[mt][0];
      Q[(8 * mt + r4) * LDQ + 8 * nt + 2 * q4 + 1] = acc[mt][1];
    }
  }
  __syncthreads();
  // ---- pass z: columns (ly, lx); R = b_B - [M_z | K_z] [Pc; Pe] ----
  for (int nt = warp; nt < NTZ; nt += NW) {
    double a0 = 0.0, a1 = 0.0;
    const int col = 8 * nt + r4, ly = col / S, lx = col - ly * S;
    const bool okc = col < S2;
#pragma unroll
    for (int kt = 0; kt < KZ; ++kt) {
      const int r = 4 * kt + q4;
      const bool second = r >= WN4;
      const int rr = second ? r - WN4 : r;
      const double bv = (okc && rr < Wn) ? Q[((second ? S : 0) + ly) * LDQ + rr * S + lx] : 0.0;
      dmma(a0, a1, azf[kt], bv);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int cc = 8 * nt + 2 * q4 + i;
      if (r4 < S && cc < S2) R[r4 * S2 + cc] = Bb[r4 * S2 + cc] - (i ? a1 : a0);
    }
  }
  __syncthreads();
  // ---- FD: six contractions out[C(i,j)] = Σ_l in[A(i,l)] B[l][j] (rows i in [0, S^2)) ----
  const double *lx_ = lamt + (int64_t)cx * S, *ly_ = lamt + (int64_t)cy * S, *lz_ = lamt + (int64_t)cz * S;
  fd3_step<S, KF, MF, NW, 0>(R, T, vf[0], lx_, ly_, lz_);   // x forward: rows (z,y)
  fd3_step<S, KF, MF, NW, 1>(T, R, vf[1], lx_, ly_, lz_);   // y forward: rows (z,x)
  fd3_step<S, KF, MF, NW, 2>(R, T, vf[2], lx_, ly_, lz_);   // z forward, / (λx + λy + λz): rows (k,j)
  fd3_step<S, KF, MF, NW, 3>(T, R, vf[3], lx_, ly_, lz_);   // z back: rows (k,j)
  fd3_step<S, KF, MF, NW, 4>(R, T, vf[4], lx_, ly_, lz_);   // y back: rows (z,j)
  fd3_step<S, KF, MF, NW, 5>(T, R, vf[5], lx_, ly_, lz_);   // x back: rows (z,y)
  // ---- x_B += δ ----
  for (int i = threadIdx.x; i < S3; i += NW * 32) {
    const int lx = i % S, ly = (i / S) % S, lz = i / S2;
    const int gx = bx + lx, gy = by + ly, gz = bz + lz;
    if (unsigned(gx) < un && unsigned(gy) < un && unsigned(gz) < un)
      x[((int64_t)(gz - zoff) * n1 + gy) * n1 + gx] = X[((lz + P) * Wn + ly + P) * LDX + lx + P] + R[i];
  }
}

template <int P, int S, int NW>
bool try_schwarz3d_mma(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                       const double *b, double *x, int c0, int c1, int c2, int D, int nb0, int nb1, int nb2, int zoff,
                       cudaStream_t st) {
  if (p != P || s != S) return false;
  constexpr size_t sm = sizeof(double) * Mma3<P, S>::SM;
  ensure_smem(k_schwarz3d_mma<P, S, NW>, sm);
  k_schwarz3d_mma<P, S, NW><<<unsigned(nb0) * unsigned(nb1) * unsigned(nb2), NW * 32, sm, st>>>(
      int(n1), K, M, V, lam, b, x, c0, c1, c2, D, nb0, nb1, zoff);
  return true;
}

// ---------------- strided batched FP64 GEMM on the tensor pipe (DMMA) ----------------------------
// C[b](m, n) = Σ_k A[b](m, k) B[b](k, n), every operand addressed by (batch, row, col) strides.
// CTA 64 x 64 (4 warps, 32 x 32 each = 4 x 4 m8n8 fragments), K chunks of 16 double-buffered in shared
// memory by cp.async (zero fill outside M, N, K).
struct GemmArgs {
  const double *A, *B;
  double *C;
  int M, N, K;
  int64_t sAb, sAm, sAk, sBb, sBk, sBn, sCb, sCm, sCn;
};

constexpr int GBM = 64, GBN = 64, GBK = 16, GLDA = GBK + 1, GLDB = GBN + 1;

__global__ void __launch_bounds__(128) k_dgemm_mma(const GemmArgs g) {
  __shared__ double As[2][GBM * GLDA], Bs[2][GBK * GLDB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r4 = lane >> 2, q4 = lane & 3;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN, b = blockIdx.z;
  const double *A = g.A + b * g.sAb, *B = g.B + b * g.sBb;
  double *C = g.C + b * g.sCb;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  auto stage = [&](int k0, int buf) {
    for (int i = threadIdx.x; i < GBM * GBK; i += 128) {
      const int mm = i / GBK, kk = i - mm * GBK, gm = m0 + mm, gk = k0 + kk;
      const bool ok = gm < g.M && gk < g.K;
      cp_async8(&As[buf][mm * GLDA + kk], ok ? A + gm * g.sAm + gk * g.sAk : A, ok);
    }
    for (int i = threadIdx.x; i < GBK * GBN; i += 128) {
      const int kk = i / GBN, nn = i - kk * GBN, gk = k0 + kk, gn = n0 + nn;
      const bool ok = gk < g.K && gn < g.N;
      cp_async8(&Bs[buf][kk * GLDB + nn], ok ? B + gk * g.sBk + gn * g.sBn : B, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = (g.K + GBK - 1) / GBK;
  stage(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nk) {
      stage((kc + 1) * GBK, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < GBK / 4; ++ks) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][(wm + 8 * i + r4) * GLDA + 4 * ks + q4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][(4 * ks + q4) * GLDB + wn + 8 * j + r4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gm = m0 + wm + 8 * i + r4, gn = n0 + wn + 8 * j + 2 * q4 + e;
        if (gm < g.M && gn < g.N) C[gm * g.sCm + gn * g.sCn] = acc[i][j][e];
      }
}

// T[idx] /= Σ_a lam[i_a]  (x-fastest multi-index over n^dim)
__global__ void k_eig_divide(double *__restrict__ T, const double *__restrict__ lam, int n, int dim, int64_t total) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double den = lam[idx % n] + lam[(idx / n) % n];
    if (dim == 3) den += lam[idx / ((int64_t)n * n)];
    T[idx] /= den;
  }
}

}  // namespace

bool launch_schwarz_colour_fast(int dim, int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                                const double *lam, const double *b, double *x, int colour, int D, cudaStream_t st,
                                SlabView sv, const ToeP *tp, const double *fb) {
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
    const char *v3 = std::getenv("IGA2L_S3D_MMA");    // 3D block solves on DMMA: opt-in (measured 2x slower
    if ((v3 && v3[0] == '1') &&                        // than the DFMA pencil kernel)
        (try_schwarz3d_mma<1, 3, 4>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, st) ||
         try_schwarz3d_mma<2, 3, 4>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, st) ||
         try_schwarz3d_mma<3, 3, 4>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, st) ||
         try_schwarz3d_mma<4, 3, 4>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, st) ||
         try_schwarz3d_mma<5, 5, 8>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, st) ||
         try_schwarz3d_mma<6, 5, 8>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, st)))
      return true;
    return try_schwarz3d<1, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, tlo, thi, st, fb) ||
           try_schwarz3d<2, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, tlo, thi, st, fb) ||
           try_schwarz3d<3, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, tlo, thi, st, fb) ||
           try_schwarz3d<4, 3>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, tlo, thi, st, fb) ||
           try_schwarz3d<5, 5>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, tlo, thi, st, fb) ||
           try_schwarz3d<6, 5>(p, s, n1, K, M, V, lam, b, x, c0, c1, f2, D, nb0, nb1, nb2, z, tlo, thi, st, fb);
  }
  if (dim != 2) return false;
  const int c0 = colour % D, c1 = (colour / D) % D;
  int f1, nb1;
  centre_range(c1, D, sv.zlo, sv.zhi, &f1, &nb1);
  if (c0 >= n1 || nb1 == 0) return true;   // empty colour
  const int nb0 = int((n1 - c0 + D - 1) / D), nblk = nb0 * nb1;
  const int z = sv.zoff;
  if (s2d_variant() == 0 || s2d_variant() == 9)   // default: FP64 tensor-pipe kernel
    if (try_schwarz2d_mma<1, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb) ||
        try_schwarz2d_mma<2, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb) ||
        try_schwarz2d_mma<3, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb) ||
        try_schwarz2d_mma<4, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb) ||
        try_schwarz2d_mma<5, 5>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb) ||
        try_schwarz2d_mma<6, 5>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb) ||
        try_schwarz2d_mma<7, 7>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb) ||
        try_schwarz2d_mma<8, 7>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, fb))
      return true;
  if (const int v = s2d_variant(); v >= 1 && v <= 4)
    if (try_schwarz2d_r<1, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, v, tp) ||
        try_schwarz2d_r<2, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, v, tp) ||
        try_schwarz2d_r<3, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, v, tp) ||
        try_schwarz2d_r<4, 3>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, v, tp) ||
        try_schwarz2d_r<5, 5>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, v, tp) ||
        try_schwarz2d_r<6, 5>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, v, tp) ||
        try_schwarz2d_r<7, 7>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, v, tp) ||
        try_schwarz2d_r<8, 7>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st, v, tp))
      return true;
  // <P, S, blocks per CTA, warps per block>
  return try_schwarz2d<1, 3, 8, 1>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st) ||
         try_schwarz2d<2, 3, 8, 1>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st) ||
         try_schwarz2d<3, 3, 8, 1>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st) ||
         try_schwarz2d<4, 3, 4, 2>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st) ||
         try_schwarz2d<5, 5, 2, 4>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st) ||
         try_schwarz2d<6, 5, 2, 4>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st) ||
         try_schwarz2d<7, 7, 2, 4>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st) ||
         try_schwarz2d<8, 7, 2, 4>(p, s, n1, K, M, V, lam, b, x, c0, f1, D, nb0, nblk, z, st);
}

// Persistent sweep dispatcher (2D).  launch = false: number of tiles (= CTAs, = progress counters)
// the kernel would use, 0 if it cannot keep all of them co-resident, -1 if (p, s) is not specialised.
int sweep2d_persist(int p, int s, int64_t n1, const double *K, const double *M, const double *V, const double *lam,
                    const double *b, double *x, unsigned *ctl, unsigned *done, int max_tiles, cudaStream_t st,
                    bool launch) {
  int r;
  // <P, S, tile blocks AX x AY, groups per CTA, warps per group>
#define IGA2L_TRY(P_, S_, AX_, AY_, NB_, G_)                                                                    \
  if ((r = try_sweep2d_persist<P_, S_, AX_, AY_, NB_, G_>(p, s, n1, K, M, V, lam, b, x, ctl, done, max_tiles, st, \
                                                          launch)) >= 0)                                         \
    return r;
  IGA2L_TRY(1, 3, 2, 2, 4, 1)
  IGA2L_TRY(2, 3, 2, 2, 4, 1)
  IGA2L_TRY(3, 3, 2, 2, 4, 1)
  IGA2L_TRY(4, 3, 2, 2, 4, 2)
  IGA2L_TRY(5, 5, 2, 2, 4, 4)
  IGA2L_TRY(6, 5, 2, 2, 4, 4)
  IGA2L_TRY(7, 7, 4, 4, 4, 4)
  IGA2L_TRY(8, 7, 4, 4, 4, 4)
#undef IGA2L_TRY
  return -1;
}

bool launch_schwarz2d_tb(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                         const double *lam, const double *b, double *x, int col0, int ncol, int kc, cudaStream_t st) {
#define IGA2L_TB(P_, S_)                                                                                      \
  if (kc == 2 && try_schwarz2d_tb<P_, S_, 2>(p, s, n1, K, M, V, lam, b, x, col0, ncol, st)) return true;    \
  if (kc == 3 && try_schwarz2d_tb<P_, S_, 3>(p, s, n1, K, M, V, lam, b, x, col0, ncol, st)) return true;
  IGA2L_TB(1, 3) IGA2L_TB(2, 3) IGA2L_TB(3, 3) IGA2L_TB(4, 3) IGA2L_TB(5, 5) IGA2L_TB(6, 5)
#undef IGA2L_TB
  return false;
}

void launch_dgemm(const double *A, const double *B, double *C, int M, int N, int K, int batch, int64_t sAb,
                  int64_t sAm, int64_t sAk, int64_t sBb, int64_t sBk, int64_t sBn, int64_t sCb, int64_t sCm,
                  int64_t sCn, cudaStream_t st) {
  GemmArgs g{A, B, C, M, N, K, sAb, sAm, sAk, sBb, sBk, sBn, sCb, sCm, sCn};
  dim3 grid((unsigned)((N + GBN - 1) / GBN), (unsigned)((M + GBM - 1) / GBM), (unsigned)batch);
  k_dgemm_mma<<<grid, 128, 0, st>>>(g);
}

int launch_coarse_fd(int dim, int n, const double *V, const double *lam, const double *d, double *e, double *t1,
                     double *t2, cudaStream_t st) {
  const int64_t n1 = n, n2 = n1 * n1, n3 = n2 * n1;
  if (dim == 2) {   // D[y][x]: S = V^T D V ./ (λ_j + λ_k);  E = V S V^T
    launch_dgemm(d, V, t1, n, n, n, 1, 0, n1, 1, 0, n1, 1, 0, n1, 1, st);      // T1[y][j] = Σ_x D[y][x] V[x][j]
    launch_dgemm(V, t1, t2, n, n, n, 1, 0, 1, n1, 0, n1, 1, 0, n1, 1, st);     // S[k][j] = Σ_y V[y][k] T1[y][j]
    k_eig_divide<<<int(std::min<int64_t>((n2 + 255) / 256, 148 * 16)), 256, 0, st>>>(t2, lam, n, 2, n2);
    launch_dgemm(t2, V, t1, n, n, n, 1, 0, n1, 1, 0, 1, n1, 0, n1, 1, st);     // T2[k][x] = Σ_j S[k][j] V[x][j]
    launch_dgemm(V, t1, e, n, n, n, 1, 0, n1, 1, 0, n1, 1, 0, n1, 1, st);      // E[y][x] = Σ_k V[y][k] T2[k][x]
    return 5;
  }
  // D[z][y][x]: forward x, y, z with V^T, divide by λ_x + λ_y + λ_z, back z, y, x with V
  launch_dgemm(d, V, t1, int(n2), n, n, 1, 0, n1, 1, 0, n1, 1, 0, n1, 1, st);          // x
  launch_dgemm(V, t1, t2, n, n, n, n, 0, 1, n1, n2, n1, 1, n2, n1, 1, st);             // y (batch z)
  launch_dgemm(V, t2, t1, n, int(n2), n, 1, 0, 1, n1, 0, n2, 1, 0, n2, 1, st);         // z
  k_eig_divide<<<int(std::min<int64_t>((n3 + 255) / 256, 148 * 16)), 256, 0, st>>>(t1, lam, n, 3, n3);
  launch_dgemm(V, t1, t2, n, int(n2), n, 1, 0, n1, 1, 0, n2, 1, 0, n2, 1, st);         // z back
  launch_dgemm(V, t2, t1, n, n, n, n, 0, n1, 1, n2, n1, 1, n2, n1, 1, st);             // y back (batch z)
  launch_dgemm(t1, V, e, int(n2), n, n, 1, 0, n1, 1, 0, 1, n1, 0, n1, 1, st);          // x back
  return 7;
}

int export_interior_frags(int p, int s, int64_t n1, const double *K, const double *M, const double *V,
                          const double *lam, double *out, cudaStream_t st) {
  const int m = int(n1) - p + 2, tlo = 2 * p - 1, thi = m - 2 - p, w = (s - 1) / 2;
  if (thi - tlo < 2 * w) return -1;
  const int cref = (tlo + thi) / 2;
#define IGA2L_EXP(P_, S_)                                                                                   \
  if (p == P_ && s == S_) {                                                                                 \
    if (!out) return (frag_count<P_, S_>() + inv_count<S_>()) * 32;                                        \
    k_export_frags<P_, S_><<<1, 32, 0, st>>>(int(n1), cref, K, M, V, lam, out);                            \
    return (frag_count<P_, S_>() + inv_count<S_>()) * 32;                                                  \
  }
  IGA2L_EXP(1, 3) IGA2L_EXP(2, 3) IGA2L_EXP(3, 3) IGA2L_EXP(4, 3) IGA2L_EXP(5, 5) IGA2L_EXP(6, 5) IGA2L_EXP(7, 7)
  IGA2L_EXP(8, 7)
#undef IGA2L_EXP
  return -1;
}

// Interior block inverse of the 3D s = 3 pencil kernel, lane-major rows: out[j * 32 + l] = A_B^{-1}[l][j],
// A_B^{-1}[(lz,ly,lx)][(kz,ky,kx)] = Σ_{a,b,c} Vz[lz][c] Vy[ly][b] Vx[lx][a] Vz[kz][c] Vy[ky][b] Vx[kx][a] / (λa+λb+λc),
// every axis at the reference centre (A27).
__global__ void k_export_inv3(int cref, const double *__restrict__ Vt, const double *__restrict__ lamt, double *out) {
  constexpr int S = 3;
  const double *V = Vt + (int64_t)cref * S * S, *L = lamt + (int64_t)cref * S;
  const int l = threadIdx.x, lx = l % 3, ly = (l / 3) % 3, lz = l / 9;
  for (int j = 0; j < 27; ++j) {
    const int kx = j % 3, ky = (j / 3) % 3, kz = j / 9;
    double acc = 0.0;
    if (l < 27)
      for (int c = 0; c < S; ++c)
        for (int bb = 0; bb < S; ++bb)
          for (int a = 0; a < S; ++a)
            acc += V[lz * S + c] * V[ly * S + bb] * V[lx * S + a] * V[kz * S + c] * V[ky * S + bb] * V[kx * S + a] /
                   (L[a] + L[bb] + L[c]);
    out[j * 32 + l] = acc;
  }
}

int export_interior_inv3(int p, int s, int64_t n1, const double *V, const double *lam, double *out, cudaStream_t st) {
  const int m = int(n1) - p + 2, tlo = 2 * p - 1, thi = m - 2 - p, w = (s - 1) / 2;
  if (s != 3 || thi - tlo < 2 * w) return -1;
  if (out) k_export_inv3<<<1, 32, 0, st>>>((tlo + thi) / 2, V, lam, out);
  return 27 * 32;
}

int batch_ps_index(int p, int s) {
  const int tab[8][2] = {{1, 3}, {2, 3}, {3, 3}, {4, 3}, {5, 5}, {6, 5}, {7, 7}, {8, 7}};
  for (int i = 0; i < 8; ++i)
    if (tab[i][0] == p && tab[i][1] == s) return i;
  return -1;
}

size_t batch_smem_bytes(int ps) {
  const size_t per[8] = {Mma2<1, 3>::PER, Mma2<2, 3>::PER, Mma2<3, 3>::PER, Mma2<4, 3>::PER,
                         Mma2<5, 5>::PER, Mma2<6, 5>::PER, Mma2<7, 7>::PER, Mma2<8, 7>::PER};
  return ps >= 0 && ps < 8 ? per[ps] * sizeof(double) : 0;
}

void launch_schwarz2d_batch(const BatchDesc &d, size_t smem, cudaStream_t st) {
  const int nb = d.beg[d.n];
  if (nb <= 0) return;
  int maxps = 0;
  for (int j = 0; j < d.n; ++j)
    if (d.beg[j + 1] > d.beg[j]) maxps = std::max(maxps, d.pr[j].ps);
  const char *e = std::getenv("IGA2L_BATCH_WPC");
  const int wpc = e ? std::atoi(e) : 4;
  const int per = int(smem / sizeof(double));
  auto go = [&](auto kern, int w) {
    ensure_smem(kern, smem * w);
    kern<<<(nb + w - 1) / w, w * 32, smem * w, st>>>(d, per, mma_inv_enabled());
  };
  if (maxps <= 5) {
    if (wpc == 1) go(k_schwarz2d_mma_batch<1, 5>, 1);
    else if (wpc == 2) go(k_schwarz2d_mma_batch<2, 5>, 2);
    else go(k_schwarz2d_mma_batch<4, 5>, 4);
  } else {
    if (wpc == 1) go(k_schwarz2d_mma_batch<1, 7>, 1);
    else if (wpc == 2) go(k_schwarz2d_mma_batch<2, 7>, 2);
    else go(k_schwarz2d_mma_batch<4, 7>, 4);
  }
}

void launch_tensor2d(const double *in, double *out, const Band1D &B, int accumulate, cudaStream_t st,
                     int iylo, int iyhi, int iyoff, int rylo, int ryhi, int ryoff) {
  if (iyhi < 0) { iylo = 0; iyhi = B.cols; iyoff = 0; }
  if (ryhi < 0) { rylo = 0; ryhi = B.rows; ryoff = 0; }
  const int64_t total = (int64_t)(ryhi - rylo) * B.rows;
  if (total <= 0) return;
  const char *te = std::getenv("IGA2L_TRANSFER_SMALL");   // 16x16 separable tiles for small grids (default on)
  const bool small_sep = !(te && te[0] == '0');
  if (g_transfer_v2 && B.lo_max_span > 0 && (total >= 200000 || small_sep)) {   // separable two-pass
    auto go = [&](auto kern, int TO, int span) {
      const int LI = span + B.W;
      const size_t sm = sizeof(double) * (size_t(LI) * LI + size_t(LI) * TO + 2 * TO * B.W) + 2 * TO * sizeof(int);
      if (sm > 200 * 1024) return false;
      ensure_smem(kern, sm);
      dim3 grid((unsigned)((B.rows + TO - 1) / TO), (unsigned)((ryhi - rylo + TO - 1) / TO));
      kern<<<grid, 256, sm, st>>>(in, out, B.cols, B.rows, B.W, B.lo, B.c, accumulate, iylo, iyhi, iyoff, rylo, ryhi,
                                  ryoff, LI);
      return true;
    };
    if (total >= 200000) {
      if (go(k_transfer2d_sep<32>, 32, B.lo_max_span)) return;
    } else if (B.lo_max_span16 > 0 && go(k_transfer2d_sep<16>, 16, B.lo_max_span16)) {
      return;
    }
  }
  const int g = grid_for(total, 128);
  if (B.W <= 4)
    k_tensor2d<4><<<g, 128, 0, st>>>(in, out, B.cols, B.rows, B.W, B.lo, B.c, accumulate, iylo, iyhi, iyoff, rylo, ryhi, ryoff);
  else if (B.W <= 8)
    k_tensor2d<8><<<g, 128, 0, st>>>(in, out, B.cols, B.rows, B.W, B.lo, B.c, accumulate, iylo, iyhi, iyoff, rylo, ryhi, ryoff);
  else
    k_tensor2d<16><<<g, 128, 0, st>>>(in, out, B.cols, B.rows, B.W, B.lo, B.c, accumulate, iylo, iyhi, iyoff, rylo, ryhi, ryoff);
}

static int g_vc_cluster[4] = {0, 0, 0, 0};

void s2d_trace_read(long long *host8) { cudaMemcpyFromSymbol(host8, g_s2d_trace, 8 * sizeof(long long)); }

void vcycle_trace_enable(unsigned long long *dev_buf) {
  cudaMemcpyToSymbol(g_vc_trace, &dev_buf, sizeof(dev_buf));
  int z = 0;
  cudaMemcpyToSymbol(g_vc_trace_n, &z, sizeof(z));
}

int vcycle_cluster_size(int dim) {   // largest schedulable cluster (16 non-portable, else 8, 4, 2)
  int &c = g_vc_cluster[dim];
  if (c) return c;
  auto kern = dim == 2 ? k_vcycle_cluster<2, 2> : k_vcycle_cluster<3, 2>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (auto k2 : {k_vcycle_cluster<2, 1>, k_vcycle_cluster<3, 1>, k_vcycle_cluster<2, 2>, k_vcycle_cluster<3, 2>})
    cudaFuncSetAttribute(k2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 16; cs >= 1; cs /= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(512, 1, 1);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) {
      c = cs;
      return c;
    }
    cudaGetLastError();
  }
  c = 1;
  return c;
}

void launch_vcycle_cta(int dim, const QLevelDev *levs_dev, int l0, int nlev, int q, cudaStream_t st) {
  const int cs = vcycle_cluster_size(dim);
  auto kern = dim == 2 ? (q == 1 ? k_vcycle_cluster<2, 1> : k_vcycle_cluster<2, 2>)
                       : (q == 1 ? k_vcycle_cluster<3, 1> : k_vcycle_cluster<3, 2>);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 1, 1);
  cfg.blockDim = dim3(512, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, levs_dev, l0, nlev);
}

}  // namespace iga2l

namespace iga2l {
namespace {
__global__ void k_axpy(double *__restrict__ y, const double *__restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += x[i];
}
}  // namespace

void launch_axpy(double *y, const double *x, int64_t n, cudaStream_t st) {
  k_axpy<<<grid_for(n, 256), 256, 0, st>>>(y, x, n);
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

// optional phase clocks (thread 0 of cluster rank 0, buffered in shared memory, written at the end;
// tools/vc_trace.cu, -DIGA2L_TRACE)
#ifdef IGA2L_TRACE
__shared__ long long s_vc_clk[128];
__shared__ int s_vc_n;
#endif
__device__ __forceinline__ void vc_mark() {
#ifdef IGA2L_TRACE
  if (threadIdx.x == 0 && cg::this_cluster().block_rank() == 0) {
    if (s_vc_n < 128) s_vc_clk[s_vc_n] = clock64();
    ++s_vc_n;
  }
#endif
}
__device__ __forceinline__ void vc_flush() {
#ifdef IGA2L_TRACE
  if (threadIdx.x == 0 && cg::this_cluster().block_rank() == 0 && g_vc_trace) {
    for (int i = 0; i < s_vc_n && i < 128; ++i) g_vc_trace[i] = (unsigned long long)s_vc_clk[i];
    g_vc_trace_n = s_vc_n;
  }
#endif
}

template <int DIM>
struct XOff {               // level values in shared memory; last-axis row j stored at row j - zoff
  const double *x;
  int n, zoff;
  __device__ __forceinline__ double operator()(int jx, int jy, int jz) const {
    return DIM == 3 ? x[((jz - zoff) * n + jy) * n + jx] : x[(jy - zoff) * n + jx];
  }
};

// Σ_j a_ij x_j over the (2Q+1)^d stencil of point (ix, iy, iz) and a_ii (tables in shared memory)
template <int DIM, int Q, class XA>
__device__ __forceinline__ double q_point_acc(int n, const double *sK, const double *sM, const XA &xa, int ix,
                                              int iy, int iz, double *diag) {
  constexpr int W = 2 * Q + 1;
  const unsigned un = unsigned(n);
  double kx[W], mx[W], ky[W], my[W];
#pragma unroll
  for (int t = 0; t < W; ++t) {
    kx[t] = sK[ix * W + t]; mx[t] = sM[ix * W + t];
    ky[t] = sK[iy * W + t]; my[t] = sM[iy * W + t];
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
    for (int t = 0; t < W; ++t) { kz[t] = sK[iz * W + t]; mz[t] = sM[iz * W + t]; }
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
      vc_mark();
    }
    vc_residual<DIM, Q>(L, v, 0, false);
    __syncthreads();
    vc_mark();
    vc_restrict<DIM>(L, v, w, 0, w.n, w.b, 0, sm, si);
    __syncthreads();
    vc_mark();
  }
}

template <int DIM, int Q>
__device__ void vc_local_up(const VcLayout &L, int lf, double *sm, const int *si) {
  constexpr int ncol = DIM == 3 ? (Q + 1) * (Q + 1) * (Q + 1) : (Q + 1) * (Q + 1);
  for (int l = L.nlev - 2; l >= lf; --l) {
    const VcLev v = vc_level<DIM>(L, l, 0, sm), w = vc_level<DIM>(L, l + 1, 0, sm);
    vc_prolong<DIM>(L, v, w, XOff<DIM>{w.x, w.n, 0}, 0, false, sm, si);
    __syncthreads();
    vc_mark();
    for (int col = 0; col < ncol; ++col) {
      vc_gs_colour<DIM, Q>(L, v, col, 0, false);
      __syncthreads();
      vc_mark();
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
#ifdef IGA2L_TRACE
  if (threadIdx.x == 0) s_vc_n = 0;
  __syncthreads();
#endif
  vc_mark();
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
  vc_mark();
  // ---- down-sweep on the spread levels ----
  for (int l = l0; l < lf; ++l) {
    const VcLev v = vc_level<DIM>(L, l, rank, sm), w = vc_level<DIM>(L, l + 1, rank, sm);
    for (int col = 0; col < ncol; ++col) {
      vc_gs_colour<DIM, Q>(L, v, col, rank, true);
      cl.sync();
      vc_mark();
    }
    vc_residual<DIM, Q>(L, v, rank, true);
    cl.sync();
    vc_mark();
    if (l + 1 < lf) {                                             // into the next spread level (own rows)
      vc_restrict<DIM>(L, v, w, w.zlo, w.zhi, w.b, w.zoff, sm, si);
    } else {                                                      // into CTA 0's first level
      double *dst = cl.map_shared_rank(sm + L.b[l + 1], 0);
      vc_restrict<DIM>(L, v, w, L.rc0[rank], L.rc0[rank + 1], dst, 0, sm, si);
    }
    cl.sync();
    vc_mark();
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
    vc_mark();
  } else if (rank == 0) {
    vc_dense(inv, NC, sm + L.b[nlev - 1], sm + L.x[nlev - 1], 0, NC);
    __syncthreads();
    vc_mark();
  }
  if (rank == 0) vc_local_up<DIM, Q>(L, lf, sm, si);
  // ---- up-sweep on the spread levels ----
  if (spread) {
    cl.sync();
    vc_mark();
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
    vc_mark();
    for (int col = 0; col < ncol; ++col) {
      vc_gs_colour<DIM, Q>(L, v, col, rank, true);
      cl.sync();
      vc_mark();
    }
  }
  {
    const VcLev v = vc_level<DIM>(L, l0, rank, sm);
    const int tot = (v.zhi - v.zlo) * v.plane;
    for (int i = tid; i < tot; i += nthr) L.gx0[(int64_t)v.zlo * v.plane + i] = v.x[(v.zlo - v.zoff) * v.plane + i];
  }
  vc_mark();
  vc_flush();
}

}  // namespace

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

void launch_vcycle_smem(int dim, int q, const VcLayout &L, cudaStream_t st) {
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = vc_config(L, st, at);
  void *args[] = {const_cast<VcLayout *>(&L)};
  cudaLaunchKernelExC(&cfg, vc_kernel_for(dim, q), args);
}

}  // namespace iga2l
