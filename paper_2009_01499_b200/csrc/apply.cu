// Fine operator y = A x / y = b - A x and small vector kernels.  See kernels.cuh.
//
// A = Σ_a ⊗_b X_b (X_b = K if b == a else M) applied matrix-free by sum factorisation from the per-row
// 1D band tables K[i*(2p+1) + t+p] (row i, column i+t; zero outside the domain).
#include "common.cuh"
#include "kernels.cuh"

namespace iga2l {
namespace {

// ============================ fine operator: apply / residual ============================
// 2D tile TX x TY outputs; window (TX+2p) x (TY+2p) staged in shared memory.
template <int TX, int TY>
__global__ void __launch_bounds__(256) k_apply2d(int p, int n1, const double *__restrict__ K,
                                                 const double *__restrict__ M, const double *__restrict__ x,
                                                 const double *__restrict__ b, double *__restrict__ y,
                                                 double *__restrict__ partial, int mode, int zoff, int zlo, int zhi,
                                                 int64_t ys) {
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
    const double *kr = K + ys + (int64_t)gy * W, *mr = M + ys + (int64_t)gy * W;   // y-axis tables
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
                                                   int zoff, int zlo, int zhi, int tlo, int thi, const ToeP tp,
                                                   int64_t ys) {
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
      cp_async8(Ky + i, K + ys + (oky ? (int64_t)gy * W + t : 0), oky);   // y-axis tables (ys: per-axis)
      cp_async8(My + i, M + ys + (oky ? (int64_t)gy * W + t : 0), oky);
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
                 double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv, const ToeP *tpp, int64_t ys) {
  if (p != P) return false;
  ToeP tp{};
  if (tpp) tp = *tpp;
  const int nz = sv.zhi - sv.zlo;
  const int m = int(n1) - P + 2;
  auto go = [&](auto kern, int at, size_t sm) {
    ensure_smem(kern, sm);
    dim3 grid((unsigned)((n1 + at - 1) / at), (unsigned)((nz + at - 1) / at));
    kern<<<grid, at * at / ARY, sm, st>>>(int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi, 2 * P - 1,
                                          m - 2 - P, tp, ys);
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
  constexpr size_t sm = sizeof(double) * Apl3<P>::SM;
  ensure_smem(k_apply3d_s<P>, sm);
  k_apply3d_s<P><<<grid, A3NT, sm, st>>>(int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi, zchunk,
                                         2 * P - 1, m - 2 - P);
  if (nparts) *nparts = int(grid.x * grid.y * grid.z);
  return true;
}

constexpr int A2X = 32, A2Y = 8, A3X = 8, A3Y = 8, A3Z = 4;

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
size_t apply_smem(int dim, int p) {
  if (dim == 2) return sizeof(double) * ((A2X + 2 * p) * (A2Y + 2 * p) + 2 * (A2Y + 2 * p) * A2X);
  const size_t wx = A3X + 2 * p, wy = A3Y + 2 * p, wz = A3Z + 2 * p;
  return sizeof(double) * (wx * wy * wz + 2 * A3X * wy * wz + 2 * A3X * A3Y * wz);
}

__global__ void k_axpy(double *__restrict__ y, const double *__restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += x[i];
}

}  // namespace

int apply_num_partials(int dim, int p, int64_t n1) {
  if (dim == 2) {   // the most tiles any 2D apply variant launches
    const int64_t v1 = ((n1 + A2X - 1) / A2X) * ((n1 + A2Y - 1) / A2Y), v2 = ((n1 + 15) / 16) * ((n1 + 15) / 16);
    int v3 = 0;
    launch_apply_stream(dim, p, n1, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, &v3, kFull,
                        nullptr, true);
    return int(std::max<int64_t>(std::max(v1, v2), v3));
  }
  const int64_t v1 = ((n1 + A3X - 1) / A3X) * ((n1 + A3Y - 1) / A3Y) * ((n1 + A3Z - 1) / A3Z);
  const int64_t v2 = ((n1 + A3TX - 1) / A3TX) * ((n1 + A3TY - 1) / A3TY) * apply3d_zchunks(n1, int(n1));
  int v3 = 0;
  launch_apply_stream(dim, p, n1, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, &v3, kFull, nullptr,
                      true);
  return int(std::max<int64_t>(std::max(v1, v2), v3));
}

inline bool apply_stream_on() {                      // IGA2L_APPLY_STREAM=0: the tiled kernels below (read per call)
  const char *e = std::getenv("IGA2L_APPLY_STREAM");
  return !(e && e[0] == '0');
}

void launch_apply(int dim, int p, int64_t n1, const double *K, const double *M, const double *x, const double *b,
                  double *y, double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv, const ToeP *tp,
                  int64_t ys) {
  if (sv.zhi < 0) sv = SlabView{0, 0, int(n1)};
  const int nz = sv.zhi - sv.zlo;
  const size_t sm = apply_smem(dim, p);
  if (nz <= 0) return;
  if (ys == 0 && apply_stream_on() && launch_apply_stream(dim, p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, false))
    return;
  if (dim == 2 &&
      (try_apply2d<1>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, ys) ||
       try_apply2d<2>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, ys) ||
       try_apply2d<3>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, ys) ||
       try_apply2d<4>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, ys) ||
       try_apply2d<5>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, ys) ||
       try_apply2d<6>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, ys) ||
       try_apply2d<7>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, ys) ||
       try_apply2d<8>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, ys)))
    return;
  if (dim == 3 &&
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
    k_apply2d<A2X, A2Y><<<grid, 256, sm, st>>>(p, int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi, ys);
    if (nparts) *nparts = int(grid.x * grid.y);
  } else {
    const unsigned nbx = unsigned((n1 + A3X - 1) / A3X), nby = unsigned((n1 + A3Y - 1) / A3Y);
    dim3 grid(nbx * nby, (unsigned)((nz + A3Z - 1) / A3Z));
    ensure_smem(k_apply3d<A3X, A3Y, A3Z>, sm);
    k_apply3d<A3X, A3Y, A3Z><<<grid, 256, sm, st>>>(p, int(n1), K, M, x, b, y, partial, mode, sv.zoff, sv.zlo, sv.zhi);
    if (nparts) *nparts = int(grid.x * grid.y);
  }
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


void launch_axpy(double *y, const double *x, int64_t n, cudaStream_t st) {
  k_axpy<<<grid_for(n, 256), 256, 0, st>>>(y, x, n);
}

}  // namespace iga2l
