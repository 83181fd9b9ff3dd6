// Streaming 3D fine-operator kernel: y = A x / y = b - A x, input staged by TMA.
//
// The grid is swept along its LAST axis (z).  A CTA owns a tile of the other axes and a
// chunk of last-axis planes; every input plane window (tile + p-wide halo) is loaded by 1D TMA row copies
// into a ring of shared-memory stages (mbarrier completion; lane 0 of every warp issues its share of the rows),
// contracted along the in-plane axes without a CTA barrier (pass x of plane g beside pass y / z of plane g - 1,
// split-phase mbarriers between them)
// (sum factorisation, band coefficients of Toeplitz tiles as constant-bank operands, reading A27), and
// the last-axis contraction is accumulated in a REGISTER ring of 2p+1 partial output planes: input plane
// g contributes tap 2p-j to output plane g-p+j, and output plane g-p is complete after plane g.
//   3D: 2(2p+1)(TY+2p)/TY + 3(2p+1) + 2(2p+1) FMAs per output, 24 B / DOF.
// TMA row copies must start 16-byte aligned: rows are loaded from the even element at or below their
// first element and read with the parity shift.
// Out-of-domain window values: the 1D tensor map zero-fills outside the stored vector; values of a
// neighbouring row that a window row overhangs into are multiplied by band coefficients that are zero
// outside the domain (band tables, kernels.cuh), and outputs outside the domain are not stored.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace iga2l {

static bool encode_1d(void *map64, const double *ptr, int64_t n, int box, CUtensorMapSwizzle swz);

bool make_tmap_1d(void *map64, const double *ptr, int64_t n, int box) {
  return encode_1d(map64, ptr, n, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

bool make_tmap_1d_swz128(void *map64, const double *ptr, int64_t n, int box) {
  return box * 8 <= 128 && encode_1d(map64, ptr, n, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  return enc;
}

bool make_tmap_rows_swz128(void *map64, const double *ptr, int64_t cols, int64_t rows, int64_t stride, int box_cols,
                           int box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = encoder();
  if (!enc || rows <= 0 || cols <= 0 || box_cols * 8 > 128 || (box_cols * 8) % 16 || box_rows > 256 ||
      (stride * 8) % 16 || (reinterpret_cast<uintptr_t>(ptr) & 15))
    return false;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(stride * 8)};
  cuuint32_t boxd[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return enc(static_cast<CUtensorMap *>(map64), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(ptr), dims,
             strides, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool encode_1d(void *map64, const double *ptr, int64_t n, int box, CUtensorMapSwizzle swz) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = encoder();
  if (!enc || n <= 0 || box <= 0 || box > 256 || (box * 8) % 16 || (reinterpret_cast<uintptr_t>(ptr) & 15)) return false;
  cuuint64_t dims[1] = {cuuint64_t(n)};
  cuuint64_t strides[1] = {0};
  cuuint32_t boxd[1] = {cuuint32_t(box)};
  cuuint32_t es[1] = {1};
  return enc(static_cast<CUtensorMap *>(map64), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, const_cast<double *>(ptr), dims,
             strides, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

// ---------------------------------------------------------------------------------------------
// 3D: work = (x,y) tiles of TX x TY outputs times the z planes, linearised tile-major; a persistent CTA
// takes one contiguous segment of it (a few tiles' z ranges, so no wave quantisation and a z-halo only
// at segment ends).  Thread (lx, ly0) owns the OY outputs (lx, ly0 .. ly0+OY-1) of every output plane.
template <int P, int TY, int NT_, int MB = 0>
struct S3 {
  // BOX = WX + 2: TMA row starts must be 16-byte aligned, so a row is loaded from the even element at or
  // below its first needed element and read with a shift of 0 or 1 (odd n1 alternates the parity)
  static constexpr int TX = 32, W = 2 * P + 1, WX = TX + 2 * P, BOX = WX + 2, ROW = ((BOX + 15) / 16) * 16;
  static constexpr int WY = TY + 2 * P;
  static constexpr int NS = 4, NT = NT_, OY = TX * TY / NT;
  static constexpr int MINB = MB ? MB : (65536 / (NT * 128) > 0 ? 65536 / (NT * 128) : 1);
  static constexpr int NB = 4;                 // Pa/Pb ring: pass x of plane g + 1 may run beside pass y/z of plane g - 2
  static constexpr int NDBL = NS * WY * ROW + 2 * NB * WY * TX + 2 * TX * W + 2 * TY * W;
  static constexpr size_t SMEM = sizeof(double) * (NDBL + 32) + 8 * (NS + 2);
};

template <int P, int TY, int NT_, int MB = 0>
__global__ void __launch_bounds__(NT_, S3<P, TY, NT_, MB>::MINB)
    k_apply3d_tma(const __grid_constant__ CUtensorMap xmap, int n1, const double *__restrict__ K,
                  const double *__restrict__ M, const double *__restrict__ b, double *__restrict__ y,
                  double *__restrict__ partial, int mode, int zoff, int zlo0, int nz, int64_t work, int tlo,
                  int thi, const ToeP tp) {
  using A = S3<P, TY, NT_, MB>;
  constexpr int TX = A::TX, W = A::W, ROW = A::ROW, WY = A::WY, NS = A::NS, NT = A::NT, OY = A::OY;
  extern __shared__ __align__(128) double sm[];
  double *stage = sm;                         // [NS][WY][ROW]  input plane windows
  double *Pa = stage + NS * WY * ROW;         // [NB][WY][TX]   K_x X
  double *Pb = Pa + A::NB * WY * TX;          // [NB][WY][TX]   M_x X
  double *ckx = Pb + A::NB * WY * TX, *cmx = ckx + TX * W;   // band rows of the tile's x rows (boundary tiles)
  double *cky = cmx + TX * W, *cmy = cky + TY * W;       // ... and y rows
  double *red = cmy + TY * W;                 // [32] block reduction scratch
  uint64_t *bar = reinterpret_cast<uint64_t *>(red + 32);
  uint64_t *px = bar + NS;                    // [2] "pass x of plane n done by every warp" (n & 1), see the plane loop
  const int tid = threadIdx.x;
  const bool tv = tp.valid != 0;
  const int64_t plane = int64_t(n1) * n1;
  const int ntx = (n1 + TX - 1) / TX;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    mbar_init(&px[0], NT / 32);
    mbar_init(&px[1], NT / 32);
    mbar_fence_init();
  }
  double sq = 0.0;
  unsigned phase = 0;
  int it = 0;                                 // planes consumed by this CTA (stage ring position)
  const int lx = tid % TX, ly0 = (tid / TX) * OY;
  const int64_t w0 = work * blockIdx.x / gridDim.x, w1 = work * (blockIdx.x + 1) / gridDim.x;
  for (int64_t w = w0; w < w1;) {
    const int64_t tile = w / nz;
    const int zlo = zlo0 + int(w - tile * nz);
    const int64_t wend = min(w1, (tile + 1) * int64_t(nz));
    const int zhi = zlo0 + int(wend - tile * nz);
    w = wend;
    const int x0 = int(tile % ntx) * TX, y0 = int(tile / ntx) * TY, gx = x0 + lx;
    const bool toex = tv && x0 >= tlo && x0 + TX - 1 <= thi, toey = tv && y0 >= tlo && y0 + TY - 1 <= thi;
    __syncthreads();                          // previous tile's passes are done with the tables
    for (int i = tid; i < TX * W; i += NT) {
      const int g = x0 + i / W;
      ckx[i] = g < n1 ? K[int64_t(g) * W + i % W] : 0.0;
      cmx[i] = g < n1 ? M[int64_t(g) * W + i % W] : 0.0;
    }
    for (int i = tid; i < TY * W; i += NT) {
      const int g = y0 + i / W;
      cky[i] = g < n1 ? K[int64_t(g) * W + i % W] : 0.0;
      cmy[i] = g < n1 ? M[int64_t(g) * W + i % W] : 0.0;
    }
    __syncthreads();
    const int gs = zlo - P, ge = zhi + P;     // input planes [gs, ge)
    // plane gi's WY window rows into stage s: lane 0 of warp w issues rows w, w + NT/32, ... (a TMA issue is
    // per thread, so one issuing warp would be WY issues late at every plane's CTA barrier: 24% of the stall
    // samples); the expect-tx arrival may follow some of the copies' complete-tx (the count is signed)
    auto issue = [&](int gi, int s) {
      if (unsigned(gi) >= unsigned(n1)) return;
      if (tid == 0) mbar_expect_tx(&bar[s], WY * A::BOX * 8);
      if ((tid & 31) == 0)
        for (int r = tid >> 5; r < WY; r += NT / 32)
          tma_load_1d(stage + (s * WY + r) * ROW, &xmap,
                      int(int64_t(gi - zoff) * plane + int64_t(y0 - P + r) * n1 + (x0 - P)) & ~1, &bar[s]);
    };
    for (int k = 0; k < NS && gs + k < ge; ++k) issue(gs + k, (it + k) % NS);
    double acc[W][OY];
#pragma unroll
    for (int j = 0; j < W; ++j)
#pragma unroll
      for (int o = 0; o < OY; ++o) acc[j][o] = 0.0;
    // Software pipeline without a CTA barrier: iteration gq runs pass x of plane gq (stage A) and then pass y / z of
    // plane gq - 1 (stage B).  A warp arrives on px[n & 1] after its pass x of the CTA's n-th plane and waits for
    // that phase only one stage later, so warps drift by up to one plane instead of meeting at every plane; the
    // Pa/Pb ring of NB = 4 keeps the plane a leading warp writes (n + 1) apart from the one a trailing warp still
    // reads (n - 2); a TMA stage is refilled after the wait that proves every warp has passed it in x.
    for (int gq = gs; gq <= ge; ++gq) {
      const int gi = gq - 1;                  // stage B's plane
      const int go = gi - P;                  // output plane completed by input plane gi
      const bool out = gq > gs && go >= zlo && go < zhi;
      double bv[OY];
#pragma unroll
      for (int o = 0; o < OY; ++o) {          // prefetch b (used after the passes)
        const int gy = y0 + ly0 + o;
        bv[o] = (mode && out && gx < n1 && gy < n1) ? b[int64_t(go - zoff) * plane + int64_t(gy) * n1 + gx] : 0.0;
      }
      if (gq < ge) {                          // ---- stage A: pass x of plane gq ----
      const int s = it % NS;
      double *pa = Pa + (it % A::NB) * WY * TX, *pb = Pb + (it % A::NB) * WY * TX;
      if (unsigned(gq) < unsigned(n1)) {
        const int gi = gq;
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
        const double *X = stage + s * WY * ROW;
        const int pbase = int(int64_t(gi - zoff) * plane + int64_t(y0 - P) * n1 + (x0 - P));
        // pass x: a task is (row, 2 outputs); a warp takes two rows of EQUAL start parity (rows wy, wy + 2), so
        // the parity shift is warp-uniform and the window comes in by 16-byte loads at a 16-byte lane stride
        // (conflict-free quarter-warps) from the even element at or below the first needed one
        constexpr int HC = (WY + 1) / 2, TC = (HC + 1) / 2;          // rows per parity class, warp tasks per class
        for (int wt = tid >> 5; wt < 2 * TC; wt += NT / 32) {
          const int cls = wt / TC, wy = cls + 2 * (2 * (wt - cls * TC) + ((tid >> 4) & 1)), l0 = (tid & 15) * 2;
          if (wy >= WY) continue;
          const double2 *Xr = reinterpret_cast<const double2 *>(X + wy * ROW + l0);
          double a0 = 0.0, a1 = 0.0, m0 = 0.0, m1 = 0.0;
          auto row = [&](auto shc) {
            constexpr int SH = decltype(shc)::value, NV = (2 + 2 * P + SH + 1) / 2;
            double v[2 * NV];
#pragma unroll
            for (int k = 0; k < NV; ++k) {
              const double2 t2 = Xr[k];
              v[2 * k] = t2.x;
              v[2 * k + 1] = t2.y;
            }
            if (toex) {
#pragma unroll
              for (int t = 0; t < W; ++t) {
                a0 = fma(tp.k[t], v[SH + t], a0);
                a1 = fma(tp.k[t], v[SH + t + 1], a1);
                m0 = fma(tp.m[t], v[SH + t], m0);
                m1 = fma(tp.m[t], v[SH + t + 1], m1);
              }
            } else {
#pragma unroll
              for (int t = 0; t < W; ++t) {
                a0 = fma(ckx[l0 * W + t], v[SH + t], a0);
                a1 = fma(ckx[(l0 + 1) * W + t], v[SH + t + 1], a1);
                m0 = fma(cmx[l0 * W + t], v[SH + t], m0);
                m1 = fma(cmx[(l0 + 1) * W + t], v[SH + t + 1], m1);
              }
            }
          };
          if ((pbase + cls * n1) & 1)             // row start parity (see S3::BOX); equal for rows cls, cls + 2, ...
            row(std::integral_constant<int, 1>{});
          else
            row(std::integral_constant<int, 0>{});
          *reinterpret_cast<double2 *>(pa + wy * TX + l0) = make_double2(a0, a1);
          *reinterpret_cast<double2 *>(pb + wy * TX + l0) = make_double2(m0, m1);
        }
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&px[it & 1]);
      ++it;
      }
      if (gq == gs) continue;                 // ---- stage B: pass y / z of plane gi = gq - 1 ----
      const int itb = it - (gq < ge ? 2 : 1);  // ring position of plane gi
      mbar_wait(&px[itb & 1], unsigned(itb >> 1) & 1u);   // Pa/Pb of plane gi ready; its stage consumed by every warp
      if (gi + NS < ge) issue(gi + NS, itb % NS);
      const bool live = unsigned(gi) < unsigned(n1);
      const double *pa = Pa + (itb % A::NB) * WY * TX, *pb = Pb + (itb % A::NB) * WY * TX;
      double c[OY], e[OY];
#pragma unroll
      for (int o = 0; o < OY; ++o) c[o] = e[o] = 0.0;
      if (live) {                             // pass y: c = My Pa + Ky Pb, e = My Pb
        double va[OY + 2 * P], vb[OY + 2 * P];
#pragma unroll
        for (int u = 0; u < OY + 2 * P; ++u) {
          va[u] = pa[(ly0 + u) * TX + lx];
          vb[u] = pb[(ly0 + u) * TX + lx];
        }
#pragma unroll
        for (int o = 0; o < OY; ++o) {
          double c1 = 0.0;
          if (toey) {
#pragma unroll
            for (int u = 0; u < W; ++u) {
              c[o] = fma(tp.m[u], va[o + u], c[o]);
              c1 = fma(tp.k[u], vb[o + u], c1);
              e[o] = fma(tp.m[u], vb[o + u], e[o]);
            }
          } else {
#pragma unroll
            for (int u = 0; u < W; ++u) {
              const double my = cmy[(ly0 + o) * W + u], ky = cky[(ly0 + o) * W + u];
              c[o] = fma(my, va[o + u], c[o]);
              c1 = fma(ky, vb[o + u], c1);
              e[o] = fma(my, vb[o + u], e[o]);
            }
          }
          c[o] += c1;
        }
      }
      // last axis: output plane gi - P + j receives tap 2P - j of this input plane
      if (tv && gi - P >= tlo && gi + P <= thi) {
#pragma unroll
        for (int j = 0; j < W; ++j)
#pragma unroll
          for (int o = 0; o < OY; ++o) acc[j][o] = fma(tp.m[2 * P - j], c[o], fma(tp.k[2 * P - j], e[o], acc[j][o]));
      } else if (live) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int gz = min(max(gi - P + j, 0), n1 - 1);     // rows outside the domain are never stored
          const double mz = __ldg(M + int64_t(gz) * W + 2 * P - j), kz = __ldg(K + int64_t(gz) * W + 2 * P - j);
#pragma unroll
          for (int o = 0; o < OY; ++o) acc[j][o] = fma(mz, c[o], fma(kz, e[o], acc[j][o]));
        }
      }
      if (out) {
#pragma unroll
        for (int o = 0; o < OY; ++o) {
          const int gy = y0 + ly0 + o;
          if (gx < n1 && gy < n1) {
            const double val = mode ? bv[o] - acc[0][o] : acc[0][o];
            y[int64_t(go - zoff) * plane + int64_t(gy) * n1 + gx] = val;
            sq = fma(val, val, sq);
          }
        }
      }
#pragma unroll
      for (int j = 0; j + 1 < W; ++j)
#pragma unroll
        for (int o = 0; o < OY; ++o) acc[j][o] = acc[j + 1][o];
#pragma unroll
      for (int o = 0; o < OY; ++o) acc[W - 1][o] = 0.0;
    }
  }
  if (partial) {
    const double t = block_sum(sq, red);
    if (tid == 0) partial[blockIdx.x] = t;
  }
}

// A/B knob IGA2L_STREAM_CFG: 1 = TY 8 / 256 threads, 2 = TY 16 / 256 threads, 3 = TY 16 / 512 threads,
// 4 / 5 = TY 8 / 256 threads at 3 / 4 CTAs per SM (80 / 64 registers)
int stream_cfg() {                                   // read per call (tests switch it within one process)
  const char *e = std::getenv("IGA2L_STREAM_CFG");
  return e ? std::atoi(e) : 0;
}

template <int P, int TY, int NT, int MB = 0>
bool go_stream3d(int64_t n1, const double *K, const double *M, const double *x, const double *b, double *y,
                 double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv, const ToeP *tpp, bool count) {
  using A = S3<P, TY, NT, MB>;
  const int nz = sv.zhi - sv.zlo;
  const int64_t tiles = ((n1 + A::TX - 1) / A::TX) * ((n1 + TY - 1) / TY), work = tiles * nz;
  // persistent: MINB CTAs per SM; segments no shorter than 8p planes (z halo <= 25%)
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(148 * A::MINB, work / (8 * P))));
  if (nparts) *nparts = grid;
  if (count) return true;
  CUtensorMap map;
  const int64_t stored = (std::min<int64_t>(n1, sv.zhi + P) - sv.zoff) * n1 * n1;
  if (!make_tmap_1d(&map, x, stored, A::BOX)) return false;
  ToeP tp{};
  if (tpp) tp = *tpp;
  const int m = int(n1) - P + 2;
  ensure_smem(k_apply3d_tma<P, TY, NT, MB>, A::SMEM);
  k_apply3d_tma<P, TY, NT, MB><<<grid, NT, A::SMEM, st>>>(map, int(n1), K, M, b, y, partial, mode, sv.zoff, sv.zlo, nz,
                                                      work, 2 * P - 1, m - 2 - P, tp);
  return true;
}

template <int P>
bool try_stream3d(int p, int64_t n1, const double *K, const double *M, const double *x, const double *b, double *y,
                  double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv, const ToeP *tpp, bool count) {
  if (p != P) return false;
  // measured (C4 p = 3, C5 p = 5): TY 8 / 256 threads at 3 CTAs per SM (80 registers) for p <= 4 (C4 65.5 us; 2 CTAs
  // 70.7, 4 CTAs at 64 registers 84), TY 16 / 256 threads at 2 CTAs per SM above (C5 510 us; TY 8 at 3 CTAs 613,
  // 512 threads 583)
  if (count) {                                        // partial-buffer sizing: the most any config writes
    int a = 0, c = 0, d = 0;
    go_stream3d<P, 8, 256>(n1, K, M, x, b, y, partial, mode, st, &a, sv, tpp, true);
    go_stream3d<P, 16, 256>(n1, K, M, x, b, y, partial, mode, st, &c, sv, tpp, true);
    go_stream3d<P, 16, 512>(n1, K, M, x, b, y, partial, mode, st, &d, sv, tpp, true);
    int e = 0, f = 0;
    go_stream3d<P, 8, 256, 3>(n1, K, M, x, b, y, partial, mode, st, &e, sv, tpp, true);
    go_stream3d<P, 8, 256, 4>(n1, K, M, x, b, y, partial, mode, st, &f, sv, tpp, true);
    if (nparts) *nparts = std::max(std::max(a, e), std::max(c, std::max(d, f)));
    return true;
  }
  const int cfg = stream_cfg() ? stream_cfg() : (P <= 4 ? 4 : 2);
  if (cfg == 1) return go_stream3d<P, 8, 256>(n1, K, M, x, b, y, partial, mode, st, nparts, sv, tpp, count);
  if (cfg == 2) return go_stream3d<P, 16, 256>(n1, K, M, x, b, y, partial, mode, st, nparts, sv, tpp, count);
  if (cfg == 4) return go_stream3d<P, 8, 256, 3>(n1, K, M, x, b, y, partial, mode, st, nparts, sv, tpp, count);
  if (cfg == 5) return go_stream3d<P, 8, 256, 4>(n1, K, M, x, b, y, partial, mode, st, nparts, sv, tpp, count);
  return go_stream3d<P, 16, 512>(n1, K, M, x, b, y, partial, mode, st, nparts, sv, tpp, count);
}

}  // namespace

bool launch_apply_stream(int dim, int p, int64_t n1, const double *K, const double *M, const double *x, const double *b,
                         double *y, double *partial, int mode, cudaStream_t st, int *nparts, SlabView sv,
                         const ToeP *tp, bool count_only) {
  if (sv.zhi < 0) sv = SlabView{0, 0, int(n1)};
  if (dim != 3 || sv.zhi - sv.zlo <= 0) return false;   // 2D: the tiled kernel (apply.cu) is faster
  return try_stream3d<1>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, count_only) ||
         try_stream3d<2>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, count_only) ||
         try_stream3d<3>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, count_only) ||
         try_stream3d<4>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, count_only) ||
         try_stream3d<5>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, count_only) ||
         try_stream3d<6>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, count_only) ||
         try_stream3d<7>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, count_only) ||
         try_stream3d<8>(p, n1, K, M, x, b, y, partial, mode, st, nparts, sv, tp, count_only);
}

}  // namespace iga2l
