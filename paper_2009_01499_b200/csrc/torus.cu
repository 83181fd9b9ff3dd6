// Torus LFA run: the two-grid error operator of Algorithm 1 on an n x n
// PERIODIC grid, applied by the hot-path kernels and power-iterated for its spectral radius.
//
// Local Fourier analysis reads the method on the infinite uniform grid, where every operator is
// a convolution; on the n-point torus the same operators are circulant, and the torus spectrum is the LFA
// symbol sampled at θ = 2πk/n.  With n = nk (s + p) (nk even) those frequencies are exactly the nk^2 Bloch
// quasi-momenta the oracle's block LFA (`oracle/lfa.py: rho_2g`, `rho_2g_ag`) samples, so the measured ρ
// pins the analysis at scale.
//
//   E = (I - P A_c^+ R A_p) S_p        (same h, q: Table 1's setting; or H = 2h, Table 3's)
//
// * S_p: the multicolour Schwarz sweep (reading A4) by the colour kernels of the Dirichlet path, run on a
//   padded grid of n + 2G points per axis (G = 2w + p) whose band tables are the interior (Toeplitz, A27)
//   rows everywhere; after each colour the ghost layers are refreshed from their periodic images.  A block
//   centred in a ghost layer is the periodic image of a real block of the same colour (n % D == 0) and
//   writes the same update into the real points it covers; blocks whose windows leave the padded grid
//   only write ghost points, which the refresh overwrites.
// * A_p: the residual kernel on the padded grid (b = 0); R = D^{-1} M_c (lumped, A6) and, for
//   H = 2h, composed with the knot-insertion restriction (A8/A9): periodic band transfers; P = R^T.
// * A_c^+: Kronecker fast diagonalisation with the circulant 1D eigen-decompositions;
//   the constant mode (A_c 1 = 0) gets 0 (pseudo-inverse, as LFA excludes θ = 0's constant).
// * Power iteration from a seeded random mean-zero start; the mean (the constant, E 1 = 1) is projected
//   out after every application.  ρ = geometric mean of the last quarter of the norm ratios.
// 2D and 3D (the padded sweep is the same construction; in 3D the rediscretised 2h operator is twice h's
// stencil, A10); the three-grid mode is 2D.
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "host_setup.h"
#include "kernels.cuh"

namespace iga2l {
namespace {

// ghost layers of an np^dim padded array (real block [G, G+n)^dim) from their periodic images
__global__ void k_ghost(double *__restrict__ x, int dim, int n, int G) {
  const int np = n + 2 * G;
  const int64_t tot = dim == 3 ? (int64_t)np * np * np : (int64_t)np * np;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = int(idx % np), j = int((idx / np) % np), k = dim == 3 ? int(idx / ((int64_t)np * np)) : G;
    const bool gh = i < G || i >= G + n || j < G || j >= G + n || k < G || k >= G + n;
    if (!gh) continue;
    const int si = G + ((i - G) % n + n) % n, sj = G + ((j - G) % n + n) % n, sk = G + ((k - G) % n + n) % n;
    x[idx] = x[dim == 3 ? ((int64_t)sk * np + sj) * np + si : (int64_t)sj * np + si];
  }
}

// compact n^dim <-> real block of the padded array; mode 0: pad = c, 1: c = pad
__global__ void k_pad(double *__restrict__ pad, double *__restrict__ c, int dim, int n, int G, int mode) {
  const int np = n + 2 * G;
  const int64_t tot = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = int(idx % n), j = int((idx / n) % n), k = dim == 3 ? int(idx / ((int64_t)n * n)) : 0;
    double *pp = pad + (dim == 3 ? ((int64_t)(k + G) * np + j + G) * np + i + G : (int64_t)(j + G) * np + i + G);
    if (mode == 0) *pp = c[idx];
    else c[idx] = *pp;
  }
}

// periodic band transfer along one axis, [outer][nin][inner] -> [outer][nout][inner].  Forward (restriction R):
//   out[i] = Σ_k c[k] in[(ratio i + o0 + k) mod nin];
// transpose (prolongation R^T): out[j] = Σ_{i, k: ratio i + o0 + k ≡ j} c[k] in[i].
__global__ void k_pband(const double *__restrict__ in, double *__restrict__ out, int nin, int nout, int64_t outer,
                        int64_t inner, const double *__restrict__ c, int W, int o0, int ratio, int transpose,
                        int accumulate) {
  const int64_t total = outer * nout * inner;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx % inner, ob = idx / inner;
    const int o = int(ob % nout);
    const int64_t u = ob / nout;
    const double *src = in + u * nin * inner + t;
    double acc = 0.0;
    if (!transpose) {
      for (int k = 0; k < W; ++k) acc = fma(c[k], src[(int64_t)(((ratio * o + o0 + k) % nin + nin) % nin) * inner], acc);
    } else {
      for (int k = 0; k < W; ++k) {
        const int r = o - o0 - k;                               // = ratio * i (mod ratio * nin)
        const int rm = ((r % (ratio * nin)) + ratio * nin) % (ratio * nin);
        if (rm % ratio) continue;
        acc = fma(c[k], src[(int64_t)(rm / ratio) * inner], acc);
      }
    }
    out[idx] = accumulate ? out[idx] + acc : acc;
  }
}

// d-dim periodic transfer, axis by axis (x first): n_in^d -> n_out^d through tmp0/tmp1 (n_max^d each)
void pband_nd(int dim, const double *in, double *out, int nin, int nout, const double *c, int W, int o0, int ratio,
              int transpose, int accumulate, double *tmp0, double *tmp1, cudaStream_t st) {
  int64_t sz[3] = {nin, nin, dim == 3 ? nin : 1};
  const double *src = in;
  for (int a = 0; a < dim; ++a) {
    const bool last = a == dim - 1;
    double *dst = last ? out : (a % 2 == 0 ? tmp0 : tmp1);
    int64_t inner = 1, outer = 1;
    for (int b = 0; b < a; ++b) inner *= sz[b];
    for (int b = a + 1; b < dim; ++b) outer *= sz[b];
    const int64_t tot = outer * nout * inner;
    k_pband<<<grid_for(tot, 256), 256, 0, st>>>(src, dst, nin, nout, outer, inner, c, W, o0, ratio, transpose,
                                                last ? accumulate : 0);
    sz[a] = nout;
    src = dst;
  }
}

// degree-q operator on the n x n torus, direct (2q+1)^2 stencil A = K ⊗ M + M ⊗ K (row stencils k, m)
__device__ __forceinline__ double torus_ax(const double *__restrict__ x, int n, int q, const double *k,
                                           const double *m, int i, int j, double *diag) {
  double acc = 0.0;
  for (int b = -q; b <= q; ++b) {
    const int jj = ((j + b) % n + n) % n;
    for (int a = -q; a <= q; ++a) {
      const int ii = ((i + a) % n + n) % n;
      acc = fma(k[a + q] * m[b + q] + m[a + q] * k[b + q], x[(int64_t)jj * n + ii], acc);
    }
  }
  *diag = 2.0 * k[q] * m[q];
  return acc;
}
struct QRows {
  double k[5], m[5];
};
// one colour (c0, c1) of the (q+1)^2-colour Gauss-Seidel (reading A11): points (q+1) apart do not couple
__global__ void k_torus_gs(double *__restrict__ x, const double *__restrict__ b, int n, int q, QRows r, int c0,
                           int c1) {
  const int st = q + 1, na = n / st;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)na * na;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = c0 + st * int(idx % na), j = c1 + st * int(idx / na);
    double dg;
    const double ax = torus_ax(x, n, q, r.k, r.m, i, j, &dg);
    x[(int64_t)j * n + i] += (b[(int64_t)j * n + i] - ax) / dg;
  }
}
__global__ void k_torus_resid(double *__restrict__ rr, const double *__restrict__ b, const double *__restrict__ x,
                              int n, int q, QRows r) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double dg;
    rr[idx] = b[idx] - torus_ax(x, n, q, r.k, r.m, int(idx % n), int(idx / n), &dg);
  }
}

// sum and sum of squares of v[0..N) (one CTA, fixed order)
__global__ void k_sums(const double *__restrict__ v, int64_t N, double *out) {
  __shared__ double red[32];
  double s = 0.0, q = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
    s += v[i];
    q = fma(v[i], v[i], q);
  }
  s = block_sum(s, red);
  __syncthreads();
  q = block_sum(q, red);
  if (threadIdx.x == 0) {
    out[0] = s;
    out[1] = q;
  }
}

// v = (v - mean) * scale
__global__ void k_shift_scale(double *__restrict__ v, int64_t N, double mean, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (v[i] - mean) * scale;
}

uint64_t splitmix(uint64_t &st) {
  uint64_t z = (st += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct DevBuf {
  std::vector<void *> ptrs;
  ~DevBuf() {
    for (void *p : ptrs) cudaFree(p);
  }
  template <typename T>
  T *get(size_t n, cudaError_t *e) {
    void *p = nullptr;
    *e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
    if (*e == cudaSuccess) ptrs.push_back(p);
    return static_cast<T *>(p);
  }
};

}  // namespace

int lfa_torus_run(int dim, int p, int q, int n, int s, int hf, int iters, unsigned long long seed, double *rho,
                  double *ratios, std::string *err) {
  auto bad = [&](const std::string &m) {
    *err = m;
    return 1;   // IGA2L_EPARAM
  };
  if (dim != 2 && dim != 3) return bad("dim must be 2 or 3");
  if (p < 1 || p > 8) return bad("p must be in 1..8");
  if (q < 1 || q > 2 || q > p) return bad("q must satisfy 1 <= q <= min(p, 2)");
  if (s != 1 && s != 3 && s != 5 && s != 7) return bad("block must be 1, 3, 5 or 7");
  if (hf < 1 || hf > 3) return bad("h_factor must be 1 (two-grid, same h), 2 (aggressive) or 3 (three-grid)");
  const bool three = hf == 3;
  if (three && dim != 2) return bad("the three-grid torus run is 2D");
  if (three && (n % 2 || n % (q + 1) || n / 2 < 2 * q + 1))
    return bad("three-grid: n must be even, a multiple of q + 1, and n / 2 >= 2q + 1");
  const int D = s + p, w = (s - 1) / 2, W = 2 * p + 1;
  if (n % D != 0 || n < 2 * D) return bad("n must be a multiple of s + p and at least 2 (s + p)");
  if (hf == 2 && (n % 2 != 0 || n / 2 < 2 * q + 1)) return bad("aggressive: n must be even and n / 2 >= 2q + 1");
  if (iters < 4 || iters > 100000) return bad("iters must be in 4..100000");
  if (!rho) return bad("rho is NULL");
  // ---- interior (Toeplitz, A27) rows from a Dirichlet grid large enough to have them ----
  const int64_t mb = 4 * (2 * p + s + 8);
  std::vector<double> Kb, Mb, Kq, Mq;
  band_tables(p, mb, Kb, Mb);
  band_tables(q, mb, Kq, Mq);
  int64_t lo, hi;
  toeplitz_rows(p, mb, &lo, &hi);
  const int64_t rp = (lo + hi) / 2;
  toeplitz_rows(q, mb, &lo, &hi);
  const int64_t rq = (lo + hi) / 2;
  const BandOp R1 = degree_restriction(p, q, mb);
  const int64_t ir = R1.rows / 2;                         // an interior row: cols ir - q + k, k = 0..p+q
  // R on the torus (q-function i and p-function j numbered by the cell their support starts in):
  // row i couples p-columns j = i + k - p with R1's interior coefficients (same h); for H = 2h the knot-
  // insertion restriction (A8/A9) is folded in: row J = Σ_k' 2^{-q} C(q+1, k') (row 2J + k' at h).
  std::vector<double> rc;
  int o0 = -p, ratio = 1;
  {
    std::vector<double> r1(R1.W);
    for (int k = 0; k < R1.W; ++k) r1[k] = R1.c[ir * R1.W + k];
    if (hf != 2) {
      rc = r1;
    } else {
      ratio = 2;
      rc.assign(R1.W + q + 1, 0.0);                        // offsets -p .. q + 1 + q
      double binom = 1.0;
      for (int kk = 0; kk <= q + 1; ++kk) {
        const double wgt = binom / double(1 << q);
        for (int k = 0; k < R1.W; ++k) rc[kk + k] += wgt * r1[k];
        binom = binom * double(q + 1 - kk) / double(kk + 1);
      }
    }
  }
  // ---- padded p-grid tables ----
  const int G = 2 * w + p, np = n + 2 * G;
  std::vector<double> K((size_t)np * W, 0.0), M((size_t)np * W, 0.0);
  for (int i = 0; i < np; ++i)
    for (int t = 0; t < W; ++t) {
      const int j = i + t - p;
      if (j < 0 || j >= np) continue;
      K[(size_t)i * W + t] = Kb[rp * W + t];
      M[(size_t)i * W + t] = Mb[rp * W + t];
    }
  std::vector<double> V, lam;
  if (!fd_tables(p, s, np, K, M, V, lam)) return bad("block matrices not SPD");
  ToeP tp{};
  for (int t = 0; t < W; ++t) {
    tp.k[t] = Kb[rp * W + t];
    tp.m[t] = Mb[rp * W + t];
  }
  const int cref = np / 2;
  for (int i = 0; i < s * s; ++i) tp.v[i] = V[(size_t)cref * s * s + i];
  for (int j = 0; j < s; ++j) tp.lam[j] = lam[(size_t)cref * s + j];
  tp.valid = 1;
  // ---- coarse level on the torus ----
  const int nc = hf == 2 ? n / 2 : n, Wq = 2 * q + 1;
  const int nfd = three ? n / 2 : nc;                    // the exactly solved level
  std::vector<double> Vc, lamc;
  if (!periodic_fd_tables(q, nfd, &Kq[rq * Wq], &Mq[rq * Wq], Vc, lamc)) return bad("coarse torus operator");
  if (dim == 3 && hf == 2)                               // rediscretised on 2h: K/2 (x) 2M (x) 2M = 2 (K M M)
    for (double &l : lamc) l *= 2.0;
  // three-grid: the q-level system by one two-grid cycle from 0 -- (q+1)^2-colour GS (A11),
  // residual, knot-insertion restriction P_m^T (A8), exact 2h solve (2D: the rediscretised 2h stencil equals
  // h's, A10), P_m, GS
  QRows qr{};
  for (int t = 0; t < Wq; ++t) {
    qr.k[t] = Kq[rq * Wq + t];
    qr.m[t] = Mq[rq * Wq + t];
  }
  std::vector<double> pm(q + 2);
  {
    double binom = 1.0;
    for (int kk = 0; kk <= q + 1; ++kk) {
      pm[kk] = binom / double(1 << q);
      binom = binom * double(q + 1 - kk) / double(kk + 1);
    }
  }
  // ---- device ----
  cudaStream_t st = nullptr;
  cudaError_t e = cudaSuccess;
  DevBuf buf;
  auto pw = [&](int64_t a) { return dim == 3 ? a * a * a : a * a; };
  const int64_t NP = pw(np), N = pw(n), NC = pw(nc);
  double *dK = buf.get<double>(K.size(), &e), *dM = buf.get<double>(M.size(), &e);
  double *dV = buf.get<double>(V.size(), &e), *dlam = buf.get<double>(lam.size(), &e);
  double *dVc = buf.get<double>(Vc.size(), &e), *dlamc = buf.get<double>(lamc.size(), &e);
  double *drc = buf.get<double>(rc.size(), &e), *dpm = buf.get<double>(pm.size(), &e);
  const int64_t N2 = (int64_t)(n / 2) * (n / 2);
  double *qr2 = buf.get<double>(three ? (int64_t)n * n : 1, &e), *d2 = buf.get<double>(three ? N2 : 1, &e),
         *e2 = buf.get<double>(three ? N2 : 1, &e);
  double *xp = buf.get<double>(NP, &e), *zp = buf.get<double>(NP, &e), *rpad = buf.get<double>(NP, &e);
  double *ec = buf.get<double>(N, &e), *rr = buf.get<double>(N, &e), *tf = buf.get<double>(N, &e);
  double *dc = buf.get<double>(NC, &e), *xc = buf.get<double>(NC, &e), *t1 = buf.get<double>(NC, &e),
         *t2 = buf.get<double>(NC, &e), *tc = buf.get<double>(N, &e), *td = buf.get<double>(N, &e);
  double *dsum = buf.get<double>(2, &e);
  const int nfr = dim == 2 ? export_interior_frags(p, s, np, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr) : -1;
  double *dfb = nfr > 0 ? buf.get<double>(nfr, &e) : nullptr;
  if (e != cudaSuccess) return (*err = "cudaMalloc failed", 6);
  auto up = [&](double *d, const std::vector<double> &h) {
    return cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice);
  };
  if (up(dK, K) || up(dM, M) || up(dV, V) || up(dlam, lam) || up(dVc, Vc) || up(dlamc, lamc) || up(drc, rc) ||
      up(dpm, pm) ||
      cudaMemset(zp, 0, NP * sizeof(double)))
    return (*err = "upload failed", 4);
  if (dfb) export_interior_frags(p, s, np, dK, dM, dV, dlam, dfb, st);
  // ---- seeded mean-zero start ----
  std::vector<double> h0(N);
  uint64_t sst = seed;
  double mean = 0.0;
  for (auto &v : h0) {
    v = 2.0 * (double(splitmix(sst) >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
    mean += v;
  }
  mean /= double(N);
  for (auto &v : h0) v -= mean;
  if (up(ec, h0)) return (*err = "upload failed", 4);
  const int gN = grid_for(N, 256), gNP = grid_for(NP, 256);
  std::vector<double> hist;
  double prev = 0.0;
  for (int it = 0; it <= iters; ++it) {
    // normalise (and project out the constant)
    k_sums<<<1, 1024, 0, st>>>(ec, N, dsum);
    double hs[2];
    if (cudaMemcpy(hs, dsum, sizeof(hs), cudaMemcpyDeviceToHost) != cudaSuccess) return (*err = "sums", 4);
    const double mu = hs[0] / double(N), nrm = std::sqrt(std::max(hs[1] - hs[0] * mu, 0.0));
    if (!(nrm > 0.0) || !std::isfinite(nrm)) return (*err = "power iteration vector vanished or not finite", 2);
    if (it > 0) hist.push_back(nrm / prev);
    if (it == iters) break;
    k_shift_scale<<<gN, 256, 0, st>>>(ec, N, mu, 1.0 / nrm);
    prev = 1.0;
    // x (padded, ghosts) = e
    k_pad<<<gN, 256, 0, st>>>(xp, ec, dim, n, G, 0);
    k_ghost<<<gNP, 256, 0, st>>>(xp, dim, n, G);
    // S_p: colour by colour, ghosts refreshed after each
    const int ncol = dim == 3 ? D * D * D : D * D;
    for (int col = 0; col < ncol; ++col) {
      if (!launch_schwarz_colour_fast(dim, p, s, np, dK, dM, dV, dlam, zp, xp, col, D, st, kFull, dfb, &tp))
        launch_schwarz_colour(dim, p, s, np, dK, dM, dV, dlam, zp, xp, col, D, st, kFull);
      k_ghost<<<gNP, 256, 0, st>>>(xp, dim, n, G);
    }
    // r = 0 - A_p x (real block), d_c = R r, e_c = A_c^+ d_c, e = x + R^T e_c
    int nparts = 0;
    launch_apply(dim, p, np, dK, dM, xp, zp, rpad, nullptr, 1, st, &nparts, kFull, &tp);
    k_pad<<<gN, 256, 0, st>>>(rpad, rr, dim, n, G, 1);
    pband_nd(dim, rr, dc, n, nc, drc, int(rc.size()), o0, ratio, 0, 0, tc, td, st);
    if (!three) {
      launch_coarse_fd(dim, nc, dVc, dlamc, dc, xc, t1, t2, st);
    } else {                                              // xc = B_q dc (one q-level two-grid cycle from 0)
      const int gq = grid_for(NC, 256), st1 = q + 1, h2 = n / 2;
      cudaMemsetAsync(xc, 0, NC * sizeof(double), st);
      for (int col = 0; col < st1 * st1; ++col)
        k_torus_gs<<<gq, 256, 0, st>>>(xc, dc, n, q, qr, col % st1, col / st1);
      k_torus_resid<<<gq, 256, 0, st>>>(qr2, dc, xc, n, q, qr);
      pband_nd(2, qr2, d2, n, h2, dpm, q + 2, 0, 2, 0, 0, tc, td, st);
      launch_coarse_fd(2, h2, dVc, dlamc, d2, e2, t1, t2, st);
      pband_nd(2, e2, xc, h2, n, dpm, q + 2, 0, 2, 1, 1, tc, td, st);
      for (int col = 0; col < st1 * st1; ++col)
        k_torus_gs<<<gq, 256, 0, st>>>(xc, dc, n, q, qr, col % st1, col / st1);
    }
    pband_nd(dim, xc, tf, nc, n, drc, int(rc.size()), o0, ratio, 1, 0, tc, td, st);
    k_pad<<<gN, 256, 0, st>>>(xp, ec, dim, n, G, 1);
    launch_axpy(ec, tf, N, st);
    if ((e = cudaGetLastError()) != cudaSuccess) return (*err = std::string("kernel launch: ") + cudaGetErrorString(e), 4);
  }
  const int tail = std::max(2, int(hist.size()) / 4);
  double lg = 0.0;
  for (int k = int(hist.size()) - tail; k < int(hist.size()); ++k) lg += std::log(hist[k]);
  *rho = std::exp(lg / tail);
  if (ratios)
    for (size_t k = 0; k < hist.size(); ++k) ratios[k] = hist[k];
  return 0;
}

}  // namespace iga2l
