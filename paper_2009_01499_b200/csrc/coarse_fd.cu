// Exact second-level solve by Kronecker fast diagonalisation on the FP64
// tensor pipe: strided batched DMMA GEMMs.  See kernels.cuh.
#include "common.cuh"
#include "kernels.cuh"

namespace iga2l {
namespace {

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
__global__ void k_eig_divide(double *__restrict__ T, const double *__restrict__ lam, int n, int dim, int64_t total,
                             int64_t lys) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double den = lam[idx % n] + lam[lys + (idx / n) % n];
    if (dim == 3) den += lam[idx / ((int64_t)n * n)];
    T[idx] = den != 0.0 ? T[idx] / den : 0.0;   // den == 0 only for the constant mode of a torus (pseudo-inverse)
  }
}

}  // namespace

void launch_dgemm(const double *A, const double *B, double *C, int M, int N, int K, int batch, int64_t sAb,
                  int64_t sAm, int64_t sAk, int64_t sBb, int64_t sBk, int64_t sBn, int64_t sCb, int64_t sCm,
                  int64_t sCn, cudaStream_t st) {
  GemmArgs g{A, B, C, M, N, K, sAb, sAm, sAk, sBb, sBk, sBn, sCb, sCm, sCn};
  dim3 grid((unsigned)((N + GBN - 1) / GBN), (unsigned)((M + GBM - 1) / GBM), (unsigned)batch);
  k_dgemm_mma<<<grid, 128, 0, st>>>(g);
}

int launch_coarse_fd(int dim, int n, const double *V, const double *lam, const double *d, double *e, double *t1,
                     double *t2, cudaStream_t st, int ax) {
  const int64_t n1 = n, n2 = n1 * n1, n3 = n2 * n1;
  if (dim == 2) {   // D[y][x]: S = Vy^T D Vx ./ (λx_j + λy_k);  E = Vy S Vx^T
    const double *Vx = V, *Vy = V + (ax ? n2 : 0);
    launch_dgemm(d, Vx, t1, n, n, n, 1, 0, n1, 1, 0, n1, 1, 0, n1, 1, st);     // T1[y][j] = Σ_x D[y][x] Vx[x][j]
    launch_dgemm(Vy, t1, t2, n, n, n, 1, 0, 1, n1, 0, n1, 1, 0, n1, 1, st);    // S[k][j] = Σ_y Vy[y][k] T1[y][j]
    k_eig_divide<<<int(std::min<int64_t>((n2 + 255) / 256, 148 * 16)), 256, 0, st>>>(t2, lam, n, 2, n2, ax ? n1 : 0);
    launch_dgemm(t2, Vx, t1, n, n, n, 1, 0, n1, 1, 0, 1, n1, 0, n1, 1, st);    // T2[k][x] = Σ_j S[k][j] Vx[x][j]
    launch_dgemm(Vy, t1, e, n, n, n, 1, 0, n1, 1, 0, n1, 1, 0, n1, 1, st);     // E[y][x] = Σ_k Vy[y][k] T2[k][x]
    return 5;
  }
  // D[z][y][x]: forward x, y, z with V^T, divide by λ_x + λ_y + λ_z, back z, y, x with V
  launch_dgemm(d, V, t1, int(n2), n, n, 1, 0, n1, 1, 0, n1, 1, 0, n1, 1, st);          // x
  launch_dgemm(V, t1, t2, n, n, n, n, 0, 1, n1, n2, n1, 1, n2, n1, 1, st);             // y (batch z)
  launch_dgemm(V, t2, t1, n, int(n2), n, 1, 0, 1, n1, 0, n2, 1, 0, n2, 1, st);         // z
  k_eig_divide<<<int(std::min<int64_t>((n3 + 255) / 256, 148 * 16)), 256, 0, st>>>(t1, lam, n, 3, n3, 0);
  launch_dgemm(V, t1, t2, n, int(n2), n, 1, 0, n1, 1, 0, n2, 1, 0, n2, 1, st);         // z back
  launch_dgemm(V, t2, t1, n, n, n, n, 0, n1, 1, n2, n1, 1, n2, n1, 1, st);             // y back (batch z)
  launch_dgemm(t1, V, e, int(n2), n, n, 1, 0, n1, 1, 0, 1, n1, 0, n1, 1, st);          // x back
  return 7;
}

}  // namespace iga2l
