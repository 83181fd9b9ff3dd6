// Probe of 1D TMA row loads (cp.async.bulk.tensor.1d) with mbarrier completion: box sizes, negative /
// out-of-range coordinates, destination offsets.  nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe
// tools/tma_probe.cu (links libcuda through the runtime entry point).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned su32(const void *p) { return unsigned(__cvta_generic_to_shared(p)); }

__global__ void k_probe(const __grid_constant__ CUtensorMap map, int c0, int box, int dst_off, double *out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(box * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                 ::"r"(su32(sm + dst_off)), "l"(&map), "r"(c0), "r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
  for (int i = threadIdx.x; i < box; i += blockDim.x) out[i] = sm[dst_off + i];
}

__global__ void k_probe_swz(const __grid_constant__ CUtensorMap map, int c0, double *out) {
  extern __shared__ __align__(1024) double smz[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(10 * 16 * 8) : "memory");
  }
  __syncthreads();
  if (threadIdx.x < 10)   // rows r = 0..9 at smem offsets 16 r doubles (128-byte aligned, NOT 1024)
    asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                 ::"r"(su32(smz + 16 * (threadIdx.x + 1))), "l"(&map), "r"(c0 + 32 * int(threadIdx.x)), "r"(su32(&bar)) : "memory");
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 16 * 11; i += blockDim.x) out[i] = smz[i];
}

int main(int argc, char **argv) {
  if (argc > 1 && argv[1][0] == 's') {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const int n = 1024;
    std::vector<double> h(n);
    for (int i = 0; i < n; ++i) h[i] = i;
    double *d, *o;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&o, 4096 * 8);
    cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[1] = {cuuint64_t(n)}, str[1] = {0};
    cuuint32_t bx[1] = {16}, es[1] = {1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemset(o, 0, 4096 * 8);
    k_probe_swz<<<1, 64, 8192>>>(map, 64, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> g(16 * 11);
    cudaMemcpy(g.data(), o, g.size() * 8, cudaMemcpyDeviceToHost);
    printf("swizzle probe: encode %d kernel %s\n", int(r), cudaGetErrorString(e));
    for (int row = 1; row <= 10; ++row) {
      printf("row %2d:", row);
      for (int c = 0; c < 16; ++c) printf(" %4d", int(g[16 * row + c]));
      printf("\n");
    }
    return 0;
  }
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int n = 225;
  std::vector<double> h(n);
  for (int i = 0; i < n; ++i) h[i] = i + 1;
  double *d, *o;
  cudaMalloc(&d, n * 8);
  cudaMalloc(&o, 4096 * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  struct Case { int box, c0, off; } cases[] = {{68, 0, 0}, {66, 0, 0}, {70, 0, 0}, {66, -1, 0}, {66, 200, 0}, {68, -2, 0},
                                               {66, 0, 80}, {64, 0, 0}, {66, 10, 16}, {80, 0, 0}, {70, -3, 0}, {66, 11, 0}, {66, 13, 16}, {64, 7, 0}, {10, 20, 2}, {16, 40, 18}, {10, 4, 10}};
  const int pick = argc > 1 ? atoi(argv[1]) : -1;
  int ci = -1;
  for (auto &c : cases) {
    if (++ci != pick && pick >= 0) continue;
    CUtensorMap map;
    cuuint64_t dims[1] = {cuuint64_t(n)}, str[1] = {0};
    cuuint32_t bx[1] = {cuuint32_t(c.box)}, es[1] = {1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemset(o, 0, 4096 * 8);
    k_probe<<<1, 64, 16384>>>(map, c.c0, c.box, c.off, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> g(c.box);
    cudaMemcpy(g.data(), o, c.box * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < c.box; ++i) {
      const int idx = c.c0 + i;
      const double want = (idx >= 0 && idx < n) ? h[idx] : 0.0;
      bad += g[i] != want;
    }
    printf("box %3d c0 %4d off %3d: encode %d, kernel %s, mismatches %d\n", c.box, c.c0, c.off, int(r),
           cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
