// Shared device helpers of libiga2l's kernels (sm_100a, fp64).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cuda_runtime.h>

namespace iga2l {

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block reduction (fixed tree); result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double *scratch) {
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

// mma.sync.m8n8k4.f64 (DMMA, the FP64 tensor pipe): A 8x4 row-major, B 4x8 column-major, C 8x8;
// per lane a = A[l/4][l%4], b = B[l%4][l/4], c[i] = C[l/4][2(l%4)+i]
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <typename F>
inline void ensure_smem(F *kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

inline int grid_for(int64_t total, int bs) {
  int64_t g = (total + bs - 1) / bs;
  return int(std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 32));
}

}  // namespace iga2l
