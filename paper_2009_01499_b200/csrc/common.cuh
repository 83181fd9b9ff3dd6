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

// ---- TMA (cp.async.bulk.tensor) + mbarrier ------------------------------------------------------
// Vectors are addressed through 1D tensor maps (element-granular coordinates, so rows of any length n1
// -- odd n1 makes 2D/3D maps impossible: their strides must be multiples of 16 bytes); coordinates
// outside [0, N) are zero-filled by the hardware.  Destination rows in shared memory are 128-byte aligned.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// count doubles from element c0 of the vector behind `map` -> dst (box = the map's box size)
__device__ __forceinline__ void tma_load_1d(double *dst, const void *map, int c0, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(smem_u32(bar))
      : "memory");
}

// 2D box load: element (c0, c1) of the box origin (c0 = column, c1 = row)
__device__ __forceinline__ void tma_load_2d(double *dst, const void *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// host: 1D tensor map over n doubles at ptr with a box of `box` elements (box * 8 % 16 == 0, box <= 256).
// Returns false if the driver entry point is missing or the encode fails.
bool make_tmap_1d(void *map64, const double *ptr, int64_t n, int box);
// the same with 128-byte swizzle (box * 8 <= 128): chunk c of a row landing at a 128-byte aligned shared
// address A goes to chunk c ^ ((A >> 7) & 7)
bool make_tmap_1d_swz128(void *map64, const double *ptr, int64_t n, int box);
// 2D map of `rows` rows of `cols` doubles, consecutive rows `stride` elements apart (stride * 8 % 16 == 0),
// box = box_cols x box_rows, 128B swizzle
bool make_tmap_rows_swz128(void *map64, const double *ptr, int64_t cols, int64_t rows, int64_t stride, int box_cols,
                           int box_rows);

template <typename F>
inline void ensure_smem(F *kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

inline int grid_for(int64_t total, int bs) {
  int64_t g = (total + bs - 1) / bs;
  return int(std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 32));
}

}  // namespace iga2l
