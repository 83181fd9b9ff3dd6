// DMMA (mma.sync m8n8k4 f64) latency and per-warp issue rate: one warp, chains of dependent MMAs,
// and 1/2/4/8 independent chains interleaved (clock64).  Design tool.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int C>
__global__ void k(double *out, long long *cyc, int n) {
  double d0[C], d1[C];
  for (int c = 0; c < C; ++c) { d0[c] = threadIdx.x; d1[c] = 1.0; }
  const double a = 1.0000001, b = 0.9999999;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < C; ++c) dmma(d0[c], d1[c], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < C; ++c) s += d0[c] + d1[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void kshfl(double *out, long long *cyc, int n) {
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31) * 1.0000001;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double *o; long long *c, h; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  const int n = 1000;
  auto run = [&](auto kern, int chains) {
    kern<<<1, 32>>>(o, c, n); cudaDeviceSynchronize();
    kern<<<1, 32>>>(o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("chains %d: %.1f cycles per DMMA step (%.1f per DMMA)\n", chains, double(h) / n, double(h) / n / chains);
  };
  run(k<1>, 1); run(k<2>, 2); run(k<4>, 4); run(k<8>, 8);
  kshfl<<<1, 32>>>(o, c, n); cudaDeviceSynchronize(); kshfl<<<1, 32>>>(o, c, n);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("shfl + dmul chain: %.1f cycles per step\n", double(h) / n);
  return 0;
}
