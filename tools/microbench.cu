// Microbenchmarks that size the design (not product code): FP64 DFMA and DMMA peak, and the
// per-step synchronisation cost options for a latency-bound multicolour sweep on B200:
//   (a) kernel boundaries replayed from a CUDA graph, (b) the same with programmatic dependent
//   launch (PDL), (c) grid-wide barriers inside one cooperative persistent kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

__global__ void k_dfma(double *out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.0) out[0] = a0;
}

__global__ void k_dmma(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double d[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[k][0]), "+d"(d[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_work(double *x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 1.0000001 + 1e-9;
}

__global__ void k_work_pdl(double *x, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 1.0000001 + 1e-9;
  asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void k_persistent(double *x, int n, int steps) {
  cg::grid_group g = cg::this_grid();
  for (int s = 0; s < steps; ++s) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      x[i] = x[i] * 1.0000001 + 1e-9;
    g.sync();
  }
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d L2 %d MB smem/block optin %zu KB clock %d MHz\n", prop.name, prop.multiProcessorCount,
         prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin >> 10, prop.clockRate / 1000);
  const int sms = prop.multiProcessorCount;
  double *d;
  CK(cudaMalloc(&d, 1 << 26));
  CK(cudaMemset(d, 0, 1 << 26));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  float ms;
  // ---- FP64 peaks ----
  for (int occ : {4, 8}) {
    int iters = 4096, threads = 256, blocks = sms * occ;
    k_dfma<<<blocks, threads, 0, st>>>(d, 16);
    cudaEventRecord(e0, st);
    k_dfma<<<blocks, threads, 0, st>>>(d, iters);
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * double(threads) * blocks;
    printf("DFMA  occ %d: %.2f TFLOP/s\n", occ, flops / ms / 1e9);
    k_dmma<<<blocks, threads, 0, st>>>(d, 16);
    cudaEventRecord(e0, st);
    k_dmma<<<blocks, threads, 0, st>>>(d, iters);
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 4 * iters * double(threads / 32) * blocks;
    printf("DMMA  occ %d: %.2f TFLOP/s\n", occ, flops / ms / 1e9);
  }
  // ---- per-step sync costs ----
  const int STEPS = 200;
  for (int grid : {sms, sms * 4, sms * 16}) {
    const int n = grid * 128;
    // (a) graph of plain launches
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int s = 0; s < STEPS; ++s) k_work<<<grid, 128, 0, st>>>(d, n);
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphLaunch(ge, st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid %5d: graph launch   %.3f us/step\n", grid, ms * 1e3 / (5 * STEPS));
    // (b) graph with PDL edges
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int s = 0; s < STEPS; ++s) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = 128;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, k_work_pdl, d, n));
    }
    CK(cudaStreamEndCapture(st, &g2));
    CK(cudaGraphInstantiate(&ge2, g2, 0));
    cudaGraphLaunch(ge2, st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge2, st);
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid %5d: graph + PDL    %.3f us/step\n", grid, ms * 1e3 / (5 * STEPS));
    // (c) cooperative persistent kernel with grid.sync per step
    int maxb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_persistent, 128, 0);
    if (grid <= maxb * sms) {
      int steps = STEPS;
      void *args[] = {&d, (void *)&n, &steps};
      CK(cudaLaunchCooperativeKernel((void *)k_persistent, grid, 128, args, 0, st));
      cudaEventRecord(e0, st);
      CK(cudaLaunchCooperativeKernel((void *)k_persistent, grid, 128, args, 0, st));
      cudaEventRecord(e1, st);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %5d: grid.sync      %.3f us/step\n", grid, ms * 1e3 / STEPS);
    }
  }
  return 0;
}
