// cluster.sync cost on B200 for cluster sizes 2..16 and 256/1024 threads per CTA (design input for
// the V-cycle tail kernel).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o clusterbench clusterbench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int steps, double *out) {
  cg::cluster_group cl = cg::this_cluster();
  double a = threadIdx.x;
  for (int s = 0; s < steps; ++s) { a = a * 1.0000001 + 1e-9; cl.sync(); }
  if (a == 1234.5) out[0] = a;
}
__global__ void k_syncthreads(int steps, double *out) {
  double a = threadIdx.x;
  for (int s = 0; s < steps; ++s) { a = a * 1.0000001 + 1e-9; __syncthreads(); }
  if (a == 1234.5) out[0] = a;
}
int main() {
  double *d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int steps = 2000;
  for (int th : {256, 1024}) {
    k_syncthreads<<<1, th>>>(10, d);
    cudaEventRecord(e0); k_syncthreads<<<1, th>>>(steps, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("syncthreads  threads %4d: %.1f ns/sync\n", th, ms * 1e6 / steps);
    for (int cs : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(th);
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int s10 = 10;
      if (cudaLaunchKernelEx(&cfg, k_sync, s10, d) != cudaSuccess) { printf("cluster %d launch failed\n", cs); cudaGetLastError(); continue; }
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, k_sync, steps, d);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("cluster %2d threads %4d: %.1f ns/sync\n", cs, th, ms * 1e6 / steps);
    }
  }
  return 0;
}
