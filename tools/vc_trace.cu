// Phase timestamps of the cluster V-cycle kernel (design/debug tool; links kernels.cu + host_setup).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../include/iga2l.h"
namespace iga2l { void vcycle_trace_enable(unsigned long long *dev_buf); }
int main(int argc, char **argv) {
  int p = argc > 1 ? atoi(argv[1]) : 3;
  iga2l_ctx *c = nullptr;
  if (iga2l_setup(argc > 2 ? atoi(argv[2]) : 2, p, argc > 3 ? atoi(argv[3]) : 1, argc > 4 ? atoi(argv[4]) : 256, p <= 4 ? 3 : (p <= 6 ? 5 : 7), p <= 4 ? 2 : (p <= 6 ? 4 : 6), &c)) { printf("setup: %s\n", iga2l_last_error()); return 1; }
  iga2l_info inf; iga2l_get_info(c, &inf);
  double *dq, *e; cudaMalloc(&dq, inf.Nc * 8); cudaMalloc(&e, inf.Nc * 8); cudaMemset(dq, 0, inf.Nc * 8);
  unsigned long long *tb; cudaMalloc(&tb, 1024 * 8);
  iga2l_coarse_solve(c, dq, e); cudaDeviceSynchronize();
  iga2l::vcycle_trace_enable(tb);
  iga2l_coarse_solve(c, dq, e); cudaDeviceSynchronize();
  std::vector<unsigned long long> h(1024); cudaMemcpy(h.data(), tb, 1024 * 8, cudaMemcpyDeviceToHost);
  int n = 0; while (n < 1023 && h[n + 1] > h[n]) ++n;
  printf("phases %d total %llu cycles (%.2f us at 1.965 GHz)\n", n, h[n] - h[0], (h[n] - h[0]) / 1965.0);
  for (int i = 1; i <= n; ++i) printf("%d:%llu ", i, h[i] - h[i - 1]);
  printf("\n");
  return 0;
}
