// Phase clocks of block 0 of a 3D Schwarz colour launch (k_schwarz3d_t; -DIGA2L_TRACE): s3d_trace p m
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../include/iga2l.h"
namespace iga2l { void s2d_trace_read(long long *host8); }
int main(int argc, char **argv) {
  const int p = argc > 1 ? atoi(argv[1]) : 3, m = argc > 2 ? atoi(argv[2]) : 128;
  const int s = p <= 4 ? 3 : (p <= 6 ? 5 : 7);
  iga2l_ctx *c = nullptr;
  if (iga2l_setup(3, p, p >= 5 ? 2 : 1, m, s, s - 1, &c)) { printf("setup: %s\n", iga2l_last_error()); return 1; }
  iga2l_info inf; iga2l_get_info(c, &inf);
  double *b, *x; cudaMalloc(&b, inf.N * 8); cudaMalloc(&x, inf.N * 8);
  cudaMemset(b, 0, inf.N * 8); cudaMemset(x, 0, inf.N * 8);
  for (int rep = 0; rep < 3; ++rep)
    for (int col = 0; col < 3; ++col) {
      iga2l_sweep(c, b, x, col, col + 1);
      cudaDeviceSynchronize();
      long long t[8];
      iga2l::s2d_trace_read(t);
      if (rep == 2)
        printf("p=%d colour %d: loads %lld, pass x %lld, pass y %lld, pass z %lld, FD+update %lld cycles\n", p, col,
               t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[5] - t[4]);
    }
  return 0;
}
