// Phase clocks of one DMMA colour-kernel block (block 0 of the colour) for a 2D config (design tool;
// build with -DIGA2L_TRACE, links the library sources): s2d_trace p m
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../include/iga2l.h"
namespace iga2l { void s2d_trace_read(long long *host8); }
int main(int argc, char **argv) {
  const int p = argc > 1 ? atoi(argv[1]) : 5, m = argc > 2 ? atoi(argv[2]) : 256;
  const int s = p <= 4 ? 3 : (p <= 6 ? 5 : 7);
  iga2l_ctx *c = nullptr;
  if (iga2l_setup(2, p, 1, m, s, s - 1, &c)) { printf("setup: %s\n", iga2l_last_error()); return 1; }
  iga2l_info inf; iga2l_get_info(c, &inf);
  double *b, *x; cudaMalloc(&b, inf.N * 8); cudaMalloc(&x, inf.N * 8);
  cudaMemset(b, 0, inf.N * 8); cudaMemset(x, 0, inf.N * 8);
  for (int rep = 0; rep < 3; ++rep) {
    for (int col = 0; col < 4; ++col) {
      iga2l_sweep(c, b, x, col, col + 1);
      cudaDeviceSynchronize();
      long long t[8];
      iga2l::s2d_trace_read(t);
      if (rep == 2)
        printf("p=%d colour %d: issue %lld  loads %lld  solve %lld (pass x %lld, pass y %lld, FD %lld, update %lld) cycles\n",
               p, col, t[0], t[1], t[2], t[6], t[7], t[3], t[4]);
    }
  }
  return 0;
}
