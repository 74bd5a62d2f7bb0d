// standalone panel trace harness: random 2048 matrix, one cluster, one panel at k=0
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "kernels.h"
#ifndef NO_TRACE_READ
namespace feast { void panel_trace_read(unsigned long long* out); void panel_ctrace_read(unsigned long long* out); }
#else
namespace feast { inline void panel_trace_read(unsigned long long*) {} inline void panel_ctrace_read(unsigned long long*) {} }
#endif
int main(int argc, char** argv) {
  int W = argc > 1 ? atoi(argv[1]) : 64, CS = argc > 2 ? atoi(argv[2]) : 16;
  int n = argc > 3 ? atoi(argv[3]) : 2048; int64_t ld = n;
  int batch = argc > 4 ? atoi(argv[4]) : 1;
  std::vector<double2> h((size_t)n * n * batch);
  srand(1);
  for (auto& v : h) { v.x = rand() / (double)RAND_MAX - 0.5; v.y = rand() / (double)RAND_MAX - 0.5; }
  double2* d; cudaMalloc(&d, h.size() * 16); cudaMemcpy(d, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  int32_t* ipiv; cudaMalloc(&ipiv, (size_t)n * 4 * batch); double* st; cudaMalloc(&st, 16 * batch);
  int32_t* inf; cudaMalloc(&inf, 4 * batch);
  feast::stats_init_launch(st, inf, batch, 0);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(d, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
    feast::panel_smem_launch(feast::Batched{d, ld, ld * n}, n, 0, W, ipiv, st, inf, batch, CS, 0);
    cudaDeviceSynchronize();
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
#ifdef NO_TRACE_READ
  return 0;
#endif
  unsigned long long t[512];
  feast::panel_trace_read(t);
  auto us = [&](int i) { return (t[i] - t[0]) / 1000.0; };
  printf("start->loaded %.2f us\n", us(1));
  for (int col = 0; col < W; ++col) {
    printf("col %2d: begin %.2f  pushed %.2f  arrived %.2f", col, us(8+4*col), us(9+4*col), us(10+4*col));
    if (col % 8 == 7 && col < 63) printf("   | chunk end wait %.2f -> %.2f, done %.2f", us(300+4*(col/8)), us(301+4*(col/8)), us(302+4*(col/8)));
    if (col % 8 == 7 && col < 63) printf("  solve-done %.2f", us(303+4*(col/8)));
    printf("\n");
  }
  printf("end loop %.2f  end %.2f\n", us(2), us(3));
  unsigned long long ct[2][16];
  feast::panel_ctrace_read(&ct[0][0]);
  const char* nm[16] = {"loop top", "key search", "warp REDUX", "rcp", "stage wrow", "syncthreads",
                        "CTA argmax", "push", "mbar wait", "global pick", "rank-1 update", "chunk store",
                        "U12 push+wait", "U12 solve+sync", "rank-8 update", "final sync"};
  for (int t = 0; t < 2; ++t) {
    printf("thread %s cycles per column:", t ? "96" : "0");
    for (int i = 0; i < 16; ++i) printf(" %s %.0f |", nm[i], ct[t][i] / (double)W);
    printf("\n");
  }
}
