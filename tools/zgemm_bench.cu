// zgemm_dmma microbenchmark: TFLOP/s vs (M, N, K, batch), CUDA events, warm L2 excluded by size.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "kernels.h"
int main() {
  struct Cfg { long M, N, K; int batch; int mode; };
  std::vector<Cfg> cfgs = {{1984, 1920, 64, 16, 0}, {1984, 1984, 128, 16, 0}, {1984, 1984, 256, 16, 0},
                           {4096, 4096, 64, 1, 0}, {4096, 4096, 256, 1, 0}, {8192, 8192, 64, 1, 0},
                           {8192, 8192, 512, 1, 0}, {4096, 4096, 4096, 1, 1}, {1984, 128, 64, 16, 0}};
  size_t maxe = 0;
  for (auto& c : cfgs) maxe = std::max(maxe, (size_t)(c.M * c.K + c.K * c.N + c.M * c.N) * c.batch);
  double2* buf; cudaMalloc(&buf, maxe * 16 + 1024);
  cudaMemset(buf, 0, maxe * 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto& c : cfgs) {
    double2* A = buf; double2* B = A + c.M * c.K * c.batch; double2* C = B + c.K * c.N * c.batch;
    feast::ZgemmArgs p{c.M, c.N, c.K, A, c.M, c.M * c.K, B, c.K, c.K * c.N, C, c.M, c.M * c.N,
                       make_double2(1, 0), make_double2(0, 0), c.batch};
    for (int w = 0; w < 2; ++w) feast::zgemm_launch(p, false, c.mode, 0);
    cudaEventRecord(e0);
    int reps = 5;
    for (int r = 0; r < reps; ++r) feast::zgemm_launch(p, false, c.mode, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 8.0 * c.M * c.N * c.K * c.batch * reps;
    printf("M=%5ld N=%5ld K=%5ld b=%2d mode=%d: %.3f ms  %.2f TF/s\n", c.M, c.N, c.K, c.batch, c.mode, ms / reps, fl / (ms * 1e-3) / 1e12);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
