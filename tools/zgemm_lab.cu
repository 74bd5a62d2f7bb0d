// zgemm_lab: the library's DMMA ZGEMM tile variants vs cuBLAS ZGEMM at the shapes of the hot
// path (trailing updates of the batched LU, substitution updates, large square), CUDA events,
// plus a max-error check of every variant against cuBLAS on random data.
//   zgemm_lab                  all configs x variants
//   zgemm_lab <cfg> <variant>  one config, one variant (-1 = cuBLAS), two launches (for ncu)
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.h"

__global__ void fill(double2* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995; x ^= x >> 15;
    unsigned y = x * 1103515245u + 12345u;
    p[i] = make_double2((x & 0xffff) / 65536.0 - 0.5, (y & 0xffff) / 65536.0 - 0.5);
  }
}

int main(int argc, char** argv) {
  struct Cfg { long M, N, K; int batch; int mode; bool conj; };
  std::vector<Cfg> cfgs = {{1792, 1792, 256, 16, 0, false}, {1792, 128, 256, 16, 0, false},
                           {1984, 1984, 64, 16, 0, false},  {4096, 4096, 256, 4, 0, false},
                           {8192, 8192, 256, 1, 0, false},  {4096, 4096, 4096, 1, 1, false},
                           {1920, 128, 128, 16, 0, false},  {2048, 128, 2048, 1, 1, true},
                           {64, 1920, 64, 16, 1, false},    {448, 128, 64, 16, 0, true},
                           // the LU's short-K updates of one 4-node group (C2): in-block (K = 32,
                           // 64) and the outer block's per-64-block sub-updates (M < 256)
                           {1984, 32, 32, 4, 0, false},    {1920, 192, 64, 4, 0, false},
                           {192, 1792, 64, 4, 0, false},   {1536, 1664, 256, 4, 0, false},
                           // C4's early trailing update (n = 16384, outer block 512; 2 of a group's nodes):
                           // for single-config ncu captures only (too large for the host-side check)
                           {16000, 16384, 512, 2, 0, false}};
  std::vector<int> variants = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9};
  int only_cfg = -2, only_var = -2;
  if (argc > 2) { only_cfg = atoi(argv[1]); only_var = atoi(argv[2]); }
  size_t maxe = 0;
  for (auto& c : cfgs) maxe = std::max(maxe, (size_t)(c.M * c.K + c.K * c.N + c.M * c.N) * c.batch);
  double2 *buf, *C0, *Cref;
  cudaMalloc(&buf, maxe * 16 + 1024);
  size_t maxc = 0;
  for (auto& c : cfgs) maxc = std::max(maxc, (size_t)c.M * c.N * c.batch);
  cudaMalloc(&C0, maxc * 16);
  cudaMalloc(&Cref, maxc * 16);
  fill<<<1024, 256>>>(buf, maxe, 1234u);
  cublasHandle_t hb;
  cublasCreate(&hb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<double2> h1, h2;
  for (size_t i = 0; i < cfgs.size(); ++i) {
    if (only_cfg >= 0 && (int)i != only_cfg) continue;
    const Cfg& c = cfgs[i];
    double2* A = buf;
    double2* B = A + c.M * c.K * c.batch;
    double2* C = B + c.K * c.N * c.batch;
    const long lda = c.conj ? c.K : c.M;
    const long sA = c.M * c.K;
    feast::ZgemmArgs p{c.M, c.N, c.K, A, lda, sA, B, c.K, c.K * c.N, C, c.M, c.M * c.N,
                       make_double2(1, 0), make_double2(0, 0), c.batch};
    const cuDoubleComplex one = make_cuDoubleComplex(1, 0), mone = make_cuDoubleComplex(-1, 0),
                          zero = make_cuDoubleComplex(0, 0);
    const size_t cn = (size_t)c.M * c.N * c.batch;
    cudaMemcpy(C0, C, cn * 16, cudaMemcpyDeviceToDevice);
    auto blas = [&](double2* Cout) {
      cublasZgemmStridedBatched(hb, c.conj ? CUBLAS_OP_C : CUBLAS_OP_N, CUBLAS_OP_N, c.M, c.N, c.K,
                                c.mode == 0 ? &mone : &one, (cuDoubleComplex*)A, lda, sA, (cuDoubleComplex*)B, c.K,
                                c.K * c.N, c.mode == 0 ? &one : &zero, (cuDoubleComplex*)Cout, c.M, c.M * c.N, c.batch);
    };
    if (only_cfg >= 0) {
      for (int r = 0; r < 2; ++r) {
        if (only_var < 0) blas(C);
        else feast::zgemm_launch_variant(p, c.conj, c.mode, only_var, 0);
      }
      continue;
    }
    if (cn > (size_t)1 << 28) continue;   // single-config (ncu) shapes only
    h1.resize(cn);
    h2.resize(cn);
    // reference once
    cudaMemcpy(Cref, C0, cn * 16, cudaMemcpyDeviceToDevice);
    blas(Cref);
    cudaMemcpy(h1.data(), Cref, cn * 16, cudaMemcpyDeviceToHost);
    const double fl = 8.0 * c.M * c.N * c.K * c.batch;
    for (int v : variants) {
      cudaMemcpy(C, C0, cn * 16, cudaMemcpyDeviceToDevice);
      feast::zgemm_launch_variant(p, c.conj, c.mode, v, 0);
      cudaMemcpy(h2.data(), C, cn * 16, cudaMemcpyDeviceToHost);
      double err = 0, ref = 0;
      for (size_t e = 0; e < cn; ++e) {
        err = std::max(err, std::fabs(h1[e].x - h2[e].x) + std::fabs(h1[e].y - h2[e].y));
        ref = std::max(ref, std::fabs(h1[e].x) + std::fabs(h1[e].y));
      }
      const int reps = 10;
      for (int w = 0; w < 2; ++w) feast::zgemm_launch_variant(p, c.conj, c.mode, v, 0);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) feast::zgemm_launch_variant(p, c.conj, c.mode, v, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("[%zu] v%-2d M=%5ld N=%5ld K=%5ld b=%2d %s%s: %8.3f ms %6.2f TF/s  relerr %.1e\n", i, v, c.M, c.N, c.K,
             c.batch, c.mode ? "GEN" : "SUB", c.conj ? " conj" : "", ms / reps, fl * reps / (ms * 1e-3) / 1e12,
             err / ref);
    }
    {
      const int reps = 10;
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) blas(C);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("[%zu] cuBLAS                                         : %8.3f ms %6.2f TF/s\n", i, ms / reps,
             fl * reps / (ms * 1e-3) / 1e12);
    }
    fflush(stdout);
  }
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
