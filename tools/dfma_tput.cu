// FP64 FMA issue throughput on one SM vs warps per CTA (independent chains).
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void tput(double* out, long long* cyc, int iters) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-9 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = fma(x[c], 0.9999999, 1e-9);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 8);
  const int iters = 4096;
  for (int th : {32, 128, 256, 512, 1024}) {
    tput<16><<<1, th>>>(out, cyc, iters); cudaDeviceSynchronize();
    tput<16><<<1, th>>>(out, cyc, iters); cudaDeviceSynchronize();
    double dfma = (double)th * iters * 16;
    printf("threads %4d: %.1f DFMA/clk/SM (%.2f cycles per warp-DFMA per SMSP)\n", th, dfma / cyc[0],
           cyc[0] / (dfma / 32 / 4 > 0 ? dfma / 32 / (th >= 128 ? 4 : th / 32) : 1));
  }
  return 0;
}
