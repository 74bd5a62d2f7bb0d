// Dependent-latency probe (one warp): DFMA, DMUL, DADD, FFMA, MUFU.RSQ64H-based rsqrt, LDS
// round trip, SHFL, __syncwarp.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double x0, float y0) {
  __shared__ double sm[64];
  double x = x0 + threadIdx.x * 1e-20;
  float y = y0;
  const int N = 1024;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { x = fma(x, 0.999999, 1e-7); x = fma(x, 0.999999, 1e-7); x = fma(x, 0.999999, 1e-7); x = fma(x, 0.999999, 1e-7); }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { y = fmaf(y, 0.999f, 1e-3f); y = fmaf(y, 0.999f, 1e-3f); y = fmaf(y, 0.999f, 1e-3f); y = fmaf(y, 0.999f, 1e-3f); }
  long long t2 = clock64();
  double r = x;
#pragma unroll 1
  for (int i = 0; i < N; ++i) { r = rsqrt(r + 1.0); }
  long long t3 = clock64();
  sm[threadIdx.x] = r;
#pragma unroll 1
  for (int i = 0; i < N; ++i) { int j = ((int)sm[threadIdx.x] & 31); sm[threadIdx.x] = sm[j] + 1.0; }
  long long t4 = clock64();
  double s = sm[threadIdx.x];
#pragma unroll 1
  for (int i = 0; i < N; ++i) { s = __shfl_sync(0xffffffffu, s, (threadIdx.x + 1) & 31) + 1.0; }
  long long t5 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { s += 1.0; __syncwarp(); }
  long long t6 = clock64();
  out[threadIdx.x] = x + y + r + s;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0); cyc[1] = (t2 - t1); cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64 * 8); cudaMallocManaged(&cyc, 8 * 8);
  for (int rep = 0; rep < 2; ++rep) { probe<<<1, 32>>>(out, cyc, 1.0, 1.0f); cudaDeviceSynchronize(); }
  const double N = 1024;
  printf("DFMA dependent latency   %.1f cycles\n", cyc[0] / (4 * N));
  printf("FFMA dependent latency   %.1f cycles\n", cyc[1] / (4 * N));
  printf("rsqrt(double)+DADD chain %.1f cycles\n", cyc[2] / N);
  printf("LDS->DADD->STS->LDS      %.1f cycles\n", cyc[3] / N);
  printf("SHFL+DADD                %.1f cycles\n", cyc[4] / N);
  printf("DADD+__syncwarp          %.1f cycles\n", cyc[5] / N);
  return 0;
}
