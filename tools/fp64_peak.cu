// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Output: TFLOP/s per variant, with CUDA-event timing. Used to fill the FP64 roofline
// denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\"}\n", p.name, p.multiProcessorCount, p.major, p.minor);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16}) {
    for (int blocks_per_sm : {1, 2}) {
      int iters = 20000;
      dim3 grid(sms * blocks_per_sm), block(32 * warps);
      dmma_kernel<8><<<grid, block>>>(d, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) dmma_kernel<8><<<grid, block>>>(d, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 5.0 * grid.x * warps * (double)iters * 8 * 512;
      printf("{\"kind\":\"dmma_m8n8k4\",\"warps\":%d,\"bps\":%d,\"tflops\":%.3f}\n", warps, blocks_per_sm, flops / (ms * 1e-3) / 1e12);
      dfma_kernel<8><<<grid, block>>>(d, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) dfma_kernel<8><<<grid, block>>>(d, iters * 4);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 5.0 * grid.x * warps * 32.0 * (double)iters * 4 * 8 * 2;
      printf("{\"kind\":\"dfma\",\"warps\":%d,\"bps\":%d,\"tflops\":%.3f}\n", warps, blocks_per_sm, flops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
