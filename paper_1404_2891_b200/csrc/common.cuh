// common.cuh — shared device/host helpers of the B200 FEAST library (product path only).
// Complex numbers are double2 (x = re, y = im): the bytes of cuDoubleComplex/torch.complex128.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#define FEAST_DEV __device__ __forceinline__

FEAST_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
FEAST_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
FEAST_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
FEAST_DEV double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// a - b*c
FEAST_DEV double2 cfms(double2 a, double2 b, double2 c) {
  return make_double2(fma(-b.x, c.x, fma(b.y, c.y, a.x)), fma(-b.x, c.y, fma(-b.y, c.x, a.y)));
}
FEAST_DEV double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
// 1/b (Smith)
FEAST_DEV double2 crcp(double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2(1.0 / d, -r / d);
  } else {
    double r = b.x / b.y, d = b.x * r + b.y;
    return make_double2(r / d, -1.0 / d);
  }
}
FEAST_DEV double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    double r = b.x / b.y, d = b.x * r + b.y;
    return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}

// Launch-count accounting (bench "gpu_launches"): every launcher bumps this counter.
namespace feast {
extern thread_local int64_t g_launches;
// Kernel attributes (dynamic smem size, non-portable clusters) belong to the CURRENT device: a
// launcher configures its kernel once per device.  Returns true the first time it is called for
// the current device with this mask (thread-safe; a race only repeats the idempotent setting).
inline bool first_use_on_device(std::atomic<uint64_t>& mask) {
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  return !(mask.fetch_or(bit) & bit);
}
inline void count_launch(int k = 1) { g_launches += k; }
}  // namespace feast
