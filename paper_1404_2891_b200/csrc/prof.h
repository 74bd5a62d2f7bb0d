// prof.h — optional per-kernel-class timing with CUDA events (bench roofline accounting).
// When enabled, every launcher brackets its launch with two events on its stream and records
// the algorithmic flops / bytes of that launch; feast_profile_summary aggregates per class.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace feast {

enum KClass { K_SHIFT = 0, K_PANEL = 1, K_LASWP = 2, K_TRSM = 3, K_ZGEMM = 4, K_PERM = 5, K_ACCUM = 6, K_OTHER = 7,
              K_NCLASS = 8 };

struct ProfRec {
  int cls;
  double flops, bytes;
  cudaEvent_t a, b;
  cudaStream_t s;
  int64_t dev_bytes = -1;   // index of a device byte counter the kernel fills (data-dependent traffic)
};

struct Prof {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  // device counters for kernels whose traffic depends on the data (row swaps: only the rows that
  // actually move); allocated on first use while profiling, read back by feast_profile_summary
  unsigned long long* counters = nullptr;
  int64_t ncounters = 0, counters_used = 0;
  // allocated by feast_profile (outside every event pair: cudaMalloc / cudaMemset synchronise)
  void ensure_counters() {
    if (counters) return;
    ncounters = 1 << 20;
    if (cudaMalloc(&counters, ncounters * sizeof(unsigned long long)) != cudaSuccess) { counters = nullptr; return; }
    cudaMemset(counters, 0, ncounters * sizeof(unsigned long long));
  }
  unsigned long long* counter() {
    if (!counters || counters_used >= ncounters) return nullptr;
    return counters + counters_used++;
  }
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};
Prof& prof();

struct ProfScope {
  bool on;
  ProfRec r;
  cudaStream_t s;
  ProfScope(int cls, double flops, double bytes, cudaStream_t st) : on(prof().on), s(st) {
    if (on) {
      r.cls = cls; r.flops = flops; r.bytes = bytes; r.s = st;
      r.a = prof().get(); r.b = prof().get();
      cudaEventRecord(r.a, s);
    }
  }
  // a device counter of this launch's bytes (the kernel adds to it); nullptr when not profiling
  unsigned long long* bytes_counter() {
    if (!on) return nullptr;
    unsigned long long* c = prof().counter();
    if (c) r.dev_bytes = c - prof().counters;
    return c;
  }
  ~ProfScope() {
    if (on) {
      cudaEventRecord(r.b, s);
      prof().recs.push_back(r);
    }
  }
};

}  // namespace feast
