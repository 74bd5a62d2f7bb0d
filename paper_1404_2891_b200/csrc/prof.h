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
};

struct Prof {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
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
  ~ProfScope() {
    if (on) {
      cudaEventRecord(r.b, s);
      prof().recs.push_back(r);
    }
  }
};

}  // namespace feast
