// trtri.cu — inverses of the 64x64 diagonal blocks of L (unit lower) and U (upper) of each
// factored node, so that every triangular solve of the LU (U12 = L11^-1 A12) and of the blocked
// substitutions (Y_k = L_kk^-1 Y_k, Y_k = U_kk^-1 Y_k, and the ^H forms of the left solves,
// P:438-439) becomes an in-place DMMA ZGEMM with M = 64 (tensor pipe instead of a latency-bound
// serial solve).
//
// Recursive doubling in shared memory: invert the eight 8x8 diagonal blocks (one thread per
// column, in registers), then combine
//   lower:  [A 0; B C]^-1 = [A^-1 0; -C^-1 B A^-1  C^-1]
//   upper:  [A B; 0 C]^-1 = [A^-1  -A^-1 B C^-1; 0  C^-1]
// for block sizes 8 -> 16 -> 32 -> 64.  A partial block (nb < 64) is padded with the identity.
#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace feast {
namespace {

constexpr int TT = 256, NB = 64, LDS = NB + 1;

template <bool UPPER, bool UNIT>
__device__ void trtri_block(const double2* __restrict__ T, int64_t ld, int nb, double2* __restrict__ out,
                            double2* S, double2* X, double2* Tmp) {
  const int tid = threadIdx.x;
  // load (padded with identity), keep only the relevant triangle
  for (int idx = tid; idx < NB * NB; idx += TT) {
    const int r = idx % NB, c = idx / NB;
    double2 v = make_double2(0.0, 0.0);
    if (r < nb && c < nb) {
      const bool keep = UPPER ? (r <= c) : (r >= c);
      if (keep) v = T[r + (int64_t)c * ld];
      if (r == c && UNIT) v = make_double2(1.0, 0.0);
    } else if (r == c) {
      v = make_double2(1.0, 0.0);
    }
    S[r * LDS + c] = v;
    X[r * LDS + c] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  // 8x8 diagonal blocks: thread = (block, column)
  if (tid < NB) {
    const int blk = tid >> 3, j = tid & 7, o = blk * 8;
    double2 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    if (!UPPER) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        x[i] = cdiv(x[i], S[(o + i) * LDS + o + i]);
#pragma unroll
        for (int r = i + 1; r < 8; ++r) x[r] = cfms(x[r], S[(o + r) * LDS + o + i], x[i]);
      }
    } else {
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        x[i] = cdiv(x[i], S[(o + i) * LDS + o + i]);
#pragma unroll
        for (int r = 0; r < i; ++r) x[r] = cfms(x[r], S[(o + r) * LDS + o + i], x[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) X[(o + i) * LDS + o + j] = x[i];
  }
  __syncthreads();
  for (int s = 8; s < NB; s *= 2) {
    const int nblk = NB / (2 * s);
    // lower: Tmp = B A^-1   (B = S[o+s.., o..], A^-1 = X[o.., o..])
    // upper: Tmp = B C^-1   (B = S[o.., o+s..], C^-1 = X[o+s.., o+s..])
    for (int idx = tid; idx < nblk * s * s; idx += TT) {
      const int blk = idx / (s * s), e = idx % (s * s), r = e / s, c = e % s, o = blk * 2 * s;
      double2 acc = make_double2(0.0, 0.0);
      if (!UPPER) {
        for (int t = 0; t < s; ++t) acc = cfms(acc, S[(o + s + r) * LDS + o + t], X[(o + t) * LDS + o + c]);
      } else {
        for (int t = 0; t < s; ++t) acc = cfms(acc, S[(o + r) * LDS + o + s + t], X[(o + s + t) * LDS + o + s + c]);
      }
      Tmp[blk * s * s + r * s + c] = acc;   // = -(product)
    }
    __syncthreads();
    // lower: X21 = C^-1 (-B A^-1) ; upper: X12 = A^-1 (-B C^-1)
    for (int idx = tid; idx < nblk * s * s; idx += TT) {
      const int blk = idx / (s * s), e = idx % (s * s), r = e / s, c = e % s, o = blk * 2 * s;
      double2 acc = make_double2(0.0, 0.0);
      if (!UPPER) {
        for (int t = 0; t < s; ++t) acc = cadd(acc, cmul(X[(o + s + r) * LDS + o + s + t], Tmp[blk * s * s + t * s + c]));
        X[(o + s + r) * LDS + o + c] = acc;
      } else {
        for (int t = 0; t < s; ++t) acc = cadd(acc, cmul(X[(o + r) * LDS + o + t], Tmp[blk * s * s + t * s + c]));
        X[(o + r) * LDS + o + s + c] = acc;
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < NB * NB; idx += TT) {
    const int r = idx % NB, c = idx / NB;
    out[r + c * NB] = X[r * LDS + c];
  }
}

// blockIdx.x = node (batch), blockIdx.y = 0 (L^-1) / 1 (U^-1), blockIdx.z = diagonal block index
// relative to kb0.  Source block j at matrix offset (o, o), o = (kb0 + j) * 64.
__global__ void __launch_bounds__(TT) trtri_kernel(Batched Cb, int64_t n, int64_t kb0, double2* __restrict__ inv,
                                                   int64_t inv_node_stride, int which) {
  extern __shared__ __align__(16) double2 sm[];
  double2* S = sm;
  double2* X = sm + NB * LDS;
  double2* Tmp = sm + 2 * NB * LDS;
  const int b = blockIdx.x;
  const int lu = (which == 2) ? (int)blockIdx.y : which;
  const int64_t kb = kb0 + blockIdx.z;
  const int64_t o = kb * NB;
  const int nb = (int)((n - o) < NB ? (n - o) : NB);
  const double2* T = Cb.p + (int64_t)b * Cb.stride + o + o * Cb.ld;
  double2* out = inv + (int64_t)b * inv_node_stride + (kb * 2 + lu) * (int64_t)NB * NB;
  if (lu == 0) trtri_block<false, true>(T, Cb.ld, nb, out, S, X, Tmp);
  else trtri_block<true, false>(T, Cb.ld, nb, out, S, X, Tmp);
}

}  // namespace

void trtri_launch(Batched C, int64_t n, int64_t kb0, int64_t nblocks, double2* inv, int64_t inv_node_stride, int which,
                  int batch, cudaStream_t s) {
  ProfScope ps_(K_TRSM, (double)batch * nblocks * (which == 2 ? 2 : 1) * 8.0 * NB * NB * NB / 3.0, 0.0, s);
  const size_t smem = (size_t)(2 * NB * LDS + NB * NB / 2) * sizeof(double2);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(trtri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  dim3 grid((unsigned)batch, which == 2 ? 2u : 1u, (unsigned)nblocks);
  trtri_kernel<<<grid, TT, smem, s>>>(C, n, kb0, inv, inv_node_stride, which);
  count_launch();
}

}  // namespace feast
