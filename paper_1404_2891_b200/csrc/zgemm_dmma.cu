// zgemm_dmma.cu — batched complex128 GEMM on the FP64 tensor pipe (DMMA) for sm_100a.
//
// The one dense contraction of the hot path: the LU trailing
// update A22 -= L21 U12, the blocked-substitution updates, R = B X and Q^H (A Q).
// tcgen05 has no f64 kind on sm_100a, so the tensor-core path for FP64 is mma.sync
// m8n8k4.f64 (SASS DMMA.8x8x4), measured at 37.17 TF/s peak on B200 (profiles/r01_fp64_peak.md).
//
// Complex product by real embedding: with C' the m x 2n real matrix of interleaved (re,im)
// columns and A' the m x 2k real matrix of interleaved A, C' = A' * Bh where Bh (2k x 2n) is
// the real 2x2-block embedding of B: [Bre Bim; -Bim Bre] per complex entry.  One DMMA
// (8x8x4 real) is then an 8(row) x 4(complex col) x 2(complex k) complex update with no
// wasted multiplies: 8 m n k real flops per complex GEMM, the LAPACK ZGEMM count.
// Fragment layout (PTX m8n8k4 .f64): lane = 4 g + t;  A[g][t], B[t][g], C[g][2t..2t+1].
//  - A' fragment: complex A[g][k = t>>1], part t&1          (conj(A): negate part 1)
//  - Bh fragment: complex B[k = t>>1][j = g>>1], part (t&1)^(g&1), negated iff t&1 && !(g&1)
//  - C' fragment: complex C[g][j = t] (re, im) — each thread owns whole complex outputs.
// Sign flips are an XOR on the high word (integer pipe), so the FP64 pipe only runs DMMA.
// C -= A B (mode SUB) folds the minus sign into the same XOR mask.
//
// Tiling: CTA 64x64 complex outputs, 4 warps of 32x32, BK = 16 complex per stage,
// 3-stage cp.async pipeline (108 KB smem -> 2 CTAs/SM).  Padded smem strides make every
// fragment load bank-conflict free (A: ld 68 complex, B: ld 18 complex).
#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace feast {
namespace {

constexpr int BK = 16, STAGES = 3;
constexpr int LDB_S = BK + 2;   // Bs[n][k]
template <int BM, int BN>
struct Tile {
  static constexpr int THREADS = 32 * (BM / 32) * (BN / 32);
  static constexpr int LDA_S = BM + 4;   // As[k][m]
  static constexpr int A_STAGE = BK * LDA_S;
  static constexpr int B_STAGE = BN * LDB_S;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double2);
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double xor_sign(double v, unsigned long long m) {
  return __longlong_as_double(__double_as_longlong(v) ^ m);
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, bool CONJA, int MODE>
__global__ void __launch_bounds__(Tile<BM, BN>::THREADS, 2) zgemm_dmma_kernel(ZgemmArgs p) {
  constexpr int THREADS = Tile<BM, BN>::THREADS, LDA_S = Tile<BM, BN>::LDA_S;
  constexpr int A_STAGE = Tile<BM, BN>::A_STAGE, B_STAGE = Tile<BM, BN>::B_STAGE;
  constexpr int WN = BN / 32;   // warps along N
  extern __shared__ __align__(128) double2 smem[];
  double2* As = smem;
  double2* Bs = smem + STAGES * A_STAGE;

  const int64_t z = blockIdx.z;
  const double2* __restrict__ A = p.A + z * p.sA;
  const double2* __restrict__ B = p.B + z * p.sB;
  double2* __restrict__ C = p.C + z * p.sC;
  const int64_t M = p.M, N = p.N, K = p.K;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = (warp / WN) * 32, wn = (warp % WN) * 32;
  const int g = lane >> 2, t = lane & 3;

  auto load_tile = [&](int stage, int64_t kt) {
    const int64_t k0 = kt * BK;
    double2* as = As + stage * A_STAGE;
    double2* bs = Bs + stage * B_STAGE;
#pragma unroll
    for (int i = 0; i < (BM * BK) / THREADS; ++i) {
      const int idx = tid + i * THREADS;
      int m, k;
      if (!CONJA) { m = idx & (BM - 1); k = idx / BM; }   // A[m][k] at m + k lda
      else { k = idx & (BK - 1); m = idx / BK; }          // Ag[k][m] at k + m lda
      const int64_t gm = m0 + m, gk = k0 + k;
      const bool pred = gm < M && gk < K;
      const double2* src = pred ? (CONJA ? A + gk + gm * p.lda : A + gm + gk * p.lda) : A;
      cp_async16(&as[k * LDA_S + m], src, pred);
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / THREADS; ++i) {
      const int idx = tid + i * THREADS;
      const int k = idx & (BK - 1), n = idx / BK;
      const int64_t gn = n0 + n, gk = k0 + k;
      const bool pred = gn < N && gk < K;
      const double2* src = pred ? B + gk + gn * p.ldb : B;
      cp_async16(&bs[n * LDB_S + k], src, pred);
    }
  };

  const int64_t KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tile(s, s);
    cp_commit();
  }

  double acc[4][8][2];
  if (MODE == ZG_SUB) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 8; ++ni) {
        const int64_t r = m0 + wm + mi * 8 + g, c = n0 + wn + ni * 4 + t;
        double2 v = make_double2(0.0, 0.0);
        if (r < M && c < N) v = C[r + c * p.ldc];
        acc[mi][ni][0] = v.x;
        acc[mi][ni][1] = v.y;
      }
  } else {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 8; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  }

  const unsigned long long SIGN = 0x8000000000000000ULL;
  const unsigned long long signA = (CONJA && (t & 1)) ? SIGN : 0ULL;
  bool negB = (t & 1) && !(g & 1);
  if (MODE == ZG_SUB) negB = !negB;
  const unsigned long long signB = negB ? SIGN : 0ULL;
  const int partA = t & 1;
  const int partB = (t & 1) ^ (g & 1);
  const int kA = t >> 1;

  for (int64_t kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + STAGES - 1;
      if (nk < KT) load_tile((int)(nk % STAGES), nk);
      cp_commit();
    }
    const double* as = reinterpret_cast<const double*>(As + (kt % STAGES) * A_STAGE);
    const double* bs = reinterpret_cast<const double*>(Bs + (kt % STAGES) * B_STAGE);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 2) {
      double af[4], bf[8];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
        af[mi] = xor_sign(as[2 * ((kk + kA) * LDA_S + wm + mi * 8 + g) + partA], signA);
#pragma unroll
      for (int ni = 0; ni < 8; ++ni)
        bf[ni] = xor_sign(bs[2 * ((wn + ni * 4 + (g >> 1)) * LDB_S + kk + kA) + partB], signB);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 8; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  cp_wait<0>();

  // epilogue
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 8; ++ni) {
      const int64_t r = m0 + wm + mi * 8 + g, c = n0 + wn + ni * 4 + t;
      if (r < M && c < N) {
        double2 v = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
        if (MODE == ZG_GEN) {
          v = cmul(p.alpha, v);
          if (p.beta.x != 0.0 || p.beta.y != 0.0) v = cadd(v, cmul(p.beta, C[r + c * p.ldc]));
        }
        C[r + c * p.ldc] = v;
      }
    }
}

template <int BM, int BN, bool CONJA, int MODE>
void launch_tile(const ZgemmArgs& p, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(zgemm_dmma_kernel<BM, BN, CONJA, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Tile<BM, BN>::SMEM_BYTES);
    configured = true;
  }
  dim3 grid((unsigned)((p.N + BN - 1) / BN), (unsigned)((p.M + BM - 1) / BM), (unsigned)p.batch);
  zgemm_dmma_kernel<BM, BN, CONJA, MODE><<<grid, Tile<BM, BN>::THREADS, Tile<BM, BN>::SMEM_BYTES, s>>>(p);
  count_launch();
}

// Tile choice: 64x64 CTAs (4 warps) normally; 32x32 CTAs (1 warp) when the 64x64 grid would not
// fill the 148 SMs twice over (small, latency-bound launches: diagonal-block applications,
// in-block updates, the substitution updates of late blocks).
template <bool CONJA, int MODE>
void launch_t(const ZgemmArgs& p, cudaStream_t s) {
  ProfScope ps_(K_ZGEMM, 8.0 * (double)p.M * (double)p.N * (double)p.K * p.batch, 0.0, s);
  const int64_t big = ((p.M + 63) / 64) * ((p.N + 63) / 64) * p.batch;
  if (p.inplace) {   // every CTA must read its whole B column block before writing it: BM >= M
    if (big < 296) launch_tile<64, 32, CONJA, MODE>(p, s);
    else launch_tile<64, 64, CONJA, MODE>(p, s);
  } else if (big < 296) {
    launch_tile<32, 32, CONJA, MODE>(p, s);
  } else {
    launch_tile<64, 64, CONJA, MODE>(p, s);
  }
}

}  // namespace

void zgemm_launch(const ZgemmArgs& p, bool conjA, int mode, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return;
  if (p.K <= 0) {
    if (mode == ZG_SUB) return;  // C -= 0
  }
  if (conjA) {
    if (mode == ZG_SUB) launch_t<true, ZG_SUB>(p, s); else launch_t<true, ZG_GEN>(p, s);
  } else {
    if (mode == ZG_SUB) launch_t<false, ZG_SUB>(p, s); else launch_t<false, ZG_GEN>(p, s);
  }
}

}  // namespace feast
