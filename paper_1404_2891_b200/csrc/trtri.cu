// trtri.cu — the small triangular pieces of the blocked LU:
//   * trsm:  op(T) X = X in place for an nb x nb diagonal block T (nb <= 64) and nb x ncols X —
//            the in-block U12 = L11^-1 A12 of the 64-column blocks;
//   * trtri: the inverses of the 64x64 diagonal blocks of L (unit lower) and U (upper) of each
//            factored node, so that every other triangular solve of the LU (the outer
//            U12 = L11^-1 A12) and of the blocked substitutions (Y_k = L_kk^-1 Y_k,
//            Y_k = U_kk^-1 Y_k and the ^H forms of the left solves) becomes an
//            in-place DMMA ZGEMM with M = 64 on the tensor pipe.
//
// Both are latency-bound chains of nb dependent steps, so the design minimises the latency of one
// step: one WARP per right-hand-side column (columns of X, or of the identity for trtri), lane l
// holding rows l and l + 32 in registers; T sits in shared memory.  Step t of a forward solve:
// x_t is broadcast from its owner lane by shuffle (scaled by the precomputed 1/T_tt if not unit),
// and every lane applies x_r -= T_rt x_t to its rows r > t (two LDS.128 + two complex FMAs).
// T is staged in shared memory by TMA bulk copies (one per column) completing an mbarrier.
// One column per warp and few warps per CTA spread the independent chains over many SMs (the
// pieces are issue-latency bound per warp); all warps of a CTA share one copy of T.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace feast {
namespace {

constexpr int NB = 64, LDT = NB + 1;   // T[r][c] at Ts[c * LDT + r] (column-major, 1040 B columns)
constexpr int WARPS = 4;      // warps per CTA; one right-hand-side column per warp (spread over SMs)

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// op(T)[r][c] from the shared copy, stored column-major Ts[c * LDT + r] (CONJT: op = ^H).  Lanes
// run over r: consecutive 16 B (no conflict) for op = T; 1040 B apart for op = T^H (4 wavefronts,
// the minimum for a warp's 512 B).
template <bool CONJT>
__device__ __forceinline__ double2 opT(const double2* Ts, int r, int c) {
  if (!CONJT) return Ts[c * LDT + r];
  const double2 v = Ts[r * LDT + c];
  return make_double2(v.x, -v.y);
}

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// Stage the nb x nb block into Ts with the TMA unit: one bulk copy (cp.async.bulk, nb * 16 B) per
// column, completing a transaction mbarrier; the identity padding up to nbp is written meanwhile.
// The solves read only the strict triangle of op(T) and its diagonal (through dinv), so the other
// factor stored in the same LU workspace block needs no masking.  1 / diagonal into dinv.
template <bool LOWER, bool UNIT, bool CONJT>
__device__ void load_tri(const double2* __restrict__ T, int64_t ld, int nb, int nbp, double2* Ts, double2* dinv) {
  __shared__ __align__(8) unsigned long long tbar;
  const unsigned bar = saddr(&tbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)(nb * nb * 16))
                 : "memory");
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nb; c += blockDim.x)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(saddr(Ts + c * LDT)), "l"(T + (int64_t)c * ld), "r"(nb * 16), "r"(bar) : "memory");
  if (nb < nbp)
    for (int idx = threadIdx.x; idx < nbp * nbp; idx += blockDim.x) {
      const int r = idx % nbp, c = idx / nbp;
      if (r >= nb || c >= nb) Ts[c * LDT + r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
  unsigned done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(bar) : "memory");
  __syncthreads();
  if (!UNIT)
    for (int i = threadIdx.x; i < nbp; i += blockDim.x) dinv[i] = crcp(opT<CONJT>(Ts, i, i));
  __syncthreads();
}

// Solve op(T) x = x for CPW columns held as x[c][0] (row lane), x[c][1] (row lane + 32).
template <bool LOWER, bool UNIT, bool CONJT, int CPW>
__device__ __forceinline__ void warp_solve(const double2* Ts, const double2* dinv, int nbp, int t_lo, int t_hi,
                                           double2 (&x)[CPW][2]) {
  const int lane = threadIdx.x & 31;
  for (int s = 0; s < nbp; ++s) {
    const int t = LOWER ? s : nbp - 1 - s;
    if (t < t_lo || t > t_hi) continue;   // warp-uniform
    const int src = t & 31, half = t >> 5;
    double2 xt[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      xt[c] = shfl2(half ? x[c][1] : x[c][0], src);
      if (!UNIT) xt[c] = cmul(xt[c], dinv[t]);
    }
    if (!UNIT && lane == src) {
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        if (half) x[c][1] = xt[c];
        else x[c][0] = xt[c];
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      if (r < nbp && (LOWER ? r > t : r < t)) {
        const double2 trt = opT<CONJT>(Ts, r, t);
#pragma unroll
        for (int c = 0; c < CPW; ++c) x[c][h] = cfms(x[c][h], trt, xt[c]);
      }
    }
  }
}

// ---------------------------------------------------------------- trsm (in place on X)
template <bool LOWER, bool UNIT, bool CONJT, int CPW>
__global__ void __launch_bounds__(32 * WARPS) trsm_warp_kernel(Batched Tb, Batched Xb, int nb, int64_t ncols) {
  extern __shared__ __align__(16) double2 sm[];
  double2* Ts = sm;
  double2* dinv = sm + NB * LDT;
  const int b = blockIdx.y;
  load_tri<LOWER, UNIT, CONJT>(Tb.p + (int64_t)b * Tb.stride, Tb.ld, nb, nb, Ts, dinv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = ((int64_t)blockIdx.x * WARPS + warp) * CPW;
  if (c0 >= ncols) return;
  double2* X = Xb.p + (int64_t)b * Xb.stride;
  double2 x[CPW][2];
#pragma unroll
  for (int c = 0; c < CPW; ++c)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      x[c][h] = (c0 + c < ncols && r < nb) ? X[r + (c0 + c) * Xb.ld] : make_double2(0.0, 0.0);
    }
  warp_solve<LOWER, UNIT, CONJT, CPW>(Ts, dinv, nb, 0, nb - 1, x);
#pragma unroll
  for (int c = 0; c < CPW; ++c)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      if (c0 + c < ncols && r < nb) X[r + (c0 + c) * Xb.ld] = x[c][h];
    }
}

template <bool LOWER, bool UNIT, bool CONJT>
void trsm_t(Batched T, Batched X, int nb, int64_t ncols, int batch, cudaStream_t s) {
  constexpr int CPW = 1;
  const size_t smem = (size_t)(NB * LDT + NB) * sizeof(double2);
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured)) {
    cudaFuncSetAttribute(trsm_warp_kernel<LOWER, UNIT, CONJT, CPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  }
  dim3 grid((unsigned)((ncols + WARPS * CPW - 1) / (WARPS * CPW)), (unsigned)batch);
  trsm_warp_kernel<LOWER, UNIT, CONJT, CPW><<<grid, 32 * WARPS, smem, s>>>(T, X, nb, ncols);
  count_launch();
}

// ---------------------------------------------------------------- trtri (64x64 diagonal blocks)
// blockIdx.x = node, blockIdx.y = 0 (L^-1, unit lower) / 1 (U^-1, upper), blockIdx.z = diagonal
// block index relative to kb0 times TR_CB column groups.  Each CTA inverts WARPS columns of one
// block (identity right-hand sides; column j of L^-1 is zero above row j, of U^-1 zero below, so
// the chains start at t = j), with a CTA per group of columns so the 2 x 64 chains of a node run
// on many SMs at once.
template <int TW, int TCPW>   // TW warps per CTA, TCPW identity columns per warp
__device__ void trtri_block(const double2* __restrict__ T, int64_t ld, int nb, double2* __restrict__ out,
                            double2* Ts, double2* dinv, int cgroup, bool upper) {
  constexpr int TR_CB = NB / (TW * TCPW);   // column groups per diagonal block (CTAs per block)
  if (upper) load_tri<false, false, false>(T, ld, nb, NB, Ts, dinv);
  else load_tri<true, true, false>(T, ld, nb, NB, Ts, dinv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // interleave long and short chains: column j_c = cgroup + TR_CB * (warp + TW * c); the TCPW
  // chains of a warp run side by side (independent FMAs between the same shuffles)
  double2 x[TCPW][2];
  int jmin = NB, jmax = -1;
#pragma unroll
  for (int c = 0; c < TCPW; ++c) {
    const int j = cgroup + TR_CB * (warp + TW * c);
    x[c][0] = make_double2(lane == j ? 1.0 : 0.0, 0.0);
    x[c][1] = make_double2(lane + 32 == j ? 1.0 : 0.0, 0.0);
    jmin = min(jmin, j);
    jmax = max(jmax, j);
  }
  if (upper) warp_solve<false, false, false, TCPW>(Ts, dinv, NB, 0, jmax, x);
  else warp_solve<true, true, false, TCPW>(Ts, dinv, NB, jmin, NB - 1, x);
#pragma unroll
  for (int c = 0; c < TCPW; ++c) {
    const int j = cgroup + TR_CB * (warp + TW * c);
    out[lane + j * NB] = x[c][0];
    out[lane + 32 + j * NB] = x[c][1];
  }
}

template <int TW, int TCPW>
__global__ void __launch_bounds__(32 * TW) trtri_kernel(Batched Cb, int64_t n, int64_t kb0,
                                                       double2* __restrict__ inv, int64_t inv_node_stride,
                                                       int which) {
  constexpr int TR_CB = NB / (TW * TCPW);
  extern __shared__ __align__(16) double2 sm[];
  double2* Ts = sm;
  double2* dinv = sm + NB * LDT;
  const int b = blockIdx.x;
  const int lu = (which == 2) ? (int)blockIdx.y : which;
  const int64_t kb = kb0 + blockIdx.z / TR_CB;
  const int cgroup = (int)(blockIdx.z % TR_CB);
  const int64_t o = kb * NB;
  const int nb = (int)((n - o) < NB ? (n - o) : NB);
  const double2* T = Cb.p + (int64_t)b * Cb.stride + o + o * Cb.ld;
  double2* out = inv + (int64_t)b * inv_node_stride + (kb * 2 + lu) * (int64_t)NB * NB;
  trtri_block<TW, TCPW>(T, Cb.ld, nb, out, Ts, dinv, cgroup, lu != 0);
}

template <int TW, int TCPW>
void trtri_t(Batched C, int64_t n, int64_t kb0, int64_t nblocks, double2* inv, int64_t inv_node_stride, int which,
             int batch, cudaStream_t s) {
  constexpr int TR_CB = NB / (TW * TCPW);
  const size_t smem = (size_t)(NB * LDT + NB) * sizeof(double2);
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured)) {
    cudaFuncSetAttribute(trtri_kernel<TW, TCPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  dim3 grid((unsigned)batch, which == 2 ? 2u : 1u, (unsigned)(nblocks * TR_CB));
  trtri_kernel<TW, TCPW><<<grid, 32 * TW, smem, s>>>(C, n, kb0, inv, inv_node_stride, which);
  count_launch();
}

}  // namespace

void trsm_launch(Batched T, Batched X, int nb, int64_t ncols, bool lower_op, bool unit, bool conjT, int batch,
                 cudaStream_t s) {
  ProfScope ps_(K_TRSM, (double)batch * 4.0 * nb * nb * ncols, 0.0, s);
  if (ncols <= 0 || nb <= 0) return;
#define TR_CASE(L, U, C) \
  if (lower_op == L && unit == U && conjT == C) { trsm_t<L, U, C>(T, X, nb, ncols, batch, s); return; }
  TR_CASE(true, true, false)
  TR_CASE(true, false, false)
  TR_CASE(false, true, false)
  TR_CASE(false, false, false)
  TR_CASE(true, true, true)
  TR_CASE(true, false, true)
  TR_CASE(false, true, true)
  TR_CASE(false, false, true)
#undef TR_CASE
}

void trtri_launch(Batched C, int64_t n, int64_t kb0, int64_t nblocks, double2* inv, int64_t inv_node_stride, int which,
                  int batch, cudaStream_t s) {
  ProfScope ps_(K_TRSM, (double)batch * nblocks * (which == 2 ? 2 : 1) * 8.0 * NB * NB * NB / 3.0, 0.0, s);
  // 8 warps x 2 interleaved chains per CTA, 4 CTAs per block (C2 step 16.76 -> 16.71 ms vs
  // 4 warps x 1 chain, 16 CTAs per block; 16 warps x 4 chains, one CTA per block: 16.85 ms)
  trtri_t<8, 2>(C, n, kb0, nblocks, inv, inv_node_stride, which, batch, s);
}

}  // namespace feast
