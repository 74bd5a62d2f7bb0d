// btrsm.cu — block triangular solve on the FP64 tensor pipe (DMMA), one kernel per <= 256-row block.
//
// Y <- op(T)^-1 Y for a triangular block of R <= 256 rows built from 64 x 64 blocks whose diagonal
// inverses were formed by trtri (SURVEY §8(a) a3 "TRSM blocks", a4 substitutions).  The one-level
// sequence this replaces is, per 64-row block kb, an in-place product Y_kb <- Inv_kb Y_kb and an
// update GEMM Y_rest -= T[rest, kb] Y_kb (K = 64): seven dependent launches per 256-row block whose
// CTAs spend most of their time filling and draining a 4-stage pipeline.  Here ONE CTA per
// 32-column tile of Y runs the whole block solve: the R x 32 tile lives in REGISTERS (each warp
// owns a 16 x 16 piece of every 64-row block, in the DMMA accumulator layout), the <= 10 operand
// blocks (diagonal inverses and off-diagonal T blocks, 64 x 64 each, from L2) stream through one
// continuous cp.async ring, and shared memory holds only that ring and the solved 64-row block
// in the B-operand layout (86 KB: two CTAs per SM, so one CTA's loads overlap the other's DMMA).
//
// The 64-row blocks are indexed by their position s in solve order (forward: block s; backward:
// block nb - 1 - s), so every register array index is a compile-time constant; block s updates
// the blocks s' > s in both directions.
//
// Arithmetic: the planar-complex DMMA product of zgemm_dmma.cu (four mma.m8n8k4.f64 per complex
// 8x8x4 block, separate re / im accumulators, signs folded into the operands); op = conjugate
// transpose reads the stored block T[kb, rb] "as rows" and negates its imaginary part.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace feast {
namespace {

constexpr int BT_TN = 32;          // columns of Y per CTA
constexpr int BT_THREADS = 256;    // 8 warps: 4 (rows of 16) x 2 (columns of 16) of a 64 x 32 block
constexpr int BT_ST = 3;           // A-ring stages (16 k each)
constexpr int BT_LDX = 64 + 4;     // Xs[col][k]
constexpr int BT_LDA = 64 + 2;     // As[k][m]
constexpr int BT_A_STAGE = 16 * BT_LDA;
constexpr size_t BT_SMEM = ((size_t)BT_TN * BT_LDX + (size_t)BT_ST * BT_A_STAGE) * sizeof(double2);

__device__ __forceinline__ void dmma_bt(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool FWD, bool CONJ, int MINB>
__global__ void __launch_bounds__(BT_THREADS, MINB) btrsm_kernel(BtrsmArgs p) {
  extern __shared__ __align__(128) double2 sm[];
  double2* Xs = sm;                                 // [BT_TN][BT_LDX]: the solved block (B operand)
  double2* As = Xs + BT_TN * BT_LDX;                // [BT_ST][16][BT_LDA]
  const int R = (int)p.R;
  const int z = blockIdx.y;
  const double2* __restrict__ T = p.T0 + (int64_t)z * p.sT;
  const double2* __restrict__ Inv = p.Inv0 + (int64_t)z * p.sInv;
  double2* __restrict__ Y = p.Y0 + (int64_t)z * p.sY;
  const int64_t n0 = (int64_t)blockIdx.x * BT_TN;
  const int tn = (int)(p.N - n0 < BT_TN ? p.N - n0 : BT_TN);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 16;
  const int nb = (R + 63) / 64;
  auto blk_of = [&](int s) { return FWD ? s : nb - 1 - s; };       // solve position -> block index
  auto rows_of = [&](int b) { return min(64, R - 64 * b); };

  // product q enumerates (position s, target position s2): s2 == s is the diagonal inverse of s,
  // s2 > s an update of block s2 by the solved block s
  auto product = [&](int q, int& s, int& s2) {
    int idx = q;
    for (int a = 0; a < nb; ++a) {
      const int nup = nb - 1 - a;
      if (idx <= nup) { s = a; s2 = a + idx; return; }
      idx -= nup + 1;
    }
    s = s2 = 0;
  };
  const int nchunk = 4 * (nb + nb * (nb - 1) / 2);

  // A-operand chunk c: k-slice (c % 4) * 16 .. +16 of op(T)[blk(s2), blk(s)] (diagonal: op(Inv))
  auto load_chunk = [&](int c, int stage) {
    int s, s2;
    product(c >> 2, s, s2);
    const int rb = blk_of(s2), kb = blk_of(s);
    const int k0 = (c & 3) * 16;
    const int M = rows_of(rb), K = rows_of(kb);
    const double2* blk;
    int64_t ld;
    if (rb == kb) { blk = Inv + (int64_t)kb * p.inv_step; ld = 64; }
    else if (!CONJ) { blk = T + (int64_t)(64 * rb) + (int64_t)(64 * kb) * p.ldt; ld = p.ldt; }
    else { blk = T + (int64_t)(64 * kb) + (int64_t)(64 * rb) * p.ldt; ld = p.ldt; }
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(As + stage * BT_A_STAGE);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int m, k;
      const double2* src;
      if (!CONJ) { m = tid & 63; k = (tid >> 6) + 4 * i; src = blk + m + (int64_t)(k0 + k) * ld; }
      else { k = tid & 15; m = (tid >> 4) + 16 * i; src = blk + (k0 + k) + (int64_t)m * ld; }
      const bool pred = m < M && k0 + k < K;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + (k * BT_LDA + m) * 16),
                   "l"(pred ? src : blk), "r"(pred ? 16 : 0));
    }
  };
#pragma unroll
  for (int c = 0; c < BT_ST - 1; ++c) {
    if (c < nchunk) load_chunk(c, c);
    asm volatile("cp.async.commit_group;\n" ::);
  }

  // ---- the Y tile in registers: y[s][mi][nj][i] = Y[64 blk(s) + wm + 8 mi + g][wn + 8 nj + 2 t + i]
  double2 y[4][2][2][2];
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = 64 * blk_of(s) + wm + 8 * mi + g, col = wn + 8 * nj + 2 * t + i;
          y[s][mi][nj][i] = (s < nb && r < R && col < tn) ? Y[r + (n0 + col) * p.ldy] : make_double2(0.0, 0.0);
        }

  double cre[2][2][2], cim[2][2][2];
  constexpr double SI = CONJ ? -1.0 : 1.0;
  int c = 0;   // next chunk to consume
  // acc = op(A product) * Xs over the product's 4 chunks (the ring advances across products)
  auto run_product = [&]() {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) cre[mi][nj][0] = cre[mi][nj][1] = cim[mi][nj][0] = cim[mi][nj][1] = 0.0;
#pragma unroll 1
    for (int kc = 0; kc < 4; ++kc, ++c) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(BT_ST - 2));
      __syncthreads();   // chunk c resident everywhere; every warp is past chunk c - 1
      if (c + BT_ST - 1 < nchunk) load_chunk(c + BT_ST - 1, (c + BT_ST - 1) % BT_ST);
      asm volatile("cp.async.commit_group;\n" ::);
      const double2* as = As + (c % BT_ST) * BT_A_STAGE;
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        double2 af[2], bf[2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) af[mi] = as[(4 * k4 + t) * BT_LDA + wm + 8 * mi + g];
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) bf[nj] = Xs[(wn + 8 * nj + g) * BT_LDX + 16 * kc + 4 * k4 + t];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const double ar = af[mi].x, ai = SI * af[mi].y;
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) {
            dmma_bt(cre[mi][nj][0], cre[mi][nj][1], ar, bf[nj].x);
            dmma_bt(cim[mi][nj][0], cim[mi][nj][1], ar, bf[nj].y);
            dmma_bt(cre[mi][nj][0], cre[mi][nj][1], -ai, bf[nj].y);
            dmma_bt(cim[mi][nj][0], cim[mi][nj][1], ai, bf[nj].x);
          }
        }
      }
    }
  };
  // write one block's registers into Xs, the B operand
  auto to_xs = [&](const double2 (&v)[2][2][2]) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
#pragma unroll
        for (int i = 0; i < 2; ++i) Xs[(wn + 8 * nj + 2 * t + i) * BT_LDX + wm + 8 * mi + g] = v[mi][nj][i];
  };

#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s >= nb) break;
    // ---- diagonal block: X_s = op(Inv) Y_s
    __syncthreads();                  // every warp is done reading Xs (the previous solved block)
    to_xs(y[s]);
    run_product();                    // (its first barrier publishes Xs)
    __syncthreads();                  // every warp is done reading Xs as the right-hand side
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
#pragma unroll
        for (int i = 0; i < 2; ++i) y[s][mi][nj][i] = make_double2(cre[mi][nj][i], cim[mi][nj][i]);
    to_xs(y[s]);                      // the solved block: operand of the updates below
    // ---- updates of the blocks still to be solved: Y_s2 -= op(T)[s2, s] X_s
#pragma unroll
    for (int s2 = s + 1; s2 < 4; ++s2) {
      if (s2 >= nb) break;
      run_product();
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            double2& v = y[s2][mi][nj][i];
            v = make_double2(v.x - cre[mi][nj][i], v.y - cim[mi][nj][i]);
          }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = 64 * blk_of(s) + wm + 8 * mi + g, col = wn + 8 * nj + 2 * t + i;
          if (s < nb && r < R && col < tn) Y[r + (n0 + col) * p.ldy] = y[s][mi][nj][i];
        }
}

template <bool FWD, bool CONJ, int MINB>
void launch_bt(const BtrsmArgs& p, cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured))
    cudaFuncSetAttribute(btrsm_kernel<FWD, CONJ, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BT_SMEM);
  dim3 grid((unsigned)((p.N + BT_TN - 1) / BT_TN), (unsigned)p.batch);
  btrsm_kernel<FWD, CONJ, MINB><<<grid, BT_THREADS, BT_SMEM, s>>>(p);
}

// FEAST_BTRSM_MINB: 2 (default) = two CTAs per SM (registers capped at 128: ~1 KB of spills at the
// product boundaries), 1 = one CTA per SM without spills
int bt_minb() {
  static const int v = [] { const char* e = getenv("FEAST_BTRSM_MINB"); return (e && e[0] == '1') ? 1 : 2; }();
  return v;
}
template <bool FWD, bool CONJ>
void launch_bt2(const BtrsmArgs& p, cudaStream_t s) {
  if (bt_minb() == 1) launch_bt<FWD, CONJ, 1>(p, s); else launch_bt<FWD, CONJ, 2>(p, s);
}

}  // namespace

void btrsm_launch(const BtrsmArgs& p, bool fwd, bool conj, cudaStream_t s) {
  if (p.R <= 0 || p.N <= 0 || p.batch <= 0) return;
  // algorithmic flops: a triangular solve of R rows against N columns, 4 R (R + 1) N (complex)
  ProfScope ps_(K_ZGEMM, 4.0 * (double)p.R * (double)(p.R + 1) * (double)p.N * p.batch,
                16.0 * ((double)p.R * p.R / 2 + 2.0 * p.R * p.N) * p.batch, s);
  if (fwd) { if (conj) launch_bt2<true, true>(p, s); else launch_bt2<true, false>(p, s); }
  else { if (conj) launch_bt2<false, true>(p, s); else launch_bt2<false, false>(p, s); }
  count_launch();
}

}  // namespace feast
