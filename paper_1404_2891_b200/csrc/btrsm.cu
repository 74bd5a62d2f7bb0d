// btrsm.cu — block triangular solve on the FP64 tensor pipe (DMMA), one kernel per <= 256-row block.
//
// Y <- op(T)^-1 Y for a triangular block of R <= 256 rows built from 64 x 64 blocks whose diagonal
// inverses were formed by trtri (SURVEY §8(a) a3 "TRSM blocks", a4 substitutions).  The one-level
// sequence this replaces is, per 64-row block kb, an in-place product Y_kb <- Inv_kb Y_kb and an
// update GEMM Y_rest -= T[rest, kb] Y_kb (K = 64): seven dependent launches per 256-row block whose
// CTAs spend most of their time filling and draining a 4-stage pipeline (5-20 TF/s measured).
// Here ONE CTA per 32-column tile of Y keeps the R x 32 tile in shared memory for the whole block
// solve and streams the <= 10 operand blocks (diagonal inverses and off-diagonal T blocks, 64 x 64
// each, from L2) through one continuous cp.async ring, so the pipeline fills once per tile.
//
// Arithmetic: the planar-complex DMMA product of zgemm_dmma.cu (four mma.m8n8k4.f64 per complex
// 8x8x4 block, separate re / im accumulators, signs folded into the operands); op = conjugate
// transpose reads the stored block T[kb, rb] "as rows" and negates its imaginary part.
//
// Shared memory (TN = 32 columns): Ys row-major R x 33 (the C-operand pattern of a DMMA fragment,
// lanes (g, 2t+i), is bank-conflict free with ld = 33), Xs = the solved 64-row block in the
// B-operand layout [n][k] (ld 68), and the A ring [stage][k][m] (ld 66): 135 + 35 + 51 KB.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace feast {
namespace {

constexpr int BT_TN = 32;          // columns of Y per CTA
constexpr int BT_THREADS = 256;    // 8 warps: 4 (rows of 16) x 2 (columns of 16) of a 64 x 32 block
constexpr int BT_ST = 3;           // A-ring stages (16 k each)
constexpr int BT_LDY = BT_TN + 1;  // Ys[row][col]
constexpr int BT_LDX = 64 + 4;     // Xs[col][k]
constexpr int BT_LDA = 64 + 2;     // As[k][m]
constexpr int BT_A_STAGE = 16 * BT_LDA;
constexpr size_t bt_smem(int R) {
  return ((size_t)R * BT_LDY + (size_t)BT_TN * BT_LDX + (size_t)BT_ST * BT_A_STAGE) * sizeof(double2);
}

__device__ __forceinline__ void dmma_bt(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool FWD, bool CONJ>
__global__ void __launch_bounds__(BT_THREADS, 1) btrsm_kernel(BtrsmArgs p) {
  extern __shared__ __align__(128) double2 sm[];
  const int R = (int)p.R;
  double2* Ys = sm;                                 // [R][BT_LDY]
  double2* Xs = Ys + (size_t)R * BT_LDY;            // [BT_TN][BT_LDX]
  double2* As = Xs + BT_TN * BT_LDX;                // [BT_ST][16][BT_LDA]
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
  auto rows_of = [&](int b) { return min(64, R - 64 * b); };

  // ---- the operand-block schedule: for each kb (in solve order) the diagonal inverse, then the
  // off-diagonal blocks of the rows still to be updated.  Product q = (rb, kb); rb == kb: inverse.
  // (at most 10 products for 4 blocks; generated on the fly from q)
  auto product = [&](int q, int& rb, int& kb) {
    // enumerate kb in solve order, each followed by its update rows
    int idx = q;
    for (int s = 0; s < nb; ++s) {
      const int k = FWD ? s : nb - 1 - s;
      const int nup = FWD ? nb - 1 - k : k;          // rows after (fwd) / before (bwd) k
      if (idx == 0) { rb = k; kb = k; return; }
      if (idx <= nup) { rb = FWD ? k + idx : k - idx; kb = k; return; }
      idx -= nup + 1;
    }
    rb = kb = -1;
  };
  const int nprod = nb + nb * (nb - 1) / 2;
  const int nchunk = 4 * nprod;

  // ---- A-operand chunk loader: chunk c = product c / 4, k-slice (c % 4) * 16 .. +16 of the 64 x 64
  // block op(T)[rb, kb] (diagonal: op(Inv_kb)), rows m < rows_of(rb), k < rows_of(kb) (else 0)
  auto load_chunk = [&](int c, int stage) {
    int rb, kb;
    product(c >> 2, rb, kb);
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

  // ---- Y tile -> Ys (rows >= R and columns >= tn zero)
  for (int e = tid; e < R * BT_TN; e += BT_THREADS) {
    const int r = e % R, c = e / R;   // consecutive threads: consecutive rows of a column (coalesced)
    Ys[r * BT_LDY + c] = c < tn ? Y[r + (n0 + c) * p.ldy] : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int s = 0; s < BT_ST - 1; ++s) {
    if (s < nchunk) load_chunk(s, s);
    asm volatile("cp.async.commit_group;\n" ::);
  }

  double cre[2][2][2], cim[2][2][2];
  auto zero_acc = [&]() {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) cre[mi][nj][0] = cre[mi][nj][1] = cim[mi][nj][0] = cim[mi][nj][1] = 0.0;
  };
  zero_acc();
  constexpr double SI = CONJ ? -1.0 : 1.0;

  for (int c = 0; c < nchunk; ++c) {
    int rb, kb;
    product(c >> 2, rb, kb);
    if ((c & 3) == 0 && rb == kb) {
      // start of block kb: its rows are final (every earlier update wrote them) -> B layout
      __syncthreads();
      for (int e = tid; e < 64 * BT_TN; e += BT_THREADS) {
        const int k = e & 63, col = e >> 6;
        Xs[col * BT_LDX + k] = 64 * kb + k < R ? Ys[(64 * kb + k) * BT_LDY + col] : make_double2(0.0, 0.0);
      }
    }
    // chunk c resident; then (every warp past chunk c - 1) refill its stage with chunk c + ST - 1
    asm volatile("cp.async.wait_group %0;\n" ::"n"(BT_ST - 2));
    __syncthreads();
    if (c + BT_ST - 1 < nchunk) load_chunk(c + BT_ST - 1, (c + BT_ST - 1) % BT_ST);
    asm volatile("cp.async.commit_group;\n" ::);
    const double2* as = As + (c % BT_ST) * BT_A_STAGE;
    const int kk0 = (c & 3) * 16;
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      double2 af[2], bf[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) af[mi] = as[(4 * k4 + t) * BT_LDA + wm + 8 * mi + g];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) bf[nj] = Xs[(wn + 8 * nj + g) * BT_LDX + kk0 + 4 * k4 + t];
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
    if ((c & 3) == 3) {
      // end of product (rb, kb)
      if (rb == kb) {
        __syncthreads();   // every warp is done reading Xs (the right-hand side) for this block
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int r = wm + 8 * mi + g, col = wn + 8 * nj + 2 * t + i;
              const double2 v = make_double2(cre[mi][nj][i], cim[mi][nj][i]);
              Xs[col * BT_LDX + r] = v;                       // solved block: operand of the updates
              if (64 * kb + r < R) Ys[(64 * kb + r) * BT_LDY + col] = v;
            }
        __syncthreads();
      } else {
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int r = 64 * rb + wm + 8 * mi + g, col = wn + 8 * nj + 2 * t + i;
              if (r < R) {
                double2& y = Ys[r * BT_LDY + col];
                y = make_double2(y.x - cre[mi][nj][i], y.y - cim[mi][nj][i]);
              }
            }
      }
      zero_acc();
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  for (int e = tid; e < R * BT_TN; e += BT_THREADS) {
    const int r = e % R, col = e / R;
    if (col < tn) Y[r + (n0 + col) * p.ldy] = Ys[r * BT_LDY + col];
  }
}

template <bool FWD, bool CONJ>
void launch_bt(const BtrsmArgs& p, cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured))
    cudaFuncSetAttribute(btrsm_kernel<FWD, CONJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bt_smem(256));
  dim3 grid((unsigned)((p.N + BT_TN - 1) / BT_TN), (unsigned)p.batch);
  btrsm_kernel<FWD, CONJ><<<grid, BT_THREADS, bt_smem((int)p.R), s>>>(p);
}

}  // namespace

void btrsm_launch(const BtrsmArgs& p, bool fwd, bool conj, cudaStream_t s) {
  if (p.R <= 0 || p.N <= 0 || p.batch <= 0) return;
  // algorithmic flops: a triangular solve of R rows against N columns, 4 R (R + 1) N (complex)
  ProfScope ps_(K_ZGEMM, 4.0 * (double)p.R * (double)(p.R + 1) * (double)p.N * p.batch,
                16.0 * ((double)p.R * p.R / 2 + 2.0 * p.R * p.N) * p.batch, s);
  if (fwd) { if (conj) launch_bt<true, true>(p, s); else launch_bt<true, false>(p, s); }
  else { if (conj) launch_bt<false, true>(p, s); else launch_bt<false, false>(p, s); }
  count_launch();
}

}  // namespace feast
