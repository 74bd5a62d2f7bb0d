// zgemm_dmma.cu — batched complex128 GEMM on the FP64 tensor pipe (DMMA) for sm_100a.
//
// The one dense contraction of the hot path: the LU trailing
// update A22 -= L21 U12, the blocked-substitution updates, R = B X and Q^H (A Q).
// tcgen05 has no f64 kind on sm_100a, so the tensor-core path for FP64 is mma.sync
// m8n8k4.f64 (SASS DMMA.8x8x4), measured at 37.17 TF/s peak on B200 (profiles/r01_fp64_peak.md).
//
// Tiling (measured, tools/zgemm_lab.cu, profiles/r01_zgemm_lab.md): CTA 32x32 complex outputs,
// 4 warps of 16x16, BK = 16 complex per stage, 4-stage cp.async ring (76 KB smem, 3 CTAs and
// 12 warps per SM).  The small CTA tile keeps more warps resident to hide shared-memory and L2
// latency behind the DMMA pipe, and fills the 148 SMs even on the narrow updates of the LU
// (N = 32..256).  In-place launches (C aliases B: the 64x64 diagonal-block inverses applied to
// a block row) use 64x32 CTAs so one CTA row covers all M <= 64 rows it overwrites.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace feast {
namespace {


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// PLANAR complex product — four real DMMAs per complex 8x8x4 block with separate real and
// imaginary accumulators:  Re += ar br - ai bi,  Im += ar bi + ai br  (conj(A): ai -> -ai;
// C -= AB: every product negated).  All sign changes are warp-uniform, so ptxas folds them
// into the DMMA operand modifiers (no integer sign flips), and each lane's A (B) fragment is
// one whole complex element: a single 16-byte LDS.128 per fragment.
//   A fragment (row g, k t) = A[m0 + g][k0 + t];  B fragment (k t, col g) = B[k0 + t][n0 + g]
//   accumulators: C[g][2t + i], i = 0, 1 (re and im in separate registers).
// Shared layout: As[k][m] with ld BM + 2 (quarter-warp rows 32 B apart: conflict-free 128-bit
// loads), Bs[n][k] with ld BK + 4.
template <int BM, int BN, int WGM, int WGN, int ST, int BK>
struct Tile {
  static constexpr int THREADS = 32 * WGM * WGN;
  static constexpr int TM = BM / WGM, TN = BN / WGN;
  static constexpr int MI = TM / 8, NJ = TN / 8;
  static constexpr int LDA_S = BM + 2, LDB_S = BK + 4;
  static constexpr int A_STAGE = BK * LDA_S;
  static constexpr int B_STAGE = BN * LDB_S;
  static constexpr size_t SMEM_BYTES = (size_t)ST * (A_STAGE + B_STAGE) * sizeof(double2);
};

template <int BM, int BN, int WGM, int WGN, int ST, int MINB, bool CONJA, int MODE, bool PREC = true, int BK = 16>
__global__ void __launch_bounds__(32 * WGM * WGN, MINB) zgemm_dmma_kernel(ZgemmArgs p) {
  using T = Tile<BM, BN, WGM, WGN, ST, BK>;
  constexpr int THREADS = T::THREADS, LDA_S = T::LDA_S, LDB3 = T::LDB_S, A_STAGE = T::A_STAGE,
                B_STAGE = T::B_STAGE;
  constexpr int MI = T::MI, NJ = T::NJ;
  constexpr int LA = (BM * BK) / THREADS, LB = (BN * BK) / THREADS;
  static_assert(MI >= 1 && NJ >= 1 && LA >= 1 && LB >= 1, "tile");
  static_assert(THREADS % BM == 0 && THREADS % BK == 0, "load mapping");
  extern __shared__ __align__(128) double2 smem[];
  double2* As = smem;
  double2* Bs = smem + ST * A_STAGE;

  const int64_t M = p.M, N = p.N, K = p.K;
  // tile coordinates: plain (grid x = N tiles, y = M tiles, z = batch) or, for large grids
  // (swz > 1), grid (swz, N tiles, M-tile groups x batch): the scheduler walks x fastest, so the
  // CTAs resident at once cover swz tile rows x ~444/swz tile columns of C and re-read their A
  // row tiles and B column tiles from L2 instead of DRAM
  unsigned mt = blockIdx.y, nt = blockIdx.x, zb = blockIdx.z;
  if (p.swz > 1) {
    const unsigned groups = (unsigned)(((p.M + BM - 1) / BM + p.swz - 1) / p.swz);
    zb = blockIdx.z / groups;
    mt = (blockIdx.z - zb * groups) * (unsigned)p.swz + blockIdx.x;
    nt = blockIdx.y;
    if ((int64_t)mt * BM >= p.M) return;   // ragged last group (the whole CTA leaves before any barrier)
  }
  const int64_t m0 = (int64_t)mt * BM, n0 = (int64_t)nt * BN;
  const int64_t z = zb;
  const double2* __restrict__ A = p.A + z * p.sA;
  const double2* __restrict__ B = p.B + z * p.sB;
  double2* __restrict__ C = p.C + z * p.sC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = (warp / WGN) * T::TM, wn = (warp % WGN) * T::TN;
  const int g = lane >> 2, t = lane & 3;

  // ---- global -> shared mapping (fixed per thread; only the k-tile base advances)
  //  A (op = N):  m = tid % BM, k = tid / BM + i * (THREADS / BM)
  //  A (op = C):  k = tid % BK, m = tid / BK + i * (THREADS / BK)     (A^H read as rows of A)
  //  B:           k = tid % BK, n = tid / BK + i * (THREADS / BK)
  const int a_m = CONJA ? tid / BK : tid % BM, a_k = CONJA ? tid % BK : tid / BM;
  constexpr int A_DI = CONJA ? THREADS / BK : THREADS / BM;   // step of the varying index
  const int b_k = tid % BK, b_n = tid / BK;
  constexpr int B_DI = THREADS / BK;
  const double2* a_src = CONJA ? A + (m0 + a_m) * p.lda + a_k : A + (m0 + a_m) + (int64_t)a_k * p.lda;
  const int64_t a_step = CONJA ? (int64_t)A_DI * p.lda : (int64_t)A_DI * p.lda;   // per i
  const int64_t a_kt = CONJA ? BK : (int64_t)BK * p.lda;                          // per k-tile
  const double2* b_src = B + (n0 + b_n) * p.ldb + b_k;
  const int64_t b_step = (int64_t)B_DI * p.ldb;
  unsigned a_ok = 0, b_ok = 0;   // bit i: row / column in range
#pragma unroll
  for (int i = 0; i < LA; ++i)
    if (CONJA ? (m0 + a_m + i * A_DI < M) : (m0 + a_m < M)) a_ok |= 1u << i;
#pragma unroll
  for (int i = 0; i < LB; ++i)
    if (n0 + b_n + i * B_DI < N) b_ok |= 1u << i;
  const uint32_t as_dst = (uint32_t)__cvta_generic_to_shared(As + a_k * LDA_S + a_m);
  const uint32_t bs_dst = (uint32_t)__cvta_generic_to_shared(Bs + b_n * LDB3 + b_k);
  constexpr uint32_t A_DST_STEP = (CONJA ? A_DI : A_DI * LDA_S) * 16;
  constexpr uint32_t B_DST_STEP = B_DI * LDB3 * 16;

  auto load_tile = [&](int stage, int kt) {
    const int64_t k0 = (int64_t)kt * BK;
    const double2* as = a_src + kt * a_kt;
    const double2* bs = b_src + k0;
    const uint32_t ad = as_dst + stage * (A_STAGE * 16), bd = bs_dst + stage * (B_STAGE * 16);
    // source pointers advanced incrementally (no per-i 64-bit offsets held in registers)
    const double2* ap = as;
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const bool kin = CONJA ? (k0 + a_k < K) : (k0 + a_k + i * A_DI < K);
      const bool pred = ((a_ok >> i) & 1u) && kin;
      const int sz = pred ? 16 : 0;
      const double2* src = pred ? ap : A;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(ad + i * A_DST_STEP), "l"(src), "r"(sz));
      ap += a_step;
    }
    const double2* bp = bs;
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const bool pred = ((b_ok >> i) & 1u) && (k0 + b_k < K);
      const int sz = pred ? 16 : 0;
      const double2* src = pred ? bp : B;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(bd + i * B_DST_STEP), "l"(src), "r"(sz));
      bp += b_step;
    }
  };

  const int KT = (int)((K + BK - 1) / BK);
#pragma unroll
  for (int s = 0; s < ST; ++s) {
    if (s < KT) load_tile(s, s);
    cp_commit();
  }

  // accumulators start at zero; C (SUB: C_old, GEN: beta C_old) joins in the epilogue.  In SUB
  // mode C_old is prefetched into registers here, so its latency overlaps the pipeline fill and
  // no DMMA waits on it.
  double cre[MI][NJ][2], cim[MI][NJ][2];
  constexpr bool PRE = MODE == ZG_SUB && PREC;   // C_old prefetched into registers
  double2 cold[PRE ? MI : 1][PRE ? NJ : 1][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        cre[mi][nj][i] = cim[mi][nj][i] = 0.0;
        if (PRE) {
          const int64_t r = m0 + wm + mi * 8 + g, c = n0 + wn + nj * 8 + 2 * t + i;
          cold[mi][nj][i] = (r < M && c < N) ? C[r + c * p.ldc] : make_double2(0.0, 0.0);
        }
      }

  const int offA = t * LDA_S + wm + g;          // complex offsets inside a stage
  const int offB = (wn + g) * LDB3 + t;
  double2 af[2][MI], bf[2][NJ];
  auto load_frags = [&](int fb, int stage, int ks) {   // ks: complex k offset (multiple of 4)
    const double2* as = As + stage * A_STAGE + offA + ks * LDA_S;
    const double2* bs = Bs + stage * B_STAGE + offB + ks;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) af[fb][mi] = as[mi * 8];
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj) bf[fb][nj] = bs[nj * 8 * LDB3];
  };
  constexpr double SA = MODE == ZG_SUB ? -1.0 : 1.0;     // sign of every product
  constexpr double SI = CONJA ? -1.0 : 1.0;             // sign of ai

  cp_wait<ST - 1>();
  __syncthreads();
  load_frags(0, 0, 0);
  int cur = 0;
  for (int kt = 0; kt < KT; ++kt) {
    const int nxt = cur + 1 == ST ? 0 : cur + 1;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int fb = k4 & 1;
      if (k4 == BK / 4 - 1) {
        cp_wait<ST - 2>();
        __syncthreads();                            // every warp is done reading buffer `cur`
        if (kt + ST < KT) load_tile(cur, kt + ST);
        cp_commit();
        if (kt + 1 < KT) load_frags(fb ^ 1, nxt, 0);
      } else {
        load_frags(fb ^ 1, cur, 4 * (k4 + 1));
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const double ar = SA * af[fb][mi].x, ai = SA * SI * af[fb][mi].y;
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) {
          dmma(cre[mi][nj][0], cre[mi][nj][1], ar, bf[fb][nj].x);
          dmma(cim[mi][nj][0], cim[mi][nj][1], ar, bf[fb][nj].y);
        }
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) {
          dmma(cre[mi][nj][0], cre[mi][nj][1], -ai, bf[fb][nj].y);
          dmma(cim[mi][nj][0], cim[mi][nj][1], ai, bf[fb][nj].x);
        }
      }
    }
    cur = nxt;
  }
  cp_wait<0>();

  const bool use_beta = MODE == ZG_GEN && (p.beta.x != 0.0 || p.beta.y != 0.0);
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int64_t r = m0 + wm + mi * 8 + g, c = n0 + wn + nj * 8 + 2 * t + i;
        if (r < M && c < N) {
          double2* cp = C + r + c * p.ldc;
          double2 v = make_double2(cre[mi][nj][i], cim[mi][nj][i]);
          if (MODE == ZG_SUB) {
            v = cadd(PRE ? cold[PRE ? mi : 0][PRE ? nj : 0][i] : *cp, v);
          } else {
            v = cmul(p.alpha, v);
            if (use_beta) v = cadd(v, cmul(p.beta, *cp));
          }
          *cp = v;
        }
      }
}
template <int BM, int BN, int WGM, int WGN, int ST, int MINB, bool CONJA, int MODE, bool PREC = true, int BK = 16>
void launch3(const ZgemmArgs& p, cudaStream_t s) {
  using T = Tile<BM, BN, WGM, WGN, ST, BK>;
  auto kern = zgemm_dmma_kernel<BM, BN, WGM, WGN, ST, MINB, CONJA, MODE, PREC, BK>;
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM_BYTES);
  }
  const int64_t tn = (p.N + BN - 1) / BN, tm = (p.M + BM - 1) / BM;
  const dim3 grid = p.swz > 1 ? dim3((unsigned)p.swz, (unsigned)tn, (unsigned)((tm + p.swz - 1) / p.swz * p.batch))
                              : dim3((unsigned)tn, (unsigned)tm, (unsigned)p.batch);
  kern<<<grid, T::THREADS, T::SMEM_BYTES, s>>>(p);
  count_launch();
}


// FEAST_SWZ: tile rows per rasterisation group of large non-in-place grids (default 16; 0/1 = off)
int swz_rows() {
  static const int v = [] { const char* e = getenv("FEAST_SWZ"); return e ? atoi(e) : 16; }();
  return v;
}

template <bool CONJA, int MODE>
void launch_t(const ZgemmArgs& p, cudaStream_t s) {
  // in place (C aliases B, BM >= M: one CTA row of tiles): 64x16 CTAs when the 64x32 grid would
  // leave most SMs idle (the substitutions' Y_k <- T_kk^-1 Y_k with N = m0)
  if (p.inplace && (p.N + 31) / 32 * p.batch < 148) launch3<64, 16, 4, 1, 4, 2, CONJA, MODE>(p, s);
  else if (p.inplace) launch3<64, 32, 2, 2, 4, 2, CONJA, MODE>(p, s);
  else {
    // large grids: rasterise in groups of swz_rows() tile rows (a wave of 444 resident CTAs then
    // spans ~16 x 28 tiles: each A row tile and B column tile is fetched from DRAM once per patch)
    ZgemmArgs q = p;
    const int g = swz_rows();
    if (g > 1 && (p.M + 31) / 32 >= 2 * g && (p.N + 31) / 32 >= 2 * g) q.swz = g;
    launch3<32, 32, 2, 2, 4, 3, CONJA, MODE>(q, s);
  }
}

// tile variants kept for tools/zgemm_lab (0 = the production choice above)
template <bool CONJA, int MODE>
void launch_variant(const ZgemmArgs& p, int v, cudaStream_t s) {
  switch (v) {
    case 1: launch3<64, 64, 2, 2, 3, 2, CONJA, MODE>(p, s); break;
    case 2: launch3<64, 32, 2, 2, 4, 2, CONJA, MODE>(p, s); break;
    case 3: launch3<32, 32, 2, 2, 3, 4, CONJA, MODE>(p, s); break;
    case 4: launch3<128, 64, 4, 2, 3, 1, CONJA, MODE>(p, s); break;
    case 5: launch3<32, 64, 2, 2, 4, 2, CONJA, MODE>(p, s); break;
    case 6: launch3<32, 32, 2, 2, 3, 2, CONJA, MODE, true, 32>(p, s); break;   // BK = 32
    case 7: launch3<32, 32, 2, 2, 4, 3, CONJA, MODE, false>(p, s); break;      // C_old read in the epilogue
    case 8: launch3<64, 64, 2, 2, 3, 2, CONJA, MODE, false>(p, s); break;      // 32x32 warp tiles
    default: launch_t<CONJA, MODE>(p, s); break;
  }
}

}  // namespace

// Algorithmic HBM bytes of one launch: op(A), B read once (once for the whole batch when the
// batch stride is 0), C read (beta != 0 or SUB) and written once.
static double zgemm_bytes(const ZgemmArgs& p, int mode) {
  const double b = p.batch;
  const bool readC = mode == ZG_SUB || p.beta.x != 0.0 || p.beta.y != 0.0;
  return 16.0 * ((p.sA ? b : 1.0) * p.M * p.K + (p.sB ? b : 1.0) * p.K * p.N +
                 b * p.M * p.N * (readC ? 2.0 : 1.0));
}

// Algorithmic flops of one launch: 8 M N K per complex GEMM; an in-place launch applies a 64x64
// TRIANGULAR inverse (L_kk^-1 or U_kk^-1) to a block, K(K+1)/2 complex multiply-adds per column,
// i.e. 4 K (K + 1) N flops (the kernel executes the dense 8 K^2 N: the zero half is not work).
static double zgemm_flops(const ZgemmArgs& p) {
  const double b = p.batch;
  if (p.inplace) return 4.0 * (double)p.K * (double)(p.K + 1) * (double)p.N * b;
  return 8.0 * (double)p.M * (double)p.N * (double)p.K * b;
}

void zgemm_launch_variant(const ZgemmArgs& p, bool conjA, int mode, int variant, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return;
  ProfScope ps_(K_ZGEMM, zgemm_flops(p), zgemm_bytes(p, mode), s);
  if (conjA) {
    if (mode == ZG_SUB) launch_variant<true, ZG_SUB>(p, variant, s); else launch_variant<true, ZG_GEN>(p, variant, s);
  } else {
    if (mode == ZG_SUB) launch_variant<false, ZG_SUB>(p, variant, s); else launch_variant<false, ZG_GEN>(p, variant, s);
  }
}

void zgemm_launch(const ZgemmArgs& p, bool conjA, int mode, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return;
  if (p.K <= 0 && mode == ZG_SUB) return;  // C -= 0
  static const int env_variant = [] {       // experiments only (FEAST_ZGEMM_VARIANT=<n>)
    const char* e = getenv("FEAST_ZGEMM_VARIANT");
    return e ? atoi(e) : 0;
  }();
  if (env_variant > 0 && !p.inplace) {
    zgemm_launch_variant(p, conjA, mode, env_variant, s);
    return;
  }
  ProfScope ps_(K_ZGEMM, zgemm_flops(p), zgemm_bytes(p, mode), s);
  if (conjA) {
    if (mode == ZG_SUB) launch_t<true, ZG_SUB>(p, s); else launch_t<true, ZG_GEN>(p, s);
  } else {
    if (mode == ZG_SUB) launch_t<false, ZG_SUB>(p, s); else launch_t<false, ZG_GEN>(p, s);
  }
}

}  // namespace feast
