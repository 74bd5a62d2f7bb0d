// panel_smem.cu — cluster panel factorisation with the panel resident in distributed shared
// memory (the latency-critical serial part of the LU).
//
// One cluster of CS CTAs per matrix factors columns [k, k+w) over rows k..n-1.  Each CTA
// holds its contiguous block of panel rows (w columns, row-major in smem) for the whole
// panel: rows are NEVER moved inside the kernel.  Partial pivoting (reading R7: argmax of
// |re|+|im|, lowest row on ties) picks, per column, the best row among the rows not yet used
// as pivots; eliminations are applied in place in the physical layout.  At the end the panel
// is stored in physical row order and the LAPACK-style ipiv (sequential swaps) is derived
// from the pivot sequence; the row-swap kernel then applies ipiv to ALL n columns (panel
// included), which yields exactly the LAPACK getrf layout.
//
// Per column: warp-shuffle argmax -> CTA argmax -> the CTA candidate (chunk row of W complex,
// |pivot|, row id) is pushed into every CTA's slot with st.async, whose bytes complete a
// transaction mbarrier in the receiving CTA -> each CTA waits on its OWN mbarrier (no
// cluster-wide barrier, no memory fence) -> identical global decision everywhere -> in-register
// rank-1 update of the W-column chunk.  Slots are double-buffered by column parity: a CTA can
// only push column c+2 after every CTA pushed column c+1, i.e. after every CTA consumed c.
// Per chunk of W columns: the chunk's W pivot rows push their remaining-panel values the same
// way, every CTA forms U12 = L11^-1 (pivot rows) and applies the rank-W update to its own
// non-pivot rows in shared memory (one smem read-modify-write per element per chunk).
#include <cooperative_groups.h>
#include <cstdlib>
#include <float.h>
#include <limits.h>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace cg = cooperative_groups;

namespace feast {
namespace {

constexpr int PT = 128;          // threads per CTA up to 256 rows (S = 1, 2 rows per thread); 2 * PT
                                 // threads for 257..512 rows (four rows per thread spill registers)
constexpr int CSM = 16;          // max cluster size
constexpr int WMAX = 64;         // max panel width

template <int WC>                 // WC = chunk width (columns held in registers)
struct __align__(16) Slot {
  double2 row[WC];
  unsigned long long key;   // pivot key (see make_key); 0 = no candidate
  unsigned long long pad;
  double2 pinv;             // 1 / pivot, computed by the candidate's owner before the exchange
};

// Pivot key: the bits of |re|+|im| (>= 0, so the IEEE pattern orders like the value) with the low
// 16 mantissa bits replaced by 0xFFFF - row: one unsigned 64-bit max picks the largest modulus
// and, among candidates equal to 2^-36 relative, the lowest row (reading R7: near-ties may be
// broken differently from the oracle; the solution Y_j agrees to kappa * u either way).
__device__ __forceinline__ unsigned long long make_key(double v, int row) {
  if (v < 0.0) return 0ull;
  return ((unsigned long long)__double_as_longlong(v) & ~0xFFFFull) | (unsigned long long)(0xFFFF - row);
}
__device__ __forceinline__ int key_row(unsigned long long k) { return 0xFFFF - (int)(k & 0xFFFFull); }
// warp-wide unsigned 64-bit max with two 32-bit REDUX operations
__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k) {
  const unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}

// 1/x for 1e-300 < x < 1e300: MUFU.RCP64H seed + two Newton steps (~1 ulp; __drcp_rn's correctly
// rounded sequence costs ~400 cycles on the per-column critical path)
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Smith's complex reciprocal for extreme magnitudes, kept out of line (it is never on the fast
// path, and inlined into every unrolled column step it only costs instruction-cache space)
__device__ __noinline__ double2 crcp_slow(double2 b) { return crcp(b); }

__device__ __forceinline__ bool better(double v, int i, double bv, int bi) {
  return v > bv || (v == bv && i < bi);
}
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async16(uint32_t raddr, double2 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
               ::"r"(raddr), "l"(__double_as_longlong(v.x)), "l"(__double_as_longlong(v.y)), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arm(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  }
}

#ifdef FEAST_PANEL_TRACE
__device__ unsigned long long g_ptrace[512];
#define PTRACE(i) do { if (blockIdx.x == 0 && threadIdx.x == 0 && k == 0) { unsigned long long t_; \
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_ptrace[(i)] = t_; } } while (0)
__device__ unsigned long long g_ctrace[2][16];
#define CT(i) do { if (ctr) { const long long t_ = clock64(); ct_[i] += t_ - ct_prev; ct_prev = t_; } } while (0)
#else
#define PTRACE(i) do {} while (0)
#define CT(i) do {} while (0)
#endif

template <int S, int WC, int NT, bool CLU>   // CLU: cluster of > 1 CTAs (else the single-CTA path)
__global__ void __launch_bounds__(NT, 1)
panel_smem_kernel(Batched Cb, int64_t n, int64_t k, int w, int64_t sc0, int64_t sc1, int32_t* __restrict__ ipiv_all,
                  double* __restrict__ stats_all, int32_t* __restrict__ info_all) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;
  double2* __restrict__ C = Cb.p + (int64_t)b * Cb.stride + k + k * Cb.ld;  // panel origin
  const int64_t ld = Cb.ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = (int)(n - k);
  const int Lc = (L + CS - 1) / CS;
  const int rbeg = crank * Lc;
  const int nrow = max(0, min(L, rbeg + Lc) - rbeg);
  const int PLD = Lc;   // column-major smem panel: P[(c - WC) * PLD + r] (consecutive rows -> conflict-free)

  // Shared memory holds only the panel columns [WC, w): the first chunk lives in registers from
  // the start, and every finished chunk is stored straight from registers to global memory, so
  // the footprint (and the number of co-resident clusters) is set by w - WC columns.
  extern __shared__ __align__(128) double2 P[];  // [w - WC][PLD]
  constexpr int SLOT_BYTES = (WC + 2) * 16;
  __shared__ Slot<WC> slots[2][CSM];
  __shared__ double2 L11s[WC][WC];               // chunk pivot rows' chunk values
  __shared__ __align__(16) double2 U12s[WC][WMAX];   // chunk pivot rows' rest-of-panel values
  __shared__ int pvt[WMAX];                      // pivot (panel row index) per column
  // per-warp candidates, double-buffered by column parity (a single-CTA "cluster" decides the
  // pivot straight from them: one __syncthreads per column, no DSMEM exchange)
  __shared__ __align__(16) unsigned long long wkey[2][NT / 32];
  __shared__ double2 wrow[2][NT / 32][WC + 1];
  __shared__ __align__(8) unsigned long long mbar[4];   // slots[0], slots[1], U12s, load
  __shared__ int pos2row[WMAX], cur[WMAX];
  __shared__ int32_t lpiv[WMAX];                 // this panel's LAPACK ipiv (absolute rows)

  PTRACE(0);
#ifdef FEAST_PANEL_TRACE
  const bool ctr = blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 96) && k == 0;
  long long ct_[16] = {0}, ct_prev = clock64();
#endif
  if (tid == 0) {
    mbar_init(saddr(&mbar[0]), 1);
    mbar_init(saddr(&mbar[1]), 1);
    mbar_init(saddr(&mbar[2]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- load own rows of the panel: one bulk (TMA) copy per column segment into the
  // column-major shared layout P[c][r], completing a local transaction mbarrier
  const uint32_t lbar = saddr(&mbar[3]);
  if (tid == 0) {
    mbar_init(lbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool tma = nrow > 0 && w > WC;
  if (tma) {
    if (tid == 0) mbar_arm(lbar, (uint32_t)((w - WC) * nrow * 16));
    for (int c = WC + tid; c < w; c += NT) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(saddr(P + (c - WC) * PLD)), "l"(C + rbeg + c * ld), "r"(nrow * 16), "r"(lbar) : "memory");
    }
  }
  // first chunk: straight from global into registers (coalesced: consecutive threads, rows)
  double2 a[S][WC];
  {
    const int wc0 = min(WC, w);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int r = tid + s * NT;
      const double2* src = C + rbeg + r;   // advanced by ld per column (no 64-bit products)
#pragma unroll
      for (int jj = 0; jj < WC; ++jj) {
        a[s][jj] = (r < nrow && jj < wc0) ? *src : make_double2(0.0, 0.0);
        src += ld;
      }
    }
  }
  cluster.sync();   // mbarrier inits visible cluster-wide before any remote st.async
  // this thread's slot elements of the per-column push (fixed for the whole panel): element e of
  // CTA dcta's slot [buf][crank] and dcta's mbarrier [buf], t = tid (+ NT) = dcta * (WC + 2) + e
  static_assert(CSM * (WC + 2) <= 2 * NT, "push covers at most two elements per thread");
  int push_e[2];
  uint32_t push_slot[2][2], push_bar[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = h * NT + tid;
    const int dcta = min(t / (WC + 2), CS - 1);
    push_e[h] = t - (t / (WC + 2)) * (WC + 2);
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      push_slot[h][bb] = mapa(saddr(&slots[bb][crank]), dcta) + push_e[h] * 16;
      push_bar[h][bb] = mapa(saddr(&mbar[bb]), dcta);
    }
  }
  if (tma) mbar_wait(lbar, 0);
  PTRACE(1);

  bool used[S];
#pragma unroll
  for (int s = 0; s < S; ++s) used[s] = false;
  double pmin = DBL_MAX, pmax = 0.0;
  int info = 0;
  int chunk = 0;

  for (int j0 = 0; j0 < w; j0 += WC, ++chunk) {
    const int wc = min(WC, w - j0);
    if (j0 > 0) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int r = tid + s * NT;
#pragma unroll
        for (int jj = 0; jj < WC; ++jj)
          a[s][jj] = (r < nrow && jj < wc) ? P[(j0 - WC + jj) * PLD + r] : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int jj = 0; jj < WC; ++jj) {
      if (jj >= wc) break;
      const int col = j0 + jj;
      const int buf = col & 1;
      const uint32_t bar = saddr(&mbar[buf]);
      PTRACE(8 + 4 * col);
      CT(0);
      if (tid == 0 && CLU) mbar_arm(bar, (uint32_t)(CS * SLOT_BYTES));
      unsigned long long bk = 0ull;
      int bs = -1;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int r = tid + s * NT;
        if (r < nrow && !used[s]) {
          const unsigned long long kk = make_key(cabs1(a[s][jj]), rbeg + r);
          if (kk > bk) { bk = kk; bs = s; }
        }
      }
      CT(1);
      // warp argmax first (the REDUX issues before the reciprocal's dependent chain), then every
      // thread inverts its own candidate while the reduction is in flight
      const unsigned long long wk = warp_max_key(bk);
      CT(2);
      // the candidate value by predicated selects (no divergent branch per row slot), then ONE
      // reciprocal chain per lane: 1/p = conj(p) / |p|^2
      double2 pv = make_double2(0.0, 0.0);
#pragma unroll
      for (int s = 0; s < S; ++s)
        if (s == bs) pv = a[s][jj];
      const double m2 = fma(pv.x, pv.x, pv.y * pv.y);
      double2 myrcp;
      if (m2 > 1e-300 && m2 < 1e300) {
        const double d = fast_rcp(m2);
        myrcp = make_double2(pv.x * d, -pv.y * d);
      } else {
        myrcp = (pv.x != 0.0 || pv.y != 0.0) ? crcp_slow(pv) : make_double2(0.0, 0.0);   // extreme magnitudes
      }
      CT(3);
      // the warp's winning lane stages its chunk row and 1/pivot; one barrier for the CTA step
      if (wk != 0ull && bk == wk) {
#pragma unroll
        for (int q = 0; q < WC; ++q) {
          double2 v = a[0][q];
#pragma unroll
          for (int s = 1; s < S; ++s)
            if (s == bs) v = a[s][q];
          wrow[buf][warp][q] = v;
        }
        wrow[buf][warp][WC] = myrcp;
      }
      if (lane == 0) wkey[buf][warp] = wk;
      CT(4);
      __syncthreads();
      CT(5);
      // CTA argmax of the NT/32 warp keys (16-byte loads; keys are distinct or 0)
      unsigned long long ck = 0ull;
      int cw = 0;
#pragma unroll
      for (int q = 0; q < NT / 32; q += 2) {
        const ulonglong2 kk = *reinterpret_cast<const ulonglong2*>(&wkey[buf][q]);
        if (kk.x > ck) { ck = kk.x; cw = q; }
        if (kk.y > ck) { ck = kk.y; cw = q + 1; }
      }
      PTRACE(9 + 4 * col);
      CT(6);
      unsigned long long gk;
      const double2* prow;
      double2 pinv;
      if (!CLU) {
        // single CTA: the CTA winner is the pivot
        gk = ck;
        prow = wrow[buf][cw];
        pinv = wrow[buf][cw][WC];
      } else {
        // push {row[WC], key, 1/pivot} into slot [buf][crank] of every CTA (st.async -> its mbarrier)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h * NT + tid >= CS * (WC + 2)) break;
          const int e = push_e[h];
          double2 v;
          if (e < WC) v = ck ? wrow[buf][cw][e] : make_double2(0.0, 0.0);
          else if (e == WC) v = make_double2(__longlong_as_double((long long)ck), 0.0);
          else v = ck ? wrow[buf][cw][WC] : make_double2(0.0, 0.0);
          st_async16(push_slot[h][buf], v, push_bar[h][buf]);
        }
        CT(7);
        mbar_wait(bar, (uint32_t)((col >> 1) & 1));
        CT(8);
        PTRACE(10 + 4 * col);
        // global pivot: lanes read the CS keys, 64-bit max by REDUX (every warp, same result)
        const unsigned long long lk = lane < CS ? slots[buf][lane].key : 0ull;
        gk = warp_max_key(lk);
        const int gb = __ffs(__ballot_sync(0xffffffffu, lane < CS && lk == gk)) - 1;
        prow = slots[buf][gb].row;
        pinv = slots[buf][gb].pinv;
      }
      CT(9);
      const int gi = key_row(gk);
      if (tid < WC) L11s[jj][tid] = prow[tid];
      if (tid == 0) pvt[col] = gi;
      const double2 p = prow[jj];
      const bool pzero = (p.x == 0.0 && p.y == 0.0);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int r = tid + s * NT;
        if (r < nrow && !used[s]) {
          if (rbeg + r == gi) {
            used[s] = true;   // pivot row: its values are U (cols >= col) and L (cols < col)
          } else {
            const double2 l = cmul(a[s][jj], pinv);
            a[s][jj] = l;
#pragma unroll
            for (int q = jj + 1; q < WC; ++q) a[s][q] = cfms(a[s][q], l, prow[q]);
          }
        }
      }
      CT(10);
      if (crank == 0 && tid == 0) {
        const double ap2 = fma(p.x, p.x, p.y * p.y);   // |p|^2; sqrt taken once at the end
        pmin = fmin(pmin, ap2);
        pmax = fmax(pmax, ap2);
        if (pzero && !info) info = (int)(k + col + 1);
      }
    }
    // ---- chunk done: its columns are final (L multipliers; U for the pivot rows) -> global
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int r = tid + s * NT;
      if (r < nrow) {
        double2* dst = C + rbeg + r + (int64_t)j0 * ld;
#pragma unroll
        for (int jj = 0; jj < WC; ++jj) {
          if (jj < wc) *dst = a[s][jj];
          dst += ld;
        }
      }
    }
    CT(11);
    const int c1 = j0 + wc;
    if (c1 < w) {
      const int rem = w - c1;
      const uint32_t ubar = saddr(&mbar[2]);
      if (tid == 0 && CLU) mbar_arm(ubar, (uint32_t)(wc * rem * 16));
      __syncthreads();
      // owners push the chunk pivot rows' rest-of-panel values to every CTA (single CTA: plain
      // shared-memory copies and a barrier)
      for (int jj = 0; jj < wc; ++jj) {
        const int pr = pvt[j0 + jj] - rbeg;
        if (pr >= 0 && pr < nrow) {
          for (int idx = tid; idx < rem * CS; idx += NT) {
            const int dcta = idx / rem, c = idx - dcta * rem;
            if (!CLU) U12s[jj][c] = P[(c1 - WC + c) * PLD + pr];
            else st_async16(mapa(saddr(&U12s[jj][c]), dcta), P[(c1 - WC + c) * PLD + pr], mapa(ubar, dcta));
          }
        }
      }
      PTRACE(300 + 4 * chunk);
      if (!CLU) __syncthreads();
      else mbar_wait(ubar, (uint32_t)(chunk & 1));
      CT(12);
      PTRACE(301 + 4 * chunk);
      // U12 = L11^-1 (pivot rows), unit lower L11 (chunk multipliers of the pivot rows)
      for (int c = tid; c < rem; c += NT) {
        double2 u[WC];
#pragma unroll
        for (int jj = 0; jj < WC; ++jj) {
          if (jj < wc) {
            double2 v = U12s[jj][c];
#pragma unroll
            for (int t = 0; t < jj; ++t) v = cfms(v, L11s[jj][t], u[t]);
            u[jj] = v;
            U12s[jj][c] = v;
          }
        }
      }
      PTRACE(303 + 4 * chunk);
      __syncthreads();
      CT(13);
      // pivot rows of this chunk take their U12 values; other rows get the rank-wc update
      for (int jj = 0; jj < wc; ++jj) {
        const int pr = pvt[j0 + jj] - rbeg;
        if (pr >= 0 && pr < nrow)
          for (int c = tid; c < rem; c += NT) P[(c1 - WC + c) * PLD + pr] = U12s[jj][c];
      }
      // rank-wc update of this thread's S rows, all rows in one pass: each U12 value (a
      // shared-memory broadcast) feeds S rows, and S x 8 independent accumulation chains keep
      // the FP64 pipe busy with one warp per SM sub-partition.  Pivot rows (used) and rows past
      // nrow are computed on zeros and not stored.
      {
        bool act[S];
        int rr[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          rr[s] = tid + s * NT;
          act[s] = rr[s] < nrow && !used[s];
        }
        double2* colp = P + (c1 - WC) * PLD;
        constexpr int CH = 8;
        int c = 0;
        for (; c + CH <= rem; c += CH) {
          double2 v[S][CH];
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int e = 0; e < CH; ++e) v[s][e] = act[s] ? colp[(c + e) * PLD + rr[s]] : make_double2(0.0, 0.0);
#pragma unroll
          for (int jj = 0; jj < WC; ++jj)
            if (jj < wc) {
#pragma unroll
              for (int e = 0; e < CH; ++e) {
                const double2 u = U12s[jj][c + e];
#pragma unroll
                for (int s = 0; s < S; ++s) v[s][e] = cfms(v[s][e], a[s][jj], u);
              }
            }
#pragma unroll
          for (int s = 0; s < S; ++s)
            if (act[s]) {
#pragma unroll
              for (int e = 0; e < CH; ++e) colp[(c + e) * PLD + rr[s]] = v[s][e];
            }
        }
        for (; c < rem; ++c) {
#pragma unroll
          for (int s = 0; s < S; ++s)
            if (act[s]) {
              double2 v = colp[c * PLD + rr[s]];
#pragma unroll
              for (int jj = 0; jj < WC; ++jj)
                if (jj < wc) v = cfms(v, a[s][jj], U12s[jj][c]);
              colp[c * PLD + rr[s]] = v;
            }
        }
      }
      CT(14);
      __syncthreads();
      CT(15);
      PTRACE(302 + 4 * chunk);
      if (chunk == 0) PTRACE(400);
    }
  }
  PTRACE(2);
#ifdef FEAST_PANEL_TRACE
  if (ctr)
    for (int i = 0; i < 16; ++i) g_ctrace[threadIdx.x == 0 ? 0 : 1][i] = (unsigned long long)ct_[i];
#endif
  // ---- LAPACK ipiv from the pivot sequence (rows / positions relative to k): every CTA derives
  // it (the pivot sequence pvt is identical in all of them); CTA 0 publishes it
  if (tid == 0) {
    for (int i = 0; i < w; ++i) { pos2row[i] = i; cur[i] = i; }
    int32_t* ipiv = ipiv_all + (int64_t)b * n + k;
    for (int col = 0; col < w; ++col) {
      const int p = pvt[col];
      const int lp = p < w ? cur[p] : p;
      const int rc = pos2row[col];
      lpiv[col] = (int32_t)(k + lp);
      if (crank == 0) ipiv[col] = (int32_t)(k + lp);
      if (lp < w) pos2row[lp] = rc;
      if (rc < w) cur[rc] = lp;
      pos2row[col] = p;
      if (p < w) cur[p] = col;
    }
    if (crank == 0) {
      stats_all[2 * b] = fmin(stats_all[2 * b], sqrt(pmin));
      stats_all[2 * b + 1] = fmax(stats_all[2 * b + 1], sqrt(pmax));
      if (info && !info_all[b]) info_all[b] = info;
    }
  }
  PTRACE(3);
  // ---- fused row swaps (sc0 < sc1): the panel's w sequential swaps applied to the columns
  // [sc0, sc1) of the outer block (the panel's own columns included: rows never moved inside the
  // kernel), one column per thread of the cluster — replaces a separate swap launch on the
  // panel chain.  The cluster barrier (release / acquire) makes every CTA's panel stores visible.
  if (sc1 > sc0) {
    if (CLU) cluster.sync(); else __syncthreads();
    double2* Cm = Cb.p + (int64_t)b * Cb.stride;
    for (int64_t col = sc0 + (int64_t)crank * NT + tid; col < sc1; col += (int64_t)CS * NT) {
      double2* Cc = Cm + col * ld;
      for (int i = 0; i < w; ++i) {
        const int64_t r1 = k + i, r2 = lpiv[i];
        if (r1 != r2) {
          const double2 t0 = Cc[r1];
          Cc[r1] = Cc[r2];
          Cc[r2] = t0;
        }
      }
    }
  }
  // No further cluster barrier: every remote write into this CTA's shared memory was a st.async
  // that this CTA waited for (the last column's slots), so it may exit.
}

template <int S, int WC, int NT>
void launch_s(Batched C, int64_t n, int64_t k, int w, int64_t sc0, int64_t sc1, int32_t* ipiv, double* stats,
              int32_t* info, int batch, int cs, cudaStream_t s) {
  const int64_t L = n - k;
  const int Lc = (int)((L + cs - 1) / cs);
  const size_t smem = (size_t)Lc * (w > WC ? w - WC : 0) * sizeof(double2);
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured)) {
    cudaFuncSetAttribute(panel_smem_kernel<S, WC, NT, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(panel_smem_kernel<S, WC, NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(panel_smem_kernel<S, WC, NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * cs), 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cs > 1) cudaLaunchKernelEx(&cfg, panel_smem_kernel<S, WC, NT, true>, C, n, k, w, sc0, sc1, ipiv, stats, info);
  else cudaLaunchKernelEx(&cfg, panel_smem_kernel<S, WC, NT, false>, C, n, k, w, sc0, sc1, ipiv, stats, info);
  count_launch();
}

}  // namespace

#ifdef FEAST_PANEL_TRACE
void panel_trace_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_ptrace, sizeof(g_ptrace)); }
void panel_ctrace_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_ctrace, sizeof(g_ctrace)); }
#endif

// Diagnostics: how many clusters of `cs` CTAs with the panel of L rows x w columns can be
// co-resident (cudaOccupancyMaxActiveClusters); decides whether a batch needs several waves.
int panel_smem_max_clusters(int64_t L, int w, int cs) {
  const int Lc = (int)((L + cs - 1) / cs);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(16 * cs), 1, 1);
  cfg.blockDim = dim3(Lc <= 2 * PT ? PT : (Lc <= 4 * PT || tall_variant() != 2 ? 2 * PT : 4 * PT), 1, 1);
  const int wc = 8;
  cfg.dynamicSmemBytes = (size_t)Lc * (w > wc ? w - wc : 0) * sizeof(double2);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nc = -1;
  const bool v5 = Lc > 4 * PT && tall_variant() == 5;
  if (v5) cfg.dynamicSmemBytes = (size_t)Lc * (w > 4 ? w - 4 : 0) * sizeof(double2);
  auto k = Lc <= PT ? panel_smem_kernel<1, 8, PT, true>
                    : (Lc <= 2 * PT ? panel_smem_kernel<2, 8, PT, true>
                                    : (Lc <= 4 * PT ? panel_smem_kernel<2, 8, 2 * PT, true>
                                                    : (tall_variant() == 2 ? panel_smem_kernel<2, 8, 4 * PT, true>
                                                                           : (v5 ? panel_smem_kernel<4, 4, 2 * PT, true>
                                                                                 : panel_smem_kernel<4, 8, 2 * PT, true>))));
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (cudaOccupancyMaxActiveClusters(&nc, k, &cfg) != cudaSuccess) { cudaGetLastError(); return -1; }
  return nc;
}

// FEAST_TALL_VARIANT for panels of 513..1024 rows per CTA: 5 (default) = 256 threads x 4 rows with
// a 4-column register chunk (no spill; 16-wide panel of 16384 rows 64.6 -> 50.6 us, C4 12.800 ->
// 12.753 s), 4 = 256 threads x 4 rows with the 8-column chunk (spills ~2 KB), 2 = 512 threads x 2
// rows; 0 = keep those panels on the register-chunk kernel (lu.cu)
// Panels of 1025..2048 rows per CTA (n - k up to 32768: C5's first half) on the cluster kernel
// too — 8 wide, 256 threads x 8 rows with a 4-column register chunk and the other 4 columns in
// shared memory (128 KB; ptxas spills ~4.7 KB at 255 registers, still far faster than the
// register-chunk kernel's ~23 us per column): C5 47.64 -> 47.06 s.  FEAST_VTALL=0: the
// register-chunk kernel (lu.cu) beyond 1024 rows per CTA.
bool very_tall_panels() {
  const char* e = getenv("FEAST_VTALL");
  return !e || e[0] != '0';
}

int tall_variant() {   // read per call (a getenv per panel launch): tests switch it per handle
  const char* e = getenv("FEAST_TALL_VARIANT");
  return e ? atoi(e) : 5;
}

bool panel_smem_fits(int64_t n, int w, int cs) {
  const int64_t Lc = (n + cs - 1) / cs;
  const int wc = 8;   // register chunk width (see panel_smem_launch)
  return w <= WMAX && (size_t)Lc * (w > wc ? w - wc : 0) * sizeof(double2) <= 190 * 1024 && Lc <= 8 * PT;
}

void panel_smem_launch(Batched C, int64_t n, int64_t k, int w, int32_t* ipiv, double* stats, int32_t* info, int batch,
                       int cs, cudaStream_t s,
                       bool one_row, int64_t sc0, int64_t sc1) {
  const double L_ = (double)(n - k);
  ProfScope ps_(K_PANEL, (double)batch * (4.0 * L_ * w * w - 4.0 * w * (double)w * w / 3.0), 0.0, s);
  // Shrink the cluster as the panel gets shorter (L = n - k): the smallest cluster that keeps
  // <= 2*PT rows per CTA.  Fewer CTAs per column exchange (cs = 1: no DSMEM at all) and fewer SMs
  // held while the latency-bound panel runs next to the trailing-update GEMMs.
  // rows per CTA: <= 2 PT (two per thread) for panels up to 32 wide; <= PT for wider ones so the
  // w - 8 shared-memory columns stay within ~112 KB
  int rowcap = w > 32 ? PT : 2 * PT;
  // FEAST_PANEL_ROWS: a larger row cap (fewer CTAs per panel cluster, e.g. 512 rows = 4 CTAs for a
  // 2048-row panel) where the w - 8 shared-memory columns still fit
  static const int rows_env = [] { const char* e = getenv("FEAST_PANEL_ROWS"); return e ? atoi(e) : 0; }();
  if (rows_env > rowcap && rows_env <= 8 * PT && (size_t)rows_env * (w > 8 ? w - 8 : 0) * 16 <= 190 * 1024)
    rowcap = rows_env;
  while (cs > 1 && (n - k + cs / 2 - 1) / (cs / 2) <= rowcap) cs /= 2;
  const int64_t Lc = (n - k + cs - 1) / cs;
  // register chunk: 8 columns (a 16-column chunk spills at 2 rows per thread)
  // one_row: 129..256 rows per CTA on 256 threads x 1 row (8 warps, faster
  // per column and in the chunk-end update, but the CTA takes most of the register file, so no
  // trailing-update GEMM CTA shares its SM): chosen by the caller when few nodes are factored
  // and the panel chain, not GEMM throughput, bounds the step
  if (Lc <= PT) launch_s<1, 8, PT>(C, n, k, w, sc0, sc1, ipiv, stats, info, batch, cs, s);
  else if (Lc <= 2 * PT && one_row) launch_s<1, 8, 2 * PT>(C, n, k, w, sc0, sc1, ipiv, stats, info, batch, cs, s);
  else if (Lc <= 2 * PT) launch_s<2, 8, PT>(C, n, k, w, sc0, sc1, ipiv, stats, info, batch, cs, s);
  else if (Lc <= 4 * PT) launch_s<2, 8, 2 * PT>(C, n, k, w, sc0, sc1, ipiv, stats, info, batch, cs, s);   // 512 rows: 256 x 2
  // 513..1024 rows per CTA (tall panels of n = 16384, w <= 16 so the w - 8 shared columns fit):
  // 256 threads x 4 rows (registers capped at 255) or 512 threads x 2 rows (capped at 128)
  else if (Lc > 8 * PT) launch_s<8, 4, 2 * PT>(C, n, k, w, sc0, sc1, ipiv, stats, info, batch, cs, s);   // very tall
  else if (tall_variant() == 2) launch_s<2, 8, 4 * PT>(C, n, k, w, sc0, sc1, ipiv, stats, info, batch, cs, s);
  // 5: 256 threads x 4 rows with a 4-column register chunk (254 registers, no spill; the w - 4
  // shared-memory columns take 192 KB at 1024 rows x 16 columns)
  else if (tall_variant() == 5) launch_s<4, 4, 2 * PT>(C, n, k, w, sc0, sc1, ipiv, stats, info, batch, cs, s);
  else launch_s<4, 8, 2 * PT>(C, n, k, w, sc0, sc1, ipiv, stats, info, batch, cs, s);
}

}  // namespace feast
