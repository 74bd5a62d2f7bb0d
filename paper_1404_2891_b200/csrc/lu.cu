// lu.cu — node shift, blocked LU pieces (cluster panel with pivot search, row swaps,
// triangular blocks), permutations, fused weighted accumulation and small iteration helpers.
//
// Paper: eq. Rasp needs, at every pole z_j, the solve (z_j B - A)^{-1} (B X);
// the paper used a sparse direct solver (MKL Pardiso).  Here the pencils are dense
// (BASELINE configs), so each shifted matrix gets a dense right-looking blocked LU with
// partial pivoting (reading R7: pivot = argmax |re|+|im|, lowest row on ties), batched
// across the nodes a rank owns (parallelism over the linear systems).
#include <cooperative_groups.h>
#include <float.h>
#include <cstdlib>
#include <limits.h>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace cg = cooperative_groups;

namespace feast {
thread_local int64_t g_launches = 0;
Prof& prof() {
  static thread_local Prof p;
  return p;
}

// ============================================================================ shift
// C_b = z_b B - A  (HBM-bound).  One thread per element of A for the whole batch: A
// and B are read once per element and the batch's C_b written from registers, so a group of
// nodes costs 32 + 16 * batch bytes per element instead of 48 * batch (A + B = 134 MB at
// n = 2048 do not stay in the 126 MB L2 between per-node passes).
__global__ void shift_kernel(Batched C, const double2* __restrict__ A, int64_t lda,
                             const double2* __restrict__ B, int64_t ldb, const double2* __restrict__ z,
                             int64_t n, int64_t c0, int batch) {
  const int64_t col = c0 + blockIdx.y;
  const double2* Ac = A + col * lda;
  const double2* Bc = B ? B + col * ldb : nullptr;
  double2* Cc = C.p + col * C.ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = Ac[i];
    const double2 bv = Bc ? Bc[i] : make_double2(i == col ? 1.0 : 0.0, 0.0);
    for (int b = 0; b < batch; ++b) Cc[b * C.stride + i] = csub(cmul(z[b], bv), a);
  }
}

void shift_launch(Batched C, const double2* A, int64_t lda, const double2* B, int64_t ldb,
                  const double2* z, int64_t n, int batch, cudaStream_t s, int64_t c0, int64_t c1) {
  if (c1 < 0) c1 = n;
  if (c1 <= c0) return;
  ProfScope ps_(K_SHIFT, 0.0, (double)(c1 - c0) * n * 16.0 * ((B ? 2 : 1) + batch), s);
  const int threads = 256;
  unsigned gx = (unsigned)((n + threads - 1) / threads);
  if (gx > 8) gx = 8;
  dim3 grid(gx, (unsigned)(c1 - c0), 1);
  shift_kernel<<<grid, threads, 0, s>>>(C, A, lda, B, ldb, z, n, c0, batch);
  count_launch();
}

// ============================================================================ panel
// One thread-block CLUSTER per matrix factors the panel of columns [k, k+w).
// Rows k..n-1 are split into CS contiguous ranges, one per CTA; thread t of a CTA owns
// rows rbeg + s*T + t (s < S) and keeps the current chunk of W columns of those rows in
// registers.  Per column: thread-local candidate -> warp-shuffle argmax -> CTA argmax ->
// the owner thread pushes (|pivot|, row, the pivot row's W values) into every CTA's shared
// memory (DSMEM); the diagonal row's owner pushes the diagonal row; ONE cluster barrier;
// every CTA then picks the same global pivot and updates its own rows (swap, scale,
// rank-1 update inside the chunk).  Between chunks: CTA 0 applies the chunk's swaps to the
// panel's other columns and forms the chunk's U rows (unit-lower solve); every CTA then
// updates its own rows of the rest of the panel.  Candidate slots are double-buffered by
// column parity, so one cluster barrier per column suffices.
namespace {
constexpr int PANEL_T = 256;
constexpr int CS_MAX = 16;
constexpr int NB_MAX = 64;

template <int W>
struct __align__(16) PivSlot {
  double2 row[W];
  double val;
  int idx;
  int pad;
};

__device__ __forceinline__ bool better(double v, int i, double bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

template <int W, int S>
__global__ void __launch_bounds__(PANEL_T, 1)
panel_kernel(Batched Cb, int64_t n, int64_t k, int w, int32_t* __restrict__ ipiv_all,
             double* __restrict__ stats_all, int32_t* __restrict__ info_all) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;
  double2* __restrict__ C = Cb.p + (int64_t)b * Cb.stride;
  const int64_t ld = Cb.ld;
  int32_t* __restrict__ ipiv = ipiv_all + (int64_t)b * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = (int)(n - k);
  const int Lc = (L + CS - 1) / CS;
  const int rbeg = crank * Lc;
  const int rend = min(L, rbeg + Lc);

  __shared__ PivSlot<W> slots[2][CS_MAX];
  __shared__ double2 diag[2][W];
  __shared__ double wv[PANEL_T / 32];
  __shared__ int wi[PANEL_T / 32];
  __shared__ double2 u12s[W][NB_MAX];

  double2 a[S][W];
  double pmin = DBL_MAX, pmax = 0.0;
  int info = 0;

  for (int j0 = 0; j0 < w; j0 += W) {
    const int wc = min(W, w - j0);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = rbeg + s * PANEL_T + tid;
#pragma unroll
      for (int jj = 0; jj < W; ++jj)
        a[s][jj] = (i < rend && i >= j0 && jj < wc) ? C[(k + i) + (k + j0 + jj) * ld] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int jj = 0; jj < W; ++jj) {
      if (jj >= wc) break;
      const int col = j0 + jj;
      const int buf = col & 1;
      // ---- thread / warp / CTA argmax of |re|+|im| over rows >= col
      double bv = -1.0;
      int bi = INT_MAX;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = rbeg + s * PANEL_T + tid;
        if (i < rend && i >= col) {
          const double v = cabs1(a[s][jj]);
          if (better(v, i, bv, bi)) { bv = v; bi = i; }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { wv[warp] = bv; wi[warp] = bi; }
      __syncthreads();
      double cv = wv[0];
      int ci = wi[0];
#pragma unroll
      for (int q = 1; q < PANEL_T / 32; ++q)
        if (better(wv[q], wi[q], cv, ci)) { cv = wv[q]; ci = wi[q]; }
      // ---- publish the CTA candidate and the diagonal row to every CTA of the cluster
      if (cv < 0.0) {
        if (tid < CS) {
          PivSlot<W>* r = cluster.map_shared_rank(&slots[buf][crank], tid);
          r->val = -1.0;
          r->idx = INT_MAX;
        }
      } else {
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const int i = rbeg + s * PANEL_T + tid;
          if (i == ci) {
            for (int d = 0; d < CS; ++d) {
              PivSlot<W>* r = cluster.map_shared_rank(&slots[buf][crank], d);
#pragma unroll
              for (int q = 0; q < W; ++q) r->row[q] = a[s][q];
              r->val = cv;
              r->idx = ci;
            }
          }
        }
      }
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = rbeg + s * PANEL_T + tid;
        if (i == col && i < rend) {
          for (int d = 0; d < CS; ++d) {
            double2* r = cluster.map_shared_rank(&diag[buf][0], d);
#pragma unroll
            for (int q = 0; q < W; ++q) r[q] = a[s][q];
          }
        }
      }
      cluster.sync();
      // ---- global pivot (identical decision in every CTA)
      int gb = 0;
      double gv = slots[buf][0].val;
      int gi = slots[buf][0].idx;
      for (int c = 1; c < CS; ++c) {
        const double v = slots[buf][c].val;
        const int i = slots[buf][c].idx;
        if (better(v, i, gv, gi)) { gv = v; gi = i; gb = c; }
      }
      const double2* prow = slots[buf][gb].row;
      const double2 p = prow[jj];
      const bool pzero = (p.x == 0.0 && p.y == 0.0);
      const double2 pinv = pzero ? make_double2(0.0, 0.0) : crcp(p);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = rbeg + s * PANEL_T + tid;
        if (i < rend && i >= col) {
          if (i == col) {
#pragma unroll
            for (int q = 0; q < W; ++q) a[s][q] = prow[q];
          } else {
            if (i == gi) {
#pragma unroll
              for (int q = 0; q < W; ++q) a[s][q] = diag[buf][q];
            }
            const double2 l = cmul(a[s][jj], pinv);
            a[s][jj] = l;
#pragma unroll
            for (int q = jj + 1; q < W; ++q) a[s][q] = cfms(a[s][q], l, prow[q]);
          }
        }
      }
      if (crank == 0 && tid == 0) {
        ipiv[k + col] = (int32_t)(k + gi);
        const double ap = hypot(p.x, p.y);
        pmin = fmin(pmin, ap);
        pmax = fmax(pmax, ap);
        if (pzero && !info) info = (int)(k + col + 1);
      }
    }
    // ---- store the factored chunk
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = rbeg + s * PANEL_T + tid;
      if (i < rend && i >= j0) {
#pragma unroll
        for (int jj = 0; jj < W; ++jj)
          if (jj < wc) C[(k + i) + (k + j0 + jj) * ld] = a[s][jj];
      }
    }
    const int c1 = j0 + wc;  // first panel column right of the chunk
    if (c1 < w || j0 > 0) {
      cluster.sync();
      if (crank == 0) {
        // swaps of this chunk applied to panel columns outside it (left: L part, right: rest)
        for (int jj = 0; jj < wc; ++jj) {
          const int64_t r1 = k + j0 + jj, r2 = ipiv[k + j0 + jj];
          if (r1 != r2) {
            for (int c = tid; c < w; c += PANEL_T) {
              if (c >= j0 && c < c1) continue;
              double2* col = C + (k + c) * ld;
              const double2 t1 = col[r1];
              col[r1] = col[r2];
              col[r2] = t1;
            }
          }
          __syncthreads();
        }
        // U rows of the chunk over the rest of the panel: unit-lower solve with L11
        for (int c = c1 + tid; c < w; c += PANEL_T) {
          double2 x[W];
          double2* col = C + (k + c) * ld + (k + j0);
#pragma unroll
          for (int jj = 0; jj < W; ++jj) {
            if (jj < wc) {
              double2 v = col[jj];
#pragma unroll
              for (int q = 0; q < jj; ++q) v = cfms(v, C[(k + j0 + jj) + (k + j0 + q) * ld], x[q]);
              x[jj] = v;
              col[jj] = v;
            }
          }
        }
      }
      if (c1 < w) {
        cluster.sync();
        const int rem = w - c1;
        for (int idx = tid; idx < wc * rem; idx += PANEL_T) {
          const int jj = idx % wc, c = idx / wc;
          u12s[jj][c] = C[(k + j0 + jj) + (k + c1 + c) * ld];
        }
        __syncthreads();
        // rest of the panel, own rows below the chunk: A22 -= L21 U12
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const int i = rbeg + s * PANEL_T + tid;
          if (i < rend && i >= c1) {
            for (int c = 0; c < rem; ++c) {
              double2* ptr = C + (k + i) + (k + c1 + c) * ld;
              double2 v = *ptr;
#pragma unroll
              for (int jj = 0; jj < W; ++jj)
                if (jj < wc) v = cfms(v, a[s][jj], u12s[jj][c]);
              *ptr = v;
            }
          }
        }
        __syncthreads();
      }
    }
  }
  if (crank == 0 && tid == 0) {
    stats_all[2 * b] = fmin(stats_all[2 * b], pmin);
    stats_all[2 * b + 1] = fmax(stats_all[2 * b + 1], pmax);
    if (info && !info_all[b]) info_all[b] = info;
  }
}

template <int W, int S>
void panel_launch_t(Batched C, int64_t n, int64_t k, int w, int32_t* ipiv, double* stats, int32_t* info,
                    int batch, int cs, cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured)) {
    cudaFuncSetAttribute(panel_kernel<W, S>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * cs), 1, 1);
  cfg.blockDim = dim3(PANEL_T, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, panel_kernel<W, S>, C, n, k, w, ipiv, stats, info);
  count_launch();
}
}  // namespace

PanelCfg panel_config(int64_t n) {
  // S * PANEL_T * cluster >= n rows (the first panel has n rows)
  if (n <= 2048) return {8, 8, 1};
  if (n <= 4096) return {8, 8, 2};
  if (n <= 8192) return {8, 8, 4};
  if (n <= 16384) return {16, 8, 4};
  if (n <= 32768) return {16, 4, 8};
  return {0, 0, 0};
}

void panel_launch(Batched C, int64_t n, int64_t k, int w, int32_t* ipiv, double* stats, int32_t* info,
                  int batch, const PanelCfg& cfg, cudaStream_t s) {
  const double L_ = (double)(n - k); ProfScope ps_(K_PANEL, (double)batch * (4.0 * L_ * w * w - 4.0 * w * (double)w * w / 3.0), 0.0, s);
  if (cfg.W == 8 && cfg.S == 1) panel_launch_t<8, 1>(C, n, k, w, ipiv, stats, info, batch, cfg.cluster, s);
  else if (cfg.W == 8 && cfg.S == 2) panel_launch_t<8, 2>(C, n, k, w, ipiv, stats, info, batch, cfg.cluster, s);
  else if (cfg.W == 8 && cfg.S == 4) panel_launch_t<8, 4>(C, n, k, w, ipiv, stats, info, batch, cfg.cluster, s);
  else if (cfg.W == 4 && cfg.S == 8) panel_launch_t<4, 8>(C, n, k, w, ipiv, stats, info, batch, cfg.cluster, s);
}

// timing ablation only (FEAST_ABLATE bit 1): identity pivots in place of a skipped panel
__global__ void ipiv_identity_kernel(int32_t* ipiv, int64_t n, int64_t k, int w, int batch) {
  const int b = blockIdx.x, i = threadIdx.x;
  if (b < batch && i < w) ipiv[(int64_t)b * n + k + i] = (int32_t)(k + i);
}

void ipiv_identity_launch(int32_t* ipiv, int64_t n, int64_t k, int w, int batch, cudaStream_t s) {
  ipiv_identity_kernel<<<batch, 64, 0, s>>>(ipiv, n, k, w, batch);
  count_launch();
}

__global__ void stats_init_kernel(double* stats, int32_t* info, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) { stats[2 * b] = DBL_MAX; stats[2 * b + 1] = 0.0; info[b] = 0; }
}

void stats_init_launch(double* stats, int32_t* info, int batch, cudaStream_t s) {
  ProfScope ps_(K_OTHER, 0.0, 0.0, s);
  stats_init_kernel<<<(batch + 127) / 128, 128, 0, s>>>(stats, info, batch);
  count_launch();
}

// ============================================================================ laswp
// Apply the cnt (<= 1024) sequential swaps ipiv[k..k+cnt) to the columns [c0, c1) of every
// matrix.  Thread per column; each swap exchanges two 16-byte complex entries.
__global__ void laswp_kernel(Batched C, int64_t n, int64_t k, int cnt, const int32_t* __restrict__ ipiv_all,
                             int64_t c0, int64_t c1, unsigned long long* moved_bytes) {
  __shared__ int32_t pv[1024];
  const int b = blockIdx.y;
  const int32_t* ipiv = ipiv_all + (int64_t)b * n;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) pv[i] = ipiv[k + i];
  __syncthreads();
  const int64_t col = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned nsw = 0;
  if (col < c1) {
    double2* Cc = C.p + (int64_t)b * C.stride + col * C.ld;
    for (int i = 0; i < cnt; ++i) {
      const int64_t r1 = k + i, r2 = pv[i];
      if (r1 != r2) {
        const double2 t = Cc[r1];
        Cc[r1] = Cc[r2];
        Cc[r2] = t;
        ++nsw;
      }
    }
  }
  if (moved_bytes) {   // profile mode: 64 B per swap (two elements read and written)
    const unsigned w = __reduce_add_sync(0xffffffffu, nsw);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(moved_bytes, 64ull * w);
  }
}

// Row swaps as ONE permutation (SURVEY G3 "row-swap kernel with coalesced 16-byte access"):
// thread 0 of every CTA composes the cnt sequential swaps into the map of the touched rows
// (positions k..k+cnt-1 and the pivot rows below), using a dense row -> slot table in shared
// memory; then each warp moves whole columns with one gather and one scatter: lane j reads the
// source row of touched slot j and writes the destination row, so the writes to the contiguous
// rows k..k+cnt-1 of a column coalesce, and no swap waits on another (a sequential swap chain
// is cnt dependent global round trips).
constexpr int LP_COLS = 1;          // columns per warp (one gather/scatter round trip each)
constexpr int LP_WARPS = 8;
__global__ void __launch_bounds__(32 * LP_WARPS) laswp_perm_kernel(Batched C, int64_t n, int64_t k, int cnt,
                                                                    const int32_t* __restrict__ ipiv_all,
                                                                    int64_t c0, int64_t c1) {
  extern __shared__ int32_t lsm[];
  const int L = (int)(n - k);
  int32_t* slot_of = lsm;                 // [L]: slot of relative row r, -1 if untouched
  int32_t* row_at = lsm + L;              // [2 cnt]: relative row of slot t (destination)
  int32_t* src_of = row_at + 2 * cnt;     // [2 cnt]: relative source row whose value ends in slot t
  __shared__ int nt_s;
  const int b = blockIdx.y;
  const int32_t* ipiv = ipiv_all + (int64_t)b * n + k;
  for (int r = threadIdx.x; r < L; r += blockDim.x) slot_of[r] = r < cnt ? r : -1;
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) { row_at[t] = t; src_of[t] = t; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nt = cnt;
    for (int i = 0; i < cnt; ++i) {
      const int p = ipiv[i] - (int)k;   // >= i (partial pivoting picks from rows i..)
      if (p == i) continue;
      int sp = slot_of[p];
      if (sp < 0) { sp = nt++; slot_of[p] = sp; row_at[sp] = p; src_of[sp] = p; }
      const int tmp = src_of[i];
      src_of[i] = src_of[sp];
      src_of[sp] = tmp;
    }
    nt_s = nt;
  }
  __syncthreads();
  const int nt = nt_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* base = C.p + (int64_t)b * C.stride + k;
  for (int q = 0; q < LP_COLS; ++q) {
    const int64_t col = c0 + ((int64_t)blockIdx.x * LP_WARPS + warp) * LP_COLS + q;
    if (col >= c1) break;
    double2* Cc = base + col * C.ld;
    // gather every touched slot's new value first, then scatter (a bijection on the slots)
    double2 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int t = lane + 32 * u;
      if (t < nt) v[u] = Cc[src_of[t]];
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int t = lane + 32 * u;
      if (t < nt) Cc[row_at[t]] = v[u];
    }
  }
}

// Row swaps, coalesced (BASELINE north_star "a row-swap kernel with coalesced 16-byte
// access").  The cnt sequential swaps ipiv[k..k+cnt) act on the touched rows only.  The swaps
// that move something (ipiv != row) are compacted in order (warp ballots); slot t names a
// DESTINATION row d_t — the block row i_j of swap j (slots < nz) or its pivot row p_j (slots
// >= nz) — and its source row is found by tracing d_t back through the nz swaps in reverse order
// (each swap is an involution), all slots in parallel (no serial composition, no row table).
// Slots whose row does not move are dropped.  Then each warp moves whole columns: lane t gathers the source of
// slot t into registers, then scatters to d_t, so the writes (and the reads of the pivot-row
// slots) to the contiguous block rows of a column coalesce into 512-byte warp transactions of
// 16-byte complex elements; the other half of the accesses are the scattered pivot rows (one
// 32-byte sector each, unavoidable in column-major storage).  In profile mode every CTA adds the
// bytes it moved (16 B read + 16 B written per moved element) to a device counter.
constexpr int LC_WARPS = 8;
template <int SPL>   // slots per lane: 2 cnt <= 32 SPL
__global__ void __launch_bounds__(32 * LC_WARPS) laswp_coalesced_kernel(Batched C, int64_t n, int64_t k, int cnt,
                                                                          const int32_t* __restrict__ ipiv_all,
                                                                          int64_t c0, int64_t c1, int cols_per_cta,
                                                                          unsigned long long* moved_bytes) {
  __shared__ int32_t s_si[16 * 32 / 2], s_sp[16 * 32 / 2];   // the non-trivial swaps, in order
  __shared__ int32_t s_src[16 * 32], s_dst[16 * 32];
  __shared__ int s_wcnt[LC_WARPS];
  __shared__ int s_nmov;
  const int b = blockIdx.y;
  const int32_t* ipiv = ipiv_all + (int64_t)b * n + k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 1. ordered compaction of the swaps that move something (p != i): pivoting close to the diagonal
  //    (the shifted matrices of the BASELINE pencils) leaves only a few of them
  const int t0 = threadIdx.x;                                   // cnt <= 256 = blockDim
  const int p0 = t0 < cnt ? ipiv[t0] - (int)k : t0;             // relative rows
  const bool nontriv = t0 < cnt && p0 != t0;
  const unsigned bal = __ballot_sync(0xffffffffu, nontriv);
  if (lane == 0) s_wcnt[warp] = __popc(bal);
  if (threadIdx.x == 0) s_nmov = 0;
  __syncthreads();
  int off = 0, nz = 0;
#pragma unroll
  for (int q = 0; q < LC_WARPS; ++q) {
    off += q < warp ? s_wcnt[q] : 0;
    nz += s_wcnt[q];
  }
  if (nontriv) {
    const int pos = off + __popc(bal & ((1u << lane) - 1u));
    s_si[pos] = t0;
    s_sp[pos] = p0;
  }
  __syncthreads();
  // 2. slots: destination rows i_j (slots < nz: ascending block rows, coalesced when most rows
  //    move) and p_j (slots >= nz); each traced back through the nz swaps to its source row.  A
  //    row named twice gives two identical slots (same source, same value): harmless.
  const int nslot = 2 * nz;
  int mov = 0;
  for (int t = threadIdx.x; t < 32 * SPL; t += blockDim.x) {
    const int d = t < nz ? s_si[t] : (t < nslot ? s_sp[t - nz] : -1);
    int src = d;
    if (d >= 0)
      for (int j = nz - 1; j >= 0; --j) {   // the value that ends in row d came from src
        const int a = s_si[j], c = s_sp[j];
        src = src == a ? c : (src == c ? a : src);
      }
    const bool mv = d >= 0 && src != d;
    s_dst[t] = mv ? d : -1;
    s_src[t] = mv ? src : 0;
    mov += mv;
  }
  if (moved_bytes && mov) atomicAdd(&s_nmov, mov);
  __syncthreads();
  double2* base = C.p + (int64_t)b * C.stride + k;
  const int64_t cbeg = c0 + (int64_t)blockIdx.x * cols_per_cta, cend = min(c1, cbeg + cols_per_cta);
  // slot tables in registers for short swap sequences, read from shared memory for long ones
  constexpr bool REG = SPL <= 4;
  int dst_r[REG ? SPL : 1], src_r[REG ? SPL : 1];
  if (REG)
#pragma unroll
    for (int u = 0; u < SPL; ++u) { dst_r[REG ? u : 0] = s_dst[lane + 32 * u]; src_r[REG ? u : 0] = s_src[lane + 32 * u]; }
#define DST(u) (REG ? dst_r[REG ? (u) : 0] : s_dst[lane + 32 * (u)])
#define SRC(u) (REG ? src_r[REG ? (u) : 0] : s_src[lane + 32 * (u)])
  constexpr bool ILP2 = SPL <= 4;   // two columns in flight per warp when the slot registers allow
  for (int64_t col = cbeg + warp; col < cend; col += (ILP2 ? 2 : 1) * LC_WARPS) {
    // gather every moved slot of the column(s) first, then scatter (a bijection on the slots)
    double2* C0 = base + col * C.ld;
    const bool two = ILP2 && col + LC_WARPS < cend;
    double2* C1 = base + (col + LC_WARPS) * C.ld;
    double2 v0[SPL], v1[ILP2 ? SPL : 1];
#pragma unroll
    for (int u = 0; u < SPL; ++u)
      if (DST(u) >= 0) {
        v0[u] = C0[SRC(u)];
        if (two) v1[ILP2 ? u : 0] = C1[SRC(u)];
      }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < SPL; ++u)
      if (DST(u) >= 0) {
        C0[DST(u)] = v0[u];
        if (two) C1[DST(u)] = v1[ILP2 ? u : 0];
      }
  }
#undef DST
#undef SRC
  if (moved_bytes && threadIdx.x == 0 && s_nmov)
    atomicAdd(moved_bytes, (unsigned long long)s_nmov * (unsigned long long)(cend > cbeg ? cend - cbeg : 0) * 32ull);
}

template <int SPL>
void laswp_coalesced_launch(Batched C, int64_t n, int64_t k, int cnt, const int32_t* ipiv, int64_t c0, int64_t c1,
                            int batch, cudaStream_t s, unsigned long long* moved) {
  // columns per CTA: enough CTAs to cover the GPU once for the smallest ranges, and at most 64
  // columns (eight per warp) so the per-CTA slot tracing (cnt steps) is amortised
  const int64_t ncol = c1 - c0;
  int cpc = 2 * LC_WARPS;
  while (cpc < 64 && (ncol + 2 * cpc - 1) / (2 * cpc) * batch >= 2 * 148) cpc *= 2;
  dim3 grid((unsigned)((ncol + cpc - 1) / cpc), (unsigned)batch);
  laswp_coalesced_kernel<SPL><<<grid, 32 * LC_WARPS, 0, s>>>(C, n, k, cnt, ipiv, c0, c1, cpc, moved);
}

void laswp_launch(Batched C, int64_t n, int64_t k, int cnt, const int32_t* ipiv, int64_t c0, int64_t c1, int batch,
                  cudaStream_t s, int variant) {
  if (c1 <= c0 || cnt <= 0) return;
  // algorithmic bytes: data-dependent (only moved rows count), filled by the kernel's counter
  ProfScope ps_(K_LASWP, 0.0, 0.0, s);
  const int64_t L = n - k;
  const size_t smem = (size_t)(L + 4 * cnt) * sizeof(int32_t);
  // coalesced kernel for the panels' swap sequences (cnt <= 64); the outer blocks' long sequences
  // (cnt = 256..1024) stay on the chain kernel: with dense pivoting (the C3 recipe) the slot
  // tracing and the 2 cnt slots per column make the coalesced kernel 3x slower there, while on the
  // panels' short sequences it is 4x faster (ncu, profiles/r02/swap_ncu.txt)
  if (variant == LASWP_COALESCED && cnt <= 64) {
    unsigned long long* moved = ps_.bytes_counter();
    if (cnt <= 32) laswp_coalesced_launch<2>(C, n, k, cnt, ipiv, c0, c1, batch, s, moved);
    else if (cnt <= 64) laswp_coalesced_launch<4>(C, n, k, cnt, ipiv, c0, c1, batch, s, moved);
    else if (cnt <= 128) laswp_coalesced_launch<8>(C, n, k, cnt, ipiv, c0, c1, batch, s, moved);
    else laswp_coalesced_launch<16>(C, n, k, cnt, ipiv, c0, c1, batch, s, moved);
  } else if (variant == LASWP_PERM && 2 * cnt <= 32 * 16 && smem <= 96 * 1024) {
    static std::atomic<uint64_t> configured{0};
    if (first_use_on_device(configured)) {
      cudaFuncSetAttribute(laswp_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    }
    const int64_t per_cta = (int64_t)LP_WARPS * LP_COLS;
    dim3 grid((unsigned)((c1 - c0 + per_cta - 1) / per_cta), (unsigned)batch);
    laswp_perm_kernel<<<grid, 32 * LP_WARPS, smem, s>>>(C, n, k, cnt, ipiv, c0, c1);
  } else {   // very tall trailing matrices (row table > 96 KB) or > 256 swaps: the swap chain per column
    const int threads = 128;
    dim3 grid((unsigned)((c1 - c0 + threads - 1) / threads), (unsigned)batch);
    laswp_kernel<<<grid, threads, 0, s>>>(C, n, k, cnt, ipiv, c0, c1, ps_.bytes_counter());
  }
  count_launch();
}

// trsm (in-block U12 = L11^-1 A12) lives in trtri.cu with the diagonal-block inverses.

// ============================================================================ permutations
// perm_b: result of applying the sequential swaps ipiv to 0..n-1 (one thread per matrix,
// the swap chain is inherently serial; kept in shared memory).
__global__ void perm_kernel(const int32_t* __restrict__ ipiv_all, int32_t* __restrict__ perm_all,
                            int32_t* __restrict__ iperm_all, int64_t n) {
  extern __shared__ int32_t ps[];
  const int b = blockIdx.x;
  const int32_t* ipiv = ipiv_all + (int64_t)b * n;
  int32_t* perm = perm_all + (int64_t)b * n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) ps[i] = (int32_t)i;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t i = 0; i < n; ++i) {
      const int32_t p = ipiv[i];
      if (p != i) { const int32_t t = ps[i]; ps[i] = ps[p]; ps[p] = t; }
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    perm[i] = ps[i];
    if (iperm_all) iperm_all[(int64_t)b * n + ps[i]] = (int32_t)i;
  }
}

void perm_launch(const int32_t* ipiv, int32_t* perm, int32_t* iperm, int64_t n, int batch, cudaStream_t s) {
  ProfScope ps_(K_PERM, 0.0, (double)batch * n * 12.0, s);
  static std::atomic<uint64_t> configured{0};
  if (first_use_on_device(configured)) {
    cudaFuncSetAttribute(perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  perm_kernel<<<batch, 256, (size_t)n * sizeof(int32_t), s>>>(ipiv, perm, iperm, n);
  count_launch();
}

__global__ void gather_rows_kernel(Batched Y, const double2* __restrict__ R, int64_t ldr, int64_t sR,
                                   const int32_t* __restrict__ perm_all, int64_t n) {
  const int b = blockIdx.z;
  const int64_t c = blockIdx.y;
  const int32_t* perm = perm_all + (int64_t)b * n;
  const double2* Rc = R + b * sR + c * ldr;
  double2* Yc = Y.p + (int64_t)b * Y.stride + c * Y.ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Yc[i] = Rc[perm[i]];
}

void gather_rows_launch(Batched Y, const double2* R, int64_t ldr, int64_t sR, const int32_t* perm, int64_t n,
                        int64_t m, int batch, cudaStream_t s) {
  ProfScope ps_(K_PERM, 0.0, (double)batch * n * m * 36.0, s);
  unsigned gx = (unsigned)((n + 255) / 256);
  if (gx > 16) gx = 16;
  gather_rows_kernel<<<dim3(gx, (unsigned)m, (unsigned)batch), 256, 0, s>>>(Y, R, ldr, sR, perm, n);
  count_launch();
}

__global__ void scatter_rows_kernel(Batched Out, const double2* __restrict__ Y, int64_t ldy, int64_t sY,
                                    const int32_t* __restrict__ perm_all, int64_t n) {
  const int b = blockIdx.z;
  const int64_t c = blockIdx.y;
  const int32_t* perm = perm_all + (int64_t)b * n;
  const double2* Yc = Y + b * sY + c * ldy;
  double2* Oc = Out.p + (int64_t)b * Out.stride + c * Out.ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Oc[perm[i]] = Yc[i];
}

void scatter_rows_launch(Batched Out, const double2* Y, int64_t ldy, int64_t sY, const int32_t* perm, int64_t n,
                         int64_t m, int batch, cudaStream_t s) {
  ProfScope ps_(K_PERM, 0.0, (double)batch * n * m * 36.0, s);
  unsigned gx = (unsigned)((n + 255) / 256);
  if (gx > 16) gx = 16;
  scatter_rows_kernel<<<dim3(gx, (unsigned)m, (unsigned)batch), 256, 0, s>>>(Out, Y, ldy, sY, perm, n);
  count_launch();
}

// Y_b[:, c] = R[:, c] (c < m) and, with mode BC_PAIR, Y_b[:, m + c] = conj(R[:, c]): the
// right-hand sides [R | conj(R)] of a conjugate-pole pair of a real pencil (one LU, both poles);
// mode BC_CONJ copies conj(R) (the left block of a complex-symmetric pencil).
__global__ void broadcast_copy_kernel(Batched Y, const double2* __restrict__ R, int64_t ldr, int64_t n, int64_t m,
                                      int mode) {
  const int b = blockIdx.z;
  const int64_t cc = blockIdx.y;
  const bool cj = cc >= m || mode == BC_CONJ;
  const int64_t c = cc >= m ? cc - m : cc;
  const double2* Rc = R + c * ldr;
  double2* Yc = Y.p + (int64_t)b * Y.stride + cc * Y.ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = Rc[i];
    Yc[i] = cj ? cconj(v) : v;
  }
}

void broadcast_copy_launch(Batched Y, const double2* R, int64_t ldr, int64_t n, int64_t m, int batch, int mode,
                           cudaStream_t s) {
  const int64_t cols = mode == BC_PAIR ? 2 * m : m;
  ProfScope ps_(K_PERM, 0.0, (double)batch * n * cols * 32.0, s);
  unsigned gx = (unsigned)((n + 255) / 256);
  if (gx > 16) gx = 16;
  broadcast_copy_kernel<<<dim3(gx, (unsigned)cols, (unsigned)batch), 256, 0, s>>>(Y, R, ldr, n, m, mode);
  count_launch();
}

// flag[0] |= 1 if any entry of the n x n matrix M has a nonzero imaginary part (real-pencil check)
__global__ void imag_check_kernel(const double2* __restrict__ M, int64_t ld, int64_t n, int32_t* flag) {
  const int64_t c = blockIdx.y;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= M[i + c * ld].y != 0.0;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

void imag_check_launch(const double2* M, int64_t ld, int64_t n, int32_t* flag, cudaStream_t s) {
  ProfScope ps_(K_OTHER, 0.0, (double)n * n * 16.0, s);
  unsigned gx = (unsigned)((n + 255) / 256);
  if (gx > 8) gx = 8;
  imag_check_kernel<<<dim3(gx, (unsigned)n), 256, 0, s>>>(M, ld, n, flag);
  count_launch();
}

// ============================================================================ accumulate
// Q (+)= sum_b w_b Y_b in increasing b (deterministic, eq. Rasp sum).  With wp
// (conjugate-pole pairs of a real pencil): + wp_b conj(Y_b[:, m + c]), the partner pole's solve
// C(conj z)^-1 R = conj(C(z)^-1 conj(R)).
__device__ __forceinline__ double2 cfma(double2 w, double2 y, double2 acc) {
  return make_double2(fma(w.x, y.x, fma(-w.y, y.y, acc.x)), fma(w.x, y.y, fma(w.y, y.x, acc.y)));
}
__global__ void accum_kernel(double2* __restrict__ Q, int64_t ldq, Batched Y, const double2* __restrict__ w,
                             const double2* __restrict__ wp, const int32_t* __restrict__ iperm, int64_t n, int64_t m,
                             int batch, bool conjw, bool accumulate, bool conj_out) {
  const int64_t c = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = accumulate ? Q[i + c * ldq] : make_double2(0.0, 0.0);
    if (conj_out) acc = cconj(acc);
    for (int b = 0; b < batch; ++b) {
      double2 wb = w[b];
      if (conjw) wb = cconj(wb);
      const int64_t src = iperm ? (int64_t)iperm[(int64_t)b * n + i] : i;
      const double2* Yb = Y.p + (int64_t)b * Y.stride + src;
      acc = cfma(wb, Yb[c * Y.ld], acc);
      if (wp) {
        double2 wq = wp[b];
        if (conjw) wq = cconj(wq);
        acc = cfma(wq, cconj(Yb[(m + c) * Y.ld]), acc);
      }
    }
    Q[i + c * ldq] = conj_out ? cconj(acc) : acc;
  }
}

void accum_launch(double2* Q, int64_t ldq, Batched Y, const double2* w, const double2* wp, const int32_t* iperm,
                  int64_t n, int64_t m, int batch, bool conjw, bool accumulate, cudaStream_t s, bool conj_out) {
  const int parts = wp ? 2 : 1;
  ProfScope ps_(K_ACCUM, (double)batch * parts * n * m * 8.0,
                (double)(batch * parts + (accumulate ? 2 : 1)) * n * m * 16.0, s);
  unsigned gx = (unsigned)((n + 255) / 256);
  if (gx > 16) gx = 16;
  accum_kernel<<<dim3(gx, (unsigned)m), 256, 0, s>>>(Q, ldq, Y, w, wp, iperm, n, m, batch, conjw, accumulate,
                                                     conj_out);
  count_launch();
}

// C = alpha * sum_s P_s + beta * C  (split-K partials, summed in s order: deterministic)
__global__ void splitk_reduce_kernel(double2* C, int64_t ldc, const double2* P, int64_t M, int64_t N, int splits,
                                     double2 alpha, double2 beta) {
  const int64_t c = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int sidx = 0; sidx < splits; ++sidx) acc = cadd(acc, P[(int64_t)sidx * M * N + c * M + i]);
    double2 v = cmul(alpha, acc);
    if (beta.x != 0.0 || beta.y != 0.0) v = cadd(v, cmul(beta, C[i + c * ldc]));
    C[i + c * ldc] = v;
  }
}

void splitk_reduce_launch(double2* C, int64_t ldc, const double2* P, int64_t M, int64_t N, int splits,
                          double2 alpha, double2 beta, cudaStream_t s) {
  ProfScope ps_(K_OTHER, 0.0, (double)(splits + 1) * M * N * 16.0, s);
  unsigned gx = (unsigned)((M + 255) / 256);
  if (gx > 16) gx = 16;
  splitk_reduce_kernel<<<dim3(gx, (unsigned)N), 256, 0, s>>>(C, ldc, P, M, N, splits, alpha, beta);
  count_launch();
}

// ============================================================================ iteration helpers
__device__ double block_sum(double v) {
  __shared__ double red[32];
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

__global__ void resid_kernel(const double2* AX, const double2* BX, const double2* X, int64_t ld,
                             const double2* lam, int64_t n, double* out, double* xn, bool squared) {
  const int64_t c = blockIdx.x;
  const double2 l = lam[c];
  double r2 = 0.0, x2 = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 rv = cfms(AX[i + c * ld], l, BX[i + c * ld]);
    r2 += rv.x * rv.x + rv.y * rv.y;
    const double2 xv = X[i + c * ld];
    x2 += xv.x * xv.x + xv.y * xv.y;
  }
  r2 = block_sum(r2);
  x2 = block_sum(x2);
  if (threadIdx.x == 0) {
    out[c] = squared ? r2 : sqrt(r2);
    if (xn) xn[c] = squared ? x2 : sqrt(x2);
  }
}

void resid_launch(const double2* AX, const double2* BX, const double2* X, int64_t ld, const double2* lam,
                  int64_t n, int64_t m, double* out, double* xn, cudaStream_t s, bool squared) {
  ProfScope ps_(K_OTHER, 0.0, 0.0, s);
  resid_kernel<<<(unsigned)m, 256, 0, s>>>(AX, BX, X, ld, lam, n, out, xn, squared);
  count_launch();
}

__global__ void frob2_kernel(const double2* A, int64_t lda, int64_t n, double* partial) {
  double s = 0.0;
  for (int64_t c = blockIdx.x; c < n; c += gridDim.x)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double2 v = A[i + c * lda];
      s += v.x * v.x + v.y * v.y;
    }
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

void frob2_launch(const double2* A, int64_t lda, int64_t n, double* partial, int nparts, cudaStream_t s) {
  ProfScope ps_(K_OTHER, 0.0, 0.0, s);
  frob2_kernel<<<nparts, 256, 0, s>>>(A, lda, n, partial);
  count_launch();
}

// partial[b] = sum over the columns c = b, b + nparts, ... of sum_i conj(U[i][c]) Q[i][c]
// (re, im) — the trace tr(U^H Q) of the count estimator, summed on the host in block order.
__global__ void cdot_kernel(const double2* U, int64_t ldu, const double2* Q, int64_t ldq, int64_t n, int64_t m,
                            double2* partial) {
  double re = 0.0, im = 0.0;
  for (int64_t c = blockIdx.x; c < m; c += gridDim.x)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double2 u = U[i + c * ldu], q = Q[i + c * ldq];
      re = fma(u.x, q.x, fma(u.y, q.y, re));
      im = fma(u.x, q.y, fma(-u.y, q.x, im));
    }
  re = block_sum(re);
  __syncthreads();
  im = block_sum(im);
  if (threadIdx.x == 0) partial[blockIdx.x] = make_double2(re, im);
}

void cdot_launch(const double2* U, int64_t ldu, const double2* Q, int64_t ldq, int64_t n, int64_t m, double2* partial,
                 int nparts, cudaStream_t s) {
  ProfScope ps_(K_OTHER, 8.0 * n * m, 32.0 * n * m, s);
  cdot_kernel<<<nparts, 256, 0, s>>>(U, ldu, Q, ldq, n, m, partial);
  count_launch();
}

// Zero the strictly lower triangle of an m x m matrix (the R factor left by geqrf).
__global__ void tril_zero_kernel(double2* M, int64_t ld, int64_t m) {
  const int64_t c = blockIdx.x;
  for (int64_t i = c + 1 + threadIdx.x; i < m; i += blockDim.x) M[i + c * ld] = make_double2(0.0, 0.0);
}

void tril_zero_launch(double2* M, int64_t ld, int64_t m, cudaStream_t s) {
  ProfScope ps_(K_OTHER, 0.0, 0.0, s);
  tril_zero_kernel<<<(unsigned)m, 128, 0, s>>>(M, ld, m);
  count_launch();
}

__global__ void colscale_kernel(double2* X, int64_t ldx, int64_t n, double2* W, int64_t ldw, int64_t m,
                                const double* xn) {
  const int64_t c = blockIdx.y;
  const double sc = xn[c] > 0.0 ? 1.0 / xn[c] : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = X[i + c * ldx];
    X[i + c * ldx] = make_double2(v.x * sc, v.y * sc);
  }
  if (blockIdx.x == 0)
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      double2 v = W[i + c * ldw];
      W[i + c * ldw] = make_double2(v.x * sc, v.y * sc);
    }
}

void colscale_launch(double2* X, int64_t ldx, int64_t n, double2* W, int64_t ldw, int64_t m, const double* xn,
                     cudaStream_t s) {
  ProfScope ps_(K_OTHER, 0.0, 0.0, s);
  unsigned gx = (unsigned)((n + 255) / 256);
  if (gx > 16) gx = 16;
  colscale_kernel<<<dim3(gx, (unsigned)m), 256, 0, s>>>(X, ldx, n, W, ldw, m, xn);
  count_launch();
}

}  // namespace feast
