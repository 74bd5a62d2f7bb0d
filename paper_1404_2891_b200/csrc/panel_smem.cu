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
// Per column: warp-shuffle argmax -> CTA argmax -> the candidate's owner pushes its chunk row
// (W complex) + |pivot| + row id into every CTA's slot (DSMEM) -> ONE cluster barrier ->
// identical global decision everywhere -> in-register rank-1 update of the W-column chunk.
// Per chunk of W columns: the chunk's W pivot rows push their remaining-panel values to every
// CTA, one more barrier, every CTA forms U12 = L11^-1 (pivot rows) and applies the rank-W
// update to its own non-pivot rows in shared memory (one smem read-modify-write per element
// per chunk, not per column).
#include <cooperative_groups.h>
#include <float.h>
#include <limits.h>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace cg = cooperative_groups;

namespace feast {
namespace {

constexpr int PT = 128;          // threads per CTA (one panel row each, S rows)
constexpr int CSM = 16;          // max cluster size
constexpr int WC = 8;            // chunk width (columns held in registers)
constexpr int WMAX = 64;         // max panel width

struct __align__(16) Slot {
  double2 row[WC];
  double val;
  int idx;
  int pad;
};

__device__ __forceinline__ bool better(double v, int i, double bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

template <int S>
__global__ void __launch_bounds__(PT, 1)
panel_smem_kernel(Batched Cb, int64_t n, int64_t k, int w, int32_t* __restrict__ ipiv_all,
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
  const int PLD = w + 1;   // smem row stride (complex) -> conflict-free column access

  extern __shared__ __align__(16) double2 P[];  // [Lc][PLD]
  __shared__ Slot slots[2][CSM];
  __shared__ double2 L11s[WC][WC];               // chunk pivot rows' chunk values
  __shared__ double2 U12s[WC][WMAX];             // chunk pivot rows' rest-of-panel values
  __shared__ int pvt[WMAX];                      // pivot (panel row index) per column
  __shared__ double wv[PT / 32];
  __shared__ int wi[PT / 32];
  __shared__ double2 cand[WC];

  // ---- load own rows of the panel (coalesced: consecutive threads = consecutive rows)
  for (int c = 0; c < w; ++c)
    for (int r = tid; r < nrow; r += PT) P[r * PLD + c] = C[(rbeg + r) + c * ld];
  __syncthreads();

  bool used[S];
#pragma unroll
  for (int s = 0; s < S; ++s) used[s] = false;
  double2 a[S][WC];
  double pmin = DBL_MAX, pmax = 0.0;
  int info = 0;

  for (int j0 = 0; j0 < w; j0 += WC) {
    const int wc = min(WC, w - j0);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int r = tid + s * PT;
#pragma unroll
      for (int jj = 0; jj < WC; ++jj)
        a[s][jj] = (r < nrow && jj < wc) ? P[r * PLD + j0 + jj] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int jj = 0; jj < WC; ++jj) {
      if (jj >= wc) break;
      const int col = j0 + jj;
      const int buf = col & 1;
      double bv = -1.0;
      int bi = INT_MAX;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int r = tid + s * PT;
        if (r < nrow && !used[s]) {
          const double v = cabs1(a[s][jj]);
          if (better(v, rbeg + r, bv, bi)) { bv = v; bi = rbeg + r; }
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
      for (int q = 1; q < PT / 32; ++q)
        if (better(wv[q], wi[q], cv, ci)) { cv = wv[q]; ci = wi[q]; }
      // the owner stages its chunk row locally, then CS*(WC+1) threads push it in parallel
#pragma unroll
      for (int s = 0; s < S; ++s)
        if (cv >= 0.0 && rbeg + tid + s * PT == ci) {
#pragma unroll
          for (int q = 0; q < WC; ++q) cand[q] = a[s][q];
        }
      __syncthreads();
      for (int t = tid; t < CS * (WC + 1); t += PT) {
        const int dcta = t / (WC + 1), e = t % (WC + 1);
        Slot* d = cluster.map_shared_rank(&slots[buf][crank], dcta);
        if (e < WC) {
          if (cv >= 0.0) d->row[e] = cand[e];
        } else {
          d->val = cv;
          d->idx = cv >= 0.0 ? ci : INT_MAX;
        }
      }
      cluster.sync();
      int gb = 0;
      double gv = slots[buf][0].val;
      int gi = slots[buf][0].idx;
      for (int c = 1; c < CS; ++c) {
        const double v = slots[buf][c].val;
        const int i = slots[buf][c].idx;
        if (better(v, i, gv, gi)) { gv = v; gi = i; gb = c; }
      }
      const double2* prow = slots[buf][gb].row;
      if (tid < WC) L11s[jj][tid] = prow[tid];
      if (tid == 0) pvt[col] = gi;
      const double2 p = prow[jj];
      const bool pzero = (p.x == 0.0 && p.y == 0.0);
      const double2 pinv = pzero ? make_double2(0.0, 0.0) : crcp(p);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int r = tid + s * PT;
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
      if (crank == 0 && tid == 0) {
        const double ap = hypot(p.x, p.y);
        pmin = fmin(pmin, ap);
        pmax = fmax(pmax, ap);
        if (pzero && !info) info = (int)(k + col + 1);
      }
    }
    // ---- chunk done: registers back to smem
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int r = tid + s * PT;
      if (r < nrow) {
#pragma unroll
        for (int jj = 0; jj < WC; ++jj)
          if (jj < wc) P[r * PLD + j0 + jj] = a[s][jj];
      }
    }
    const int c1 = j0 + wc;
    if (c1 < w) {
      const int rem = w - c1;
      __syncthreads();
      // owners push the chunk pivot rows' rest-of-panel values to every CTA
      for (int jj = 0; jj < wc; ++jj) {
        const int pr = pvt[j0 + jj] - rbeg;
        if (pr >= 0 && pr < nrow) {
          for (int idx = tid; idx < rem * CS; idx += PT) {
            const int c = idx % rem, dcta = idx / rem;
            double2* d = cluster.map_shared_rank(&U12s[jj][c], dcta);
            *d = P[pr * PLD + c1 + c];
          }
        }
      }
      cluster.sync();
      // U12 = L11^-1 (pivot rows), unit lower L11 (chunk multipliers of the pivot rows)
      for (int c = tid; c < rem; c += PT) {
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
      __syncthreads();
      // pivot rows of this chunk take their U12 values; other rows get the rank-wc update
      for (int jj = 0; jj < wc; ++jj) {
        const int pr = pvt[j0 + jj] - rbeg;
        if (pr >= 0 && pr < nrow)
          for (int c = tid; c < rem; c += PT) P[pr * PLD + c1 + c] = U12s[jj][c];
      }
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int r = tid + s * PT;
        if (r < nrow && !used[s]) {
          double2* row = P + r * PLD + c1;
          for (int c = 0; c < rem; ++c) {
            double2 v = row[c];
#pragma unroll
            for (int jj = 0; jj < WC; ++jj)
              if (jj < wc) v = cfms(v, a[s][jj], U12s[jj][c]);
            row[c] = v;
          }
        }
      }
      // the next chunk's slots/U12s writes by other CTAs happen after the next cluster barrier
      cluster.sync();
    }
  }
  __syncthreads();
  // ---- store own rows back (physical order)
  for (int c = 0; c < w; ++c)
    for (int r = tid; r < nrow; r += PT) C[(rbeg + r) + c * ld] = P[r * PLD + c];
  // ---- LAPACK ipiv from the pivot sequence (rows / positions relative to k)
  if (crank == 0 && tid == 0) {
    int pos2row[WMAX], cur[WMAX];
    for (int i = 0; i < w; ++i) { pos2row[i] = i; cur[i] = i; }
    int32_t* ipiv = ipiv_all + (int64_t)b * n + k;
    for (int col = 0; col < w; ++col) {
      const int p = pvt[col];
      const int lp = p < w ? cur[p] : p;
      const int rc = pos2row[col];
      ipiv[col] = (int32_t)(k + lp);
      if (lp < w) pos2row[lp] = rc;
      if (rc < w) cur[rc] = lp;
      pos2row[col] = p;
      if (p < w) cur[p] = col;
    }
    stats_all[2 * b] = fmin(stats_all[2 * b], pmin);
    stats_all[2 * b + 1] = fmax(stats_all[2 * b + 1], pmax);
    if (info && !info_all[b]) info_all[b] = info;
  }
  // keep every CTA's shared memory alive until remote writes into it are complete
  cluster.sync();
}

template <int S>
void launch_s(Batched C, int64_t n, int64_t k, int w, int32_t* ipiv, double* stats, int32_t* info, int batch, int cs,
              cudaStream_t s) {
  const int64_t L = n - k;
  const int Lc = (int)((L + cs - 1) / cs);
  const size_t smem = (size_t)Lc * (w + 1) * sizeof(double2);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(panel_smem_kernel<S>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(panel_smem_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * cs), 1, 1);
  cfg.blockDim = dim3(PT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, panel_smem_kernel<S>, C, n, k, w, ipiv, stats, info);
  count_launch();
}

}  // namespace

bool panel_smem_fits(int64_t n, int w, int cs) {
  const int64_t Lc = (n + cs - 1) / cs;
  return w <= WMAX && (size_t)Lc * (w + 1) * sizeof(double2) <= 190 * 1024 && Lc <= 2 * PT;
}

void panel_smem_launch(Batched C, int64_t n, int64_t k, int w, int32_t* ipiv, double* stats, int32_t* info, int batch,
                       int cs, cudaStream_t s) {
  const double L_ = (double)(n - k);
  ProfScope ps_(K_PANEL, (double)batch * (4.0 * L_ * w * w - 4.0 * w * (double)w * w / 3.0), 0.0, s);
  const int64_t Lc = (n + cs - 1) / cs;
  if (Lc <= PT) launch_s<1>(C, n, k, w, ipiv, stats, info, batch, cs, s);
  else launch_s<2>(C, n, k, w, ipiv, stats, info, batch, cs, s);
}

}  // namespace feast
