// reduced_eig.cu — the m0 x m0 reduced eigenproblem of a FEAST iteration on one CTA (SURVEY §8(a)
// "outside the timed path": R-FEAST step 5; Bi-FEAST step 7), for
// m0 <= RE_MAXM.  cuSOLVER's Xgeev (a hybrid host/device solver) takes ~25 ms at m0 = 128 on
// B200 — longer than the projector of C2 — so small reduced problems are solved here:
//
//   1. Householder reduction to upper Hessenberg form, in global memory (L2-resident):
//      H = P^H M P, P = P_1 ... P_{m-2}, P_j = I - 2 u u^H (||u|| = 1); Z = P.
//   2. Complex single-shift QR iteration (Wilkinson shift, exceptional shifts every 10
//      iterations, deflation |h_{l,l-1}| <= eps (|h_ll| + |h_{l-1,l-1}|)) on the Hessenberg
//      matrix held PACKED in shared memory (column j keeps rows 0..j+1: ~m^2/2 entries), the
//      bulge as a separate scalar.  Each step's rotation G = [[a, b], [-conj(b), conj(a)]]
//      (a = conj(f)/r, b = conj(g)/r, one reciprocal square root) is chased by ONE warp inside a
//      sliding window of RE_W steps (one lane per row / column of the window); the CTA applies
//      the window's rotations to the rest of H after each window and to Z after each sweep.
//   Measured on B200 (m = 64 / 128 / 160): 6.1 / 26 / 42 ms; at m = 128 the chase is ~28k
//   dependent steps of ~1.1k cycles (single-warp latency: rsqrt, shared-memory round trips),
//   the Householder phase 4.4 ms.  cuSOLVER Xgeev (26 ms at m = 128) stays the default; this
//   solver is device-resident (FEAST_EIG=own, feast_small_eig).  FEAST_RE_DEBUG=1 prints the
//   per-phase cycle counts.
//   3. Eigenvectors of T by back-substitution (one thread per eigenvector):
//      y_i = e_i, y_j = -(sum_{l=j+1..i} t_jl y_l) / (t_jj - t_ii), j < i.
//   The caller forms W = Z Y (a DMMA ZGEMM).  info = 0, or 1 if the QR iteration did not
//   converge within 30 m sweeps (the caller then falls back to cuSOLVER).
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace feast {
namespace {

constexpr int RE_T = 256;   // threads
constexpr int RE_W = 29;    // chase window: rows k0-1 .. k1+1 and columns k0-1 .. k1+1 fit 32 lanes

__device__ double block_sum_re(double v, double* red) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < RE_T / 32; ++i) s += red[i];
  return s;
}

__device__ __forceinline__ double cabs2d(double2 a) { return hypot(a.x, a.y); }

// packed Hessenberg: column j holds rows 0 .. min(j+1, m-1)
__host__ __device__ __forceinline__ int poff(int j, int m) {
  // sum_{l<j} min(l+2, m): for l <= m-2 the length is l+2
  const int jj = min(j, m - 1);
  int o = jj * (jj + 3) / 2;            // sum_{l<jj} (l + 2)
  if (j > m - 1) o += (j - (m - 1)) * m;
  return o;
}

__global__ void __launch_bounds__(RE_T) reduced_eig_kernel(double2* __restrict__ H, int m, int64_t ldh,
                                                           double2* __restrict__ Z, int64_t ldz,
                                                           double2* __restrict__ lam, double2* __restrict__ Y,
                                                           int64_t ldy, int32_t* __restrict__ info, int dbg) {
  extern __shared__ __align__(16) double2 S[];   // packed Hessenberg / Schur form
  __shared__ double red[RE_T / 32];
  __shared__ double2 rot_c[RE_MAXM], rot_s[RE_MAXM];   // a and b of each sweep step's rotation
  __shared__ double2 u_s[RE_MAXM], w_s[RE_MAXM];
  __shared__ int lo_s, conv_s, hi_s;
  const int tid = threadIdx.x;
  const long long t_begin = clock64();
  long long t_hess = 0, t_qr = 0;
  long long nsteps = 0, c_defl = 0, c_chase = 0, c_defer = 0, c_z = 0, cA;

  // ---- 1. Householder Hessenberg reduction in global memory; Z = I then Z <- Z P_j
  for (int idx = tid; idx < m * m; idx += RE_T) {
    const int i = idx % m, j = idx / m;
    Z[i + j * ldz] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  for (int j = 0; j + 2 < m; ++j) {
    const int len = m - j - 1;   // x = H[j+1 : m, j]
    double part = 0.0;
    for (int i = tid; i < len; i += RE_T) {
      const double2 v = H[(j + 1 + i) + j * ldh];
      part += v.x * v.x + v.y * v.y;
    }
    const double xn2 = block_sum_re(part, red);
    const double2 x0 = H[(j + 1) + j * ldh];
    const double xn = sqrt(xn2), ax0 = cabs2d(x0);
    if (xn == 0.0 || xn2 - ax0 * ax0 <= 1e-300 * xn2) { __syncthreads(); continue; }   // already reduced
    // alpha = -e^{i arg x0} ||x||;  u = (x - alpha e1) / ||x - alpha e1||
    const double2 ph = ax0 > 0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
    const double2 alpha = make_double2(-ph.x * xn, -ph.y * xn);
    const double2 u0 = make_double2(x0.x - alpha.x, x0.y - alpha.y);
    const double un = sqrt(xn2 - ax0 * ax0 + u0.x * u0.x + u0.y * u0.y);
    for (int i = tid; i < len; i += RE_T) {
      const double2 v = i == 0 ? u0 : H[(j + 1 + i) + j * ldh];
      u_s[i] = make_double2(v.x / un, v.y / un);
    }
    __syncthreads();
    // left: rows j+1.., columns j..m-1:  H <- H - 2 u (u^H H); w = u^H H by one warp per column
    // (lanes over rows: coalesced column reads, shuffle reduction)
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int c = j + warp; c < m; c += RE_T / 32) {
        double sx = 0.0, sy = 0.0;
        for (int i = lane; i < len; i += 32) {
          const double2 uh = cconj(u_s[i]), hv = H[(j + 1 + i) + c * ldh];
          sx += uh.x * hv.x - uh.y * hv.y;
          sy += uh.x * hv.y + uh.y * hv.x;
        }
        for (int off = 16; off > 0; off >>= 1) {
          sx += __shfl_xor_sync(0xffffffffu, sx, off);
          sy += __shfl_xor_sync(0xffffffffu, sy, off);
        }
        if (lane == 0) w_s[c - j] = make_double2(sx, sy);
      }
    }
    __syncthreads();
    for (int idx = tid; idx < len * (m - j); idx += RE_T) {
      const int i = idx % len, c = j + idx / len;
      const double2 t = cmul(u_s[i], w_s[c - j]);
      double2* hp = H + (j + 1 + i) + c * ldh;
      *hp = make_double2(hp->x - 2.0 * t.x, hp->y - 2.0 * t.y);
    }
    __syncthreads();
    // right: all rows, columns j+1..:  H <- H - 2 (H u) u^H ;  same for Z
    for (int pass = 0; pass < 2; ++pass) {
      double2* A = pass ? Z : H;
      const int64_t lda = pass ? ldz : ldh;
      for (int r = tid; r < m; r += RE_T) {   // consecutive rows per thread: coalesced
        double2 s0 = make_double2(0.0, 0.0), s1 = s0, s2 = s0, s3 = s0;
        int i = 0;
        for (; i + 4 <= len; i += 4) {        // four independent chains, loads in flight
          s0 = cadd(s0, cmul(A[r + (j + 1 + i) * lda], u_s[i]));
          s1 = cadd(s1, cmul(A[r + (j + 2 + i) * lda], u_s[i + 1]));
          s2 = cadd(s2, cmul(A[r + (j + 3 + i) * lda], u_s[i + 2]));
          s3 = cadd(s3, cmul(A[r + (j + 4 + i) * lda], u_s[i + 3]));
        }
        for (; i < len; ++i) s0 = cadd(s0, cmul(A[r + (j + 1 + i) * lda], u_s[i]));
        w_s[r] = cadd(cadd(s0, s1), cadd(s2, s3));
      }
      __syncthreads();
      for (int idx = tid; idx < m * len; idx += RE_T) {
        const int r = idx % m, i = idx / m;
        const double2 t = cmul(w_s[r], cconj(u_s[i]));
        double2* ap = A + r + (j + 1 + i) * lda;
        *ap = make_double2(ap->x - 2.0 * t.x, ap->y - 2.0 * t.y);
      }
      __syncthreads();
    }
  }
  t_hess = clock64();
  // ---- 2. packed copy into shared memory (entries below the subdiagonal are zero)
  for (int j = 0; j < m; ++j)
    for (int i = tid; i <= min(j + 1, m - 1); i += RE_T) S[poff(j, m) + i] = H[i + j * ldh];
  __syncthreads();
  auto at = [&](int i, int j) -> double2& { return S[poff(j, m) + i]; };

  const double eps = DBL_EPSILON;
  const int warp = tid >> 5, lane = tid & 31;
  // The bulge of a sweep is chased by WARP 0 alone inside a sliding window of RE_W steps
  // (lanes over the window's rows / columns, __syncwarp between the dependent passes): step k
  // updates rows k, k+1 only up to column cmax = k1 + 1 and columns k, k+1 only from row
  // k0 - 1, so each step touches <= 32 entries per pass whatever m is.  Left and right
  // rotations commute, and columns right of the window / rows above it never feed back into
  // it, so after each window the whole CTA applies the window's rotations to those parts
  // (one thread per column: the left chain down rows k0..k1; one thread per row: the right
  // chain across columns k0..k1) and, after the sweep, to Z.
  int hi = m - 1, its = 0, total = 0;
  const int maxit = 30 * m;
  bool failed = false;
  double2 f = make_double2(0.0, 0.0), g = f, bulge = f;   // warp 0: the chase state
  while (true) {
    cA = clock64();
    if (warp == 0) {
      int lo = 0;
      bool sweep = false;
      while (hi > 0 && !sweep) {
        // deflation: largest l in (0, hi] with negligible h_{l,l-1} (lanes test 32 l's at a time)
        int l = 0;
        for (int base = hi; base > 0; base -= 32) {
          const int cand = base - lane;
          bool neg = false;
          if (cand > 0) {
            const double tst = cabs1(at(cand, cand)) + cabs1(at(cand - 1, cand - 1));
            neg = cabs1(at(cand, cand - 1)) <= eps * tst;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, neg);
          if (bal) { l = base - (__ffs(bal) - 1); break; }
        }
        __syncwarp();
        if (l > 0 && lane == 0) at(l, l - 1) = make_double2(0.0, 0.0);
        __syncwarp();
        lo = l;
        if (lo == hi) { --hi; its = 0; continue; }
        if (++total > maxit) { failed = true; break; }
        ++its;
        sweep = true;
      }
      if (sweep) {
        // shift (every lane computes it: no broadcast needed)
        double2 mu;
        {
          const double2 a = at(hi - 1, hi - 1), b = at(hi - 1, hi), c = at(hi, hi - 1), d = at(hi, hi);
          if (its % 10 == 0) {
            const double e = cabs1(c) + (hi - 2 >= lo ? cabs1(at(hi - 1, hi - 2)) : 0.0);
            mu = make_double2(d.x + 0.75 * e, d.y);
          } else {
            const double2 hf = make_double2(0.5 * (a.x - d.x), 0.5 * (a.y - d.y));
            const double2 disc = cadd(cmul(hf, hf), cmul(b, c));
            const double r = cabs2d(disc);
            const double t = sqrt(0.5 * (r + fabs(disc.x)));
            double2 sq = make_double2(0.0, 0.0);
            if (t > 0.0)
              sq = disc.x >= 0.0 ? make_double2(t, disc.y / (2.0 * t)) : make_double2(fabs(disc.y) / (2.0 * t), copysign(t, disc.y));
            const double2 mid = make_double2(0.5 * (a.x + d.x), 0.5 * (a.y + d.y));
            const double2 l1 = cadd(mid, sq), l2 = csub(mid, sq);
            mu = cabs1(csub(l1, d)) <= cabs1(csub(l2, d)) ? l1 : l2;
          }
        }
        f = csub(at(lo, lo), mu);
        g = at(lo + 1, lo);
        bulge = make_double2(0.0, 0.0);
      }
      if (lane == 0) { lo_s = sweep ? lo : -1; conv_s = failed ? -1 : (hi <= 0 ? 1 : 0); hi_s = hi; }
    }
    __syncthreads();
    const int lo = lo_s, hiv = hi_s;
    c_defl += clock64() - cA; cA = clock64();
    if (lo >= 0) {
      for (int k0 = lo; k0 < hiv; k0 += RE_W) {
        const int k1 = min(k0 + RE_W, hiv);
        const int cmax = min(k1 + 1, m - 1);
        const int rmin = max(k0 - 1, 0);
        nsteps += k1 - k0;
        const long long cB = clock64();
        if (warp == 0) {
          for (int k = k0; k < k1; ++k) {
            // rotation G = [[a, b], [-conj(b), conj(a)]], a = conj(f)/nrm, b = conj(g)/nrm, so that
            // G [f; g] = [nrm; 0]: one reciprocal square root on the dependent chain (every lane)
            double2 a = make_double2(1.0, 0.0), b = make_double2(0.0, 0.0);
            {
              double n2 = f.x * f.x + f.y * f.y + g.x * g.x + g.y * g.y;
              if (n2 > 0.0) {
                double sc = 1.0;
                if (n2 < 1e-280 || n2 > 1e280) {   // rescale before squaring (rare)
                  sc = fmax(fmax(fabs(f.x), fabs(f.y)), fmax(fabs(g.x), fabs(g.y)));
                  sc = 1.0 / sc;
                  const double2 fs = make_double2(f.x * sc, f.y * sc), gs = make_double2(g.x * sc, g.y * sc);
                  n2 = fs.x * fs.x + fs.y * fs.y + gs.x * gs.x + gs.y * gs.y;
                }
                const double in = rsqrt(n2) * sc;
                a = make_double2(f.x * in, -f.y * in);
                b = make_double2(g.x * in, -g.y * in);
              }
            }
            if (lane == 0) { rot_c[k] = a; rot_s[k] = b; }
            // rows k, k+1, columns (k-1 or lo) .. cmax: <= RE_W + 3 = 32 entries, one per lane
            {
              const int col = (k > lo ? k - 1 : lo) + lane;
              if (col <= cmax) {
                const double2 hk = at(k, col);
                const double2 hk1 = (k + 1 <= col + 1) ? at(k + 1, col) : bulge;
                at(k, col) = cadd(cmul(a, hk), cmul(b, hk1));
                if (k + 1 <= col + 1) at(k + 1, col) = csub(cmul(cconj(a), hk1), cmul(cconj(b), hk));
              }
            }
            __syncwarp();
            // columns k, k+1, rows rmin .. min(k+2, hi): <= 32 entries, one per lane; (k+2, k) is
            // zero before, the new bulge after
            const int r1 = min(k + 2, hiv);
            double2 nb = make_double2(0.0, 0.0);
            {
              const int row = rmin + lane;
              if (row <= r1) {
                const double2 hik = (row <= k + 1) ? at(row, k) : make_double2(0.0, 0.0);
                const double2 hik1 = at(row, k + 1);
                const double2 nk = cadd(cmul(cconj(a), hik), cmul(cconj(b), hik1));
                if (row <= k + 1) at(row, k) = nk;
                at(row, k + 1) = csub(cmul(a, hik1), cmul(b, hik));
                nb = nk;
              }
            }
            __syncwarp();
            // next rotation's pair: (h_{k+1,k}, bulge (k+2, k)), broadcast from the owning lane
            if (k + 1 < hiv) {
              const int ob = (k + 2 - rmin) & 31;
              bulge = make_double2(__shfl_sync(0xffffffffu, nb.x, ob), __shfl_sync(0xffffffffu, nb.y, ob));
              f = at(k + 1, k);
              g = bulge;
            }
          }
        }
        __syncthreads();
        c_chase += clock64() - cB;
        const long long cC = clock64();
        // the window's rotations on the columns right of it (left chain down rows k0..k1) and
        // on the rows above it (right chain across columns k0..k1)
        const int ncol = m - 1 - cmax, nrow = rmin;
        for (int t = tid; t < ncol + nrow; t += RE_T) {
          if (t < ncol) {
            const int col = cmax + 1 + t;
            double2 x = at(k0, col);
            for (int k = k0; k < k1; ++k) {
              const double2 a = rot_c[k], b = rot_s[k], y = at(k + 1, col);
              at(k, col) = cadd(cmul(a, x), cmul(b, y));
              x = csub(cmul(cconj(a), y), cmul(cconj(b), x));
            }
            at(k1, col) = x;
          } else {
            const int row = t - ncol;
            double2 x = at(row, k0);
            for (int k = k0; k < k1; ++k) {
              const double2 a = rot_c[k], b = rot_s[k], y = at(row, k + 1);
              at(row, k) = cadd(cmul(cconj(a), x), cmul(cconj(b), y));
              x = csub(cmul(a, y), cmul(b, x));
            }
            at(row, k1) = x;
          }
        }
        __syncthreads();
      }
      c_defer += clock64() - cA; cA = clock64();
      // Z <- Z G_k^H, k = lo..hiv-1, one thread per row; the row segment is prefetched 8 at a time
      for (int row = tid; row < m; row += RE_T) {
        double2* zr = Z + row;
        double2 zk = zr[(int64_t)lo * ldz];
        for (int k0 = lo; k0 < hiv; k0 += 8) {
          double2 nx[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (k0 + 1 + e <= hiv) nx[e] = zr[(int64_t)(k0 + 1 + e) * ldz];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int k = k0 + e;
            if (k < hiv) {
              const double2 a = rot_c[k], b = rot_s[k];
              const double2 nk = cadd(cmul(cconj(a), zk), cmul(cconj(b), nx[e]));
              zk = csub(cmul(a, nx[e]), cmul(b, zk));
              zr[(int64_t)k * ldz] = nk;
            }
          }
        }
        zr[(int64_t)hiv * ldz] = zk;
      }
    }
    __syncthreads();
    if (lo >= 0) c_z += clock64() - cA;
    if (conv_s != 0) break;
  }
  t_qr = clock64();
  if (dbg && tid == 0)
    printf("reduced_eig m=%d: hessenberg %lld cyc, qr %lld cyc, sweeps %d, steps %lld; defl+shift %lld, chase %lld, "
           "windows %lld, Z %lld\n", m, t_hess - t_begin, t_qr - t_hess, total, nsteps, c_defl, c_chase, c_defer, c_z);
  if (conv_s < 0) {
    if (tid == 0) info[0] = 1;
    return;
  }
  // ---- 3. eigenvalues and eigenvectors of T (upper triangular part of S)
  for (int i = tid; i < m; i += RE_T) lam[i] = at(i, i);
  const double smlnum = DBL_MIN * (double)m / eps;
  for (int i = tid; i < m; i += RE_T) {
    const double2 ti = at(i, i);
    double2* y = Y + (int64_t)i * ldy;
    for (int j = i + 1; j < m; ++j) y[j] = make_double2(0.0, 0.0);
    y[i] = make_double2(1.0, 0.0);
    for (int j = i - 1; j >= 0; --j) {
      double2 sacc = make_double2(0.0, 0.0);
      for (int l = j + 1; l <= i; ++l) sacc = cadd(sacc, cmul(at(j, l), y[l]));
      double2 den = csub(at(j, j), ti);
      if (cabs1(den) < smlnum) den = make_double2(smlnum, 0.0);
      y[j] = cdiv(make_double2(-sacc.x, -sacc.y), den);
    }
  }
  if (tid == 0) info[0] = 0;
  if (dbg && tid == 0) printf("reduced_eig m=%d: vectors %lld cyc\n", m, clock64() - t_qr);
}

}  // namespace

bool reduced_eig_launch(double2* H, int m, int64_t ldh, double2* Z, int64_t ldz, double2* lam, double2* Y, int64_t ldy,
                        int32_t* info, cudaStream_t s) {
  if (m < 1 || m > RE_MAXM) return false;
  ProfScope ps_(K_OTHER, 0.0, 0.0, s);
  const size_t smem = (size_t)poff(m, m) * sizeof(double2);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(reduced_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    configured = true;
  }
  static const int dbg = getenv("FEAST_RE_DEBUG") ? 1 : 0;
  reduced_eig_kernel<<<1, RE_T, smem, s>>>(H, m, ldh, Z, ldz, lam, Y, ldy, info, dbg);
  count_launch();
  return true;
}

}  // namespace feast
