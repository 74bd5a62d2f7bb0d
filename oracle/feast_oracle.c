/*
 * feast_oracle.c — plain, slow, obviously-correct CPU oracle for the non-Hermitian
 * FEAST quadrature projector (Tang, Kestyn & Polizzi, arXiv 1404.2891).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1404_2891_b200/) never links, imports or calls it, and shares no code,
 * header, helper or constant with it.
 *
 * Citations "P:n" are lines of the paper text PAPER.md (LaTeX source); the section /
 * equation label is named beside each.  Readings of ambiguous passages are the
 * DESIGN.md "Readings" list (R1..).
 *
 * Arithmetic: IEEE binary64, complex numbers written out in (re, im) pairs, compiled
 * with -O2 -fno-fast-math -ffp-contract=off (no FMA contraction).  Matrices are
 * column-major, complex interleaved (re, im), leading dimension given explicitly.
 * OpenMP is used across independent quadrature nodes (a lone node: across the independent
 * columns of its rank-1 updates and its right-hand sides); the node sum is formed in
 * increasing node order afterwards, so results do not depend on the thread count.
 *
 * Pinning (tests/test_oracle_*.py, -m "not gpu"): quadrature closed forms, the
 * closed-form filters 1/(1+x^q) and 1/(1-x^q), the S:263 worked example, LU
 * reconstruction, spectral identity rho(B^-1 A) = X rho(Lambda) X^-1,
 * brute force vs scipy at n <= 64, Rayleigh-Ritz exactness on the full space.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double re, im; } cx;

static inline cx cmk(double r, double i) { cx z; z.re = r; z.im = i; return z; }
static inline cx cadd(cx a, cx b) { return cmk(a.re + b.re, a.im + b.im); }
static inline cx csub(cx a, cx b) { return cmk(a.re - b.re, a.im - b.im); }
static inline cx cmul(cx a, cx b) { return cmk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static inline cx cconj(cx a) { return cmk(a.re, -a.im); }
static inline cx cscale(cx a, double s) { return cmk(a.re * s, a.im * s); }
static inline double cabs1(cx a) { return fabs(a.re) + fabs(a.im); }
static inline double cabs2(cx a) { return hypot(a.re, a.im); }
static inline cx cdiv(cx a, cx b) {
  /* Smith's algorithm (robust complex division). */
  if (fabs(b.re) >= fabs(b.im)) {
    double r = b.im / b.re, d = b.re + b.im * r;
    return cmk((a.re + a.im * r) / d, (a.im - a.re * r) / d);
  } else {
    double r = b.re / b.im, d = b.re * r + b.im;
    return cmk((a.re * r + a.im) / d, (a.im * r - a.re) / d);
  }
}

#define AT(M, ld, i, j) ((M)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

/* ------------------------------------------------------------------------------
 * O1 — quadrature rules on [-1,1] and the partial-fraction filter (§3)
 * ------------------------------------------------------------------------------ */

/* Gauss–Legendre K-point rule: Newton on P_K from Chebyshev initial guesses
 * (S:157-165).  Nodes ascending. */
int orc_gauss_legendre(int K, double* t, double* w) {
  if (K < 1) return -1;
  for (int i = 0; i < K; ++i) {
    double x = cos(M_PI * (i + 0.75) / (K + 0.5)); /* Chebyshev-like guess, descending */
    double pk = 0.0, pkm1 = 0.0, dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      /* three-term recurrence (k+1) P_{k+1} = (2k+1) x P_k - k P_{k-1} */
      pkm1 = 1.0; pk = x;
      for (int k = 1; k < K; ++k) {
        double pn = ((2.0 * k + 1.0) * x * pk - k * pkm1) / (k + 1.0);
        pkm1 = pk; pk = pn;
      }
      dp = K * (x * pk - pkm1) / (x * x - 1.0); /* P_K'(x) */
      double dx = pk / dp;
      x -= dx;
      if (fabs(dx) < 1e-16) break;
    }
    pkm1 = 1.0; pk = x;
    for (int k = 1; k < K; ++k) {
      double pn = ((2.0 * k + 1.0) * x * pk - k * pkm1) / (k + 1.0);
      pkm1 = pk; pk = pn;
    }
    dp = K * (x * pk - pkm1) / (x * x - 1.0);
    t[K - 1 - i] = x;
    w[K - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  return 0;
}

/* Trapezoidal rule with both endpoints (Fig. 3 caption P:461-465):
 * t_k = -1 + 2k/(K-1), weights 2/(K-1) interior, 1/(K-1) at the ends. */
int orc_trapezoid_endpoint(int K, double* t, double* w) {
  if (K < 2) return -1;
  for (int k = 0; k < K; ++k) {
    t[k] = -1.0 + 2.0 * k / (K - 1);
    w[k] = (k == 0 || k == K - 1) ? 1.0 / (K - 1) : 2.0 / (K - 1);
  }
  return 0;
}

/* Composite midpoint rule on [-1,1] (reading R1: the "N_e-point trapezoidal rule" of
 * BASELINE.json whose circle filter is 1/(1+x^N_e)): t_k = -1 + (2k+1)/K, w_k = 2/K. */
int orc_midpoint(int K, double* t, double* w) {
  if (K < 1) return -1;
  for (int k = 0; k < K; ++k) { t[k] = -1.0 + (2.0 * k + 1.0) / K; w[k] = 2.0 / K; }
  return 0;
}

/* Ellipse phi(t) = c + R( cos(pi/2 (1+t)) + i a sin(pi/2 (1+t)) ) (eq. ellipses)
 * and its derivative in t. */
static void phi_ellipse(double c_re, double c_im, double R, double a, double t, cx* ph, cx* dph) {
  double th = 0.5 * M_PI * (1.0 + t);
  *ph = cmk(c_re + R * cos(th), c_im + R * a * sin(th));
  *dph = cmk(-R * 0.5 * M_PI * sin(th), R * a * 0.5 * M_PI * cos(th));
}

/* rule: 0 = midpoint ("trapezoid", R1), 1 = trapezoid with endpoints, 2 = Gauss–Legendre.
 * n_e: number of poles q for rules 0 and 1 (R1); nodes per half K for rule 2 (R3).
 * Output: q poles z (phi_k) and weights w (sigma_k) of eq. quadrature_for_pi:
 *   sigma = w_k phi'(t)/(2 pi i) for t = t_k and t~ = 2 - t_k; coinciding poles
 *   (t_k = +-1 with the endpoint rule) are merged by summing their sigma.
 * Returns q (>0) or -1 on bad arguments.  z, w must hold 2*q doubles (q <= 2*K). */
int orc_nodes(double c_re, double c_im, double R, double a, int n_e, int rule, double* z, double* w) {
  int K;
  double tk[4096], wk[4096];
  if (R <= 0 || a <= 0) return -1;
  if (rule == 0) { if (n_e < 2 || n_e % 2) return -1; K = n_e / 2; orc_midpoint(K, tk, wk); }
  else if (rule == 1) { if (n_e < 2 || n_e % 2) return -1; K = n_e / 2 + 1; orc_trapezoid_endpoint(K, tk, wk); }
  else if (rule == 2) { if (n_e < 1) return -1; K = n_e; orc_gauss_legendre(K, tk, wk); }
  else return -1;
  if (K > 2048) return -1;
  int q = 0;
  cx poles[8192], sig[8192];
  const cx two_pi_i = cmk(0.0, 2.0 * M_PI);
  for (int half = 0; half < 2; ++half) {
    for (int k = 0; k < K; ++k) {
      double t = half == 0 ? tk[k] : 2.0 - tk[k];
      cx ph, dph;
      phi_ellipse(c_re, c_im, R, a, t, &ph, &dph);
      cx s = cdiv(cscale(dph, wk[k]), two_pi_i);
      /* merge with an existing equal pole (endpoint rule only: t = +-1 give the same phi) */
      int merged = 0;
      for (int j = 0; j < q; ++j) {
        if (cabs2(csub(poles[j], ph)) <= 1e-12 * R) { sig[j] = cadd(sig[j], s); merged = 1; break; }
      }
      if (!merged) { poles[q] = ph; sig[q] = s; ++q; }
    }
  }
  for (int j = 0; j < q; ++j) {
    z[2 * j] = poles[j].re; z[2 * j + 1] = poles[j].im;
    w[2 * j] = sig[j].re; w[2 * j + 1] = sig[j].im;
  }
  return q;
}

/* Composite ("glued") contours (§5.4 "General Domain Shapes": the region is bounded
 * by segments of curves or lines parameterized separately and glued together; only phi(t)
 * changes).  Segment s is parameterized on t in [-1, 1]:
 *   kind 0, line a -> b:        phi(t) = a + (b - a)(1 + t)/2,          phi'(t) = (b - a)/2
 *   kind 1, arc c, R, th0->th1:  phi(t) = c + R e^{i th(t)}, th(t) = th0 + (th1 - th0)(1 + t)/2,
 *                                 phi'(t) = i R e^{i th(t)} (th1 - th0)/2
 * params: 5 doubles per segment (line: a_re, a_im, b_re, b_im, unused; arc: c_re, c_im, R, th0, th1).
 * The rule (0 = midpoint trapezoid, reading R18; 2 = Gauss-Legendre) with K nodes is applied on
 * every segment: pole phi(t_k), weight sigma = w_k phi'(t_k)/(2 pi i) (eq. pi / quadrature_for_pi
 * with one parameter interval per segment).  Returns q = nseg*K or -1. */
static void phi_segment(int kind, const double* p, double t, cx* ph, cx* dph) {
  if (kind == 0) {
    const double s = 0.5 * (1.0 + t);
    *ph = cmk(p[0] + (p[2] - p[0]) * s, p[1] + (p[3] - p[1]) * s);
    *dph = cmk(0.5 * (p[2] - p[0]), 0.5 * (p[3] - p[1]));
  } else {
    const double th = p[3] + (p[4] - p[3]) * 0.5 * (1.0 + t), half = 0.5 * (p[4] - p[3]);
    *ph = cmk(p[0] + p[2] * cos(th), p[1] + p[2] * sin(th));
    *dph = cmk(-p[2] * sin(th) * half, p[2] * cos(th) * half);
  }
}

int orc_contour_nodes(int nseg, const int* kind, const double* params, int K, int rule, double* z, double* w) {
  double tk[4096], wk[4096];
  if (nseg < 1 || K < 1 || K > 4096) return -1;
  if (rule == 0) orc_midpoint(K, tk, wk);
  else if (rule == 2) orc_gauss_legendre(K, tk, wk);
  else return -1;
  const cx two_pi_i = cmk(0.0, 2.0 * M_PI);
  int q = 0;
  for (int s = 0; s < nseg; ++s) {
    if (kind[s] != 0 && kind[s] != 1) return -1;
    for (int k = 0; k < K; ++k) {
      cx ph, dph;
      phi_segment(kind[s], params + 5 * s, tk[k], &ph, &dph);
      const cx sg = cdiv(cscale(dph, wk[k]), two_pi_i);
      z[2 * q] = ph.re; z[2 * q + 1] = ph.im;
      w[2 * q] = sg.re; w[2 * q + 1] = sg.im;
      ++q;
    }
  }
  return q;
}

/* rho(mu) = sum_k sigma_k / (phi_k - mu)  (eq. quadrature_for_pi). */
void orc_rho(int q, const double* z, const double* w, int nmu, const double* mu, double* out) {
  for (int i = 0; i < nmu; ++i) {
    cx m = cmk(mu[2 * i], mu[2 * i + 1]);
    cx s = cmk(0, 0);
    for (int k = 0; k < q; ++k) {
      s = cadd(s, cdiv(cmk(w[2 * k], w[2 * k + 1]), csub(cmk(z[2 * k], z[2 * k + 1]), m)));
    }
    out[2 * i] = s.re; out[2 * i + 1] = s.im;
  }
}

/* ------------------------------------------------------------------------------
 * O3/O4 — naive LU with partial pivoting and substitution (the solves of eq. Rasp,
 * P:338-345 "solving q linear systems each with BU as the right-hand-side").
 * ------------------------------------------------------------------------------ */

/* In-place LU of the n x n column-major matrix M: P M = L U, L unit lower.
 * Pivot = argmax |re|+|im| over the column, lowest row index on ties (reading R7).
 * ipiv[k] = row swapped with row k at step k (0-based, LAPACK style).
 * stats[0] = min|u_ii|, stats[1] = max|u_ii|.  Returns 0, or k+1 if u_kk == 0. */
int orc_lu(int64_t n, double* Md, int64_t ld, int32_t* ipiv, double* stats) {
  cx* M = (cx*)Md;
  int info = 0;
  double umin = INFINITY, umax = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    double best = cabs1(AT(M, ld, k, k));
    for (int64_t i = k + 1; i < n; ++i) {
      double v = cabs1(AT(M, ld, i, k));
      if (v > best) { best = v; p = i; }
    }
    ipiv[k] = (int32_t)p;
    if (p != k) {
      for (int64_t j = 0; j < n; ++j) {
        cx tmp = AT(M, ld, k, j); AT(M, ld, k, j) = AT(M, ld, p, j); AT(M, ld, p, j) = tmp;
      }
    }
    cx piv = AT(M, ld, k, k);
    double a = cabs2(piv);
    if (a < umin) umin = a;
    if (a > umax) umax = a;
    if (piv.re == 0.0 && piv.im == 0.0) { if (!info) info = (int)k + 1; continue; }
    for (int64_t i = k + 1; i < n; ++i) AT(M, ld, i, k) = cdiv(AT(M, ld, i, k), piv);
    /* the columns j of the rank-1 update are independent: threads split them (each element's
     * update sequence, and so every result bit, is the same for any thread count) */
#pragma omp parallel for schedule(static) if (n - k > 512)
    for (int64_t j = k + 1; j < n; ++j) {
      cx ukj = AT(M, ld, k, j);
      if (ukj.re == 0.0 && ukj.im == 0.0) continue;
      for (int64_t i = k + 1; i < n; ++i)
        AT(M, ld, i, j) = csub(AT(M, ld, i, j), cmul(AT(M, ld, i, k), ukj));
    }
  }
  if (stats) { stats[0] = umin; stats[1] = umax; }
  return info;
}

/* Solve with the factors of orc_lu.  trans = 0: M X = Bm;  trans = 2: M^H X = Bm
 * (the conjugate-transposed systems of eq. Lasp, reusing the same factors).
 * Bm (n x nrhs, ld ldb) is overwritten with X. */
void orc_lu_solve(int64_t n, const double* LUd, int64_t ld, const int32_t* ipiv, int64_t nrhs,
                  double* Bd, int64_t ldb, int trans) {
  const cx* LU = (const cx*)LUd;
  cx* Bm = (cx*)Bd;
  /* right-hand sides are independent (threads split them; results independent of the count) */
#pragma omp parallel for schedule(dynamic, 1) if (nrhs > 1 && n > 256)
  for (int64_t r = 0; r < nrhs; ++r) {
    cx* b = Bm + (size_t)r * (size_t)ldb;
    if (trans == 0) {
      for (int64_t k = 0; k < n; ++k) if (ipiv[k] != k) { cx t = b[k]; b[k] = b[ipiv[k]]; b[ipiv[k]] = t; }
      for (int64_t i = 0; i < n; ++i) {            /* L y = P b, L unit lower */
        cx s = b[i];
        for (int64_t j = 0; j < i; ++j) s = csub(s, cmul(AT(LU, ld, i, j), b[j]));
        b[i] = s;
      }
      for (int64_t i = n - 1; i >= 0; --i) {       /* U x = y */
        cx s = b[i];
        for (int64_t j = i + 1; j < n; ++j) s = csub(s, cmul(AT(LU, ld, i, j), b[j]));
        b[i] = cdiv(s, AT(LU, ld, i, i));
      }
    } else {
      /* M^H = U^H L^H P  =>  U^H y = b, L^H z = y, x = P^T z */
      for (int64_t i = 0; i < n; ++i) {            /* U^H lower triangular */
        cx s = b[i];
        for (int64_t j = 0; j < i; ++j) s = csub(s, cmul(cconj(AT(LU, ld, j, i)), b[j]));
        b[i] = cdiv(s, cconj(AT(LU, ld, i, i)));
      }
      for (int64_t i = n - 1; i >= 0; --i) {       /* L^H unit upper */
        cx s = b[i];
        for (int64_t j = i + 1; j < n; ++j) s = csub(s, cmul(cconj(AT(LU, ld, j, i)), b[j]));
        b[i] = s;
      }
      for (int64_t k = n - 1; k >= 0; --k) if (ipiv[k] != k) { cx t = b[k]; b[k] = b[ipiv[k]]; b[ipiv[k]] = t; }
    }
  }
}

/* C (m x p) = op(A) (m x k or k x m) * Bm (k x p); opa 0 = N, 2 = conjugate transpose.
 * Plain triple loop (the reduced matrices of R-FEAST step 4). */
void orc_gemm(int64_t m, int64_t p, int64_t k, int opa, const double* Ad, int64_t lda,
              const double* Bd, int64_t ldb, double* Cd, int64_t ldc) {
  const cx* A = (const cx*)Ad; const cx* Bm = (const cx*)Bd; cx* C = (cx*)Cd;
#pragma omp parallel for schedule(dynamic, 1) if (m * k > 65536)
  for (int64_t j = 0; j < p; ++j)
    for (int64_t i = 0; i < m; ++i) {
      cx s = cmk(0, 0);
      for (int64_t l = 0; l < k; ++l) {
        cx a = opa == 0 ? AT(A, lda, i, l) : cconj(AT(A, lda, l, i));
        s = cadd(s, cmul(a, AT(Bm, ldb, l, j)));
      }
      AT(C, ldc, i, j) = s;
    }
}

/* ------------------------------------------------------------------------------
 * O2-O6 — the projector actions (eq. Rasp; eq. Lasp P:424-439 read as R4)
 * ------------------------------------------------------------------------------ */

/* Q = sum_{j=j0}^{j1-1} w_j (z_j B - A)^{-1} (B X)      (left = 0)
 * Q = sum_{j=j0}^{j1-1} conj(w_j) (z_j B - A)^{-H} (B^H X)   (left = 1)
 * B == NULL means B = I.  stats (optional, 2*q doubles): min|u_ii|, max|u_ii| per node.
 * Returns 0, or -(j+1) for the first node with an exactly singular factor. */
int orc_project(int64_t n, int64_t m0, const double* A, int64_t lda, const double* B, int64_t ldb,
                const double* X, int64_t ldx, int q, const double* z, const double* w,
                int j0, int j1, int left, double* Q, int64_t ldq, double* stats) {
  (void)q;
  size_t nn = (size_t)n * (size_t)n, nm = (size_t)n * (size_t)m0;
  cx* R = (cx*)malloc(nm * sizeof(cx));        /* R = B X  or  B^H X */
  const cx* Ac = (const cx*)A; const cx* Bc = (const cx*)B; const cx* Xc = (const cx*)X;
#pragma omp parallel for schedule(dynamic, 1) if (n > 256)
  for (int64_t c = 0; c < m0; ++c)
    for (int64_t i = 0; i < n; ++i) {
      if (!B) { R[i + c * n] = AT(Xc, ldx, i, c); continue; }
      cx s = cmk(0, 0);
      for (int64_t l = 0; l < n; ++l) {
        cx b = left ? cconj(AT(Bc, ldb, l, i)) : AT(Bc, ldb, i, l);
        s = cadd(s, cmul(b, AT(Xc, ldx, l, c)));
      }
      R[i + c * n] = s;
    }
  int nodes = j1 - j0;
  cx* Y = (cx*)malloc((size_t)nodes * nm * sizeof(cx));
  int err = 0;
  /* nodes in parallel; a single node gets every thread inside its LU and solves instead (the
   * inner regions are inactive while this one is) */
#pragma omp parallel for schedule(dynamic, 1) if (nodes > 1)
  for (int jj = 0; jj < nodes; ++jj) {
    int j = j0 + jj;
    cx zj = cmk(z[2 * j], z[2 * j + 1]);
    cx* C = (cx*)malloc(nn * sizeof(cx));
    int32_t* piv = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    for (int64_t c = 0; c < n; ++c)                 /* C_j = z_j B - A */
      for (int64_t i = 0; i < n; ++i) {
        cx b = Bc ? AT(Bc, ldb, i, c) : cmk(i == c ? 1.0 : 0.0, 0.0);
        C[i + c * n] = csub(cmul(zj, b), AT(Ac, lda, i, c));
      }
    double st[2];
    int info = orc_lu(n, (double*)C, n, piv, st);
    if (stats) { stats[2 * j] = st[0]; stats[2 * j + 1] = st[1]; }
    if (info) {
#pragma omp critical
      { if (!err || -(j + 1) > err) err = -(j + 1); }
    }
    cx* Yj = Y + (size_t)jj * nm;
    memcpy(Yj, R, nm * sizeof(cx));
    orc_lu_solve(n, (double*)C, n, piv, m0, (double*)Yj, n, left ? 2 : 0);
    free(C); free(piv);
  }
  cx* Qc = (cx*)Q;
  for (int64_t c = 0; c < m0; ++c)
    for (int64_t i = 0; i < n; ++i) AT(Qc, ldq, i, c) = cmk(0, 0);
  for (int jj = 0; jj < nodes; ++jj) {              /* sum in increasing node order */
    int j = j0 + jj;
    cx wj = cmk(w[2 * j], w[2 * j + 1]);
    if (left) wj = cconj(wj);
    const cx* Yj = Y + (size_t)jj * nm;
    for (int64_t c = 0; c < m0; ++c)
      for (int64_t i = 0; i < n; ++i)
        AT(Qc, ldq, i, c) = cadd(AT(Qc, ldq, i, c), cmul(wj, Yj[i + c * n]));
  }
  free(R); free(Y);
  return err;
}

/* ------------------------------------------------------------------------------
 * O7 — reduced dense eigenproblem  A^ W = B^ W Lambda^  (R-FEAST step 5, P:511-512;
 * Bi-FEAST step 7, P:530-532 read as R5).  M = B^-1 A^, Householder Hessenberg,
 * complex single-shift QR (Wilkinson shift), eigenvectors by back substitution.
 * ------------------------------------------------------------------------------ */

/* Upper Hessenberg reduction H = Z^H M Z by Householder reflectors; M overwritten by H,
 * Z (m x m, ld m) receives the accumulated unitary. */
static void hessenberg(int m, cx* H, cx* Z) {
  for (int i = 0; i < m * m; ++i) Z[i] = cmk(0, 0);
  for (int i = 0; i < m; ++i) Z[i + i * m] = cmk(1, 0);
  cx* v = (cx*)malloc((size_t)m * sizeof(cx));
  for (int k = 0; k < m - 2; ++k) {
    double alpha2 = 0.0;
    for (int i = k + 1; i < m; ++i) { cx x = H[i + k * m]; alpha2 += x.re * x.re + x.im * x.im; }
    double alpha = sqrt(alpha2);
    if (alpha == 0.0) continue;
    cx x0 = H[(k + 1) + k * m];
    double ax0 = cabs2(x0);
    cx ph = ax0 > 0 ? cscale(x0, 1.0 / ax0) : cmk(1, 0);
    /* v = x + ph*alpha e1, reflector P = I - 2 v v^H / (v^H v) */
    for (int i = 0; i < m; ++i) v[i] = cmk(0, 0);
    for (int i = k + 1; i < m; ++i) v[i] = H[i + k * m];
    v[k + 1] = cadd(v[k + 1], cscale(ph, alpha));
    double vn2 = 0.0;
    for (int i = k + 1; i < m; ++i) vn2 += v[i].re * v[i].re + v[i].im * v[i].im;
    if (vn2 == 0.0) continue;
    double beta = 2.0 / vn2;
    /* H = P H */
    for (int j = 0; j < m; ++j) {
      cx s = cmk(0, 0);
      for (int i = k + 1; i < m; ++i) s = cadd(s, cmul(cconj(v[i]), H[i + j * m]));
      s = cscale(s, beta);
      for (int i = k + 1; i < m; ++i) H[i + j * m] = csub(H[i + j * m], cmul(v[i], s));
    }
    /* H = H P ; Z = Z P */
    for (int i = 0; i < m; ++i) {
      cx s = cmk(0, 0), t = cmk(0, 0);
      for (int j = k + 1; j < m; ++j) {
        s = cadd(s, cmul(H[i + j * m], v[j]));
        t = cadd(t, cmul(Z[i + j * m], v[j]));
      }
      s = cscale(s, beta); t = cscale(t, beta);
      for (int j = k + 1; j < m; ++j) {
        H[i + j * m] = csub(H[i + j * m], cmul(s, cconj(v[j])));
        Z[i + j * m] = csub(Z[i + j * m], cmul(t, cconj(v[j])));
      }
    }
    for (int i = k + 2; i < m; ++i) H[i + k * m] = cmk(0, 0);
  }
  free(v);
}

/* Complex Schur form of Hessenberg H by shifted QR with Givens rotations; Z accumulates.
 * Returns 0 or -1 if not converged within 30*m sweeps. */
static int schur_qr(int m, cx* H, cx* Z) {
  const double eps = 2.220446049250313e-16;
  int hi = m - 1, iter = 0, total = 0;
  cx* cs = (cx*)malloc((size_t)m * sizeof(cx));
  double* cc = (double*)malloc((size_t)m * sizeof(double));
  while (hi > 0) {
    /* find lo: deflation |h_{l,l-1}| <= eps (|h_ll| + |h_{l-1,l-1}|) */
    int lo = hi;
    while (lo > 0) {
      double s = cabs1(H[lo + lo * m]) + cabs1(H[(lo - 1) + (lo - 1) * m]);
      if (s == 0.0) s = 1.0;
      if (cabs1(H[lo + (lo - 1) * m]) <= eps * s) { H[lo + (lo - 1) * m] = cmk(0, 0); break; }
      --lo;
    }
    if (lo == hi) { --hi; iter = 0; continue; }
    if (++total > 30 * m) { free(cs); free(cc); return -1; }
    ++iter;
    /* Wilkinson shift from the trailing 2x2 of the active block */
    cx a = H[(hi - 1) + (hi - 1) * m], b = H[(hi - 1) + hi * m];
    cx c = H[hi + (hi - 1) * m], d = H[hi + hi * m];
    cx mu;
    if (iter % 11 == 10) {
      /* exceptional shift */
      mu = cadd(d, cmk(0.75 * cabs1(H[hi + (hi - 1) * m]), 0.0));
    } else {
      cx tr2 = cscale(cadd(a, d), 0.5);
      cx det = csub(cmul(a, d), cmul(b, c));
      cx disc = csub(cmul(tr2, tr2), det);
      /* complex sqrt */
      double r = cabs2(disc);
      double sr = sqrt(0.5 * (r + fabs(disc.re)));
      cx sq;
      if (sr == 0.0) sq = cmk(0, 0);
      else if (disc.re >= 0) sq = cmk(sr, disc.im / (2 * sr));
      else sq = cmk(fabs(disc.im) / (2 * sr), disc.im >= 0 ? sr : -sr);
      cx l1 = cadd(tr2, sq), l2 = csub(tr2, sq);
      mu = cabs2(csub(l1, d)) < cabs2(csub(l2, d)) ? l1 : l2;
    }
    /* explicit single-shift QR sweep on rows/cols lo..hi: H - mu I = QR, H = RQ + mu I */
    for (int k = lo; k <= hi; ++k) H[k + k * m] = csub(H[k + k * m], mu);
    for (int k = lo; k < hi; ++k) {
      /* Givens G_k zeroing H[k+1][k] against H[k][k]: [c s; -conj(s) c] with c real */
      cx x = H[k + k * m], y = H[(k + 1) + k * m];
      double nx = cabs2(x), ny = cabs2(y);
      double r = hypot(nx, ny);
      double cr; cx s;
      if (r == 0.0) { cr = 1.0; s = cmk(0, 0); }
      else if (nx == 0.0) { cr = 0.0; s = cscale(cconj(y), 1.0 / ny); }
      else {
        cr = nx / r;
        cx ph = cscale(x, 1.0 / nx);           /* x/|x| */
        s = cscale(cmul(ph, cconj(y)), 1.0 / r); /* s = (x/|x|) conj(y) / r */
      }
      cc[k] = cr; cs[k] = s;
      (void)ny;
      /* apply G to rows k,k+1 for columns k..m-1:  [r1; r2] = [c s; -conj(s) c][r1; r2] */
      for (int j = k; j < m; ++j) {
        cx h1 = H[k + j * m], h2 = H[(k + 1) + j * m];
        H[k + j * m] = cadd(cscale(h1, cr), cmul(s, h2));
        H[(k + 1) + j * m] = csub(cscale(h2, cr), cmul(cconj(s), h1));
      }
      (void)nx;
    }
    /* H = R G^H for columns: for each k apply to columns k,k+1, rows 0..min(k+2,hi) */
    for (int k = lo; k < hi; ++k) {
      double cr = cc[k]; cx s = cs[k];
      int rmax = k + 1;
      for (int i = 0; i <= rmax; ++i) {
        cx h1 = H[i + k * m], h2 = H[i + (k + 1) * m];
        H[i + k * m] = cadd(cscale(h1, cr), cmul(cconj(s), h2));
        H[i + (k + 1) * m] = csub(cscale(h2, cr), cmul(s, h1));
      }
      for (int i = 0; i < m; ++i) {
        cx z1 = Z[i + k * m], z2 = Z[i + (k + 1) * m];
        Z[i + k * m] = cadd(cscale(z1, cr), cmul(cconj(s), z2));
        Z[i + (k + 1) * m] = csub(cscale(z2, cr), cmul(s, z1));
      }
    }
    for (int k = lo; k <= hi; ++k) H[k + k * m] = cadd(H[k + k * m], mu);
  }
  free(cs); free(cc);
  return 0;
}

/* Reduced eigenproblem of (Ah, Bh), m x m column-major.  lam: 2m doubles; W: m x m right
 * eigenvectors (columns unit 2-norm).  Returns 0, -1 (B^ singular), -2 (QR failed). */
int orc_eig(int m, const double* Ahd, const double* Bhd, double* lam, double* Wd) {
  size_t mm = (size_t)m * (size_t)m;
  cx* Mx = (cx*)malloc(mm * sizeof(cx));
  cx* Bf = (cx*)malloc(mm * sizeof(cx));
  cx* Z = (cx*)malloc(mm * sizeof(cx));
  cx* T = Mx;
  int32_t* piv = (int32_t*)malloc((size_t)m * sizeof(int32_t));
  memcpy(Bf, Bhd, mm * sizeof(cx));
  memcpy(Mx, Ahd, mm * sizeof(cx));
  double st[2];
  int info = orc_lu(m, (double*)Bf, m, piv, st);
  if (info || st[0] < 1e-14 * st[1]) { free(Mx); free(Bf); free(Z); free(piv); return -1; }
  orc_lu_solve(m, (double*)Bf, m, piv, m, (double*)Mx, m, 0);   /* M = B^-1 A */
  hessenberg(m, T, Z);
  if (schur_qr(m, T, Z)) { free(Mx); free(Bf); free(Z); free(piv); return -2; }
  /* eigenvectors of upper-triangular T, then W = Z V */
  cx* V = Bf; /* reuse */
  double tnorm = 0.0;
  for (size_t i = 0; i < mm; ++i) tnorm = fmax(tnorm, cabs1(T[i]));
  double smin = fmax(2.220446049250313e-16 * tnorm, 1e-300);
  for (int k = 0; k < m; ++k) {
    cx lk = T[k + k * m];
    lam[2 * k] = lk.re; lam[2 * k + 1] = lk.im;
    for (int i = 0; i < m; ++i) V[i + k * m] = cmk(0, 0);
    V[k + k * m] = cmk(1, 0);
    for (int i = k - 1; i >= 0; --i) {
      cx s = cmk(0, 0);
      for (int j = i + 1; j <= k; ++j) s = cadd(s, cmul(T[i + j * m], V[j + k * m]));
      cx den = csub(T[i + i * m], lk);
      if (cabs1(den) < smin) den = cmk(smin, 0);
      V[i + k * m] = cdiv(cmk(-s.re, -s.im), den);
    }
  }
  cx* W = (cx*)Wd;
  for (int k = 0; k < m; ++k) {
    double nrm = 0.0;
    for (int i = 0; i < m; ++i) {
      cx s = cmk(0, 0);
      for (int j = 0; j <= k; ++j) s = cadd(s, cmul(Z[i + j * m], V[j + k * m]));
      W[i + k * m] = s;
      nrm += s.re * s.re + s.im * s.im;
    }
    nrm = sqrt(nrm);
    for (int i = 0; i < m; ++i) W[i + k * m] = cscale(W[i + k * m], 1.0 / nrm);
  }
  free(Mx); free(Bf); free(Z); free(piv);
  return 0;
}

/* Orthonormalise the columns of Y (n x m, ld n) in place by classical Gram–Schmidt applied
 * twice ("CGS2").  Used on U^ (and V^) before the Rayleigh–Ritz step (reading R13: P:652-653
 * "especially if orthogonalization is applied"; S:392 default ON).  A column whose norm
 * collapses below 1e-14 of its original norm is left as the (renormalised) remainder. */
static void orth_cgs2(int64_t n, int64_t m, cx* Y) {
  for (int64_t c = 0; c < m; ++c) {
    cx* y = Y + (size_t)c * (size_t)n;
    for (int pass = 0; pass < 2; ++pass) {
      for (int64_t p = 0; p < c; ++p) {
        const cx* qp = Y + (size_t)p * (size_t)n;
        cx s = cmk(0, 0);
        for (int64_t i = 0; i < n; ++i) s = cadd(s, cmul(cconj(qp[i]), y[i]));
        for (int64_t i = 0; i < n; ++i) y[i] = csub(y[i], cmul(qp[i], s));
      }
    }
    double nrm = 0.0;
    for (int64_t i = 0; i < n; ++i) nrm += y[i].re * y[i].re + y[i].im * y[i].im;
    nrm = sqrt(nrm);
    double sc = nrm > 0 ? 1.0 / nrm : 0.0;
    for (int64_t i = 0; i < n; ++i) y[i] = cscale(y[i], sc);
  }
}

/* ------------------------------------------------------------------------------
 * One FEAST iteration (R-FEAST P:503-517; Bi-FEAST P:520-537).
 * X (n x m0) in: U^(k-1); out: U^(k) = U^ W with unit columns (R14).
 * V (bi only, NULL otherwise) in: V^(k-1); out: V^(k) = V^ Z, Z = (B^ W)^-H (R5).
 * Outputs (host): lam (2*m0), resid (m0) = ||A x - l B x|| / (||A||_F ||x||) (R11),
 * resid_paper (m0) = ||A x - l B x|| / ||x||, flags (m0): bit0 inside,
 * bit1 candidate (inside and resid_paper <= 1e-4).
 * ortho != 0: orthonormalise U^ (and V^) before the reduction (reading R13).
 * Returns 0 or a negative error.
 * ------------------------------------------------------------------------------ */
int orc_feast_iterate(int64_t n, int64_t m0, const double* A, int64_t lda, const double* B, int64_t ldb,
                      int q, const double* z, const double* w, double c_re, double c_im, double R, double a,
                      double* X, int64_t ldx, double* V, int64_t ldv,
                      double* lam, double* resid, double* resid_paper, int32_t* flags, int ortho) {
  size_t nm = (size_t)n * (size_t)m0, mm = (size_t)m0 * (size_t)m0;
  cx* Q = (cx*)malloc(nm * sizeof(cx));
  cx* QL = V ? (cx*)malloc(nm * sizeof(cx)) : NULL;
  int e = orc_project(n, m0, A, lda, B, ldb, X, ldx, q, z, w, 0, q, 0, (double*)Q, n, NULL);
  if (e) { free(Q); free(QL); return -3; }
  if (V) {
    e = orc_project(n, m0, A, lda, B, ldb, V, ldv, q, z, w, 0, q, 1, (double*)QL, n, NULL);
    if (e) { free(Q); free(QL); return -3; }
  }
  if (ortho) { orth_cgs2(n, m0, Q); if (QL) orth_cgs2(n, m0, QL); }
  const cx* Ql = V ? QL : Q;
  cx* AQ = (cx*)malloc(nm * sizeof(cx));
  cx* BQ = (cx*)malloc(nm * sizeof(cx));
  orc_gemm(n, m0, n, 0, A, lda, (double*)Q, n, (double*)AQ, n);
  if (B) orc_gemm(n, m0, n, 0, B, ldb, (double*)Q, n, (double*)BQ, n);
  else memcpy(BQ, Q, nm * sizeof(cx));
  cx* Ah = (cx*)malloc(mm * sizeof(cx));
  cx* Bh = (cx*)malloc(mm * sizeof(cx));
  orc_gemm(m0, m0, n, 2, (double*)Ql, n, (double*)AQ, n, (double*)Ah, m0);
  orc_gemm(m0, m0, n, 2, (double*)Ql, n, (double*)BQ, n, (double*)Bh, m0);
  cx* W = (cx*)malloc(mm * sizeof(cx));
  e = orc_eig((int)m0, (double*)Ah, (double*)Bh, lam, (double*)W);
  if (e) { free(Q); free(QL); free(AQ); free(BQ); free(Ah); free(Bh); free(W); return e == -1 ? -7 : -8; }
  /* X = Q W, columns scaled to unit norm (scale folded into W) */
  cx* Xc = (cx*)X;
  orc_gemm(n, m0, m0, 0, (double*)Q, n, (double*)W, m0, X, ldx);
  double anorm = 0.0;
  const cx* Ac = (const cx*)A;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) { cx v = AT(Ac, lda, i, j); anorm += v.re * v.re + v.im * v.im; }
  anorm = sqrt(anorm);
  for (int64_t c = 0; c < m0; ++c) {
    double nrm = 0.0;
    for (int64_t i = 0; i < n; ++i) { cx v = AT(Xc, ldx, i, c); nrm += v.re * v.re + v.im * v.im; }
    nrm = sqrt(nrm);
    double s = nrm > 0 ? 1.0 / nrm : 0.0;
    for (int64_t i = 0; i < n; ++i) AT(Xc, ldx, i, c) = cscale(AT(Xc, ldx, i, c), s);
    for (int64_t i = 0; i < m0; ++i) W[i + c * m0] = cscale(W[i + c * m0], s);
  }
  if (V) {
    /* Z = (B^ W)^-H  => solve (B^ W)^H Z = I */
    cx* BW = (cx*)malloc(mm * sizeof(cx));
    cx* Zm = (cx*)malloc(mm * sizeof(cx));
    orc_gemm(m0, m0, m0, 0, (double*)Bh, m0, (double*)W, m0, (double*)BW, m0);
    int32_t* piv = (int32_t*)malloc((size_t)m0 * sizeof(int32_t));
    double st[2];
    orc_lu(m0, (double*)BW, m0, piv, st);
    for (size_t i = 0; i < mm; ++i) Zm[i] = cmk(0, 0);
    for (int64_t i = 0; i < m0; ++i) Zm[i + i * m0] = cmk(1, 0);
    orc_lu_solve(m0, (double*)BW, m0, piv, m0, (double*)Zm, m0, 2);
    orc_gemm(n, m0, m0, 0, (double*)QL, n, (double*)Zm, m0, V, ldv);
    free(BW); free(Zm); free(piv);
  }
  /* residuals with the normalised Ritz vectors (R11) and flags */
  orc_gemm(n, m0, m0, 0, (double*)AQ, n, (double*)W, m0, (double*)Q, n);   /* Q <- A X */
  orc_gemm(n, m0, m0, 0, (double*)BQ, n, (double*)W, m0, (double*)AQ, n);  /* AQ <- B X */
  for (int64_t c = 0; c < m0; ++c) {
    cx l = cmk(lam[2 * c], lam[2 * c + 1]);
    double r2 = 0.0, x2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      cx rv = csub(Q[i + c * n], cmul(l, AQ[i + c * n]));
      r2 += rv.re * rv.re + rv.im * rv.im;
      cx xv = AT(Xc, ldx, i, c);
      x2 += xv.re * xv.re + xv.im * xv.im;
    }
    double rp = sqrt(r2) / sqrt(x2);
    resid_paper[c] = rp;
    resid[c] = rp / anorm;
    double u = (l.re - c_re) / R, v = (l.im - c_im) / (R * a);
    int inside = (u * u + v * v) < 1.0;
    flags[c] = (inside ? 1 : 0) | ((inside && rp <= 1e-4) ? 2 : 0);
  }
  free(Q); free(QL); free(AQ); free(BQ); free(Ah); free(Bh); free(W);
  return 0;
}

/* Host-thread control for the timing legs (bench.py cpu_baseline / --impl reference): the OpenMP
 * team size used across nodes (a launcher may have set OMP_NUM_THREADS=1 before this library
 * was loaded).  n > 0 sets it; returns the current maximum.  No arithmetic. */
int orc_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}
