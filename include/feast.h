/*
 * feast.h — C ABI of the B200-native non-Hermitian FEAST quadrature projector
 * (Tang, Kestyn & Polizzi, arXiv 1404.2891).  Library: paper_1404_2891_b200/libfeast_b200.so
 *
 * Problem (§2): A x = lambda B x, A, B dense n x n complex128.
 * The contour (eq. ellipses) is the ellipse
 *     phi(t) = c + r ( cos(pi/2 (1+t)) + i * aspect * sin(pi/2 (1+t)) ),  t in [-1, 3]
 * with real semi-axis r and imaginary semi-axis r*aspect (reading R2 in DESIGN.md).
 * A quadrature rule on [-1,1], applied on both halves t and 2-t (eq. pi), gives
 * q poles z_j = phi_k and weights w_j = sigma_k (eq. quadrature_for_pi), i.e. the
 * rational filter rho(mu) = sum_j w_j / (z_j - mu).
 *
 * The hot path (eq. Rasp; eq. Lasp, P:424-439 read as R4):
 *     Q  = sum_j      w_j  (z_j B - A)^{-1} (B X)
 *     QL = sum_j conj(w_j) (z_j B - A)^{-H} (B^H V)
 * computed as: shift C_j = z_j B - A, blocked LU with partial pivoting P_j C_j = L_j U_j,
 * multi-RHS substitution, fused weighted accumulation — all in this library's sm_100a kernels.
 *
 * CONVENTIONS (every entry point)
 *   - Matrices are COLUMN-MAJOR complex128, interleaved (re, im) — the bytes of
 *     torch.complex128 / cuDoubleComplex / C99 double _Complex.  "ld" is the leading
 *     dimension in complex elements, ld >= n (or >= m0 for m0 x m0 matrices).
 *   - Matrix arguments are DEVICE pointers (16-byte aligned), unless marked (host).
 *   - Streams: every call is ordered after the work already enqueued on the stream given to
 *     feast_init (the caller's stream) and before anything enqueued there afterwards.  The
 *     library runs its kernels on its own stream (forked from / joined to the caller's with
 *     events) so that a repeated projector call can be captured once into a CUDA graph and
 *     replayed (2nd identical call captured, later ones replayed; FEAST_GRAPH=0 disables).
 *     Calls return after synchronising the library stream (host outputs valid on return).
 *   - The caller owns every matrix and the workspace; the library never frees caller memory.
 *   - Return value: 0 = ok, < 0 = error (result not valid), > 0 = warning (result valid).
 *     No exception or exit() crosses the ABI; feast_last_error() has the message.
 *   - A handle is not re-entrant; use one handle per stream.
 *
 * MULTI-GPU (§5.5: parallelism over the linear systems)
 *   Rank r of `world` owns the contiguous node block [r q/world, (r+1) q/world) (reading R17);
 *   q % world must be 0.  Every projector call (feast_project, _left, _bi, feast_estimate_count,
 *   feast_iterate) returns the FULL node sum on every rank: after its own nodes it performs the
 *   node sum across ranks (§8(a) a6) as one SUM all-reduce of the n x m0 block(s) (Q and QL
 *   packed into one buffer) through the callback registered with feast_set_allreduce (the
 *   Python binding registers torch.distributed.all_reduce: NCCL on GPUs).  With world > 1 and
 *   no callback these calls return FEAST_E_COMM, unless feast_set_partial(h, 1) asked for this
 *   rank's partial sum (the caller then sums over ranks itself).
 */
#ifndef FEAST_B200_H
#define FEAST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct feast_ctx* feast_handle;

/* Quadrature rules (readings R1, R3):
 *  FEAST_RULE_TRAPEZOID           composite midpoint rule with K = n_e/2 points on [-1,1]:
 *                                 q = n_e poles at theta_j = 2 pi (j + 1/2)/q on a circle,
 *                                 rho = 1/(1 + x^q) (BASELINE.json closed form); n_e even >= 2.
 *  FEAST_RULE_TRAPEZOID_ENDPOINT  the paper's trapezoid with both endpoints:
 *                                 K = n_e/2 + 1 points, q = 2(K-1) = n_e poles, rho = 1/(1 - x^q).
 *  FEAST_RULE_GAUSS_LEGENDRE      K = n_e Gauss-Legendre points per half, q = 2 n_e. */
enum { FEAST_RULE_TRAPEZOID = 0, FEAST_RULE_TRAPEZOID_ENDPOINT = 1, FEAST_RULE_GAUSS_LEGENDRE = 2 };

/* R-FEAST (right projector only) or Bi-FEAST (both projectors). */
enum { FEAST_RIGHT = 0, FEAST_BI = 1 };

enum {
  FEAST_OK = 0,
  FEAST_E_ARG = -1,       /* invalid argument (sizes, radii, rule, q % world, null pointer, ld) */
  FEAST_E_NOMEM = -2,     /* workspace missing or too small */
  FEAST_E_SINGULAR = -3,  /* some node's min|u_ii|/max|u_ii| < 1e-14 or an exact zero pivot;
                             Q is still written; feast_node_stats names the node */
  FEAST_E_CUDA = -4,      /* CUDA / cuSOLVER failure (message in feast_last_error) */
  FEAST_E_COMM = -5,      /* the registered all-reduce callback failed, or world > 1 without one */
  FEAST_E_STATE = -6,     /* call out of order (e.g. no workspace bound) */
  FEAST_E_REDUCED = -7,   /* reduced eigenproblem failed (B^ singular / QR failure) */
  FEAST_W_ILLCOND = 1     /* some node's pivot ratio < 1e-10 (near-singular shifted matrix) */
};

/* Create a handle.
 *  n >= 1, 1 <= m0 <= n         problem size and subspace width (p in the paper)
 *  c_re, c_im, r, aspect        contour centre, real semi-axis r > 0, aspect a > 0
 *  n_e, rule                    quadrature (see FEAST_RULE_*)
 *  mode                         FEAST_RIGHT or FEAST_BI
 *  b_is_identity                non-zero when B = I (B pointers may then be NULL)
 *  rank, world                  node sharding (world >= 1, 0 <= rank < world, q % world == 0)
 *  max_batch                    nodes factored concurrently (0 = all owned nodes that fit:
 *                               feast_workspace_bytes shrinks the batch until the workspace
 *                               takes at most 90 % of the free device memory); bounds the
 *                               workspace at max_batch * 16 n^2 bytes plus blocks
 *  cuda_stream                  cudaStream_t the work is enqueued on (NULL = legacy stream)
 * Errors: FEAST_E_ARG, FEAST_E_CUDA. */
int feast_init(feast_handle* h, int64_t n, int64_t m0, double c_re, double c_im, double r,
               double aspect, int32_t n_e, int32_t rule, int32_t mode, int32_t b_is_identity,
               int32_t rank, int32_t world, int32_t max_batch, void* cuda_stream);

/* Real-pencil mode (SURVEY NEXT-2b; the paper's real application pencils): when A and B
 * are real-valued (zero imaginary parts) and the contour is symmetric about the real axis
 * (c_im = 0), the pole pair {z, conj z} shares one LU, since C(conj z) = conj(C(z)):
 *     (conj z B - A)^-1 R = conj( (z B - A)^-1 conj(R) ),
 * so each pair is factored once with the right-hand sides [R | conj R] (left solves alike with
 * [R_L | conj R_L]) — half the LU work.  Poles on the real axis stay single units.  The
 * factorisation units are then the orbits: rank ownership, max_batch and feast_nodes' j0/j1
 * count orbits (orbits % world must be 0).  Must be called before feast_workspace_bytes /
 * feast_bind_workspace (the augmented block is n x (n + 2 m0) per unit).  Returns FEAST_E_ARG if
 * the contour is not symmetric or the poles do not pair up, FEAST_E_STATE after the workspace
 * is bound or with the factor cache on.  Every projector call checks the premise on the device:
 * FEAST_E_ARG ("A or B has a nonzero imaginary part") and Q invalid if it fails.
 * enable = 0 restores per-node factorisation. */
int feast_set_real_pencil(feast_handle h, int32_t enable);

/* Complex-symmetric pencil mode (SURVEY NEXT-2a; the paper's complex-symmetric FEM / PML
 * pencils with Bi-FEAST): the caller asserts A^T = A and B^T = B.  Then
 * C_j^T = C_j and the left solve is a right solve of the conjugated block,
 *     C_j^-H (B^H V) = conj( C_j^-1 conj(B^H V) ),
 * so in FEAST_BI handles the left block rides along the right solves as m0 extra columns of the
 * augmented system (fused forward substitution, one back substitution for both blocks) instead
 * of a separate conjugate-transposed substitution.  Q_L = conj(sum_j w_j C_j^-1 conj(B^H V)).
 * Same ordering rule as feast_set_real_pencil (before the workspace); exclusive with it.
 * The symmetry is the caller's premise (not checked). */
int feast_set_complex_symmetric(feast_handle h, int32_t enable);

/* Composite ("glued") contour (§5.4 "General Domain Shapes": only the
 * parameterization phi(t) changes).  Replaces the ellipse of feast_init by nseg segments, each on
 * t in [-1, 1], counter-clockwise, end of segment s = start of segment s+1 (closed):
 *   kind[s] = 0  line a -> b:        params[5s..5s+3] = a_re, a_im, b_re, b_im   (5s+4 unused)
 *   kind[s] = 1  arc  c + R e^{i th}: params[5s..5s+4] = c_re, c_im, R, th0, th1 (th1 > th0: ccw)
 * rule: FEAST_RULE_TRAPEZOID (composite midpoint rule, reading R18) or FEAST_RULE_GAUSS_LEGENDRE,
 * k_per_segment nodes on every segment: poles phi(t_k), weights w_k phi'(t_k)/(2 pi i), q = nseg*k.
 * Before the workspace is bound (FEAST_E_STATE after); FEAST_E_ARG for an open or clockwise chain,
 * bad kinds/radii, or q % world != 0.  feast_iterate's inside flags then use the crossing number
 * of the contour polyline. */
int feast_set_contour(feast_handle h, int32_t nseg, const int32_t* kind, const double* params, int32_t k_per_segment,
                      int32_t rule);

/* The rational filter of the handle's quadrature, rho(mu) = sum_j w_j / (z_j - mu) (eq.
 * quadrature_for_pi), at npts host points mu (2*npts doubles, complex interleaved)
 * into rho (host, 2*npts doubles): the eta(r) / filter-gap diagnostics. */
int feast_filter(feast_handle h, int64_t npts, const double* mu, double* rho);

/* Device workspace size in bytes for this handle (caller allocates, e.g. with torch). */
int feast_workspace_bytes(feast_handle h, size_t* bytes);

/* Bind caller-owned device memory (>= feast_workspace_bytes, 256-byte aligned). */
int feast_bind_workspace(feast_handle h, void* dev_ptr, size_t bytes);

/* Quadrature data (host outputs): *q; z, w = 2*q doubles each (complex interleaved poles
 * z_j and weights w_j); *j0, *j1 = this rank's owned range of factorisation units (nodes; in
 * real-pencil mode, conjugate-pole orbits in increasing primary-node order).  Any pointer may
 * be NULL. */
int feast_nodes(feast_handle h, int32_t* q, double* z, double* w, int32_t* j0, int32_t* j1);

/* Right projector (eq. Rasp), node-summed over the ranks (see MULTI-GPU):
 *   Q = sum_j w_j (z_j B - A)^{-1} (B X)       (B = NULL when b_is_identity)
 * A, B: n x n; X, Q: n x m0.  Q is overwritten (X and Q must not alias).
 * Returns FEAST_OK, FEAST_W_ILLCOND, FEAST_E_SINGULAR, FEAST_E_ARG, FEAST_E_STATE, FEAST_E_CUDA,
 * FEAST_E_COMM (world > 1: no callback registered and partial mode off, or the callback failed). */
int feast_project(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb,
                  const void* X, int64_t ldx, void* Q, int64_t ldq);

/* Left projector (eq. Lasp, P:424-439 read as R4), node-summed over the ranks:
 *   QL = sum_j conj(w_j) (z_j B - A)^{-H} (B^H V)
 * solved with the conjugate-transposed factors of the same LU. */
int feast_project_left(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb,
                       const void* V, int64_t ldv, void* QL, int64_t ldql);

/* Both projectors from ONE factorisation per node (Bi-FEAST steps 4-5):
 * Q as feast_project (from X) and QL as feast_project_left (from V). */
int feast_project_bi(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb,
                     const void* X, int64_t ldx, const void* V, int64_t ldv,
                     void* Q, int64_t ldq, void* QL, int64_t ldql);

/* Reduced matrices (R-FEAST step 4; Bi-FEAST step 6):
 *   Ahat = QL^H A Q,  Bhat = QL^H B Q      (QL = Q in R-FEAST: pass QL = NULL)
 * Ahat, Bhat: m0 x m0 device, ld >= m0.  B = NULL when b_is_identity.  Q (QL) must be the
 * node-summed block.  With world > 1 and an all-reduce callback registered, the rows are
 * sharded: rank r multiplies rows [r n/P, (r+1) n/P) of A (B) and the m0 x m0 partials are
 * all-reduced through the callback, so every rank returns the complete Ahat, Bhat. */
int feast_reduce(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb,
                 const void* Q, int64_t ldq, const void* QL, int64_t ldql,
                 void* Ahat, int64_t ldah, void* Bhat, int64_t ldbh);

/* Eigenvalue-count estimate (the count m of eigenvalues inside the
 * contour decides whether m0 >= m): Q = rho(B^-1 A) U for a caller-supplied random block U
 * (n x m0, entries with E[u u^H] = I, e.g. CN(0,1)), then the Hutchinson trace estimate
 *     *estimate = Re tr(U^H Q) / m0  ~  Re tr rho(B^-1 A) = Re sum_i rho(lambda_i)  ~  m,
 * since rho ~ 1 inside and ~ 0 outside the contour (the expectation is exact; the standard
 * deviation falls like 1/sqrt(m0)).  With world > 1, Q is all-reduced over the ranks (through
 * the registered callback) before the trace, so every rank returns the same estimate.
 * U, Q: device, column-major, ld >= n; estimate: host. */
int feast_estimate_count(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb,
                         const void* U, int64_t ldu, void* Q, int64_t ldq, double* estimate);

/* All-reduce callback for world > 1: sum `count` float64 values at device pointer `buf`
 * across ranks, in place, ordered on `cuda_stream` (the library's stream: the callback must
 * enqueue its collective there, or complete it before returning); return 0 on success. */
typedef int (*feast_allreduce_fn)(void* buf, int64_t count, void* cuda_stream, void* user);
int feast_set_allreduce(feast_handle h, feast_allreduce_fn fn, void* user);

/* Partial mode (world > 1): enable = 1 makes feast_project / _left / _bi / feast_estimate_count
 * return this rank's PARTIAL sum over its own nodes [j0, j1) with no collective (for callers
 * that reduce over ranks themselves, or several "virtual ranks" driven from one process).
 * feast_iterate then returns FEAST_E_STATE.  Default 0 (full node sum through the callback). */
int feast_set_partial(feast_handle h, int32_t enable);

/* One FEAST iteration (R-FEAST P:503-517 / Bi-FEAST P:520-537):
 *   project (+ node sum over the ranks), orthonormalise U^ (and V^) (reading R13), reduce (with
 *   world > 1 the rows of A Q, B Q and of the residual block A x - l B x are sharded over the
 *   ranks: the m0 x m0 partials and the m0 squared residual norms are all-reduced), solve the
 *   m0 x m0 eigenproblem (outside the hot path; cuSOLVER), X <- U^ W with unit columns,
 *   Bi: V <- V^ Z with Z = (B^ W)^-H (reading R5).
 * X (n x m0, device) in/out; V (bi only, else NULL) in/out.
 * Host outputs (may be NULL): ritz (2*m0 doubles, complex interleaved), resid (m0) =
 *   ||A x - l B x||_2 / (||A||_F ||x||_2) (reading R11), flags (m0): bit0 = Ritz value
 *   inside the contour, bit1 = candidate (inside and ||A x - l B x||/||x|| <= 1e-4).
 * Returns as feast_project, plus FEAST_E_REDUCED, FEAST_E_COMM. */
int feast_iterate(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb,
                  void* X, int64_t ldx, void* V, int64_t ldv,
                  double* ritz, double* resid, int32_t* flags);

/* ---- NEXT-3: count estimate, candidate monitors, filter-gap report ---------- */

/* Eigenvalue-count estimate of Bi-FEAST ("the eigenvalues of V^^H B U^ (U^, V^ from
 * Steps 4 and 5 of Bi-FEAST)"): U^ = rho(B^-1 A) U into Q and V^ = the left projector of V into
 * QL (as feast_project_bi, node-summed over the ranks), then the eigenvalues mu of the m0 x m0
 * matrix V^^H B U^ (cuSOLVER Xgeev; outside the hot path), sorted by decreasing modulus into mu
 * (host, 2*m0 doubles, complex interleaved; may be NULL), and *count = #{|mu| >= 1/4}.
 * Reading R21: with V^H B U = I (e.g. V = U (U^H B U)^-H, reading R6, or any Bi-FEAST iterate),
 * V^^H B U^ = V^H B rho(B^-1 A)^2 U, whose eigenvalues are rho(lambda_i)^2 when U spans
 * eigenvectors (or is square) and approach the dominant rho(lambda_i)^2 as the iteration
 * converges; 1/4 = (1/2)^2 counts |rho(lambda)| >= 1/2, the filter's half height (on a circle
 * exactly the eigenvalues inside).  From random U, V at the first iteration the estimate is rough.
 * FEAST_BI handles only (FEAST_E_STATE otherwise).  Returns as feast_project_bi, plus
 * FEAST_E_REDUCED if the eigensolver fails. */
int feast_estimate_count_bi(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb,
                            const void* U, int64_t ldu, const void* V, int64_t ldv,
                            void* Q, int64_t ldq, void* QL, int64_t ldql, double* mu, int32_t* count);

/* enable = 1: every Bi-FEAST feast_iterate also forms V^^H B U^ of its steps 4-5 (from the R factors
 * of the orthonormalisation: R_l^H (V_o^H B U_o) R_q, m0^3 work) and its eigenvalues (Xgeev, no
 * vectors): the count estimate above, tracked along the iteration (feast_monitors). */
int feast_set_count_estimate(feast_handle h, int32_t enable);

/* Monitors of the last feast_iterate (host outputs, any may be NULL), P:695-712:
 *   *res_k   = Res_(k) = max ||A u_j - l_j B u_j|| / ||u_j|| over the candidates (-1: none)
 *   trace_k  = trace_(k) = sum of the candidate Ritz values l_j (2 doubles: re, im)
 *   *ncand   = number of candidates (inside the contour and that residual <= 1e-4)
 *   mu, *count: eig(V^^H B U^) sorted by decreasing modulus and the count estimate of that
 *              iteration (feast_set_count_estimate on, Bi-FEAST; else *count = -1, mu zeros). */
int feast_monitors(feast_handle h, double* res_k, double* trace_k, int32_t* ncand, double* mu, int32_t* count);

/* Filter-gap report (§4; SPEC FilterGapReport): for nl eigenvalues lam (host, 2*nl
 * doubles, e.g. a full spectrum of a small or synthetic problem), gamma_j = rho(lambda_j) of this
 * handle's quadrature, numbered |gamma_1| >= ... >= |gamma_nl| (stable on ties):
 *   abs_sorted (nl) = |gamma_j| in that order, order (nl) = the input index of each,
 *   *m_inside = #{lambda inside the contour}, *m_prime = the smallest l >= (last position of an
 *   inside eigenvalue) with a strict gap |gamma_{l+1}| < |gamma_l| (a relative difference <= 1e-12
 *   is a tie, reading R22), *eps = |gamma_{p+1} / gamma_{m'}|, *log10_gap =
 *   log10 |rho(lambda_{p+1}) / rho(lambda_m)|; NaN when p >= nl or m (m') = 0.
 * Host computation; any output may be NULL. */
int feast_filter_gap(feast_handle h, int64_t nl, const double* lam, int64_t p, double* abs_sorted, int32_t* order,
                     int32_t* m_inside, int32_t* m_prime, double* eps, double* log10_gap);

/* Asynchronous mode (enable = 1): feast_project / _left / _bi and feast_reduce return as soon as
 * their work (including the node-sum collective) is enqueued on the stream, without a host
 * synchronisation, so consecutive calls pipeline.  The pivot statistics of each projection are
 * copied to pinned host memory on the stream; feast_sync (or feast_node_stats) waits for them
 * and returns the status the synchronous call would have returned (FEAST_OK, FEAST_W_ILLCOND,
 * FEAST_E_SINGULAR for the LAST projection).  Results are valid on the caller's stream order as
 * usual.  feast_iterate and the count estimates read results on the host and always judge.
 * Default 0 (every call synchronises and returns its own status). */
int feast_set_async(feast_handle h, int32_t enable);
int feast_sync(feast_handle h);

/* Pivot diagnostics of the last projection (host outputs): min_rel_pivot[q] =
 * min|u_ii| / max|u_ii| per node (owned nodes only; others are set to -1), *worst_node =
 * index of the smallest ratio.  Either pointer may be NULL. */
int feast_node_stats(feast_handle h, double* min_rel_pivot, int32_t* worst_node);

/* Factor-once reuse across calls (the paper's lever P:912-913 "each linear system
 * can be factored just once for the entire iterative process").  enable = 1 turns it on and
 * invalidates any cached factors; while on, a projection whose A and B pointers equal those of
 * the call that factored skips a2-a3 and runs only the substitutions on the cached L_j, U_j, P_j.
 * The caller must call feast_factor_cache(h, 1) again after modifying A or B in place.
 * Requires all owned nodes resident (max_batch 0 or >= q/world): FEAST_E_NOMEM otherwise.
 * enable = 0 turns it off (every call refactors: the timed hot path of bench.py). */
int feast_factor_cache(feast_handle h, int32_t enable);

/* Number of this library's kernels launched by the last call (for bench accounting). */
int64_t feast_last_launch_count(feast_handle h);

/* Per-kernel-class timing (bench roofline accounting).  feast_profile(h, 1) starts recording
 * a CUDA-event pair around every launch of this library on the launching stream (and clears
 * earlier records); feast_profile(h, 2) does the same with every launch serialised on one
 * stream (no lookahead, no concurrent node groups, no graph), so an event pair brackets only
 * its own kernel; feast_profile(h, 0) stops.  feast_profile_summary aggregates the records of
 * one class: launches, summed event time (ms), algorithmic flops and algorithmic bytes
 * (DESIGN.md "Roofline" defines them per class).  Classes: */
enum { FEAST_K_SHIFT = 0, FEAST_K_PANEL = 1, FEAST_K_LASWP = 2, FEAST_K_TRSM = 3, FEAST_K_ZGEMM = 4,
       FEAST_K_PERM = 5, FEAST_K_ACCUM = 6, FEAST_K_OTHER = 7 };
int feast_profile(feast_handle h, int32_t enable);
int feast_profile_summary(feast_handle h, int32_t kclass, int64_t* launches, double* ms, double* flops,
                          double* bytes);
/* The recorded launches one by one (a timeline; tools/timeline.py): class, stream (2g = node
 * group g's main stream, 2g + 1 its lookahead side stream; group 0 = the handle's own stream
 * pair; -1 other), start / end in ms relative to the first
 * record's start, algorithmic flops.  Host arrays of max_records entries (any may be NULL);
 * *count = number of records.  Synchronises the device. */
int feast_profile_records(feast_handle h, int64_t max_records, int32_t* kclass, int32_t* stream, double* t0_ms,
                          double* t1_ms, double* flops, int64_t* count);

/* Message for the last error on this handle ("" if none).  Valid until the next call. */
const char* feast_last_error(feast_handle h);

/* Library version string. */
const char* feast_version(void);

/* Free the handle (not the caller's memory). */
void feast_destroy(feast_handle h);

#ifdef __cplusplus
}
#endif
#endif /* FEAST_B200_H */
