// feast_api.cu — the C ABI (include/feast.h): handle, contour nodes, workspace, the projector
// driver (shift -> blocked LU -> multi-RHS substitution -> weighted accumulation, batched over
// the nodes this rank owns), the reduced matrices and one FEAST iteration.
//
// Paper map: nodes = eq. ellipses / pi / quadrature_for_pi; projector = eq. Rasp
// and eq. Lasp (reading R4); iteration = Algorithms R-FEAST
// and Bi-FEAST; monitoring = P:695-712.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/feast.h"
#include "common.cuh"
#include "kernels.h"
#include "prof.h"

using feast::Batched;
using feast::ZgemmArgs;

struct feast_ctx {
  int64_t n = 0, m0 = 0;
  double c_re = 0, c_im = 0, r = 0, aspect = 1;
  int n_e = 0, rule = 0, mode = 0;
  bool b_id = true;
  int rank = 0, world = 1, q = 0, j0 = 0, j1 = 0, batch = 1, max_batch = 0;
  std::vector<double2> z, w;
  // Factorisation UNITS: the nodes, or in real-pencil mode (NEXT-2b) the orbits {z, conj z} of
  // conjugate poles, which share one LU (C(conj z) = conj(C(z)) for real A, B).  j0/j1 and the
  // batches index units.  Per unit: pole zu (primary node), weight wu, partner weight wpu (0 if
  // the pole is real), primary node unode, partner node upart (-1).
  // composite contour (NEXT-4): segments replace the ellipse when non-empty
  struct Seg { int kind; double p[5]; };
  std::vector<Seg> segs;
  int seg_k = 0, seg_rule = 0;
  std::vector<double2> poly;          // closed polyline of the contour (inside test)
  bool real = false;
  bool csym = false;                  // A^T = A, B^T = B: left block through the right solves (NEXT-2a)
  int nu = 0;
  int64_t mr = 0;                     // right-hand-side columns per unit: m0, or 2 m0 ([R | conj R])
  std::vector<double2> zu, wu, wpu;
  std::vector<int> unode, upart;
  cudaStream_t stream = nullptr;      // the library's own stream (capturable into CUDA graphs)
  cudaStream_t caller = nullptr;      // the caller's stream: every call is ordered after / before it
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  bool own_stream = false;
  int nb = 64;
  feast::PanelCfg pcfg{};
  int smem_cs = 0;   // cluster size of the shared-memory panel kernel for the full height (0: too tall)
  int smem_cs_max = 16;  // largest cluster the shared-memory panel may use (FEAST_CS_MAX)
  bool panel_one_row = false;  // 256 threads x 1 row panels: set when <= 4 units are owned (latency-bound)
  bool lookahead = true;
  bool cache_on = false, cache_valid = false;   // factor-once reuse across calls
  const void *cache_A = nullptr, *cache_B = nullptr;
  int64_t nbo = 256;                  // outer block (trailing-update K); multiple of 64
  int64_t solve_nb = 256;             // outer block of the substitutions (FEAST_SOLVE_NB, multiple of 64)
  // fused DMMA block triangular solves (btrsm.cu) instead of the 64-row launch chains (FEAST_BTRSM=1).
  // Correct (tests) but not faster on B200: C2 17.26 vs 16.43 ms, C4 13.020 vs 13.022 s per step —
  // its parallelism is N/32 x batch CTAs that each run the whole <= 256-row solve, which delays a
  // node group's chain (C2) and under-fills the GPU in the substitutions (N = m0)
  bool btrsm = false;
  // FEAST_SUBST_DOT=1 (default for n >= 8192): substitutions in dot form (left-looking): before its diagonal block is
  // solved, an outer block takes ALL the solved rows' contribution in one GEMM with a long K
  // (M = N-block rows, K = rows solved so far) instead of pushing its own contribution to every
  // later block (right-looking: M = rows still to solve, K = the block)
  bool subst_dot = false;
  // FEAST_U12_DOT: the outer U12 = L11^-1 A12 in dot form (left-looking): the 64-row block i of
  // the outer block first takes the solved blocks' contribution in ONE GEMM (M = 64, K = 64 i)
  // and is then multiplied by its 64x64 inverse — C read / written once per block instead of the
  // right-looking K = 64 updates of every later block (M = NBO - 64 (i + 1)).  1: when the dot
  // grid (64-row tiles x N tiles x batch) fills a wave of 444 CTAs; 2: always (tests); 0: off
  int u12_dot = 0;
  // FEAST_SUBST_INNER_DOT: the 64-row blocks INSIDE a substitution outer block in dot form too
  // (M = 64, K = the block's solved rows, C read / written once per block); 1: with subst_dot when
  // the grid (64-row tiles x N tiles x batch) fills a wave of 444 CTAs; 2: always (tests); 0: off
  int inner_dot = 1;
  // FEAST_SUBST_JOIN=1: substitutions once over the whole batch after joining the node groups
  // (measured no faster: C2 16.52 vs 16.39 ms, C4 12.972 vs 12.967 s)
  bool subst_join = false;
  bool panel_swap = true;             // swaps fused into the shared-memory panel (FEAST_PANEL_SWAP=0: separate)
  int64_t wp = 32;                    // cluster-panel width (divides 64)
  int64_t wide_panel_rows = 768;      // 64-wide cluster panels once n - k <= this (FEAST_WIDE_ROWS)
  cudaStream_t side = nullptr;        // high-priority stream for the lookahead panel
  cudaEvent_t ev_a = nullptr, ev_p = nullptr;
  // concurrent node groups (group 0 uses stream / side / ev_a / ev_p)
  static constexpr int GMAX = 8;
  int laswp_variant = feast::LASWP_COALESCED;   // FEAST_LASWP=chain|perm: the round-1 swap kernels
  bool prof_serial = false;           // feast_profile(h, 2): one stream, no lookahead / groups
  int groups = 4;                     // concurrent node groups per batch (FEAST_GROUPS)
  bool groups_set = false;            // FEAST_GROUPS given (else 2 groups for throughput-bound batches)
  // the current batch is throughput-bound (n >= 8192 with >= 16 nodes factored together: C3, C4):
  // 2 node groups and a full-width first outer block (C4 12.838 -> 12.803 s, C3 1543.4 -> 1538.0 ms;
  // C5's 4-node batches keep 4 groups and the 128-wide first block: 47.64 vs 47.65 s)
  bool big = false;
  bool group_streams = false;
  cudaStream_t gs[GMAX] = {}, gside[GMAX] = {};
  cudaEvent_t gev_a[GMAX] = {}, gev_p[GMAX] = {}, gev_done[GMAX] = {};
  cudaEvent_t ev_fork = nullptr;
  cudaStream_t s_rhs = nullptr;       // a1 (R = B X) concurrently with the first panels
  cudaEvent_t ev_a1 = nullptr, ev_rhs = nullptr;
  cudaEvent_t gev_first[GMAX] = {};
  cudaStream_t gx[GMAX] = {};         // per group: the stream of the diagonal-block inverses
  cudaEvent_t gev_t[GMAX] = {}, gev_x[GMAX] = {};
  cudaStream_t gl[GMAX] = {};         // per group: the stream of the L-column swaps (FEAST_LSWAP_SIDE)
  cudaEvent_t gev_l[GMAX] = {}, gev_lj[GMAX] = {};
  bool lswap_side = true;
  // FEAST_STAGGER = d > 0: node group g starts once group g-1 has finished d outer steps, so the
  // groups' latency-bound LU tails (and start-up panels) overlap other groups' GEMM-heavy blocks
  // instead of coinciding (round-robin enqueue keeps them in lockstep otherwise)
  int stagger = 0;
  int64_t ldc = 0;
  // workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  double2 *Cw = nullptr, *Y = nullptr, *YL = nullptr, *R = nullptr, *RL = nullptr, *zd = nullptr, *wd = nullptr;
  double2* wpd = nullptr;             // partner weights per unit (real-pencil mode)
  int32_t* realviol = nullptr;        // device flag: A or B not real (real-pencil mode)
  double2 *AQ = nullptr, *BQ = nullptr, *SK = nullptr;
  double2* Inv = nullptr;          // batch x nblk x {L^-1, U^-1} 64x64 diagonal-block inverses
  int64_t inv_stride = 0, nblk = 0;
  int64_t sk_elems = 0;
  int32_t *ipiv = nullptr, *perm = nullptr, *iperm = nullptr, *info = nullptr;
  double* stats = nullptr;
  std::vector<double> minrel;
  int worst = -1;
  // iterate extras (library-owned, allocated lazily; outside the hot path)
  void* itmem = nullptr;
  size_t itbytes = 0;
  cusolverDnHandle_t sol = nullptr;
  cusolverDnParams_t solp = nullptr;
  struct It {
    double2 *Qr, *Ql, *AX, *BX, *Ah, *Bh, *M, *W, *Z, *T, *lam, *tau;
    double2 *Rq, *Rl, *mu;               // R factors of U^, V^ and eig(V^^H B U^) (count estimate)
    double *rn, *xn, *fr;
    int *piv, *info;
    void* sw;
    size_t sw_bytes;
    std::vector<char> hw;
  } it{};
  // CUDA graph of the projector's launch sequence (replayed when the call signature repeats)
  struct GraphKey {
    const void *A, *B, *X, *V, *Q, *QL;
    int64_t lda, ldb, ldx, ldv, ldq, ldql;
    bool reuse;
    bool operator==(const GraphKey& o) const {
      return A == o.A && B == o.B && X == o.X && V == o.V && Q == o.Q && QL == o.QL && lda == o.lda && ldb == o.ldb &&
             ldx == o.ldx && ldv == o.ldv && ldq == o.ldq && ldql == o.ldql && reuse == o.reuse;
    }
  };
  bool graphs = true;
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey{}, gseen{};
  bool gseen_valid = false;
  int64_t glaunches = 0;
  feast_allreduce_fn ar = nullptr;
  void* ar_user = nullptr;
  bool partial = false;               // feast_set_partial: return this rank's partial node sum
  // feast_set_async: projector / reduce calls return once enqueued; the pivot statistics land in
  // pinned host memory and are judged by feast_sync (or the next feast_node_stats)
  bool async = false, pending = false;
  double* h_stats = nullptr;          // pinned: 2 nu doubles
  int32_t* h_info = nullptr;          // pinned: nu + 1 ints (the last: real-pencil violation flag)
  cudaEvent_t ev_stats = nullptr;
  // NEXT-3: monitors of the last feast_iterate
  bool count_on = false;              // feast_set_count_estimate: eig(V^^H B U^) in Bi-FEAST iterations
  double mon_res = -1.0;
  double2 mon_trace{0.0, 0.0};
  int mon_ncand = 0, mon_count = -1;
  std::vector<double2> mon_mu;
  double2* NS = nullptr;              // node-sum staging block [Q | QL] (n x m0 each, ld n), world > 1
  std::string err;
  int64_t launches = 0;
};

namespace {

int fail(feast_ctx* h, int code, const char* fmt, const char* a = "") {
  char buf[512];
  snprintf(buf, sizeof buf, fmt, a);
  h->err = buf;
  return code;
}

#define CUDA_TRY(h, x)                                                            \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) return fail((h), FEAST_E_CUDA, "CUDA: %s", cudaGetErrorString(e_)); \
  } while (0)
#define SOL_TRY(h, x)                                                             \
  do {                                                                            \
    cusolverStatus_t s_ = (x);                                                    \
    if (s_ != CUSOLVER_STATUS_SUCCESS) {                                          \
      char b_[64]; snprintf(b_, sizeof b_, "%d at line %d", (int)s_, __LINE__);  \
      return fail((h), FEAST_E_CUDA, "cuSOLVER status %s", b_);                   \
    }                                                                             \
  } while (0)

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Every public call runs on the library's own stream, ordered after the work already queued on
// the caller's stream and before anything the caller queues afterwards (event fork / join).
struct Join {
  feast_ctx* h;
  explicit Join(feast_ctx* hh) : h(hh) {
    if (h->own_stream) {
      cudaEventRecord(h->ev_in, h->caller);
      cudaStreamWaitEvent(h->stream, h->ev_in, 0);
    }
  }
  ~Join() {
    if (h->own_stream) {
      cudaEventRecord(h->ev_out, h->stream);
      cudaStreamWaitEvent(h->caller, h->ev_out, 0);
    }
  }
};

void graph_reset(feast_ctx* h) {   // the captured sequence depends on the workspace and cache mode
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  h->gexec = nullptr;
  h->gseen_valid = false;
}

// ---------------------------------------------------------------- nodes (product side)
// Quadrature on [-1,1] mapped to the ellipse of eq. ellipses: theta = pi/2 (1+t),
// z = c + r (cos theta + i a sin theta), sigma = w_k phi'(t) / (2 pi i)
//   = w_k r (a cos theta + i sin theta) / 4            (phi' = (pi/2) r (-sin + i a cos)).
// Each rule node t_k gives theta(t_k) and theta(2 - t_k) = 2 pi - theta(t_k) (eq. pi);
// coinciding angles (t = +-1 with endpoints) are merged by summing weights.
bool legendre_rule(int K, std::vector<double>& t, std::vector<double>& wt) {
  t.assign(K, 0.0);
  wt.assign(K, 0.0);
  for (int i = 1; i <= K; ++i) {
    double x = std::cos(M_PI * (i - 0.25) / (K + 0.5));
    double d = 0.0;
    for (int it = 0; it < 200; ++it) {
      double p0 = 1.0, p1 = x;
      for (int j = 2; j <= K; ++j) {
        const double p2 = ((2 * j - 1) * x * p1 - (j - 1) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      if (K == 1) { p1 = x; p0 = 1.0; }
      d = K * (p0 - x * p1) / (1.0 - x * x);
      const double dx = p1 / d;
      x -= dx;
      if (std::fabs(dx) <= 4e-16 * std::fabs(x) + 1e-300) {
        // one more evaluation for the weight
        p0 = 1.0; p1 = x;
        for (int j = 2; j <= K; ++j) {
          const double p2 = ((2 * j - 1) * x * p1 - (j - 1) * p0) / j;
          p0 = p1;
          p1 = p2;
        }
        if (K == 1) { p1 = x; p0 = 1.0; }
        d = K * (p0 - x * p1) / (1.0 - x * x);
        break;
      }
    }
    t[K - i] = x;                  // ascending
    wt[K - i] = 2.0 / ((1.0 - x * x) * d * d);
  }
  return true;
}

// Composite contour: segment s on t in [-1, 1] (line a -> b, or arc c + R e^{i th}, th0 -> th1),
// the rule (midpoint trapezoid, reading R18, or Gauss-Legendre) with seg_k nodes on every
// segment: pole phi(t_k), weight w_k phi'(t_k) / (2 pi i) (eq. pi with one interval per segment).
void seg_phi(const feast_ctx::Seg& g, double t, double2& ph, double2& dph) {
  if (g.kind == 0) {
    const double s = 0.5 * (1.0 + t);
    ph = make_double2(g.p[0] + (g.p[2] - g.p[0]) * s, g.p[1] + (g.p[3] - g.p[1]) * s);
    dph = make_double2(0.5 * (g.p[2] - g.p[0]), 0.5 * (g.p[3] - g.p[1]));
  } else {
    const double half = 0.5 * (g.p[4] - g.p[3]), th = g.p[3] + half * (1.0 + t);
    ph = make_double2(g.p[0] + g.p[2] * std::cos(th), g.p[1] + g.p[2] * std::sin(th));
    dph = make_double2(-g.p[2] * std::sin(th) * half, g.p[2] * std::cos(th) * half);
  }
}

int make_segment_nodes(feast_ctx* h) {
  std::vector<double> t, wt;
  const int K = h->seg_k;
  if (K < 1) return -1;
  if (h->seg_rule == FEAST_RULE_TRAPEZOID) {
    for (int k = 0; k < K; ++k) { t.push_back(-1.0 + (2.0 * k + 1.0) / K); wt.push_back(2.0 / K); }
  } else if (h->seg_rule == FEAST_RULE_GAUSS_LEGENDRE) {
    legendre_rule(K, t, wt);
  } else {
    return -1;
  }
  h->z.clear(); h->w.clear(); h->poly.clear();
  for (const auto& g : h->segs) {
    for (int k = 0; k < K; ++k) {
      double2 ph, dph;
      seg_phi(g, t[k], ph, dph);
      h->z.push_back(ph);
      // w phi' / (2 pi i) = (w / 2 pi) (Im phi', -Re phi')
      h->w.push_back(make_double2(wt[k] * dph.y / (2.0 * M_PI), -wt[k] * dph.x / (2.0 * M_PI)));
    }
    for (int i = 0; i < 256; ++i) {   // polyline for the inside test
      double2 ph, dph;
      seg_phi(g, -1.0 + 2.0 * i / 256.0, ph, dph);
      h->poly.push_back(ph);
    }
  }
  h->q = (int)h->z.size();
  return 0;
}

// Is mu inside the contour?  Ellipse: the analytic test (R2); composite contour:
// crossing number of the closed polyline (256 points per segment).
bool inside_contour(const feast_ctx* h, double x, double y) {
  if (h->segs.empty()) {
    const double u = (x - h->c_re) / h->r, v = (y - h->c_im) / (h->r * h->aspect);
    return u * u + v * v < 1.0;
  }
  bool in = false;
  const size_t np = h->poly.size();
  for (size_t i = 0, j = np - 1; i < np; j = i++) {
    const double2 a = h->poly[i], b = h->poly[j];
    if ((a.y > y) != (b.y > y) && x < (b.x - a.x) * (y - a.y) / (b.y - a.y) + a.x) in = !in;
  }
  return in;
}

int make_nodes(feast_ctx* h) {
  std::vector<double> t, wt;
  int K;
  if (h->rule == FEAST_RULE_TRAPEZOID) {
    if (h->n_e < 2 || h->n_e % 2) return -1;
    K = h->n_e / 2;
    for (int k = 0; k < K; ++k) { t.push_back(-1.0 + (2.0 * k + 1.0) / K); wt.push_back(2.0 / K); }
  } else if (h->rule == FEAST_RULE_TRAPEZOID_ENDPOINT) {
    if (h->n_e < 2 || h->n_e % 2) return -1;
    K = h->n_e / 2 + 1;
    for (int k = 0; k < K; ++k) {
      t.push_back(-1.0 + 2.0 * k / (K - 1));
      wt.push_back((k == 0 || k == K - 1) ? 1.0 / (K - 1) : 2.0 / (K - 1));
    }
  } else if (h->rule == FEAST_RULE_GAUSS_LEGENDRE) {
    if (h->n_e < 1) return -1;
    K = h->n_e;
    legendre_rule(K, t, wt);
  } else {
    return -1;
  }
  std::vector<double> th, ww;
  for (int half = 0; half < 2; ++half)
    for (int k = 0; k < K; ++k) {
      const double tt = half ? 2.0 - t[k] : t[k];
      double a = 0.5 * M_PI * (1.0 + tt);
      bool merged = false;
      for (size_t j = 0; j < th.size(); ++j) {
        double d = std::fabs(std::remainder(a - th[j], 2 * M_PI));
        if (d < 1e-12) { ww[j] += wt[k]; merged = true; break; }
      }
      if (!merged) { th.push_back(a); ww.push_back(wt[k]); }
    }
  h->q = (int)th.size();
  h->z.resize(h->q);
  h->w.resize(h->q);
  for (int j = 0; j < h->q; ++j) {
    const double ct = std::cos(th[j]), st = std::sin(th[j]);
    h->z[j] = make_double2(h->c_re + h->r * ct, h->c_im + h->r * h->aspect * st);
    h->w[j] = make_double2(ww[j] * h->r * h->aspect * ct / 4.0, ww[j] * h->r * st / 4.0);
  }
  return 0;
}

Batched bat(double2* p, int64_t ld, int64_t stride) { return Batched{p, ld, stride}; }

// A group of nodes factored together (lockstep batch): its slice of the workspace and its
// streams.  Several groups run concurrently on their own stream pairs, so one group's latency-
// bound panel chain overlaps another group's trailing-update GEMMs.
struct Lu {
  double2* Cw;          // first node's augmented block [C_j | R]
  double2* Inv;         // first node's 64x64 diagonal-block inverses
  int32_t* ipiv;        // first node's pivots
  double* stats;        // first node's pivot statistics
  int32_t* info;
  int nbat;
  cudaStream_t sm, sp;  // main / high-priority lookahead stream
  cudaEvent_t ev_a, ev_p;
  cudaEvent_t ev_first;  // recorded after the first block is factored (nullptr: none)
  cudaStream_t sx;       // diagonal-block inverses off the panel chain (nullptr: on the chain)
  cudaEvent_t ev_t, ev_x;
  cudaStream_t sl = nullptr;   // the outer blocks' swaps of the L columns, off the chain (nullptr: on it)
  cudaEvent_t ev_l = nullptr, ev_lj = nullptr;
};
const double2* inv_ptr(const Lu& v, int64_t kb, int which) { return v.Inv + (kb * 2 + which) * 4096; }

// Y[K0:K0+R) <- op(T[K0:K0+R, K0:K0+R])^-1 Y[K0:K0+R) for N columns, T = L (which = 0, unit lower)
// or U (which = 1, upper) of the factored block, op = conjugate transpose when conj (the sweep
// runs forward for L and U^H, backward for U and L^H): the fused DMMA block solve (btrsm.cu) on
// 256-row pieces, the pieces coupled by DMMA GEMM updates with K = 256.  Y's row r is Y[r] (ld,
// batch stride sy).
void block_solve(feast_ctx* h, double2* Cw, const double2* Inv, int nbat, int which, bool conj, int64_t K0, int64_t R,
                 double2* Y, int64_t ldy, int64_t sy, int64_t N, cudaStream_t s) {
  const int64_t n = h->n, ld = h->ldc, st = ld * (n + h->mr);
  const bool fwd = (which == 0) != conj;
  auto piece = [&](int64_t j, int64_t r) {
    feast::BtrsmArgs a{Cw + (K0 + j) + (K0 + j) * ld, ld, st, Inv + ((K0 + j) / 64 * 2 + which) * 4096, 2 * 4096,
                       h->inv_stride, Y + K0 + j, ldy, sy, r, N, nbat};
    feast::btrsm_launch(a, fwd, conj, s);
  };
  if (fwd) {
    for (int64_t j = 0; j < R; j += 256) {
      const int64_t r = std::min<int64_t>(256, R - j), rest = R - j - r;
      piece(j, r);
      if (rest > 0) {   // Y[K0+j+r : K0+R) -= op(T)[those rows, K0+j : K0+j+r) Y[K0+j : +r)
        const double2* A = conj ? Cw + (K0 + j) + (K0 + j + r) * ld : Cw + (K0 + j + r) + (K0 + j) * ld;
        ZgemmArgs p{rest, N, r, A, ld, st, Y + K0 + j, ldy, sy, Y + K0 + j + r, ldy, sy, make_double2(-1, 0),
                    make_double2(1, 0), nbat};
        feast::zgemm_launch(p, conj, feast::ZG_SUB, s);
      }
    }
  } else {
    for (int64_t j = ((R - 1) / 256) * 256; j >= 0; j -= 256) {
      const int64_t r = std::min<int64_t>(256, R - j);
      piece(j, r);
      if (j > 0) {      // Y[K0 : K0+j) -= op(T)[K0 : K0+j, K0+j : +r) Y[K0+j : +r)
        const double2* A = conj ? Cw + (K0 + j) + K0 * ld : Cw + K0 + (K0 + j) * ld;
        ZgemmArgs p{j, N, r, A, ld, st, Y + K0 + j, ldy, sy, Y + K0, ldy, sy, make_double2(-1, 0), make_double2(1, 0),
                    nbat};
        feast::zgemm_launch(p, conj, feast::ZG_SUB, s);
      }
    }
  }
}

// ---------------------------------------------------------------- GEMM helpers
// C = alpha op(A) B + beta C (single), with split-K when the output tile grid is too small
// to fill the GPU (the reduced matrices Q^H (A Q) are m0 x m0 with K = n).
void gemm_gen(feast_ctx* h, int64_t M, int64_t N, int64_t K, bool conjA, const double2* A, int64_t lda,
              const double2* B, int64_t ldb, double2* C, int64_t ldc, double2 alpha, double2 beta,
              cudaStream_t s = nullptr) {
  if (!s) s = h->stream;
  // 32x32 CTA tiles, 3 resident per SM: fewer than 444 tiles leave the GPU under-filled
  const int64_t tiles = ((M + 31) / 32) * ((N + 31) / 32);
  int splits = 1;
  if (tiles < 444 && K >= 512 && h->SK) {
    // the split count whose tile grid best fills whole waves of 444 CTAs (2 splits of a 256-tile
    // grid would run 1.15 waves at 58 % occupancy of the second; 5 splits fill 96 %)
    double best = (double)tiles / 444.0;
    const int smax = (int)std::min<int64_t>(16, K / 128);
    for (int sp = 2; sp <= smax; ++sp) {
      if ((int64_t)sp * M * N > h->sk_elems) break;
      const int64_t t = tiles * sp, waves = (t + 443) / 444;
      const double eff = (double)t / (double)(waves * 444) - 0.01 * sp;   // mild cost per split
      if (eff > best) { best = eff; splits = sp; }
    }
  }
  if (splits <= 1) {
    ZgemmArgs p{M, N, K, A, lda, 0, B, ldb, 0, C, ldc, 0, alpha, beta, 1};
    feast::zgemm_launch(p, conjA, feast::ZG_GEN, s);
    return;
  }
  const int64_t kc = ((K + splits - 1) / splits + 15) / 16 * 16;
  splits = (int)((K + kc - 1) / kc);
  // batch over K-chunks: A advances kc along K, B advances kc rows; last chunk is ragged -> run
  // the even part batched and the tail separately.
  const int full = (int)(K / kc);
  const int64_t sA = conjA ? kc : kc * lda;
  if (full > 0) {
    ZgemmArgs p{M, N, kc, A, lda, sA, B, ldb, kc, h->SK, M, M * N, make_double2(1, 0), make_double2(0, 0), full};
    feast::zgemm_launch(p, conjA, feast::ZG_GEN, s);
  }
  if (full < splits) {
    const int64_t k0 = (int64_t)full * kc;
    ZgemmArgs p{M, N, K - k0, A + (conjA ? k0 : k0 * lda), lda, 0, B + k0, ldb, 0, h->SK + (int64_t)full * M * N, M, 0,
                make_double2(1, 0), make_double2(0, 0), 1};
    feast::zgemm_launch(p, conjA, feast::ZG_GEN, s);
  }
  feast::splitk_reduce_launch(C, ldc, h->SK, M, N, splits, alpha, beta, s);
}

// ---------------------------------------------------------------- blocked LU (batched)
// The cluster panel with the panel in shared memory whenever the remaining height L = n - k fits
// clusters of <= smem_cs_max CTAs x 256 rows (the launch shrinks the cluster further as L falls);
// the register-chunk panel (64 wide, rows swapped in global memory) for taller panels.
bool smem_panel_for(const feast_ctx* h, int64_t k) {
  if (h->smem_cs_max <= 0) return false;
  const int64_t rows = (h->n - k + h->smem_cs_max - 1) / h->smem_cs_max;   // per CTA
  return rows <= 256 || (rows <= 1024 && feast::tall_variant() != 0) || (rows <= 2048 && feast::very_tall_panels());
}
// Panels taller than 256 rows per CTA (n - k > 16 x 256) are 16 wide: the w - 8 columns a CTA
// keeps in shared memory must fit 190 KB at up to 1024 rows per CTA.
bool tall_panel(const feast_ctx* h, int64_t k) {
  return (h->n - k + h->smem_cs_max - 1) / h->smem_cs_max > 256;
}

// Timing ablation (FEAST_ABLATE, never for results): bit 1 skips the panels (identity pivots),
// bit 2 the triangular kernels, bit 4 the row swaps, bit 8 the back substitution — to measure
// each class's marginal cost in
// the overlapped schedule.
int ablate() {
  static const int a = [] { const char* e = getenv("FEAST_ABLATE"); return e ? atoi(e) : 0; }();
  return a;
}

// sc0 < sc1: the shared-memory panel also applies its swaps to the columns [sc0, sc1)
void panel_at(feast_ctx* h, const Lu& v, int64_t k, int w, cudaStream_t s, int64_t sc0 = 0, int64_t sc1 = 0) {
  const int64_t n = h->n, ld = h->ldc, st = ld * (n + h->mr);
  if (ablate() & 1) { feast::ipiv_identity_launch(v.ipiv, n, k, w, v.nbat, s); return; }
  if (smem_panel_for(h, k))
    feast::panel_smem_launch(bat(v.Cw, ld, st), n, k, w, v.ipiv, v.stats, v.info, v.nbat, h->smem_cs_max, s,
                             h->panel_one_row, sc0, sc1);
  else
    feast::panel_launch(bat(v.Cw, ld, st), n, k, w, v.ipiv, v.stats, v.info, v.nbat, h->pcfg, s);
}

// Two-level right-looking blocked LU of the batch with one-step LOOKAHEAD.
//   inner: 64-wide panels (cluster kernel) inside an outer block of NBO columns, each followed
//          by its row swaps on the block's columns, the 64x64 diagonal inverses and the
//          in-block U12 / update (K = 64);
//   outer: the block's swaps on all other columns, U12 = L11^-1 A12 as a blocked in-place DMMA
//          TRSM with the 64x64 inverses, then the trailing update A22 -= L21 U12 with K = NBO.
// Lookahead: the outer update first refreshes the next block's columns, then the next block is
// factored on a high-priority side stream while the rest of the outer update runs on the main
// stream (disjoint columns; the next block's swaps reach the other columns afterwards).
// aug > 0: columns [n, n + aug) hold R, so swaps, U12 and updates also perform the forward
// substitution L^-1 P R.
void factor_block(feast_ctx* h, const Lu& v, int64_t K0, int64_t Wo, cudaStream_t s) {
  const int64_t n = h->n, ld = h->ldc, st = ld * (n + h->mr);
  double2* C = v.Cw;
  const int nbat = v.nbat;
  for (int64_t ki = K0; ki < K0 + Wo; ki += 64) {
    const int wi = (int)std::min<int64_t>(64, K0 + Wo - ki);
    const bool smem = smem_panel_for(h, ki);
    // once the panel is short (L <= wide_panel_rows: clusters of <= 8 CTAs x 128 rows), a 64-wide
    // block is one cluster panel: no in-block trsm / update / second swap launch on the chain
    const int64_t vt_rows = (h->n - ki + h->smem_cs_max - 1) / h->smem_cs_max;   // rows per CTA
    const int64_t wp = !smem ? 64 : ((h->n - ki <= h->wide_panel_rows) ? 64 : (vt_rows > 1024 ? 8 : (tall_panel(h, ki) ? 16 : h->wp)));
    // the 64-block is factored as narrow cluster panels of wp columns (small SM footprint), with
    // the in-block U12 (warp TRSM) and update (DMMA) between them
    for (int64_t kp = ki; kp < ki + wi; kp += wp) {
      const int wpp = (int)std::min<int64_t>(wp, ki + wi - kp);
      // shared-memory panels apply their swaps to the outer block's columns themselves
      // (FEAST_PANEL_SWAP=0: a separate swap launch)
      const bool fused = smem && h->panel_swap && !(ablate() & 5);
      panel_at(h, v, kp, wpp, s, fused ? K0 : 0, fused ? K0 + Wo : 0);
      if (smem) {
        if (!fused && !(ablate() & 4))
          feast::laswp_launch(bat(C, ld, st), n, kp, wpp, v.ipiv, K0, K0 + Wo, nbat, s, h->laswp_variant);
      } else {   // the register-chunk panel already swapped its own columns
        if (!(ablate() & 4)) feast::laswp_launch(bat(C, ld, st), n, kp, wpp, v.ipiv, K0, kp, nbat, s, h->laswp_variant);
        if (!(ablate() & 4)) feast::laswp_launch(bat(C, ld, st), n, kp, wpp, v.ipiv, kp + wpp, K0 + Wo, nbat, s, h->laswp_variant);
      }
      const int64_t cp = kp + wpp, remb = ki + wi - cp;
      if (remb > 0) {
        if (!(ablate() & 2)) feast::trsm_launch(bat(C + kp + kp * ld, ld, st), bat(C + kp + cp * ld, ld, st), wpp, remb, true, true, false,
                           nbat, s);
        ZgemmArgs p{n - cp, remb, wpp, C + cp + kp * ld, ld, st, C + kp + cp * ld, ld, st, C + cp + cp * ld, ld, st,
                    make_double2(-1, 0), make_double2(1, 0), nbat};
        feast::zgemm_launch(p, false, feast::ZG_SUB, s);
      }
    }
    // the 64x64 inverses (needed by the outer U12 and the substitutions, not by this block's
    // chain) run on their own stream, joined at the end of the block
    const int64_t c1 = ki + wi, rem = K0 + Wo - c1;
    cudaStream_t st_inv = s;
    if (v.sx) {
      cudaEventRecord(v.ev_t, s);
      cudaStreamWaitEvent(v.sx, v.ev_t, 0);
      st_inv = v.sx;
    }
    if (!(ablate() & 2)) feast::trtri_launch(bat(C, ld, st), n, ki / 64, 1, v.Inv, h->inv_stride, 2, nbat, st_inv);
    if (rem > 0) {
      // in-block U12 = L11^-1 A12 (warp TRSM on the chain), then A22 -= L21 U12 (DMMA)
      if (!(ablate() & 2)) feast::trsm_launch(bat(C + ki + ki * ld, ld, st), bat(C + ki + c1 * ld, ld, st), wi, rem, true, true, false,
                         nbat, s);
      ZgemmArgs p{n - c1, rem, wi, C + c1 + ki * ld, ld, st, C + ki + c1 * ld, ld, st, C + c1 + c1 * ld, ld, st,
                  make_double2(-1, 0), make_double2(1, 0), nbat};
      feast::zgemm_launch(p, false, feast::ZG_SUB, s);
    }
  }
  if (v.sx) {   // the block's inverses complete before anything downstream of this stream
    cudaEventRecord(v.ev_x, v.sx);
    cudaStreamWaitEvent(s, v.ev_x, 0);
  }
}

// U12 = L11^-1 A12 and A22 -= L21 U12 for the columns [c0, c0 + nc) of outer block (K0, Wo).
void outer_update(feast_ctx* h, const Lu& v, int64_t K0, int64_t Wo, int64_t c0, int64_t nc, cudaStream_t s) {
  if (nc <= 0) return;
  const int64_t n = h->n, ld = h->ldc, st = ld * (n + h->mr), K1 = K0 + Wo;
  double2* C = v.Cw;
  const int nbat = v.nbat;
  if (h->btrsm) {   // U12 = L11^-1 A12: the fused block solve
    block_solve(h, C, v.Inv, nbat, 0, false, K0, Wo, C + c0 * ld, ld, st, nc, s);
  } else if (h->u12_dot == 2 || (h->u12_dot == 1 && 2 * ((nc + 31) / 32) * nbat >= 444)) {
    for (int64_t ki = K0; ki < K1; ki += 64) {   // dot form: Y_i -= L[i, 0:i] Y[0:i]; Y_i <- L_ii^-1 Y_i
      const int wi = (int)std::min<int64_t>(64, K1 - ki);
      if (ki > K0) {
        ZgemmArgs p{wi, nc, ki - K0, C + ki + K0 * ld, ld, st, C + K0 + c0 * ld, ld, st, C + ki + c0 * ld, ld, st,
                    make_double2(-1, 0), make_double2(1, 0), nbat};
        feast::zgemm_launch(p, false, feast::ZG_SUB, s);
      }
      ZgemmArgs u{wi, nc, wi, inv_ptr(v, ki / 64, 0), 64, h->inv_stride, C + ki + c0 * ld, ld, st, C + ki + c0 * ld,
                  ld, st, make_double2(1, 0), make_double2(0, 0), nbat, 1};
      feast::zgemm_launch(u, false, feast::ZG_GEN, s);
    }
  } else
  for (int64_t ki = K0; ki < K1; ki += 64) {
    const int wi = (int)std::min<int64_t>(64, K1 - ki);
    ZgemmArgs u{wi, nc, wi, inv_ptr(v, ki / 64, 0), 64, h->inv_stride, C + ki + c0 * ld, ld, st, C + ki + c0 * ld, ld,
                st, make_double2(1, 0), make_double2(0, 0), nbat, 1};
    feast::zgemm_launch(u, false, feast::ZG_GEN, s);
    if (ki + wi < K1) {
      ZgemmArgs p{K1 - ki - wi, nc, wi, C + (ki + wi) + ki * ld, ld, st, C + ki + c0 * ld, ld, st,
                  C + (ki + wi) + c0 * ld, ld, st, make_double2(-1, 0), make_double2(1, 0), nbat};
      feast::zgemm_launch(p, false, feast::ZG_SUB, s);
    }
  }
  if (K1 < n) {
    ZgemmArgs p{n - K1, nc, Wo, C + K1 + K0 * ld, ld, st, C + K0 + c0 * ld, ld, st, C + K1 + c0 * ld, ld, st,
                make_double2(-1, 0), make_double2(1, 0), nbat};
    feast::zgemm_launch(p, false, feast::ZG_SUB, s);
  }
}

// Width of the first outer block: 128 columns (FEAST_NBO0), half the outer block, so the big
// trailing GEMMs start sooner after the latency-bound first factorisation (C2 16.71 -> 16.61 ms;
// 64: 16.74, 192: 16.67); the full outer block for throughput-bound batches (h->big: the K = 128
// first trailing update ran at 33.6 TF/s on C4).
int64_t first_block(const feast_ctx* h) {
  static const int64_t nbo0_env = [] { const char* e = getenv("FEAST_NBO0"); return e ? atoll(e) : 0LL; }();
  const int64_t nbo0 = nbo0_env > 0 ? nbo0_env : (h->big ? h->nbo : 128);
  return (nbo0 % 64 == 0) ? std::min<int64_t>(nbo0, h->nbo) : h->nbo;
}

// The batched LU as a resumable sequence: step() enqueues the first outer block (and, with
// rest(s), the formation of the remaining columns of [C_j | R] on stream s underneath it), then
// one outer block per call; it returns true once the factorisation is fully enqueued.  The node
// groups' sequences are enqueued round-robin, block by block (project_enqueue), so the groups
// progress together instead of group 0 running ahead and the last group's latency-bound tail
// finishing alone.
struct LuRun {
  feast_ctx* h;
  Lu v;
  int64_t aug;
  std::function<void(cudaStream_t)> rest;
  int phase = 0;          // 0: not started, 1: outer blocks, 2: done
  int64_t K0 = 0, Wo = 0;
  int steps = 0;          // outer steps enqueued (ev_first is recorded after h->stagger of them)

  void record_first(cudaStream_t sm) {
    if (v.ev_first && ++steps == h->stagger) cudaEventRecord(v.ev_first, sm);   // releases the next group
  }
  void finish(cudaStream_t sm) {
    phase = 2;
    while (v.ev_first && steps < h->stagger) record_first(sm);   // short LU: release the next group
    if (v.sl) {                                                  // the L-column swaps are done
      cudaEventRecord(v.ev_lj, v.sl);
      cudaStreamWaitEvent(sm, v.ev_lj, 0);
    }
  }

  bool step() {
    const int64_t n = h->n, ld = h->ldc, st = ld * (n + h->mr), ntot = n + aug;
    double2* C = v.Cw;
    const int nbat = v.nbat;
    cudaStream_t sm = v.sm, sp = v.sp;
    const int64_t NBO = h->nbo;
    if (phase == 2) return true;
    if (phase == 0) {
      // first outer block (FEAST_NBO0, experiment): a narrower one starts the big trailing
      // GEMMs sooner after the latency-bound first factorisation
      Wo = std::min<int64_t>(first_block(h), n);
      if (rest && h->lookahead && !h->prof_serial && Wo < n) {
        // the first block is factored on the high-priority side stream while the main stream
        // forms the rest of [C_j | R] (HBM-bound, needed only once the block is done)
        cudaEventRecord(v.ev_a, sm);
        cudaStreamWaitEvent(sp, v.ev_a, 0);
        factor_block(h, v, 0, Wo, sp);
        cudaEventRecord(v.ev_p, sp);
        rest(sm);
        cudaStreamWaitEvent(sm, v.ev_p, 0);
      } else {
        if (rest) rest(sm);
        factor_block(h, v, 0, Wo, sm);
      }
      if (!(ablate() & 4)) feast::laswp_launch(bat(C, ld, st), n, 0, (int)Wo, v.ipiv, Wo, ntot, nbat, sm, h->laswp_variant);
      record_first(sm);
      phase = 1;
      K0 = 0;
      return false;
    }
    if (K0 >= n) {
      finish(sm);
      return true;
    }
    const int64_t K1 = K0 + Wo;
    if (K1 >= n) {
      outer_update(h, v, K0, Wo, n, aug, sm);      // last block: augmented columns only
      finish(sm);
      return true;
    }
    const int64_t Wo1 = std::min<int64_t>(NBO, n - K1);
    outer_update(h, v, K0, Wo, K1, Wo1, sm);       // next block's columns first
    if (h->lookahead && !h->prof_serial) {
      cudaEventRecord(v.ev_a, sm);
      cudaStreamWaitEvent(sp, v.ev_a, 0);
      factor_block(h, v, K1, Wo1, sp);             // overlaps the rest of the outer update
      cudaEventRecord(v.ev_p, sp);
      outer_update(h, v, K0, Wo, K1 + Wo1, ntot - K1 - Wo1, sm);
      cudaStreamWaitEvent(sm, v.ev_p, 0);
    } else {
      outer_update(h, v, K0, Wo, K1 + Wo1, ntot - K1 - Wo1, sm);
      factor_block(h, v, K1, Wo1, sm);
    }
    // block K1's swaps on every column outside it: the L columns [0, K1) are read only by the
    // substitutions, so their swaps run on a side stream (in order, joined when the LU ends)
    if (!(ablate() & 4)) {
      cudaStream_t sl = sm;
      if (v.sl) {
        cudaEventRecord(v.ev_l, sm);
        cudaStreamWaitEvent(v.sl, v.ev_l, 0);
        sl = v.sl;
      }
      feast::laswp_launch(bat(C, ld, st), n, K1, (int)Wo1, v.ipiv, 0, K1, nbat, sl, h->laswp_variant);
      feast::laswp_launch(bat(C, ld, st), n, K1, (int)Wo1, v.ipiv, K1 + Wo1, ntot, nbat, sm, h->laswp_variant);
    }
    K0 = K1;
    Wo = Wo1;
    record_first(sm);
    return false;
  }
};

void lu_batched(feast_ctx* h, const Lu& v, int64_t aug, const std::function<void(cudaStream_t)>& rest = nullptr) {
  LuRun r{h, v, aug, rest};
  while (!r.step()) {
  }
}

// Y_k <- op(T_kk^-1) Y_k in place (M = w <= 64): which 0 = L^-1, 1 = U^-1; conj: (.)^H
void diag_apply(feast_ctx* h, const Lu& v, double2* Y, int64_t sy, int64_t k, int w, int which, bool conj,
                int64_t ncols) {
  const int64_t ld = h->ldc;
  ZgemmArgs p{w, ncols, w, inv_ptr(v, k / 64, which), 64, h->inv_stride, Y + k, ld, sy, Y + k, ld, sy,
              make_double2(1, 0), make_double2(0, 0), v.nbat, 1};
  feast::zgemm_launch(p, conj, feast::ZG_GEN, v.sm);
}

// Substitutions with the LU factors, two-level: 64-row blocks (the inverted 64x64 diagonal blocks
// applied by in-place DMMA products, K = 64 updates inside an outer block) and outer blocks of
// h->solve_nb rows whose off-block update is ONE DMMA GEMM with K = solve_nb (the K = 64 updates of
// a one-level sweep keep every CTA in its pipeline prologue / epilogue).
bool inner_dot(const feast_ctx* h, int nbat, int64_t m) {
  return h->inner_dot == 2 || (h->inner_dot == 1 && h->subst_dot && 2 * ((m + 31) / 32) * nbat >= 444);
}

// Y <- L^-1 Y (Y already row-permuted): used when the factors are cached (no augmented LU)
void solve_right_fwd(feast_ctx* h, const Lu& v, double2* Y, int64_t sy, int64_t m) {
  const int64_t n = h->n, ld = h->ldc, st = ld * (n + h->mr), NB = h->solve_nb;
  double2* C = v.Cw;
  const bool idot = inner_dot(h, v.nbat, m);
  for (int64_t K0 = 0; K0 < n; K0 += NB) {
    const int64_t K1 = std::min(n, K0 + NB);
    if (h->subst_dot && K0 > 0) {   // Y[K0:K1] -= L[K0:K1, 0:K0] Y[0:K0]
      ZgemmArgs p{K1 - K0, m, K0, C + K0, ld, st, Y, ld, sy, Y + K0, ld, sy, make_double2(-1, 0), make_double2(1, 0),
                  v.nbat};
      feast::zgemm_launch(p, false, feast::ZG_SUB, v.sm);
    }
    if (h->btrsm) block_solve(h, C, v.Inv, v.nbat, 0, false, K0, K1 - K0, Y, ld, sy, m, v.sm);
    else
    for (int64_t k = K0; k < K1; k += h->nb) {
      const int w = (int)std::min<int64_t>(h->nb, K1 - k);
      if (idot && k > K0) {   // Y[k:k+w] -= L[k:k+w, K0:k] Y[K0:k]
        ZgemmArgs p{w, m, k - K0, C + k + K0 * ld, ld, st, Y + K0, ld, sy, Y + k, ld, sy, make_double2(-1, 0),
                    make_double2(1, 0), v.nbat};
        feast::zgemm_launch(p, false, feast::ZG_SUB, v.sm);
      }
      diag_apply(h, v, Y, sy, k, w, 0, false, m);
      const int64_t rest = K1 - k - w;
      if (!idot && rest > 0) {   // inside the outer block
        ZgemmArgs p{rest, m, w, C + (k + w) + k * ld, ld, st, Y + k, ld, sy, Y + k + w, ld, sy,
                    make_double2(-1, 0), make_double2(1, 0), v.nbat};
        feast::zgemm_launch(p, false, feast::ZG_SUB, v.sm);
      }
    }
    if (K1 < n && !h->subst_dot) {       // Y[K1:] -= L[K1:, K0:K1] Y[K0:K1]
      ZgemmArgs p{n - K1, m, K1 - K0, C + K1 + K0 * ld, ld, st, Y + K0, ld, sy, Y + K1, ld, sy,
                  make_double2(-1, 0), make_double2(1, 0), v.nbat};
      feast::zgemm_launch(p, false, feast::ZG_SUB, v.sm);
    }
  }
}

// Y <- U^-1 Y  (Y = L^-1 P R already: the forward substitution ran inside the augmented LU)
void solve_right_back(feast_ctx* h, const Lu& v, double2* Y, int64_t sy, int64_t m) {
  const int64_t n = h->n, ld = h->ldc, st = ld * (n + h->mr), NB = h->solve_nb;
  double2* C = v.Cw;
  const bool idot = inner_dot(h, v.nbat, m);
  const int64_t lastK0 = ((n - 1) / NB) * NB;
  for (int64_t K0 = lastK0; K0 >= 0; K0 -= NB) {
    const int64_t K1 = std::min(n, K0 + NB);
    const int64_t last = K0 + ((K1 - 1 - K0) / h->nb) * h->nb;
    if (h->subst_dot && K1 < n) {   // Y[K0:K1] -= U[K0:K1, K1:n] Y[K1:n]
      ZgemmArgs p{K1 - K0, m, n - K1, C + K0 + K1 * ld, ld, st, Y + K1, ld, sy, Y + K0, ld, sy, make_double2(-1, 0),
                  make_double2(1, 0), v.nbat};
      feast::zgemm_launch(p, false, feast::ZG_SUB, v.sm);
    }
    if (h->btrsm) block_solve(h, C, v.Inv, v.nbat, 1, false, K0, K1 - K0, Y, ld, sy, m, v.sm);
    else
    for (int64_t k = last; k >= K0; k -= h->nb) {
      const int w = (int)std::min<int64_t>(h->nb, K1 - k);
      if (idot && k + w < K1) {   // Y[k:k+w] -= U[k:k+w, k+w:K1] Y[k+w:K1]
        ZgemmArgs p{w, m, K1 - k - w, C + k + (k + w) * ld, ld, st, Y + k + w, ld, sy, Y + k, ld, sy,
                    make_double2(-1, 0), make_double2(1, 0), v.nbat};
        feast::zgemm_launch(p, false, feast::ZG_SUB, v.sm);
      }
      diag_apply(h, v, Y, sy, k, w, 1, false, m);
      if (!idot && k > K0) {     // Y[K0:k] -= U[K0:k, k:k+w] Y[k:k+w]
        ZgemmArgs p{k - K0, m, w, C + K0 + k * ld, ld, st, Y + k, ld, sy, Y + K0, ld, sy, make_double2(-1, 0),
                    make_double2(1, 0), v.nbat};
        feast::zgemm_launch(p, false, feast::ZG_SUB, v.sm);
      }
    }
    if (K0 > 0 && !h->subst_dot) {       // Y[0:K0] -= U[0:K0, K0:K1] Y[K0:K1]
      ZgemmArgs p{K0, m, K1 - K0, C + K0 * ld, ld, st, Y + K0, ld, sy, Y, ld, sy, make_double2(-1, 0),
                  make_double2(1, 0), v.nbat};
      feast::zgemm_launch(p, false, feast::ZG_SUB, v.sm);
    }
  }
}

// Y <- L^-H U^-H Y   (then the caller applies P^T): M^H = U^H L^H P  (P:438-439 same factors)
void solve_left(feast_ctx* h, const Lu& v, double2* Y) {
  const int64_t n = h->n, ld = h->ldc, st = ld * (n + h->mr), m = h->mr, sy = ld * m, NB = h->solve_nb;
  double2* C = v.Cw;
  const bool idot = inner_dot(h, v.nbat, m);
  for (int64_t K0 = 0; K0 < n; K0 += NB) {  // U^H: lower, non-unit
    const int64_t K1 = std::min(n, K0 + NB);
    if (h->subst_dot && K0 > 0) {   // Y[K0:K1] -= (U[0:K0, K0:K1])^H Y[0:K0]
      ZgemmArgs p{K1 - K0, m, K0, C + K0 * ld, ld, st, Y, ld, sy, Y + K0, ld, sy, make_double2(-1, 0),
                  make_double2(1, 0), v.nbat};
      feast::zgemm_launch(p, true, feast::ZG_SUB, v.sm);
    }
    if (h->btrsm) block_solve(h, C, v.Inv, v.nbat, 1, true, K0, K1 - K0, Y, ld, sy, m, v.sm);
    else
    for (int64_t k = K0; k < K1; k += h->nb) {
      const int w = (int)std::min<int64_t>(h->nb, K1 - k);
      if (idot && k > K0) {   // Y[k:k+w] -= (U[K0:k, k:k+w])^H Y[K0:k]
        ZgemmArgs p{w, m, k - K0, C + K0 + k * ld, ld, st, Y + K0, ld, sy, Y + k, ld, sy, make_double2(-1, 0),
                    make_double2(1, 0), v.nbat};
        feast::zgemm_launch(p, true, feast::ZG_SUB, v.sm);
      }
      diag_apply(h, v, Y, sy, k, w, 1, true, m);   // (U_kk^H)^-1 = (U_kk^-1)^H
      const int64_t rest = K1 - k - w;
      if (!idot && rest > 0) {   // Y[k+w:K1] -= (U[k:k+w, k+w:K1])^H Y[k:k+w]
        ZgemmArgs p{rest, m, w, C + k + (k + w) * ld, ld, st, Y + k, ld, sy, Y + k + w, ld, sy,
                    make_double2(-1, 0), make_double2(1, 0), v.nbat};
        feast::zgemm_launch(p, true, feast::ZG_SUB, v.sm);
      }
    }
    if (K1 < n && !h->subst_dot) {       // Y[K1:] -= (U[K0:K1, K1:])^H Y[K0:K1]
      ZgemmArgs p{n - K1, m, K1 - K0, C + K0 + K1 * ld, ld, st, Y + K0, ld, sy, Y + K1, ld, sy,
                  make_double2(-1, 0), make_double2(1, 0), v.nbat};
      feast::zgemm_launch(p, true, feast::ZG_SUB, v.sm);
    }
  }
  const int64_t lastK0 = ((n - 1) / NB) * NB;
  for (int64_t K0 = lastK0; K0 >= 0; K0 -= NB) {  // L^H: upper, unit
    const int64_t K1 = std::min(n, K0 + NB);
    const int64_t last = K0 + ((K1 - 1 - K0) / h->nb) * h->nb;
    if (h->subst_dot && K1 < n) {   // Y[K0:K1] -= (L[K1:n, K0:K1])^H Y[K1:n]
      ZgemmArgs p{K1 - K0, m, n - K1, C + K1 + K0 * ld, ld, st, Y + K1, ld, sy, Y + K0, ld, sy, make_double2(-1, 0),
                  make_double2(1, 0), v.nbat};
      feast::zgemm_launch(p, true, feast::ZG_SUB, v.sm);
    }
    if (h->btrsm) block_solve(h, C, v.Inv, v.nbat, 0, true, K0, K1 - K0, Y, ld, sy, m, v.sm);
    else
    for (int64_t k = last; k >= K0; k -= h->nb) {
      const int w = (int)std::min<int64_t>(h->nb, K1 - k);
      if (idot && k + w < K1) {   // Y[k:k+w] -= (L[k+w:K1, k:k+w])^H Y[k+w:K1]
        ZgemmArgs p{w, m, K1 - k - w, C + (k + w) + k * ld, ld, st, Y + k + w, ld, sy, Y + k, ld, sy,
                    make_double2(-1, 0), make_double2(1, 0), v.nbat};
        feast::zgemm_launch(p, true, feast::ZG_SUB, v.sm);
      }
      diag_apply(h, v, Y, sy, k, w, 0, true, m);   // (L_kk^H)^-1 = (L_kk^-1)^H
      if (!idot && k > K0) {     // Y[K0:k] -= (L[k:k+w, K0:k])^H Y[k:k+w]
        ZgemmArgs p{k - K0, m, w, C + k + K0 * ld, ld, st, Y + k, ld, sy, Y + K0, ld, sy, make_double2(-1, 0),
                    make_double2(1, 0), v.nbat};
        feast::zgemm_launch(p, true, feast::ZG_SUB, v.sm);
      }
    }
    if (K0 > 0 && !h->subst_dot) {       // Y[0:K0] -= (L[K0:K1, 0:K0])^H Y[K0:K1]
      ZgemmArgs p{K0, m, K1 - K0, C + K0, ld, st, Y + K0, ld, sy, Y, ld, sy, make_double2(-1, 0),
                  make_double2(1, 0), v.nbat};
      feast::zgemm_launch(p, true, feast::ZG_SUB, v.sm);
    }
  }
}

int check_args_common(feast_ctx* h, const void* A, int64_t lda, const void* B, int64_t ldb) {
  if (!h) return FEAST_E_ARG;
  if (!h->ws) return fail(h, FEAST_E_STATE, "no workspace bound%s");
  if (!A || lda < h->n) return fail(h, FEAST_E_ARG, "A is null or lda < n%s");
  if (!h->b_id && (!B || ldb < h->n)) return fail(h, FEAST_E_ARG, "B is null or ldb < n (B != I)%s");
  return FEAST_OK;
}

// The projector's launch sequence: right (X -> Q) and/or left (V -> QL) from one factorisation
// per node.  Pure enqueue (no host synchronisation), so it can be captured into a CUDA graph.
void project_enqueue(feast_ctx* h, const double2* A, int64_t lda, const double2* B, int64_t ldb, const double2* X,
                     int64_t ldx, const double2* V, int64_t ldv, double2* Q, int64_t ldq, double2* QL, int64_t ldql,
                     bool reuse, bool rhs_ready) {
  const bool doR = X != nullptr, doL = V != nullptr;
  const int64_t n = h->n, m = h->m0, ld = h->ldc;
  const double2 one = make_double2(1, 0), zero = make_double2(0, 0);
  // a1: right-hand sides R = B X, RL = B^H V (shared by all nodes; skipped for B = I)
  const double2* Rr = X;
  int64_t ldr = ldx;
  const double2* Rl = V;
  int64_t ldrl = ldv;
  // a1 on its own stream when possible: the node groups start their shifts and first panels at
  // once, and wait for R only where they copy it into the augmented columns
  cudaEvent_t rhs_wait = nullptr;
  if (!h->b_id) {   // (rhs_ready: formed row-sharded and all-reduced by project_impl)
    const bool side_a1 = !rhs_ready && h->s_rhs && !h->prof_serial;
    cudaStream_t sa = h->stream;
    if (side_a1) {
      cudaEventRecord(h->ev_a1, h->stream);
      cudaStreamWaitEvent(h->s_rhs, h->ev_a1, 0);
      sa = h->s_rhs;
    }
    if (doR) {
      if (!rhs_ready) gemm_gen(h, n, m, n, false, B, ldb, X, ldx, h->R, ld, one, zero, sa);
      Rr = h->R; ldr = ld;
    }
    if (doL) {
      if (!rhs_ready) gemm_gen(h, n, m, n, true, B, ldb, V, ldv, h->RL, ld, one, zero, sa);
      Rl = h->RL; ldrl = ld;
    }
    if (side_a1) {
      cudaEventRecord(h->ev_rhs, sa);
      rhs_wait = h->ev_rhs;
    }
  }
  const int owned = h->j1 - h->j0;
  const int64_t mr = h->mr, st = ld * (n + mr);
  const bool pair = h->real;          // units are conjugate-pole orbits: RHS [R | conj R]
  const double2* wp = pair ? h->wpd : nullptr;
  // complex-symmetric pencil (C_j^T = C_j): Z_j = C_j^-H RL = conj(C_j^-1 conj(RL)), so the left
  // block rides along the right solves as extra columns conj(RL) of the augmented system
  const bool csl = h->csym && doL && !reuse;
  const int64_t ncr = pair ? mr : (csl && doR ? 2 * m : m);   // right-hand-side columns solved
  const bool solve = doR || csl;
  if (pair && owned > 0) {            // the real-pencil premise, checked on the device
    cudaMemsetAsync(h->realviol, 0, 4, h->stream);
    feast::imag_check_launch(A, lda, n, h->realviol, h->stream);
    if (!h->b_id) feast::imag_check_launch(B, ldb, n, h->realviol, h->stream);
  }
  for (int jb = 0; jb < owned; jb += h->batch) {
    const int nbat = std::min(h->batch, owned - jb);
    const int j = h->j0 + jb;
    // split the batch into G concurrent groups (group 0 on the handle's stream)
    h->big = h->n >= 8192 && nbat >= 16;
    const int gmax = (h->big && !h->groups_set) ? std::min(2, h->groups) : h->groups;
    const int G = (h->group_streams && !h->prof_serial) ? std::max(1, std::min(gmax, nbat)) : 1;
    if (G > 1) cudaEventRecord(h->ev_fork, h->stream);
    // pass 1: per group, the fork, the shift of the first outer block and the LU sequence object
    std::vector<Lu> vs;
    std::vector<LuRun> runs;
    for (int g = 0; g < G; ++g) {
      const int b0 = g * nbat / G, b1 = (g + 1) * nbat / G;
      Lu v{h->Cw + b0 * st, h->Inv + b0 * h->inv_stride, h->ipiv + (int64_t)b0 * n, h->stats + 2 * (j + b0),
           h->info + (j + b0), b1 - b0, g ? h->gs[g] : h->stream, g ? h->gside[g] : h->side, g ? h->gev_a[g] : h->ev_a,
           g ? h->gev_p[g] : h->ev_p, (h->stagger && g + 1 < G) ? h->gev_first[g] : nullptr,
           h->prof_serial ? nullptr : h->gx[g], h->gev_t[g], h->gev_x[g],
           (h->prof_serial || !h->lswap_side) ? nullptr : h->gl[g], h->gev_l[g], h->gev_lj[g]};
      if (g) cudaStreamWaitEvent(v.sm, h->ev_fork, 0);
      vs.push_back(v);
      if (!reuse) {
        feast::stats_init_launch(v.stats, v.info, v.nbat, v.sm);
        // a2: C_j = z_j B - A ; R appended as extra columns (augmented system [C_j | R]).  Only the
        // first outer block's columns are formed before its factorisation starts; the LU forms
        // the rest underneath it (needed only once the block is factored).
        const int64_t w0 = std::min<int64_t>(first_block(h), n);
        const double2* zj = h->zd + j + b0;
        feast::shift_launch(bat(v.Cw, ld, st), A, lda, B, ldb, zj, n, v.nbat, v.sm, 0, w0);
        // (invoked later, from the round-robin pass 2: the block-scoped values are captured by copy)
        auto rest = [&, zj, v, w0](cudaStream_t sr) {
          feast::shift_launch(bat(v.Cw, ld, st), A, lda, B, ldb, zj, n, v.nbat, sr, w0, n);
          if (rhs_wait) cudaStreamWaitEvent(sr, rhs_wait, 0);
          if (doR)
            feast::broadcast_copy_launch(bat(v.Cw + n * ld, ld, st), Rr, ldr, n, m, v.nbat,
                                         pair ? feast::BC_PAIR : feast::BC_COPY, sr);
          if (csl)
            feast::broadcast_copy_launch(bat(v.Cw + (n + (doR ? m : 0)) * ld, ld, st), Rl, ldrl, n, m, v.nbat,
                                         feast::BC_CONJ, sr);
        };
        // a3 (+ forward substitution of a4): P_j [C_j | R] -> [U_j | L_j^-1 P_j R]
        runs.push_back(LuRun{h, v, solve ? ncr : 0, rest});
      }
    }
    // pass 2: the groups' LU sequences enqueued round-robin, one outer block each per turn; with
    // FEAST_STAGGER = d, group g joins once group g - 1 has enqueued d outer steps (its stream then
    // waits on the event group g - 1 records after them)
    std::vector<char> started(runs.size(), 0);
    for (bool all = runs.empty(); !all;) {
      all = true;
      for (size_t g = 0; g < runs.size(); ++g) {
        if (!started[g]) {
          if (g > 0 && h->stagger > 0) {
            const LuRun& prev = runs[g - 1];
            if (prev.phase != 2 && prev.steps < h->stagger) { all = false; continue; }
            cudaStreamWaitEvent(runs[g].v.sm, h->gev_first[g - 1], 0);
          }
          started[g] = 1;
        }
        all = runs[g].step() && all;
      }
    }
    // pass 3: the substitutions, per node group on its stream (FEAST_SUBST_JOIN=1: the groups,
    // whose LU sequences were enqueued round-robin and finish together, are joined first and the
    // substitutions run once over the whole batch: G times fewer, G times wider launches).
    auto subst = [&](const Lu& v, int b0) {
      if (!reuse) {
        if (doL || h->cache_on)
          feast::perm_launch(v.ipiv, h->perm + (int64_t)b0 * n, h->iperm + (int64_t)b0 * n, n, v.nbat, v.sm);
        // a4: Y_j = U_j^-1 (L_j^-1 P_j R)
        if (solve && !(ablate() & 8)) solve_right_back(h, v, v.Cw + n * ld, st, ncr);
      } else if (doR) {
        // cached factors (NEXT-1, "factored just once"): Y_j = U^-1 L^-1 P_j R
        double2* Yg = h->Y + b0 * ld * mr;   // (factor cache and real-pencil mode are exclusive: mr = m)
        if (rhs_wait) cudaStreamWaitEvent(v.sm, rhs_wait, 0);
        feast::gather_rows_launch(bat(Yg, ld, ld * mr), Rr, ldr, 0, h->perm + (int64_t)b0 * n, n, m, v.nbat, v.sm);
        solve_right_fwd(h, v, Yg, ld * mr, m);
        solve_right_back(h, v, Yg, ld * mr, m);
      }
      if (doL && !csl) {
        // Z_j = P^T L^-H U^-H RL  (P^T folded into the accumulate below)
        double2* Yg = h->YL + b0 * ld * mr;
        if (rhs_wait) cudaStreamWaitEvent(v.sm, rhs_wait, 0);
        feast::broadcast_copy_launch(bat(Yg, ld, ld * mr), Rl, ldrl, n, m, v.nbat, pair, v.sm);
        solve_left(h, v, Yg);
      }
    };
    if (h->subst_join && G > 1) {
      for (int g = 1; g < G; ++g) {
        cudaEventRecord(h->gev_done[g], vs[g].sm);
        cudaStreamWaitEvent(h->stream, h->gev_done[g], 0);
      }
      Lu all = vs[0];
      all.nbat = nbat;
      subst(all, 0);
    } else {
      for (int g = 0; g < G; ++g) {
        subst(vs[g], g * nbat / G);
        if (g) {
          cudaEventRecord(h->gev_done[g], vs[g].sm);
          cudaStreamWaitEvent(h->stream, h->gev_done[g], 0);
        }
      }
    }
    // a5: Q (+)= sum_j w_j Y_j, QL (+)= sum_j conj(w_j) Z_j over the batch in node order
    const double2* wpj = wp ? wp + j : nullptr;
    if (doR) {
      if (!reuse)
        feast::accum_launch(Q, ldq, bat(h->Cw + n * ld, ld, st), h->wd + j, wpj, nullptr, n, m, nbat, false, jb > 0,
                            h->stream);
      else
        feast::accum_launch(Q, ldq, bat(h->Y, ld, ld * mr), h->wd + j, wpj, nullptr, n, m, nbat, false, jb > 0,
                            h->stream);
    }
    if (csl)   // QL (+)= sum_j conj(w_j) conj(C_j^-1 conj RL) = conj(sum_j w_j C_j^-1 conj RL)
      feast::accum_launch(QL, ldql, bat(h->Cw + (n + (doR ? m : 0)) * ld, ld, st), h->wd + j, nullptr, nullptr, n, m,
                          nbat, false, jb > 0, h->stream, true);
    else if (doL)
      feast::accum_launch(QL, ldql, bat(h->YL, ld, ld * mr), h->wd + j, wpj, h->iperm, n, m, nbat, true, jb > 0,
                          h->stream);
  }
  if (owned == 0) {
    if (doR) cudaMemset2DAsync(Q, ldq * 16, 0, n * 16, m, h->stream);
    if (doL) cudaMemset2DAsync(QL, ldql * 16, 0, n * 16, m, h->stream);
  }
}

// Driver: enqueue the sequence (replaying a CUDA graph of it when the call repeats with the same
// pointers: the second identical call is captured, later ones replay it), then read back the
// pivot diagnostics.
// a6: the node sum over ranks (parallelism over the linear systems): one SUM all-reduce
// through the registered callback of the n x m0 block(s) this rank accumulated.  Q and QL are
// packed into the contiguous staging block [Q | QL] (ld = n) so that the callback sees one flat
// float64 buffer (any caller ld) and Bi-FEAST's two blocks travel in one collective.
int node_sum(feast_ctx* h, double2* Q, int64_t ldq, double2* QL, int64_t ldql) {
  if (h->world <= 1 || h->partial) return FEAST_OK;
  if (!h->ar) return fail(h, FEAST_E_COMM, "world > 1 needs feast_set_allreduce (or feast_set_partial)%s");
  const int64_t n = h->n, m = h->m0;
  double2* blk[2] = {Q, QL};
  const int64_t lds[2] = {ldq, ldql};
  int nb = 0;
  for (int k = 0; k < 2; ++k)
    if (blk[k]) {
      CUDA_TRY(h, cudaMemcpy2DAsync(h->NS + nb * n * m, n * 16, blk[k], lds[k] * 16, n * 16, m, cudaMemcpyDeviceToDevice,
                                    h->stream));
      ++nb;
    }
  if (nb == 0) return FEAST_OK;
  if (h->ar(h->NS, 2 * n * m * nb, h->stream, h->ar_user)) return fail(h, FEAST_E_COMM, "all-reduce failed%s");
  nb = 0;
  for (int k = 0; k < 2; ++k)
    if (blk[k]) {
      CUDA_TRY(h, cudaMemcpy2DAsync(blk[k], lds[k] * 16, h->NS + nb * n * m, n * 16, n * 16, m, cudaMemcpyDeviceToDevice,
                                    h->stream));
      ++nb;
    }
  return FEAST_OK;
}

int judge_stats(feast_ctx* h);

int project_impl(feast_ctx* h, const double2* A, int64_t lda, const double2* B, int64_t ldb, const double2* X,
                 int64_t ldx, const double2* V, int64_t ldv, double2* Q, int64_t ldq, double2* QL, int64_t ldql) {
  if (h->world > 1 && !h->partial && !h->ar)
    return fail(h, FEAST_E_COMM, "world > 1 needs feast_set_allreduce (or feast_set_partial)%s");
  const int64_t t0 = feast::g_launches;
  const int owned = h->j1 - h->j0;
  const bool reuse = h->cache_on && h->cache_valid && h->batch >= owned && h->cache_A == A && h->cache_B == B;
  const feast_ctx::GraphKey key{A, B, X, V, Q, QL, lda, ldb, ldx, ldv, ldq, ldql, reuse};
  // a1 with world > 1: rank r forms rows [r n/P, (r+1) n/P) of R = B X (R_L = B^H V), the rest
  // zero, and the all-reduce (sum) through the callback assembles the full block on every rank
  // (an all-gather), before the (graph-captured) node loop reads it
  const bool rhs_ready = !h->b_id && h->world > 1 && h->ar != nullptr && owned > 0;
  if (rhs_ready) {
    const int64_t n = h->n, m = h->m0, ld = h->ldc;
    const int64_t r0 = h->rank * n / h->world, r1 = (h->rank + 1) * n / h->world;
    const double2 one = make_double2(1, 0), zero = make_double2(0, 0);
    for (int k = 0; k < 2; ++k) {
      if (k == 0 ? X == nullptr : V == nullptr) continue;
      double2* R = k == 0 ? h->R : h->RL;
      CUDA_TRY(h, cudaMemsetAsync(R, 0, (size_t)ld * m * 16, h->stream));
      if (k == 0) gemm_gen(h, r1 - r0, m, n, false, B + r0, ldb, X, ldx, R + r0, ld, one, zero);
      else gemm_gen(h, r1 - r0, m, n, true, B + r0 * ldb, ldb, V, ldv, R + r0, ld, one, zero);
      if (h->ar(R, 2 * ld * m, h->stream, h->ar_user)) return fail(h, FEAST_E_COMM, "all-reduce failed%s");
    }
  }
  const bool use_graph = h->graphs && !feast::prof().on;
  if (use_graph && h->gexec && h->gkey == key) {
    CUDA_TRY(h, cudaGraphLaunch(h->gexec, h->stream));
    feast::count_launch((int)h->glaunches);
  } else if (use_graph && h->gseen_valid && h->gseen == key) {
    // second identical call: capture, instantiate, launch
    if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
    cudaGraph_t g = nullptr;
    const int64_t c0 = feast::g_launches;
    CUDA_TRY(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    project_enqueue(h, A, lda, B, ldb, X, ldx, V, ldv, Q, ldq, QL, ldql, reuse, rhs_ready);
    const cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
    h->glaunches = feast::g_launches - c0;
    feast::g_launches = c0;
    if (ce != cudaSuccess ||
        cudaGraphInstantiateWithFlags(&h->gexec, g, cudaGraphInstantiateFlagUseNodePriority) != cudaSuccess) {
      cudaGetLastError();
      if (g) cudaGraphDestroy(g);
      h->gexec = nullptr;
      h->graphs = false;   // capture unsupported here: keep launching the same kernels eagerly
      project_enqueue(h, A, lda, B, ldb, X, ldx, V, ldv, Q, ldq, QL, ldql, reuse, rhs_ready);
    } else {
      cudaGraphDestroy(g);
      h->gkey = key;
      CUDA_TRY(h, cudaGraphLaunch(h->gexec, h->stream));
      feast::count_launch((int)h->glaunches);
    }
  } else {
    project_enqueue(h, A, lda, B, ldb, X, ldx, V, ldv, Q, ldq, QL, ldql, reuse, rhs_ready);
    h->gseen = key;
    h->gseen_valid = true;
  }
  if (!reuse && h->cache_on && h->batch >= owned) { h->cache_valid = true; h->cache_A = A; h->cache_B = B; }
  CUDA_TRY(h, cudaGetLastError());
  if (int e = node_sum(h, Q, ldq, QL, ldql)) return e;
  h->launches = feast::g_launches - t0;
  // pivot diagnostics of the owned units into pinned host memory; judged now (synchronous calls)
  // or by feast_sync (async mode: the call returns once everything is enqueued)
  CUDA_TRY(h, cudaMemcpyAsync(h->h_stats, h->stats, 2 * (size_t)h->nu * 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->h_info, h->info, (size_t)h->nu * 4, cudaMemcpyDeviceToHost, h->stream));
  h->h_info[h->nu] = 0;
  if (h->real) CUDA_TRY(h, cudaMemcpyAsync(h->h_info + h->nu, h->realviol, 4, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaEventRecord(h->ev_stats, h->stream));
  h->pending = true;
  if (h->async) return FEAST_OK;
  return judge_stats(h);
}

// Evaluate the pivot statistics of the last projection (waits for them): FEAST_E_SINGULAR if some
// node's min|u_ii|/max|u_ii| < 1e-14 or an exact zero pivot, FEAST_W_ILLCOND below 1e-10.
int judge_stats(feast_ctx* h) {
  if (!h->pending) return FEAST_OK;
  CUDA_TRY(h, cudaEventSynchronize(h->ev_stats));
  h->pending = false;
  const double* st = h->h_stats;
  const int32_t* inf = h->h_info;
  if (inf[h->nu]) return fail(h, FEAST_E_ARG, "real-pencil mode: A or B has a nonzero imaginary part%s");
  h->minrel.assign(h->q, -1.0);
  h->worst = -1;
  double wr = INFINITY;
  bool singular = false, ill = false;
  for (int u = h->j0; u < h->j1; ++u) {
    const double ratio = st[2 * u + 1] > 0 ? st[2 * u] / st[2 * u + 1] : 0.0;
    const int jj = h->unode[u];
    h->minrel[jj] = inf[u] ? 0.0 : ratio;
    if (h->upart[u] >= 0) h->minrel[h->upart[u]] = h->minrel[jj];
    if (h->minrel[jj] < wr) { wr = h->minrel[jj]; h->worst = jj; }
    if (inf[u] || ratio < 1e-14) singular = true;
    else if (ratio < 1e-10) ill = true;
  }
  if (singular && !(ablate() & 1)) {   // (a timing ablation has no pivots to judge)
    char b[64];
    snprintf(b, sizeof b, "%d", h->worst);
    return fail(h, FEAST_E_SINGULAR, "shifted matrix at node %s is singular (pivot ratio < 1e-14)", b);
  }
  h->err.clear();
  return ill ? FEAST_W_ILLCOND : FEAST_OK;
}

int ensure_iter_mem(feast_ctx* h) {
  if (h->itmem) return FEAST_OK;
  if (!h->sol) {
    SOL_TRY(h, cusolverDnCreate(&h->sol));
    SOL_TRY(h, cusolverDnSetStream(h->sol, h->stream));
    SOL_TRY(h, cusolverDnCreateParams(&h->solp));
  }
  const int64_t n = h->n, m = h->m0;
  // buffers: Qr, Ql (n x m), AX, BX (n x m), Ah, Bh, M, W, Z, T (m x m), lam (m), rn, xn (m),
  // frob partials (256), ipiv (m), info, cusolver workspace
  size_t ws_geqrf = 0, ws_getrf = 0, ws_geev_d = 0, ws_geev_h = 0;
  int lw = 0;
  SOL_TRY(h, cusolverDnZgeqrf_bufferSize(h->sol, (int)n, (int)m, nullptr, (int)n, &lw));
  ws_geqrf = std::max<size_t>(ws_geqrf, (size_t)lw * 16);
  SOL_TRY(h, cusolverDnZungqr_bufferSize(h->sol, (int)n, (int)m, (int)m, nullptr, (int)n, nullptr, &lw));
  ws_geqrf = std::max<size_t>(ws_geqrf, (size_t)lw * 16);
  SOL_TRY(h, cusolverDnZgetrf_bufferSize(h->sol, (int)m, (int)m, nullptr, (int)m, &lw));
  ws_getrf = (size_t)lw * 16;
  SOL_TRY(h, cusolverDnXgeev_bufferSize(h->sol, h->solp, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, m,
                                        CUDA_C_64F, nullptr, m, CUDA_C_64F, nullptr, CUDA_C_64F, nullptr, m,
                                        CUDA_C_64F, nullptr, m, CUDA_C_64F, &ws_geev_d, &ws_geev_h));
  size_t ws_nn_d = 0, ws_nn_h = 0;
  SOL_TRY(h, cusolverDnXgeev_bufferSize(h->sol, h->solp, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_NOVECTOR, m,
                                        CUDA_C_64F, nullptr, m, CUDA_C_64F, nullptr, CUDA_C_64F, nullptr, m,
                                        CUDA_C_64F, nullptr, m, CUDA_C_64F, &ws_nn_d, &ws_nn_h));
  ws_geev_d = std::max(ws_geev_d, ws_nn_d);
  ws_geev_h = std::max(ws_geev_h, ws_nn_h);
  const size_t nm = (size_t)n * m * 16, mm = (size_t)m * m * 16;
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += align256(b); return o; };
  size_t o_q = take(nm), o_ql = take(nm), o_ax = take(nm), o_bx = take(nm);
  size_t o_ah = take(mm), o_bh = take(mm), o_m = take(mm), o_w = take(mm), o_z = take(mm), o_t = take(mm);
  size_t o_rq = take(mm), o_rl = take(mm), o_mu = take(m * 16);
  size_t o_lam = take(m * 16), o_rn = take(m * 8), o_xn = take(m * 8), o_fr = take(256 * 8);
  size_t o_tau = take(m * 16), o_piv = take(m * 4), o_info = take(16);
  size_t o_sw = take(std::max({ws_geqrf, ws_getrf, ws_geev_d, (size_t)256}));
  h->itbytes = off;
  CUDA_TRY(h, cudaMalloc(&h->itmem, off));
  char* base = (char*)h->itmem;
  h->it.Qr = (double2*)(base + o_q);
  h->it.Ql = (double2*)(base + o_ql);
  h->it.AX = (double2*)(base + o_ax);
  h->it.BX = (double2*)(base + o_bx);
  h->it.Ah = (double2*)(base + o_ah);
  h->it.Bh = (double2*)(base + o_bh);
  h->it.M = (double2*)(base + o_m);
  h->it.W = (double2*)(base + o_w);
  h->it.Z = (double2*)(base + o_z);
  h->it.T = (double2*)(base + o_t);
  h->it.Rq = (double2*)(base + o_rq);
  h->it.Rl = (double2*)(base + o_rl);
  h->it.mu = (double2*)(base + o_mu);
  h->it.lam = (double2*)(base + o_lam);
  h->it.rn = (double*)(base + o_rn);
  h->it.xn = (double*)(base + o_xn);
  h->it.fr = (double*)(base + o_fr);
  h->it.tau = (double2*)(base + o_tau);
  h->it.piv = (int*)(base + o_piv);
  h->it.info = (int*)(base + o_info);
  h->it.sw = (void*)(base + o_sw);
  h->it.sw_bytes = std::max({ws_geqrf, ws_getrf, ws_geev_d, (size_t)256});
  h->it.hw.resize(std::max<size_t>(ws_geev_h, 16));
  return FEAST_OK;
}

// NEXT-3 count estimate: eigenvalues of the m0 x m0 matrix V^^H B U^ (device, ld m,
// destroyed) by cuSOLVER Xgeev without vectors, sorted by decreasing modulus (stable in index);
// count = #{|mu| >= 1/4}: |rho(lambda)| >= 1/2, the filter's half height (reading R21), since
// V^^H B U^ = V^H B rho(B^-1 A)^2 U with V^H B U = I.
int bhat_count(feast_ctx* h, double2* M) {
  const int64_t m = h->m0;
  auto& it = h->it;
  SOL_TRY(h, cusolverDnXgeev(h->sol, h->solp, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_NOVECTOR, m, CUDA_C_64F, M,
                             m, CUDA_C_64F, it.mu, CUDA_C_64F, nullptr, m, CUDA_C_64F, nullptr, m, CUDA_C_64F, it.sw,
                             it.sw_bytes, it.hw.data(), it.hw.size(), it.info));
  std::vector<double2> mu(m);
  int hinfo = 0;
  CUDA_TRY(h, cudaMemcpyAsync(mu.data(), it.mu, m * 16, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(&hinfo, it.info, 4, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (hinfo != 0) return fail(h, FEAST_E_REDUCED, "eig(V^H B U) failed%s");
  std::vector<int> ord(m);
  for (int64_t i = 0; i < m; ++i) ord[i] = (int)i;
  std::stable_sort(ord.begin(), ord.end(),
                   [&](int a, int b) { return std::hypot(mu[a].x, mu[a].y) > std::hypot(mu[b].x, mu[b].y); });
  h->mon_mu.resize(m);
  h->mon_count = 0;
  for (int64_t i = 0; i < m; ++i) {
    h->mon_mu[i] = mu[ord[i]];
    if (std::hypot(mu[ord[i]].x, mu[ord[i]].y) >= 0.25) ++h->mon_count;
  }
  return FEAST_OK;
}

// Factorisation units and their ownership (reading R17 applied to units): plain nodes, or in
// real-pencil mode the orbits of conjugate poles {z, conj z} (NEXT-2b; P:899-905 / S:282, S:291:
// for real A, B, C(conj z) = conj(C(z)), so the partner's solve is conj(C(z)^-1 conj R)).
int setup_units(feast_ctx* h) {
  h->zu.clear(); h->wu.clear(); h->wpu.clear(); h->unode.clear(); h->upart.clear();
  if (!h->real) {
    h->zu = h->z; h->wu = h->w;
    for (int j = 0; j < h->q; ++j) { h->unode.push_back(j); h->upart.push_back(-1); }
  } else {
    const double tol = 1e-12 * h->r;
    std::vector<bool> taken(h->q, false);
    for (int j = 0; j < h->q; ++j) {
      if (h->z[j].y < -tol) continue;        // lower half plane: a partner, found below
      int p = -1;
      if (h->z[j].y > tol)
        for (int k = 0; k < h->q; ++k)
          if (!taken[k] && h->z[k].y < -tol && std::fabs(h->z[k].x - h->z[j].x) <= tol &&
              std::fabs(h->z[k].y + h->z[j].y) <= tol) { p = k; break; }
      if (h->z[j].y > tol && p < 0) return -1;   // contour not symmetric about the real axis
      if (p >= 0) taken[p] = true;
      h->zu.push_back(h->z[j]);
      h->wu.push_back(h->w[j]);
      h->wpu.push_back(p >= 0 ? h->w[p] : make_double2(0.0, 0.0));
      h->unode.push_back(j);
      h->upart.push_back(p);
    }
    for (int k = 0; k < h->q; ++k)
      if (h->z[k].y < -tol && !taken[k]) return -1;
  }
  h->nu = (int)h->zu.size();
  if (h->nu % h->world != 0) return -1;
  h->j0 = h->rank * (h->nu / h->world);
  h->j1 = (h->rank + 1) * (h->nu / h->world);
  const int owned = h->j1 - h->j0;
  h->batch = std::max(1, h->max_batch == 0 ? owned : std::min<int>(h->max_batch, owned));
  h->mr = (h->real || (h->csym && h->mode == FEAST_BI)) ? 2 * h->m0 : h->m0;
  // few concurrent LUs: the panel chain bounds the step, so panels take the faster 8-warp form
  // (measured C2 rank shares: 4 nodes 7.5 -> 7.2 ms, 2 nodes 6.4 -> 6.2 ms; 16 nodes lose 4 %)
  h->panel_one_row = h->batch <= 4;
  if (const char* e = getenv("FEAST_PANEL_1ROW")) h->panel_one_row = e[0] == '1';
  return 0;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* feast_version(void) { return "feast_b200 0.1 (sm_100a)"; }

int feast_init(feast_handle* out, int64_t n, int64_t m0, double c_re, double c_im, double r, double aspect,
               int32_t n_e, int32_t rule, int32_t mode, int32_t b_is_identity, int32_t rank, int32_t world,
               int32_t max_batch, void* cuda_stream) {
  if (!out) return FEAST_E_ARG;
  *out = nullptr;
  if (n < 1 || m0 < 1 || m0 > n || !(r > 0) || !(aspect > 0) || world < 1 || rank < 0 || rank >= world ||
      (mode != FEAST_RIGHT && mode != FEAST_BI) || max_batch < 0)
    return FEAST_E_ARG;
  feast_ctx* h = new feast_ctx();
  h->n = n; h->m0 = m0; h->c_re = c_re; h->c_im = c_im; h->r = r; h->aspect = aspect;
  h->n_e = n_e; h->rule = rule; h->mode = mode; h->b_id = b_is_identity != 0;
  h->rank = rank; h->world = world;
  h->stream = h->caller = (cudaStream_t)cuda_stream;
  h->max_batch = max_batch;
  if (make_nodes(h) != 0 || h->q % world != 0 || setup_units(h) != 0) { delete h; return FEAST_E_ARG; }
  h->pcfg = feast::panel_config(n);
  if (h->pcfg.cluster == 0) { delete h; return FEAST_E_ARG; }
  // panel strategy: shared-memory cluster panel when the n x nb panel fits in <= 16 CTAs
  h->smem_cs = 0;
  h->nb = 64;   // the diagonal-block inverses (trtri) use 64-row blocks
  if (const char* e = getenv("FEAST_WP")) {
    const long v = atol(e);
    if (v == 8 || v == 16 || v == 32 || v == 64) h->wp = v;
  }
  // smallest cluster whose CTAs hold <= 256 panel rows (two per thread: no register spills)
  for (int cs = 1; cs <= 16; cs *= 2)
    if (feast::panel_smem_fits(n, (int)h->wp, cs) && (n + cs - 1) / cs <= 256) { h->smem_cs = cs; break; }
  if (const char* e = getenv("FEAST_CS")) {
    const int v = atoi(e);
    if (v >= 1 && v <= 16 && feast::panel_smem_fits(n, (int)h->wp, v)) h->smem_cs = v;
  }
  h->smem_cs_max = std::max(h->smem_cs, 16);
  if (const char* e = getenv("FEAST_CS_MAX")) {
    const int v = atoi(e);
    if (v == 0 || v == 1 || v == 2 || v == 4 || v == 8 || v == 16) h->smem_cs_max = v;
  }
  if (const char* e = getenv("FEAST_PANEL")) {   // debugging override: "reg" = register-chunk kernel
    if (e[0] == 'r') { h->smem_cs = 0; h->smem_cs_max = 0; h->nb = 64; }
  }
  if (const char* e = getenv("FEAST_LOOKAHEAD")) h->lookahead = e[0] != '0';
  if (const char* e = getenv("FEAST_GRAPH")) h->graphs = e[0] != '0';
  if (const char* e = getenv("FEAST_LASWP"))
    h->laswp_variant = e[0] == 'p' ? feast::LASWP_PERM : (e[0] == 'c' && e[1] == 'h') ? feast::LASWP_CHAIN : feast::LASWP_COALESCED;
  if (const char* e = getenv("FEAST_STAGGER")) h->stagger = std::max(0, atoi(e));
  if (const char* e = getenv("FEAST_WIDE_ROWS")) h->wide_panel_rows = atol(e);
  if (const char* e = getenv("FEAST_GROUPS")) {
    const int v = atoi(e);
    if (v >= 1 && v <= feast_ctx::GMAX) { h->groups = v; h->groups_set = true; }
  }
  // large n: wider outer blocks (trailing updates with K = 512) and substitution blocks (measured
  // C3 / C4 / C5: -0.4 / -0.7 / -1.6 % per step with 512 instead of 256)
  if (n >= 8192) { h->nbo = 512; h->solve_nb = 512; }
  // dot-form substitutions from n = 8192 (C4 12.898 -> 12.838 s, C3 1544.6 -> 1543.3 ms; C2 16.51 vs
  // 16.57 ms right-looking: its short K = 256 blocks do not pay)
  h->subst_dot = n >= 8192;
  if (const char* e = getenv("FEAST_BTRSM")) h->btrsm = e[0] == '1';
  if (const char* e = getenv("FEAST_SUBST_DOT")) h->subst_dot = e[0] == '1';
  h->u12_dot = n >= 8192 ? 1 : 0;
  if (const char* e = getenv("FEAST_SUBST_INNER_DOT")) h->inner_dot = std::max(0, std::min(2, atoi(e)));
  if (const char* e = getenv("FEAST_U12_DOT")) h->u12_dot = std::max(0, std::min(2, atoi(e)));
  if (const char* e = getenv("FEAST_SUBST_JOIN")) h->subst_join = e[0] == '1';
  if (const char* e = getenv("FEAST_PANEL_SWAP")) h->panel_swap = e[0] != '0';
  if (const char* e = getenv("FEAST_LSWAP_SIDE")) h->lswap_side = e[0] != '0';
  if (const char* e = getenv("FEAST_SOLVE_NB")) {
    const long v = atol(e);
    if (v >= 64 && v % 64 == 0) h->solve_nb = v;
  }
  if (const char* e = getenv("FEAST_NBO")) {
    const long v = atol(e);
    if (v >= 64 && v <= 1024 && v % 64 == 0) h->nbo = v;
  }
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_p, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      h->lookahead = false;   // no CUDA context (CPU-only validation): launches never happen
    } else if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) == cudaSuccess &&
               cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming) == cudaSuccess &&
               cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming) == cudaSuccess) {
      h->own_stream = true;
      bool ok = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
                cudaStreamCreateWithFlags(&h->s_rhs, cudaStreamNonBlocking) == cudaSuccess &&
                cudaEventCreateWithFlags(&h->ev_a1, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&h->ev_rhs, cudaEventDisableTiming) == cudaSuccess;
      for (int g = 1; g < feast_ctx::GMAX && ok; ++g)
        ok = cudaStreamCreateWithFlags(&h->gs[g], cudaStreamNonBlocking) == cudaSuccess &&
             cudaStreamCreateWithPriority(&h->gside[g], cudaStreamNonBlocking, hi) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->gev_a[g], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->gev_p[g], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->gev_done[g], cudaEventDisableTiming) == cudaSuccess;
      for (int g = 0; g < feast_ctx::GMAX && ok; ++g)
        ok = cudaStreamCreateWithPriority(&h->gl[g], cudaStreamNonBlocking, lo) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->gev_l[g], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->gev_lj[g], cudaEventDisableTiming) == cudaSuccess;
      for (int g = 0; g < feast_ctx::GMAX && ok; ++g)
        ok = cudaEventCreateWithFlags(&h->gev_first[g], cudaEventDisableTiming) == cudaSuccess &&
             cudaStreamCreateWithFlags(&h->gx[g], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->gev_t[g], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->gev_x[g], cudaEventDisableTiming) == cudaSuccess;
      if (!ok) { cudaGetLastError(); h->groups = 1; h->group_streams = false; }
      else h->group_streams = true;
    } else {
      cudaGetLastError();
      h->stream = h->caller;
    }
  }
  h->ldc = (n + 7) / 8 * 8;
  *out = h;
  return FEAST_OK;
}

// Workspace layout.  base == nullptr: size only (the handle's pointers are left untouched, so the
// call is safe after a workspace is bound).
static size_t layout(feast_ctx* h, char* base) {
  const int64_t n = h->n, m = h->m0, ld = h->ldc;
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += align256(b); return o; };
  auto set = [&](auto*& ptr, size_t b, bool want = true) {
    if (!want) { if (base) ptr = nullptr; return; }
    const size_t o = take(b);
    if (base) ptr = reinterpret_cast<std::remove_reference_t<decltype(ptr)>>(base + o);
  };
  const int64_t mr = h->mr;
  const bool bi = h->mode == FEAST_BI;
  set(h->Cw, (size_t)h->batch * ld * (n + mr) * 16);  // [C_j | R (| conj R)] (augmented)
  set(h->Y, (size_t)h->batch * ld * mr * 16);           // right solves with cached factors
  set(h->YL, (size_t)h->batch * ld * mr * 16, bi);
  set(h->R, (size_t)ld * m * 16, !h->b_id);
  set(h->RL, (size_t)ld * m * 16, !h->b_id && bi);
  set(h->AQ, (size_t)ld * m * 16);
  set(h->BQ, (size_t)ld * m * 16, !h->b_id);
  // split-K partials: up to 6 n x m0 slices (grids that small need splits; large ones do not),
  // capped at 512 MB
  h->sk_elems = std::max<int64_t>(16 * m * m, std::min<int64_t>((int64_t)6 * ld * m, (int64_t)1 << 25));
  set(h->SK, (size_t)h->sk_elems * 16);
  h->nblk = (n + 63) / 64;
  h->inv_stride = h->nblk * 2 * 4096;
  set(h->Inv, (size_t)h->batch * h->inv_stride * 16);
  set(h->ipiv, (size_t)h->batch * n * 4);
  set(h->perm, (size_t)h->batch * n * 4);
  set(h->iperm, (size_t)h->batch * n * 4);
  set(h->zd, (size_t)h->nu * 16);
  set(h->wd, (size_t)h->nu * 16);
  set(h->wpd, (size_t)h->nu * 16, h->real);
  set(h->stats, (size_t)h->nu * 16);
  set(h->info, (size_t)h->nu * 4);
  set(h->realviol, 16);
  set(h->NS, (size_t)n * m * (bi ? 2 : 1) * 16, h->world > 1);   // node-sum staging [Q | QL]
  return off;
}

int feast_workspace_bytes(feast_handle h, size_t* bytes) {
  if (!h || !bytes) return FEAST_E_ARG;
  *bytes = layout(h, nullptr);
  if (h->ws) return FEAST_OK;   // bound: the batch (and the layout) stay frozen
  if (h->max_batch == 0) {
    // "all owned nodes" means all that fit: shrink the concurrent batch until the workspace
    // takes at most 90 % of the device memory free now (C5 on one B200: 16 nodes x 17.7 GB of
    // augmented blocks do not fit next to A and B; 4 do)
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && free_b > 0) {
      const size_t cap = free_b / 10 * 9;
      while (*bytes > cap && h->batch > 1) {
        h->batch = std::max(1, h->batch * 3 / 4);
        *bytes = layout(h, nullptr);
      }
      if (!getenv("FEAST_PANEL_1ROW")) h->panel_one_row = h->batch <= 4;
    } else {
      cudaGetLastError();
    }
  }
  return FEAST_OK;
}

int feast_bind_workspace(feast_handle h, void* p, size_t bytes) {
  if (!h || !p) return FEAST_E_ARG;
  const size_t need = layout(h, nullptr);
  if (bytes < need) return fail(h, FEAST_E_NOMEM, "workspace too small%s");
  if (((uintptr_t)p) & 255) return fail(h, FEAST_E_ARG, "workspace not 256-byte aligned%s");
  graph_reset(h);
  if (!h->h_stats) {
    CUDA_TRY(h, cudaMallocHost(&h->h_stats, 2 * (size_t)h->q * 8 + 64));
    CUDA_TRY(h, cudaMallocHost(&h->h_info, ((size_t)h->q + 1) * 4 + 64));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_stats, cudaEventDisableTiming));
  }
  h->ws = p;
  h->ws_bytes = bytes;
  layout(h, (char*)p);
  CUDA_TRY(h, cudaMemcpyAsync(h->zd, h->zu.data(), h->nu * 16, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->wd, h->wu.data(), h->nu * 16, cudaMemcpyHostToDevice, h->stream));
  if (h->real)
    CUDA_TRY(h, cudaMemcpyAsync(h->wpd, h->wpu.data(), h->nu * 16, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return FEAST_OK;
}

int feast_nodes(feast_handle h, int32_t* q, double* z, double* w, int32_t* j0, int32_t* j1) {
  if (!h) return FEAST_E_ARG;
  if (q) *q = h->q;
  if (z) std::memcpy(z, h->z.data(), h->q * 16);
  if (w) std::memcpy(w, h->w.data(), h->q * 16);
  if (j0) *j0 = h->j0;
  if (j1) *j1 = h->j1;
  return FEAST_OK;
}

int feast_project(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb, const void* X, int64_t ldx,
                  void* Q, int64_t ldq) {
  int e = check_args_common(h, A, lda, B, ldb);
  if (e) return e;
  if (!X || !Q || ldx < h->n || ldq < h->n) return fail(h, FEAST_E_ARG, "X/Q null or ld < n%s");
  Join j_(h);
  return project_impl(h, (const double2*)A, lda, (const double2*)B, ldb, (const double2*)X, ldx, nullptr, 0,
                      (double2*)Q, ldq, nullptr, 0);
}

int feast_project_left(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb, const void* V,
                       int64_t ldv, void* QL, int64_t ldql) {
  int e = check_args_common(h, A, lda, B, ldb);
  if (e) return e;
  if (h->mode != FEAST_BI) return fail(h, FEAST_E_STATE, "left projector needs a FEAST_BI handle%s");
  if (!V || !QL || ldv < h->n || ldql < h->n) return fail(h, FEAST_E_ARG, "V/QL null or ld < n%s");
  Join j_(h);
  return project_impl(h, (const double2*)A, lda, (const double2*)B, ldb, nullptr, 0, (const double2*)V, ldv, nullptr,
                      0, (double2*)QL, ldql);
}

int feast_project_bi(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb, const void* X, int64_t ldx,
                     const void* V, int64_t ldv, void* Q, int64_t ldq, void* QL, int64_t ldql) {
  int e = check_args_common(h, A, lda, B, ldb);
  if (e) return e;
  if (h->mode != FEAST_BI) return fail(h, FEAST_E_STATE, "bi projector needs a FEAST_BI handle%s");
  if (!X || !Q || !V || !QL || ldx < h->n || ldq < h->n || ldv < h->n || ldql < h->n)
    return fail(h, FEAST_E_ARG, "X/V/Q/QL null or ld < n%s");
  Join j_(h);
  return project_impl(h, (const double2*)A, lda, (const double2*)B, ldb, (const double2*)X, ldx, (const double2*)V, ldv,
                      (double2*)Q, ldq, (double2*)QL, ldql);
}

}  // extern "C"

namespace {
// a7 with the rows of A Q (B Q) split over the ranks when `shard` (world > 1 and an all-reduce
// callback): rank r forms AQ for rows [r n/P, (r+1) n/P) and the partial QL_r^H AQ_r; one
// all-reduce of the two m0 x m0 partials completes Ahat, Bhat ("must be
// row-sharded across ranks").  Without sharding every rank forms the whole product (AQ / BQ
// stay complete in the workspace, as feast_iterate's residuals need).
int reduce_impl(feast_ctx* h, const void* A, int64_t lda, const void* B, int64_t ldb, const void* Q, int64_t ldq,
                const void* QL, int64_t ldql, void* Ahat, int64_t ldah, void* Bhat, int64_t ldbh, bool shard) {
  const int64_t n = h->n, m = h->m0, ld = h->ldc;
  const double2 one = make_double2(1, 0), zero = make_double2(0, 0);
  const double2* Qr = (const double2*)Q;
  const double2* Ql = QL ? (const double2*)QL : Qr;
  if (!QL) ldql = ldq;
  const int64_t t0 = feast::g_launches;
  shard = shard && h->world > 1 && h->ar != nullptr;
  const int64_t r0 = shard ? h->rank * n / h->world : 0, r1 = shard ? (h->rank + 1) * n / h->world : n, nr = r1 - r0;
  // a7: AQ = A Q, BQ = B Q, Ahat = QL^H AQ, Bhat = QL^H BQ  (rows [r0, r1) when sharded)
  gemm_gen(h, nr, m, n, false, (const double2*)A + r0, lda, Qr, ldq, h->AQ + r0, ld, one, zero);
  gemm_gen(h, m, m, nr, true, Ql + r0, ldql, h->AQ + r0, ld, (double2*)Ahat, ldah, one, zero);
  if (!h->b_id) {
    gemm_gen(h, nr, m, n, false, (const double2*)B + r0, ldb, Qr, ldq, h->BQ + r0, ld, one, zero);
    gemm_gen(h, m, m, nr, true, Ql + r0, ldql, h->BQ + r0, ld, (double2*)Bhat, ldbh, one, zero);
  } else {
    gemm_gen(h, m, m, nr, true, Ql + r0, ldql, Qr + r0, ldq, (double2*)Bhat, ldbh, one, zero);
  }
  CUDA_TRY(h, cudaGetLastError());
  if (shard) {
    for (int k = 0; k < 2; ++k) {
      double2* M = (double2*)(k ? Bhat : Ahat);
      const int64_t ldm = k ? ldbh : ldah;
      if (ldm == m) {
        if (h->ar(M, 2 * m * m, h->stream, h->ar_user)) return fail(h, FEAST_E_COMM, "all-reduce failed%s");
      } else {
        for (int64_t c = 0; c < m; ++c)
          if (h->ar(M + c * ldm, 2 * m, h->stream, h->ar_user)) return fail(h, FEAST_E_COMM, "all-reduce failed%s");
      }
    }
  }
  if (!h->async) CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->launches = feast::g_launches - t0;
  return FEAST_OK;
}
}  // namespace

extern "C" {

int feast_reduce(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb, const void* Q, int64_t ldq,
                 const void* QL, int64_t ldql, void* Ahat, int64_t ldah, void* Bhat, int64_t ldbh) {
  int e = check_args_common(h, A, lda, B, ldb);
  if (e) return e;
  if (!Q || !Ahat || !Bhat || ldq < h->n || ldah < h->m0 || ldbh < h->m0 || (QL && ldql < h->n))
    return fail(h, FEAST_E_ARG, "reduce: null pointer or bad ld%s");
  Join j_(h);
  return reduce_impl(h, A, lda, B, ldb, Q, ldq, QL, ldql, Ahat, ldah, Bhat, ldbh, true);
}

int feast_estimate_count(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb, const void* U,
                         int64_t ldu, void* Q, int64_t ldq, double* estimate) {
  int e = check_args_common(h, A, lda, B, ldb);
  if (e) return e;
  if (!U || !Q || !estimate || ldu < h->n || ldq < h->n) return fail(h, FEAST_E_ARG, "U/Q/estimate null or ld < n%s");
  Join j_(h);
  const int64_t n = h->n, m = h->m0;
  // Q = rho(B^-1 A) U (this rank's nodes, then the node sum over ranks inside project_impl)
  int pst = project_impl(h, (const double2*)A, lda, (const double2*)B, ldb, (const double2*)U, ldu, nullptr, 0,
                               (double2*)Q, ldq, nullptr, 0);
  if (pst < 0) return pst;
  if (h->async && (pst = judge_stats(h)) < 0) return pst;   // these calls read their results now
  // Hutchinson trace estimate: m ~ tr rho(B^-1 A) ~ Re tr(U^H Q) / m0 (deterministic block sums)
  constexpr int NP = 64;
  feast::cdot_launch((const double2*)U, ldu, (const double2*)Q, ldq, n, m, h->SK, NP, h->stream);
  std::vector<double2> part(NP);
  CUDA_TRY(h, cudaMemcpyAsync(part.data(), h->SK, NP * 16, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  double re = 0.0;
  for (const double2& p : part) re += p.x;
  *estimate = re / (double)m;
  return pst;
}

int feast_set_allreduce(feast_handle h, feast_allreduce_fn fn, void* user) {
  if (!h) return FEAST_E_ARG;
  h->ar = fn;
  h->ar_user = user;
  return FEAST_OK;
}

int feast_set_partial(feast_handle h, int32_t enable) {
  if (!h) return FEAST_E_ARG;
  h->partial = enable != 0;
  return FEAST_OK;
}

int feast_iterate(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb, void* X, int64_t ldx,
                  void* V, int64_t ldv, double* ritz, double* resid, int32_t* flags) {
  int e = check_args_common(h, A, lda, B, ldb);
  if (e) return e;
  const bool bi = h->mode == FEAST_BI;
  if (!X || ldx < h->n || (bi && (!V || ldv < h->n))) return fail(h, FEAST_E_ARG, "X/V null or ld < n%s");
  if (h->world > 1 && !h->ar) return fail(h, FEAST_E_COMM, "world > 1 needs feast_set_allreduce%s");
  if (h->world > 1 && h->partial) return fail(h, FEAST_E_STATE, "feast_iterate needs the full node sum (partial mode on)%s");
  Join j_(h);
  e = ensure_iter_mem(h);
  if (e) return e;
  const int64_t n = h->n, m = h->m0, ld = h->ldc;
  auto& it = h->it;
  const double2 one = make_double2(1, 0), zero = make_double2(0, 0);
  // steps 3 (and 4-5 Bi): projector(s)
  int pst = bi ? project_impl(h, (const double2*)A, lda, (const double2*)B, ldb, (const double2*)X, ldx,
                              (const double2*)V, ldv, it.Qr, n, it.Ql, n)
               : project_impl(h, (const double2*)A, lda, (const double2*)B, ldb, (const double2*)X, ldx, nullptr, 0,
                              it.Qr, n, nullptr, 0);
  if (pst < 0) return pst;   // (node-summed over the ranks inside project_impl)
  if (h->async && (pst = judge_stats(h)) < 0) return pst;
  // orthonormalise U^ (and V^) (reading R13), cuSOLVER Householder QR
  // FEAST_TIMING=1: host wall time of the iteration phases (stream-synchronised), to stderr
  static const bool timing = getenv("FEAST_TIMING") != nullptr;
  auto tmark = [&](const char* what) {
    if (!timing) return;
    static double last = 0.0;
    cudaStreamSynchronize(h->stream);
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    const double now = ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
    if (what) fprintf(stderr, "feast_iterate %-12s %8.3f ms\n", what, now - last);
    last = now;
  };
  tmark(nullptr);
  const bool count = bi && h->count_on;
  auto orth = [&](double2* Qb, double2* Rk) -> int {
    SOL_TRY(h, cusolverDnZgeqrf(h->sol, (int)n, (int)m, (cuDoubleComplex*)Qb, (int)n, (cuDoubleComplex*)it.tau,
                                (cuDoubleComplex*)it.sw, (int)(it.sw_bytes / 16), it.info));
    if (Rk) {   // keep R (U^ = Q_o R) for the count estimate: V^^H B U^ = R_l^H (V_o^H B U_o) R_q
      CUDA_TRY(h, cudaMemcpy2DAsync(Rk, m * 16, Qb, n * 16, m * 16, m, cudaMemcpyDeviceToDevice, h->stream));
      feast::tril_zero_launch(Rk, m, m, h->stream);
    }
    SOL_TRY(h, cusolverDnZungqr(h->sol, (int)n, (int)m, (int)m, (cuDoubleComplex*)Qb, (int)n, (cuDoubleComplex*)it.tau,
                                (cuDoubleComplex*)it.sw, (int)(it.sw_bytes / 16), it.info));
    return 0;
  };
  tmark("project");
  if ((e = orth(it.Qr, count ? it.Rq : nullptr))) return e;
  if (bi && (e = orth(it.Ql, count ? it.Rl : nullptr))) return e;
  // step 4 / 6: reduced matrices, rows of A Q (B Q) sharded over the ranks
  e = reduce_impl(h, A, lda, B, ldb, it.Qr, n, bi ? it.Ql : nullptr, n, it.Ah, m, it.Bh, m, true);
  if (e) return e;
  h->mon_count = -1;
  h->mon_mu.clear();
  if (count) {   // NEXT-3: eig(V^^H B U^) of this iteration's steps 4-5
    gemm_gen(h, m, m, m, false, it.Bh, m, it.Rq, m, it.W, m, one, zero);
    gemm_gen(h, m, m, m, true, it.Rl, m, it.W, m, it.Z, m, one, zero);
    if ((e = bhat_count(h, it.Z))) return e;
  }
  tmark("qr+reduce");
  // step 5 / 7 (outside the hot path): M = Bh^-1 Ah, eig(M) -> lam, W
  CUDA_TRY(h, cudaMemcpyAsync(it.T, it.Bh, m * m * 16, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(it.M, it.Ah, m * m * 16, cudaMemcpyDeviceToDevice, h->stream));
  SOL_TRY(h, cusolverDnZgetrf(h->sol, (int)m, (int)m, (cuDoubleComplex*)it.T, (int)m, (cuDoubleComplex*)it.sw,
                              it.piv, it.info));
  SOL_TRY(h, cusolverDnZgetrs(h->sol, CUBLAS_OP_N, (int)m, (int)m, (cuDoubleComplex*)it.T, (int)m, it.piv,
                              (cuDoubleComplex*)it.M, (int)m, it.info));
  int hinfo = 0;
  SOL_TRY(h, cusolverDnXgeev(h->sol, h->solp, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, m, CUDA_C_64F,
                             it.M, m, CUDA_C_64F, it.lam, CUDA_C_64F, nullptr, m, CUDA_C_64F, it.W, m, CUDA_C_64F,
                             it.sw, it.sw_bytes, it.hw.data(), it.hw.size(), it.info));
  CUDA_TRY(h, cudaMemcpyAsync(&hinfo, it.info, 4, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (hinfo != 0) {
    char b[32];
    snprintf(b, sizeof b, "%d", hinfo);
    return fail(h, FEAST_E_REDUCED, "reduced eigensolver info = %s", b);
  }
  tmark("reduced-eig");
  // step 6 / 8: X = U^ W with unit columns (scale folded into W)
  gemm_gen(h, n, m, m, false, it.Qr, n, it.W, m, (double2*)X, ldx, one, zero);
  feast::resid_launch((double2*)X, (double2*)X, (double2*)X, ldx, it.lam, n, m, it.rn, it.xn, h->stream);
  feast::colscale_launch((double2*)X, ldx, n, it.W, m, m, it.xn, h->stream);
  if (bi) {
    // Z = (Bh W)^-H ; V = V^ Z
    gemm_gen(h, m, m, m, false, it.Bh, m, it.W, m, it.T, m, one, zero);
    SOL_TRY(h, cusolverDnZgetrf(h->sol, (int)m, (int)m, (cuDoubleComplex*)it.T, (int)m, (cuDoubleComplex*)it.sw,
                                it.piv, it.info));
    std::vector<double2> I((size_t)m * m, make_double2(0, 0));
    for (int64_t i = 0; i < m; ++i) I[i + i * m] = make_double2(1, 0);
    CUDA_TRY(h, cudaMemcpyAsync(it.Z, I.data(), m * m * 16, cudaMemcpyHostToDevice, h->stream));
    SOL_TRY(h, cusolverDnZgetrs(h->sol, CUBLAS_OP_C, (int)m, (int)m, (cuDoubleComplex*)it.T, (int)m, it.piv,
                                (cuDoubleComplex*)it.Z, (int)m, it.info));
    gemm_gen(h, n, m, m, false, it.Ql, n, it.Z, m, (double2*)V, ldv, one, zero);
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  }
  // residuals (reading R11): A x - l B x with x = U^ W (unit columns), over this rank's rows of
  // A Q (B Q) when a7 was sharded: squared column norms, summed over the ranks (one m-vector)
  const bool shard = h->world > 1 && h->ar != nullptr;
  const int64_t r0 = shard ? h->rank * n / h->world : 0, r1 = shard ? (h->rank + 1) * n / h->world : n, nr = r1 - r0;
  gemm_gen(h, nr, m, m, false, h->AQ + r0, ld, it.W, m, it.AX + r0, n, one, zero);
  const double2* BXp = (const double2*)X;
  int64_t ldbx = ldx;
  if (!h->b_id) { gemm_gen(h, nr, m, m, false, h->BQ + r0, ld, it.W, m, it.BX + r0, n, one, zero); BXp = it.BX; ldbx = n; }
  if (ldbx != n) {  // resid kernel uses one ld: copy X into BX when B = I and ldx != n
    CUDA_TRY(h, cudaMemcpy2DAsync(it.BX, n * 16, X, ldx * 16, n * 16, m, cudaMemcpyDeviceToDevice, h->stream));
    BXp = it.BX;
  }
  feast::resid_launch(it.AX + r0, BXp + r0, BXp + r0, n, it.lam, nr, m, it.rn, nullptr, h->stream, true);
  if (shard && h->ar(it.rn, m, h->stream, h->ar_user)) return fail(h, FEAST_E_COMM, "all-reduce failed%s");
  feast::frob2_launch((const double2*)A, lda, n, it.fr, 256, h->stream);
  std::vector<double2> lam(m);
  std::vector<double> rn(m), fr(256);
  CUDA_TRY(h, cudaMemcpyAsync(lam.data(), it.lam, m * 16, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(rn.data(), it.rn, m * 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(fr.data(), it.fr, 256 * 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  double an = 0.0;
  for (double v : fr) an += v;
  an = std::sqrt(an);
  tmark("ritz+resid");
  h->mon_res = -1.0;
  h->mon_trace = make_double2(0.0, 0.0);
  h->mon_ncand = 0;
  for (int64_t c = 0; c < m; ++c) {
    if (ritz) { ritz[2 * c] = lam[c].x; ritz[2 * c + 1] = lam[c].y; }
    const double rp = std::sqrt(rn[c]);  // ||x|| = 1
    if (resid) resid[c] = an > 0 ? rp / an : rp;
    const bool inside = inside_contour(h, lam[c].x, lam[c].y);
    if (flags) flags[c] = (inside ? 1 : 0) | ((inside && rp <= 1e-4) ? 2 : 0);
    if (inside && rp <= 1e-4) {   // candidate: Res_(k) and trace_(k)
      ++h->mon_ncand;
      h->mon_res = std::max(h->mon_res, rp);
      h->mon_trace.x += lam[c].x;
      h->mon_trace.y += lam[c].y;
    }
  }
  return pst;
}

int feast_set_count_estimate(feast_handle h, int32_t enable) {
  if (!h) return FEAST_E_ARG;
  h->count_on = enable != 0;
  return FEAST_OK;
}

int feast_monitors(feast_handle h, double* res_k, double* trace_k, int32_t* ncand, double* mu, int32_t* count) {
  if (!h) return FEAST_E_ARG;
  if (res_k) *res_k = h->mon_res;
  if (trace_k) { trace_k[0] = h->mon_trace.x; trace_k[1] = h->mon_trace.y; }
  if (ncand) *ncand = h->mon_ncand;
  if (count) *count = h->mon_count;
  if (mu)
    for (int64_t i = 0; i < h->m0; ++i) {
      const bool have = i < (int64_t)h->mon_mu.size();
      mu[2 * i] = have ? h->mon_mu[i].x : 0.0;
      mu[2 * i + 1] = have ? h->mon_mu[i].y : 0.0;
    }
  return FEAST_OK;
}

int feast_estimate_count_bi(feast_handle h, const void* A, int64_t lda, const void* B, int64_t ldb, const void* U,
                            int64_t ldu, const void* V, int64_t ldv, void* Q, int64_t ldq, void* QL, int64_t ldql,
                            double* mu, int32_t* count) {
  int e = check_args_common(h, A, lda, B, ldb);
  if (e) return e;
  if (h->mode != FEAST_BI) return fail(h, FEAST_E_STATE, "the bi count estimate needs a FEAST_BI handle%s");
  if (!U || !V || !Q || !QL || ldu < h->n || ldv < h->n || ldq < h->n || ldql < h->n)
    return fail(h, FEAST_E_ARG, "U/V/Q/QL null or ld < n%s");
  if (h->world > 1 && h->partial) return fail(h, FEAST_E_STATE, "the count estimate needs the full node sum%s");
  Join j_(h);
  if ((e = ensure_iter_mem(h))) return e;
  const int64_t n = h->n, m = h->m0, ld = h->ldc;
  const double2 one = make_double2(1, 0), zero = make_double2(0, 0);
  // Bi-FEAST steps 4-5: U^ = rho U, V^ = left projector of V (node sums over the ranks inside)
  int pst = project_impl(h, (const double2*)A, lda, (const double2*)B, ldb, (const double2*)U, ldu,
                               (const double2*)V, ldv, (double2*)Q, ldq, (double2*)QL, ldql);
  if (pst < 0) return pst;
  if (h->async && (pst = judge_stats(h)) < 0) return pst;   // these calls read their results now
  // V^^H B U^ (m0 x m0; B U^ on the rows this rank owns when sharded: partials all-reduced)
  const bool shard = h->world > 1 && h->ar != nullptr;
  const int64_t r0 = shard ? h->rank * n / h->world : 0, r1 = shard ? (h->rank + 1) * n / h->world : n, nr = r1 - r0;
  const double2* BU = (const double2*)Q + r0;
  int64_t ldbu = ldq;
  if (!h->b_id) {
    gemm_gen(h, nr, m, n, false, (const double2*)B + r0, ldb, (const double2*)Q, ldq, h->BQ + r0, ld, one, zero);
    BU = h->BQ + r0;
    ldbu = ld;
  }
  gemm_gen(h, m, m, nr, true, (const double2*)QL + r0, ldql, BU, ldbu, h->it.Z, m, one, zero);
  if (shard && h->ar(h->it.Z, 2 * m * m, h->stream, h->ar_user)) return fail(h, FEAST_E_COMM, "all-reduce failed%s");
  if ((e = bhat_count(h, h->it.Z))) return e;
  if (count) *count = h->mon_count;
  if (mu)
    for (int64_t i = 0; i < m; ++i) { mu[2 * i] = h->mon_mu[i].x; mu[2 * i + 1] = h->mon_mu[i].y; }
  return pst;
}

int feast_filter_gap(feast_handle h, int64_t nl, const double* lam, int64_t p, double* abs_sorted, int32_t* order,
                     int32_t* m_inside, int32_t* m_prime, double* eps, double* log10_gap) {
  if (!h || nl < 1 || !lam || p < 0) return FEAST_E_ARG;
  // gamma_j = rho(lambda_j) (eq. quadrature_for_pi), numbered |gamma_1| >= ... >= |gamma_n| (
  // stable in the input order on ties); m, m' and eps = |gamma_{p+1} / gamma_{m'}|
  std::vector<double> rr(2 * nl);
  feast_filter(h, nl, lam, rr.data());
  std::vector<double> a(nl);
  for (int64_t j = 0; j < nl; ++j) a[j] = std::hypot(rr[2 * j], rr[2 * j + 1]);
  std::vector<int32_t> ord(nl);
  for (int64_t j = 0; j < nl; ++j) ord[j] = (int32_t)j;
  std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return a[x] > a[y]; });
  int64_t m = 0, last = 0;
  for (int64_t pos = 0; pos < nl; ++pos)
    if (inside_contour(h, lam[2 * ord[pos]], lam[2 * ord[pos] + 1])) { ++m; last = pos + 1; }
  int64_t mp = last;   // smallest l >= last with a strict gap |gamma_{l+1}| < |gamma_l| (a tie: reading R22)
  while (mp < nl && mp > 0 && !(a[ord[mp]] < (1.0 - 1e-12) * a[ord[mp - 1]])) ++mp;
  const double nan = std::nan("");
  if (abs_sorted)
    for (int64_t j = 0; j < nl; ++j) abs_sorted[j] = a[ord[j]];
  if (order) std::memcpy(order, ord.data(), nl * 4);
  if (m_inside) *m_inside = (int32_t)m;
  if (m_prime) *m_prime = (int32_t)mp;
  if (eps) *eps = (p < nl && mp >= 1) ? a[ord[p]] / a[ord[mp - 1]] : nan;
  if (log10_gap) *log10_gap = (p < nl && m >= 1) ? std::log10(a[ord[p]] / a[ord[m - 1]]) : nan;
  return FEAST_OK;
}

int feast_set_async(feast_handle h, int32_t enable) {
  if (!h) return FEAST_E_ARG;
  h->async = enable != 0;
  return FEAST_OK;
}

int feast_sync(feast_handle h) {
  if (!h) return FEAST_E_ARG;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return judge_stats(h);
}

int feast_node_stats(feast_handle h, double* min_rel_pivot, int32_t* worst_node) {
  if (!h) return FEAST_E_ARG;
  if (h->pending) judge_stats(h);
  if (min_rel_pivot)
    for (int j = 0; j < h->q; ++j) min_rel_pivot[j] = j < (int)h->minrel.size() ? h->minrel[j] : -1.0;
  if (worst_node) *worst_node = h->worst;
  return FEAST_OK;
}

int64_t feast_last_launch_count(feast_handle h) { return h ? h->launches : 0; }

int feast_factor_cache(feast_handle h, int32_t enable) {
  if (!h) return FEAST_E_ARG;
  if (enable && h->real) return fail(h, FEAST_E_STATE, "factor cache is not combined with real-pencil mode%s");
  graph_reset(h);
  h->cache_on = enable != 0;
  h->cache_valid = false;
  h->cache_A = h->cache_B = nullptr;
  if (h->cache_on && h->batch < h->j1 - h->j0)
    return fail(h, FEAST_E_NOMEM, "factor cache needs max_batch >= owned nodes (all factors resident)%s");
  return FEAST_OK;
}

int feast_set_contour(feast_handle h, int32_t nseg, const int32_t* kind, const double* params, int32_t k_per_segment,
                      int32_t rule) {
  if (!h) return FEAST_E_ARG;
  if (h->ws) return fail(h, FEAST_E_STATE, "feast_set_contour must precede feast_workspace_bytes/bind%s");
  if (nseg < 1 || !kind || !params || k_per_segment < 1 || k_per_segment > 2048 ||
      (rule != FEAST_RULE_TRAPEZOID && rule != FEAST_RULE_GAUSS_LEGENDRE))
    return fail(h, FEAST_E_ARG, "feast_set_contour: bad segment count, rule or nodes per segment%s");
  std::vector<feast_ctx::Seg> segs(nseg);
  for (int s = 0; s < nseg; ++s) {
    if (kind[s] != 0 && kind[s] != 1) return fail(h, FEAST_E_ARG, "segment kind must be 0 (line) or 1 (arc)%s");
    segs[s].kind = kind[s];
    for (int i = 0; i < 5; ++i) segs[s].p[i] = params[5 * s + i];
    if (kind[s] == 1 && !(segs[s].p[2] > 0)) return fail(h, FEAST_E_ARG, "arc radius must be > 0%s");
  }
  // closure and orientation (counter-clockwise: positive signed area of the polyline)
  auto ends = [](const feast_ctx::Seg& g, double t) { double2 a, b; seg_phi(g, t, a, b); return a; };
  double diam = 0.0, area = 0.0;
  for (int s = 0; s < nseg; ++s) {
    const double2 a = ends(segs[s], -1.0), b = ends(segs[(s + 1) % nseg], -1.0);
    diam = std::max(diam, std::hypot(a.x - b.x, a.y - b.y));
  }
  for (int s = 0; s < nseg; ++s) {
    const double2 e = ends(segs[s], 1.0), b = ends(segs[(s + 1) % nseg], -1.0);
    if (std::hypot(e.x - b.x, e.y - b.y) > 1e-10 * std::max(diam, 1e-300))
      return fail(h, FEAST_E_ARG, "contour segments do not close (end of segment s != start of s+1)%s");
    for (int i = 0; i < 64; ++i) {
      const double2 p0 = ends(segs[s], -1.0 + 2.0 * i / 64), p1 = ends(segs[s], -1.0 + 2.0 * (i + 1) / 64);
      area += p0.x * p1.y - p1.x * p0.y;
    }
  }
  if (!(area > 0)) return fail(h, FEAST_E_ARG, "contour must be counter-clockwise%s");
  const auto old_segs = h->segs;
  const int old_k = h->seg_k, old_rule = h->seg_rule;
  h->segs = segs; h->seg_k = k_per_segment; h->seg_rule = rule;
  if (make_segment_nodes(h) != 0 || h->q % h->world != 0 || setup_units(h) != 0) {
    h->segs = old_segs; h->seg_k = old_k; h->seg_rule = old_rule;
    if (h->segs.empty()) make_nodes(h); else make_segment_nodes(h);
    setup_units(h);
    return fail(h, FEAST_E_ARG, "contour: nodes do not divide over the ranks (or do not pair in real mode)%s");
  }
  // c_re, c_im: the centroid of the polyline (used only by diagnostics); r: half the diameter
  double cx = 0, cy = 0;
  for (const auto& p : h->poly) { cx += p.x; cy += p.y; }
  h->c_re = cx / h->poly.size(); h->c_im = cy / h->poly.size(); h->r = 0.5 * diam;
  return FEAST_OK;
}

int feast_filter(feast_handle h, int64_t npts, const double* mu, double* rho) {
  if (!h || npts < 0 || (npts > 0 && (!mu || !rho))) return FEAST_E_ARG;
  for (int64_t i = 0; i < npts; ++i) {
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < h->q; ++j) {   // w_j / (z_j - mu)  (eq. quadrature_for_pi)
      const double dr = h->z[j].x - mu[2 * i], di = h->z[j].y - mu[2 * i + 1];
      const double d2 = dr * dr + di * di;
      sr += (h->w[j].x * dr + h->w[j].y * di) / d2;
      si += (h->w[j].y * dr - h->w[j].x * di) / d2;
    }
    rho[2 * i] = sr;
    rho[2 * i + 1] = si;
  }
  return FEAST_OK;
}

int feast_set_complex_symmetric(feast_handle h, int32_t enable) {
  if (!h) return FEAST_E_ARG;
  if (h->ws) return fail(h, FEAST_E_STATE, "feast_set_complex_symmetric must precede feast_workspace_bytes/bind%s");
  if (enable && h->real) return fail(h, FEAST_E_STATE, "complex-symmetric and real-pencil modes are exclusive%s");
  h->csym = enable != 0;
  setup_units(h);
  return FEAST_OK;
}

int feast_set_real_pencil(feast_handle h, int32_t enable) {
  if (!h) return FEAST_E_ARG;
  if (h->ws) return fail(h, FEAST_E_STATE, "feast_set_real_pencil must precede feast_workspace_bytes/bind%s");
  if (enable && h->cache_on) return fail(h, FEAST_E_STATE, "factor cache is not combined with real-pencil mode%s");
  if (enable && h->segs.empty() && h->c_im != 0.0)
    return fail(h, FEAST_E_ARG, "real-pencil mode needs a contour centre on the real axis%s");
  if (enable && h->csym) return fail(h, FEAST_E_STATE, "complex-symmetric and real-pencil modes are exclusive%s");
  h->real = enable != 0;
  if (setup_units(h) != 0) {
    h->real = false;
    setup_units(h);
    return fail(h, FEAST_E_ARG, "real-pencil mode: poles do not pair up or units %% world != 0%s");
  }
  return FEAST_OK;
}

int feast_profile(feast_handle h, int32_t enable) {
  if (!h) return FEAST_E_ARG;
  feast::Prof& p = feast::prof();
  p.on = enable != 0;
  h->prof_serial = enable == 2;
  p.recs.clear();
  p.used = 0;
  if (p.on) p.ensure_counters();
  if (p.counters && p.counters_used) cudaMemset(p.counters, 0, p.counters_used * sizeof(unsigned long long));
  p.counters_used = 0;
  CUDA_TRY(h, cudaDeviceSynchronize());
  return FEAST_OK;
}

int feast_profile_summary(feast_handle h, int32_t kclass, int64_t* launches, double* ms, double* flops,
                          double* bytes) {
  if (!h || kclass < 0 || kclass >= feast::K_NCLASS) return FEAST_E_ARG;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaDeviceSynchronize());
  int64_t c = 0;
  double t = 0, f = 0, b = 0;
  const auto& P = feast::prof();
  std::vector<unsigned long long> cnt;
  if (P.counters && P.counters_used > 0) {
    cnt.resize(P.counters_used);
    CUDA_TRY(h, cudaMemcpy(cnt.data(), P.counters, cnt.size() * 8, cudaMemcpyDeviceToHost));
  }
  for (const auto& r : P.recs) {
    if (r.cls != kclass) continue;
    float e = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&e, r.a, r.b));
    ++c; t += e; f += r.flops;
    b += (r.dev_bytes >= 0 && r.dev_bytes < (int64_t)cnt.size()) ? (double)cnt[r.dev_bytes] : r.bytes;
  }
  if (launches) *launches = c;
  if (ms) *ms = t;
  if (flops) *flops = f;
  if (bytes) *bytes = b;
  return FEAST_OK;
}

int feast_profile_records(feast_handle h, int64_t max_records, int32_t* kclass, int32_t* stream, double* t0_ms,
                          double* t1_ms, double* flops, int64_t* count) {
  if (!h || max_records < 0) return FEAST_E_ARG;
  CUDA_TRY(h, cudaDeviceSynchronize());
  const auto& recs = feast::prof().recs;
  const int64_t nrec = (int64_t)recs.size();
  if (count) *count = nrec;
  for (int64_t i = 0; i < nrec && i < max_records; ++i) {
    const auto& r = recs[(size_t)i];
    float e0 = 0.f, e1 = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&e0, recs[0].a, r.a));
    CUDA_TRY(h, cudaEventElapsedTime(&e1, recs[0].a, r.b));
    if (kclass) kclass[i] = r.cls;
    if (stream) {
      int tag = r.s == h->stream ? 0 : (r.s == h->side ? 1 : -1);
      for (int g = 1; g < feast_ctx::GMAX && tag < 0; ++g)
        if (r.s == h->gs[g]) tag = 2 * g; else if (r.s == h->gside[g]) tag = 2 * g + 1;
      stream[i] = tag;
    }
    if (t0_ms) t0_ms[i] = e0;
    if (t1_ms) t1_ms[i] = e1;
    if (flops) flops[i] = r.flops;
  }
  return FEAST_OK;
}

const char* feast_last_error(feast_handle h) { return h ? h->err.c_str() : "null handle"; }

void feast_destroy(feast_handle h) {
  if (!h) return;
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->ev_a) cudaEventDestroy(h->ev_a);
  if (h->ev_p) cudaEventDestroy(h->ev_p);
  if (h->side) cudaStreamDestroy(h->side);
  for (int g = 1; g < feast_ctx::GMAX; ++g) {
    if (h->gs[g]) cudaStreamDestroy(h->gs[g]);
    if (h->gside[g]) cudaStreamDestroy(h->gside[g]);
    if (h->gev_a[g]) cudaEventDestroy(h->gev_a[g]);
    if (h->gev_p[g]) cudaEventDestroy(h->gev_p[g]);
    if (h->gev_done[g]) cudaEventDestroy(h->gev_done[g]);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->s_rhs) cudaStreamDestroy(h->s_rhs);
  if (h->ev_a1) cudaEventDestroy(h->ev_a1);
  if (h->ev_rhs) cudaEventDestroy(h->ev_rhs);
  for (int g = 0; g < feast_ctx::GMAX; ++g) {
    if (h->gev_first[g]) cudaEventDestroy(h->gev_first[g]);
    if (h->gl[g]) cudaStreamDestroy(h->gl[g]);
    if (h->gev_l[g]) cudaEventDestroy(h->gev_l[g]);
    if (h->gev_lj[g]) cudaEventDestroy(h->gev_lj[g]);
    if (h->gx[g]) cudaStreamDestroy(h->gx[g]);
    if (h->gev_t[g]) cudaEventDestroy(h->gev_t[g]);
    if (h->gev_x[g]) cudaEventDestroy(h->gev_x[g]);
  }
  if (h->own_stream) {
    cudaStreamSynchronize(h->stream);
    cudaStreamDestroy(h->stream);
    cudaEventDestroy(h->ev_in);
    cudaEventDestroy(h->ev_out);
  }
  if (h->itmem) cudaFree(h->itmem);
  if (h->h_stats) cudaFreeHost(h->h_stats);
  if (h->h_info) cudaFreeHost(h->h_info);
  if (h->ev_stats) cudaEventDestroy(h->ev_stats);
  if (h->solp) cusolverDnDestroyParams(h->solp);
  if (h->sol) cusolverDnDestroy(h->sol);
  delete h;
}

}  // extern "C"
