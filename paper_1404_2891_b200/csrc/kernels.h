// kernels.h — internal launcher interfaces of the B200 FEAST library (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace feast {

// ---------------------------------------------------------------- ZGEMM (DMMA)
enum { ZG_SUB = 0,   // C -= op(A) B
       ZG_GEN = 1 }; // C = alpha op(A) B + beta C
struct ZgemmArgs {
  int64_t M, N, K;
  const double2* A; int64_t lda, sA;  // op(A) is M x K; A is M x K (N) or K x M (conj-transpose)
  const double2* B; int64_t ldb, sB;  // K x N
  double2* C; int64_t ldc, sC;        // M x N
  double2 alpha, beta;
  int batch;                          // batch index z adds z*sA, z*sB, z*sC
  int inplace = 0;                    // 1: C aliases B (requires M <= 64: one CTA row of tiles)
  int swz = 0;                        // > 1: tile rasterisation in groups of swz tile rows (set by the launcher)
};
void zgemm_launch(const ZgemmArgs& p, bool conjA, int mode, cudaStream_t s);
// tile-variant selection (tools/zgemm_lab): 0 = the launcher's heuristic
void zgemm_launch_variant(const ZgemmArgs& p, bool conjA, int mode, int variant, cudaStream_t s);

// ---------------------------------------------------------------- block triangular solve (DMMA)
// Y <- op(T)^-1 Y for an R x R (R <= 256) triangular block T made of 64 x 64 blocks whose diagonal
// blocks' inverses are precomputed (trtri): one CTA per 32-column tile of Y keeps the R x 32 tile
// in shared memory and runs the whole block solve (diagonal-inverse products and the in-block
// updates) on DMMA, streaming the 64 x 64 operand blocks from L2.
//   fwd   : blocks in increasing order (op(T) lower: L, or U^H), else decreasing (U, or L^H)
//   conj  : op = conjugate transpose (the block (rb, kb) of op(T) is T[kb, rb]^H)
//   T0    : T's top-left element (column-major, ld ldt), batch stride sT
//   Inv0  : the first diagonal block's inverse (64 x 64, ld 64), the next at + inv_step, batch sInv
//   Y0    : Y's first row (ld ldy), N columns, batch stride sY; R rows (ragged last 64-block ok)
struct BtrsmArgs {
  const double2* T0; int64_t ldt, sT;
  const double2* Inv0; int64_t inv_step, sInv;
  double2* Y0; int64_t ldy, sY;
  int64_t R, N;
  int batch;
};
void btrsm_launch(const BtrsmArgs& p, bool fwd, bool conj, cudaStream_t s);

// ---------------------------------------------------------------- LU pieces
// Batched matrices: matrix b at base + b*stride (complex elements), column-major, ld.
struct Batched {
  double2* p;
  int64_t ld, stride;
};

// C_b = z_b B - A   (B == nullptr: B = I).  z: device array of batch poles.  Columns [c0, c1)
// only (c1 < 0: to n).
void shift_launch(Batched C, const double2* A, int64_t lda, const double2* B, int64_t ldb,
                  const double2* z, int64_t n, int batch, cudaStream_t s, int64_t c0 = 0, int64_t c1 = -1);

// Panel factorisation with partial pivoting of columns [k, k+w) (rows k..n-1) of each matrix.
// ipiv: batch x n int32 (absolute row index swapped with row k+i), stats: batch x 2 doubles
// (running min / max |u_ii|), info: batch int32 (first exact zero pivot, 1-based; 0 none).
struct PanelCfg { int cluster; int W; int S; };
PanelCfg panel_config(int64_t n);
void panel_launch(Batched C, int64_t n, int64_t k, int w, int32_t* ipiv, double* stats, int32_t* info,
                  int batch, const PanelCfg& cfg, cudaStream_t s);

// Row swaps ipiv[k..k+cnt) applied to columns [c0, c1) (variant: LASWP_COALESCED = slot-traced
// gather/scatter with coalesced block rows (default), LASWP_CHAIN = one thread per column running
// the swap chain, LASWP_PERM = permutation composed per CTA with a row table).
enum { LASWP_COALESCED = 0, LASWP_CHAIN = 1, LASWP_PERM = 2 };
void laswp_launch(Batched C, int64_t n, int64_t k, int cnt, const int32_t* ipiv, int64_t c0, int64_t c1, int batch,
                  cudaStream_t s, int variant = LASWP_COALESCED);
// Cluster panel with the panel resident in shared memory (rows never moved; see panel_smem.cu).
int tall_variant();
bool very_tall_panels();   // 1025..2048 rows per CTA on the cluster kernel (FEAST_VTALL)
bool panel_smem_fits(int64_t n, int w, int cs);
int panel_smem_max_clusters(int64_t L, int w, int cs);
// sc0 < sc1: the panel's row swaps are also applied to the columns [sc0, sc1) (fused; no laswp launch)
void panel_smem_launch(Batched C, int64_t n, int64_t k, int w, int32_t* ipiv, double* stats, int32_t* info, int batch,
                       int cs, cudaStream_t s,
                       bool one_row = false, int64_t sc0 = 0, int64_t sc1 = 0);

// Triangular solve op(T) X = X in place, T = nb x nb diagonal block (nb <= 64),
// X = nb x ncols.  lower_op: op(T) lower (forward); unit: unit diagonal; conjT: op = ^H.
void trsm_launch(Batched T, Batched X, int nb, int64_t ncols, bool lower_op, bool unit, bool conjT,
                 int batch, cudaStream_t s);

// Inverses of the 64x64 diagonal blocks kb0 .. kb0+nblocks-1 of every factored node:
// inv + b*inv_node_stride + (kb*2 + 0) * 4096 = L_kk^-1 (unit lower), (kb*2 + 1) * 4096 = U_kk^-1,
// each 64 x 64 column-major (ld 64), identity-padded for a partial last block.
// which: 0 = L only, 1 = U only, 2 = both.
void trtri_launch(Batched C, int64_t n, int64_t kb0, int64_t nblocks, double2* inv, int64_t inv_node_stride, int which,
                  int batch, cudaStream_t s);
void ipiv_identity_launch(int32_t* ipiv, int64_t n, int64_t k, int w, int batch, cudaStream_t s);
void stats_init_launch(double* stats, int32_t* info, int batch, cudaStream_t s);
// perm_b from ipiv_b (sequential swaps of rows 0..n-1); iperm (optional) = inverse permutation
void perm_launch(const int32_t* ipiv, int32_t* perm, int32_t* iperm, int64_t n, int batch, cudaStream_t s);
// gather: Y_b[i][c] = R[perm_b[i]][c]   (R shared by the batch: sR = 0 allowed)
void gather_rows_launch(Batched Y, const double2* R, int64_t ldr, int64_t sR, const int32_t* perm,
                        int64_t n, int64_t m, int batch, cudaStream_t s);
// scatter: Out_b[perm_b[i]][c] = Y_b[i][c]
void scatter_rows_launch(Batched Out, const double2* Y, int64_t ldy, int64_t sY, const int32_t* perm,
                         int64_t n, int64_t m, int batch, cudaStream_t s);
// copy R (shared) into every Y_b; BC_PAIR: and conj(R) into Y_b's columns [m, 2m); BC_CONJ: conj(R)
enum { BC_COPY = 0, BC_PAIR = 1, BC_CONJ = 2 };
void broadcast_copy_launch(Batched Y, const double2* R, int64_t ldr, int64_t n, int64_t m, int batch, int mode,
                           cudaStream_t s);
// flag |= 1 if M (n x n) has any nonzero imaginary part
void imag_check_launch(const double2* M, int64_t ld, int64_t n, int32_t* flag, cudaStream_t s);

// Q (+)= sum_b w_b Y_b[iperm_b[i]] (+ wp_b conj(Y_b[iperm_b[i], m + c]) when wp != null) with
// conj(w), conj(wp) if conjw; iperm null = identity; b increasing; accumulate=false overwrites Q;
// conj_out: Q = conj(conj(Q_old) + sum) (the left block of a complex-symmetric pencil).
void accum_launch(double2* Q, int64_t ldq, Batched Y, const double2* w, const double2* wp, const int32_t* iperm,
                  int64_t n, int64_t m, int batch, bool conjw, bool accumulate, cudaStream_t s, bool conj_out = false);
// C = alpha * sum_s P_s + beta C, P_s = M x N (ld M) partials at P + s*M*N
void splitk_reduce_launch(double2* C, int64_t ldc, const double2* P, int64_t M, int64_t N, int splits,
                          double2 alpha, double2 beta, cudaStream_t s);

// Column residual norms over n rows: out[c] = || AX[:,c] - lam_c BX[:,c] ||_2 and xn[c] = || X[:,c] ||_2
// (xn may be null); squared = true writes the squared norms (partial sums of a row-sharded block).
void resid_launch(const double2* AX, const double2* BX, const double2* X, int64_t ld, const double2* lam,
                  int64_t n, int64_t m, double* out, double* xn, cudaStream_t s, bool squared = false);
// || A ||_F^2 partial sums into out (one double, must be zeroed) — deterministic two-pass.
void frob2_launch(const double2* A, int64_t lda, int64_t n, double* partial, int nparts, cudaStream_t s);
// partial[b] = sum_{c = b mod nparts} sum_i conj(U[i][c]) Q[i][c]  (nparts blocks, host sums in order)
void cdot_launch(const double2* U, int64_t ldu, const double2* Q, int64_t ldq, int64_t n, int64_t m, double2* partial,
                 int nparts, cudaStream_t s);
// Zero the strictly lower triangle of an m x m matrix.
void tril_zero_launch(double2* M, int64_t ld, int64_t m, cudaStream_t s);
// Scale columns of X by 1/xn[c] and rows of W by same: X[:,c] /= xn[c], W[:,c] /= xn[c]
void colscale_launch(double2* X, int64_t ldx, int64_t n, double2* W, int64_t ldw, int64_t m,
                     const double* xn, cudaStream_t s);

}  // namespace feast
