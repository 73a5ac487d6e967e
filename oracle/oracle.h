/*
 * oracle/oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of Tall-Skinny QR (TSQR)
 * from arXiv 0808.2664 ("Communication-optimal parallel and sequential QR and LU
 * factorizations", Demmel, Grigori, Hoemmen, Langou).  Citations "P:n" are lines
 * of /root/reference/PAPER.md (LaTeX source), with the section / equation /
 * algorithm they fall in.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.  It shares NO code, headers, tables or helpers with
 * the CUDA product path (paper_0808_2664_b200/csrc, include/tsqr.h).
 *
 * Conventions:
 *   - all matrices fp64, column-major, element (i,j) at a[i + j*ld];
 *   - inner products and norms accumulate in long double (x87 80-bit);
 *   - Householder reflectors follow LAPACK dlarfg: H = I - tau v v^T, v(0)=1,
 *     beta = -sign(alpha)*||x||, sign(0)=+1 (reading R1; the paper only fixes
 *     "normalized so that v(1)=1", P:1967-1968 [Alg. QR:qnxn]);
 *   - T factors follow LAPACK dlarft: H_0 H_1 ... H_{k-1} = I - Y T Y^T with
 *     T(j,j)=tau_j, i.e. the NEGATIVE of Alg. YT:scaled's T (
 *     reading R3).
 * Parity status of each function is stated beside it ("pinned by" = the test
 * in tests/test_oracle_pins.py that ties it to something other than itself).
 */
#ifndef TSQR_ORACLE_H
#define TSQR_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* House(w) of Alg. QR:qnxn line 4.  On entry x[0..len-1] = w.
 * On exit x[1..len-1] = v(1..len-1) (v(0)=1 implicit), x[0] untouched;
 * *tau, *beta set so that (I - tau v v^T) w = beta e_0.
 * sigma^2 = sum_{i>=1} x_i^2 == 0  =>  tau = 0, beta = x[0] (reading R2).
 * Pinned by: worked example x=(3,4) -> v=(1,0.5), tau=1.6, beta=-5; special
 * cases x=(c,0,0), x=0; H w = beta e_0 on random w. */
void orc_house(int64_t len, double *x, double *tau, double *beta);

/* Unblocked Householder QR (= LAPACK DGEQR2), the "sequential Householder QR"
 * of Alg. TSQR:par line 1 and the leaf QR of Eq. 1.
 * A (m x n, m >= n) is overwritten: upper triangle = R, strictly lower = v's;
 * tau[n] receives the scaling factors.
 * Pinned by: long-double MGS on tiny inputs, LAPACK (torch.linalg.qr), A=I(:,1:n),
 * the invariants ||A-QR||, ||Q^TQ-I||, R^TR = A^TA. */
void orc_hqr(int64_t m, int64_t n, double *A, int64_t lda, double *tau);

/* Flat-tree ("sequential") TSQR of one tile over chunks of c rows (
 * [TR] Alg. sequential TSQR P:1725-1753): chunk k (rows r0 = kc .. r0+h-1) is
 * merged into the running R by qr([R; A_k]); R is upper trapezoidal and its
 * row j is the tile's row j, so reflector j of chunk k acts on
 *   rows {j} u [r0, r0+h)   if j < r0        (pivot = R row j, tail = chunk),
 *   rows [j, r0+h)          if r0 <= j < r0+h (pivot inside the chunk),
 * and is absent otherwise (tau = 0).  c <= 0 or c >= rows: orc_hqr exactly.
 * On exit R is in the upper triangle of the first n rows, every reflector's
 * tail in place below the diagonal, tau[k*n + j] for chunk k.
 * Pinned by: c = 0 equals orc_hqr bit for bit; R vs LAPACK / flat QR
 * (uniqueness modulo signs); the invariants of the explicit Q
 * built from the stored reflectors; the executed row sets (chain_rows) vs
 * the sparsity of [R; A_k]. */
void orc_chain_qr(int64_t rows, int64_t n, double *A, int64_t lda, int64_t c, double *tau);

/* Structured QR of two stacked n x n upper triangles [Ra; Rb], Alg. QR:qnxn with
 * q = 2 (sparsity eq. fact_2rs).  Reflector j acts on
 * the index set I_j = {row j of Ra} u {rows 0..j of Rb}.
 * On exit Ra's upper triangle = R, Rb's upper triangle (incl. diagonal) = Y1
 * (the nonunit part of the vectors [e_j; y_j]), tau[n].  Entries of Ra/Rb
 * strictly below the diagonal are neither read nor written.
 * *flops (may be NULL) receives the executed flop count (2 per mul-add pair,
 * 1 per other arithmetic op) for the (2/3)n^3 pin.
 * Pinned by: dense orc_hqr of the explicitly stacked 2n x n matrix; Y1 strictly
 * lower exactly zero; R_a=I,R_b=0 -> R=I,tau=0; flop window. */
void orc_combine(int64_t n, double *Ra, int64_t lda, double *Rb, int64_t ldb,
                 double *tau, double *flops);

/* LAPACK-sign T factor (dlarft, forward, columnwise) of k reflectors whose
 * vectors are the columns of the unit lower trapezoidal rows x k matrix Y
 * (strictly-lower part read from Y, unit diagonal implicit, upper ignored):
 * H_0 ... H_{k-1} = I - Y T Y^T.  Alg. YT:scaled with T := -T'
 * (reading R3).  T is k x k upper triangular (lower part set to 0).
 * Pinned by: I - Y T Y^T equals the explicit product of the reflectors. */
void orc_build_t(int64_t rows, int64_t k, const double *Y, int64_t ldy,
                 const double *tau, double *T, int64_t ldt);

/* Same for a tree node, whose vectors are [e_j; Y1(:,j)] with Y1 n x n upper
 * triangular (eq. fact_2rs; T for the node P:2225-2230). */
void orc_build_t_node(int64_t n, const double *Y1, int64_t ldy, const double *tau,
                      double *T, int64_t ldt);

/* ---------------- the reduction-tree plan ----------
 * Three nested levels, all binary with the paper's pairing (Alg. TSQR:par,
 * P:1687-1696; reading R5): tiles inside a row block, row blocks inside a
 * rank, ranks (G a power of two; the cross-rank butterfly of Alg. TSQR:par is
 * a binary tree over rank roots, every rank holding a replica).
 * Row blocks: b rows each from row 0; remainder r = m mod b becomes its own
 * block if r >= n, else is merged into the last block (reading R6).
 * Ranks: contiguous runs of whole blocks, the first (nblocks mod G) ranks get
 * one extra block.
 * Tiles: a block of h rows is split into t = min(ceil(h/s), floor(h/n)) (at
 * least 1) tiles of near-equal EVEN height: the floor(h/2) row pairs split
 * near-equally (the first (floor(h/2) mod t) tiles one pair taller), the last
 * tile taking the rest; when that leaves a tile shorter than n, plain
 * near-equal heights (the first (h mod t) tiles one row taller); s = 0 means
 * one tile per block (the paper's plan, tiles = row blocks).
 * Nodes are listed in execution order: level by level inside every block,
 * then level by level over the blocks of each rank, then the rank levels.
 * A node is the pair (a, b) of the leftmost tiles of its left and right
 * subtrees; its level counts from 1 within its tree stage.
 * Returns 0 on success, -1 on an invalid shape (m < n, a tile < n rows, a rank
 * with no block, G not a power of two). */
int orc_plan_count(int64_t m, int64_t n, int64_t b, int64_t s, int64_t G,
                   int64_t *ntiles, int64_t *nnodes);
int orc_plan_fill(int64_t m, int64_t n, int64_t b, int64_t s, int64_t G,
                  int64_t *tile_row0, int64_t *tile_rows, int64_t *tile_rank,
                  int64_t *node_a, int64_t *node_b, int64_t *node_stage,
                  int64_t *node_level);

/* TSQR factorization over an explicit plan (Eqs. 1-4).
 * Every tile (leaf) is factored by orc_chain_qr with chunk rows c (c = 0: the
 * paper's plain leaf QR); A (m x n, global) is overwritten tile by tile;
 * tau_tile[nchunks*n] (chunks of tile 0 first, ceil(rows/c) chunks per tile); node factors Y1[nnodes*n*n] (node k at Y1 + k*n*n,
 * column-major n x n, upper triangle) and tau_node[nnodes*n]; R (n x n, ldr)
 * receives the final R (zeros below the diagonal).
 * Pinned by: flat orc_hqr R (uniqueness modulo signs), tree
 * independence, R^TR = A^TA (Cor. 1). */
void orc_tsqr_factor(int64_t m, int64_t n, double *A, int64_t lda, int64_t c,
                     int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                     int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                     double *tau_tile, double *Y1, double *tau_node,
                     double *R, int64_t ldr);

/* The same factorization with the leaf QRs (Eq. 1, independent per leaf)
 * spread over nthreads host threads (contiguous runs of tiles); the nodes run
 * in plan order on the calling thread.  Bitwise equal to orc_tsqr_factor (each
 * tile's arithmetic is unchanged; only which thread runs it differs).  Y1 may
 * be NULL.  The only parallelism in the oracle ("parallel over
 * leaves"), used to time it on all host cores and to check full-size configs. */
void orc_tsqr_factor_mt(int64_t m, int64_t n, double *A, int64_t lda, int64_t c,
                        int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                        int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                        double *tau_tile, double *Y1, double *tau_node,
                        double *R, int64_t ldr, int64_t nthreads);

/* C <- Q^T C in "tree order" (leaves first, then nodes in factor order;
 * reading R4): tile stage [TR] P:1915-1938, node stage eq. localQTupdate
 * applied reflector by reflector.  Global rows 0..n-1 end
 * holding Q_thin^T C.  Pinned by: Q^T A = [R; 0]; ||Q^T C|| = ||C||;
 * apply_q(apply_qt(C)) = C; thin part = (formed Q)^T C. */
void orc_tsqr_apply_qt(int64_t m, int64_t n, const double *A, int64_t lda, int64_t c,
                       int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                       int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                       const double *tau_tile, const double *Y1, const double *tau_node,
                       double *C, int64_t ldc, int64_t k);

/* C <- Q C, the exact reverse traversal of orc_tsqr_apply_qt. */
void orc_tsqr_apply_q(int64_t m, int64_t n, const double *A, int64_t lda, int64_t c,
                      int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                      int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                      const double *tau_tile, const double *Y1, const double *tau_node,
                      double *C, int64_t ldc, int64_t k);

/* Explicit thin Q (m x n) = Q [I_n; 0]. */
void orc_tsqr_form_q(int64_t m, int64_t n, const double *A, int64_t lda, int64_t c,
                     int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                     int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                     const double *tau_tile, const double *Y1, const double *tau_node,
                     double *Q, int64_t ldq);

/* Modified Gram-Schmidt in long double (test tool required by north_star;
 * P:1205-1207 names MGS).  Q (m x n), R (n x n upper, positive diagonal). */
void orc_mgs_ld(int64_t m, int64_t n, const double *A, int64_t lda,
                double *Q, int64_t ldq, double *R, int64_t ldr);

/* CholeskyQR, Alg. CholeskyQR ([TR] P:1410-1419) -- the comparison method of
 * SURVEY 8(f) row 4, NOT part of TSQR:
 *   line 1  W := A^T A        (each entry an inner product, long double sum, then
 *                              rounded to double: the fp64 W of the algorithm)
 *   line 2  W = L L^T         (Cholesky, row by row; R := L^T, positive diagonal)
 *   line 3  Q := A L^{-T}     (Q = A R^{-1}: forward substitution q_i^T R = a_i^T
 *                              for every row i)
 * Returns 0, or j+1 when the leading minor of order j+1 of the computed W is not
 * positive (R, Q then incomplete).  Q may be NULL (R only).
 * Pinned by: a hand-worked 2x2 example (golden cholqr_2x2.txt); R vs LAPACK's
 * Householder R (uniqueness modulo signs); Q vs an independent
 * triangular solve; orthonormal A -> R = I, Q = A; a zero column -> breakdown at
 * that column; the loss of orthogonality growing as kappa^2. */
int orc_cholqr(int64_t m, int64_t n, const double *A, int64_t lda, double *R, int64_t ldr,
               double *Q, int64_t ldq);

#ifdef __cplusplus
}
#endif
#endif
