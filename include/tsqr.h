/*
 * include/tsqr.h -- C-ABI of libtsqr.so, a B200-native (sm_100a) Tall-Skinny QR
 * (TSQR) after arXiv 0808.2664 (Demmel, Grigori, Hoemmen, Langou).
 * "P:n" = line n of the paper's LaTeX source, with its section /
 * equation / algorithm.  DESIGN.md states the plan rules and the readings R1-R13.
 *
 * Conventions for every call
 *   - Matrices are fp64, COLUMN-MAJOR: element (i,j) of X lives at X[i + j*ldx].
 *   - Pointers named "device" must be CUDA device (or managed) memory on the
 *     current device; "host" pointers are ordinary host memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Every device call is asynchronous and stream-ordered.
 *   - Arguments are validated on the host BEFORE anything is enqueued: a status
 *     other than TSQR_OK means nothing was enqueued and nothing was modified.
 *   - Asynchronous device faults surface as TSQR_ERR_CUDA from a later call or
 *     at the caller's own synchronisation.  No exception or abort crosses the ABI.
 *   - A tree handle must be used on one device by one host thread at a time.
 */
#ifndef TSQR_H
#define TSQR_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TSQR_OK = 0,
    TSQR_ERR_INVALID = 1,      /* null pointer, ld too small, k < 0, bad round / rank  */
    TSQR_ERR_SHAPE = 2,        /* m < n, a tile or row block with < n rows, no block   */
    TSQR_ERR_UNSUPPORTED = 3,  /* n > TSQR_MAX_N, tile_rows above the kernel capacity,
                                  nranks not a power of two                             */
    TSQR_ERR_ALLOC = 4,        /* device or host allocation failed                      */
    TSQR_ERR_CUDA = 5,         /* a CUDA runtime error (message: tsqr_last_error())     */
    TSQR_ERR_NCCL = 6          /* an NCCL error or a failed exchange of a butterfly
                                  round (message: tsqr_last_error())                    */
} tsqr_status_t;

#define TSQR_MAX_N 256         /* widest n the kernels support: n <= 64 on the
                                  register-resident chunk chains, 64 < n <= 256 on
                                  the wide engine (tiles of at most 2304 rows)   */

/* Plan options.
 *  block_rows: b, the paper's row-block height (A_i of Eq. 1); the
 *              row blocks of a rank are reduced by a binary tree (Eqs. 1-4).
 *  tile_rows:  s, the SM-resident tile height: each row block is split into
 *              ceil(h/s) near-equal tiles, the leaves of the tree, reduced by a
 *              binary sub-tree inside the block ("any tree").
 *              0 = library default for n (tsqr_plan_info reports it).
 *  nranks, rank: the row-sharded multi-GPU layout (Alg. TSQR:par);
 *              nranks = 1 for a single GPU.  A rank's slab must be the one
 *              tsqr_slab() assigns.
 *  flags:      bit 0 = synchronise and check after every launch (debug);
 *              bit 1 = record CUDA events around tsqr_factor's leaf and tree
 *              stages on its stream (read back with tsqr_tree_stage_ms);
 *              bit 2 = TSQR_FLAG_ROBUST: dlarfg's rescaling in every leaf and
 *              tree Householder step (reading R23 of DESIGN.md).  Without it the
 *              leaf kernels form sums of squares unscaled and are exact (to
 *              rounding, normwise) when the nonzero entries of A have magnitudes
 *              in [2^-400, 2^400] (about 1e-120 .. 1e+120); outside that range
 *              set the flag (it costs 3-8 % of the factor).  The cross-rank and
 *              q-ary combines always rescale. */
#define TSQR_FLAG_DEBUG_SYNC 1
#define TSQR_FLAG_STAGE_TIMING 2
#define TSQR_FLAG_ROBUST 4
typedef struct {
    int64_t block_rows;
    int64_t tile_rows;
    int32_t nranks;
    int32_t rank;
    int32_t flags;
    int32_t reserved;
} tsqr_opts_t;

typedef struct tsqr_tree_s *tsqr_tree_t;   /* opaque implicit Q (D5 of SURVEY §2.2) */

typedef struct {
    int64_t m_local, n, block_rows, tile_rows;
    int64_t ntiles;        /* leaves of the local tree                           */
    int64_t nnodes;        /* local combine nodes (= ntiles - 1)                 */
    int64_t nblocks;       /* row blocks of this rank                            */
    int64_t depth;         /* levels of the local tree (tile + block stages)     */
    int64_t cross_rounds;  /* log2(nranks): butterfly rounds (Table 1) */
    int64_t max_tile_rows, min_tile_rows;
    int64_t tile_capacity; /* tallest tile the kernels accept                     */
    int64_t chunk_rows;    /* c: every tile is factored as a flat chain ("sequential
                              TSQR") over chunks of c rows  */
    int64_t nchunks;       /* chunks of all tiles = rows of the tau export        */
} tsqr_plan_info_t;

/* ---------------------------------------------------------------- host-only
 * These never touch a GPU and may be called on a machine without one. */

const char *tsqr_status_string(tsqr_status_t s);
/* Text of the last CUDA error seen by this thread (or "" ). */
const char *tsqr_last_error(void);

/* Rank slab of the global m x n problem: contiguous
 * runs of whole row blocks, the first (nblocks mod nranks) ranks one block more.
 * Outputs the slab's first global row and its row count. */
tsqr_status_t tsqr_slab(int64_t m, int64_t n, int64_t block_rows, int32_t nranks,
                        int32_t rank, int64_t *row0, int64_t *m_local);

/* Plan summary for a rank's slab (m_local rows). */
tsqr_status_t tsqr_plan_info(int64_t m_local, int64_t n, const tsqr_opts_t *opts,
                             tsqr_plan_info_t *info);

/* Plan arrays (host buffers sized from tsqr_plan_info): per tile its first
 * local row and row count; per node in execution order the leftmost tiles
 * (a, b) of its two subtrees, its stage (0 = tiles in a block, 1 = blocks) and
 * level within the stage.  Used by the tests to compare with the oracle's plan. */
tsqr_status_t tsqr_plan_export(int64_t m_local, int64_t n, const tsqr_opts_t *opts,
                               int64_t *tile_row0, int64_t *tile_rows,
                               int64_t *node_a, int64_t *node_b,
                               int64_t *node_stage, int64_t *node_level);

/* Butterfly indexing of Alg. TSQR:par: in round
 * k = 1..log2(nranks), rank r pairs with r XOR 2^(k-1); the lower rank's R is
 * stacked on top ("by order of processor ids").
 * *is_lower = 1 if rank < partner.  *head_role: 1 if this rank is the leftmost
 * rank of the lower group (its C head keeps the R coordinates), 2 if it is the
 * leftmost of the upper group (its C head receives this node's complement),
 * 0 otherwise.  Words per message: n(n+1)/2 (factor, Cor. 2 P:5084-5091),
 * n*k (apply). */
tsqr_status_t tsqr_cross_partner(int32_t nranks, int32_t rank, int32_t round,
                                 int32_t *partner, int32_t *is_lower, int32_t *head_role);

/* ---------------------------------------------------------------- device */

/* Factor the rank's slab (Eqs. 1-4; Alg. TSQR:par line 1 P:1679).
 *  A (device, m_local x n, lda >= m_local): IN the slab, OUT the tile
 *    reflectors in place (strictly lower part of each tile) and
 *    the node factors Y1 of eq. fact_2rs (upper triangle of the head n x n
 *    block of each node's right subtree's first tile).  A is BORROWED by the
 *    tree until tsqr_tree_free: do not modify or free it before then.
 *  R (device, n x n, ldr >= n): OUT the R of the slab (nranks = 1: of A),
 *    upper triangular, exact zeros below the diagonal.  May be NULL.
 *  *tree: OUT a new handle; if *tree is non-NULL on entry and was built for the
 *    same (m_local, n, opts), its device workspace is reused (no allocation).
 * With nranks > 1 follow with tsqr_cross_factor for every round. */
tsqr_status_t tsqr_factor(int64_t m_local, int64_t n, double *A, int64_t lda,
                          double *R, int64_t ldr, const tsqr_opts_t *opts,
                          void *stream, tsqr_tree_t *tree);

/* Pack the tree's current R (upper triangle, column by column) into
 * packed[n(n+1)/2] (device): the message of one butterfly round (Cor. 2). */
tsqr_status_t tsqr_pack_r(tsqr_tree_t tree, double *packed, void *stream);

/* Butterfly round `round` (1..log2 nranks) of Alg. TSQR:par:
 * stack [R_lower; R_upper] from the tree's R and partner_packed (device,
 * n(n+1)/2, the partner's tsqr_pack_r output of the same round), factor it with
 * the structured combine (Alg. QR:qnxn), keep the node factor in the tree and
 * make the new R current.  R (device, may be NULL) receives it, zeros below. */
tsqr_status_t tsqr_cross_factor(tsqr_tree_t tree, int32_t round, const double *partner_packed,
                                double *R, int64_t ldr, void *stream);

/* All rounds of the butterfly at once from an all-gather of the leaf R's (one
 * collective instead of log2(nranks) exchanges; "any tree"
 * P:928-932): all_packed (device, nranks * n(n+1)/2) holds every rank's
 * tsqr_pack_r output, rank i at offset i*n(n+1)/2.  Each rank recomputes the
 * sibling groups' R's it needs (nranks - 1 - log2(nranks) extra combines) with
 * the same kernels, then runs its own rounds as tsqr_cross_factor would: the
 * tree ends in the same state and R is bitwise the butterfly's.  Only on a tree
 * with no round done yet.  R (device, may be NULL) receives the final R. */
tsqr_status_t tsqr_cross_factor_gathered(tsqr_tree_t tree, const double *all_packed, double *R,
                                         int64_t ldr, void *stream);

/* C <- Q^T C over the local tree ([TR] P:1915-1938; eq. localQTupdate
 * P:2193-2212).  C (device, m_local x k, ldc >= m_local) is overwritten in
 * "tree order": rows 0..n-1 of the slab hold the R coordinates (for nranks = 1,
 * Q_thin^T C); every other tile head holds its node's complement coordinates.
 * top (device, n x k, ldtop >= n, may be NULL) receives a copy of rows 0..n-1.
 * k = 0 is a no-op. */
tsqr_status_t tsqr_apply_qt(tsqr_tree_t tree, double *C, int64_t ldc, int64_t k,
                            double *top, int64_t ldtop, void *stream);

/* Butterfly round of apply Q^T: top (device, n x k, ldtop) holds this rank's
 * R coordinates, partner_top (device, n x k, ld = n) the partner's.  Both ranks
 * apply the round's node reflectors to [top_lower; top_upper]; top becomes the
 * new R coordinates; if head_role = 1 they are also written to C's rows
 * 0..n-1, if head_role = 2 the complement coordinates are. */
tsqr_status_t tsqr_cross_apply_qt(tsqr_tree_t tree, int32_t round, double *top, int64_t ldtop,
                                  const double *partner_top, double *C, int64_t ldc,
                                  int64_t k, void *stream);

/* C <- Q C, the inverse of tsqr_apply_qt (the reverse traversal: node stages
 * top-down with T in place of T^T, then the leaves' reflectors in reverse order;
 * [TR] P:1919-1925 with an arbitrary C in place of [I_n; 0]).
 * C (device, m_local x k, ldc >= m_local) is read in tree order -- rows 0..n-1
 * of the slab are the R coordinates, every other tile head its node's
 * complement coordinates -- so tsqr_apply_q(tsqr_apply_qt(C)) = C, and C =
 * [X; 0] gives Q[X; 0] (X = I: the explicit thin Q of tsqr_form_q).  With
 * butterfly rounds (nranks > 1) the rounds go first, top-down, through
 * tsqr_cross_apply_q; this call is then the local tree's part.
 * k = 0 is a no-op. */
tsqr_status_t tsqr_apply_q(tsqr_tree_t tree, double *C, int64_t ldc, int64_t k, void *stream);

/* Butterfly round of apply Q, rounds log2(nranks) .. 1 in that order, called by
 * the two group heads of the round only (head_role 1 or 2 of
 * tsqr_cross_partner; any other rank gets TSQR_ERR_INVALID and has nothing to
 * do).  top (device, n x k, ldtop) holds this rank's C head rows (the group's R
 * coordinates for head_role 1, the node's complement for head_role 2),
 * partner_top (device, n x k, ld = n) the partner's; both compute
 * Q_node [lower; upper] and keep their own half, written to top and to C's rows
 * 0..n-1 (C: device, m_local x k, ldc >= m_local). */
tsqr_status_t tsqr_cross_apply_q(tsqr_tree_t tree, int32_t round, double *top, int64_t ldtop,
                                 const double *partner_top, double *C, int64_t ldc,
                                 int64_t k, void *stream);

/* Explicit thin Q of the rank's slab: Q (device, m_local x n, ldq >= m_local) =
 * rows of Q [I_n; 0].  Needs no communication: the
 * cross-rank node factors are replicated on every rank. */
tsqr_status_t tsqr_form_q(tsqr_tree_t tree, double *Q, int64_t ldq, void *stream);

/* Sequential (out-of-HBM) TSQR: R of a HOST-resident m x n matrix streamed
 * through the GPU in row slabs -- a flat tree over the slabs ([TR] Alg.
 * sequential TSQR P:1725-1753; flat tree P:954-993; model Eq. 6).
 * Slab k (rows k*slab_rows .., a remainder of fewer than n rows joins the last
 * slab) is copied to the device (cudaMemcpy2DAsync on an internal copy stream,
 * overlapping the previous slab's factorization; page-locked A makes the copy
 * asynchronous), factored by tsqr_factor with opts (nranks must be 0 or 1), and
 * the running R absorbs it by the structured combine of [R; R_slab] (Alg.
 * QR:qnxn, q = 2).  A (host, lda >= m) is read only.  Y (host, ldy >= m, may be
 * NULL) receives every factored slab (its tiles' reflectors below their
 * diagonals, as tsqr_factor leaves A).  R (device, n x n, ldr >= n) receives R,
 * exact zeros below.  Device memory: two slabs plus O(n^2).  Synchronous: returns
 * after `stream` has completed the factorization. */
tsqr_status_t tsqr_factor_streamed(int64_t m, int64_t n, const double *A, int64_t lda, int64_t slab_rows,
                                   double *Y, int64_t ldy, double *R, int64_t ldr,
                                   const tsqr_opts_t *opts, void *stream);

/* The streamed factor with its implicit Q kept ([TR] Alg. sequential TSQR
 * P:1725-1753 writes every slab's Q factors to slow memory): as
 * tsqr_factor_streamed, Y (host, ldy >= m) REQUIRED -- it receives the reflectors
 * and is borrowed by the handle until tsqr_stream_tree_free -- and *out receives a
 * handle holding, in page-locked host memory, each slab tree's taus and cached T's
 * and each flat-tree node's factors (O(mn/c + S n^2) words).  Then, slab by slab
 * through the GPU (device memory: one slab of Y and of C plus O(n k)), with HOST
 * matrices:
 *   tsqr_streamed_apply_qt  C (m x k, ldc >= m) <- Q^T C in the streamed tree's
 *                           order (rows 0..n-1 = Q_thin^T C; top, host n x k,
 *                           ldtop >= n, may be NULL, receives it too);
 *   tsqr_streamed_apply_q   C <- Q C (C in that order): the exact inverse;
 *   tsqr_streamed_form_q    Q (m x n, ldq >= m) <- the explicit thin Q.
 * Synchronous (they return after `stream` has finished).  Page-locked C / Q make
 * the copies asynchronous DMA. */
typedef struct tsqr_stream_tree_s *tsqr_stream_tree_t;
tsqr_status_t tsqr_factor_streamed_q(int64_t m, int64_t n, const double *A, int64_t lda, int64_t slab_rows,
                                     double *Y, int64_t ldy, double *R, int64_t ldr, const tsqr_opts_t *opts,
                                     void *stream, tsqr_stream_tree_t *out);
tsqr_status_t tsqr_streamed_apply_qt(tsqr_stream_tree_t t, double *C, int64_t ldc, int64_t k, double *top,
                                     int64_t ldtop, void *stream);
tsqr_status_t tsqr_streamed_apply_q(tsqr_stream_tree_t t, double *C, int64_t ldc, int64_t k, void *stream);
tsqr_status_t tsqr_streamed_form_q(tsqr_stream_tree_t t, double *Q, int64_t ldq, void *stream);
tsqr_status_t tsqr_stream_tree_free(tsqr_stream_tree_t t);

/* q-ary structured combine, Alg. QR:qnxn ([TR] P:1957-1979): the QR of q stacked
 * n x n upper triangles [R_1; ...; R_q], reflector j acting on {row j of R_1} U
 * {rows 0..j of R_2..R_q} ((2/3)(q-1)n^3 flops; q = 2 is the tree's
 * binary node).  packed (device, q * n(n+1)/2 words, triangle i at offset
 * i*n(n+1)/2, each packed column by column as tsqr_pack_r): IN R_1..R_q, OUT R in
 * slot 0 and the reflectors' v parts Y_2..Y_q (upper triangles, v(1) = 1
 * implicit) in slots 1..q-1.  tau (device, n): OUT.  One CTA; asynchronous. */
tsqr_status_t tsqr_combine_stacked(int32_t q, int64_t n, double *packed, double *tau, void *stream);

/* ---------------------------------------------------------------- CAQR
 * Right-looking QR of an m x N matrix (N may exceed TSQR_MAX_N) with TSQR
 * panels: "CAQR simply implements the right-looking QR factorization using ...
 * TSQR as the panel factorization" (Sec. 3); Alg. CAQR:j ([TR]
 * P:3992-4048) on one GPU (one process row).  Panel j = columns c0..c0+w-1
 * (c0 = j*panel_cols, w = min(panel_cols, N - c0)) is factored by tsqr_factor
 * over rows c0..m-1 (line 1), then Q_j^T is applied to the trailing columns by
 * tsqr_apply_qt (line 3 and the tree stages, lines 4-9); rows c0..c0+w-1 of the
 * update are R's row block, rows c0+w.. (panel j's tree order) the next panel.
 * Q = Q_1 diag(I, Q_2) ... ; Q_j acts on rows c0_j..m-1. */
typedef struct tsqr_caqr_s *tsqr_caqr_t;

/* A (device, m x N, lda >= m, m >= N): IN the matrix, OUT the panels' reflectors
 * and the trailing updates; BORROWED until tsqr_caqr_free.  R (device, N x N,
 * ldr >= N): OUT upper triangular, exact zeros below.  opts: as tsqr_factor's,
 * used for every panel (nranks must be 0 or 1: TSQR_ERR_UNSUPPORTED otherwise).
 * panel_cols in [1, TSQR_MAX_N].  *caqr: OUT a new handle, or IN a handle of the
 * same (m, N, panel_cols, block_rows, tile_rows) whose panel trees are reused
 * (TSQR_ERR_INVALID for another shape).  Errors of a panel's TSQR are returned
 * as they are (e.g. TSQR_ERR_SHAPE when a panel's row block has < w rows). */
tsqr_status_t tsqr_caqr_factor(int64_t m, int64_t N, double *A, int64_t lda, int64_t panel_cols,
                               double *R, int64_t ldr, const tsqr_opts_t *opts, void *stream,
                               tsqr_caqr_t *caqr);

/* C <- Q^T C (C: device, m x k, ldc >= m), the panels' trees in order, each in
 * its own tree order on rows c0_j..m-1: rows 0..N-1 become Q_thin^T C. */
tsqr_status_t tsqr_caqr_apply_qt(tsqr_caqr_t caqr, double *C, int64_t ldc, int64_t k, void *stream);

/* C <- Q C, the inverse of tsqr_caqr_apply_qt (panels in reverse order). */
tsqr_status_t tsqr_caqr_apply_q(tsqr_caqr_t caqr, double *C, int64_t ldc, int64_t k, void *stream);

/* Explicit thin Q (device, m x N, ldq >= m) = Q [I_N; 0]. */
tsqr_status_t tsqr_caqr_form_q(tsqr_caqr_t caqr, double *Q, int64_t ldq, void *stream);

/* Release the handle and its panel trees. */
tsqr_status_t tsqr_caqr_free(tsqr_caqr_t caqr);

/* Release the tree's device memory (stream-ordered on the last stream used). */
tsqr_status_t tsqr_tree_free(tsqr_tree_t tree);

/* Test hook: copy the tree's leaf taus (nchunks*n: chunk k of the tiles in
 * order, reflector j at [k*n + j], 0 where chunk k has no reflector j) and the
 * node taus (by node b index, ntiles*n; row 0 unused) to host buffers (either
 * may be NULL).
 * Synchronises the tree's stream. */
tsqr_status_t tsqr_tree_export_tau(tsqr_tree_t tree, double *tau_tile_host, double *tau_node_host);

/* Measurement hook: device time (ms) of the last tsqr_factor's leaf stage
 * (a2+a3: the dominant kernel) and of its tree stage (a4+a6), from CUDA events
 * recorded on the factor's stream when opts.flags bit 1 was set (else
 * TSQR_ERR_INVALID).  Either pointer may be NULL.  Waits for the last event. */
tsqr_status_t tsqr_tree_stage_ms(tsqr_tree_t tree, float *leaf_ms, float *tree_ms);

/* ---------------------------------------------------------------- communicator
 * Row-sharded multi-GPU TSQR as ONE collective call per operation:
 * Alg. TSQR:par ([TR] P:1667-1707) with the butterfly indexing of [TR]
 * each rank factors its slab (tsqr_factor), then log2(nranks)
 * rounds, each one grouped ncclSend/ncclRecv of the packed R (n(n+1)/2 words,
 * the Cor. 2 minimum) with partner rank XOR 2^(k-1) on the caller's
 * stream followed by the structured combine; R ends replicated.
 * Everything is enqueued on `stream` (no host synchronisation), so the calls
 * can be captured in a CUDA graph.  One context per process (= per GPU).
 * Every ctx call on a context with nranks > 1 is COLLECTIVE over its ranks, with
 * the same n, k and plan options on every rank; m_local, A, C and Q are the
 * rank's slab (tsqr_slab); R and top are replicated.  SURVEY 8(b) writes
 * tsqr_factor(ctx, ...): that is tsqr_ctx_factor below; tsqr_factor without a
 * context is its local (one-rank) layer. */
typedef struct tsqr_ctx_s *tsqr_ctx_t;

/* A context on CUDA device `device` (nranks = 1 until a communicator is set). */
tsqr_status_t tsqr_ctx_create(int device, tsqr_ctx_t *out);

/* ncclGetUniqueId into uid128 (host, 128 bytes): rank 0 calls it and hands the
 * bytes to every rank (any host channel, e.g. torch.distributed). */
tsqr_status_t tsqr_get_unique_id(void *uid128);

/* ncclCommInitRank(nranks, uid, rank) on the context's device (collective and
 * blocking across the ranks).  nranks must be a power of two (the butterfly;
 * TSQR_ERR_UNSUPPORTED otherwise).  Replaces an earlier communicator. */
tsqr_status_t tsqr_ctx_set_comm(tsqr_ctx_t ctx, const void *uid128, int32_t nranks, int32_t rank);

/* Test transport: the ranks of one process exchange through a host mailbox
 * (each side synchronises its stream, then copies its partner's message) instead
 * of NCCL -- kernels of one rank never wait on another's.  hub from
 * tsqr_loopback_create(nranks); ctx takes rank `rank` of it. */
typedef struct tsqr_loopback_s *tsqr_loopback_t;
tsqr_status_t tsqr_loopback_create(int32_t nranks, tsqr_loopback_t *out);
tsqr_status_t tsqr_loopback_destroy(tsqr_loopback_t hub);
tsqr_status_t tsqr_ctx_set_loopback(tsqr_ctx_t ctx, tsqr_loopback_t hub, int32_t rank);

/* Ranks and rank of the context. */
tsqr_status_t tsqr_ctx_info(tsqr_ctx_t ctx, int32_t *nranks, int32_t *rank);

/* Release the communicator and the context's exchange buffers. */
tsqr_status_t tsqr_ctx_destroy(tsqr_ctx_t ctx);

/* Collective factor: tsqr_factor of this rank's slab (opts' nranks and rank are
 * taken from the context), then every butterfly round inside the call.  R (device,
 * n x n, ldr >= n, may be NULL) receives the replicated R.  *tree as tsqr_factor. */
tsqr_status_t tsqr_ctx_factor(tsqr_ctx_t ctx, int64_t m_local, int64_t n, double *A, int64_t lda,
                              double *R, int64_t ldr, const tsqr_opts_t *opts, void *stream,
                              tsqr_tree_t *tree);

/* Collective C <- Q^T C: the local tree (tsqr_apply_qt), then per round one
 * exchange of the n x k R coordinates (n k words, Table 1) and the
 * round's node reflectors on [top_lower; top_upper] (eq. localQTupdate
 * P:2193-2212).  C (device, m_local x k, ldc) ends in tree order (rank 0's rows
 * 0..n-1 = Q_thin^T C); top (device, n x k, ldtop >= n, may be NULL) receives the
 * replicated Q_thin^T C on every rank. */
tsqr_status_t tsqr_ctx_apply_qt(tsqr_ctx_t ctx, tsqr_tree_t tree, double *C, int64_t ldc, int64_t k,
                                double *top, int64_t ldtop, void *stream);

/* Collective C <- Q C (C in tree order), the inverse of tsqr_ctx_apply_qt: the
 * rounds top-down between the two group heads of each round, then the local tree. */
tsqr_status_t tsqr_ctx_apply_q(tsqr_ctx_t ctx, tsqr_tree_t tree, double *C, int64_t ldc, int64_t k, void *stream);

/* Explicit thin Q rows of this rank: no communication (the butterfly replicates
 * every cross-rank node factor, [TR] P:1919-1925); = tsqr_form_q. */
tsqr_status_t tsqr_ctx_form_q(tsqr_ctx_t ctx, tsqr_tree_t tree, double *Q, int64_t ldq, void *stream);

/* ---------------------------------------------------------------- CholeskyQR
 * The comparison method of SURVEY 8(f) row 4 -- NOT the TSQR path.  Alg.
 * CholeskyQR ([TR] P:1410-1419): W := A^T A (line 1), W = L L^T (line 2),
 * Q := A L^{-T} (line 3); R = L^T.  Its Q "loses orthogonality proportionally
 * to kappa_2(A)^2" where TSQR's stays orthogonal: the stability
 * half of "only parallel TSQR is simultaneously fastest and stable"
 * (P:1347-1354).  A^T A and A R^{-1} run on FP64 DMMA.
 * A (device, m x n, lda >= m) is read only.  R (device, n x n, ldr >= n)
 * receives the upper triangular factor with a positive diagonal (zeros below).
 * Q (device, m x n, ldq >= m, may be NULL: R only) receives A R^{-1}.
 * info (DEVICE int) receives 0, or j + 1 when the computed W's leading minor of
 * order j + 1 is not positive (Cholesky breakdown -- kappa(A)^2 beyond 1/eps);
 * R and Q are then unspecified.  Workspace is stream-ordered (cudaMallocAsync
 * on `stream`); TSQR_ERR_ALLOC if it cannot be had.  n <= TSQR_MAX_N. */
tsqr_status_t tsqr_cholqr(int64_t m, int64_t n, const double *A, int64_t lda, double *R, int64_t ldr,
                          double *Q, int64_t ldq, int *info, void *stream);

/* Collective CholeskyQR over the context's ranks (row slabs as tsqr_ctx_factor):
 * each rank's A_i^T A_i, then the all-reduction of line 1 as log2(nranks)
 * butterfly rounds of n^2 words (lower rank's W + upper rank's W in that order,
 * so W -- hence R -- is bitwise identical on every rank; Table "CholeskyQR
 * counts": log P messages), then lines 2-3 locally.  R replicated;
 * Q = this rank's rows. */
tsqr_status_t tsqr_ctx_cholqr(tsqr_ctx_t ctx, int64_t m_local, int64_t n, const double *A, int64_t lda,
                              double *R, int64_t ldr, double *Q, int64_t ldq, int *info, void *stream);

/* ---------------------------------------------------------------- host
 * End-to-end QR with HOST buffers on one GPU (the e2e path of bench.py): A (host,
 * m x n, lda >= m) is copied to the device, factored (tsqr_factor with opts;
 * nranks must be 0 or 1), R (host, n x n, ldr >= n) receives R (zeros below);
 * if Q (host, ldq >= m) is non-NULL it receives the explicit thin Q (tsqr_form_q);
 * if k > 0, C (host, m x k, ldc >= m) is replaced by Q^T C in tree order
 * (tsqr_apply_qt).  Every copy and kernel is enqueued on `stream`; page-locked
 * host buffers make the copies asynchronous DMA.  Returns after the outputs
 * have landed in host memory (synchronises `stream`).  *ws: device workspace
 * and tree, created on first use (pass a NULL-initialised handle) and reused
 * while (m, n) match; release with tsqr_host_ws_free. */
typedef struct tsqr_host_ws_s *tsqr_host_ws_t;
tsqr_status_t tsqr_qr_host(tsqr_host_ws_t *ws, int64_t m, int64_t n, const double *A, int64_t lda,
                           double *R, int64_t ldr, double *Q, int64_t ldq, double *C, int64_t ldc,
                           int64_t k, const tsqr_opts_t *opts, void *stream);
tsqr_status_t tsqr_host_ws_free(tsqr_host_ws_t ws);

/* ---------------------------------------------------------------- measurement
 * FP64 pipe peak of the current device (TFLOP/s, best of 3): DMMA.8x8x4 chains and
 * DFMA chains on every SM (the roofline denominator of SURVEY 8(d)).  Synchronises
 * `stream`.  Not on the TSQR path. */
tsqr_status_t tsqr_measure_fp64_peak(double *dmma_tflops, double *dfma_tflops, void *stream);

#ifdef __cplusplus
}
#endif
#endif
