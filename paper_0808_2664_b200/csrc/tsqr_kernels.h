// Host-side declarations of the kernel launchers (tsqr_chain.cu, tsqr_cs.cu,
// tsqr_tree.cu, tsqr_wide.cu, tsqr_wy.cu), called by the C-ABI in tsqr_api.cu.
#pragma once
#include "../../include/tsqr.h"

#include <cstdint>
#include <cuda_runtime.h>
#include <vector>


namespace tsqr {

// The text tsqr_last_error() returns (tsqr_api.cu); for the C-ABI entry points in other files.
void set_last_error(const char *where, cudaError_t e);
void set_last_error_text(const char *text);
}  // namespace tsqr
struct tsqr_tree_s;
namespace tsqr {
// Shape of a tree handle (tsqr_api.cu), for the communicator layer (tsqr_comm.cu).
bool tree_shape(const tsqr_tree_s *t, int64_t *m_local, int64_t *n, int *nranks, int *rank, int *rounds_done);
// A local tree's implicit-Q state besides the reflectors in A (taus, cached T's):
// its size in doubles, and a packed stream-ordered copy to / from host memory
// (tsqr_api.cu; used by the streamed factor's Q, tsqr_stream.cu).
// full = false: the compact state (the chain engine's chunk T cache left out and rebuilt
// from Y and the taus on import -- the tree must already be bound to its reflectors).
size_t tree_state_words(const tsqr_tree_s *t, bool full);
tsqr_status_t tree_state_words_for(int64_t m_local, int64_t n, const tsqr_opts_t *opts, bool full, size_t *words);
cudaError_t tree_state_copy(tsqr_tree_s *t, double *host, bool to_host, bool full, cudaStream_t st);
// after a compact import: the chain engine's chunk T cache from the bound reflectors and taus
cudaError_t tree_rebuild_tcache(tsqr_tree_s *t, cudaStream_t st);
// A tree of the plan (m_local, n, opts) bound to reflectors in A without a factor
// (for an imported state); reuses *tree when the plan matches.
tsqr_status_t tree_bind(int64_t m_local, int64_t n, double *A, int64_t lda, const tsqr_opts_t *opts,
                        cudaStream_t st, tsqr_tree_s **tree);
// The host-buffer QR + explicit Q pipelined over S slabs of tiles (tsqr_api.cu; n <= 64, one
// rank; TSQR_ERR_UNSUPPORTED otherwise, before anything is enqueued).
tsqr_status_t qr_host_pipelined(tsqr_tree_s **tree, int64_t m, int64_t n, const double *A, int64_t lda, double *dA,
                                double *dR, double *dQ, double *R, int64_t ldr, double *Q, int64_t ldq,
                                const tsqr_opts_t *opts, cudaStream_t st, cudaStream_t up, cudaStream_t down, int S);

// Leaf stage on the chunk engine (tsqr_chain.cu).
struct ChainArgs {
    double *A; int64_t lda; int n;
    int64_t m = 0;               // rows of A (the TMA tensor map's extent; 0 = no TMA)
    int chunk_rows;              // the plan's c (chain_chunk_rows(n))
    const int64_t *tile_row0; const int *tile_rows; const int64_t *tile_chunk0;
    const int *cta_tile0; int grid;
    double *tau;                 // [chunks][n]
    double *tcache;              // [chunks][NCB][8][8]: the panels' T (compact WY), may be null
    bool robust = false;         // the rescaled steps of reading R23 (opts.flags bit 2)
};
// Leaf stage of Q^T C (forward) or of form Q (Q = Q_leaves [X; 0], !forward).
struct ChainApplyArgs {
    const double *A; int64_t lda; int n;
    int chunk_rows;
    const int64_t *tile_row0; const int *tile_rows; const int64_t *tile_chunk0;
    const int *cta_tile0; int grid;
    const double *tcache;        // the factor's T cache
    double *C; int64_t ldc; int k;
    int forward;
    const double *xbuf;          // !forward: per-tile X (n x n) from the node stage (form Q);
                                 // nullptr: C <- Q C in place (the head rows hold C_R)
    bool bulk = false;           // Y / T staged by bulk copies (every tile starts on an even row)
};
// Chain engine (tsqr_chain.cu): chunk rows, column blocks, persistent grid, factor.
int chain_chunk_rows(int n);
int chain_ncb(int n);
int chain_grid(int n);
int cs_apply_grid(int n);   // SMs x resident apply CTAs
cudaError_t launch_chain_factor(const ChainArgs &f, cudaStream_t st);
// The factor's T cache recomputed from the stored reflectors and chunk taus (streamed Q).
cudaError_t launch_chain_rebuild_t(const double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows,
                                   const int64_t *tile_chunk0, int ntiles, int64_t nchunks, const double *tau,
                                   double *tcache, cudaStream_t st);
// Leaf stage of Q^T C / form Q on the chain representation (tsqr_cs.cu).
cudaError_t launch_cs_apply(const ChainApplyArgs &f, cudaStream_t st);
// Wide-n engine (tsqr_wide.cu, 64 < n <= 256): one CTA per leaf / node problem.
int wide_max_rows();
cudaError_t launch_wide_leaves(double *A, int64_t lda, int n, const int64_t *row0, const int *rows, int L,
                               int max_rows, double *tau, double *tcache, double *tpair, bool robust, cudaStream_t st);
cudaError_t launch_wide_nodes(double *A, int64_t lda, int n, const int64_t *row0, const int *node_a, const int *ids,
                              int count, double *tau_node, double *tcache_node, cudaStream_t st);
cudaError_t launch_wide_node1(double *Ra, int64_t lda, double *Rb, int64_t ldb, int n, double *tau, double *tcache,
                              cudaStream_t st);
cudaError_t launch_wide_apply_leaves(const double *A, int64_t lda, int n, const int64_t *row0, const int *rows,
                                     int L, int max_rows, const double *tcache, const double *tpair, double *C,
                                     int64_t ldc, int k, int forward, cudaStream_t st);
cudaError_t launch_node_apply(const double *A, int64_t lda, int n, const int64_t *row0, const int *node_a,
                                    const int *ids, int count, const double *tcache_node, double *C, int64_t ldc,
                                    int k, int forward, int xbuf_mode, cudaStream_t st);
cudaError_t launch_node_apply_pipe(const double *A, int64_t lda, int n, const int64_t *row0, const int *node_a,
                                   const int *ids, int count, const int *dep0, const int *dep1, int *flags, int L,
                                   const double *tcache_node, double *C, int64_t ldc, int k, int forward,
                                   int xbuf_mode, cudaStream_t st);
cudaError_t launch_wide_apply_node1(const double *Y1, int64_t ldy, int n, const double *tcache, double *Ca,
                                    int64_t ldca, double *Cb, int64_t ldcb, int k, int forward, cudaStream_t st);
cudaError_t launch_wide_formq_init(const int64_t *row0, const int *rows, int L, int n, const double *xbuf, double *Q,
                                   int64_t ldq, cudaStream_t st);
cudaError_t launch_extract_r(const double *A, int64_t lda, int n, double *R, int64_t ldr, cudaStream_t st);
cudaError_t launch_wide_cross_factor(double *A, int64_t lda, int n, const double *packed, int is_lower, double *tmp,
                                     double *Y1, double *tau, double *tcache, double *R, int64_t ldr,
                                     cudaStream_t st);
cudaError_t launch_wide_cross_apply(const double *Y1, const double *tcache, double *top, int64_t ldtop,
                                    const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n, int k,
                                    double *tmp, int forward, cudaStream_t st);
cudaError_t launch_wide_cross_root_x(const double *Y1s, const double *tcaches, int64_t tstride, int rounds, int rank,
                                     int n, double *tmp, double *X0, cudaStream_t st);
// Balanced contiguous split of the tiles over `grid` persistent CTAs by chunk count.
void chain_partition(const std::vector<int64_t> &tile_rows, int chunk_rows, int grid, std::vector<int> &cta_tile0);
// Pipelined node combines for n <= 64 (tsqr_tree.cu): nodes (ids, bottom-up),
// prod_l/prod_r = producing node of each child (-1: leaf), flags L x NCB ints.
cudaError_t launch_tree_pipe(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a,
                             const int *nodes, int count, const int *prod_l, const int *prod_r, int *flags,
                             double *tau_node, int root, double *R, int64_t ldr, double *tcache_node,
                             cudaStream_t st);
// The same for 64 < n <= 224: one CTA per node (flags L x 28 ints).
bool wide_tree_pipe_ok(int n);
cudaError_t launch_wide_tree_pipe(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a,
                                  const int *nodes, int count, const int *prod_l, const int *prod_r, int *flags,
                                  double *tau_node, double *tcache_node, bool robust, cudaStream_t st);
cudaError_t launch_identity(double *X, int n, cudaStream_t st);
cudaError_t launch_pack_r(const double *A, int64_t lda, int n, double *packed, cudaStream_t st);
cudaError_t launch_unpack_r(const double *packed, int n, double *A, int64_t lda, cudaStream_t st);
cudaError_t launch_copy_block(const double *src, int64_t lds, double *dst, int64_t ldd, int n, int k,
                              cudaStream_t st);
cudaError_t launch_cross_factor(int NP, double *A, int64_t lda, int n, const double *pp, int is_lower,
                                double *Y1, double *tau, double *R, int64_t ldr, cudaStream_t st);
cudaError_t launch_cross_apply(int NP, const double *Y1, const double *tau, double *top, int64_t ldtop,
                               const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n,
                               int k, int forward, cudaStream_t st);
cudaError_t launch_cross_root_x(int NP, const double *Y1s, const double *taus, int rounds, int rank, int n,
                                double *X0, cudaStream_t st);


// CholeskyQR comparison path (tsqr_cholqr.cu): workspace and stages.
struct CholqrWs {
    double *base = nullptr, *W = nullptr, *Rinv = nullptr, *part = nullptr;
    int nsplit = 1;
    int64_t rows_per_split = 0;
    ~CholqrWs();
};
cudaError_t cholqr_alloc(CholqrWs &w, int64_t m, int n, cudaStream_t st);
void cholqr_free(CholqrWs &w, cudaStream_t st);
cudaError_t cholqr_gram(const double *A, int64_t lda, int64_t m, int n, CholqrWs &w, cudaStream_t st);   // w.W = A^T A
cudaError_t cholqr_add_ordered(double *W, const double *P, int64_t count, int is_lower, cudaStream_t st);
cudaError_t cholqr_finish(const double *A, int64_t lda, int64_t m, int n, CholqrWs &w, double *R, int64_t ldr,
                          double *Q, int64_t ldq, int *info, cudaStream_t st);
}  // namespace tsqr
