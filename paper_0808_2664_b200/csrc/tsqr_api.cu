// C-ABI of libtsqr.so (include/tsqr.h): validation, tree handles, launch order.
// Product code.  Every device call validates all arguments on the host first;
// an error status means nothing was enqueued.
#include "../../include/tsqr.h"
#include "plan.h"
#include "tsqr_kernels.h"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

using namespace tsqr;

static thread_local std::string g_last_error;

// NVTX range over a device entry point (named in nsys / ncu --nvtx timelines; a no-op
// without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

struct tsqr_tree_s {
    Plan plan;
    tsqr_opts_t opts{};
    int NP = 64;
    int device = 0;
    double *A = nullptr;
    int64_t lda = 0;
    cudaStream_t stream = nullptr;
    // device arrays
    int64_t *d_row0 = nullptr;
    int *d_rows = nullptr, *d_node_a = nullptr;
    double *d_tau_node = nullptr;
    double *d_cross_y1 = nullptr, *d_cross_tau = nullptr;
    int cross_rounds = 0, cross_done = 0;
    double *d_xbuf = nullptr;
    int *d_step_ids = nullptr;
    int *d_pipe_nodes = nullptr, *d_prod_l = nullptr, *d_prod_r = nullptr, *d_pipe_flags = nullptr;
    int *d_parent = nullptr, *d_node_flags = nullptr;   // the one-launch node stages of apply / form Q
    // the pipelined host path (tsqr_qr_host): per-slab CTA partitions of the leaf and form-Q
    // kernels, slab k's at d_slab_part + slab_off[k] (leaves) / + slab_off[S + k] (form Q)
    int slab_S = 0;
    std::vector<int> slab_t0, slab_grid, slab_off;
    int *d_slab_part = nullptr;
    int pipe_count = 0, pipe_root = -1;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};   // stage timing (opts.flags bit 1)
    bool ev_recorded = false;
    // completion of the last call on the tree (recorded on its stream): a call on another
    // stream first waits for it, so the handle may move between streams
    cudaEvent_t done = nullptr;
    bool done_valid = false;
    // chunk-chain leaf stage
    int64_t *d_tile_chunk0 = nullptr;
    int *d_cta_tile0 = nullptr, *d_apply_cta_tile0 = nullptr;
    int chain_grid = 0, apply_grid = 0;
    bool rows_even = false;           // every tile starts on an even row (TMA boxes need 16-byte aligned starts)
    double *d_tau_chunk = nullptr;
    double *d_tcache = nullptr;       // [chunks][NCB][8][8] panel T factors (compact WY)
    int64_t nchunks = 0;
    // wide n (> 64): per-node T cache, butterfly T caches, a stacking buffer
    bool wide = false;
    int npan = 0;
    double *d_tcache_node = nullptr, *d_cross_tcache = nullptr, *d_wtmp = nullptr;
    double *d_tcache_pair = nullptr;   // wide leaves: T01 of each pair of panels (tiles <= 1024 rows)
    double *d_gather = nullptr;        // all-gathered cross variant: n x n scratch + G packed group R's
    int64_t wtmp_size = 0;
    std::vector<int> step_off;   // top-down: groups [step_off[g], step_off[g+1])
};

void tsqr::set_last_error(const char *where, cudaError_t e) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
}

void tsqr::set_last_error_text(const char *text) { g_last_error = text; }

bool tsqr::tree_shape(const tsqr_tree_s *t, int64_t *m_local, int64_t *n, int *nranks, int *rank, int *rounds_done) {
    if (!t) return false;
    *m_local = t->plan.m_local;
    *n = t->plan.n;
    *nranks = t->opts.nranks;
    *rank = t->opts.rank;
    *rounds_done = t->cross_done;
    return true;
}

static tsqr_status_t cuda_fail(cudaError_t e, const char *where) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return TSQR_ERR_CUDA;
}

#define CUDA_TRY(expr, where)                               \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, where); \
    } while (0)

static tsqr_status_t debug_sync(const tsqr_tree_s *t, cudaStream_t st, const char *where) {
    if (t->opts.flags & 1) CUDA_TRY(cudaStreamSynchronize(st), where);
    return TSQR_OK;
}
static tsqr_status_t leave(tsqr_tree_s *t, cudaStream_t st);
static tsqr_status_t enter(tsqr_tree_s *t, cudaStream_t st);
static tsqr_status_t finish(tsqr_tree_s *t, cudaStream_t st, const char *where) {
    tsqr_status_t s = leave(t, st);
    return s != TSQR_OK ? s : debug_sync(t, st, where);
}
#define ENTER(t, st)                                   \
    do {                                               \
        tsqr_status_t _s = enter((t), (st));           \
        if (_s != TSQR_OK) return _s;                  \
    } while (0)

// Stream ordering of a tree's calls: every device entry point runs enter() before its
// first launch and leave() after its last one.
static tsqr_status_t enter(tsqr_tree_s *t, cudaStream_t st) {
    if (t->done_valid && st != t->stream) CUDA_TRY(cudaStreamWaitEvent(st, t->done, 0), "stream order");
    return TSQR_OK;
}
static tsqr_status_t leave(tsqr_tree_s *t, cudaStream_t st) {
    if (!t->done) CUDA_TRY(cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming), "stream order");
    CUDA_TRY(cudaEventRecord(t->done, st), "stream order");
    t->stream = st;
    t->done_valid = true;
    return TSQR_OK;
}

// Device memory of a tree is stream-ordered (cudaMallocAsync / cudaFreeAsync on the
// call's stream): nothing here synchronises the host.
static void free_tree_memory(tsqr_tree_s *t, cudaStream_t st) {
    void *ptrs[] = {t->d_row0, t->d_rows, t->d_node_a,
                    t->d_tau_node, t->d_cross_y1, t->d_cross_tau, t->d_xbuf,
                    t->d_step_ids, t->d_pipe_nodes, t->d_prod_l, t->d_prod_r, t->d_pipe_flags, t->d_parent,
                    t->d_node_flags, t->d_slab_part,
                    t->d_tile_chunk0, t->d_cta_tile0, t->d_apply_cta_tile0, t->d_tau_chunk, t->d_tcache,
                    t->d_tcache_node, t->d_cross_tcache, t->d_wtmp, t->d_tcache_pair, t->d_gather};
    for (void *p : ptrs)
#ifdef TSQR_PLAIN_MALLOC
        if (p) cudaFree(p);
#else
        if (p) cudaFreeAsync(p, st);
#endif
}

// The wide path's stacking buffer (2n x max(n, cols) doubles), grown on demand.
static tsqr_status_t wide_tmp(tsqr_tree_s *t, int64_t cols, cudaStream_t st) {
    const int64_t need = 2 * t->plan.n * std::max<int64_t>(cols, t->plan.n);
    if (t->d_wtmp && t->wtmp_size >= need) return TSQR_OK;
    if (t->d_wtmp) cudaFreeAsync(t->d_wtmp, st);
    t->d_wtmp = nullptr;
    if (cudaMallocAsync((void **)&t->d_wtmp, sizeof(double) * need, st) != cudaSuccess) {
        cudaGetLastError();
        t->wtmp_size = 0;
        return TSQR_ERR_ALLOC;
    }
    t->wtmp_size = need;
    return TSQR_OK;
}

static int ilog2(int x) {
    int r = 0;
    while ((1 << r) < x) ++r;
    return r;
}

// The node stages of Q^T C (forward: bottom-up, after the leaves) or of Q C / form Q
// (top-down, before the leaves) on C's tile heads (xbuf_mode: the per-tile X blocks):
// one pipelined launch over the whole tree when the node kernel fits (n <= 224), else
// one launch per tree step.
static cudaError_t node_stages(tsqr_tree_s *t, double *C, int64_t ldc, int k, bool forward, int xbuf_mode,
                               cudaStream_t st) {
    const int n = (int)t->plan.n, L = t->plan.ntiles();
    const int count = t->step_off.back();
    if (count == 0) return cudaSuccess;
    if ((n + 7) / 8 <= 28) {
        return forward ? launch_node_apply_pipe(t->A, t->lda, n, t->d_row0, t->d_node_a, t->d_pipe_nodes, count,
                                                t->d_prod_l, t->d_prod_r, t->d_node_flags, L, t->d_tcache_node, C,
                                                ldc, k, 1, xbuf_mode, st)
                       : launch_node_apply_pipe(t->A, t->lda, n, t->d_row0, t->d_node_a, t->d_step_ids, count,
                                                t->d_parent, nullptr, t->d_node_flags, L, t->d_tcache_node, C, ldc,
                                                k, 0, xbuf_mode, st);
    }
    if (forward) {
        for (size_t g = t->step_off.size() - 1; g-- > 0;) {             // tree steps bottom-up
            const int cnt = t->step_off[g + 1] - t->step_off[g];
            if (cnt == 0) continue;
            const cudaError_t e = launch_node_apply(t->A, t->lda, n, t->d_row0, t->d_node_a,
                                                    t->d_step_ids + t->step_off[g], cnt, t->d_tcache_node, C, ldc,
                                                    k, 1, xbuf_mode, st);
            if (e != cudaSuccess) return e;
        }
    } else {
        for (size_t g = 0; g + 1 < t->step_off.size(); ++g) {             // tree steps top-down
            const int cnt = t->step_off[g + 1] - t->step_off[g];
            if (cnt == 0) continue;
            const cudaError_t e = launch_node_apply(t->A, t->lda, n, t->d_row0, t->d_node_a,
                                                    t->d_step_ids + t->step_off[g], cnt, t->d_tcache_node, C, ldc,
                                                    k, 0, xbuf_mode, st);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

extern "C" {

const char *tsqr_status_string(tsqr_status_t s) {
    switch (s) {
        case TSQR_OK: return "ok";
        case TSQR_ERR_INVALID: return "invalid argument";
        case TSQR_ERR_SHAPE: return "invalid shape (m < n, or a tile / row block with fewer than n rows)";
        case TSQR_ERR_UNSUPPORTED: return "unsupported (n > TSQR_MAX_N, tile_rows above capacity, or nranks not a power of two)";
        case TSQR_ERR_ALLOC: return "allocation failed";
        case TSQR_ERR_CUDA: return "CUDA error";
        case TSQR_ERR_NCCL: return "NCCL error or failed butterfly exchange";
    }
    return "unknown status";
}

const char *tsqr_last_error(void) { return g_last_error.c_str(); }

tsqr_status_t tsqr_slab(int64_t m, int64_t n, int64_t block_rows, int32_t nranks, int32_t rank,
                        int64_t *row0, int64_t *m_local) {
    if (!row0 || !m_local) return TSQR_ERR_INVALID;
    return (tsqr_status_t)rank_slab(m, n, block_rows, nranks, rank, row0, m_local);
}

static tsqr_opts_t resolve_opts(int64_t m_local, const tsqr_opts_t *o) {
    tsqr_opts_t r{};
    if (o) r = *o;
    if (r.block_rows == 0) r.block_rows = m_local;
    if (r.nranks == 0) r.nranks = 1;
    return r;
}

static int plan_for(int64_t m_local, int64_t n, const tsqr_opts_t *opts, Plan *p, tsqr_opts_t *ro) {
    *ro = resolve_opts(m_local, opts);
    if (ro->block_rows < 0) return TSQR_ERR_INVALID;
    return build_plan(m_local, n, ro->block_rows, ro->tile_rows, ro->nranks, ro->rank, p);
}

tsqr_status_t tsqr_plan_info(int64_t m_local, int64_t n, const tsqr_opts_t *opts, tsqr_plan_info_t *info) {
    if (!info) return TSQR_ERR_INVALID;
    Plan p;
    tsqr_opts_t ro;
    int rc;
    try { rc = plan_for(m_local, n, opts, &p, &ro); } catch (const std::bad_alloc &) { return TSQR_ERR_ALLOC; }
    if (rc) return (tsqr_status_t)rc;
    info->m_local = m_local;
    info->n = n;
    info->block_rows = p.b;
    info->tile_rows = p.s;
    info->ntiles = p.ntiles();
    info->nnodes = (int64_t)p.nodes.size();
    info->nblocks = (int64_t)p.blk_tile0.size() - 1;
    info->depth = p.nsteps;
    info->cross_rounds = ilog2(ro.nranks);
    info->max_tile_rows = p.max_rows;
    info->min_tile_rows = p.min_rows;
    info->tile_capacity = tile_capacity(n);
    info->chunk_rows = p.c;
    info->nchunks = p.tile_chunk0.back();
    return TSQR_OK;
}

tsqr_status_t tsqr_plan_export(int64_t m_local, int64_t n, const tsqr_opts_t *opts, int64_t *tile_row0,
                               int64_t *tile_rows, int64_t *node_a, int64_t *node_b, int64_t *node_stage,
                               int64_t *node_level) {
    Plan p;
    tsqr_opts_t ro;
    int rc;
    try { rc = plan_for(m_local, n, opts, &p, &ro); } catch (const std::bad_alloc &) { return TSQR_ERR_ALLOC; }
    if (rc) return (tsqr_status_t)rc;
    for (int t = 0; t < p.ntiles(); ++t) {
        if (tile_row0) tile_row0[t] = p.tile_row0[t];
        if (tile_rows) tile_rows[t] = p.tile_rows[t];
    }
    for (size_t i = 0; i < p.nodes.size(); ++i) {
        if (node_a) node_a[i] = p.nodes[i].a;
        if (node_b) node_b[i] = p.nodes[i].b;
        if (node_stage) node_stage[i] = p.nodes[i].stage;
        if (node_level) node_level[i] = p.nodes[i].level;
    }
    return TSQR_OK;
}

tsqr_status_t tsqr_cross_partner(int32_t nranks, int32_t rank, int32_t round, int32_t *partner,
                                 int32_t *is_lower, int32_t *head_role) {
    if (nranks < 1 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks) return TSQR_ERR_INVALID;
    if (round < 1 || round > ilog2(nranks)) return TSQR_ERR_INVALID;
    const int half = 1 << (round - 1);
    const int p = rank ^ half;
    if (partner) *partner = p;
    if (is_lower) *is_lower = rank < p;
    if (head_role) {
        const int pos = rank & (2 * half - 1);          // position inside the 2^round group
        *head_role = pos == 0 ? 1 : (pos == half ? 2 : 0);
    }
    return TSQR_OK;
}

static tsqr_status_t create_tree(int64_t m_local, int64_t n, double *A, int64_t lda, const tsqr_opts_t *opts,
                                 cudaStream_t st, tsqr_tree_s **out) {
    tsqr_tree_s *t = new (std::nothrow) tsqr_tree_s();
    if (!t) return TSQR_ERR_ALLOC;
    tsqr_opts_t ro;
    int rc;
    try { rc = plan_for(m_local, n, opts, &t->plan, &ro); } catch (const std::bad_alloc &) { rc = TSQR_ERR_ALLOC; }
    if (rc) { delete t; return (tsqr_status_t)rc; }
    t->opts = ro;
    t->NP = padded_width(n);
    cudaGetDevice(&t->device);
    const Plan &p = t->plan;
    const int L = p.ntiles();
    // top-down form-Q schedule: node ids grouped by step, highest step first
    std::vector<int> ids;
    t->step_off.push_back(0);
    for (int s = p.nsteps; s >= 1; --s) {
        for (const auto &nd : p.nodes)
            if (nd.step == s) ids.push_back(nd.b);
        t->step_off.push_back((int)ids.size());
    }
    t->cross_rounds = ilog2(ro.nranks);
    cudaError_t e = cudaSuccess;
    auto alloc = [&](void **ptr, size_t bytes) {
#ifdef TSQR_PLAIN_MALLOC            // measurement variant
        if (e == cudaSuccess) e = cudaMalloc(ptr, bytes < 16 ? 16 : bytes);
#else
        if (e == cudaSuccess) e = cudaMallocAsync(ptr, bytes < 16 ? 16 : bytes, st);
#endif
    };
    alloc((void **)&t->d_row0, sizeof(int64_t) * L);
    alloc((void **)&t->d_rows, sizeof(int) * L);
    alloc((void **)&t->d_node_a, sizeof(int) * L);
    alloc((void **)&t->d_tau_node, sizeof(double) * L * n);
    alloc((void **)&t->d_cross_y1, sizeof(double) * (t->cross_rounds + 1) * n * n);
    alloc((void **)&t->d_cross_tau, sizeof(double) * (t->cross_rounds + 1) * n);
    alloc((void **)&t->d_step_ids, sizeof(int) * (ids.size() + 1));
    // pipelined tree (n <= 64): nodes bottom-up; each child's producing node
    std::vector<int> pipe(ids.rbegin(), ids.rend()), prod_l(L, -1), prod_r(L, -1), last(L, -1);
    for (int b : pipe) {
        const int a = p.node_a[b];
        prod_l[b] = last[a];
        prod_r[b] = last[b];
        last[a] = b;
    }
    t->pipe_count = (int)pipe.size();
    t->pipe_root = L > 1 ? last[0] : -1;
    alloc((void **)&t->d_pipe_nodes, sizeof(int) * L);
    alloc((void **)&t->d_prod_l, sizeof(int) * L);
    alloc((void **)&t->d_prod_r, sizeof(int) * L);
    alloc((void **)&t->d_pipe_flags, sizeof(int) * (L * 32 + 1));   // L x panels (<= 28 wide, 8 narrow) + ticket
    // top-down dependency of the node stages: each node's parent (the node that writes the
    // head block this node reads); bottom-up it is prod_l / prod_r
    std::vector<int> parent(L, -1);
    for (int b : pipe) {
        if (prod_l[b] >= 0) parent[prod_l[b]] = b;
        if (prod_r[b] >= 0) parent[prod_r[b]] = b;
    }
    alloc((void **)&t->d_parent, sizeof(int) * L);
    alloc((void **)&t->d_node_flags, sizeof(int) * (L + 1));
    const int64_t nchunks = p.tile_chunk0[L];
    t->wide = n > 64;
    t->npan = (int)((n + 7) / 8);
    int grid = 1;
    std::vector<int> cta_tile0(2, 0);
    if (!t->wide) {
        grid = chain_grid((int)n);
        if (grid > L) grid = L;
        chain_partition(p.tile_rows, p.c, grid, cta_tile0);
    } else {
        cta_tile0[1] = L;
    }
    t->chain_grid = grid;
    int agrid = 1;                         // the apply / form-Q kernels' own split (higher occupancy)
    std::vector<int> apply_tile0(2, 0);
    if (!t->wide) {
        agrid = std::min(L, cs_apply_grid((int)n));
        chain_partition(p.tile_rows, p.c, agrid, apply_tile0);
    } else {
        apply_tile0[1] = L;
    }
    t->apply_grid = agrid;
    alloc((void **)&t->d_apply_cta_tile0, sizeof(int) * (agrid + 1));
    alloc((void **)&t->d_tile_chunk0, sizeof(int64_t) * (L + 1));
    alloc((void **)&t->d_cta_tile0, sizeof(int) * (grid + 1));
    alloc((void **)&t->d_tau_chunk, sizeof(double) * nchunks * n);
    const int ncb_cache = t->wide ? t->npan : chain_ncb((int)n);
    alloc((void **)&t->d_tcache, sizeof(double) * nchunks * ncb_cache * 64);
    alloc((void **)&t->d_tcache_node, sizeof(double) * L * t->npan * 64);    // node panel T's (both engines)
    if (t->wide) {
        alloc((void **)&t->d_cross_tcache, sizeof(double) * (ilog2(ro.nranks) + 1) * t->npan * 64);
        alloc((void **)&t->d_tcache_pair, sizeof(double) * L * ((t->npan + 1) / 2) * 64);
    }
    t->nchunks = nchunks;
    t->rows_even = std::all_of(p.tile_row0.begin(), p.tile_row0.end(), [](int64_t r) { return (r & 1) == 0; });
    if (e != cudaSuccess) {
        free_tree_memory(t, st);
        delete t;
        g_last_error = std::string("tsqr_factor alloc: ") + cudaGetErrorString(e);
        cudaGetLastError();
        return TSQR_ERR_ALLOC;
    }
    // plan arrays: stream-ordered copies on the call's stream (pageable sources are
    // staged by the driver before cudaMemcpyAsync returns, so the vectors may go)
    std::vector<int> rows(p.tile_rows.begin(), p.tile_rows.end());
    auto h2d = [&](void *dst, const void *src, size_t bytes) {
        if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
    };
    h2d(t->d_row0, p.tile_row0.data(), sizeof(int64_t) * L);
    h2d(t->d_rows, rows.data(), sizeof(int) * L);
    h2d(t->d_node_a, p.node_a.data(), sizeof(int) * L);
    h2d(t->d_step_ids, ids.data(), sizeof(int) * ids.size());
    h2d(t->d_pipe_nodes, pipe.data(), sizeof(int) * pipe.size());
    h2d(t->d_prod_l, prod_l.data(), sizeof(int) * L);
    h2d(t->d_prod_r, prod_r.data(), sizeof(int) * L);
    h2d(t->d_parent, parent.data(), sizeof(int) * L);
    h2d(t->d_tile_chunk0, p.tile_chunk0.data(), sizeof(int64_t) * (L + 1));
    h2d(t->d_cta_tile0, cta_tile0.data(), sizeof(int) * (grid + 1));
    h2d(t->d_apply_cta_tile0, apply_tile0.data(), sizeof(int) * (agrid + 1));
    if (e == cudaSuccess) e = cudaMemsetAsync(t->d_tau_node, 0, sizeof(double) * L * n, st);
    if (e != cudaSuccess) {
        free_tree_memory(t, st);
        delete t;
        return cuda_fail(e, "tsqr_factor setup");
    }
    *out = t;
    return TSQR_OK;
}

tsqr_status_t tsqr_factor(int64_t m_local, int64_t n, double *A, int64_t lda, double *R, int64_t ldr,
                          const tsqr_opts_t *opts, void *stream, tsqr_tree_t *tree) {
    NvtxRange nvtx_("tsqr_factor");
    if (!tree || !A) return TSQR_ERR_INVALID;
    if (n < 1 || m_local < n) return TSQR_ERR_SHAPE;
    if (lda < m_local) return TSQR_ERR_INVALID;
    if (R && ldr < n) return TSQR_ERR_INVALID;
    if (n > TSQR_MAX_N) return TSQR_ERR_UNSUPPORTED;
    {   // validate the plan before touching the handle
        Plan p;
        tsqr_opts_t ro;
        int rc;
        try { rc = plan_for(m_local, n, opts, &p, &ro); } catch (const std::bad_alloc &) { return TSQR_ERR_ALLOC; }
        if (rc) return (tsqr_status_t)rc;
    }
    tsqr_tree_s *t = *tree;
    const tsqr_opts_t ro = resolve_opts(m_local, opts);
    const bool reuse = t && t->plan.m_local == m_local && t->plan.n == n && t->opts.block_rows == ro.block_rows &&
                       (ro.tile_rows == 0 || t->plan.s == ro.tile_rows) && t->opts.nranks == ro.nranks &&
                       t->opts.rank == ro.rank;
    if (!reuse) {
        tsqr_tree_s *nt = nullptr;
        if (t) {                                  // the old tree's last work precedes the new one's
            tsqr_status_t s0 = enter(t, (cudaStream_t)stream);
            if (s0 != TSQR_OK) return s0;
        }
        tsqr_status_t s = create_tree(m_local, n, A, lda, opts, (cudaStream_t)stream, &nt);
        if (s != TSQR_OK) return s;
        if (t) {
            t->stream = (cudaStream_t)stream;     // stream-ordered release behind the new tree's setup
            tsqr_tree_free(t);
        }
        t = nt;
        *tree = t;
    } else {
        tsqr_status_t s0 = enter(t, (cudaStream_t)stream);
        if (s0 != TSQR_OK) return s0;
    }
    t->opts.flags = ro.flags;
    t->A = A;
    t->lda = lda;
    t->stream = (cudaStream_t)stream;
    t->cross_done = 0;
    const bool timed = (ro.flags & 2) != 0;
    t->ev_recorded = false;
    if (timed)
        for (cudaEvent_t &e : t->ev)
            if (!e) CUDA_TRY(cudaEventCreate(&e), "tsqr_factor events");
    auto mark = [&](int i) -> cudaError_t { return timed ? cudaEventRecord(t->ev[i], t->stream) : cudaSuccess; };
    ChainArgs ca;
    ca.A = A; ca.lda = lda; ca.n = (int)n; ca.m = t->rows_even ? m_local : 0; ca.chunk_rows = t->plan.c;
    ca.tile_row0 = t->d_row0; ca.tile_rows = t->d_rows; ca.tile_chunk0 = t->d_tile_chunk0;
    ca.cta_tile0 = t->d_cta_tile0; ca.grid = t->chain_grid; ca.tau = t->d_tau_chunk; ca.tcache = t->d_tcache;
    const bool robust = (ro.flags & TSQR_FLAG_ROBUST) != 0;     // reading R23
    ca.robust = robust;
    if (t->wide) {
        const int L = t->plan.ntiles();
        CUDA_TRY(mark(0), "tsqr_factor events");
        CUDA_TRY(launch_wide_leaves(A, lda, (int)n, t->d_row0, t->d_rows, L, (int)t->plan.max_rows, t->d_tau_chunk,
                                    t->d_tcache, t->d_tcache_pair, robust, t->stream),
                 "tsqr_factor leaves");
        CUDA_TRY(mark(1), "tsqr_factor events");
        if (wide_tree_pipe_ok((int)n)) {
            CUDA_TRY(launch_wide_tree_pipe(A, lda, (int)n, t->d_row0, t->d_node_a, t->d_pipe_nodes, t->pipe_count,
                                           t->d_prod_l, t->d_prod_r, t->d_pipe_flags, t->d_tau_node,
                                           t->d_tcache_node, robust, t->stream),
                     "tsqr_factor tree");
        } else {
            for (size_t g = t->step_off.size() - 1; g-- > 0;) {     // tree steps bottom-up
                const int cnt = t->step_off[g + 1] - t->step_off[g];
                if (cnt == 0) continue;
                CUDA_TRY(launch_wide_nodes(A, lda, (int)n, t->d_row0, t->d_node_a, t->d_step_ids + t->step_off[g],
                                           cnt, t->d_tau_node, t->d_tcache_node, t->stream),
                         "tsqr_factor tree");
            }
        }
        if (R) CUDA_TRY(launch_extract_r(A, lda, (int)n, R, ldr, t->stream), "tsqr_factor R");
        CUDA_TRY(mark(2), "tsqr_factor events");
        t->ev_recorded = timed;
        return finish(t, t->stream, "tsqr_factor");
    }
    CUDA_TRY(mark(0), "tsqr_factor events");
    CUDA_TRY(launch_chain_factor(ca, t->stream), "tsqr_factor leaves");
    CUDA_TRY(mark(1), "tsqr_factor events");
    if (t->pipe_count == 0) {
        if (R) CUDA_TRY(launch_extract_r(A, lda, (int)n, R, ldr, t->stream), "tsqr_factor R");
    } else {
        CUDA_TRY(launch_tree_pipe(A, lda, (int)n, t->d_row0, t->d_node_a, t->d_pipe_nodes, t->pipe_count, t->d_prod_l,
                                  t->d_prod_r, t->d_pipe_flags, t->d_tau_node, t->pipe_root, R, ldr,
                                  t->d_tcache_node, t->stream),
                 "tsqr_factor tree");
    }
    CUDA_TRY(mark(2), "tsqr_factor events");
    t->ev_recorded = timed;
    return finish(t, t->stream, "tsqr_factor");
}

tsqr_status_t tsqr_pack_r(tsqr_tree_t t, double *packed, void *stream) {
    NvtxRange nvtx_("tsqr_pack_r");
    if (!t || !t->A || !packed) return TSQR_ERR_INVALID;
    ENTER(t, (cudaStream_t)stream);
    CUDA_TRY(launch_pack_r(t->A, t->lda, (int)t->plan.n, packed, (cudaStream_t)stream), "tsqr_pack_r");
    return finish(t, (cudaStream_t)stream, "tsqr_pack_r");
}

tsqr_status_t tsqr_cross_factor(tsqr_tree_t t, int32_t round, const double *partner_packed, double *R,
                                int64_t ldr, void *stream) {
    NvtxRange nvtx_("tsqr_cross_factor");
    if (!t || !t->A || !partner_packed) return TSQR_ERR_INVALID;
    if (round != t->cross_done + 1 || round > t->cross_rounds) return TSQR_ERR_INVALID;
    if (R && ldr < t->plan.n) return TSQR_ERR_INVALID;
    int32_t partner, lower, role;
    if (tsqr_cross_partner(t->opts.nranks, t->opts.rank, round, &partner, &lower, &role) != TSQR_OK)
        return TSQR_ERR_INVALID;
    ENTER(t, (cudaStream_t)stream);
    const int n = (int)t->plan.n;
    if (t->wide) {
        tsqr_status_t ws = wide_tmp(t, n, (cudaStream_t)stream);
        if (ws != TSQR_OK) return ws;
        CUDA_TRY(launch_wide_cross_factor(t->A, t->lda, n, partner_packed, lower, t->d_wtmp,
                                          t->d_cross_y1 + (int64_t)(round - 1) * n * n,
                                          t->d_cross_tau + (int64_t)(round - 1) * n,
                                          t->d_cross_tcache + (int64_t)(round - 1) * t->npan * 64, R, ldr,
                                          (cudaStream_t)stream),
                 "tsqr_cross_factor");
    } else {
        CUDA_TRY(launch_cross_factor(t->NP, t->A, t->lda, n, partner_packed, lower,
                                     t->d_cross_y1 + (int64_t)(round - 1) * n * n,
                                     t->d_cross_tau + (int64_t)(round - 1) * n, R, ldr, (cudaStream_t)stream),
                 "tsqr_cross_factor");
    }
    t->cross_done = round;
    return finish(t, (cudaStream_t)stream, "tsqr_cross_factor");
}

// Packed R of rank group g at butterfly level r (ranks g*2^r .. (g+1)*2^r - 1) from the
// all-gathered leaf R's, by the same structured-combine kernels as the butterfly rounds
// (so bitwise the R the group's ranks hold after round r).  Slot: heap index (G >> r) + g.
static tsqr_status_t gathered_group_r(tsqr_tree_s *t, const double *all, int r, int g, const double **out,
                                      cudaStream_t st) {
    const int n = (int)t->plan.n, G = t->opts.nranks;
    const int64_t np = (int64_t)n * (n + 1) / 2;
    if (r == 0) {
        *out = all + (int64_t)g * np;
        return TSQR_OK;
    }
    const double *lo = nullptr, *hi = nullptr;
    tsqr_status_t s = gathered_group_r(t, all, r - 1, 2 * g, &lo, st);
    if (s == TSQR_OK) s = gathered_group_r(t, all, r - 1, 2 * g + 1, &hi, st);
    if (s != TSQR_OK) return s;
    double *scr = t->d_gather, *dst = t->d_gather + (int64_t)n * n + (int64_t)((G >> r) + g) * np;
    const int jr = t->cross_rounds;                 // the spare round slot takes the node factors
    CUDA_TRY(launch_unpack_r(lo, n, scr, n, st), "tsqr_cross_factor_gathered");
    if (t->wide) {
        CUDA_TRY(launch_wide_cross_factor(scr, n, n, hi, 1, t->d_wtmp, t->d_cross_y1 + (int64_t)jr * n * n,
                                          t->d_cross_tau + (int64_t)jr * n,
                                          t->d_cross_tcache + (int64_t)jr * t->npan * 64, nullptr, 0, st),
                 "tsqr_cross_factor_gathered");
    } else {
        CUDA_TRY(launch_cross_factor(t->NP, scr, n, n, hi, 1, t->d_cross_y1 + (int64_t)jr * n * n,
                                     t->d_cross_tau + (int64_t)jr * n, nullptr, 0, st),
                 "tsqr_cross_factor_gathered");
    }
    CUDA_TRY(launch_pack_r(scr, n, n, dst, st), "tsqr_cross_factor_gathered");
    *out = dst;
    return TSQR_OK;
}

tsqr_status_t tsqr_cross_factor_gathered(tsqr_tree_t t, const double *all_packed, double *R, int64_t ldr,
                                         void *stream) {
    NvtxRange nvtx_("tsqr_cross_factor_gathered");
    if (!t || !t->A || !all_packed) return TSQR_ERR_INVALID;
    if (t->cross_done != 0) return TSQR_ERR_INVALID;
    if (R && ldr < t->plan.n) return TSQR_ERR_INVALID;
    const int n = (int)t->plan.n, G = t->opts.nranks;
    cudaStream_t st = (cudaStream_t)stream;
    ENTER(t, st);
    if (t->cross_rounds == 0) {
        if (R) CUDA_TRY(launch_extract_r(t->A, t->lda, n, R, ldr, st), "tsqr_cross_factor_gathered");
        return finish(t, st, "tsqr_cross_factor_gathered");
    }
    if (!t->d_gather) {
        const size_t words = (size_t)n * n + (size_t)G * n * (n + 1) / 2;
        if (cudaMallocAsync((void **)&t->d_gather, sizeof(double) * words, st) != cudaSuccess) {
            cudaGetLastError();
            t->d_gather = nullptr;
            return TSQR_ERR_ALLOC;
        }
    }
    if (t->wide) {
        tsqr_status_t ws = wide_tmp(t, n, st);
        if (ws != TSQR_OK) return ws;
    }
    for (int r = 1; r <= t->cross_rounds; ++r) {
        // this rank's node of round r: its own R (the tree's current R) and the sibling group's
        const int sib = (t->opts.rank >> (r - 1)) ^ 1;
        const double *sp = nullptr;
        tsqr_status_t s = gathered_group_r(t, all_packed, r - 1, sib, &sp, st);
        if (s == TSQR_OK) s = tsqr_cross_factor(t, r, sp, r == t->cross_rounds ? R : nullptr, ldr, stream);
        if (s != TSQR_OK) return s;
    }
    return TSQR_OK;
}

tsqr_status_t tsqr_apply_qt(tsqr_tree_t t, double *C, int64_t ldc, int64_t k, double *top, int64_t ldtop,
                            void *stream) {
    NvtxRange nvtx_("tsqr_apply_qt");
    if (!t || !t->A) return TSQR_ERR_INVALID;
    if (k < 0 || k > INT32_MAX) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    if (!C || ldc < t->plan.m_local) return TSQR_ERR_INVALID;
    if (top && ldtop < t->plan.n) return TSQR_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    ENTER(t, st);
    ChainApplyArgs ca;
    ca.A = t->A; ca.lda = t->lda; ca.n = (int)t->plan.n; ca.chunk_rows = t->plan.c; ca.bulk = t->rows_even;
    ca.tile_row0 = t->d_row0; ca.tile_rows = t->d_rows; ca.tile_chunk0 = t->d_tile_chunk0;
    ca.cta_tile0 = t->d_apply_cta_tile0; ca.grid = t->apply_grid; ca.tcache = t->d_tcache;
    ca.C = C; ca.ldc = ldc; ca.k = (int)k; ca.forward = 1; ca.xbuf = nullptr;
    if (t->wide) {
        const int n = (int)t->plan.n;
        CUDA_TRY(launch_wide_apply_leaves(t->A, t->lda, n, t->d_row0, t->d_rows, t->plan.ntiles(),
                                          (int)t->plan.max_rows, t->d_tcache, t->d_tcache_pair, C, ldc, (int)k, 1,
                                          st),
                 "tsqr_apply_qt leaves");
        CUDA_TRY(node_stages(t, C, ldc, (int)k, true, 0, st), "tsqr_apply_qt nodes");
    } else {
        CUDA_TRY(launch_cs_apply(ca, st), "tsqr_apply_qt leaves");
        CUDA_TRY(node_stages(t, C, ldc, (int)k, true, 0, st), "tsqr_apply_qt nodes");
    }
    if (top) CUDA_TRY(launch_copy_block(C, ldc, top, ldtop, (int)t->plan.n, (int)k, st), "tsqr_apply_qt top");
    return finish(t, st, "tsqr_apply_qt");
}

tsqr_status_t tsqr_cross_apply_qt(tsqr_tree_t t, int32_t round, double *top, int64_t ldtop,
                                  const double *partner_top, double *C, int64_t ldc, int64_t k, void *stream) {
    NvtxRange nvtx_("tsqr_cross_apply_qt");
    if (!t || !t->A || !top || !partner_top) return TSQR_ERR_INVALID;
    if (round < 1 || round > t->cross_done) return TSQR_ERR_INVALID;
    if (k < 0 || k > INT32_MAX || ldtop < t->plan.n) return TSQR_ERR_INVALID;
    int32_t partner, lower, role;
    if (tsqr_cross_partner(t->opts.nranks, t->opts.rank, round, &partner, &lower, &role) != TSQR_OK)
        return TSQR_ERR_INVALID;
    if (role != 0 && (!C || ldc < t->plan.m_local)) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    ENTER(t, (cudaStream_t)stream);
    const int n = (int)t->plan.n;
    if (t->wide) {
        tsqr_status_t ws = wide_tmp(t, k, (cudaStream_t)stream);
        if (ws != TSQR_OK) return ws;
        CUDA_TRY(launch_wide_cross_apply(t->d_cross_y1 + (int64_t)(round - 1) * n * n,
                                         t->d_cross_tcache + (int64_t)(round - 1) * t->npan * 64, top, ldtop,
                                         partner_top, lower, role, C, ldc, n, (int)k, t->d_wtmp, 1,
                                         (cudaStream_t)stream),
                 "tsqr_cross_apply_qt");
    } else {
        CUDA_TRY(launch_cross_apply(t->NP, t->d_cross_y1 + (int64_t)(round - 1) * n * n,
                                    t->d_cross_tau + (int64_t)(round - 1) * n, top, ldtop, partner_top, lower, role,
                                    C, ldc, n, (int)k, 1, (cudaStream_t)stream),
                 "tsqr_cross_apply_qt");
    }
    return finish(t, (cudaStream_t)stream, "tsqr_cross_apply_qt");
}

tsqr_status_t tsqr_cross_apply_q(tsqr_tree_t t, int32_t round, double *top, int64_t ldtop,
                                 const double *partner_top, double *C, int64_t ldc, int64_t k, void *stream) {
    NvtxRange nvtx_("tsqr_cross_apply_q");
    if (!t || !t->A || !top || !partner_top) return TSQR_ERR_INVALID;
    if (round < 1 || round > t->cross_done) return TSQR_ERR_INVALID;
    if (k < 0 || k > INT32_MAX || ldtop < t->plan.n) return TSQR_ERR_INVALID;
    if (!C || ldc < t->plan.m_local) return TSQR_ERR_INVALID;
    int32_t partner, lower, role;
    if (tsqr_cross_partner(t->opts.nranks, t->opts.rank, round, &partner, &lower, &role) != TSQR_OK)
        return TSQR_ERR_INVALID;
    if (role == 0) return TSQR_ERR_INVALID;        // only the group heads take part in this round
    if (k == 0) return TSQR_OK;
    ENTER(t, (cudaStream_t)stream);
    const int n = (int)t->plan.n;
    if (t->wide) {
        tsqr_status_t ws = wide_tmp(t, k, (cudaStream_t)stream);
        if (ws != TSQR_OK) return ws;
        CUDA_TRY(launch_wide_cross_apply(t->d_cross_y1 + (int64_t)(round - 1) * n * n,
                                         t->d_cross_tcache + (int64_t)(round - 1) * t->npan * 64, top, ldtop,
                                         partner_top, lower, role, C, ldc, n, (int)k, t->d_wtmp, 0,
                                         (cudaStream_t)stream),
                 "tsqr_cross_apply_q");
    } else {
        CUDA_TRY(launch_cross_apply(t->NP, t->d_cross_y1 + (int64_t)(round - 1) * n * n,
                                    t->d_cross_tau + (int64_t)(round - 1) * n, top, ldtop, partner_top, lower, role,
                                    C, ldc, n, (int)k, 0, (cudaStream_t)stream),
                 "tsqr_cross_apply_q");
    }
    return finish(t, (cudaStream_t)stream, "tsqr_cross_apply_q");
}

tsqr_status_t tsqr_apply_q(tsqr_tree_t t, double *C, int64_t ldc, int64_t k, void *stream) {
    NvtxRange nvtx_("tsqr_apply_q");
    if (!t || !t->A) return TSQR_ERR_INVALID;
    if (k < 0 || k > INT32_MAX) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    if (!C || ldc < t->plan.m_local) return TSQR_ERR_INVALID;
    const int n = (int)t->plan.n;
    cudaStream_t st = (cudaStream_t)stream;
    ENTER(t, st);
    CUDA_TRY(node_stages(t, C, ldc, (int)k, false, 0, st), "tsqr_apply_q nodes");
    if (t->wide) {
        CUDA_TRY(launch_wide_apply_leaves(t->A, t->lda, n, t->d_row0, t->d_rows, t->plan.ntiles(),
                                          (int)t->plan.max_rows, t->d_tcache, t->d_tcache_pair, C, ldc, (int)k, 0, st),
                 "tsqr_apply_q leaves");
    } else {
        ChainApplyArgs ca;
        ca.A = t->A; ca.lda = t->lda; ca.n = n; ca.chunk_rows = t->plan.c; ca.bulk = t->rows_even; ca.bulk = t->rows_even;
        ca.tile_row0 = t->d_row0; ca.tile_rows = t->d_rows; ca.tile_chunk0 = t->d_tile_chunk0;
        ca.cta_tile0 = t->d_apply_cta_tile0; ca.grid = t->apply_grid; ca.tcache = t->d_tcache;
        ca.C = C; ca.ldc = ldc; ca.k = (int)k; ca.forward = 0; ca.xbuf = nullptr;
        CUDA_TRY(launch_cs_apply(ca, st), "tsqr_apply_q leaves");
    }
    return finish(t, st, "tsqr_apply_q");
}

tsqr_status_t tsqr_form_q(tsqr_tree_t t, double *Q, int64_t ldq, void *stream) {
    NvtxRange nvtx_("tsqr_form_q");
    if (!t || !t->A || !Q) return TSQR_ERR_INVALID;
    if (ldq < t->plan.m_local) return TSQR_ERR_INVALID;
    if (t->cross_done != t->cross_rounds) return TSQR_ERR_INVALID;
    const int n = (int)t->plan.n;
    const int L = t->plan.ntiles();
    cudaStream_t st = (cudaStream_t)stream;
    ENTER(t, st);
    if (!t->d_xbuf) {
        cudaError_t e = cudaMallocAsync((void **)&t->d_xbuf, sizeof(double) * (size_t)L * n * n, st);
        if (e != cudaSuccess) {
            t->d_xbuf = nullptr;
            cudaGetLastError();
            g_last_error = std::string("tsqr_form_q alloc: ") + cudaGetErrorString(e);
            return TSQR_ERR_ALLOC;
        }
    }
    if (t->wide) {
        tsqr_status_t ws = wide_tmp(t, n, st);
        if (ws != TSQR_OK) return ws;
        CUDA_TRY(cudaMemsetAsync(t->d_xbuf, 0, sizeof(double) * (size_t)L * n * n, st), "tsqr_form_q");
        CUDA_TRY(launch_wide_cross_root_x(t->d_cross_y1, t->d_cross_tcache, (int64_t)t->npan * 64, t->cross_rounds,
                                          t->opts.rank, n, t->d_wtmp, t->d_xbuf, st),
                 "tsqr_form_q root");
        CUDA_TRY(node_stages(t, t->d_xbuf, n, n, false, 1, st), "tsqr_form_q nodes");
        CUDA_TRY(launch_wide_formq_init(t->d_row0, t->d_rows, L, n, t->d_xbuf, Q, ldq, st), "tsqr_form_q");
        CUDA_TRY(launch_wide_apply_leaves(t->A, t->lda, n, t->d_row0, t->d_rows, L, (int)t->plan.max_rows,
                                          t->d_tcache, t->d_tcache_pair, Q, ldq, n, 0, st),
                 "tsqr_form_q leaves");
        return finish(t, st, "tsqr_form_q");
    }
    // root X of this rank: I (one GPU) or the butterfly path (no communication)
    // the node stages read X_b = 0 below every subtree's X ([X; 0])
    if (L > 1) CUDA_TRY(cudaMemsetAsync(t->d_xbuf, 0, sizeof(double) * (size_t)L * n * n, st), "tsqr_form_q");
    if (t->cross_rounds == 0) CUDA_TRY(launch_identity(t->d_xbuf, n, st), "tsqr_form_q identity");
    else
        CUDA_TRY(launch_cross_root_x(t->NP, t->d_cross_y1, t->d_cross_tau, t->cross_rounds, t->opts.rank, n,
                                     t->d_xbuf, st),
                 "tsqr_form_q root");
    CUDA_TRY(node_stages(t, t->d_xbuf, n, n, false, 1, st), "tsqr_form_q nodes");
    ChainApplyArgs ca;
    ca.A = t->A; ca.lda = t->lda; ca.n = n; ca.chunk_rows = t->plan.c; ca.bulk = t->rows_even;
    ca.tile_row0 = t->d_row0; ca.tile_rows = t->d_rows; ca.tile_chunk0 = t->d_tile_chunk0;
    ca.cta_tile0 = t->d_apply_cta_tile0; ca.grid = t->apply_grid; ca.tcache = t->d_tcache;
    ca.C = Q; ca.ldc = ldq; ca.k = n; ca.forward = 0; ca.xbuf = t->d_xbuf;
    CUDA_TRY(launch_cs_apply(ca, st), "tsqr_form_q leaves");
    return finish(t, st, "tsqr_form_q");
}

tsqr_status_t tsqr_tree_free(tsqr_tree_t t) {
    if (!t) return TSQR_OK;
    // stream-ordered: the memory is released behind the tree's last call on its stream
    // (no host synchronisation); events are destroyed once their work completes
    for (cudaEvent_t &e : t->ev)
        if (e) cudaEventDestroy(e);
    if (t->done) cudaEventDestroy(t->done);
    free_tree_memory(t, t->stream);
    delete t;
    return TSQR_OK;
}

tsqr_status_t tsqr_tree_stage_ms(tsqr_tree_t t, float *leaf_ms, float *tree_ms) {
    if (!t || !t->ev_recorded) return TSQR_ERR_INVALID;
    CUDA_TRY(cudaEventSynchronize(t->ev[2]), "tsqr_tree_stage_ms");
    float a = 0.f, b = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&a, t->ev[0], t->ev[1]), "tsqr_tree_stage_ms");
    CUDA_TRY(cudaEventElapsedTime(&b, t->ev[1], t->ev[2]), "tsqr_tree_stage_ms");
    if (leaf_ms) *leaf_ms = a;
    if (tree_ms) *tree_ms = b;
    return TSQR_OK;
}

tsqr_status_t tsqr_tree_export_tau(tsqr_tree_t t, double *tau_tile_host, double *tau_node_host) {
    if (!t) return TSQR_ERR_INVALID;
    const size_t bytes = sizeof(double) * (size_t)t->plan.ntiles() * t->plan.n;
    const size_t cbytes = sizeof(double) * (size_t)t->nchunks * t->plan.n;
    if (t->stream) CUDA_TRY(cudaStreamSynchronize(t->stream), "tsqr_tree_export_tau");
    if (tau_tile_host) CUDA_TRY(cudaMemcpy(tau_tile_host, t->d_tau_chunk, cbytes, cudaMemcpyDeviceToHost), "export");
    if (tau_node_host) CUDA_TRY(cudaMemcpy(tau_node_host, t->d_tau_node, bytes, cudaMemcpyDeviceToHost), "export");
    return TSQR_OK;
}

}  // extern "C"

// --------------------------------------------------- tree state (streamed Q)
// The device arrays that, with the reflectors in A, make up a local tree's implicit
// Q (everything tsqr_apply_qt / tsqr_apply_q / tsqr_form_q read): chunk and node taus
// and the cached panel T's.  tsqr_stream.cu keeps them in host memory per slab
// ([TR] Alg. sequential TSQR P:1725-1753: "write Q factors to slow memory").
namespace {
struct StateArr {
    double *p;
    size_t words;
};
// the chain engine's chunk T cache (a fifth of Y's size at n = 64) is left out of the
// compact state: tree_rebuild_tcache recomputes it from Y and the chunk taus
std::vector<StateArr> state_arrays(const tsqr_tree_s *t, bool full) {
    const int64_t L = t->plan.ntiles(), n = t->plan.n;
    const int ncb_cache = t->wide ? t->npan : chain_ncb((int)n);
    std::vector<StateArr> v = {{t->d_tau_chunk, (size_t)(t->nchunks * n)},
                               {t->d_tau_node, (size_t)(L * n)},
                               {t->d_tcache_node, (size_t)(L * t->npan * 64)}};
    if (full || t->wide) v.push_back({t->d_tcache, (size_t)(t->nchunks * ncb_cache * 64)});
    if (t->wide) v.push_back({t->d_tcache_pair, (size_t)(L * ((t->npan + 1) / 2) * 64)});
    return v;
}
}  // namespace

size_t tsqr::tree_state_words(const tsqr_tree_s *t, bool full) {
    size_t w = 0;
    for (const StateArr &a : state_arrays(t, full)) w += a.words;
    return w;
}

tsqr_status_t tsqr::tree_state_words_for(int64_t m_local, int64_t n, const tsqr_opts_t *opts, bool full,
                                         size_t *words) {
    Plan p;
    tsqr_opts_t ro;
    int rc;
    try { rc = plan_for(m_local, n, opts, &p, &ro); } catch (const std::bad_alloc &) { return TSQR_ERR_ALLOC; }
    if (rc) return (tsqr_status_t)rc;
    const int64_t L = p.ntiles(), nchunks = p.tile_chunk0[L], npan = (n + 7) / 8;
    const bool wide = n > 64;
    const int64_t ncb_cache = wide ? npan : chain_ncb((int)n);
    size_t w = (size_t)(nchunks * n + L * n + L * npan * 64);
    if (full || wide) w += (size_t)(nchunks * ncb_cache * 64);
    if (wide) w += (size_t)(L * ((npan + 1) / 2) * 64);
    *words = w;
    return TSQR_OK;
}

cudaError_t tsqr::tree_state_copy(tsqr_tree_s *t, double *host, bool to_host, bool full, cudaStream_t st) {
    size_t off = 0;
    for (const StateArr &a : state_arrays(t, full)) {
        const cudaError_t e = to_host
            ? cudaMemcpyAsync(host + off, a.p, sizeof(double) * a.words, cudaMemcpyDeviceToHost, st)
            : cudaMemcpyAsync(a.p, host + off, sizeof(double) * a.words, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return e;
        off += a.words;
    }
    return cudaSuccess;
}

cudaError_t tsqr::tree_rebuild_tcache(tsqr_tree_s *t, cudaStream_t st) {
    if (t->wide) return cudaSuccess;                // the compact state of a wide tree is complete
    return launch_chain_rebuild_t(t->A, t->lda, (int)t->plan.n, t->d_row0, t->d_rows, t->d_tile_chunk0,
                                  t->plan.ntiles(), t->nchunks, t->d_tau_chunk, t->d_tcache, st);
}

tsqr_status_t tsqr::tree_bind(int64_t m_local, int64_t n, double *A, int64_t lda, const tsqr_opts_t *opts,
                              cudaStream_t st, tsqr_tree_s **tree) {
    // a tree for the plan of (m_local, n, opts) bound to the reflectors in A, without
    // factoring (its state is imported next); an existing handle of the same plan is kept
    tsqr_tree_s *t = *tree;
    const tsqr_opts_t ro = resolve_opts(m_local, opts);
    const bool reuse = t && t->plan.m_local == m_local && t->plan.n == n && t->opts.block_rows == ro.block_rows &&
                       (ro.tile_rows == 0 || t->plan.s == ro.tile_rows) && t->opts.nranks == ro.nranks;
    if (!reuse) {
        if (t) {
            t->stream = st;
            tsqr_tree_free(t);
        }
        t = nullptr;
        const tsqr_status_t s = create_tree(m_local, n, A, lda, opts, st, &t);
        if (s != TSQR_OK) return s;
        *tree = t;
    } else {
        ENTER(t, st);
    }
    t->A = A;
    t->lda = lda;
    t->stream = st;
    t->cross_done = 0;
    return TSQR_OK;
}


// ------------------------------------------------- pipelined host path (e2e)
// tsqr_qr_host with a HOST A and the explicit Q (n <= 64, one rank): the tiles are cut
// into S slabs of whole tiles; slab k's rows go host->device on `up` and its leaves are
// factored on `st` as soon as they land (the leaf QRs are independent, Eq. 1),
// so the copy-in hides the leaf stage; then the tree and the form-Q node stages; then slab
// k's form-Q leaves and its Q rows device->host on `down`, so the copy-out hides the
// leaf stage of form Q.  Same kernels, same plan, same results as tsqr_factor +
// tsqr_form_q (the CTA partition of the leaf kernels is per slab; no kernel's arithmetic
// depends on it).
tsqr_status_t tsqr::qr_host_pipelined(tsqr_tree_s **tree, int64_t m, int64_t n, const double *A, int64_t lda,
                                      double *dA, double *dR, double *dQ, double *R, int64_t ldr, double *Q,
                                      int64_t ldq, const tsqr_opts_t *opts, cudaStream_t st, cudaStream_t up,
                                      cudaStream_t down, int S) {
    if (n > 64 || (opts && opts->nranks > 1)) return TSQR_ERR_UNSUPPORTED;
    // the tree of the plan, bound to dA (lda = m), exactly as tsqr_factor prepares it
    {
        Plan p;
        tsqr_opts_t ro;
        int rc;
        try { rc = plan_for(m, n, opts, &p, &ro); } catch (const std::bad_alloc &) { return TSQR_ERR_ALLOC; }
        if (rc) return (tsqr_status_t)rc;
    }
    tsqr_status_t s = tree_bind(m, n, dA, m, opts, st, tree);
    if (s != TSQR_OK) return s;
    tsqr_tree_s *t = *tree;
    const int L = t->plan.ntiles();
    S = std::max(1, std::min(S, L));
    const Plan &p = t->plan;
    if (t->slab_S != S || !t->d_slab_part) {       // the slabs' CTA partitions, once per (tree, S)
        t->slab_t0.assign(S + 1, L);
        const int64_t per = (m + S - 1) / S;
        int tt = 0;
        for (int k = 0; k < S; ++k) {
            t->slab_t0[k] = tt;
            while (tt < L && (p.tile_row0[tt] + p.tile_rows[tt] <= (int64_t)(k + 1) * per || k == S - 1)) ++tt;
        }
        t->slab_t0[S] = L;
        std::vector<int> all;
        t->slab_grid.assign(2 * S, 0);
        t->slab_off.assign(2 * S, 0);
        for (int pass = 0; pass < 2; ++pass)
            for (int k = 0; k < S; ++k) {
                const int a = t->slab_t0[k], b = t->slab_t0[k + 1];
                std::vector<int64_t> rows(p.tile_rows.begin() + a, p.tile_rows.begin() + b);
                const int g = std::max(1, std::min(b - a, pass == 0 ? chain_grid((int)n) : cs_apply_grid((int)n)));
                std::vector<int> part;
                if (b > a) chain_partition(rows, p.c, g, part);
                else part.assign(g + 1, 0);
                t->slab_grid[pass * S + k] = b > a ? g : 0;
                t->slab_off[pass * S + k] = (int)all.size();
                for (int v : part) all.push_back(v + a);
            }
        if (t->d_slab_part) cudaFreeAsync(t->d_slab_part, st);
        t->d_slab_part = nullptr;
        CUDA_TRY(cudaMallocAsync((void **)&t->d_slab_part, sizeof(int) * all.size(), st), "tsqr_qr_host slabs");
        CUDA_TRY(cudaMemcpyAsync(t->d_slab_part, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice, st),
                 "tsqr_qr_host slabs");
        CUDA_TRY(cudaStreamSynchronize(st), "tsqr_qr_host slabs");   // the pageable source goes out of scope
        t->slab_S = S;
    }
    std::vector<cudaEvent_t> ev(2 * S + 1, nullptr);
    struct EvGuard {
        std::vector<cudaEvent_t> &v;
        ~EvGuard() {
            for (cudaEvent_t e : v)
                if (e) cudaEventDestroy(e);
        }
    } guard{ev};
    for (cudaEvent_t &e : ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "tsqr_qr_host events");
    const size_t D = sizeof(double);
    // the side streams start behind the work already on st (allocations, the partition upload)
    CUDA_TRY(cudaEventRecord(ev[2 * S], st), "tsqr_qr_host");
    CUDA_TRY(cudaStreamWaitEvent(up, ev[2 * S], 0), "tsqr_qr_host");
    CUDA_TRY(cudaStreamWaitEvent(down, ev[2 * S], 0), "tsqr_qr_host");
    auto slab_rows = [&](int k, int64_t *r0, int64_t *rows) {
        const int a = t->slab_t0[k], b = t->slab_t0[k + 1];
        *r0 = a < L ? p.tile_row0[a] : m;
        *rows = (b > a) ? p.tile_row0[b - 1] + p.tile_rows[b - 1] - *r0 : 0;
    };
    for (int k = 0; k < S; ++k) {                  // copy-in, slab by slab
        int64_t r0, rows;
        slab_rows(k, &r0, &rows);
        if (rows > 0)
            CUDA_TRY(cudaMemcpy2DAsync(dA + r0, D * m, A + r0, D * lda, D * rows, n, cudaMemcpyHostToDevice, up),
                     "tsqr_qr_host copy in");
        CUDA_TRY(cudaEventRecord(ev[k], up), "tsqr_qr_host");
    }
    t->opts.flags = resolve_opts(m, opts).flags & ~2;
    t->ev_recorded = false;
    ChainArgs ca;
    ca.A = dA; ca.lda = m; ca.n = (int)n; ca.m = t->rows_even ? m : 0; ca.chunk_rows = p.c;
    ca.tile_row0 = t->d_row0; ca.tile_rows = t->d_rows; ca.tile_chunk0 = t->d_tile_chunk0;
    ca.tau = t->d_tau_chunk; ca.tcache = t->d_tcache; ca.robust = (t->opts.flags & TSQR_FLAG_ROBUST) != 0;
    for (int k = 0; k < S; ++k) {                  // each slab's leaves as soon as it has landed
        CUDA_TRY(cudaStreamWaitEvent(st, ev[k], 0), "tsqr_qr_host");
        if (t->slab_grid[k] == 0) continue;
        ca.cta_tile0 = t->d_slab_part + t->slab_off[k];
        ca.grid = t->slab_grid[k];
        CUDA_TRY(launch_chain_factor(ca, st), "tsqr_qr_host leaves");
    }
    if (t->pipe_count == 0) CUDA_TRY(launch_extract_r(dA, m, (int)n, dR, n, st), "tsqr_qr_host R");
    else
        CUDA_TRY(launch_tree_pipe(dA, m, (int)n, t->d_row0, t->d_node_a, t->d_pipe_nodes, t->pipe_count, t->d_prod_l,
                                  t->d_prod_r, t->d_pipe_flags, t->d_tau_node, t->pipe_root, dR, n, t->d_tcache_node,
                                  st),
                 "tsqr_qr_host tree");
    // form Q: the root X = I, the node stages, then slab by slab the leaves and the copy-out
    if (!t->d_xbuf) CUDA_TRY(cudaMallocAsync((void **)&t->d_xbuf, D * (size_t)L * n * n, st), "tsqr_qr_host xbuf");
    if (L > 1) CUDA_TRY(cudaMemsetAsync(t->d_xbuf, 0, D * (size_t)L * n * n, st), "tsqr_qr_host");
    CUDA_TRY(launch_identity(t->d_xbuf, (int)n, st), "tsqr_qr_host identity");
    CUDA_TRY(node_stages(t, t->d_xbuf, n, (int)n, false, 1, st), "tsqr_qr_host nodes");
    ChainApplyArgs qa;
    qa.A = dA; qa.lda = m; qa.n = (int)n; qa.chunk_rows = p.c; qa.bulk = t->rows_even;
    qa.tile_row0 = t->d_row0; qa.tile_rows = t->d_rows; qa.tile_chunk0 = t->d_tile_chunk0; qa.tcache = t->d_tcache;
    qa.C = dQ; qa.ldc = m; qa.k = (int)n; qa.forward = 0; qa.xbuf = t->d_xbuf;
    for (int k = 0; k < S; ++k) {
        int64_t r0, rows;
        slab_rows(k, &r0, &rows);
        if (t->slab_grid[S + k] > 0) {
            qa.cta_tile0 = t->d_slab_part + t->slab_off[S + k];
            qa.grid = t->slab_grid[S + k];
            CUDA_TRY(launch_cs_apply(qa, st), "tsqr_qr_host form Q leaves");
        }
        CUDA_TRY(cudaEventRecord(ev[S + k], st), "tsqr_qr_host");
        CUDA_TRY(cudaStreamWaitEvent(down, ev[S + k], 0), "tsqr_qr_host");
        if (rows > 0)
            CUDA_TRY(cudaMemcpy2DAsync(Q + r0, D * ldq, dQ + r0, D * m, D * rows, n, cudaMemcpyDeviceToHost, down),
                     "tsqr_qr_host copy out");
    }
    CUDA_TRY(cudaMemcpy2DAsync(R, D * ldr, dR, D * n, D * n, n, cudaMemcpyDeviceToHost, st), "tsqr_qr_host R out");
    CUDA_TRY(cudaEventRecord(ev[2 * S], down), "tsqr_qr_host");
    CUDA_TRY(cudaStreamWaitEvent(st, ev[2 * S], 0), "tsqr_qr_host");
    s = leave(t, st);
    if (s != TSQR_OK) return s;
    CUDA_TRY(cudaStreamSynchronize(st), "tsqr_qr_host");
    return TSQR_OK;
}
