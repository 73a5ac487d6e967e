// Sequential (out-of-HBM) TSQR: R of a host-resident m x n
// matrix streamed through the GPU in row slabs -- a flat tree over the slabs
// ([TR] Alg. sequential TSQR P:1725-1753; flat tree P:954-993; the B200 analogue
// of the paper's out-of-DRAM experiment, model Eq. 6): each slab is
// factored on the device by the parallel TSQR (tsqr_factor), then the running R
// absorbs it by the structured combine of [R; R_slab] (Alg. QR:qnxn, q = 2; the
// same kernels as the butterfly rounds).  Slab k+1's host->device copy runs on a
// copy stream while slab k is factored; the factored slab (its reflectors) can be
// copied back to the host.  tsqr_factor_streamed_q also keeps the rest of the
// implicit Q in host memory -- each slab tree's taus and cached T's and each
// flat-tree node's factors ("write Q factors to slow memory", Alg. TSQR:seq) -- so
// that Q^T C, Q C and the explicit Q of a host-resident matrix stream through the
// GPU slab by slab afterwards (tsqr_streamed_*).  Product code.
#include "../../include/tsqr.h"
#include "plan.h"
#include "tsqr_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

using namespace tsqr;

namespace {

struct Slab {
    int64_t r0, rows;
};

// R6 at slab granularity: slabs of slab_rows; a remainder of fewer than n rows joins the last.
std::vector<Slab> slabs_of(int64_t m, int64_t n, int64_t s) {
    std::vector<Slab> out;
    const int64_t full = m / s, rem = m % s;
    if (full == 0) return {Slab{0, m}};
    for (int64_t k = 0; k < full; ++k) out.push_back(Slab{k * s, s});
    if (rem >= n) out.push_back(Slab{full * s, rem});
    else if (rem) out.back().rows += rem;
    return out;
}

struct Res {
    cudaStream_t copy = nullptr, down = nullptr;          // host->device, device->host (full duplex)
    cudaEvent_t loaded[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr};
    double *slab[2] = {nullptr, nullptr};
    double *rk = nullptr, *run = nullptr, *packed = nullptr, *y1 = nullptr, *tau = nullptr, *tc = nullptr,
           *wtmp = nullptr, *nodes = nullptr;
    tsqr_tree_t tree[2] = {nullptr, nullptr};
    ~Res() {
        if (copy) cudaStreamSynchronize(copy);
        if (down) cudaStreamSynchronize(down);
        for (int i = 0; i < 2; ++i) {
            if (tree[i]) tsqr_tree_free(tree[i]);
            if (slab[i]) cudaFree(slab[i]);
            if (loaded[i]) cudaEventDestroy(loaded[i]);
            if (used[i]) cudaEventDestroy(used[i]);
        }
        for (double *p : {rk, run, packed, y1, tau, tc, wtmp, nodes})
            if (p) cudaFree(p);
        if (copy) cudaStreamDestroy(copy);
        if (down) cudaStreamDestroy(down);
    }
};

}  // namespace

// The implicit Q of a streamed factor, kept in host memory (the reflectors are the
// caller's Y): per slab, its tree's state (tree_state_copy); per flat-tree node
// k >= 1 (the combine of [R_{0..k-1}; R_k]), Y1 (n x n), tau (n) and the panel T's.
struct tsqr_stream_tree_s {
    int64_t m = 0, n = 0;
    tsqr_opts_t o{};
    std::vector<Slab> sl;
    const double *Y = nullptr;
    int64_t ldy = 0;
    double *host = nullptr;                  // pinned: every slab's compact tree state, then the nodes
    std::vector<size_t> state_off;           // slab k's state at host + state_off[k]
    double *nodes = nullptr;                 // node k at nodes + (k - 1) * node_words
    size_t node_words = 0;
    ~tsqr_stream_tree_s() {
        if (host) cudaFreeHost(host);
    }
};

#define S_TRY(expr)                                          \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) {                             \
            cudaGetLastError();                              \
            set_last_error("tsqr_factor_streamed", _e);      \
            return _e == cudaErrorMemoryAllocation ? TSQR_ERR_ALLOC : TSQR_ERR_CUDA; \
        }                                                    \
    } while (0)

extern "C" {

static tsqr_status_t factor_streamed_impl(int64_t m, int64_t n, const double *A, int64_t lda, int64_t slab_rows,
                                          double *Y, int64_t ldy, double *R, int64_t ldr, const tsqr_opts_t *opts,
                                          void *stream, tsqr_stream_tree_s *keep) {
    if (!A || !R) return TSQR_ERR_INVALID;
    if (n < 1 || m < n) return TSQR_ERR_SHAPE;
    if (n > TSQR_MAX_N) return TSQR_ERR_UNSUPPORTED;
    if (lda < m || ldr < n || slab_rows < n || (Y && ldy < m)) return TSQR_ERR_INVALID;
    tsqr_opts_t o{};
    if (opts) o = *opts;
    if (o.nranks > 1) return TSQR_ERR_UNSUPPORTED;
    o.nranks = 1;
    o.rank = 0;
    const std::vector<Slab> sl = slabs_of(m, n, slab_rows);
    // every slab's plan must be valid before anything is enqueued
    for (const Slab &s : sl) {
        tsqr_plan_info_t info;
        tsqr_status_t ps = tsqr_plan_info(s.rows, n, &o, &info);
        if (ps != TSQR_OK) return ps;
    }
    int64_t maxrows = 0;
    for (const Slab &s : sl) maxrows = s.rows > maxrows ? s.rows : maxrows;
    cudaStream_t st = (cudaStream_t)stream;
    Res r;
    S_TRY(cudaStreamCreateWithFlags(&r.copy, cudaStreamNonBlocking));
    S_TRY(cudaStreamCreateWithFlags(&r.down, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        S_TRY(cudaEventCreateWithFlags(&r.loaded[i], cudaEventDisableTiming));
        S_TRY(cudaEventCreateWithFlags(&r.used[i], cudaEventDisableTiming));
        if (i < (int)sl.size()) S_TRY(cudaMalloc((void **)&r.slab[i], sizeof(double) * maxrows * n));
    }
    const int npan = (int)((n + 7) / 8);
    S_TRY(cudaMalloc((void **)&r.rk, sizeof(double) * n * n));
    S_TRY(cudaMalloc((void **)&r.run, sizeof(double) * n * n));
    S_TRY(cudaMalloc((void **)&r.packed, sizeof(double) * n * (n + 1) / 2));
    S_TRY(cudaMalloc((void **)&r.y1, sizeof(double) * n * n));
    S_TRY(cudaMalloc((void **)&r.tau, sizeof(double) * n));
    S_TRY(cudaMalloc((void **)&r.tc, sizeof(double) * npan * 64));
    S_TRY(cudaMalloc((void **)&r.wtmp, sizeof(double) * 2 * n * n));
    if (keep) {
        keep->m = m;
        keep->n = n;
        keep->o = o;
        keep->sl = sl;
        keep->Y = Y;
        keep->ldy = ldy;
        // one page-locked block for the whole Q state, sized from the slabs' plans: the
        // compact tree states (taus + node T's; the chunk T's are rebuilt on use) and the nodes
        keep->state_off.assign(sl.size() + 1, 0);
        for (size_t k = 0; k < sl.size(); ++k) {
            size_t w = 0;
            const tsqr_status_t ws = tree_state_words_for(sl[k].rows, n, &o, false, &w);
            if (ws != TSQR_OK) return ws;
            keep->state_off[k + 1] = keep->state_off[k] + w;
        }
        keep->node_words = (size_t)(n * n + n + npan * 64);
        const size_t total = keep->state_off[sl.size()] + keep->node_words * (sl.size() - 1);
        S_TRY(cudaMallocHost((void **)&keep->host, sizeof(double) * std::max<size_t>(total, 1)));
        keep->nodes = keep->host + keep->state_off[sl.size()];
        if (sl.size() > 1) S_TRY(cudaMalloc((void **)&r.nodes, sizeof(double) * keep->node_words * (sl.size() - 1)));
    }
    // the copy stream starts after the work already queued on `stream`
    S_TRY(cudaEventRecord(r.used[0], st));
    S_TRY(cudaStreamWaitEvent(r.copy, r.used[0], 0));
    auto load = [&](size_t k) -> cudaError_t {
        const int b = (int)(k & 1);
        cudaError_t e = cudaMemcpy2DAsync(r.slab[b], sizeof(double) * sl[k].rows, A + sl[k].r0, sizeof(double) * lda,
                                          sizeof(double) * sl[k].rows, n, cudaMemcpyHostToDevice, r.copy);
        if (e == cudaSuccess) e = cudaEventRecord(r.loaded[b], r.copy);
        return e;
    };
    S_TRY(load(0));
    for (size_t k = 0; k < sl.size(); ++k) {
        const int b = (int)(k & 1);
        if (k + 1 < sl.size()) {
            // slab k+1 goes into the other buffer once slab k-1 (its last user) is done
            if (k >= 1) S_TRY(cudaStreamWaitEvent(r.copy, r.used[b ^ 1], 0));
            S_TRY(load(k + 1));
        }
        S_TRY(cudaStreamWaitEvent(st, r.loaded[b], 0));
        // reuse the buffer's tree when the slab has the same height (all but possibly the last)
        if (r.tree[b] && k + 1 == sl.size() && sl[k].rows != sl[0].rows) {
            tsqr_tree_free(r.tree[b]);
            r.tree[b] = nullptr;
        }
        tsqr_status_t s = tsqr_factor(sl[k].rows, n, r.slab[b], sl[k].rows, k == 0 ? r.run : r.rk, n, &o, stream,
                                      &r.tree[b]);
        if (s != TSQR_OK) return s;
        if (k > 0) {
            // R <- structured QR of [R; R_k] (the running R covers the earlier rows: on top)
            S_TRY(launch_pack_r(r.rk, n, (int)n, r.packed, st));
            if (n > 64) S_TRY(launch_wide_cross_factor(r.run, n, (int)n, r.packed, 1, r.wtmp, r.y1, r.tau, r.tc,
                                                       nullptr, 0, st));
            else S_TRY(launch_cross_factor(padded_width(n), r.run, n, (int)n, r.packed, 1, r.y1, r.tau, nullptr, 0,
                                           st));
            if (keep) {                         // node k's factors into its device slot (kernels, on st)
                double *h = r.nodes + (k - 1) * keep->node_words;
                S_TRY(launch_copy_block(r.y1, n * n, h, n * n, (int)(n * n), 1, st));
                S_TRY(launch_copy_block(r.tau, n, h + n * n, n, (int)n, 1, st));
                if (n > 64) S_TRY(launch_copy_block(r.tc, npan * 64, h + n * n + n, npan * 64, npan * 64, 1, st));
            }
        }
        if (Y) {
            // the factored slab (reflectors below each tile's diagonal) back to the host, and
            // with keep the tree's compact state and the node, all on the device->host stream
            // (a copy on st would queue behind them in the copy engine and stall the factor)
            S_TRY(cudaEventRecord(r.used[b], st));
            S_TRY(cudaStreamWaitEvent(r.down, r.used[b], 0));
            S_TRY(cudaMemcpy2DAsync(Y + sl[k].r0, sizeof(double) * ldy, r.slab[b], sizeof(double) * sl[k].rows,
                                    sizeof(double) * sl[k].rows, n, cudaMemcpyDeviceToHost, r.down));
            if (keep) {
                S_TRY(tree_state_copy(r.tree[b], keep->host + keep->state_off[k], true, false, r.down));
                if (k > 0)
                    S_TRY(cudaMemcpyAsync(keep->nodes + (k - 1) * keep->node_words, r.nodes + (k - 1) * keep->node_words,
                                          sizeof(double) * keep->node_words, cudaMemcpyDeviceToHost, r.down));
            }
            S_TRY(cudaEventRecord(r.used[b], r.down));
        } else {
            S_TRY(cudaEventRecord(r.used[b], st));
        }
    }
    S_TRY(launch_copy_block(r.run, n, R, ldr, (int)n, (int)n, st));
    S_TRY(cudaStreamWaitEvent(st, r.used[(sl.size() - 1) & 1], 0));
    S_TRY(cudaStreamSynchronize(st));
    return TSQR_OK;
}

tsqr_status_t tsqr_factor_streamed(int64_t m, int64_t n, const double *A, int64_t lda, int64_t slab_rows,
                                   double *Y, int64_t ldy, double *R, int64_t ldr, const tsqr_opts_t *opts,
                                   void *stream) {
    return factor_streamed_impl(m, n, A, lda, slab_rows, Y, ldy, R, ldr, opts, stream, nullptr);
}

tsqr_status_t tsqr_factor_streamed_q(int64_t m, int64_t n, const double *A, int64_t lda, int64_t slab_rows,
                                     double *Y, int64_t ldy, double *R, int64_t ldr, const tsqr_opts_t *opts,
                                     void *stream, tsqr_stream_tree_t *out) {
    if (!out || !Y) return TSQR_ERR_INVALID;
    tsqr_stream_tree_s *h = new (std::nothrow) tsqr_stream_tree_s();
    if (!h) return TSQR_ERR_ALLOC;
    const tsqr_status_t s = factor_streamed_impl(m, n, A, lda, slab_rows, Y, ldy, R, ldr, opts, stream, h);
    if (s != TSQR_OK) {
        delete h;
        return s;
    }
    if (*out) delete *out;
    *out = h;
    return TSQR_OK;
}

tsqr_status_t tsqr_stream_tree_free(tsqr_stream_tree_t t) {
    delete t;
    return TSQR_OK;
}

// Q^T C (forward), Q C (!forward) or, with formq, Q [I; 0] of a streamed factor on a
// HOST matrix, slab by slab.  Forward: slab k's local tree (tsqr_apply_qt), then node
// k on [top; slab head] (the running top is the earlier rows: lower); Q C: the reverse,
// nodes S-1 .. 1 split [top; slab head] into both halves, then each slab's tree.
// Pipelined over two device buffers and three streams: slab j+1's Y and C come in on
// `up` and slab j-1's result goes out on `down` while slab j is computed on `st`
// (host links are full duplex), so the call runs at about max(bytes in, bytes out)
// over the link.
static tsqr_status_t streamed_apply(tsqr_stream_tree_s *t, double *C, int64_t ldc, int64_t k, bool forward,
                                    bool formq, double *top_out, int64_t ldtop, cudaStream_t st) {
    const int64_t n = t->n;
    int64_t maxrows = 0;
    for (const Slab &s : t->sl) maxrows = std::max(maxrows, s.rows);
    struct Dev {
        double *yb[2] = {nullptr, nullptr}, *cb[2] = {nullptr, nullptr};
        double *top = nullptr, *ta = nullptr, *tb = nullptr, *node[2] = {nullptr, nullptr}, *wtmp = nullptr;
        tsqr_tree_t tree[2] = {nullptr, nullptr};
        cudaStream_t st = nullptr, up = nullptr, down = nullptr;
        cudaEvent_t loaded[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
        ~Dev() {
            if (up) cudaStreamSynchronize(up);
            if (down) cudaStreamSynchronize(down);
            if (st) cudaStreamSynchronize(st);
            for (tsqr_tree_t &x : tree)
                if (x) tsqr_tree_free(x);
            for (double *p : {yb[0], yb[1], cb[0], cb[1], top, ta, tb, node[0], node[1], wtmp})
                if (p) cudaFreeAsync(p, st);
            for (int i = 0; i < 2; ++i)
                for (cudaEvent_t e : {loaded[i], done[i], freed[i]})
                    if (e) cudaEventDestroy(e);
            if (up) cudaStreamDestroy(up);
            if (down) cudaStreamDestroy(down);
        }
    } d;
    d.st = st;
    const int64_t kw = std::max<int64_t>(k, n);
    S_TRY(cudaStreamCreateWithFlags(&d.up, cudaStreamNonBlocking));
    S_TRY(cudaStreamCreateWithFlags(&d.down, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        S_TRY(cudaEventCreateWithFlags(&d.loaded[i], cudaEventDisableTiming));
        S_TRY(cudaEventCreateWithFlags(&d.done[i], cudaEventDisableTiming));
        S_TRY(cudaEventCreateWithFlags(&d.freed[i], cudaEventDisableTiming));
        S_TRY(cudaMallocAsync((void **)&d.yb[i], sizeof(double) * maxrows * n, st));
        S_TRY(cudaMallocAsync((void **)&d.cb[i], sizeof(double) * maxrows * k, st));
        S_TRY(cudaMallocAsync((void **)&d.node[i], sizeof(double) * t->node_words, st));
    }
    S_TRY(cudaMallocAsync((void **)&d.top, sizeof(double) * n * k, st));
    S_TRY(cudaMallocAsync((void **)&d.ta, sizeof(double) * n * k, st));
    S_TRY(cudaMallocAsync((void **)&d.tb, sizeof(double) * n * k, st));
    S_TRY(cudaMallocAsync((void **)&d.wtmp, sizeof(double) * 2 * n * kw, st));
    // the side streams start behind the allocations and the caller's earlier work
    S_TRY(cudaEventRecord(d.done[0], st));
    S_TRY(cudaStreamWaitEvent(d.up, d.done[0], 0));
    S_TRY(cudaStreamWaitEvent(d.down, d.done[0], 0));
    const size_t D = sizeof(double);
    const size_t S = t->sl.size();
    // processing order of the slabs and the copies of slab order[i] into buffer i & 1
    std::vector<size_t> order(S);
    for (size_t i = 0; i < S; ++i) order[i] = forward ? i : S - 1 - i;
    // everything slab i needs from the host -- Y, C, its tree's compact state, its node --
    // goes over `up`, so `st` only runs kernels (an H2D copy on `st` would queue behind
    // the next slab's copies in the copy engine and serialise the pipeline)
    auto issue_load = [&](size_t i) -> tsqr_status_t {
        const int b = (int)(i & 1);
        const size_t j = order[i];
        const Slab &sj = t->sl[j];
        tsqr_tree_t &tr = d.tree[b];
        const tsqr_tree_t before = tr;
        const tsqr_status_t bs = tree_bind(sj.rows, n, d.yb[b], sj.rows, &t->o, st, &tr);
        if (bs != TSQR_OK) return bs;
        cudaError_t e = cudaSuccess;
        if (tr != before) {                                               // a new tree: its arrays were made on st
            e = cudaEventRecord(d.done[b], st);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(d.up, d.done[b], 0);
        }
        if (e == cudaSuccess && i >= 2) e = cudaStreamWaitEvent(d.up, d.freed[b], 0);   // slab i-2 left buffer b
        if (e == cudaSuccess) e = tree_state_copy(tr, t->host + t->state_off[j], false, false, d.up);
        if (e == cudaSuccess && j > 0)
            e = cudaMemcpyAsync(d.node[b], t->nodes + (j - 1) * t->node_words, D * t->node_words,
                                cudaMemcpyHostToDevice, d.up);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(d.yb[b], D * sj.rows, t->Y + sj.r0, D * t->ldy, D * sj.rows, n,
                                  cudaMemcpyHostToDevice, d.up);
        if (e == cudaSuccess && !formq)
            e = cudaMemcpy2DAsync(d.cb[b], D * sj.rows, C + sj.r0, D * ldc, D * sj.rows, k, cudaMemcpyHostToDevice,
                                  d.up);
        if (e == cudaSuccess) e = cudaEventRecord(d.loaded[b], d.up);
        if (e != cudaSuccess) {
            cudaGetLastError();
            set_last_error("tsqr_streamed (load)", e);
            return TSQR_ERR_CUDA;
        }
        return TSQR_OK;
    };
    const double *y1 = nullptr, *tau = nullptr, *tc = nullptr;
    auto cross = [&](double *top, int64_t ldt, const double *ptop, int is_lower, int role, double *Cc, int64_t ldcc,
                     int fwd) -> cudaError_t {
        if (n > 64)
            return launch_wide_cross_apply(y1, tc, top, ldt, ptop, is_lower, role, Cc, ldcc, (int)n, (int)k, d.wtmp,
                                           fwd, st);
        return launch_cross_apply(padded_width(n), y1, tau, top, ldt, ptop, is_lower, role, Cc, ldcc, (int)n, (int)k,
                                  fwd, st);
    };
    if (!forward) {
        if (formq) S_TRY(launch_identity(d.top, (int)n, st));
        else S_TRY(cudaMemcpy2DAsync(d.top, D * n, C, D * ldc, D * n, k, cudaMemcpyHostToDevice, st));
    }
    tsqr_status_t s = issue_load(0);
    if (s != TSQR_OK) return s;
    for (size_t i = 0; i < S; ++i) {
        const size_t j = order[i];
        const int b = (int)(i & 1);
        const Slab &sj = t->sl[j];
        double *cb = d.cb[b];
        tsqr_tree_t tr = d.tree[b];
        S_TRY(cudaStreamWaitEvent(st, d.loaded[b], 0));
        if (i + 1 < S && (s = issue_load(i + 1)) != TSQR_OK) return s;
        S_TRY(tree_rebuild_tcache(tr, st));
        y1 = d.node[b];
        tau = y1 + n * n;
        tc = tau + n;
        if (forward) {
            if ((s = tsqr_apply_qt(tr, cb, sj.rows, k, nullptr, 0, st)) != TSQR_OK) return s;
            if (j == 0) {
                S_TRY(launch_copy_block(cb, sj.rows, d.top, n, (int)n, (int)k, st));
            } else {
                S_TRY(launch_copy_block(cb, sj.rows, d.ta, n, (int)n, (int)k, st));
                // [top; slab head] <- Q_node^T [top; slab head]: top keeps the R coordinates,
                // the slab head rows the node's complement (head role 2)
                S_TRY(cross(d.top, n, d.ta, 1, 2, cb, sj.rows, 1));
            }
        } else {
            if (formq) S_TRY(cudaMemsetAsync(cb, 0, D * sj.rows * k, st));
            if (j > 0) {
                S_TRY(launch_copy_block(cb, sj.rows, d.ta, n, (int)n, (int)k, st));
                S_TRY(launch_copy_block(cb, sj.rows, d.tb, n, (int)n, (int)k, st));
                // Q_node [top; slab head]: the slab's half into its head rows, then the running half
                S_TRY(cross(d.ta, n, d.top, 0, 1, cb, sj.rows, 0));
                S_TRY(cross(d.top, n, d.tb, 1, 1, d.top, n, 0));
            } else {
                S_TRY(launch_copy_block(d.top, n, cb, sj.rows, (int)n, (int)k, st));
            }
            if ((s = tsqr_apply_q(tr, cb, sj.rows, k, st)) != TSQR_OK) return s;
        }
        S_TRY(cudaEventRecord(d.done[b], st));
        S_TRY(cudaStreamWaitEvent(d.down, d.done[b], 0));
        S_TRY(cudaMemcpy2DAsync(C + sj.r0, D * ldc, cb, D * sj.rows, D * sj.rows, k, cudaMemcpyDeviceToHost, d.down));
        S_TRY(cudaEventRecord(d.freed[b], d.down));
    }
    if (forward) {
        // the global head rows (slab 0's, already out) receive Q_thin^T C
        S_TRY(cudaEventRecord(d.done[0], d.down));
        S_TRY(cudaStreamWaitEvent(st, d.done[0], 0));
        S_TRY(cudaMemcpy2DAsync(C, D * ldc, d.top, D * n, D * n, k, cudaMemcpyDeviceToHost, st));
        if (top_out)
            S_TRY(cudaMemcpy2DAsync(top_out, D * ldtop, d.top, D * n, D * n, k, cudaMemcpyDeviceToHost, st));
    }
    S_TRY(cudaStreamSynchronize(d.down));
    S_TRY(cudaStreamSynchronize(st));
    return TSQR_OK;
}

tsqr_status_t tsqr_streamed_apply_qt(tsqr_stream_tree_t t, double *C, int64_t ldc, int64_t k, double *top,
                                     int64_t ldtop, void *stream) {
    if (!t || k < 0 || (k > 0 && (!C || ldc < t->m)) || (top && ldtop < t->n)) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    return streamed_apply(t, C, ldc, k, true, false, top, ldtop, (cudaStream_t)stream);
}

tsqr_status_t tsqr_streamed_apply_q(tsqr_stream_tree_t t, double *C, int64_t ldc, int64_t k, void *stream) {
    if (!t || k < 0 || (k > 0 && (!C || ldc < t->m))) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    return streamed_apply(t, C, ldc, k, false, false, nullptr, 0, (cudaStream_t)stream);
}

tsqr_status_t tsqr_streamed_form_q(tsqr_stream_tree_t t, double *Q, int64_t ldq, void *stream) {
    if (!t || !Q || ldq < t->m) return TSQR_ERR_INVALID;
    return streamed_apply(t, Q, ldq, t->n, false, true, nullptr, 0, (cudaStream_t)stream);
}

}  // extern "C"
