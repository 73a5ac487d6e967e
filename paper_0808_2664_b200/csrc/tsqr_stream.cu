// Sequential (out-of-HBM) TSQR: R of a host-resident m x n
// matrix streamed through the GPU in row slabs -- a flat tree over the slabs
// ([TR] Alg. sequential TSQR P:1725-1753; flat tree P:954-993; the B200 analogue
// of the paper's out-of-DRAM experiment, model Eq. 6): each slab is
// factored on the device by the parallel TSQR (tsqr_factor), then the running R
// absorbs it by the structured combine of [R; R_slab] (Alg. QR:qnxn, q = 2; the
// same kernels as the butterfly rounds).  Slab k+1's host->device copy runs on a
// copy stream while slab k is factored; the factored slab (its reflectors) can be
// copied back to the host.  Product code.
#include "../../include/tsqr.h"
#include "plan.h"
#include "tsqr_kernels.h"

#include <cuda_runtime.h>

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
    cudaStream_t copy = nullptr;
    cudaEvent_t loaded[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr};
    double *slab[2] = {nullptr, nullptr};
    double *rk = nullptr, *run = nullptr, *packed = nullptr, *y1 = nullptr, *tau = nullptr, *tc = nullptr,
           *wtmp = nullptr;
    tsqr_tree_t tree[2] = {nullptr, nullptr};
    ~Res() {
        if (copy) cudaStreamSynchronize(copy);
        for (int i = 0; i < 2; ++i) {
            if (tree[i]) tsqr_tree_free(tree[i]);
            if (slab[i]) cudaFree(slab[i]);
            if (loaded[i]) cudaEventDestroy(loaded[i]);
            if (used[i]) cudaEventDestroy(used[i]);
        }
        for (double *p : {rk, run, packed, y1, tau, tc, wtmp})
            if (p) cudaFree(p);
        if (copy) cudaStreamDestroy(copy);
    }
};

}  // namespace

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

tsqr_status_t tsqr_factor_streamed(int64_t m, int64_t n, const double *A, int64_t lda, int64_t slab_rows,
                                   double *Y, int64_t ldy, double *R, int64_t ldr, const tsqr_opts_t *opts,
                                   void *stream) {
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
        }
        if (Y) {
            // the factored slab (reflectors below each tile's diagonal) back to the host
            S_TRY(cudaEventRecord(r.used[b], st));
            S_TRY(cudaStreamWaitEvent(r.copy, r.used[b], 0));
            S_TRY(cudaMemcpy2DAsync(Y + sl[k].r0, sizeof(double) * ldy, r.slab[b], sizeof(double) * sl[k].rows,
                                    sizeof(double) * sl[k].rows, n, cudaMemcpyDeviceToHost, r.copy));
            S_TRY(cudaEventRecord(r.used[b], r.copy));
        } else {
            S_TRY(cudaEventRecord(r.used[b], st));
        }
    }
    S_TRY(launch_copy_block(r.run, n, R, ldr, (int)n, (int)n, st));
    S_TRY(cudaStreamWaitEvent(st, r.used[(sl.size() - 1) & 1], 0));
    S_TRY(cudaStreamSynchronize(st));
    return TSQR_OK;
}

}  // extern "C"
