// End-to-end QR with HOST buffers (include/tsqr.h "host"): the call a user makes
// with a matrix in host memory -- copy A in, factor (Eqs. 1-4), then
// the explicit thin Q and/or Q^T C ([TR] P:1915-1938), copy the
// results out.  Host orchestration only; the arithmetic is tsqr_factor /
// tsqr_form_q / tsqr_apply_qt.  Product code.
#include "../../include/tsqr.h"
#include "tsqr_kernels.h"

#include <algorithm>
#include <new>

struct tsqr_host_ws_s {
    int64_t m = 0, n = 0, k = 0;
    bool want_q = false;
    double *A = nullptr, *R = nullptr, *Q = nullptr, *C = nullptr;
    tsqr_tree_t tree = nullptr;
    cudaStream_t st = nullptr;
    cudaStream_t up = nullptr, down = nullptr;   // the pipelined path's copy streams
};

namespace {

tsqr_status_t fail(cudaError_t e, const char *where) {
    tsqr::set_last_error(where, e);
    return TSQR_ERR_CUDA;
}

void release(tsqr_host_ws_s *w) {
    for (cudaStream_t *sp : {&w->up, &w->down}) {
        if (*sp) {
            cudaStreamSynchronize(*sp);
            cudaStreamDestroy(*sp);
        }
        *sp = nullptr;
    }
    if (w->tree) tsqr_tree_free(w->tree);
    w->tree = nullptr;
    for (double **p : {&w->A, &w->R, &w->Q, &w->C}) {
        if (*p) cudaFreeAsync(*p, w->st);
        *p = nullptr;
    }
}

}  // namespace

extern "C" {

tsqr_status_t tsqr_qr_host(tsqr_host_ws_t *ws, int64_t m, int64_t n, const double *A, int64_t lda, double *R,
                           int64_t ldr, double *Q, int64_t ldq, double *C, int64_t ldc, int64_t k,
                           const tsqr_opts_t *opts, void *stream) {
    if (!ws || !A || !R) return TSQR_ERR_INVALID;
    if (n < 1 || m < n) return TSQR_ERR_SHAPE;
    if (lda < m || ldr < n || (Q && ldq < m) || k < 0 || (k > 0 && (!C || ldc < m))) return TSQR_ERR_INVALID;
    if (opts && opts->nranks > 1) return TSQR_ERR_UNSUPPORTED;
    {   // validate the plan before anything is enqueued
        tsqr_plan_info_t info;
        const tsqr_status_t s = tsqr_plan_info(m, n, opts, &info);
        if (s != TSQR_OK) return s;
    }
    cudaStream_t st = (cudaStream_t)stream;
    tsqr_host_ws_s *w = *ws;
    if (!w) {
        w = new (std::nothrow) tsqr_host_ws_s();
        if (!w) return TSQR_ERR_ALLOC;
        *ws = w;
    }
    if (w->m != m || w->n != n || w->k < k || (Q && !w->want_q)) {      // (re)allocate, stream-ordered
        release(w);
        w->st = st;
        cudaError_t e = cudaMallocAsync((void **)&w->A, sizeof(double) * m * n, st);
        if (e == cudaSuccess) e = cudaMallocAsync((void **)&w->R, sizeof(double) * n * n, st);
        if (e == cudaSuccess && Q) e = cudaMallocAsync((void **)&w->Q, sizeof(double) * m * n, st);
        if (e == cudaSuccess && k) e = cudaMallocAsync((void **)&w->C, sizeof(double) * m * k, st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            release(w);
            w->m = w->n = w->k = 0;
            return TSQR_ERR_ALLOC;
        }
        w->m = m;
        w->n = n;
        w->k = k;
        w->want_q = Q != nullptr;
    }
    w->st = st;
    const size_t d = sizeof(double);
    if (Q && k == 0 && n <= 64) {
        // factor + explicit Q pipelined over slabs of tiles: the copy-in hides the leaf stage
        // and the copy-out the form-Q leaves (tsqr::qr_host_pipelined); slabs of >= 128 MB
        const int S = (int)std::max<int64_t>(1, std::min<int64_t>(8, (int64_t)(d * m * n) >> 27));
        cudaError_t e = cudaSuccess;
        if (!w->up) e = cudaStreamCreateWithFlags(&w->up, cudaStreamNonBlocking);
        if (e == cudaSuccess && !w->down) e = cudaStreamCreateWithFlags(&w->down, cudaStreamNonBlocking);
        if (e != cudaSuccess) return fail(e, "tsqr_qr_host streams");
        return tsqr::qr_host_pipelined(&w->tree, m, n, A, lda, w->A, w->R, w->Q, R, ldr, Q, ldq, opts, st, w->up,
                                       w->down, S);
    }
    cudaError_t e = cudaMemcpy2DAsync(w->A, d * m, A, d * lda, d * m, n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && k) e = cudaMemcpy2DAsync(w->C, d * m, C, d * ldc, d * m, k, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(e, "tsqr_qr_host copy in");
    tsqr_status_t s = tsqr_factor(m, n, w->A, m, w->R, n, opts, stream, &w->tree);
    if (s != TSQR_OK) return s;
    if (Q) {
        if ((s = tsqr_form_q(w->tree, w->Q, m, stream)) != TSQR_OK) return s;
        e = cudaMemcpy2DAsync(Q, d * ldq, w->Q, d * m, d * m, n, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return fail(e, "tsqr_qr_host copy out");
    }
    if (k) {
        if ((s = tsqr_apply_qt(w->tree, w->C, m, k, nullptr, 0, stream)) != TSQR_OK) return s;
        e = cudaMemcpy2DAsync(C, d * ldc, w->C, d * m, d * m, k, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return fail(e, "tsqr_qr_host copy out");
    }
    e = cudaMemcpy2DAsync(R, d * ldr, w->R, d * n, d * n, n, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(e, "tsqr_qr_host");
    return TSQR_OK;
}

tsqr_status_t tsqr_host_ws_free(tsqr_host_ws_t w) {
    if (!w) return TSQR_OK;
    release(w);
    delete w;
    return TSQR_OK;
}

}  // extern "C"
