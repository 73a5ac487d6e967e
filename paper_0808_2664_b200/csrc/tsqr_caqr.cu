// CAQR on one GPU: the right-looking QR of an m x N matrix
// with TSQR panels -- "CAQR simply implements the right-looking QR factorization
// using ... TSQR as the panel factorization.  The rest is bookkeeping" (Sec. 3,
// P:2944-2946); Alg. CAQR:j ([TR] P:3992-4048) with one process row.  Product
// code: host-side orchestration of the TSQR entry points (tsqr_api.cu) plus two
// small fill kernels; every panel factor and trailing update runs in the TSQR
// kernels.
#include "../../include/tsqr.h"
#include "tsqr_kernels.h"

#include <cuda_runtime.h>

#include <new>
#include <vector>

struct tsqr_caqr_s {
    int64_t m = 0, N = 0, panel = 0;
    tsqr_opts_t opts{};
    std::vector<tsqr_tree_t> trees;   // one per panel: its TSQR over rows c0..m-1
    double *A = nullptr;
    int64_t lda = 0;
};

namespace {

__global__ void k_caqr_zero_below(double *R, int64_t ldr, int64_t N, int64_t c0, int64_t w) {
    // rows c0+w..N-1 of columns c0..c0+w-1 of R (the panel's zero block below its diagonal block)
    const int64_t rows = N - c0 - w;
    for (int64_t e = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; e < rows * w;
         e += (int64_t)blockDim.x * gridDim.x)
        R[c0 + w + e % rows + (c0 + e / rows) * ldr] = 0.0;
}

__global__ void k_caqr_eye(double *Q, int64_t ldq, int64_t m, int64_t N) {
    // Q <- [I_N; 0] (m x N)
    for (int64_t e = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; e < m * N;
         e += (int64_t)blockDim.x * gridDim.x) {
        const int64_t r = e % m, c = e / m;
        Q[r + c * ldq] = r == c ? 1.0 : 0.0;
    }
}

int grid_for(int64_t elems) {
    const int64_t g = (elems + 255) / 256;
    return (int)(g < 1 ? 1 : (g > 4 * 148 * 8 ? 4 * 148 * 8 : g));
}

tsqr_status_t free_trees(tsqr_caqr_s *c) {
    for (tsqr_tree_t &t : c->trees)
        if (t) tsqr_tree_free(t);
    c->trees.clear();
    return TSQR_OK;
}

}  // namespace

extern "C" {

tsqr_status_t tsqr_caqr_factor(int64_t m, int64_t N, double *A, int64_t lda, int64_t panel_cols, double *R,
                               int64_t ldr, const tsqr_opts_t *opts, void *stream, tsqr_caqr_t *caqr) {
    if (!A || !R || !caqr) return TSQR_ERR_INVALID;
    if (N < 1 || m < N) return TSQR_ERR_SHAPE;
    if (lda < m || ldr < N || panel_cols < 1) return TSQR_ERR_INVALID;
    if (panel_cols > TSQR_MAX_N) return TSQR_ERR_UNSUPPORTED;
    tsqr_opts_t o{};
    if (opts) o = *opts;
    if (o.nranks > 1) return TSQR_ERR_UNSUPPORTED;    // one GPU (one process row)
    o.nranks = 1;
    o.rank = 0;
    const int64_t np = (N + panel_cols - 1) / panel_cols;
    tsqr_caqr_s *c = *caqr;
    // a handle of the same shape keeps its panel trees (their workspaces are reused)
    if (c && !(c->m == m && c->N == N && c->panel == panel_cols && c->opts.block_rows == o.block_rows &&
               c->opts.tile_rows == o.tile_rows && (int64_t)c->trees.size() == np))
        return TSQR_ERR_INVALID;
    const bool fresh = c == nullptr;
    if (fresh) {
        c = new (std::nothrow) tsqr_caqr_s();
        if (!c) return TSQR_ERR_ALLOC;
        c->m = m; c->N = N; c->panel = panel_cols; c->opts = o;
        c->trees.assign(np, nullptr);
    }
    c->A = A;
    c->lda = lda;
    cudaStream_t st = (cudaStream_t)stream;
    for (int64_t j = 0; j < np; ++j) {
        const int64_t c0 = j * panel_cols, w = N - c0 < panel_cols ? N - c0 : panel_cols;
        // line 1: TSQR of the panel's rows c0..m-1; its R is R's diagonal block
        tsqr_status_t s = tsqr_factor(m - c0, w, A + c0 + c0 * lda, lda, R + c0 + c0 * ldr, ldr, &o, stream,
                                      &c->trees[j]);
        if (s == TSQR_OK && c0 + w < N) {
            // zero block below the diagonal block, then line 3 (+ the tree stages): Q_j^T on the
            // trailing columns; rows 0..w-1 of the result are R's row block
            k_caqr_zero_below<<<grid_for((N - c0 - w) * w), 256, 0, st>>>(R, ldr, N, c0, w);
            const cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) {
                tsqr::set_last_error("tsqr_caqr_factor", e);
                s = TSQR_ERR_CUDA;
            }
            if (s == TSQR_OK)
                s = tsqr_apply_qt(c->trees[j], A + c0 + (c0 + w) * lda, lda, N - c0 - w, R + c0 + (c0 + w) * ldr,
                                  ldr, stream);
        }
        if (s != TSQR_OK) {
            if (fresh) {
                free_trees(c);
                delete c;
            }
            return s;
        }
    }
    *caqr = c;
    return TSQR_OK;
}

tsqr_status_t tsqr_caqr_apply_qt(tsqr_caqr_t c, double *C, int64_t ldc, int64_t k, void *stream) {
    if (!c || !c->A) return TSQR_ERR_INVALID;
    if (k < 0) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    if (!C || ldc < c->m) return TSQR_ERR_INVALID;
    for (size_t j = 0; j < c->trees.size(); ++j) {
        const int64_t c0 = (int64_t)j * c->panel;
        tsqr_status_t s = tsqr_apply_qt(c->trees[j], C + c0, ldc, k, nullptr, 0, stream);
        if (s != TSQR_OK) return s;
    }
    return TSQR_OK;
}

tsqr_status_t tsqr_caqr_apply_q(tsqr_caqr_t c, double *C, int64_t ldc, int64_t k, void *stream) {
    if (!c || !c->A) return TSQR_ERR_INVALID;
    if (k < 0) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    if (!C || ldc < c->m) return TSQR_ERR_INVALID;
    for (size_t j = c->trees.size(); j-- > 0;) {
        const int64_t c0 = (int64_t)j * c->panel;
        tsqr_status_t s = tsqr_apply_q(c->trees[j], C + c0, ldc, k, stream);
        if (s != TSQR_OK) return s;
    }
    return TSQR_OK;
}

tsqr_status_t tsqr_caqr_form_q(tsqr_caqr_t c, double *Q, int64_t ldq, void *stream) {
    if (!c || !c->A || !Q || ldq < c->m) return TSQR_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    k_caqr_eye<<<grid_for(c->m * c->N), 256, 0, st>>>(Q, ldq, c->m, c->N);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        tsqr::set_last_error("tsqr_caqr_form_q", e);
        return TSQR_ERR_CUDA;
    }
    // Q = Q_1 ... Q_p [I_N; 0]: Q_j acts on rows c0_j.. where only columns >= c0_j are nonzero
    for (size_t j = c->trees.size(); j-- > 0;) {
        const int64_t c0 = (int64_t)j * c->panel;
        tsqr_status_t s = tsqr_apply_q(c->trees[j], Q + c0 + c0 * ldq, ldq, c->N - c0, stream);
        if (s != TSQR_OK) return s;
    }
    return TSQR_OK;
}

tsqr_status_t tsqr_caqr_free(tsqr_caqr_t c) {
    if (!c) return TSQR_OK;
    free_trees(c);
    delete c;
    return TSQR_OK;
}

}  // extern "C"
