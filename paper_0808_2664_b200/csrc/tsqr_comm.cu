// Communicator layer of libtsqr.so (include/tsqr.h "communicator"): row-sharded
// multi-GPU TSQR as one collective C call per operation.  Alg. TSQR:par ([TR]
// P:1667-1707) as a butterfly all-reduction (indices [TR] P:3955-3975): after the
// local tree, log2(G) rounds, each a grouped ncclSend/ncclRecv with partner
// rank XOR 2^(k-1) on the caller's stream, then the round's structured combine.
// Host code only: every arithmetic step is one of the tree's kernels (the local
// entry points of tsqr_api.cu).  Product code.
#include "../../include/tsqr.h"
#include "tsqr_kernels.h"

#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

using namespace tsqr;

// In-process mailbox of the loopback transport (tests): message (from -> to) and
// its acknowledgement carry a per-pair sequence number.
struct tsqr_loopback_s {
    int nranks = 0;
    std::mutex mu;
    std::condition_variable cv;
    struct Msg {
        const double *ptr = nullptr;
        int64_t count = 0, seq = 0, ack = 0;
    };
    std::vector<Msg> box;                     // [from * nranks + to]
};

struct tsqr_ctx_s {
    int device = 0;
    int nranks = 1, rank = 0;
    ncclComm_t comm = nullptr;
    tsqr_loopback_s *hub = nullptr;
    std::vector<int64_t> pair_seq;            // loopback: exchanges done with each peer
    double *send = nullptr, *recv = nullptr;  // exchange buffers (device), `words` each
    int64_t words = 0;
    cudaStream_t buf_stream = nullptr;        // stream of the buffers' last use
};

namespace {

int ilog2(int x) {
    int r = 0;
    while ((1 << r) < x) ++r;
    return r;
}

int head_role(int rank, int round) {
    const int half = 1 << (round - 1), pos = rank & (2 * half - 1);
    return pos == 0 ? 1 : (pos == half ? 2 : 0);
}

tsqr_status_t nccl_fail(ncclResult_t r, const char *where) {
    const std::string msg = std::string(where) + ": " + ncclGetErrorString(r);
    set_last_error_text(msg.c_str());
    return TSQR_ERR_NCCL;
}

tsqr_status_t cuda_fail(cudaError_t e, const char *where) {
    set_last_error(where, e);
    return TSQR_ERR_CUDA;
}

// current device = the context's, restored on exit
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// exchange buffers of at least `need` words, stream-ordered on st
tsqr_status_t ensure_buffers(tsqr_ctx_s *c, int64_t need, cudaStream_t st) {
    if (c->words >= need) return TSQR_OK;
    if (c->send) cudaFreeAsync(c->send, st);
    if (c->recv) cudaFreeAsync(c->recv, st);
    c->send = c->recv = nullptr;
    c->words = 0;
    cudaError_t e = cudaMallocAsync((void **)&c->send, sizeof(double) * need, st);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&c->recv, sizeof(double) * need, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return TSQR_ERR_ALLOC;
    }
    c->words = need;
    c->buf_stream = st;
    return TSQR_OK;
}

// One message each way between this rank and `partner`, stream-ordered on st:
// recv[0..count) <- the partner's send[0..count).
tsqr_status_t exchange(tsqr_ctx_s *c, const double *send, double *recv, int64_t count, int partner, cudaStream_t st) {
    if (c->comm) {
        ncclResult_t r = ncclGroupStart();
        if (r == ncclSuccess) r = ncclSend(send, (size_t)count, ncclDouble, partner, c->comm, st);
        if (r == ncclSuccess) r = ncclRecv(recv, (size_t)count, ncclDouble, partner, c->comm, st);
        const ncclResult_t g = ncclGroupEnd();
        if (r == ncclSuccess) r = g;
        return r == ncclSuccess ? TSQR_OK : nccl_fail(r, "butterfly exchange");
    }
    if (!c->hub) {
        set_last_error_text("butterfly exchange: the context has no communicator (tsqr_ctx_set_comm)");
        return TSQR_ERR_NCCL;
    }
    // loopback: post the (complete) message, copy the partner's, wait for its copy of ours
    tsqr_loopback_s *h = c->hub;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "loopback exchange");
    const int64_t seq = ++c->pair_seq[partner];
    tsqr_loopback_s::Msg *mine = &h->box[c->rank * h->nranks + partner];
    tsqr_loopback_s::Msg *theirs = &h->box[partner * h->nranks + c->rank];
    {
        std::unique_lock<std::mutex> lk(h->mu);
        mine->ptr = send;
        mine->count = count;
        mine->seq = seq;
        h->cv.notify_all();
        h->cv.wait(lk, [&] { return theirs->seq == seq; });
    }
    if (theirs->count != count) {
        set_last_error_text("loopback exchange: message sizes differ between partners");
        return TSQR_ERR_NCCL;
    }
    e = cudaMemcpyAsync(recv, theirs->ptr, sizeof(double) * count, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "loopback exchange");
    {
        std::unique_lock<std::mutex> lk(h->mu);
        theirs->ack = seq;                     // we are done with the partner's buffer
        h->cv.notify_all();
        h->cv.wait(lk, [&] { return mine->ack == seq; });
    }
    return TSQR_OK;
}

bool valid(const tsqr_ctx_s *c) { return c != nullptr && c->nranks >= 1; }

}  // namespace

extern "C" {

tsqr_status_t tsqr_ctx_create(int device, tsqr_ctx_t *out) {
    if (!out) return TSQR_ERR_INVALID;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "tsqr_ctx_create");
    if (device < 0 || device >= count) return TSQR_ERR_INVALID;
    tsqr_ctx_s *c = new (std::nothrow) tsqr_ctx_s();
    if (!c) return TSQR_ERR_ALLOC;
    c->device = device;
    c->pair_seq.assign(1, 0);
    *out = c;
    return TSQR_OK;
}

tsqr_status_t tsqr_get_unique_id(void *uid128) {
    if (!uid128) return TSQR_ERR_INVALID;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "tsqr_get_unique_id");
    std::memcpy(uid128, &id, sizeof(id));
    return TSQR_OK;
}

static void drop_comm(tsqr_ctx_s *c) {
    if (c->comm) ncclCommDestroy(c->comm);
    c->comm = nullptr;
    c->hub = nullptr;
    c->nranks = 1;
    c->rank = 0;
    c->pair_seq.assign(1, 0);
}

tsqr_status_t tsqr_ctx_set_comm(tsqr_ctx_t c, const void *uid128, int32_t nranks, int32_t rank) {
    if (!valid(c) || !uid128) return TSQR_ERR_INVALID;
    if (nranks < 1 || rank < 0 || rank >= nranks) return TSQR_ERR_INVALID;
    if (nranks & (nranks - 1)) return TSQR_ERR_UNSUPPORTED;
    DeviceGuard g(c->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "tsqr_ctx_set_comm");
    drop_comm(c);
    ncclUniqueId id;
    std::memcpy(&id, uid128, sizeof(id));
    const ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        return nccl_fail(r, "tsqr_ctx_set_comm (ncclCommInitRank)");
    }
    c->nranks = nranks;
    c->rank = rank;
    c->pair_seq.assign(nranks, 0);
    return TSQR_OK;
}

tsqr_status_t tsqr_loopback_create(int32_t nranks, tsqr_loopback_t *out) {
    if (!out || nranks < 1) return TSQR_ERR_INVALID;
    if (nranks & (nranks - 1)) return TSQR_ERR_UNSUPPORTED;
    tsqr_loopback_s *h = new (std::nothrow) tsqr_loopback_s();
    if (!h) return TSQR_ERR_ALLOC;
    h->nranks = nranks;
    h->box.resize((size_t)nranks * nranks);
    *out = h;
    return TSQR_OK;
}

tsqr_status_t tsqr_loopback_destroy(tsqr_loopback_t h) {
    delete h;
    return TSQR_OK;
}

tsqr_status_t tsqr_ctx_set_loopback(tsqr_ctx_t c, tsqr_loopback_t h, int32_t rank) {
    if (!valid(c) || !h || rank < 0 || rank >= h->nranks) return TSQR_ERR_INVALID;
    drop_comm(c);
    c->hub = h;
    c->nranks = h->nranks;
    c->rank = rank;
    c->pair_seq.assign(h->nranks, 0);
    return TSQR_OK;
}

tsqr_status_t tsqr_ctx_info(tsqr_ctx_t c, int32_t *nranks, int32_t *rank) {
    if (!valid(c)) return TSQR_ERR_INVALID;
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    return TSQR_OK;
}

tsqr_status_t tsqr_ctx_destroy(tsqr_ctx_t c) {
    if (!c) return TSQR_OK;
    {
        DeviceGuard g(c->device);
        if (c->send) cudaFreeAsync(c->send, c->buf_stream);
        if (c->recv) cudaFreeAsync(c->recv, c->buf_stream);
        drop_comm(c);
    }
    delete c;
    return TSQR_OK;
}

tsqr_status_t tsqr_ctx_factor(tsqr_ctx_t c, int64_t m_local, int64_t n, double *A, int64_t lda, double *R,
                              int64_t ldr, const tsqr_opts_t *opts, void *stream, tsqr_tree_t *tree) {
    if (!valid(c)) return TSQR_ERR_INVALID;
    DeviceGuard g(c->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "tsqr_ctx_factor");
    tsqr_opts_t o{};
    if (opts) o = *opts;
    o.nranks = c->nranks;
    o.rank = c->rank;
    const int rounds = ilog2(c->nranks);
    cudaStream_t st = (cudaStream_t)stream;
    // Alg. TSQR:par line 1: the local tree of the slab
    tsqr_status_t s = tsqr_factor(m_local, n, A, lda, rounds ? nullptr : R, ldr, &o, stream, tree);
    if (s != TSQR_OK || rounds == 0) return s;
    const int64_t np = n * (n + 1) / 2;                 // Cor. 2: the packed triangle
    if ((s = ensure_buffers(c, np, st)) != TSQR_OK) return s;
    for (int r = 1; r <= rounds; ++r) {                 // lines 2-8: the butterfly rounds
        const int partner = c->rank ^ (1 << (r - 1));
        if ((s = tsqr_pack_r(*tree, c->send, stream)) != TSQR_OK) return s;
        if ((s = exchange(c, c->send, c->recv, np, partner, st)) != TSQR_OK) return s;
        if ((s = tsqr_cross_factor(*tree, r, c->recv, r == rounds ? R : nullptr, ldr, stream)) != TSQR_OK) return s;
    }
    c->buf_stream = st;
    return TSQR_OK;
}

tsqr_status_t tsqr_ctx_apply_qt(tsqr_ctx_t c, tsqr_tree_t tree, double *C, int64_t ldc, int64_t k, double *top,
                                int64_t ldtop, void *stream) {
    if (!valid(c) || !tree) return TSQR_ERR_INVALID;
    int64_t ml, n;
    int nr, rk, done;
    tree_shape(tree, &ml, &n, &nr, &rk, &done);
    if (nr != c->nranks || rk != c->rank) return TSQR_ERR_INVALID;    // a tree of another layout
    if (k < 0) return TSQR_ERR_INVALID;
    if (top && ldtop < n) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    DeviceGuard g(c->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "tsqr_ctx_apply_qt");
    const int rounds = ilog2(c->nranks);
    cudaStream_t st = (cudaStream_t)stream;
    if (rounds == 0) return tsqr_apply_qt(tree, C, ldc, k, top, ldtop, stream);
    if (done != rounds) return TSQR_ERR_INVALID;                      // factor's rounds not all done
    tsqr_status_t s = ensure_buffers(c, n * k, st);
    if (s != TSQR_OK) return s;
    // the local tree; c->send holds this rank's R coordinates (n x k, ld n), then per
    // round: exchange them, apply the round's node (eq. localQTupdate)
    if ((s = tsqr_apply_qt(tree, C, ldc, k, c->send, n, stream)) != TSQR_OK) return s;
    for (int r = 1; r <= rounds; ++r) {
        const int partner = c->rank ^ (1 << (r - 1));
        if ((s = exchange(c, c->send, c->recv, n * k, partner, st)) != TSQR_OK) return s;
        if ((s = tsqr_cross_apply_qt(tree, r, c->send, n, c->recv, C, ldc, k, stream)) != TSQR_OK) return s;
    }
    if (top) {
        const cudaError_t e = cudaMemcpy2DAsync(top, sizeof(double) * ldtop, c->send, sizeof(double) * n,
                                                sizeof(double) * n, k, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "tsqr_ctx_apply_qt top");
    }
    c->buf_stream = st;
    return TSQR_OK;
}

tsqr_status_t tsqr_ctx_apply_q(tsqr_ctx_t c, tsqr_tree_t tree, double *C, int64_t ldc, int64_t k, void *stream) {
    if (!valid(c) || !tree) return TSQR_ERR_INVALID;
    int64_t ml, n;
    int nr, rk, done;
    tree_shape(tree, &ml, &n, &nr, &rk, &done);
    if (nr != c->nranks || rk != c->rank) return TSQR_ERR_INVALID;
    if (k < 0 || !C || ldc < ml) return TSQR_ERR_INVALID;
    if (k == 0) return TSQR_OK;
    DeviceGuard g(c->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "tsqr_ctx_apply_q");
    const int rounds = ilog2(c->nranks);
    cudaStream_t st = (cudaStream_t)stream;
    if (rounds && done != rounds) return TSQR_ERR_INVALID;
    tsqr_status_t s = rounds ? ensure_buffers(c, n * k, st) : TSQR_OK;
    if (s != TSQR_OK) return s;
    for (int r = rounds; r >= 1; --r) {                 // top-down: only the round's two group heads
        if (head_role(c->rank, r) == 0) continue;
        const int partner = c->rank ^ (1 << (r - 1));
        const cudaError_t e = cudaMemcpy2DAsync(c->send, sizeof(double) * n, C, sizeof(double) * ldc,
                                                sizeof(double) * n, k, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "tsqr_ctx_apply_q head");
        if ((s = exchange(c, c->send, c->recv, n * k, partner, st)) != TSQR_OK) return s;
        if ((s = tsqr_cross_apply_q(tree, r, c->send, n, c->recv, C, ldc, k, stream)) != TSQR_OK) return s;
    }
    if (rounds) c->buf_stream = st;
    return tsqr_apply_q(tree, C, ldc, k, stream);
}

tsqr_status_t tsqr_ctx_form_q(tsqr_ctx_t c, tsqr_tree_t tree, double *Q, int64_t ldq, void *stream) {
    if (!valid(c) || !tree) return TSQR_ERR_INVALID;
    int64_t ml, n;
    int nr, rk, done;
    tree_shape(tree, &ml, &n, &nr, &rk, &done);
    if (nr != c->nranks || rk != c->rank) return TSQR_ERR_INVALID;
    DeviceGuard g(c->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "tsqr_ctx_form_q");
    return tsqr_form_q(tree, Q, ldq, stream);
}

tsqr_status_t tsqr_ctx_cholqr(tsqr_ctx_t c, int64_t m_local, int64_t n, const double *A, int64_t lda, double *R,
                              int64_t ldr, double *Q, int64_t ldq, int *info, void *stream) {
    if (!valid(c) || !A || !R || !info) return TSQR_ERR_INVALID;
    if (n < 1 || m_local < n) return TSQR_ERR_SHAPE;
    if (n > TSQR_MAX_N) return TSQR_ERR_UNSUPPORTED;
    if (lda < m_local || ldr < n || (Q && ldq < m_local)) return TSQR_ERR_INVALID;
    DeviceGuard g(c->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "tsqr_ctx_cholqr");
    const int rounds = ilog2(c->nranks);
    cudaStream_t st = (cudaStream_t)stream;
    tsqr_status_t s = rounds ? ensure_buffers(c, n * n, st) : TSQR_OK;
    if (s != TSQR_OK) return s;
    CholqrWs w;
    cudaError_t e = cholqr_alloc(w, m_local, (int)n, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return TSQR_ERR_ALLOC;
    }
    e = cholqr_gram(A, lda, m_local, (int)n, w, st);                       // line 1, this rank's A_i^T A_i
    for (int r = 1; r <= rounds && e == cudaSuccess && s == TSQR_OK; ++r) {  // line 1's all-reduction
        const int partner = c->rank ^ (1 << (r - 1));
        e = cudaMemcpyAsync(c->send, w.W, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess) s = exchange(c, c->send, c->recv, n * n, partner, st);
        if (e == cudaSuccess && s == TSQR_OK) e = cholqr_add_ordered(w.W, c->recv, n * n, c->rank < partner, st);
    }
    if (e == cudaSuccess && s == TSQR_OK) e = cholqr_finish(A, lda, m_local, (int)n, w, R, ldr, Q, ldq, info, st);
    cholqr_free(w, st);
    if (rounds) c->buf_stream = st;
    if (s != TSQR_OK) return s;
    return e == cudaSuccess ? TSQR_OK : cuda_fail(e, "tsqr_ctx_cholqr");
}

}  // extern "C"

