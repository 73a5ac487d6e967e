// Pipelined reduction tree for n <= 64 (a4, a6).  Product code.
//
// Every tree node (Alg. QR:qnxn with q = 2 on [R_a; R_b], eq. fact_2rs;
// Alg. TSQR:par P:1681-1692) is one warp.  R_b's upper block-triangle lives in
// the warp's registers as DMMA fragments (blocks k <= cb of 8x8, the zero
// blocks never exist); the pivot rows 8P..8P+7 of R_a of panel P sit in a small
// per-warp smem buffer.  Panel P of a node needs only row block P of each
// child's R (R's rows 8P..8P+7 are final once the child has finished its panel
// P), so a node starts panel P as soon as both children have published it:
// the levels of the tree overlap, and the critical path is about
// (depth + panels) panel latencies instead of depth x node latencies.
// Outputs per panel: the node's R rows 8P..8P+7 -> the left subtree's head
// (tile a), Y1 columns 8P..8P+7 -> the right subtree's head (tile b), both
// upper triangles only (the leaf reflectors below stay); tau -> tau_node.
// Nodes are numbered bottom-up, so a node depends only on lower-numbered
// nodes; blocks take their node range from a ticket counter when they start,
// so a lower-numbered node always belongs to a block that is already resident
// or finished: the spin-waits cannot deadlock.
#include "tsqr_kernels.h"
#include "chunk.cuh"

#include <vector>

namespace tsqr {
namespace tree {

using chunk::build_t;
using chunk::House;
using chunk::house_bf;
using wy::dmma;
constexpr unsigned FULL = 0xffffffffu;
#ifndef TSQR_TREE_NW
#define TSQR_TREE_NW 4
#endif
constexpr int NW = TSQR_TREE_NW;   // nodes (warps) per block: 4 spreads a level over twice the SMs of 8 (C5 tree 0.229 -> 0.189 ms, C4 0.307 -> 0.293, C2 0.126 -> 0.121)

template <int NCB_>
struct TCfg {
    static constexpr int NCB = NCB_, NP = 8 * NCB;
    static constexpr int LDA = NP + 2;                      // R_a row block (8 x NP, row-major)
    static constexpr int RA = 0, YS = RA + 8 * LDA, GS = YS + NP * 8, TS = GS + 64, T8 = TS + 64, XS = T8 + 8;
    static constexpr int WS = XS + 2 * NP;                  // per warp (doubles)
    static constexpr size_t BYTES = (size_t)NW * WS * sizeof(double);
};

template <class C>
struct NodeRegs {
    double a[C::NCB][C::NCB][2];     // only k <= cb is ever touched
};

__device__ __forceinline__ void wait_flag(const int *f) {
    if ((threadIdx.x & 31) == 0) {
        while (*reinterpret_cast<const volatile int *>(f) == 0) __nanosleep(64);
    }
    __syncwarp();
    __threadfence();
}

#ifdef TSQR_NTREE_PROBE
__device__ unsigned long long g_ntprobe[8 * 8 * 2];
#define NTPROBE(i) do { if ((threadIdx.x & 31) == 0 && (fme == g_nt_root || fme == g_nt_leaf)) { \
    unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
    g_ntprobe[(fme == g_nt_root ? 64 : 0) + P * 8 + (i)] = t_; } } while (0)
__device__ int *g_nt_root, *g_nt_leaf;
#else
#define NTPROBE(i)
#endif

template <class C, int P>
__device__ __forceinline__ void node_panel(NodeRegs<C> &rg, double *Ahead_a, double *Ahead_b, int64_t lda, int n,
                                           double *ws, double *tau_out, const int *fl, const int *fr, int *fme,
                                           double *R, int64_t ldr, double *tc) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    double *Ra = ws + C::RA, *Ys = ws + C::YS, *Gs = ws + C::GS, *Ts = ws + C::TS, *t8 = ws + C::T8, *xs = ws + C::XS;
    NTPROBE(0);
    if (fl) wait_flag(fl + P);
    if (fr) wait_flag(fr + P);
    NTPROBE(1);
    // R_a rows 8P..8P+7 (upper part) -> smem; R_b row block P (upper part) -> registers
    double ra[2 * C::NCB];              // all loads in flight before the first use
#pragma unroll
    for (int u = 0; u < 2 * C::NCB; ++u) {
        const int e = lane + 32 * u, r = e & 7, c = e >> 3, i = 8 * P + r;
        ra[u] = (c >= i && c < n) ? __ldcg(Ahead_a + i + (int64_t)c * lda) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 2 * C::NCB; ++u) {
        const int e = lane + 32 * u;
        Ra[(e & 7) * C::LDA + (e >> 3)] = ra[u];
    }
#pragma unroll
    for (int cb = P; cb < C::NCB; ++cb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = 8 * P + 2 * q + e, c = 8 * cb + l4;
            rg.a[P][cb][e] = (c >= i && c < n) ? __ldcg(Ahead_b + i + (int64_t)c * lda) : 0.0;
        }
    // pivot column broadcast row (x = column 8P of R_b rows 0..8P+7)
    if (l4 == 0) {
#pragma unroll
        for (int k = 0; k <= P; ++k)
            *reinterpret_cast<double2 *>(xs + 8 * k + 2 * q) = make_double2(rg.a[k][P][0], rg.a[k][P][1]);
    }
    __syncwarp();
    const int jn = (P + 1 < C::NCB) ? 8 : n - 8 * P;
#pragma unroll 1
    for (int jj = 0; jj < jn; ++jj) {
        const double *xr = xs + (jj & 1) * C::NP;
        double d0 = 0.0, d1 = 0.0, s0 = 0.0, s1 = 0.0;
        double x[P + 1][2];
#pragma unroll
        for (int k = 0; k <= P; ++k) {
            const double2 v = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
            x[k][0] = v.x;
            x[k][1] = v.y;
            d0 = fma(x[k][0], rg.a[k][P][0], d0);
            d1 = fma(x[k][1], rg.a[k][P][1], d1);
            s0 = fma(x[k][0], x[k][0], s0);
            s1 = fma(x[k][1], x[k][1], s1);
        }
        double d, s2;
        chunk::quad_sums(d, s2, d0 + d1, s0 + s1);
        const double alpha = Ra[jj * C::LDA + 8 * P + jj];
        const double rj = Ra[jj * C::LDA + 8 * P + l4];
        House h = house_bf(alpha, s2);
        double sc = 1.0;
        double sx = h.scale;                                        // the scale of the unscaled x
        if (__any_sync(0xffffffffu, wy::house_unsafe(alpha, s2))) {  // warp-uniform, R23
            chunk::rescaled_sums<P + 1>(x, [&](int k, int e) { return rg.a[k][P][e]; }, alpha, d, s2, sc);
            h = house_bf(sc * alpha, s2);
            h.beta = h.beta / sc;
            sx = h.scale * sc;
        }
        const double w = fma(h.scale, d, rj);
        const double u = (l4 > jj) ? h.tau * sx * w : (l4 == jj ? 1.0 : 0.0);
        const double g = (l4 == jj) ? sx : 0.0;
        const double rnew = (l4 == jj) ? h.beta : fma(-h.tau, w, rj);
#pragma unroll
        for (int k = 0; k <= P; ++k) {
            rg.a[k][P][0] = fma(g, x[k][0], fma(-u, x[k][0], rg.a[k][P][0]));
            rg.a[k][P][1] = fma(g, x[k][1], fma(-u, x[k][1], rg.a[k][P][1]));
        }
        if (l4 == jj + 1) {
            double *xw = xs + ((jj + 1) & 1) * C::NP;
#pragma unroll
            for (int k = 0; k <= P; ++k)
                *reinterpret_cast<double2 *>(xw + 8 * k + 2 * q) = make_double2(rg.a[k][P][0], rg.a[k][P][1]);
        }
        __syncwarp();
        if (q == 0 && l4 >= jj) Ra[jj * C::LDA + 8 * P + l4] = rnew;
        if (q == 0 && l4 < jj) Gs[l4 * 8 + jj] = h.scale * d;
        if (lane == 0) t8[jj] = h.tau;
        __syncwarp();
    }
    chunk::pad_steps(Gs, t8, jn);
    __syncwarp();
    if (lane < 8 && 8 * P + lane < n) tau_out[8 * P + lane] = t8[lane];
    // Y of the panel (rows 0..8P+7 of R_b, i.e. Y1's columns 8P..8P+7) for the update
#pragma unroll
    for (int k = 0; k <= P; ++k) {
        Ys[(8 * k + 2 * q) * 8 + l4] = rg.a[k][P][0];
        Ys[(8 * k + 2 * q + 1) * 8 + l4] = rg.a[k][P][1];
    }
    __syncwarp();
    NTPROBE(2);
    build_t(Gs, t8, Ts);
    *reinterpret_cast<double2 *>(tc + 64 * P + 2 * lane) = *reinterpret_cast<const double2 *>(Ts + 2 * lane);
    if constexpr (P + 1 < C::NCB) {
        const double tb0 = Ts[(2 * q) * 8 + l4], tb1 = Ts[(2 * q + 1) * 8 + l4];
#pragma unroll
        for (int cb = P + 1; cb < C::NCB; ++cb) {
            double w0 = 0.0, w1 = 0.0;
#pragma unroll
            for (int k = 0; k <= P; ++k) {
                dmma(w0, w1, rg.a[k][cb][0], rg.a[k][P][0]);
                dmma(w0, w1, rg.a[k][cb][1], rg.a[k][P][1]);
            }
            double *rp = Ra + (2 * q) * C::LDA + 8 * cb + l4;
            w0 += rp[0];
            w1 += rp[C::LDA];
            double p0 = 0.0, p1 = 0.0;
            dmma(p0, p1, w0, tb0);
            dmma(p0, p1, w1, tb1);
            rp[0] -= p0;
            rp[C::LDA] -= p1;
#pragma unroll
            for (int k = 0; k <= P; ++k) {
                const double2 yt = *reinterpret_cast<const double2 *>(Ys + (8 * k + l4) * 8 + 2 * q);
                dmma(rg.a[k][cb][0], rg.a[k][cb][1], -p0, yt.x);
                dmma(rg.a[k][cb][0], rg.a[k][cb][1], -p1, yt.y);
            }
        }
    }
    __syncwarp();
    // publish: R rows 8P..8P+7 -> tile a's head, Y1 columns 8P..8P+7 -> tile b's head
#pragma unroll
    for (int u = 0; u < 2 * C::NCB; ++u) {
        const int e = lane + 32 * u, r = e & 7, c = e >> 3, i = 8 * P + r;
        if (c >= i && c < n) Ahead_a[i + (int64_t)c * lda] = Ra[r * C::LDA + c];
        if (R && i < n && c < n) R[i + (int64_t)c * ldr] = c >= i ? Ra[r * C::LDA + c] : 0.0;
    }
#pragma unroll
    for (int k = 0; k <= P; ++k)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = 8 * k + 2 * q + e, c = 8 * P + l4;
            if (i <= c && c < n) Ahead_b[i + (int64_t)c * lda] = rg.a[k][P][e];
        }
    NTPROBE(3);
    __threadfence();
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile int *>(fme + P) = 1;
    NTPROBE(4);
    if constexpr (P + 1 < C::NCB) node_panel<C, P + 1>(rg, Ahead_a, Ahead_b, lda, n, ws, tau_out, fl, fr, fme, R, ldr, tc);
}

}  // namespace tree

using namespace tree;

// nodes[i]: node id (b) in bottom-up order; prod_l / prod_r: the node ids that
// produce the left / right child's R (-1: a leaf tile, ready); flags[b][NCB].
template <class C>
__global__ void __launch_bounds__(NW * 32)
k_tree_pipe(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a, const int *nodes, int count,
            const int *prod_l, const int *prod_r, int *flags, double *tau_node, int root, double *R, int64_t ldr,
            double *tcache_node) {
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5;
    // logical block index from a ticket taken at start, so that every node a
    // resident warp waits on belongs to a block that started earlier (is resident
    // or done) whatever order the hardware dispatches blocks in
    __shared__ int s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(flags + (count + 1) * C::NCB, 1);
    __syncthreads();
    const int i = s_ticket * NW + warp;
    if (i >= count) return;
    const int b = nodes[i], a = node_a[b];
    double *ws = sm + warp * C::WS;
    NodeRegs<C> rg;
#pragma unroll
    for (int k = 0; k < C::NCB; ++k)
#pragma unroll
        for (int cb = 0; cb < C::NCB; ++cb) rg.a[k][cb][0] = rg.a[k][cb][1] = 0.0;
    const int pl = prod_l[b], pr = prod_r[b];
#ifdef TSQR_NTREE_PROBE
    if (i == 0 && (threadIdx.x & 31) == 0) g_nt_leaf = flags + b * C::NCB;
    if (b == root && (threadIdx.x & 31) == 0) g_nt_root = flags + b * C::NCB;
#endif
    node_panel<C, 0>(rg, A + tile_row0[a], A + tile_row0[b], lda, n, ws, tau_node + (int64_t)b * n,
                     pl >= 0 ? flags + pl * C::NCB : nullptr, pr >= 0 ? flags + pr * C::NCB : nullptr,
                     flags + b * C::NCB, b == root ? R : nullptr, ldr, tcache_node + (int64_t)b * C::NCB * 64);
}

template <class F>
static cudaError_t tree_dispatch(int n, F &&fn) {
    switch ((n + 7) / 8) {
        case 1: return fn(TCfg<1>());
        case 2: return fn(TCfg<2>());
        case 3: return fn(TCfg<3>());
        case 4: return fn(TCfg<4>());
        case 5: return fn(TCfg<5>());
        case 6: return fn(TCfg<6>());
        case 7: return fn(TCfg<7>());
        default: return fn(TCfg<8>());
    }
}

cudaError_t launch_tree_pipe(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a,
                             const int *nodes, int count, const int *prod_l, const int *prod_r, int *flags,
                             double *tau_node, int root, double *R, int64_t ldr, double *tcache_node,
                             cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    return tree_dispatch(n, [&](auto c) {
        using C = decltype(c);
        // node flags (ids <= count) and the block ticket counter after them
        cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * ((size_t)(count + 1) * C::NCB + 1), st);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute((const void *)k_tree_pipe<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)C::BYTES);
        if (e != cudaSuccess) return e;
        k_tree_pipe<C><<<(count + NW - 1) / NW, NW * 32, C::BYTES, st>>>(A, lda, n, tile_row0, node_a, nodes, count,
                                                                         prod_l, prod_r, flags, tau_node, root, R,
                                                                         ldr, tcache_node);
        return cudaGetLastError();
    });
}


// =====================================================================
// Pipelined reduction tree for 64 < n <= 224 (a4, a6): one CTA per node.
// R_b's upper block-triangle sits in shared memory as 8x8 column-major blocks
// (block (k, cb), k <= cb; element (r, c) at [8c + r], which is exactly the
// DMMA fragment order: lane (q, l4) reads rows 2q, 2q+1 of column l4 as one
// double2), R_a's pivot rows of the current panel likewise (one block per
// column block).  Panel P: wait for both children's panel P, load R_a's and
// R_b's row block P (the only rows of them reflectors < 8P have not touched),
// warp 0 runs the 8 structured Householder steps on column block P (rows
// 0..8P+7 of R_b), builds T, then all warps update the trailing column blocks
// with DMMA (W^T = R_a rows + Y^T R_b, W'^T = W^T T, R_a rows -= W'^T,
// R_b -= Y W'^T).  The node's R rows 8P..8P+7 go to the left subtree's head,
// Y1's columns 8P..8P+7 to the right subtree's head, then the panel flag.
namespace wtree {

#ifdef TSQR_TREE_PROBE
__device__ unsigned long long g_tprobe[32 * 8];
#define TPROBE(i) do { if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned long long t; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); g_tprobe[P * 8 + (i)] = t; } } while (0)
#define SPROBE(i) do { if (threadIdx.x == 0 && blockIdx.x == 0 && P == 20 && jj < 4) { unsigned long long t; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); g_tprobe[208 + jj * 8 + (i)] = t; } } while (0)
#else
#define TPROBE(i)
#define SPROBE(i)
#endif

constexpr int NT = 256;
constexpr int MAX_NPAN = 28;

__host__ __device__ constexpr int nblk(int npan) { return npan * (npan + 1) / 2; }
// Block (k, cb) of R_b (k <= cb) is live from panel k (its row block arrives)
// to panel cb (its column is published as Y1), so at panel P only the blocks
// with k <= P <= cb exist: at most max_P (P+1)(npan-P) of them, about a
// quarter of the triangle.  A host-side greedy colouring of these intervals
// (by start panel) gives every block a slot that no live block shares;
// the tables for every npan <= MAX_NPAN sit in constant memory, block (k, cb)
// of width npan at c_slot[slot_off(npan) + cb(cb+1)/2 + k].
__host__ __device__ constexpr int slot_off(int npan) { return (npan - 1) * npan * (npan + 1) / 6; }   // sum nblk(j<npan)
constexpr int SLOT_TABLE = slot_off(MAX_NPAN + 1);
__constant__ unsigned short c_slot[SLOT_TABLE];

__host__ __device__ inline int max_live(int npan) {
    int m = 0;
    for (int P = 0; P < npan; ++P) m = (P + 1) * (npan - P) > m ? (P + 1) * (npan - P) : m;
    return m;
}
__host__ __device__ inline size_t smem_doubles(int npan) {
    return (size_t)(max_live(npan) + npan + 1) * 64 + 64 + 64 + 8 + 2 * 8 * npan + 8 * 9;
}

__device__ __forceinline__ double *blk(double *Rb, int so, int k, int cb) {
    return Rb + 64 * c_slot[so + cb * (cb + 1) / 2 + k];
}

__device__ __forceinline__ void wait_flag_cta(const int *f) {
    if (threadIdx.x == 0) {
        while (*reinterpret_cast<const volatile int *>(f) == 0) __nanosleep(100);
        __threadfence();
    }
    __syncthreads();
}

}  // namespace wtree

template <bool kRobust>
__global__ void __launch_bounds__(wtree::NT, 1)
k_wide_tree_pipe(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a, const int *nodes,
                 int count, const int *prod_l, const int *prod_r, int *flags, double *tau_node, double *tcache_node) {
    using namespace wtree;
    extern __shared__ __align__(16) double sm[];
    const int npan = (n + 7) / 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    double *Rb = sm;                                 // max_live(npan) block slots (see c_slot)
    // npan + 1 blocks shared by the panel's column of R_b, contiguous (PB(k) =
    // Wb + 64 k, k <= P: the steps, T, the update's Y and the Y1 publish read it
    // without slot lookups) and R_a's pivot rows (Ra(cb) = Wb + 64 (cb + 1), cb >= P)
    double *Wb = Rb + 64 * max_live(npan);
    double *Ra = Wb + 64;                            // Ra + 64 cb = Wb + 64 (cb + 1)
    double *Gs = Wb + 64 * (npan + 1), *Ts = Gs + 64, *t8 = Ts + 64, *xs = t8 + 8;   // xs: 2 x 8 npan
    double *part = xs + 2 * 8 * npan;                // per-warp partial dots of a step (8 x 9)
    __shared__ int s_ticket;                         // logical block index (see k_tree_pipe)
    if (threadIdx.x == 0) s_ticket = atomicAdd(flags + (count + 1) * MAX_NPAN, 1);
    __syncthreads();
    const int b = nodes[s_ticket], a = node_a[b];
    const int so = slot_off(npan);
    double *Ha = A + tile_row0[a], *Hb = A + tile_row0[b];
    const int pl = prod_l[b], pr = prod_r[b];
    double *tau_out = tau_node + (int64_t)b * n;
    double *tc = tcache_node + (int64_t)b * npan * 64;
    for (int P = 0; P < npan; ++P) {
        TPROBE(0);
        if (pl >= 0) wait_flag_cta(flags + pl * MAX_NPAN + P);
        if (pr >= 0) wait_flag_cta(flags + pr * MAX_NPAN + P);
        // row block P of R_a and R_b (upper part), column blocks P..npan-1
        // L2 loads (ld.cg: the rows were written by other CTAs of this launch;
        // L1 may hold stale lines), all of a thread's loads in flight at once
        {
            constexpr int MAXL = (64 * MAX_NPAN + NT - 1) / NT;
            double va[MAXL], vb[MAXL];
#pragma unroll
            for (int u = 0; u < MAXL; ++u) {
                const int e = threadIdx.x + u * NT;
                const int cb = P + (e >> 6), cl = (e >> 3) & 7, r = e & 7;
                const int i = 8 * P + r, c = 8 * cb + cl;
                const bool ok = e < 64 * (npan - P) && c >= i && c < n;
                va[u] = ok ? __ldcg(Ha + i + (int64_t)c * lda) : 0.0;
                vb[u] = ok ? __ldcg(Hb + i + (int64_t)c * lda) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < MAXL; ++u) {
                const int e = threadIdx.x + u * NT;
                if (e < 64 * (npan - P)) {
                    const int cb = P + (e >> 6), cl = (e >> 3) & 7, r = e & 7;
                    Ra[64 * cb + 8 * cl + r] = va[u];
                    (cb == P ? Wb + 64 * P : blk(Rb, so, P, cb))[8 * cl + r] = vb[u];
                }
            }
            // the panel's column blocks (k, P), k < P, from their slots into PB
            for (int e = threadIdx.x; e < 32 * P; e += NT) {
                const int k = e >> 5, o = 2 * (e & 31);
                *reinterpret_cast<double2 *>(Wb + 64 * k + o) =
                    *reinterpret_cast<const double2 *>(blk(Rb, so, k, P) + o);
            }
        }
        __syncthreads();
        TPROBE(1);
        // the 8 structured Householder steps of panel P, all warps: warp w owns
        // the panel's row blocks k = w, w + 8, ... (k <= P); per step the warps'
        // partial dots meet in smem, every warp sums them in the same order and
        // runs the same dlarfg, then updates its own blocks
        double *RaP = Ra + 64 * P;
        for (int k = warp; k <= P; k += NT / 32)          // pivot column 8P -> xs[0]
            if (l4 == 0)
                *reinterpret_cast<double2 *>(xs + 8 * k + 2 * q) =
                    *reinterpret_cast<const double2 *>(Wb + 64 * k + 2 * q);
        __syncthreads();
        {
            const int jn = min(8, n - 8 * P);
#pragma unroll 1
            for (int jj = 0; jj < jn; ++jj) {
                const double *xr = xs + (jj & 1) * 8 * npan;
                double *xw = xs + ((jj + 1) & 1) * 8 * npan;
                SPROBE(0);
                double d0 = 0.0, d1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll 4
                for (int k = warp; k <= P; k += NT / 32) {
                    const double2 x = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                    const double2 v = *reinterpret_cast<const double2 *>(Wb + 64 * k + 8 * l4 + 2 * q);
                    d0 = fma(x.x, v.x, d0);
                    d1 = fma(x.y, v.y, d1);
                    s0 = fma(x.x, x.x, s0);
                    s1 = fma(x.y, x.y, s1);
                }
                double dw, sw;
                chunk::quad_sums(dw, sw, d0 + d1, s0 + s1);
                if (q == 0) part[warp * 9 + l4] = dw;
                if (lane == 0) part[warp * 9 + 8] = sw;
                __syncthreads();
                SPROBE(1);
                double d = 0.0, s2 = 0.0;
#pragma unroll
                for (int w2 = 0; w2 < NT / 32; ++w2) {
                    d += part[w2 * 9 + l4];
                    s2 += part[w2 * 9 + 8];
                }
                SPROBE(2);
                const double alpha = RaP[8 * jj + jj];
                const double rj = RaP[8 * l4 + jj];
                House h = house_bf(alpha, s2);
                double sc = 1.0;
                double sx = h.scale;                                        // the scale of the unscaled x
                if (kRobust && wy::house_unsafe(alpha, s2)) {   // block-uniform, rescaled step (R23)
                    double mx = fabs(alpha);
                    for (int k = warp; k <= P; k += NT / 32) {
                        const double2 x = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                        mx = fmax(mx, fmax(fabs(x.x), fabs(x.y)));
                    }
                    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
                    __syncthreads();                             // every warp has read the sums
                    if (lane == 0) part[warp * 9] = mx;
                    __syncthreads();
                    for (int w2 = 0; w2 < NT / 32; ++w2) mx = fmax(mx, part[w2 * 9]);
                    sc = wy::pow2_scale(mx);
                    __syncthreads();                             // every warp has read the maxima
                    d0 = d1 = s0 = s1 = 0.0;
                    for (int k = warp; k <= P; k += NT / 32) {
                        const double2 x = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                        const double2 v = *reinterpret_cast<const double2 *>(Wb + 64 * k + 8 * l4 + 2 * q);
                        d0 = fma(sc * x.x, v.x, d0);
                        d1 = fma(sc * x.y, v.y, d1);
                        s0 = fma(sc * x.x, sc * x.x, s0);
                        s1 = fma(sc * x.y, sc * x.y, s1);
                    }
                    chunk::quad_sums(dw, sw, d0 + d1, s0 + s1);
                    if (q == 0) part[warp * 9 + l4] = dw;
                    if (lane == 0) part[warp * 9 + 8] = sw;
                    __syncthreads();
                    d = 0.0;
                    s2 = 0.0;
#pragma unroll
                    for (int w2 = 0; w2 < NT / 32; ++w2) {
                        d += part[w2 * 9 + l4];
                        s2 += part[w2 * 9 + 8];
                    }
                    h = house_bf(sc * alpha, s2);
                    h.beta = h.beta / sc;
                    sx = h.scale * sc;
                }
                const double w = fma(h.scale, d, rj);
                const double u = (l4 > jj) ? h.tau * sx * w : (l4 == jj ? 1.0 : 0.0);
                const double g = (l4 == jj) ? sx : 0.0;
                const double rnew = (l4 == jj) ? h.beta : fma(-h.tau, w, rj);
                SPROBE(3);
#pragma unroll 4
                for (int k = warp; k <= P; k += NT / 32) {
                    const double2 x = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                    double2 *vp = reinterpret_cast<double2 *>(Wb + 64 * k + 8 * l4 + 2 * q);
                    double2 v = *vp;
                    v.x = fma(g, x.x, fma(-u, x.x, v.x));
                    v.y = fma(g, x.y, fma(-u, x.y, v.y));
                    *vp = v;
                    if (l4 == jj + 1) *reinterpret_cast<double2 *>(xw + 8 * k + 2 * q) = v;
                }
                SPROBE(4);
                if (warp == 0) {
                    if (q == 0 && l4 < jj) Gs[l4 * 8 + jj] = h.scale * d;
                    if (lane == 0) t8[jj] = h.tau;
                }
                __syncthreads();          // xw complete; part free; every warp has read R_a row jj
                if (warp == 0 && q == 0 && l4 >= jj) RaP[8 * l4 + jj] = rnew;   // read again only after the panel
            }
            if (warp == 0) {
                chunk::pad_steps(Gs, t8, jn);
                __syncwarp();
                if (lane < 8 && 8 * P + lane < n) tau_out[8 * P + lane] = t8[lane];
                build_t(Gs, t8, Ts);
                *reinterpret_cast<double2 *>(tc + 64 * P + 2 * lane) =
                    *reinterpret_cast<const double2 *>(Ts + 2 * lane);
            }
        }
        __syncthreads();
        TPROBE(2);
        // trailing column blocks, split over the warps
        {
            const double tb0 = Ts[(2 * q) * 8 + l4], tb1 = Ts[(2 * q + 1) * 8 + l4];
            for (int cb = P + 1 + warp; cb < npan; cb += NT / 32) {
                double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
#pragma unroll 4
                for (int k = 0; k <= P; ++k) {
                    const double2 c = *reinterpret_cast<const double2 *>(blk(Rb, so, k, cb) + 8 * l4 + 2 * q);
                    const double2 y = *reinterpret_cast<const double2 *>(Wb + 64 * k + 8 * l4 + 2 * q);
                    dmma(w0[k & 1], w1[k & 1], c.x, y.x);
                    dmma(w0[k & 1], w1[k & 1], c.y, y.y);
                }
                double2 *rp = reinterpret_cast<double2 *>(Ra + 64 * cb + 8 * l4 + 2 * q);
                double2 rv = *rp;
                const double wt0 = w0[0] + w0[1] + rv.x, wt1 = w1[0] + w1[1] + rv.y;
                double p0 = 0.0, p1 = 0.0;
                dmma(p0, p1, wt0, tb0);
                dmma(p0, p1, wt1, tb1);
                rv.x -= p0;
                rv.y -= p1;
                *rp = rv;
#pragma unroll 4
                for (int k = 0; k <= P; ++k) {
                    const double *yb = Wb + 64 * k;
                    const double yt0 = yb[8 * (2 * q) + l4], yt1 = yb[8 * (2 * q + 1) + l4];
                    double2 *cp = reinterpret_cast<double2 *>(blk(Rb, so, k, cb) + 8 * l4 + 2 * q);
                    double2 c = *cp;
                    dmma(c.x, c.y, -p0, yt0);
                    dmma(c.x, c.y, -p1, yt1);
                    *cp = c;
                }
            }
        }
        __syncthreads();
        TPROBE(3);
        // publish: R rows 8P..8P+7 -> tile a's head, Y1 columns 8P..8P+7 -> tile b's head
        for (int e = threadIdx.x; e < 64 * (npan - P); e += NT) {
            const int cb = P + (e >> 6), cl = (e >> 3) & 7, r = e & 7;
            const int i = 8 * P + r, c = 8 * cb + cl;
            if (c >= i && c < n) Ha[i + (int64_t)c * lda] = Ra[64 * cb + 8 * cl + r];
        }
        for (int e = threadIdx.x; e < 64 * (P + 1); e += NT) {
            const int k = e >> 6, cl = (e >> 3) & 7, r = e & 7;
            const int i = 8 * k + r, c = 8 * P + cl;
            if (i <= c && c < n) Hb[i + (int64_t)c * lda] = Wb[64 * k + 8 * cl + r];
        }
        __threadfence();
        __syncthreads();
        TPROBE(4);
        if (threadIdx.x == 0) *reinterpret_cast<volatile int *>(flags + b * MAX_NPAN + P) = 1;
    }
}

#ifdef TSQR_NTREE_PROBE
extern "C" int tsqr_ntree_probe_dump(unsigned long long *host) {
    return (int)cudaMemcpyFromSymbol(host, g_ntprobe, sizeof(unsigned long long) * 128);
}
#endif
#ifdef TSQR_TREE_PROBE
extern "C" int tsqr_tree_probe_dump(unsigned long long *host) {
    return (int)cudaMemcpyFromSymbol(host, wtree::g_tprobe, sizeof(unsigned long long) * 32 * 8);
}
#endif

bool wide_tree_pipe_ok(int n) { return (n + 7) / 8 <= wtree::MAX_NPAN; }

cudaError_t launch_wide_tree_pipe(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a,
                                  const int *nodes, int count, const int *prod_l, const int *prod_r, int *flags,
                                  double *tau_node, double *tcache_node, bool robust, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const int npan = (n + 7) / 8;
    if (npan > wtree::MAX_NPAN) return cudaErrorInvalidValue;
    static bool tables = false;                      // slot colourings, once per process
    if (!tables) {
        std::vector<unsigned short> tab(wtree::SLOT_TABLE);
        for (int np = 1; np <= wtree::MAX_NPAN; ++np) {
            std::vector<int> end;                        // per slot: last panel of its occupant
            for (int k = 0; k < np; ++k)                 // blocks by start panel k, then by cb
                for (int cb = k; cb < np; ++cb) {
                    int sl = 0;
                    while (sl < (int)end.size() && end[sl] >= k) ++sl;
                    if (sl == (int)end.size()) end.push_back(cb);
                    else end[sl] = cb;
                    tab[wtree::slot_off(np) + cb * (cb + 1) / 2 + k] = (unsigned short)sl;
                }
            if ((int)end.size() > wtree::max_live(np)) return cudaErrorInvalidValue;
        }
        cudaError_t e = cudaMemcpyToSymbol(wtree::c_slot, tab.data(), sizeof(unsigned short) * tab.size());
        if (e != cudaSuccess) return e;
        tables = true;
    }
    const size_t bytes = wtree::smem_doubles(npan) * sizeof(double);
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * ((size_t)(count + 1) * wtree::MAX_NPAN + 1), st);
    if (e != cudaSuccess) return e;
    auto kern = robust ? k_wide_tree_pipe<true> : k_wide_tree_pipe<false>;
    e = cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    kern<<<count, wtree::NT, bytes, st>>>(A, lda, n, tile_row0, node_a, nodes, count, prod_l, prod_r, flags, tau_node,
                                          tcache_node);
    return cudaGetLastError();
}

}  // namespace tsqr
