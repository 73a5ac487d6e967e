// Leaf-stage kernels of the B200 TSQR path on the register-resident chunk
// engine (chunk.cuh).  Product code.
//
//  k_chain_factor  (a2)+(a3)+(a6 for each tile): persistent CTAs; CTA i owns a
//      contiguous run of tiles and walks their chunks in order; chunk g goes to
//      warp g mod NW.  The running R of a tile sits in one of two smem buffers
//      (tiles alternate); consecutive chunks of a tile hand R row block p over
//      through a counter in smem, so the warps form a software pipeline (chunk g+1
//      runs panel p as soon as chunk g has finished panel p).  The last chunk
//      of a tile writes the tile's R into the upper triangle of its head rows.
#include "tsqr_kernels.h"
#include "chunk.cuh"

#include <algorithm>
#include <vector>

namespace tsqr {
using namespace chunk;

template <class C, int P>
__device__ __forceinline__ void chunk_panels(Chunk<C> &ch, int r0, bool last, double *Rb, const Sync &sy,
                                             double *ws, double *tau_out, int n, double *Ahead, int64_t lda,
                                             double *tg) {
    const int lane = threadIdx.x & 31;
    const int kind = (8 * P < r0) ? 0 : (8 * P < r0 + C::CH ? 1 : 2);
    const int kb = (8 * P - r0) >> 3;
    factor_panel<C, P>(ch, kind, kb, Rb, ws, tau_out, n, sy, last, tg);
    if (last) {                                   // R rows 8P .. 8P+7 of the tile are final
        const int w = n - 8 * P;
        for (int e = lane; e < 8 * w; e += 32) {
            const int i = 8 * P + (e & 7), c = 8 * P + (e >> 3);
            if (i <= c && i < n) Ahead[i + (int64_t)c * lda] = Rb[i * C::LDR + c];
        }
        sync_publish(sy.tr + P, sy.s + 1);        // the buffer's next user may overwrite them
    }
    PROBE(8);
    if constexpr (P + 1 < C::NCB) chunk_panels<C, P + 1>(ch, r0, last, Rb, sy, ws, tau_out, n, Ahead, lda, tg);
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1)
k_chain_factor(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows,
               const int64_t *tile_chunk0, const int *cta_tile0, double *tau, double *tcache) {
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane & 3, l4 = lane >> 2;
    int *sync = reinterpret_cast<int *>(sm + C::OFF_SYNC);
    for (int i = threadIdx.x; i < 2 * C::SYNC_INTS; i += C::NT) sync[i] = 0;
    PROBE_INIT();
    __syncthreads();
    double *ws = sm + C::OFF_WS + warp * C::WS;
    const int tb = cta_tile0[blockIdx.x], te = cta_tile0[blockIdx.x + 1];
    int cnt[2] = {0, 0};
    int g = 0;
    for (int t = tb; t < te; ++t) {
        const int b = (t - tb) & 1;
        const int h = tile_rows[t];
        const int nch = (h + C::CH - 1) / C::CH;
        const int64_t row0 = tile_row0[t];
        for (int c = 0; c < nch; ++c, ++g) {
            const int s = cnt[b]++;
            if (g % C::NW != warp) continue;
            const int r0 = c * C::CH, hk = min(C::CH, h - r0);
            Chunk<C> ch;
            const double *src = A + row0 + r0;
#pragma unroll
            for (int k = 0; k < C::KM; ++k)
#pragma unroll
                for (int cb = 0; cb < C::NCB; ++cb) {
                    const int r = 8 * k + 2 * q, col = 8 * cb + l4;
                    const double *p = src + r + (int64_t)col * lda;
                    ch.a[k][cb][0] = (col < n && r < hk) ? __ldg(p) : 0.0;
                    ch.a[k][cb][1] = (col < n && r + 1 < hk) ? __ldg(p + 1) : 0.0;
                }
            PROBE(0);
            double *tau_out = tau + (tile_chunk0[t] + c) * n;
            const Sync sy{sync + b * C::SYNC_INTS, sync + b * C::SYNC_INTS + C::NP, s};
            double *tg = tcache ? tcache + (tile_chunk0[t] + c) * (C::NCB * 64) : nullptr;
            chunk_panels<C, 0>(ch, r0, c == nch - 1, sm + b * C::RBUF, sy, ws, tau_out, n, A + row0, lda, tg);
            double *dst = A + row0 + r0;
#pragma unroll
            for (int k = 0; k < C::KM; ++k)
#pragma unroll
                for (int cb = 0; cb < C::NCB; ++cb)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int r = 8 * k + 2 * q + e, col = 8 * cb + l4;
                        if (col < n && r < hk && r0 + r > col) dst[r + (int64_t)col * lda] = ch.a[k][cb][e];
                    }
        }
    }
    PROBE_FLUSH();
}

// ============================================================ apply / form Q
// k_chain_apply<C, kFwd>: the leaf stage of C <- Q^T C (kFwd, (a7)) or of
// Q = Q_leaves [X; 0] (!kFwd, form Q (a10)) on the same chunk chains.  Work
// items are (slab of SW = 8 NCBC columns, tile); every item is a chain over
// the tile's chunks (forward order for Q^T, reverse for Q) handing the
// "R-row coordinates" C_R (NP x SW, smem) from chunk to chunk exactly as the
// factor hands R over: the chunk's panel p acts on [C_R rows 8p..8p+7; chunk]
// with the block reflector I - Y T^T Y^T (Q^T) or I - Y T Y^T (Q), Y read from
// the chunk's rows of A, T from the factor's cache.
template <class C, int NCBC>
struct ApplyCfg {
    static constexpr int SW = 8 * NCBC;                  // slab width (columns of C)
    static constexpr int LDC = SW + 2;                   // C_R row-major ld
    static constexpr int CBUF = C::NP * LDC;
    static constexpr int YS = 0, WS = C::CH * 8;         // per-warp: Y panel (CH x 8 row-major)
    static constexpr int OFF_WS = 2 * CBUF;
    static constexpr int OFF_SYNC = OFF_WS + C::NW * WS;
    static constexpr size_t BYTES = (size_t)OFF_SYNC * sizeof(double) + 2 * C::NCB * sizeof(int);
};

template <class C, class AC, int P, bool kFwd>
__device__ __forceinline__ void apply_panel(double (&cc)[C::KM][AC::SW / 8][2], int r0, int hk, const double *Ak,
                                            int64_t lda, int n, const double *tg, double *CR, double *ws,
                                            int *tr, int s, bool first, bool last, const double *X, int c0,
                                            int kc, double *Chead, int64_t ldc) {
    constexpr int NC = AC::SW / 8;
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int kind = (8 * P < r0) ? 0 : (8 * P < r0 + C::CH ? 1 : 2);
    const int kb = (8 * P - r0) >> 3;
    sync_wait(tr + P, s);
    if (first && !kFwd) {                  // C_R := X (the tile's head coordinates) for this row block
        for (int e = lane; e < 8 * AC::SW; e += 32) {
            const int r = 8 * P + (e / AC::SW), col = e % AC::SW;
            CR[r * AC::LDC + col] = (r < n && c0 + col < n && col < kc) ? X[r + (int64_t)(c0 + col) * n] : 0.0;
        }
        __syncwarp();
    }
    if (kind != 2) {
        double yv[C::KM][2];
        const int piv = 8 * kb + l4;
        const int col = 8 * P + l4;
#pragma unroll
        for (int k = 0; k < C::KM; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = 8 * k + 2 * q + e;
                double v = (col < n && r < hk) ? __ldg(Ak + r + (int64_t)col * lda) : 0.0;
                if (kind == 1) v = r > piv ? v : (r == piv && col < n ? 1.0 : 0.0);
                yv[k][e] = v;
            }
        double *Ys = ws + AC::YS;
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            Ys[(8 * k + 2 * q) * 8 + l4] = yv[k][0];
            Ys[(8 * k + 2 * q + 1) * 8 + l4] = yv[k][1];
        }
        if (!kFwd && kind == 1) {          // the pivot rows take their R-row coordinates back
#pragma unroll
            for (int k = 0; k < C::KM; ++k)
                if (k == kb) {
#pragma unroll
                    for (int cb = 0; cb < NC; ++cb) {
                        cc[k][cb][0] = CR[(8 * P + 2 * q) * AC::LDC + 8 * cb + l4];
                        cc[k][cb][1] = CR[(8 * P + 2 * q + 1) * AC::LDC + 8 * cb + l4];
                    }
                }
        }
        __syncwarp();
        double yt[C::KM][2];
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            const double2 v = *reinterpret_cast<const double2 *>(Ys + (8 * k + l4) * 8 + 2 * q);
            yt[k][0] = v.x;
            yt[k][1] = v.y;
        }
        // B operand of W'^T = W^T op(T): op = T (Q^T, W' = T^T W) or T^T (Q, W' = T W)
        const double tb0 = kFwd ? tg[(2 * q) * 8 + l4] : tg[l4 * 8 + 2 * q];
        const double tb1 = kFwd ? tg[(2 * q + 1) * 8 + l4] : tg[l4 * 8 + 2 * q + 1];
#pragma unroll
        for (int cb = 0; cb < NC; ++cb) {
            double w0 = 0.0, w1 = 0.0;
#pragma unroll
            for (int k = 0; k < C::KM; ++k) {
                dmma(w0, w1, cc[k][cb][0], yv[k][0]);
                dmma(w0, w1, cc[k][cb][1], yv[k][1]);
            }
            double *crp = CR + (8 * P + 2 * q) * AC::LDC + 8 * cb + l4;
            if (kind == 0) {
                w0 += crp[0];
                w1 += crp[AC::LDC];
            }
            double p0 = 0.0, p1 = 0.0;
            dmma(p0, p1, w0, tb0);
            dmma(p0, p1, w1, tb1);
            if (kind == 0) {
                crp[0] -= p0;
                crp[AC::LDC] -= p1;
            }
#pragma unroll
            for (int k = 0; k < C::KM; ++k) {
                dmma(cc[k][cb][0], cc[k][cb][1], -p0, yt[k][0]);
                dmma(cc[k][cb][0], cc[k][cb][1], -p1, yt[k][1]);
            }
        }
        if (kFwd && kind == 1) {           // the pivot rows become R-row coordinates
#pragma unroll
            for (int k = 0; k < C::KM; ++k)
                if (k == kb) {
#pragma unroll
                    for (int cb = 0; cb < NC; ++cb) {
                        CR[(8 * P + 2 * q) * AC::LDC + 8 * cb + l4] = cc[k][cb][0];
                        CR[(8 * P + 2 * q + 1) * AC::LDC + 8 * cb + l4] = cc[k][cb][1];
                    }
                }
        }
    }
    if (kFwd && last) {                    // the tile's head rows receive C_R (rows < n)
        __syncwarp();
        for (int e = lane; e < 8 * AC::SW; e += 32) {
            const int r = 8 * P + (e & 7), col = e >> 3;
            if (r < n && col < kc) Chead[r + (int64_t)col * ldc] = CR[r * AC::LDC + col];
        }
    }
    sync_publish(tr + P, s + 1);
}

template <class C, class AC, int P, bool kFwd>
__device__ __forceinline__ void apply_panels(double (&cc)[C::KM][AC::SW / 8][2], int r0, int hk, const double *Ak,
                                             int64_t lda, int n, const double *tg, double *CR, double *ws, int *tr,
                                             int s, bool first, bool last, const double *X, int c0, int kc,
                                             double *Chead, int64_t ldc) {
    constexpr int PP = kFwd ? P : C::NCB - 1 - P;
    apply_panel<C, AC, PP, kFwd>(cc, r0, hk, Ak, lda, n, tg + PP * 64, CR, ws, tr, s, first, last, X, c0, kc, Chead,
                                  ldc);
    if constexpr (P + 1 < C::NCB)
        apply_panels<C, AC, P + 1, kFwd>(cc, r0, hk, Ak, lda, n, tg, CR, ws, tr, s, first, last, X, c0, kc, Chead,
                                         ldc);
}

template <class C, class AC, bool kFwd>
__global__ void __launch_bounds__(C::NT, 1)
k_chain_apply(const double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows,
              const int64_t *tile_chunk0, const int *cta_tile0, const double *tcache, double *Cm, int64_t ldc,
              int k, const double *xbuf) {
    constexpr int NC = AC::SW / 8;
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane & 3, l4 = lane >> 2;
    int *sync = reinterpret_cast<int *>(sm + AC::OFF_SYNC);
    for (int i = threadIdx.x; i < 2 * C::NCB; i += C::NT) sync[i] = 0;
    __syncthreads();
    double *ws = sm + AC::OFF_WS + warp * AC::WS;
    const int tb = cta_tile0[blockIdx.x], te = cta_tile0[blockIdx.x + 1];
    const int nslab = (k + AC::SW - 1) / AC::SW;
    int cnt[2] = {0, 0};
    int g = 0, item = 0;
    for (int sl = 0; sl < nslab; ++sl) {
        const int c0 = sl * AC::SW, kc = min(AC::SW, k - c0);
        for (int t = tb; t < te; ++t, ++item) {
            const int b = item & 1;
            const int h = tile_rows[t];
            const int nch = (h + C::CH - 1) / C::CH;
            const int64_t row0 = tile_row0[t];
            for (int cc_ = 0; cc_ < nch; ++cc_, ++g) {
                const int s = cnt[b]++;
                if (g % C::NW != warp) continue;
                const int c = kFwd ? cc_ : nch - 1 - cc_;
                const int r0 = c * C::CH, hk = min(C::CH, h - r0);
                double cc[C::KM][NC][2];
                double *Ck = Cm + row0 + r0 + (int64_t)c0 * ldc;
#pragma unroll
                for (int kk = 0; kk < C::KM; ++kk)
#pragma unroll
                    for (int cb = 0; cb < NC; ++cb) {
                        const int r = 8 * kk + 2 * q, col = 8 * cb + l4;
                        const double *p = Ck + r + (int64_t)col * ldc;
                        cc[kk][cb][0] = (kFwd && col < kc && r < hk) ? p[0] : 0.0;
                        cc[kk][cb][1] = (kFwd && col < kc && r + 1 < hk) ? p[1] : 0.0;
                    }
                const double *tg = tcache + (tile_chunk0[t] + c) * (C::NCB * 64);
                const double *X = kFwd ? nullptr : xbuf + (int64_t)t * n * n;
                apply_panels<C, AC, 0, kFwd>(cc, r0, hk, A + row0 + r0, lda, n, tg, sm + b * AC::CBUF, ws,
                                             sync + b * C::NCB, s, cc_ == 0, cc_ == nch - 1, X, c0, kc,
                                             Cm + row0 + (int64_t)c0 * ldc, ldc);
#pragma unroll
                for (int kk = 0; kk < C::KM; ++kk)
#pragma unroll
                    for (int cb = 0; cb < NC; ++cb)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int r = 8 * kk + 2 * q + e, col = 8 * cb + l4;
                            if (col < kc && r < hk && (!kFwd || r0 + r >= n)) Ck[r + (int64_t)col * ldc] = cc[kk][cb][e];
                        }
            }
        }
    }
}

// ================================================================= launchers
template <class C>
static cudaError_t launch_chain_factor_t(const ChainArgs &f, cudaStream_t st) {
    const size_t sm = C::BYTES;
    cudaError_t e = cudaFuncSetAttribute((const void *)k_chain_factor<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm);
    if (e != cudaSuccess) return e;
    k_chain_factor<C><<<f.grid, C::NT, sm, st>>>(f.A, f.lda, f.n, f.tile_row0, f.tile_rows, f.tile_chunk0,
                                                 f.cta_tile0, f.tau, f.tcache);
    return cudaGetLastError();
}

int chain_chunk_rows(int n) { return n <= 32 ? 64 : 32; }

// Dispatch on (n, chunk rows) to the compiled configurations.
template <class F>
static cudaError_t chain_dispatch(int n, int chunk_rows, F &&fn) {
    const int ncb = (n + 7) / 8;
    if (chunk_rows == 64) {
        switch (ncb) {
            case 1: case 2: return fn(Cfg<2, 8, 8>());
            case 3: case 4: return fn(Cfg<4, 8, 8>());
            default: return cudaErrorInvalidValue;
        }
    }
    switch (ncb) {
        case 1: case 2: return fn(Cfg<2, 4, 8>());
        case 3: case 4: return fn(Cfg<4, 4, 8>());
        case 5: case 6: return fn(Cfg<6, 4, 8>());
        case 7: return fn(Cfg<7, 4, 8>());
        default: return fn(Cfg<8, 4, 8>());
    }
}

cudaError_t launch_chain_factor(const ChainArgs &f, cudaStream_t st) {
    return chain_dispatch(f.n, f.chunk_rows, [&](auto c) { return launch_chain_factor_t<decltype(c)>(f, st); });
}

template <class C, bool kFwd>
static cudaError_t launch_chain_apply_t(const ChainApplyArgs &f, cudaStream_t st) {
    using AC = ApplyCfg<C, C::KM == 4 ? 8 : 4>;
    const size_t sm = AC::BYTES;
    cudaError_t e = cudaFuncSetAttribute((const void *)k_chain_apply<C, AC, kFwd>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_chain_apply<C, AC, kFwd><<<f.grid, C::NT, sm, st>>>(f.A, f.lda, f.n, f.tile_row0, f.tile_rows, f.tile_chunk0,
                                                          f.cta_tile0, f.tcache, f.C, f.ldc, f.k, f.xbuf);
    return cudaGetLastError();
}

cudaError_t launch_chain_apply(const ChainApplyArgs &f, cudaStream_t st) {
    return chain_dispatch(f.n, f.chunk_rows, [&](auto c) {
        using C = decltype(c);
        return f.forward ? launch_chain_apply_t<C, true>(f, st) : launch_chain_apply_t<C, false>(f, st);
    });
}

int chain_ncb(int n, int chunk_rows) {
    int ncb = 0;
    chain_dispatch(n, chunk_rows, [&](auto c) {
        ncb = decltype(c)::NCB;
        return cudaSuccess;
    });
    return ncb;
}

// Resident CTAs of the factor kernel on the current device (the persistent grid).
int chain_grid(int n, int chunk_rows) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = chain_dispatch(n, chunk_rows, [&](auto c) {
        using C = decltype(c);
        cudaError_t r = cudaFuncSetAttribute((const void *)k_chain_factor<C>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
        if (r != cudaSuccess) return r;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_chain_factor<C>, C::NT, C::BYTES);
    });
    if (e != cudaSuccess || occ < 1) occ = 1;
    return sms * occ;
}

// Balanced split of the tiles over `grid` CTAs by chunk count (contiguous runs).
void chain_partition(const std::vector<int64_t> &tile_rows, int chunk_rows, int grid, std::vector<int> &cta_tile0) {
    const int L = (int)tile_rows.size();
    std::vector<int64_t> pre(L + 1, 0);
    for (int t = 0; t < L; ++t) pre[t + 1] = pre[t] + (tile_rows[t] + chunk_rows - 1) / chunk_rows;
    cta_tile0.assign(grid + 1, L);
    cta_tile0[0] = 0;
    int t = 0;
    for (int i = 1; i < grid; ++i) {
        const int64_t target = (pre[L] * i + grid - 1) / grid;
        while (t < L && pre[t] < target) ++t;
        // choose the closer cut of t-1 / t
        if (t > 0 && t < L && (target - pre[t - 1]) < (pre[t] - target)) --t;
        t = std::max(t, cta_tile0[i - 1]);
        cta_tile0[i] = t;
    }
    cta_tile0[grid] = L;
}

}  // namespace tsqr
