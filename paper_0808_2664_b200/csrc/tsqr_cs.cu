// Leaf stage of the apply / form-Q kernels (a7, a10) on the chunk-chain
// factor's representation (chunk.cuh).  Product code.
#include "tsqr_kernels.h"
#include "chunk.cuh"

#include <algorithm>
#include <vector>

namespace tsqr {
using namespace chunk;

// ============================================================ apply / form Q
// k_cs_apply<C, kFwd, kX>: the leaf stage of C <- Q^T C (kFwd, (a7)), of the
// explicit Q = Q_leaves [X; 0] (!kFwd, kX, (a10)) or of C <- Q C (!kFwd, !kX:
// the reverse traversal) on the factor's chunk chains
// (C: the factor's chunk configuration).  The 8 warps of a CTA work on the same
// chunk; warp w owns an 8-column slab of C (column block w of the current
// pass) for the chunk's CH rows (registers, DMMA accumulator layout) and the
// slab's "R-row coordinates" C_R (NP x 8, registers: cr[p] = C_R rows
// 8p..8p+7), which play the role R plays in the factor.  Chunk by chunk
// (forward order for Q^T, reverse for Q) the CTA stages the chunk's Y (CH x NP
// from its rows of A) and its panels' T (the factor's cache) into a
// double-buffered smem slot with cp.async, one __syncthreads per chunk; every
// warp then applies the chunk's block reflectors panel by panel to
// [C_R rows 8p..8p+7; its chunk slab].
template <class C>
struct ApplyCs {
    static constexpr int NW = 8, NT = 256;
    // Y twice, so that both DMMA operand reads are bank-conflict free: row-major Yr (CH x NP,
    // row stride LDY = NP + 2) for W^T = C^T Y (rows 2q+e, column l4 of a lane) and column-major
    // Yt (NP x CH, stride LDT = CH + 2) for C -= Y W' (rows l4, columns 2q+e); then the T's
    static constexpr int LDY = C::NP + 2, LDT = C::CH + 2;
    static constexpr int OFF_YT = C::CH * LDY, OFF_T = OFF_YT + C::NP * LDT;
    static constexpr int YS = OFF_T + C::NCB * 64;
    static constexpr size_t BYTES = (size_t)2 * YS * sizeof(double);
};

__device__ __forceinline__ void cp8(double *sm, const double *g, bool ok) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0) : "memory");
}

// Stage the chunk's Y (zero outside [0, hk) x [0, n) and on/above the pivot
// of a column whose pivot lies in the chunk -- chunk row col - r0; fix_dense
// then adds the unit diagonal) and its T's.
template <class C>
__device__ __forceinline__ void stage_chunk(double *slot, const double *Ak, int64_t lda, int hk, int n,
                                            const double *tch, int r0) {
    for (int i = threadIdx.x; i < C::CH * C::NP; i += blockDim.x) {
        const int col = i / C::CH, row = i % C::CH;
        const bool ok = row < hk && col < n && row > col - r0;
        const double *src = Ak + row + (int64_t)(ok ? col : 0) * lda;
        cp8(slot + row * ApplyCs<C>::LDY + col, src, ok);
        cp8(slot + ApplyCs<C>::OFF_YT + col * ApplyCs<C>::LDT + row, src, ok);
    }
    for (int i = threadIdx.x; i < C::NCB * 64; i += blockDim.x) cp8(slot + ApplyCs<C>::OFF_T + i, tch + i, true);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <class C>
__device__ __forceinline__ void fix_dense(double *slot, int n, int r0) {
    for (int c = threadIdx.x; c < C::NP; c += blockDim.x)
        if (c < n && c >= r0 && c < r0 + C::CH) {
            slot[(c - r0) * ApplyCs<C>::LDY + c] = 1.0;
            slot[ApplyCs<C>::OFF_YT + c * ApplyCs<C>::LDT + (c - r0)] = 1.0;
        }
}

template <class C, bool kFwd>
__device__ __forceinline__ void cs_apply_panel(double (&cc)[C::KM][2], double (&cr)[C::NCB][2], int p, int r0,
                                               const double *slot, bool &czero) {
    // czero (form Q only): the chunk's rows of C are still all zero -- they become
    // nonzero with the first panel applied to the chunk -- so W^T = C^T Y is skipped
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    constexpr int KM = C::KM, NP = ApplyCs<C>::LDY, LDT = ApplyCs<C>::LDT;   // Yr / Yt strides
    if (8 * p >= r0 + C::CH) return;           // no reflector of panel p in this chunk
    const bool dense = 8 * p >= r0;            // pivots inside the chunk: row block kb
    const int kb = dense ? (8 * p - r0) >> 3 : -1;
    const double *ys = slot + 8 * p;
    const double *Tg = slot + ApplyCs<C>::OFF_T + 64 * p;
    const double *yt = slot + ApplyCs<C>::OFF_YT + 8 * p * LDT;       // Yt column 8p
    double crp0 = 0.0, crp1 = 0.0;
#pragma unroll
    for (int i = 0; i < C::NCB; ++i) {
        crp0 = (i == p) ? cr[i][0] : crp0;
        crp1 = (i == p) ? cr[i][1] : crp1;
    }
    if (!kFwd && dense) {                     // Q: the pivot rows take their R-row coordinates back
#pragma unroll
        for (int k = 0; k < KM; ++k) {
            cc[k][0] = (k == kb) ? crp0 : cc[k][0];
            cc[k][1] = (k == kb) ? crp1 : cc[k][1];
        }
    }
    double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
    if (!(kFwd == false && czero && !dense)) {
#pragma unroll
        for (int k = 0; k < KM; ++k) {
            const double y0 = ys[(8 * k + 2 * q) * NP + l4], y1 = ys[(8 * k + 2 * q + 1) * NP + l4];
            dmma(w0[k & 1], w1[k & 1], cc[k][0], y0);
            dmma(w0[k & 1], w1[k & 1], cc[k][1], y1);
        }
    }
    czero = false;
    double wt0 = w0[0] + w0[1], wt1 = w1[0] + w1[1];
    if (!dense) {
        wt0 += crp0;
        wt1 += crp1;
    }
    const double tb0 = kFwd ? Tg[(2 * q) * 8 + l4] : Tg[l4 * 8 + 2 * q];
    const double tb1 = kFwd ? Tg[(2 * q + 1) * 8 + l4] : Tg[l4 * 8 + 2 * q + 1];
    double p0 = 0.0, p1 = 0.0;
    dmma(p0, p1, wt0, tb0);
    dmma(p0, p1, wt1, tb1);
    if (!dense) {
        crp0 -= p0;
        crp1 -= p1;
    }
#pragma unroll
    for (int k = 0; k < KM; ++k) {
        const double y0 = yt[(2 * q) * LDT + 8 * k + l4], y1 = yt[(2 * q + 1) * LDT + 8 * k + l4];
        dmma(cc[k][0], cc[k][1], -p0, y0);
        dmma(cc[k][0], cc[k][1], -p1, y1);
    }
    if (kFwd && dense) {                      // Q^T: the pivot rows become R-row coordinates
#pragma unroll
        for (int k = 0; k < KM; ++k) {
            crp0 = (k == kb) ? cc[k][0] : crp0;
            crp1 = (k == kb) ? cc[k][1] : crp1;
        }
    }
#pragma unroll
    for (int i = 0; i < C::NCB; ++i) {
        cr[i][0] = (i == p) ? crp0 : cr[i][0];
        cr[i][1] = (i == p) ? crp1 : cr[i][1];
    }
}

// this lane's slab of C (column col, rows 8kk+2q+{0,1}) for chunk c of a tile
template <class C>
__device__ __forceinline__ void load_cslab(double (&v)[C::KM][2], const double *Cm, int64_t ldc, int k, int64_t row0,
                                           int h, int c, int col, int q) {
    const int r0 = c * C::CH, hk = min(C::CH, h - r0);
    const double *Ck = Cm + row0 + r0 + (int64_t)(col < k ? col : 0) * ldc;
#pragma unroll
    for (int kk = 0; kk < C::KM; ++kk) {
        const int r = 8 * kk + 2 * q;
        v[kk][0] = (col < k && r < hk) ? Ck[r] : 0.0;
        v[kk][1] = (col < k && r + 1 < hk) ? Ck[r + 1] : 0.0;
    }
}

template <class C, bool kFwd, bool kX>
__global__ void __launch_bounds__(256, 2)
k_cs_apply(const double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows,
           const int64_t *tile_chunk0, const int *cta_tile0, const double *tcache, double *Cm, int64_t ldc, int k,
           const double *xbuf) {
    using AC = ApplyCs<C>;
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int tb = cta_tile0[blockIdx.x], te = cta_tile0[blockIdx.x + 1];
    const int pw = blockDim.x >> 2;                               // columns per pass (8 per warp)
    const int npass = (k + pw - 1) / pw;
    const int np = (n + 7) / 8;
    // the CTA's work list: (tile, pass) items, each a chain over the tile's chunks
    int cur = 0;                                                  // staging parity
    bool staged = false;
    auto chunk_of = [&](int t, int cc_) {
        const int nch = (tile_rows[t] + C::CH - 1) / C::CH;
        return kFwd ? cc_ : nch - 1 - cc_;
    };
    double ccv[C::KM][2];
    if (!kX && tb < te) load_cslab<C>(ccv, Cm, ldc, k, tile_row0[tb], tile_rows[tb], chunk_of(tb, 0), 8 * warp + l4, q);
    for (int t = tb; t < te; ++t) {
        const int h = tile_rows[t];
        const int nch = (h + C::CH - 1) / C::CH;
        const int64_t row0 = tile_row0[t];
        for (int pass = 0; pass < npass; ++pass) {
            const int col = pw * pass + 8 * warp + l4;            // this lane's column of C
            const bool okc = col < k;
            double cr[C::NCB][2];
#pragma unroll
            for (int i = 0; i < C::NCB; ++i) {
                cr[i][0] = cr[i][1] = 0.0;
                const int r = 8 * i + 2 * q;
                if (kX) {                                         // C_R := X (rows < n, columns < n)
                    const double *X = xbuf + (int64_t)t * n * n;
                    cr[i][0] = (okc && r < n) ? X[r + (int64_t)col * n] : 0.0;
                    cr[i][1] = (okc && r + 1 < n) ? X[r + 1 + (int64_t)col * n] : 0.0;
                } else if (!kFwd) {
                    // Q C: C_R := the tile's head rows, including the padding rows n..8np-1 of
                    // the last panel's row block: they are passive in C_R (zero Y columns and T
                    // rows) and the dense chunk takes the whole row block back
                    const double *Ch = Cm + row0 + (int64_t)col * ldc;
                    cr[i][0] = (okc && r < h) ? Ch[r] : 0.0;
                    cr[i][1] = (okc && r + 1 < h) ? Ch[r + 1] : 0.0;
                }
            }
            for (int cc_ = 0; cc_ < nch; ++cc_) {
                const int c = chunk_of(t, cc_);
                const int r0 = c * C::CH, hk = min(C::CH, h - r0);
                const bool dense = r0 < C::NP;                    // a head chunk (holds pivots)
                if (!staged)
                    stage_chunk<C>(sm + cur * AC::YS, A + row0 + r0, lda, hk, n,
                                   tcache + (tile_chunk0[t] + c) * (C::NCB * 64), r0);
                // prefetch the next chunk of the work list: Y/T into the other
                // slot, C into registers
                int tn = t, pn = pass, cn = cc_ + 1;
                if (cn == nch) { cn = 0; if (++pn == npass) { pn = 0; ++tn; } }
                double ccn[C::KM][2];
                if (tn < te) {
                    const int cnn = chunk_of(tn, cn), hn = tile_rows[tn], r0n = cnn * C::CH;
                    stage_chunk<C>(sm + (cur ^ 1) * AC::YS, A + tile_row0[tn] + r0n, lda, min(C::CH, hn - r0n), n,
                                   tcache + (tile_chunk0[tn] + cnn) * (C::NCB * 64), r0n);
                    if (!kX) load_cslab<C>(ccn, Cm, ldc, k, tile_row0[tn], hn, cnn, pw * pn + 8 * warp + l4, q);
                    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
                    staged = true;
                } else {
                    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                    staged = false;
                }
                if (kX) {
#pragma unroll
                    for (int kk = 0; kk < C::KM; ++kk) ccv[kk][0] = ccv[kk][1] = 0.0;
                }
                __syncthreads();
                double *slot = sm + cur * AC::YS;
                if (dense) {
                    fix_dense<C>(slot, n, r0);
                    __syncthreads();
                }
                double *Ck = Cm + row0 + r0;
                bool czero = kX;
#pragma unroll 1
                for (int pp = 0; pp < np; ++pp)
                    cs_apply_panel<C, kFwd>(ccv, cr, kFwd ? pp : np - 1 - pp, r0, slot, czero);
#pragma unroll
                for (int kk = 0; kk < C::KM; ++kk)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int r = 8 * kk + 2 * q + e;
                        if (okc && r < hk && (!kFwd || r0 + r >= n)) Ck[r + (int64_t)col * ldc] = ccv[kk][e];
                    }
                if (!kX && tn < te) {
#pragma unroll
                    for (int kk = 0; kk < C::KM; ++kk) {
                        ccv[kk][0] = ccn[kk][0];
                        ccv[kk][1] = ccn[kk][1];
                    }
                }
                __syncthreads();                                  // the slot may be refilled
                cur ^= 1;
            }
            if (kFwd && okc) {                                    // the tile's head rows receive C_R
#pragma unroll
                for (int i = 0; i < C::NCB; ++i)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int r = 8 * i + 2 * q + e;
                        if (r < n) Cm[row0 + r + (int64_t)col * ldc] = cr[i][e];
                    }
            }
        }
    }
}

// ================================================================= launchers
// The apply kernel on the chain factor's representation (chunk.cuh, 32-row chunks).
template <class F>
static cudaError_t chain_cfg_dispatch(int n, F &&fn) {
    const int ncb = (n + 7) / 8;
    switch (ncb) {
        case 1: case 2: return fn(chunk::Cfg<2, 8, 8>());
        case 3: case 4: return fn(chunk::Cfg<TSQR_CFG32>());
        case 5: case 6: return fn(chunk::Cfg<6, 6, 8>());
        case 7: return fn(chunk::Cfg<7, 5, 8>());
        default: return fn(chunk::Cfg<8, 5, 8, 1>());
    }
}

int cs_apply_grid(int n) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = chain_cfg_dispatch(n, [&](auto c) {
        using C = decltype(c);
        using AC = ApplyCs<C>;
        cudaError_t r = cudaFuncSetAttribute((const void *)k_cs_apply<C, true, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AC::BYTES);
        if (r != cudaSuccess) return r;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cs_apply<C, true, false>, AC::NT, AC::BYTES);
    });
    if (e != cudaSuccess || occ < 1) occ = 1;
    return sms * occ;
}

cudaError_t launch_cs_apply(const ChainApplyArgs &f, cudaStream_t st) {
    return chain_cfg_dispatch(f.n, [&](auto c) {
        using C = decltype(c);
        using AC = ApplyCs<C>;
        auto kern = f.forward ? k_cs_apply<C, true, false>
                              : (f.xbuf ? k_cs_apply<C, false, true> : k_cs_apply<C, false, false>);
        cudaError_t e = cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)AC::BYTES);
        if (e != cudaSuccess) return e;
        const int nw = f.k >= 64 ? 8 : (f.k + 7) / 8;           // one warp per 8-column slab
        kern<<<f.grid, 32 * (nw < 1 ? 1 : nw), AC::BYTES, st>>>(f.A, f.lda, f.n, f.tile_row0, f.tile_rows, f.tile_chunk0, f.cta_tile0,
                                                f.tcache, f.C, f.ldc, f.k, f.xbuf);
        return cudaGetLastError();
    });
}

}  // namespace tsqr
