// Leaf stage of the apply / form-Q kernels (a7, a10) on the chunk-chain
// factor's representation (chunk.cuh).  Product code.
#include "tsqr_kernels.h"
#include "chunk.cuh"
#include "tma.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace tsqr {
using namespace chunk;

// TSQR_NO_TMA=1: per-element cp.async staging here too (A/B checks)
static bool apply_no_bulk() {
    static const int v = [] {
        const char *e = std::getenv("TSQR_NO_TMA");
        return (e && *e == '1') ? 1 : 0;
    }();
    return v != 0;
}

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
    // Y column-major (Yt: NP x CH, stride LDT = CH + 2), read bank-conflict free by both DMMA
    // operand patterns: W^T = C^T Y (a lane's rows 2q, 2q+1 of column l4: one 16-byte load;
    // LDT = 2 mod 4 doubles spreads the 8 columns over the banks) and C -= Y W' (rows l4,
    // columns 2q+e); then the T's.
    static constexpr int LDT = C::CH + 2;
#ifdef TSQR_APPLY_OLD_SLOT
    static constexpr int OFF_YT = C::CH * (C::NP + 2);   // variant: the old row-major region kept, unused
#else
    static constexpr int OFF_YT = 0;
#endif
    static constexpr int OFF_T = OFF_YT + C::NP * LDT;
    static constexpr int YS = OFF_T + C::NCB * 64;
    static_assert(LDT % 2 == 0 && OFF_YT % 2 == 0 && OFF_T % 2 == 0 && YS % 2 == 0, "bulk copy targets 16-byte aligned");
    static constexpr size_t BYTES = (size_t)2 * YS * sizeof(double) + 2 * sizeof(uint64_t);   // + two mbarriers
};

__device__ __forceinline__ void bulk_g2s(double *dst, const double *src, unsigned bytes, uint64_t *bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}

// Bulk staging (even row starts, even lda, hk even): each of Y's n columns (hk rows,
// 16-byte aligned both sides) is one cp.async.bulk into the column-major copy Yt,
// the T's one more; all complete on the slot's mbarrier.  After the wait,
// finish_bulk_stage() zeroes what the factor stores but Y does not contain (rows past
// the tile, the R entries on/above the pivots of a head chunk), sets the unit
// diagonal and writes the row-major copy Yr.
template <class C>
__device__ __forceinline__ void stage_chunk_bulk(double *slot, const double *Ak, int64_t lda, int hk, int n,
                                                 const double *tch, uint64_t *bar) {
    using AC = ApplyCs<C>;
    if (threadIdx.x == 0)
        tma::mbar_arrive_expect_tx(bar, (unsigned)(n * hk + C::NCB * 64) * (unsigned)sizeof(double));
    tma::fence_proxy_async_smem();
    for (int col = threadIdx.x; col <= n; col += blockDim.x) {
        if (col < n) bulk_g2s(slot + AC::OFF_YT + col * AC::LDT, Ak + (int64_t)col * lda, (unsigned)hk * 8u, bar);
        else bulk_g2s(slot + AC::OFF_T, tch, C::NCB * 64 * 8u, bar);
    }
}
// (only for a ragged or head chunk: a full chunk below the pivots is Y as staged)
template <class C>
__device__ __forceinline__ void finish_bulk_stage(double *slot, int hk, int n, int r0) {
    using AC = ApplyCs<C>;
    for (int i = threadIdx.x; i < C::CH * C::NP; i += blockDim.x) {
        const int col = i / C::CH, row = i - col * C::CH;
        const double v = slot[AC::OFF_YT + col * AC::LDT + row];
        const double y = (col < n && row < hk && row > col - r0) ? v : ((col < n && row == col - r0) ? 1.0 : 0.0);
        slot[AC::OFF_YT + col * AC::LDT + row] = y;
    }
}

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
        cp8(slot + ApplyCs<C>::OFF_YT + col * ApplyCs<C>::LDT + row, src, ok);
    }
    for (int i = threadIdx.x; i < C::NCB * 64; i += blockDim.x) cp8(slot + ApplyCs<C>::OFF_T + i, tch + i, true);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <class C>
__device__ __forceinline__ void fix_dense(double *slot, int n, int r0) {
    for (int c = threadIdx.x; c < C::NP; c += blockDim.x)
        if (c < n && c >= r0 && c < r0 + C::CH) slot[ApplyCs<C>::OFF_YT + c * ApplyCs<C>::LDT + (c - r0)] = 1.0;
}

template <class C, bool kFwd, int p>
__device__ __forceinline__ void cs_apply_panel(double (&cc)[C::KM][2], double (&cr)[C::NCB][2], int r0,
                                               const double *slot, bool &czero) {
    // czero (form Q only): the chunk's rows of C are still all zero -- they become
    // nonzero with the first panel applied to the chunk -- so W^T = C^T Y is skipped
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    constexpr int KM = C::KM, LDT = ApplyCs<C>::LDT;                          // Yt stride
    if (8 * p >= r0 + C::CH) return;           // no reflector of panel p in this chunk
    const bool dense = 8 * p >= r0;            // pivots inside the chunk: row block kb
    const int kb = dense ? (8 * p - r0) >> 3 : -1;
    const double *ycol = slot + ApplyCs<C>::OFF_YT + (8 * p + l4) * LDT;   // this lane's column of the panel
    const double *Tg = slot + ApplyCs<C>::OFF_T + 64 * p;
    const double *yt = slot + ApplyCs<C>::OFF_YT + 8 * p * LDT;       // Yt column 8p
    double crp0 = cr[p][0], crp1 = cr[p][1];
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
            const double2 yv = *reinterpret_cast<const double2 *>(ycol + 8 * k + 2 * q);
            const double y0 = yv.x, y1 = yv.y;
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
    cr[p][0] = crp0;
    cr[p][1] = crp1;
}

// the chunk's panels in order (Q^T: 0 .. np-1) or reverse (Q: np-1 .. 0), the
// panel index a compile-time constant so C_R's row block is a plain register
template <class C, bool kFwd, int I>
__device__ __forceinline__ void cs_apply_panels(double (&cc)[C::KM][2], double (&cr)[C::NCB][2], int r0, int np,
                                                const double *slot, bool &czero) {
    if constexpr (kFwd) {
        if (I < np) cs_apply_panel<C, kFwd, I>(cc, cr, r0, slot, czero);
    } else {
        constexpr int p = C::NCB - 1 - I;
        if (p < np) cs_apply_panel<C, kFwd, p>(cc, cr, r0, slot, czero);
    }
    if constexpr (I + 1 < C::NCB) cs_apply_panels<C, kFwd, I + 1>(cc, cr, r0, np, slot, czero);
}

// this lane's slab of C (column col, rows 8kk+2q+{0,1}) for chunk c of a tile
// (vec: C's rows pairs 16-byte aligned -- even tile starts, even ldc, aligned base)
template <class C>
__device__ __forceinline__ void load_cslab(double (&v)[C::KM][2], const double *Cm, int64_t ldc, int k, int64_t row0,
                                           int h, int c, int col, int q, bool vec) {
    const int r0 = c * C::CH, hk = min(C::CH, h - r0);
    const double *Ck = Cm + row0 + r0 + (int64_t)(col < k ? col : 0) * ldc;
    if (vec && hk == C::CH) {
#pragma unroll
        for (int kk = 0; kk < C::KM; ++kk) {
            const double2 x = col < k ? *reinterpret_cast<const double2 *>(Ck + 8 * kk + 2 * q) : make_double2(0.0, 0.0);
            v[kk][0] = x.x;
            v[kk][1] = x.y;
        }
        return;
    }
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
           const double *xbuf, int bulk, int vecc) {
    using AC = ApplyCs<C>;
    extern __shared__ __align__(16) double sm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + 2 * AC::YS);
    if (bulk) {                                                   // padding columns of Yt stay zero
        for (int i = threadIdx.x; i < 2 * (C::NP - n) * AC::LDT; i += blockDim.x) {
            const int sl = i / ((C::NP - n) * AC::LDT), j = i - sl * (C::NP - n) * AC::LDT;
            sm[sl * AC::YS + AC::OFF_YT + n * AC::LDT + j] = 0.0;
        }
        if (threadIdx.x == 0) {
            tma::mbar_init(bars, 1);
            tma::mbar_init(bars + 1, 1);
            tma::fence_mbar_init();
        }
        __syncthreads();
    }
    unsigned phase = 0u, sbulk = 0u;                              // per slot (bit i): mbarrier parity, bulk-staged
    auto stage = [&](int slot_i, int t_, int c_, int hk_, int r0_) {
        const double *Ak = A + tile_row0[t_] + r0_;
        const double *tch = tcache + (tile_chunk0[t_] + c_) * (C::NCB * 64);
        const bool bk = bulk && !(hk_ & 1);
        sbulk = bk ? (sbulk | (1u << slot_i)) : (sbulk & ~(1u << slot_i));
        if (bk) {
            stage_chunk_bulk<C>(sm + slot_i * AC::YS, Ak, lda, hk_, n, tch, bars + slot_i);
            asm volatile("cp.async.commit_group;\n" ::: "memory");    // an empty group: wait_group counts stay aligned
        } else {
            stage_chunk<C>(sm + slot_i * AC::YS, Ak, lda, hk_, n, tch, r0_);
        }
    };
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
    if (!kX && tb < te) load_cslab<C>(ccv, Cm, ldc, k, tile_row0[tb], tile_rows[tb], chunk_of(tb, 0), 8 * warp + l4, q, vecc);
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
                if (!staged) stage(cur, t, c, hk, r0);
                // prefetch the next chunk of the work list: Y/T into the other
                // slot, C into registers
                int tn = t, pn = pass, cn = cc_ + 1;
                if (cn == nch) { cn = 0; if (++pn == npass) { pn = 0; ++tn; } }
                double ccn[C::KM][2];
                if (tn < te) {
                    const int cnn = chunk_of(tn, cn), hn = tile_rows[tn], r0n = cnn * C::CH;
                    stage(cur ^ 1, tn, cnn, min(C::CH, hn - r0n), r0n);
                    if (!kX) load_cslab<C>(ccn, Cm, ldc, k, tile_row0[tn], hn, cnn, pw * pn + 8 * warp + l4, q, vecc);
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
                double *slot = sm + cur * AC::YS;
                if ((sbulk >> cur) & 1u) {
                    tma::mbar_wait(bars + cur, (phase >> cur) & 1u);
                    phase ^= 1u << cur;
                    if (hk < C::CH || r0 < C::NP) {       // ragged or head chunk: Yt is fixed up
                        finish_bulk_stage<C>(slot, hk, n, r0);
                        __syncthreads();
                    }                                     // (else every thread waited on the TMA itself)
                } else {
                    __syncthreads();
                    if (dense) {
                        fix_dense<C>(slot, n, r0);
                        __syncthreads();
                    }
                }
                double *Ck = Cm + row0 + r0;
                bool czero = kX;
                cs_apply_panels<C, kFwd, 0>(ccv, cr, r0, np, slot, czero);
                if (vecc && hk == C::CH && (!kFwd || r0 >= C::NP)) {   // aligned row pairs, every row stored
                    if (okc) {
#pragma unroll
                        for (int kk = 0; kk < C::KM; ++kk)
                            *reinterpret_cast<double2 *>(Ck + 8 * kk + 2 * q + (int64_t)col * ldc) =
                                make_double2(ccv[kk][0], ccv[kk][1]);
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < C::KM; ++kk)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int r = 8 * kk + 2 * q + e;
                            if (okc && r < hk && (!kFwd || r0 + r >= n)) Ck[r + (int64_t)col * ldc] = ccv[kk][e];
                        }
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
        const bool bulk = f.bulk && !apply_no_bulk() && !(reinterpret_cast<uintptr_t>(f.A) & 15) && !(f.lda & 1) &&
                          !(reinterpret_cast<uintptr_t>(f.tcache) & 15);
        // C's row pairs aligned: even tile starts (f.bulk), even ldc, 16-byte aligned base
        const bool vecc = f.bulk && !(f.ldc & 1) && !(reinterpret_cast<uintptr_t>(f.C) & 15);
        kern<<<f.grid, 32 * (nw < 1 ? 1 : nw), AC::BYTES, st>>>(f.A, f.lda, f.n, f.tile_row0, f.tile_rows, f.tile_chunk0, f.cta_tile0,
                                                f.tcache, f.C, f.ldc, f.k, f.xbuf, bulk ? 1 : 0, vecc ? 1 : 0);
        return cudaGetLastError();
    });
}

}  // namespace tsqr
