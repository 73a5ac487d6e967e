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
#include "tma.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace tsqr {
using namespace chunk;

// TSQR_NO_TMA=1 in the environment: the per-element cp.async staging everywhere (A/B checks)
static bool chain_no_tma() {
    static const int v = [] {
        const char *e = std::getenv("TSQR_NO_TMA");
        return (e && *e == '1') ? 1 : 0;
    }();
    return v != 0;
}

template <class C, int P, bool kRobust, bool kAllStruct>
__device__ __forceinline__ void chunk_panels(Chunk<C> &ch, int r0, bool last, double *Rb, const Sync &sy,
                                             double *ws, double *tau_out, int n, double *Ahead, int64_t lda,
                                             double *tg, double *ydst) {
    const int lane = threadIdx.x & 31;
    const int kind = kAllStruct ? 0 : ((8 * P < r0) ? 0 : (8 * P < r0 + C::CH ? 1 : 2));
    const int kb = (8 * P - r0) >> 3;
    factor_panel<C, P, kRobust>(ch, kind, kb, Rb, ws, tau_out, n, sy, last, tg, ydst, lda);
    if (last) {                                   // R rows 8P .. 8P+7 of the tile are final
        const int w = n - 8 * P;
        for (int e = lane; e < 8 * w; e += 32) {
            const int i = 8 * P + (e & 7), c = 8 * P + (e >> 3);
            if (i <= c && i < n) Ahead[i + (int64_t)c * lda] = Rb[i * C::LDR + c];
        }
        sync_publish(sy.tr + P, sy.s + 1);        // the buffer's next user may overwrite them
    }
    PROBE(8);
    if constexpr (P + 1 < C::NCB)
        chunk_panels<C, P + 1, kRobust, kAllStruct>(ch, r0, last, Rb, sy, ws, tau_out, n, Ahead, lda, tg, ydst);
}

// Prefetch a chunk (rows [r0, r0 + hk) of the tile at A + row0, all n columns)
// into the warp's staging buffer (col-major CH x NP, zero-filled) with cp.async.
template <class C>
__device__ __forceinline__ void prefetch_chunk(double *stg, const double *src, int64_t lda, int hk, int n) {
    const int lane = threadIdx.x & 31;
#pragma unroll 4
    for (int i = lane; i < C::CH * C::NP; i += 32) {
        const int col = i / C::CH, row = i % C::CH;
        const bool ok = row < hk && col < n;
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(stg + i));
        const double *g = src + (ok ? row + (int64_t)col * lda : 0);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// kRobust: the rescaled Householder steps of reading R23 (inputs outside
// [2^-400, 2^400]); a separate instantiation chosen at launch (opts.flags bit 2)
// so the default kernel carries no trace of the slow path (measured 3-8 %).
// kTma: the next chunk is staged by one TMA box copy (tensor map `tmap` of A,
// box CH x n, rows past the matrix zero-filled, the slot's padding columns
// n..NP-1 zeroed once; rows past the tile are zeroed on the register load)
// completing on the warp's mbarrier;
// otherwise by per-element cp.async (any lda / alignment).
template <class C, bool kRobust, bool kTma>
__global__ void __launch_bounds__(C::NT, 1)
k_chain_factor(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows,
               const int64_t *tile_chunk0, const int *cta_tile0, double *tau, double *tcache,
               const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane & 3, l4 = lane >> 2;
    int *sync = reinterpret_cast<int *>(sm + C::OFF_SYNC);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + C::OFF_BAR) + warp;
    for (int i = threadIdx.x; i < C::NBUF * C::SYNC_INTS; i += C::NT) sync[i] = 0;
    if (kTma && lane == 0) {
        tma::mbar_init(bar, 1);
        tma::fence_mbar_init();
        tma::prefetch_map(&tmap);
    }
    PROBE_INIT();
    __syncthreads();
    double *ws = sm + C::OFF_WS + warp * C::WS;
    double *stg = sm + C::OFF_STG + warp * C::STG;
    unsigned phase = 0;
    if constexpr (kTma) {                                 // the box is CH x n: padding columns stay zero
        for (int i = lane; i < (C::NP - n) * C::CH; i += 32) stg[n * C::CH + i] = 0.0;
        __syncwarp();
    }
    // stream rows [r0, r0 + hk) of tile t into the staging slot
    auto stage = [&](int t, int r0, int hk) {
        if constexpr (kTma) {
            if (lane == 0) {
                tma::fence_proxy_async_smem();        // the slot's generic reads precede the async write
                tma::mbar_arrive_expect_tx(bar, C::CH * n * (unsigned)sizeof(double));
                tma::load_2d(stg, &tmap, (int)(tile_row0[t] + r0), 0, bar);
            }
        } else {
            prefetch_chunk<C>(stg, A + tile_row0[t] + r0, lda, hk, n);
        }
    };
    const int tb = cta_tile0[blockIdx.x], te = cta_tile0[blockIdx.x + 1];
    // Walk the CTA's chunk sequence (all warps identically); this warp owns
    // every NW-th chunk.  When the warp finds its next chunk it computes the
    // previous one (pend), whose data was prefetched into its staging buffer,
    // and streams the new one in meanwhile.
    int cnt[2] = {0, 0};
    int g = 0;
    int pt = -1, pc = 0, ps = 0, pb = 0;                  // the pending chunk
    int t = tb, c = 0, b = 0, nch = tb < te ? (tile_rows[tb] + C::CH - 1) / C::CH : 0;
    for (;;) {
        // advance to this warp's next chunk (or the end)
        int nt = -1, ncix = 0, ns = 0, nb = 0;
        while (t < te) {
            if (c == nch) {
                ++t;
                c = 0;
                if (t >= te) break;
                b = C::NBUF == 2 ? (t - tb) & 1 : 0;
                nch = (tile_rows[t] + C::CH - 1) / C::CH;
                continue;
            }
            const int s = cnt[b]++;
            // n = 64 and n = 32: consecutive chunks go to the two warps of one SMSP (warp w
            // runs on SMSP w % 4), chunk i -> warp (i >> 1) + 4 (i & 1), so those two warps run
            // about one panel apart, mostly in the same phase -- both in latency-bound
            // Householder steps or both in DMMA-bound trailing updates -- instead of one's
            // DMMAs delaying the other's step chain on the shared FP64 pipe (C4 leaf 15.33 ->
            // 14.84 ms, C5 10.46 -> 10.41 ms; C2's n = 50 configuration measured 1 % slower)
            constexpr bool kPairSmsp = C::NW == 8 && (C::NCB == 8 || C::NCB == 4);
            const int gi = g % C::NW;
            const bool mine = (kPairSmsp ? (gi >> 1) + 4 * (gi & 1) : gi) == warp;
            ++g;
            const int cc = c++;
            if (mine) {
                nt = t; ncix = cc; ns = s; nb = b;
                break;
            }
        }
        if (pt < 0) {                                     // first chunk: stream it in
            if (nt < 0) break;
            const int r0 = ncix * C::CH;
            stage(nt, r0, min(C::CH, tile_rows[nt] - r0));
            pt = nt; pc = ncix; ps = ns; pb = nb;
            continue;
        }
        // compute the pending chunk
        const int h = tile_rows[pt];
        const int pnch = (h + C::CH - 1) / C::CH;
        const int64_t row0 = tile_row0[pt];
        const int r0 = pc * C::CH, hk = min(C::CH, h - r0);
        if constexpr (kTma) {
            tma::mbar_wait(bar, phase);
            phase ^= 1;
        } else {
            asm volatile("cp.async.wait_all;\n" ::: "memory");
        }
        __syncwarp();
        Chunk<C> ch;
#pragma unroll
        for (int k = 0; k < C::KM; ++k)
#pragma unroll
            for (int cb = 0; cb < C::NCB; ++cb) {
                const double2 v = *reinterpret_cast<const double2 *>(stg + (8 * cb + l4) * C::CH + 8 * k + 2 * q);
                ch.a[k][cb][0] = v.x;
                ch.a[k][cb][1] = v.y;
            }
        if (kTma && hk < C::CH) {                         // the box ran into the next tile: zero those rows
#pragma unroll
            for (int k = 0; k < C::KM; ++k)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (8 * k + 2 * q + e >= hk)
#pragma unroll
                        for (int cb = 0; cb < C::NCB; ++cb) ch.a[k][cb][e] = 0.0;
        }
        __syncwarp();
        if (nt >= 0) {                                    // the next chunk streams in meanwhile
            const int r0n = ncix * C::CH;
            stage(nt, r0n, min(C::CH, tile_rows[nt] - r0n));
        }
        PROBE(0);
        double *tau_out = tau + (tile_chunk0[pt] + pc) * n;
        const Sync sy{sync + pb * C::SYNC_INTS, sync + pb * C::SYNC_INTS + C::NP, ps};
        double *tg = tcache ? tcache + (tile_chunk0[pt] + pc) * (C::NCB * 64) : nullptr;
        double *dst = A + row0 + r0;
        // A full chunk below the pivots: every element is a reflector entry, and with the TMA
        // layout conditions (even tile starts, even lda) each lane's row pair is one aligned
        // 16-byte store; each panel's reflectors are stored as soon as its steps end (spread
        // over the chunk: C4 leaf 14.58 -> 14.06 ms, C2 0.810 -> 0.799 ms against one burst of
        // stores after the last panel).  Other chunks store after the last panel, masked.
        const bool full = kTma && hk == C::CH && r0 >= C::NP;
        if constexpr (C::NCB <= 4) {
            // n <= 32: a chunk below the pivots runs structured panels only, in its own
            // instantiation, so its code is contiguous (the head chunks' dense / mixed path is
            // laid out elsewhere): C5 leaf 10.25 -> 10.0 ms.  For n > 32 the same split measured
            // slower (C4 +2.8 %, C2 +6 %; profiles/r02_split_paths_ab.txt).
            if (__builtin_expect(r0 >= C::NP, 1))
                chunk_panels<C, 0, kRobust, true>(ch, r0, pc == pnch - 1, sm + pb * C::RBUF, sy, ws, tau_out, n,
                                                  A + row0, lda, tg, full ? dst : nullptr);
            else
                chunk_panels<C, 0, kRobust, false>(ch, r0, pc == pnch - 1, sm + pb * C::RBUF, sy, ws, tau_out, n,
                                                   A + row0, lda, tg, nullptr);
        } else {
            chunk_panels<C, 0, kRobust, false>(ch, r0, pc == pnch - 1, sm + pb * C::RBUF, sy, ws, tau_out, n, A + row0,
                                               lda, tg, full ? dst : nullptr);
        }
        if (!full) {
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
        if (nt < 0) break;
        pt = nt; pc = ncix; ps = ns; pb = nb;
    }
    PROBE_FLUSH();
}

// ================================================================= launchers
// Dispatch on n to the compiled configurations of the chain engine (32-row chunks).
template <class F>
static cudaError_t chain_dispatch(int n, F &&fn) {
    const int ncb = (n + 7) / 8;
    switch (ncb) {
        case 1: case 2: return fn(Cfg<2, 8, 8>());
        case 3: case 4: return fn(Cfg<TSQR_CFG32>());
        case 5: case 6: return fn(Cfg<6, 6, 8>());
        case 7: return fn(Cfg<7, 5, 8>());
        default: return fn(Cfg<8, 5, 8, 1>());          // one R buffer: room for 40-row chunks
    }
}

// Tensor map of an m x n column-major fp64 matrix (tma.cuh), through the driver
// entry point (no libcuda link dependency).
bool make_tmap_colmajor(CUtensorMap *map, const double *base, int64_t m, int64_t n, int64_t ld, int box_rows,
                        int box_cols) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool looked = false;
    if (!looked) {
        looked = true;
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        cudaGetLastError();
    }
    if (!encode || m < 1 || n < 1 || m > INT32_MAX || n > INT32_MAX) return false;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 8) & 15) || ld >= (int64_t(1) << 37)) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
    const cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
    const cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class C, bool kRobust, bool kTma>
static cudaError_t launch_chain_factor_t(const ChainArgs &f, const CUtensorMap &map, cudaStream_t st) {
    const size_t sm = C::BYTES;
    cudaError_t e = cudaFuncSetAttribute((const void *)k_chain_factor<C, kRobust, kTma>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_chain_factor<C, kRobust, kTma><<<f.grid, C::NT, sm, st>>>(f.A, f.lda, f.n, f.tile_row0, f.tile_rows,
                                                               f.tile_chunk0, f.cta_tile0, f.tau, f.tcache, map);
    return cudaGetLastError();
}

cudaError_t launch_chain_factor(const ChainArgs &f, cudaStream_t st) {
    return chain_dispatch(f.n, [&](auto c) {
        using C = decltype(c);
        CUtensorMap map;
        std::memset(&map, 0, sizeof(map));
        // the robust instantiation keeps the cp.async staging (one fewer kernel per configuration)
        const bool tma = !f.robust && f.m > 0 && !chain_no_tma() &&
                         make_tmap_colmajor(&map, f.A, f.m, f.n, f.lda, C::CH, f.n);
        if (f.robust) return launch_chain_factor_t<C, true, false>(f, map, st);
        return tma ? launch_chain_factor_t<C, false, true>(f, map, st) : launch_chain_factor_t<C, false, false>(f, map, st);
    });
}

int chain_chunk_rows(int n) {
    int ch = 0;
    chain_dispatch(n, [&](auto c) {
        ch = decltype(c)::CH;
        return cudaSuccess;
    });
    return ch;
}

int chain_ncb(int n) {
    int ncb = 0;
    chain_dispatch(n, [&](auto c) {
        ncb = decltype(c)::NCB;
        return cudaSuccess;
    });
    return ncb;
}

// Resident CTAs of the factor kernel on the current device (the persistent grid).
int chain_grid(int n) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = chain_dispatch(n, [&](auto c) {
        using C = decltype(c);
        cudaError_t r = cudaFuncSetAttribute((const void *)k_chain_factor<C, false, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
        if (r != cudaSuccess) return r;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_chain_factor<C, false, false>, C::NT, C::BYTES);
    });
    if (e != cudaSuccess || occ < 1) occ = 1;
    return sms * occ;
}

// Split of the tiles over `grid` CTAs in contiguous runs that minimises the
// largest run's chunk count (the kernel ends with its busiest CTA): binary
// search on the capacity, runs filled greedily.
void chain_partition(const std::vector<int64_t> &tile_rows, int chunk_rows, int grid, std::vector<int> &cta_tile0) {
    const int L = (int)tile_rows.size();
    std::vector<int64_t> w(L);
    int64_t lo = 0, hi = 0;
    for (int t = 0; t < L; ++t) {
        w[t] = (tile_rows[t] + chunk_rows - 1) / chunk_rows;
        lo = std::max(lo, w[t]);
        hi += w[t];
    }
    auto runs = [&](int64_t cap) {
        int k = 0;
        int64_t acc = 0;
        for (int t = 0; t < L; ++t) {
            if (k == 0 || acc + w[t] > cap) { ++k; acc = 0; }
            acc += w[t];
        }
        return k;
    };
#ifdef TSQR_PARTITION_NEAREST
    // variant: cuts at the tile nearest to each equal-share target
    std::vector<int64_t> pre(L + 1, 0);
    for (int t = 0; t < L; ++t) pre[t + 1] = pre[t] + w[t];
    cta_tile0.assign(grid + 1, L);
    cta_tile0[0] = 0;
    int t = 0;
    for (int i = 1; i < grid; ++i) {
        const int64_t target = (pre[L] * i + grid - 1) / grid;
        while (t < L && pre[t] < target) ++t;
        if (t > 0 && t < L && (target - pre[t - 1]) < (pre[t] - target)) --t;
        t = std::max(t, cta_tile0[i - 1]);
        cta_tile0[i] = t;
    }
    cta_tile0[grid] = L;
    return;
#endif
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (runs(mid) <= grid) hi = mid;
        else lo = mid + 1;
    }
    cta_tile0.assign(grid + 1, L);
    cta_tile0[0] = 0;
    int k = 0;
    int64_t acc = 0;
    for (int t = 0; t < L; ++t) {
        if (t > 0 && acc + w[t] > lo) { cta_tile0[++k] = t; acc = 0; }
        acc += w[t];
    }
}

// ================================================================ T rebuild
// k_chain_rebuild_t: the factor's T cache (tcache[chunk][panel] = the 8 x 8 T of
// the panel's reflectors, row-major, LAPACK sign, reading R3) recomputed from the
// stored reflectors and taus alone -- the streamed factor keeps only Y and tau
// as its Q factors in host memory ([TR] Alg. TSQR:seq P:1725-1753 writes Y and
// tau; T is derived data, Alg. YT:scaled P:2007-2028).  One warp per (chunk,
// panel): the chunk-local part of each reflector is
//     structured column j < r0:   y_j(i) = A(r0 + i, j), i < hk   (its R-row part
//                                 e_j is orthogonal to the others' in the panel)
//     dense column r0 <= j:       1 at i = j - r0, A(r0 + i, j) below, 0 above,
// (a panel never mixes the two: CH is a multiple of 8); the lanes split the rows
// for the 28 Gram entries G(l, c) = v_l^T v_c (l < c), a warp reduction, then T by
// the recurrence T(r,c) = -tau_c sum_{l=r}^{c-1} T(r,l) G(l,c).  Absent columns
// (tau = 0) give zero rows/columns, as in the factor.
__global__ void __launch_bounds__(256)
k_chain_rebuild_t(const double *A, int64_t lda, int n, int ch, int ncb, const int64_t *tile_row0, const int *tile_rows,
                  const int64_t *tile_chunk0, int ntiles, const double *tau, double *tcache) {
    const int lane = threadIdx.x & 31;
    const int64_t nchunks = tile_chunk0[ntiles];
    const int64_t task = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (task >= nchunks * ncb) return;
    const int64_t g = task / ncb;
    const int P = (int)(task - g * ncb);
    int lo = 0, hi = ntiles - 1;                          // tile of chunk g
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_chunk0[mid] <= g) lo = mid;
        else hi = mid - 1;
    }
    const int t = lo;
    const int r0 = (int)(g - tile_chunk0[t]) * ch;
    const int hk = min(ch, tile_rows[t] - r0);
    const double *Ak = A + tile_row0[t] + r0;
    double gs[28];
#pragma unroll
    for (int i = 0; i < 28; ++i) gs[i] = 0.0;
    for (int i = lane; i < hk; i += 32) {
        double v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int j = 8 * P + c;
            double x = 0.0;
            if (j < n) {
                if (j < r0) x = Ak[i + (int64_t)j * lda];
                else x = (i == j - r0) ? 1.0 : (i > j - r0 ? Ak[i + (int64_t)j * lda] : 0.0);
            }
            v[c] = x;
        }
        int e = 0;
#pragma unroll
        for (int c = 1; c < 8; ++c)
#pragma unroll
            for (int l = 0; l < c; ++l) {
                gs[e] = fma(v[l], v[c], gs[e]);
                ++e;
            }
    }
#pragma unroll
    for (int i = 0; i < 28; ++i)
#pragma unroll
        for (int o = 16; o; o >>= 1) gs[i] += __shfl_xor_sync(0xffffffffu, gs[i], o);
    const double *tp = tau + g * n;
    const int r = lane & 7;
    double row[8], tt[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) tt[c] = (8 * P + c < n) ? tp[8 * P + c] : 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) row[c] = (c == r) ? tt[r] : 0.0;
    int e = 0;
#pragma unroll
    for (int c = 1; c < 8; ++c) {
        double s2 = 0.0;
#pragma unroll
        for (int l = 0; l < c; ++l) s2 = fma(row[l], gs[e + l], s2);
        e += c;
        row[c] = (r < c) ? -tt[c] * s2 : row[c];
    }
    if (lane < 8) {
        double *dst = tcache + (g * ncb + P) * 64 + r * 8;
#pragma unroll
        for (int c = 0; c < 8; ++c) dst[c] = row[c];
    }
}

cudaError_t launch_chain_rebuild_t(const double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows,
                                   const int64_t *tile_chunk0, int ntiles, int64_t nchunks, const double *tau,
                                   double *tcache, cudaStream_t st) {
    const int ch = chain_chunk_rows(n), ncb = chain_ncb(n);
    const int64_t tasks = nchunks * ncb;
    if (tasks == 0) return cudaSuccess;
    k_chain_rebuild_t<<<(unsigned)((tasks + 7) / 8), 256, 0, st>>>(A, lda, n, ch, ncb, tile_row0, tile_rows, tile_chunk0,
                                                                   ntiles, tau, tcache);
    return cudaGetLastError();
}

}  // namespace tsqr
