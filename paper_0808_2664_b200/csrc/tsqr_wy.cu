// Butterfly-round kernels (a5, a8 and a9 across ranks, n <= 64) on the blocked
// compact-WY tile engine (wy.cuh), plus small utility kernels, and their host
// launchers.  Product code.
//
//  k_cross_factor  (a5): one round's node [R_lower; R_upper] of the cross-GPU
//                  butterfly (Alg. TSQR:par P:1667-1707): structured combine of
//                  this rank's R and the partner's packed R, identical on both.
//  k_cross_apply   (a8): the round's reflectors applied to the stacked heads of
//                  Q^T C (this rank's and the partner's), keeping the R coordinates;
//                  or of Q C (reverse traversal), keeping this rank's half.
//  k_cross_root_x  (a9): the root X of this rank for form Q, from the replicated
//                  round factors (no communication).
//  k_identity, k_pack_r, k_copy_block: X = I, R -> packed upper triangle, and
//                  block copies for the exchanges.
#include "tsqr_kernels.h"
#include "wy.cuh"

namespace tsqr {

template <int NCB_, int NRB_, int NW_>
struct Geo {
    static constexpr int NCB = NCB_;                 // 8-column blocks (n <= 8 NCB)
    static constexpr int NRB = NRB_;                 // 8-row blocks of a tile (S = 8 NRB)
    static constexpr int NW = NW_;
    static constexpr int NT = 32 * NW;
    static constexpr int NP = 8 * NCB, S = 8 * NRB;
    static constexpr int NROWS = S > 2 * NP ? S : 2 * NP;       // node tiles are [R_a; R_b]
    static constexpr int LD = ((NROWS + 13) / 16) * 16 + 2;     // = 2 mod 16, >= NROWS
    static constexpr int KMAX = NRB > NCB + 1 ? NRB : NCB + 1;  // panel register blocks
};

// Shared-memory carve-up common to the kernels.
template <class G, int CCOLS, int YCOLS = G::NP>
struct Smem {
    static constexpr int tile = 0;                                 // CCOLS x LD
    static constexpr int ys = tile + CCOLS * G::LD;                // Y: YCOLS x LD (one panel or all)
    static constexpr int ts = ys + YCOLS * G::LD;                  // T of all panels: NCB x 64
    static constexpr int gs = ts + G::NCB * 64;                    // 64 (per warp) Gram scratch
    static constexpr int wb = gs + 64 * G::NW;                     // 72 per warp
    static constexpr int taus = wb + 72 * G::NW;                   // NP
    static constexpr int betas = taus + G::NP;                     // NP
    static constexpr int flag = betas + G::NP;                     // 2
    static constexpr size_t bytes = (size_t)(flag + 2) * sizeof(double);
};

template <int NT>
__device__ __forceinline__ void cp_async8(double *sm, const double *g, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// global (rows x ncols, ldg) -> smem (cap_rows x cap_cols, lds), zero padded.
template <int NT>
__device__ __forceinline__ void stage_in(double *sm, int lds, const double *g, int64_t ldg, int rows, int ncols,
                                         int cap_rows, int cap_cols) {
    for (int c = 0; c < cap_cols; ++c) {
        const double *gc = g + (int64_t)(c < ncols ? c : 0) * ldg;
        for (int r = threadIdx.x; r < cap_rows; r += NT) {
            const bool ok = (c < ncols) && (r < rows);
            cp_async8<NT>(sm + c * lds + r, ok ? gc + r : g, ok);
        }
    }
    cp_async_wait_all();
}

template <int NT>
__device__ __forceinline__ void stage_out(const double *sm, int lds, double *g, int64_t ldg, int rows, int ncols) {
    for (int c = 0; c < ncols; ++c) {
        double *gc = g + (int64_t)c * ldg;
        for (int r = threadIdx.x; r < rows; r += NT) gc[r] = sm[c * lds + r];
    }
}

template <int NT>
__device__ __forceinline__ void zero(double *p, int count) {
    for (int e = threadIdx.x; e < count; e += NT) p[e] = 0.0;
}

// Blocked Householder QR of the tile in smem (dense rows [0, rows) or the
// structured node [R_a; R_b] with na = NCB).  Leaves R and the reflector
// entries in place, taus/betas in smem, T of every panel in Ts.
template <class G, bool kNode>
__device__ __forceinline__ void blocked_qr(double *sm, int n, int rows) {
    using SM = Smem<G, G::NP, 8>;
    const int warp = threadIdx.x >> 5;
    double *tile = sm + SM::tile, *Ys = sm + SM::ys;
    const int npan = (n + 7) / 8, nrb = (rows + 7) / 8;
    zero<G::NT>(Ys, 8 * G::LD);
    zero<G::NT>(sm + SM::taus, G::NP);      // padding reflectors (columns >= n) stay H = I
    __syncthreads();
    for (int p = 0; p < npan; ++p) {
        const wy::Rows R{p, nrb, kNode ? G::NCB : -1, p};
        if (warp == p % G::NW) {
            if (p > 0) {
                const int lane = threadIdx.x & 31;
                for (int e = lane; e < 64; e += 32) Ys[(e >> 3) * G::LD + 8 * (p - 1) + (e & 7)] = 0.0;
                __syncwarp();
            }
            wy::panel_qr<G::KMAX>(tile, G::LD, n, R, Ys, G::LD, sm + SM::taus, sm + SM::betas);
            __syncwarp();
            wy::build_t(Ys, G::LD, R, sm + SM::taus + 8 * p, sm + SM::gs + 64 * warp, sm + SM::ts);
        }
        __syncthreads();
        for (int cb = warp; cb < npan; cb += G::NW)
            if (cb > p) wy::wy_update_block<true>(tile, G::LD, cb, Ys, G::LD, R, sm + SM::ts, sm + SM::wb + 72 * warp);
        __syncthreads();
    }
}

// Build the T factors of all panels of a Y held in sm+ys (Y with unit diagonal
// and zeros above, ld LD), warps splitting the panels.
template <class G, int CCOLS, bool kNode>
__device__ __forceinline__ void build_all_t(double *sm, int n, int rows) {
    using SM = Smem<G, CCOLS>;
    const int warp = threadIdx.x >> 5;
    const int npan = (n + 7) / 8, nrb = (rows + 7) / 8;
    for (int p = warp; p < npan; p += G::NW) {
        const wy::Rows R{p, nrb, kNode ? G::NCB : -1, p};
        wy::build_t(sm + SM::ys + 8 * p * G::LD, G::LD, R, sm + SM::taus + 8 * p, sm + SM::gs + 64 * warp,
                    sm + SM::ts + 64 * p);
    }
    __syncthreads();
}

// Apply the panels of the Y in smem to the C tile in smem (kcols columns):
// Q^T (kFwd: panels 0..npan-1, op = T^T) or Q (panels npan-1..0, op = T).
template <class G, int CCOLS, bool kNode, bool kFwd>
__device__ __forceinline__ void apply_panels(double *sm, int n, int rows, int kcols) {
    using SM = Smem<G, CCOLS>;
    const int warp = threadIdx.x >> 5;
    const int npan = (n + 7) / 8, nrb = (rows + 7) / 8, ncb = (kcols + 7) / 8;
    for (int pp = 0; pp < npan; ++pp) {
        const int p = kFwd ? pp : npan - 1 - pp;
        const wy::Rows R{p, nrb, kNode ? G::NCB : -1, p};
        for (int cb = warp; cb < ncb; cb += G::NW)
            wy::wy_update_block<kFwd>(sm + SM::tile, G::LD, cb, sm + SM::ys + 8 * p * G::LD, G::LD, R,
                                      sm + SM::ts + 64 * p, sm + SM::wb + 72 * warp);
    }
    __syncthreads();
}

// Load the n x n upper triangle at g (ld) into smem rows r0.. of a tile (ld LD).
template <class G>
__device__ __forceinline__ void load_upper_cg(double *tile, int r0, const double *g, int64_t ld, int n) {
    for (int e = threadIdx.x; e < G::NP * G::NP; e += G::NT) {
        const int r = e % G::NP, c = e / G::NP;
        const bool ok = r <= c && c < n;
        const double v = __ldcg(g + (ok ? r + (int64_t)c * ld : 0));
        tile[c * G::LD + r0 + r] = ok ? v : 0.0;
    }
}

template <class G>
__device__ __forceinline__ void store_upper(const double *tile, int r0, double *g, int64_t ld, int n) {
    for (int e = threadIdx.x; e < n * n; e += G::NT) {
        const int r = e % n, c = e / n;
        if (r <= c) g[r + (int64_t)c * ld] = tile[c * G::LD + r0 + r];
    }
}

// Node Y = [I; Y1] in smem (rows 0..NP-1: identity on the first n, rows NP..: Y1).
template <class G>
__device__ __forceinline__ void load_node_y(double *Ys, const double *y1, int64_t ld, int n, bool cg) {
    for (int e = threadIdx.x; e < G::NP * G::NP; e += G::NT) {
        const int r = e % G::NP, c = e / G::NP;
        const bool ok = r <= c && c < n;
        double v = 0.0;
        if (ok) v = cg ? __ldcg(y1 + r + (int64_t)c * ld) : y1[r + (int64_t)c * ld];
        Ys[c * G::LD + r] = (r == c && c < n) ? 1.0 : 0.0;
        Ys[c * G::LD + G::NP + r] = v;
    }
}

// ===================================================== factor, warp per tile
// One warp owns one tile and the chain of Householder steps through it: the
// panel chain (latency-bound) of many tiles then overlaps on each SM with no
// block barriers.  Node combines stream R_a row block p through two 8-row
// slots under R_b (rows [0, NP) = R_b, rows [NP, NP+16) = R_a blocks p and
// p+1, the next one loaded into registers while panel p updates), so a node
// needs NP + 16 rows of shared memory instead of 2 NP.
template <int NCB_, int NRB_>
struct WGeo {
    static constexpr int NCB = NCB_, NRB = NRB_;
    static constexpr int NP = 8 * NCB, S = 8 * NRB;
    static constexpr int NROWS = S > NP + 16 ? S : NP + 16;
    static constexpr int LD = ((NROWS + 13) / 16) * 16 + 2;     // = 2 mod 16
    static constexpr int KMAX = NRB > NCB + 1 ? NRB : NCB + 1;
    static constexpr int NB = 4;                                // update blocks per pass
};

template <class G>
struct WSmem {
    static constexpr int tile = 0;                              // NP x LD
    static constexpr int ys = tile + G::NP * G::LD;             // 8 x LD (one panel)
    static constexpr int ts = ys + 8 * G::LD;                   // 64
    static constexpr int gs = ts + 64;                          // 64
    static constexpr int wb = gs + 64;                          // 72 NB
    static constexpr int taus = wb + 72 * G::NB;                // NP
    static constexpr int betas = taus + G::NP;                  // NP
    static constexpr size_t bytes = (size_t)(betas + G::NP) * sizeof(double);
};

// Householder QR of the warp's tile (dense, nrb row blocks) or of the node
// [R_a; R_b] (kNode: R_b in rows [0, NP), R_a read and written at Ra in global
// memory one row block per panel through the slot).
// R_a rows 8pp..8pp+7 (upper part, zero below the diagonal), one warp: lane
// element e = lane + 32 i, i < 16, of the 8 x (NP - 8pp) block.  L2 loads
// (ld.global.cg): the heads are written by warps on other SMs and L1 is not
// coherent.
template <class G>
__device__ __forceinline__ void slot_fetch(double (&v)[16], const double *Ra, int64_t lda, int n, int pp) {
    const int lane = threadIdx.x & 31, w = G::NP - 8 * pp;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int e = lane + 32 * i, c = 8 * pp + (e >> 3), r = 8 * pp + (e & 7);
        const bool ok = e < 8 * w && r <= c && c < n;
        v[i] = ok ? __ldcg(Ra + r + (int64_t)c * lda) : 0.0;
    }
}
template <class G>
__device__ __forceinline__ void slot_put(const double (&v)[16], double *tile, int pp) {
    const int lane = threadIdx.x & 31, w = G::NP - 8 * pp, slot = G::NP + 8 * (pp & 1);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int e = lane + 32 * i;
        if (e < 8 * w) tile[(8 * pp + (e >> 3)) * G::LD + slot + (e & 7)] = v[i];
    }
}

template <class G, bool kNode>
__device__ __forceinline__ void warp_qr(double *sm, int n, int nrb, double *Ra, int64_t lda) {
    using SM = WSmem<G>;
    const int lane = threadIdx.x & 31;
    double *tile = sm + SM::tile, *Ys = sm + SM::ys;
    const int npan = (n + 7) / 8;
    double nxt[16];
    if (kNode) {
        slot_fetch<G>(nxt, Ra, lda, n, 0);
        slot_put<G>(nxt, tile, 0);
        __syncwarp();
    }
    for (int p = 0; p < npan; ++p) {
        const int slot = G::NP + 8 * (p & 1);
        const wy::Rows R = kNode ? wy::Rows{p, nrb, 0, slot / 8} : wy::Rows{p, nrb, -1, p};
        wy::panel_qr<G::KMAX>(tile, G::LD, n, R, Ys, G::LD, sm + SM::taus, sm + SM::betas, sm + SM::gs);
        __syncwarp();
        if (kNode && p + 1 < npan) slot_fetch<G>(nxt, Ra, lda, n, p + 1);   // in flight during T + update
        wy::build_t_gram(sm + SM::gs, sm + SM::taus + 8 * p, sm + SM::ts);
        for (int cb = p + 1; cb < npan; cb += G::NB)
            wy::wy_update_multi<true, G::NB>(tile, G::LD, cb, min(G::NB, npan - cb), Ys, G::LD, R, sm + SM::ts,
                                              sm + SM::wb);
        if (kNode) {                                   // R rows 8p..8p+7 of the merged subtree
            const int w = n - 8 * p;
            for (int e = lane; e < 8 * w; e += 32) {
                const int i = e & 7, c = 8 * p + (e >> 3), r = 8 * p + i;
                if (r <= c) Ra[r + (int64_t)c * lda] = tile[c * G::LD + slot + i];
            }
            if (p + 1 < npan) slot_put<G>(nxt, tile, p + 1);
            __syncwarp();
        }
    }
}

__global__ void k_identity(double *X, int n) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x)
        X[e] = (e % n == e / n) ? 1.0 : 0.0;
}

// ================================================================ output / comm
__global__ void k_pack_r(const double *A, int64_t lda, int n, double *packed) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x) {
        const int r = e % n, c = e / n;
        if (r <= c) packed[(int64_t)c * (c + 1) / 2 + r] = A[r + (int64_t)c * lda];
    }
}

__global__ void k_unpack_r(const double *packed, int n, double *A, int64_t lda) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x) {
        const int r = e % n, c = e / n;
        A[r + (int64_t)c * lda] = r <= c ? packed[(int64_t)c * (c + 1) / 2 + r] : 0.0;
    }
}

__global__ void k_copy_block(const double *src, int64_t lds, double *dst, int64_t ldd, int n, int k) {
    for (int64_t e = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; e < (int64_t)n * k;
         e += (int64_t)blockDim.x * gridDim.x) {
        const int r = (int)(e % n);
        const int64_t c = e / n;
        dst[r + c * ldd] = src[r + c * lds];
    }
}

// Butterfly round of the factorization: [R_lower; R_upper] -> structured QR.
template <class G>
__global__ void __launch_bounds__(G::NT)
k_cross_factor(double *A, int64_t lda, int n, const double *partner_packed, int is_lower, double *Y1_out,
               double *tau_out, double *R, int64_t ldr) {
    using SM = Smem<G, G::NP, 8>;
    extern __shared__ __align__(16) double sm[];
    double *tile = sm + SM::tile;
    zero<G::NT>(tile, G::NP * G::LD);
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += G::NT) {
        const int r = e % n, c = e / n;
        if (r <= c) {
            const double mine = A[r + (int64_t)c * lda];
            const double theirs = partner_packed[(int64_t)c * (c + 1) / 2 + r];
            tile[c * G::LD + r] = is_lower ? mine : theirs;
            tile[c * G::LD + G::NP + r] = is_lower ? theirs : mine;
        }
    }
    __syncthreads();
    blocked_qr<G, true>(sm, n, 2 * G::NP);
    for (int e = threadIdx.x; e < n * n; e += G::NT) {
        const int r = e % n, c = e / n;
        const double rv = (r <= c) ? tile[c * G::LD + r] : 0.0;
        if (r <= c) A[r + (int64_t)c * lda] = rv;                          // the new current R
        if (R) R[r + (int64_t)c * ldr] = rv;
        Y1_out[r + (int64_t)c * n] = (r <= c) ? tile[c * G::LD + G::NP + r] : 0.0;
    }
    for (int j = threadIdx.x; j < n; j += G::NT) tau_out[j] = sm[SM::taus + j];
}

// Butterfly round of apply Q^T on the R coordinates (n x k tops).
template <class G, bool kFwd>
__global__ void __launch_bounds__(G::NT)
k_cross_apply(const double *Y1g, const double *taug, double *top, int64_t ldtop, const double *partner_top,
              int is_lower, int head_role, double *C, int64_t ldc, int n, int k) {
    using SM = Smem<G, G::NP>;
    extern __shared__ __align__(16) double sm[];
    double *tile = sm + SM::tile;
    for (int j = threadIdx.x; j < G::NP; j += G::NT) sm[SM::taus + j] = j < n ? taug[j] : 0.0;
    zero<G::NT>(sm + SM::ys, G::NP * G::LD);
    __syncthreads();
    load_node_y<G>(sm + SM::ys, Y1g, n, n, false);
    __syncthreads();
    build_all_t<G, G::NP, true>(sm, n, 2 * G::NP);
    for (int c0 = 0; c0 < k; c0 += G::NP) {
        const int kc = min(G::NP, k - c0);
        for (int e = threadIdx.x; e < G::NP * 2 * G::NP; e += G::NT) {
            const int r = e % (2 * G::NP), c = e / (2 * G::NP);
            const bool topblk = r < G::NP;
            const int rr = topblk ? r : r - G::NP;
            double v = 0.0;
            if (rr < n && c < kc) {
                const bool mine = (topblk == (is_lower != 0));
                v = mine ? top[rr + (int64_t)(c0 + c) * ldtop] : partner_top[rr + (int64_t)(c0 + c) * n];
            }
            tile[c * G::LD + r] = v;
        }
        __syncthreads();
        apply_panels<G, G::NP, true, kFwd>(sm, n, 2 * G::NP, kc);
        for (int e = threadIdx.x; e < kc * n; e += G::NT) {
            const int r = e % n, c = e / n;
            // Q^T: the new R coordinates; Q C (!kFwd): this rank's half of the result
            const double ra = tile[c * G::LD + (kFwd || is_lower ? 0 : G::NP) + r];
            top[r + (int64_t)(c0 + c) * ldtop] = ra;
            if (!kFwd || head_role == 1) C[r + (int64_t)(c0 + c) * ldc] = ra;
            if (head_role == 2) C[r + (int64_t)(c0 + c) * ldc] = tile[c * G::LD + G::NP + r];
        }
        __syncthreads();
    }
}

// Root X of this rank for form-Q: top-down over the butterfly nodes.
template <class G>
__global__ void __launch_bounds__(G::NT)
k_cross_root_x(const double *Y1s, const double *taus_g, int rounds, int rank, int n, double *X0) {
    using SM = Smem<G, G::NP>;
    extern __shared__ __align__(16) double sm[];
    double *tile = sm + SM::tile;
    // X lives in tile rows 0..NP-1 between rounds; rows NP.. receive X_b.
    zero<G::NT>(tile, G::NP * G::LD);
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += G::NT) tile[e * G::LD + e] = 1.0;
    for (int kr = rounds; kr >= 1; --kr) {
        for (int j = threadIdx.x; j < G::NP; j += G::NT) sm[SM::taus + j] = j < n ? taus_g[(kr - 1) * n + j] : 0.0;
        zero<G::NT>(sm + SM::ys, G::NP * G::LD);
        for (int e = threadIdx.x; e < G::NP * G::NP; e += G::NT) {
            const int r = e % G::NP, c = e / G::NP;
            tile[c * G::LD + G::NP + r] = 0.0;               // [X; 0]
        }
        __syncthreads();
        load_node_y<G>(sm + SM::ys, Y1s + (int64_t)(kr - 1) * n * n, n, n, false);
        __syncthreads();
        build_all_t<G, G::NP, true>(sm, n, 2 * G::NP);
        apply_panels<G, G::NP, true, false>(sm, n, 2 * G::NP, n);
        const bool lower = ((rank >> (kr - 1)) & 1) == 0;
        if (!lower) {
            for (int e = threadIdx.x; e < G::NP * G::NP; e += G::NT) {
                const int r = e % G::NP, c = e / G::NP;
                tile[c * G::LD + r] = tile[c * G::LD + G::NP + r];
            }
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < n * n; e += G::NT) {
        const int r = e % n, c = e / n;
        X0[r + (int64_t)c * n] = tile[c * G::LD + r];
    }
}

// ================================================================= launchers
static cudaError_t set_smem(const void *fn, size_t bytes) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Geometries: n <= 32 (4 column blocks, 4 warps), n <= 64 (8 column blocks, 8 warps);
// tiles of 64 / 128 / 192 rows.
template <int NCB, int NRB> struct GeoFor { using type = Geo<NCB, NRB, NCB>; };


cudaError_t launch_identity(double *X, int n, cudaStream_t st) {
    k_identity<<<(n * n + 255) / 256, 256, 0, st>>>(X, n);
    return cudaGetLastError();
}

cudaError_t launch_pack_r(const double *A, int64_t lda, int n, double *packed, cudaStream_t st) {
    k_pack_r<<<(n * n + 255) / 256, 256, 0, st>>>(A, lda, n, packed);
    return cudaGetLastError();
}

cudaError_t launch_unpack_r(const double *packed, int n, double *A, int64_t lda, cudaStream_t st) {
    k_unpack_r<<<(n * n + 255) / 256, 256, 0, st>>>(packed, n, A, lda);
    return cudaGetLastError();
}

cudaError_t launch_copy_block(const double *src, int64_t lds, double *dst, int64_t ldd, int n, int k,
                              cudaStream_t st) {
    const int64_t tot = (int64_t)n * k;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > 1184) blocks = 1184;
    if (blocks < 1) blocks = 1;
    k_copy_block<<<blocks, 256, 0, st>>>(src, lds, dst, ldd, n, k);
    return cudaGetLastError();
}

template <class G>
static cudaError_t launch_cross_factor_t(double *A, int64_t lda, int n, const double *pp, int is_lower, double *Y1,
                                         double *tau, double *R, int64_t ldr, cudaStream_t st) {
    const size_t sm = Smem<G, G::NP, 8>::bytes;
    cudaError_t e = set_smem((const void *)k_cross_factor<G>, sm);
    if (e != cudaSuccess) return e;
    k_cross_factor<G><<<1, G::NT, sm, st>>>(A, lda, n, pp, is_lower, Y1, tau, R, ldr);
    return cudaGetLastError();
}

cudaError_t launch_cross_factor(int NP, double *A, int64_t lda, int n, const double *pp, int is_lower, double *Y1,
                                double *tau, double *R, int64_t ldr, cudaStream_t st) {
    return NP <= 32 ? launch_cross_factor_t<Geo<4, 8, 4>>(A, lda, n, pp, is_lower, Y1, tau, R, ldr, st)
                    : launch_cross_factor_t<Geo<8, 8, 8>>(A, lda, n, pp, is_lower, Y1, tau, R, ldr, st);
}

template <class G>
static cudaError_t launch_cross_apply_t(const double *Y1, const double *tau, double *top, int64_t ldtop,
                                        const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n,
                                        int k, int forward, cudaStream_t st) {
    const size_t sm = Smem<G, G::NP>::bytes;
    auto kern = forward ? k_cross_apply<G, true> : k_cross_apply<G, false>;
    cudaError_t e = set_smem((const void *)kern, sm);
    if (e != cudaSuccess) return e;
    kern<<<1, G::NT, sm, st>>>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k);
    return cudaGetLastError();
}

cudaError_t launch_cross_apply(int NP, const double *Y1, const double *tau, double *top, int64_t ldtop,
                               const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n, int k,
                               int forward, cudaStream_t st) {
    return NP <= 32
               ? launch_cross_apply_t<Geo<4, 8, 4>>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, forward, st)
               : launch_cross_apply_t<Geo<8, 8, 8>>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, forward, st);
}

template <class G>
static cudaError_t launch_cross_root_x_t(const double *Y1s, const double *taus, int rounds, int rank, int n,
                                         double *X0, cudaStream_t st) {
    const size_t sm = Smem<G, G::NP>::bytes;
    cudaError_t e = set_smem((const void *)k_cross_root_x<G>, sm);
    if (e != cudaSuccess) return e;
    k_cross_root_x<G><<<1, G::NT, sm, st>>>(Y1s, taus, rounds, rank, n, X0);
    return cudaGetLastError();
}

cudaError_t launch_cross_root_x(int NP, const double *Y1s, const double *taus, int rounds, int rank, int n,
                                double *X0, cudaStream_t st) {
    return NP <= 32 ? launch_cross_root_x_t<Geo<4, 8, 4>>(Y1s, taus, rounds, rank, n, X0, st)
                    : launch_cross_root_x_t<Geo<8, 8, 8>>(Y1s, taus, rounds, rank, n, X0, st);
}

}  // namespace tsqr
