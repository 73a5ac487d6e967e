// Kernels of the B200 TSQR hot path (sm_100a) on the blocked compact-WY engine
// (wy.cuh) and their host launchers.  Product code.
//
//  k_factor_w    (a2)+(a3)+(a4)+(a6): one warp per tile: panel QR (shuffles,
//                Gram on the fly) -> T (a3) -> DMMA trailing update, panel by
//                panel; then the single-pass ticketed tree: the second warp to
//                finish below a node runs the structured combine of [R_a; R_b]
//                (Alg. QR:qnxn on the same engine, structured row blocks) and
//                climbs; the root writes R.
//  k_apply_qt    (a7)+(a8): C <- Q_tile^T C panel by panel (W = Y^T C,
//                W <- T^T W, C -= Y W on DMMA), then the ticketed climb applying
//                each node's [I; Y1] reflectors to the head rows.
//  k_formq_node  (a9): one top-down tree step [X_a; X_b] = Q_node [X; 0].
//  k_formq_leaf  (a10): Q_t = Q_tile [X_t; 0].
//  k_cross_*     (a5): butterfly round compute.
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

template <class G, bool kLeaf>
__global__ void __launch_bounds__(32)
k_factor_w(double *A, int64_t lda, int n, DevPlan plan, double *tau_tile, double *tau_node, int *counters, double *R,
           int64_t ldr) {
    using SM = WSmem<G>;
    extern __shared__ __align__(16) double sm[];
    double *tile = sm + SM::tile;
    const int lane = threadIdx.x;
    const int t = blockIdx.x;
    if (kLeaf) {
        const int64_t row0 = plan.tile_row0[t];
        const int rows = plan.tile_rows[t];
        double *At = A + row0;
        for (int j = lane; j < G::NP; j += 32) sm[SM::taus + j] = 0.0;   // padding reflectors: H = I
        stage_in<32>(tile, G::LD, At, lda, rows, n, G::S, G::NP);
        __syncwarp();
        warp_qr<G, false>(sm, n, (rows + 7) / 8, nullptr, 0);
        stage_out<32>(tile, G::LD, At, lda, rows, n);
        for (int j = lane; j < n; j += 32) tau_tile[(int64_t)t * n + j] = sm[SM::taus + j];
    }

    int p = plan.tile_parent[t];
    bool root = (p < 0);
    while (p >= 0) {
        // ticket: the second warp to arrive at node p runs it
        __threadfence();
        __syncwarp();
        int old = 0;
        if (lane == 0) {
            old = atomicAdd(counters + p, 1);
            if (old == 1) counters[p] = 0;
        }
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old != 1) return;
        __threadfence();
        const int64_t ra = plan.tile_row0[plan.node_a[p]], rb = plan.tile_row0[p];
        for (int e0 = 0; e0 < G::NP * G::NP; e0 += 32 * 16) {     // R_b (upper) -> rows [0, NP), L2 loads
            double v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int e = e0 + lane + 32 * i, r = e % G::NP, c = e / G::NP;
                const bool ok = e < G::NP * G::NP && r <= c && c < n;
                v[i] = ok ? __ldcg(A + rb + r + (int64_t)c * lda) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int e = e0 + lane + 32 * i;
                if (e < G::NP * G::NP) tile[(e / G::NP) * G::LD + e % G::NP] = v[i];
            }
        }
        __syncwarp();
        warp_qr<G, true>(sm, n, G::NCB, A + ra, lda);
        for (int e = lane; e < n * n; e += 32) {                   // Y1 of the node (eq. fact_2rs)
            const int r = e % n, c = e / n;
            if (r <= c) A[rb + r + (int64_t)c * lda] = tile[c * G::LD + r];
        }
        for (int j = lane; j < n; j += 32) tau_node[(int64_t)p * n + j] = sm[SM::taus + j];
        const int q = plan.node_parent[p];
        if (q < 0) root = true;
        p = q;
    }
    if (root && R != nullptr) {
        __threadfence();
        __syncwarp();
        for (int e = lane; e < n * n; e += 32) {
            const int r = e % n, c = e / n;
            R[r + (int64_t)c * ldr] = (r <= c) ? __ldcg(A + r + (int64_t)c * lda) : 0.0;
        }
    }
}

// ========================================================= apply Q^T (a7,a8)
// The tile's Y (unit lower, zeros above) into sm+ys.
template <class G, int CCOLS>
__device__ __forceinline__ void load_tile_y(double *sm, const double *At, int64_t lda, int rows, int n) {
    using SM = Smem<G, CCOLS>;
    double *Ys = sm + SM::ys;
    stage_in<G::NT>(Ys, G::LD, At, lda, rows, n, G::S, G::NP);
    __syncthreads();
    for (int e = threadIdx.x; e < G::NP * 8; e += G::NT) {
        const int c = e / 8, r8 = e % 8;
        const int r = (c / 8) * 8 + r8;                      // rows of the pivot block of c's panel
        if (r <= c || c >= n) Ys[c * G::LD + r] = (r == c && c < n) ? 1.0 : 0.0;
    }
    // rows above the pivot block of every panel are zero
    for (int e = threadIdx.x; e < G::NP * G::S; e += G::NT) {
        const int c = e / G::S, r = e % G::S;
        if (r < (c / 8) * 8 || c >= n) Ys[c * G::LD + r] = 0.0;
    }
    __syncthreads();
}

template <class G, int CCOLS, bool kLeaf>
__global__ void __launch_bounds__(G::NT)
k_apply_qt(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_tile, const double *tau_node,
           int *counters, double *C, int64_t ldc, int k) {
    using SM = Smem<G, CCOLS>;
    extern __shared__ __align__(16) double sm[];
    int *flag = reinterpret_cast<int *>(sm + SM::flag);
    double *tile = sm + SM::tile;
    const int t = blockIdx.x;
    if (kLeaf) {
        const int64_t row0 = plan.tile_row0[t];
        const int rows = plan.tile_rows[t];
        for (int j = threadIdx.x; j < G::NP; j += G::NT) sm[SM::taus + j] = j < n ? tau_tile[(int64_t)t * n + j] : 0.0;
        load_tile_y<G, CCOLS>(sm, A + row0, lda, rows, n);
        build_all_t<G, CCOLS, false>(sm, n, rows);
        double *Ct = C + row0;
        for (int c0 = 0; c0 < k; c0 += CCOLS) {
            const int kc = min(CCOLS, k - c0);
            stage_in<G::NT>(tile, G::LD, Ct + (int64_t)c0 * ldc, ldc, rows, kc, G::S, CCOLS);
            __syncthreads();
            apply_panels<G, CCOLS, false, true>(sm, n, rows, kc);
            stage_out<G::NT>(tile, G::LD, Ct + (int64_t)c0 * ldc, ldc, rows, kc);
            __syncthreads();
        }
    }
    // node stage (eq. localQTupdate) on the head rows, climbing the tree
    int p = plan.tile_parent[t];
    while (p >= 0) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const int old = atomicAdd(counters + p, 1);
            if (old == 1) counters[p] = 0;
            *flag = old;
        }
        __syncthreads();
        if (*flag != 1) return;
        __threadfence();
        const int a_t = plan.node_a[p];
        const int64_t ra = plan.tile_row0[a_t], rb = plan.tile_row0[p];
        for (int j = threadIdx.x; j < G::NP; j += G::NT)
            sm[SM::taus + j] = j < n ? tau_node[(int64_t)p * n + j] : 0.0;
        zero<G::NT>(sm + SM::ys, G::NP * G::LD);
        __syncthreads();
        load_node_y<G>(sm + SM::ys, A + rb, lda, n, true);
        __syncthreads();
        build_all_t<G, CCOLS, true>(sm, n, 2 * G::NP);
        for (int c0 = 0; c0 < k; c0 += CCOLS) {
            const int kc = min(CCOLS, k - c0);
            for (int e = threadIdx.x; e < CCOLS * 2 * G::NP; e += G::NT) {
                const int r = e % (2 * G::NP), c = e / (2 * G::NP);
                const bool top = r < G::NP;
                const int rr = top ? r : r - G::NP;
                const bool ok = rr < n && c < kc;
                const double v = __ldcg(C + (top ? ra : rb) + (ok ? rr + (int64_t)(c0 + c) * ldc : 0));
                tile[c * G::LD + r] = ok ? v : 0.0;
            }
            __syncthreads();
            apply_panels<G, CCOLS, true, true>(sm, n, 2 * G::NP, kc);
            for (int e = threadIdx.x; e < kc * n; e += G::NT) {
                const int r = e % n, c = e / n;
                C[ra + r + (int64_t)(c0 + c) * ldc] = tile[c * G::LD + r];
                C[rb + r + (int64_t)(c0 + c) * ldc] = tile[c * G::LD + G::NP + r];
            }
            __syncthreads();
        }
        p = plan.node_parent[p];
    }
}

// ============================================================ form Q (a9,a10)
template <class G>
__global__ void __launch_bounds__(G::NT)
k_formq_node(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_node, const int *ids,
             double *xbuf) {
    using SM = Smem<G, G::NP>;
    extern __shared__ __align__(16) double sm[];
    double *tile = sm + SM::tile;
    const int p = ids[blockIdx.x];
    const int a_t = plan.node_a[p];
    const int64_t nn = (int64_t)n * n;
    for (int j = threadIdx.x; j < G::NP; j += G::NT) sm[SM::taus + j] = j < n ? tau_node[(int64_t)p * n + j] : 0.0;
    zero<G::NT>(sm + SM::ys, G::NP * G::LD);
    zero<G::NT>(tile, G::NP * G::LD);
    __syncthreads();
    load_node_y<G>(sm + SM::ys, A + plan.tile_row0[p], lda, n, false);
    for (int e = threadIdx.x; e < n * n; e += G::NT) {
        const int r = e % n, c = e / n;
        tile[c * G::LD + r] = xbuf[a_t * nn + r + (int64_t)c * n];       // [X; 0]
    }
    __syncthreads();
    build_all_t<G, G::NP, true>(sm, n, 2 * G::NP);
    apply_panels<G, G::NP, true, false>(sm, n, 2 * G::NP, n);
    for (int e = threadIdx.x; e < n * n; e += G::NT) {
        const int r = e % n, c = e / n;
        xbuf[a_t * nn + r + (int64_t)c * n] = tile[c * G::LD + r];
        xbuf[(int64_t)p * nn + r + (int64_t)c * n] = tile[c * G::LD + G::NP + r];
    }
}

template <class G, int CCOLS>
__global__ void __launch_bounds__(G::NT)
k_formq_leaf(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_tile, const double *xbuf,
             double *Q, int64_t ldq) {
    using SM = Smem<G, CCOLS>;
    extern __shared__ __align__(16) double sm[];
    double *tile = sm + SM::tile;
    const int t = blockIdx.x;
    const int64_t row0 = plan.tile_row0[t];
    const int rows = plan.tile_rows[t];
    for (int j = threadIdx.x; j < G::NP; j += G::NT) sm[SM::taus + j] = j < n ? tau_tile[(int64_t)t * n + j] : 0.0;
    load_tile_y<G, CCOLS>(sm, A + row0, lda, rows, n);
    build_all_t<G, CCOLS, false>(sm, n, rows);
    const double *Xt = xbuf + (int64_t)t * n * n;
    for (int c0 = 0; c0 < n; c0 += CCOLS) {
        const int kc = min(CCOLS, n - c0);
        stage_in<G::NT>(tile, G::LD, Xt + (int64_t)c0 * n, n, n, kc, G::S, CCOLS);   // [X_t; 0]
        __syncthreads();
        apply_panels<G, CCOLS, false, false>(sm, n, rows, kc);
        stage_out<G::NT>(tile, G::LD, Q + row0 + (int64_t)c0 * ldq, ldq, rows, kc);
        __syncthreads();
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
template <class G>
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
        apply_panels<G, G::NP, true, true>(sm, n, 2 * G::NP, kc);
        for (int e = threadIdx.x; e < kc * n; e += G::NT) {
            const int r = e % n, c = e / n;
            const double ra = tile[c * G::LD + r];
            top[r + (int64_t)(c0 + c) * ldtop] = ra;
            if (head_role == 1) C[r + (int64_t)(c0 + c) * ldc] = ra;
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

int team_rows_for(int64_t max_rows) {
    if (max_rows <= 64) return 64;
    if (max_rows <= 128) return 128;
    return 192;
}

template <class G, bool kLeaf = true>
static cudaError_t launch_factor_w_t(const FactorArgs &f, cudaStream_t st) {
    const size_t sm = WSmem<G>::bytes;
    cudaError_t e = set_smem((const void *)k_factor_w<G, kLeaf>, sm);
    if (e != cudaSuccess) return e;
    k_factor_w<G, kLeaf><<<f.plan.L, 32, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile, f.tau_node, f.counters, f.R,
                                                    f.ldr);
    return cudaGetLastError();
}

cudaError_t launch_tree(const FactorArgs &f, cudaStream_t st) {
    switch ((f.n + 7) / 8) {
        case 1: case 2: return launch_factor_w_t<WGeo<2, 8>, false>(f, st);
        case 3: case 4: return launch_factor_w_t<WGeo<4, 8>, false>(f, st);
        case 5: case 6: return launch_factor_w_t<WGeo<6, 8>, false>(f, st);
        case 7: return launch_factor_w_t<WGeo<7, 8>, false>(f, st);
        default: return launch_factor_w_t<WGeo<8, 8>, false>(f, st);
    }
}

template <int NCB>
static cudaError_t launch_factor_w_n(const FactorArgs &f, cudaStream_t st) {
    if (f.max_rows <= 64) return launch_factor_w_t<WGeo<NCB, 8>>(f, st);
    if (f.max_rows <= 96) return launch_factor_w_t<WGeo<NCB, 12>>(f, st);
    if (f.max_rows <= 128) return launch_factor_w_t<WGeo<NCB, 16>>(f, st);
    return launch_factor_w_t<WGeo<NCB, 24>>(f, st);
}

cudaError_t launch_factor(const FactorArgs &f, cudaStream_t st) {
    const int ncb = (f.n + 7) / 8;
    switch (ncb) {
        case 1: case 2: return launch_factor_w_n<2>(f, st);
        case 3: case 4: return launch_factor_w_n<4>(f, st);
        case 5: case 6: return launch_factor_w_n<6>(f, st);
        case 7: return launch_factor_w_n<7>(f, st);
        default: return launch_factor_w_n<8>(f, st);
    }
}

template <class G, int CCOLS>
static cudaError_t launch_apply_t(const ApplyArgs &f, cudaStream_t st) {
    const size_t sm = Smem<G, CCOLS>::bytes;
    cudaError_t e;
    if (f.form_q) {
        e = set_smem((const void *)k_formq_leaf<G, CCOLS>, sm);
        if (e != cudaSuccess) return e;
        k_formq_leaf<G, CCOLS><<<f.plan.L, G::NT, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile, f.xbuf, f.C, f.ldc);
    } else {
        e = set_smem((const void *)k_apply_qt<G, CCOLS, true>, sm);
        if (e != cudaSuccess) return e;
        k_apply_qt<G, CCOLS, true><<<f.plan.L, G::NT, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile, f.tau_node,
                                                                f.counters, f.C, f.ldc, f.k);
    }
    return cudaGetLastError();
}

template <int NCB>
static cudaError_t launch_apply_n(const ApplyArgs &f, cudaStream_t st) {
    switch (team_rows_for(f.max_rows)) {
        case 64: return launch_apply_t<Geo<NCB, 8, NCB>, 8 * NCB>(f, st);
        case 128: return launch_apply_t<Geo<NCB, 16, NCB>, 8 * NCB>(f, st);
        default: return launch_apply_t<Geo<NCB, 24, NCB>, 8 * NCB>(f, st);
    }
}

// Node stage only of Q^T C (eq. localQTupdate on the tile heads), after the leaf stage.
template <class G>
static cudaError_t launch_apply_nodes_t(const ApplyArgs &f, cudaStream_t st) {
    constexpr int CCOLS = G::NP;
    const size_t sm = Smem<G, CCOLS>::bytes;
    cudaError_t e = set_smem((const void *)k_apply_qt<G, CCOLS, false>, sm);
    if (e != cudaSuccess) return e;
    k_apply_qt<G, CCOLS, false><<<f.plan.L, G::NT, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile, f.tau_node,
                                                             f.counters, f.C, f.ldc, f.k);
    return cudaGetLastError();
}

cudaError_t launch_apply_nodes(const ApplyArgs &f, cudaStream_t st) {
    return f.NP <= 32 ? launch_apply_nodes_t<Geo<4, 8, 4>>(f, st) : launch_apply_nodes_t<Geo<8, 8, 8>>(f, st);
}

cudaError_t launch_apply(const ApplyArgs &f, cudaStream_t st) {
    return f.NP <= 32 ? launch_apply_n<4>(f, st) : launch_apply_n<8>(f, st);
}

template <class G>
static cudaError_t launch_formq_nodes_t(const double *A, int64_t lda, int n, const DevPlan &plan,
                                        const double *tau_node, const int *ids, int count, double *xbuf,
                                        cudaStream_t st) {
    const size_t sm = Smem<G, G::NP>::bytes;
    cudaError_t e = set_smem((const void *)k_formq_node<G>, sm);
    if (e != cudaSuccess) return e;
    k_formq_node<G><<<count, G::NT, sm, st>>>(A, lda, n, plan, tau_node, ids, xbuf);
    return cudaGetLastError();
}

cudaError_t launch_formq_nodes(int NP, const double *A, int64_t lda, int n, const DevPlan &plan,
                               const double *tau_node, const int *ids, int count, double *xbuf, cudaStream_t st) {
    return NP <= 32 ? launch_formq_nodes_t<Geo<4, 8, 4>>(A, lda, n, plan, tau_node, ids, count, xbuf, st)
                    : launch_formq_nodes_t<Geo<8, 8, 8>>(A, lda, n, plan, tau_node, ids, count, xbuf, st);
}

cudaError_t launch_identity(double *X, int n, cudaStream_t st) {
    k_identity<<<(n * n + 255) / 256, 256, 0, st>>>(X, n);
    return cudaGetLastError();
}

cudaError_t launch_pack_r(const double *A, int64_t lda, int n, double *packed, cudaStream_t st) {
    k_pack_r<<<(n * n + 255) / 256, 256, 0, st>>>(A, lda, n, packed);
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
                                        int k, cudaStream_t st) {
    const size_t sm = Smem<G, G::NP>::bytes;
    cudaError_t e = set_smem((const void *)k_cross_apply<G>, sm);
    if (e != cudaSuccess) return e;
    k_cross_apply<G><<<1, G::NT, sm, st>>>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k);
    return cudaGetLastError();
}

cudaError_t launch_cross_apply(int NP, const double *Y1, const double *tau, double *top, int64_t ldtop,
                               const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n, int k,
                               cudaStream_t st) {
    return NP <= 32 ? launch_cross_apply_t<Geo<4, 8, 4>>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, st)
                    : launch_cross_apply_t<Geo<8, 8, 8>>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, st);
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
