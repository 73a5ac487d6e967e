// Kernels of the B200 TSQR hot path (sm_100a) and their host launchers.
// Product code; see tsqr_device.cuh for the column-owner team layout.
//
//  k_factor      (a2)+(a4)+(a6): tile Householder QR by one team per tile, then
//                the single-pass ticketed tree: the second team to finish below a
//                node runs the structured combine (Alg. QR:qnxn) and climbs; the
//                root writes R.
//  k_apply_qt    (a7)+(a8): tile reflectors on C (Q^T, forward), then the same
//                ticketed climb applying node reflectors to head rows.
//  k_formq_node  (a9): one tree step of the top-down pass [X_a; X_b] = Q_node [X; 0].
//  k_formq_leaf  (a10): Q_t = Q_tile [X_t; 0].
//  k_cross_*     (a5): butterfly round compute (stack by rank, combine / apply).
#include "tsqr_device.cuh"
#include "tsqr_kernels.h"

namespace tsqr {

// ============================================================== factor (a2,a4)
template <class T>
struct FactorSmem {
    static constexpr int SLD = T::S + 1;                       // odd: conflict-free column reads
    static constexpr int stage0 = SLD * T::NPAD;
    static constexpr int node = T::NPAD * T::LDR;
    static constexpr int stage = ((stage0 > node ? stage0 : node) + 1) / 2 * 2;
    static constexpr int xs = stage;                            // 2 * max(S, NPAD)
    static constexpr int xlen = 2 * (T::S > T::NPAD ? T::S : T::NPAD);
    static constexpr int red = xs + xlen;                       // 2 * 2 * G * NPAD
    static constexpr int alph = red + 4 * T::G * T::NPAD;
    static constexpr int taus = alph + 2;
    static constexpr int betas = taus + T::NPAD;
    static constexpr int scales = betas + T::NPAD;
    static constexpr int flag = scales + T::NPAD;
    static constexpr size_t bytes = (size_t)(flag + 2) * sizeof(double);
};

template <class T>
__device__ __forceinline__ void factor_combine(double *A, int64_t lda, int n, int64_t row_a, int64_t row_b, double *tau_out,
                               double *sm) {
    using F = FactorSmem<T>;
    constexpr int NP = T::NPAD, LDR = T::LDR;
    double *Ra = sm;
    const int c = T::col();
    // Ra: upper triangle of the left subtree's head (cross-team data: L2 loads)
    for (int e = threadIdx.x; e < NP * NP; e += T::NT) {
        const int r = e % NP, cc = e / NP;
        const bool ok = r <= cc && cc < n;
        const double v = __ldcg(A + row_a + (ok ? r + (int64_t)cc * lda : 0));
        Ra[cc * LDR + r] = ok ? v : 0.0;
    }
    double rb[NP];
    {
        const double *gb = A + row_b + (int64_t)(c < n ? c : 0) * lda;
        const int lim = c < n ? c : -1;                        // rows 0..c of column c
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            rb[i] = 0.0;
            if (i <= lim) rb[i] = __ldcg(gb + i);
        }
    }
    team_sync<T::NW>();
    team_node_qr<T>(Ra, rb, n, sm + F::xs, sm + F::red, sm + F::taus, sm + F::betas, sm + F::scales);
    for (int e = threadIdx.x; e < n * n; e += T::NT) {
        const int r = e % n, cc = e / n;
        if (r <= cc) A[row_a + r + (int64_t)cc * lda] = Ra[cc * LDR + r];
    }
    if (T::grp() == 0 && c < n) {
        double *gb = A + row_b + (int64_t)c * lda;
#pragma unroll
        for (int i = 0; i < NP; ++i)
            if (i <= c) gb[i] = rb[i];                          // Y1(:, c), eq. fact_2rs
    }
    for (int j = threadIdx.x; j < n; j += T::NT) tau_out[j] = sm[F::taus + j];
    team_sync<T::NW>();
}

template <class T>
__global__ void __launch_bounds__(T::NT)
k_factor(double *A, int64_t lda, int n, DevPlan plan, double *tau_tile, double *tau_node, int *counters,
         double *R, int64_t ldr) {
    using F = FactorSmem<T>;
    extern __shared__ __align__(16) double sm[];
    double *stage = sm;
    int *flag = reinterpret_cast<int *>(sm + F::flag);
    const int t = blockIdx.x;
    const int64_t row0 = plan.tile_row0[t];
    const int rows = plan.tile_rows[t];
    double *At = A + row0;
    const int c = T::col(), r0 = T::row0();

    stage_in_async<T::NT>(stage, F::SLD, At, lda, rows, n, T::S, T::NPAD);
    cp_async_wait_all();
    team_sync<T::NW>();
    double a[T::RT];
#pragma unroll
    for (int i = 0; i < T::RT; ++i) a[i] = stage[c * F::SLD + r0 + i];
    team_tile_qr<T>(a, n, sm + F::xs, sm + F::red, sm + F::alph, sm + F::taus, sm + F::betas, sm + F::scales);
#pragma unroll
    for (int i = 0; i < T::RT; ++i) stage[c * F::SLD + r0 + i] = a[i];
    team_sync<T::NW>();
    stage_out<T::NT>(stage, F::SLD, At, lda, rows, n);
    for (int j = threadIdx.x; j < n; j += T::NT) tau_tile[(int64_t)t * n + j] = sm[F::taus + j];

    // single-pass tree: climb while this team is the last arriver
    int p = plan.tile_parent[t];
    bool root = (p < 0);
    while (p >= 0) {
        if (!ticket<T::NW>(counters, p, flag)) return;
        const int a_t = plan.node_a[p];
        factor_combine<T>(A, lda, n, plan.tile_row0[a_t], plan.tile_row0[p], tau_node + (int64_t)p * n, sm);
        const int q = plan.node_parent[p];
        if (q < 0) root = true;
        p = q;
    }
    if (root && R != nullptr) {
        __threadfence();
        team_sync<T::NW>();
        for (int e = threadIdx.x; e < n * n; e += T::NT) {
            const int r = e % n, cc = e / n;
            R[r + (int64_t)cc * ldr] = (r <= cc) ? __ldcg(A + r + (int64_t)cc * lda) : 0.0;
        }
    }
}

// ========================================================= apply Q^T (a7,a8)
// Y tile (S x NPY) in smem with the unit diagonal and zeros above made explicit.
template <int NT>
__device__ __forceinline__ void load_y_tile(double *Ys, int yld, const double *At, int64_t lda, int rows, int n, int S, int NPY) {
    stage_in_async<NT>(Ys, yld, At, lda, rows, n, S, NPY);
    cp_async_wait_all();
    __syncthreads();
    for (int e = threadIdx.x; e < NPY * NPY; e += NT) {
        const int r = e % NPY, cc = e / NPY;
        if (r <= cc) Ys[cc * yld + r] = (r == cc && cc < n) ? 1.0 : 0.0;
    }
    __syncthreads();
}

template <class T, int NPY>
struct ApplySmem {
    static constexpr int YLD = T::S + 2;                        // even: 16-byte column reads
    static constexpr int LDY1 = NPY + 2;                        // Y1 columns: even (double2 reads)
    static constexpr int LDY = NPY + 1;                         // Ca columns: odd (per-lane reads)
    static constexpr int tile = YLD * NPY;
    static constexpr int node = NPY * LDY1 + T::NPAD * LDY;     // Y1 + Ca
    static constexpr int base = ((tile > node ? tile : node) + 1) / 2 * 2;
    static constexpr int red = base;                            // 2 * G * NPAD
    static constexpr int taus = red + 2 * T::G * T::NPAD;
    static constexpr int flag = taus + NPY;
    static constexpr size_t bytes = (size_t)(flag + 2) * sizeof(double);
};

// Band of C (rows [r0, r0+RT) of the tile, column c0 + c) <-> registers.
template <class T>
__device__ __forceinline__ void load_band(double (&cb)[T::RT], const double *Ct, int64_t ldc, int rows, int kc) {
    const int c = T::col(), r0 = T::row0();
    const double *g = Ct + (int64_t)(c < kc ? c : 0) * ldc + r0;
    const int lim = c < kc ? rows - r0 : 0;                    // valid rows of my band
    if (lim >= T::RT) {
#pragma unroll
        for (int i = 0; i < T::RT; ++i) cb[i] = g[i];
    } else {
#pragma unroll
        for (int i = 0; i < T::RT; ++i) {
            cb[i] = 0.0;
            if (i < lim) cb[i] = g[i];
        }
    }
}

template <class T>
__device__ __forceinline__ void store_band(const double (&cb)[T::RT], double *Ct, int64_t ldc, int rows, int kc) {
    const int c = T::col(), r0 = T::row0();
    if (c >= kc) return;
    double *g = Ct + (int64_t)c * ldc + r0;
    if (r0 + T::RT <= rows) {
#pragma unroll
        for (int i = 0; i < T::RT; ++i) g[i] = cb[i];
    } else {
#pragma unroll
        for (int i = 0; i < T::RT; ++i)
            if (r0 + i < rows) g[i] = cb[i];
    }
}

// Node stage of apply Q^T at node p for columns [c0, c0+kc) of C: heads of the
// node's two subtrees (rows ra.. and rb.. of C), Y1 from A (head of tile p).
template <class T, int NPY>
__device__ __forceinline__ void apply_node(const double *A, int64_t lda, int n, int64_t ra, int64_t rb, const double *taug,
                           double *C, int64_t ldc, int c0, int kc, double *sm) {
    using F = ApplySmem<T, NPY>;
    constexpr int LDY = F::LDY, LDY1 = F::LDY1;
    double *Y1 = sm, *Ca = sm + NPY * LDY1;
    double *taus = sm + F::taus;
    const int c = T::col();
    for (int e = threadIdx.x; e < NPY * NPY; e += T::NT) {
        const int r = e % NPY, cc = e / NPY;
        const bool ok = r <= cc && cc < n;
        const double v = __ldcg(A + rb + (ok ? r + (int64_t)cc * lda : 0));
        Y1[cc * LDY1 + r] = ok ? v : 0.0;
    }
    for (int j = threadIdx.x; j < NPY; j += T::NT) taus[j] = j < n ? taug[j] : 0.0;
    for (int e = threadIdx.x; e < NPY * T::NPAD; e += T::NT) {
        const int r = e % NPY, cc = e / NPY;
        const bool ok = r < n && cc < kc;
        const double v = __ldcg(C + ra + (ok ? r + (int64_t)(c0 + cc) * ldc : 0));
        Ca[cc * LDY + r] = ok ? v : 0.0;
    }
    double cbh[NPY];
    {
        const double *g = C + rb + (int64_t)(c0 + (c < kc ? c : 0)) * ldc;
        const int lim = c < kc ? n : 0;
#pragma unroll
        for (int i = 0; i < NPY; ++i) {
            cbh[i] = 0.0;
            if (i < lim) cbh[i] = __ldcg(g + i);
        }
    }
    team_sync<T::NW>();
    const bool act = T::grp() == 0;         // row groups > 0 own the same columns: idle
    if (act) team_node_apply<NPY, LDY1, LDY, true>(Y1, taus, Ca, cbh, n, c);
    team_sync<T::NW>();
    for (int e = threadIdx.x; e < n * kc; e += T::NT) {
        const int r = e % n, cc = e / n;
        C[ra + r + (int64_t)(c0 + cc) * ldc] = Ca[cc * LDY + r];
    }
    if (act && c < kc) {
        double *g = C + rb + (int64_t)(c0 + c) * ldc;
#pragma unroll
        for (int i = 0; i < NPY; ++i)
            if (i < n) g[i] = cbh[i];
    }
    team_sync<T::NW>();
}

template <class T, int NPY>
__global__ void __launch_bounds__(T::NT)
k_apply_qt(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_tile, const double *tau_node,
           int *counters, double *C, int64_t ldc, int k) {
    using F = ApplySmem<T, NPY>;
    extern __shared__ __align__(16) double sm[];
    double *Ys = sm;
    double *taus = sm + F::taus;
    int *flag = reinterpret_cast<int *>(sm + F::flag);
    const int t = blockIdx.x;
    const int64_t row0 = plan.tile_row0[t];
    const int rows = plan.tile_rows[t];
    load_y_tile<T::NT>(Ys, F::YLD, A + row0, lda, rows, n, T::S, NPY);
    for (int j = threadIdx.x; j < NPY; j += T::NT) taus[j] = j < n ? tau_tile[(int64_t)t * n + j] : 0.0;
    team_sync<T::NW>();
    double *Ct = C + row0;
#pragma unroll 1
    for (int c0 = 0; c0 < k; c0 += T::NPAD) {
        const int kc = min(T::NPAD, k - c0);
        double cb[T::RT];
        load_band<T>(cb, Ct + (int64_t)c0 * ldc, ldc, rows, kc);
        team_tile_apply<T, true>(cb, n, Ys, F::YLD, taus, sm + F::red);
        store_band<T>(cb, Ct + (int64_t)c0 * ldc, ldc, rows, kc);
    }
    // node stage (eq. localQTupdate) on the head rows, climbing the tree
    int p = plan.tile_parent[t];
    while (p >= 0) {
        if (!ticket<T::NW>(counters, p, flag)) return;
        const int a_t = plan.node_a[p];
        for (int c0 = 0; c0 < k; c0 += T::NPAD)
            apply_node<T, NPY>(A, lda, n, plan.tile_row0[a_t], plan.tile_row0[p], tau_node + (int64_t)p * n, C, ldc,
                               c0, min(T::NPAD, k - c0), sm);
        p = plan.node_parent[p];
    }
}

// ============================================================ form Q (a9,a10)
// One top-down step: every node id in ids[] computes [X_a; X_b] = Q_node [X; 0]
// with X = xbuf[a] (n x n, ld n), storing X_a -> xbuf[a], X_b -> xbuf[b].
template <int NPY>
struct NodeSmem {
    static constexpr int LDY1 = NPY + 2, LDY = NPY + 1;
    static constexpr int taus = NPY * LDY1 + NPY * LDY + 1;
    static constexpr size_t bytes = (size_t)(taus + NPY + 2) * sizeof(double);
};

template <int NPY>
__global__ void __launch_bounds__(NPY)
k_formq_node(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_node, const int *ids,
             double *xbuf) {
    using N = NodeSmem<NPY>;
    constexpr int LDY = N::LDY, LDY1 = N::LDY1, NT = NPY;
    extern __shared__ __align__(16) double sm[];
    double *Y1 = sm, *Xa = sm + NPY * LDY1, *taus = sm + N::taus;
    const int p = ids[blockIdx.x];
    const int a_t = plan.node_a[p];
    const int64_t nn = (int64_t)n * n;
    const int c = threadIdx.x;
    for (int e = threadIdx.x; e < NPY * NPY; e += NT) {
        const int r = e % NPY, cc = e / NPY;
        Y1[cc * LDY1 + r] = (r <= cc && cc < n) ? A[plan.tile_row0[p] + r + (int64_t)cc * lda] : 0.0;
        Xa[cc * LDY + r] = (r < n && cc < n) ? xbuf[a_t * nn + r + (int64_t)cc * n] : 0.0;
    }
    for (int j = threadIdx.x; j < NPY; j += NT) taus[j] = j < n ? tau_node[(int64_t)p * n + j] : 0.0;
    __syncthreads();
    double xb[NPY];
#pragma unroll
    for (int i = 0; i < NPY; ++i) xb[i] = 0.0;
    team_node_apply<NPY, LDY1, LDY, false>(Y1, taus, Xa, xb, n, c);
    __syncthreads();
    if (c < n) {
#pragma unroll
        for (int i = 0; i < NPY; ++i)
            if (i < n) {
                xbuf[a_t * nn + i + (int64_t)c * n] = Xa[c * LDY + i];
                xbuf[(int64_t)p * nn + i + (int64_t)c * n] = xb[i];
            }
    }
}

template <class T, int NPY>
__global__ void __launch_bounds__(T::NT)
k_formq_leaf(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_tile, const double *xbuf,
             double *Q, int64_t ldq) {
    using F = ApplySmem<T, NPY>;
    extern __shared__ __align__(16) double sm[];
    double *Ys = sm;
    double *taus = sm + F::taus;
    const int t = blockIdx.x;
    const int64_t row0 = plan.tile_row0[t];
    const int rows = plan.tile_rows[t];
    const int c = T::col(), r0 = T::row0();
    load_y_tile<T::NT>(Ys, F::YLD, A + row0, lda, rows, n, T::S, NPY);
    for (int j = threadIdx.x; j < NPY; j += T::NT) taus[j] = j < n ? tau_tile[(int64_t)t * n + j] : 0.0;
    team_sync<T::NW>();
    const double *Xt = xbuf + (int64_t)t * n * n;
#pragma unroll 1
    for (int c0 = 0; c0 < n; c0 += T::NPAD) {
        const int kc = min(T::NPAD, n - c0);
        double cb[T::RT];
        // [X_t; 0]
        const double *xg = Xt + (int64_t)(c0 + (c < kc ? c : 0)) * n + r0;
        const int lim = c < kc ? n - r0 : 0;
#pragma unroll
        for (int i = 0; i < T::RT; ++i) {
            cb[i] = 0.0;
            if (i < lim) cb[i] = xg[i];
        }
        team_tile_apply<T, false>(cb, n, Ys, F::YLD, taus, sm + F::red);
        store_band<T>(cb, Q + row0 + (int64_t)c0 * ldq, ldq, rows, kc);
    }
}

__global__ void k_identity(double *X, int n) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x)
        X[e] = (e % n == e / n) ? 1.0 : 0.0;
}

// ================================================================ output / comm
__global__ void k_write_r(const double *A, int64_t lda, int n, double *R, int64_t ldr) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x) {
        const int r = e % n, c = e / n;
        R[r + (int64_t)c * ldr] = (r <= c) ? A[r + (int64_t)c * lda] : 0.0;
    }
}

__global__ void k_pack_r(const double *A, int64_t lda, int n, double *packed) {
    // column-packed upper triangle: column c holds rows 0..c at offset c(c+1)/2
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
template <class T>
__global__ void __launch_bounds__(T::NT)
k_cross_factor(double *A, int64_t lda, int n, const double *partner_packed, int is_lower, double *Y1_out,
               double *tau_out, double *R, int64_t ldr) {
    using F = FactorSmem<T>;
    constexpr int NP = T::NPAD, LDR = T::LDR;
    extern __shared__ __align__(16) double sm[];
    double *Ra = sm;
    const int c = T::col();
    auto mine_at = [&](int r, int cc) { return A[r + (int64_t)cc * lda]; };
    auto theirs_at = [&](int r, int cc) { return partner_packed[(int64_t)cc * (cc + 1) / 2 + r]; };
    for (int e = threadIdx.x; e < NP * NP; e += T::NT) {
        const int r = e % NP, cc = e / NP;
        const bool ok = r <= cc && cc < n;
        Ra[cc * LDR + r] = ok ? (is_lower ? mine_at(r, cc) : theirs_at(r, cc)) : 0.0;
    }
    double rb[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        const bool ok = i <= c && c < n;
        rb[i] = ok ? (is_lower ? theirs_at(i, c) : mine_at(i, c)) : 0.0;
    }
    team_sync<T::NW>();
    team_node_qr<T>(Ra, rb, n, sm + F::xs, sm + F::red, sm + F::taus, sm + F::betas, sm + F::scales);
    for (int e = threadIdx.x; e < n * n; e += T::NT) {
        const int r = e % n, cc = e / n;
        if (r <= cc) A[r + (int64_t)cc * lda] = Ra[cc * LDR + r];          // new current R
        if (R) R[r + (int64_t)cc * ldr] = (r <= cc) ? Ra[cc * LDR + r] : 0.0;
    }
    if (c < n) {
#pragma unroll
        for (int i = 0; i < NP; ++i)
            if (i < n) Y1_out[i + (int64_t)c * n] = (i <= c) ? rb[i] : 0.0;
    }
    for (int j = threadIdx.x; j < n; j += T::NT) tau_out[j] = sm[F::taus + j];
}

// Butterfly round of apply Q^T on the R coordinates (n x k tops).
template <int NPY>
__global__ void __launch_bounds__(64)
k_cross_apply(const double *Y1g, const double *taug, double *top, int64_t ldtop, const double *partner_top,
              int is_lower, int head_role, double *C, int64_t ldc, int n, int k) {
    constexpr int LDY = NPY + 1, LDY1 = NPY + 2, NT = 64;
    extern __shared__ __align__(16) double sm[];
    double *Y1 = sm, *Ca = sm + NPY * LDY1, *taus = Ca + NT * LDY;
    const int c = threadIdx.x;
    for (int e = threadIdx.x; e < NPY * NPY; e += NT) {
        const int r = e % NPY, cc = e / NPY;
        Y1[cc * LDY1 + r] = (r < n && cc < n) ? Y1g[r + (int64_t)cc * n] : 0.0;
    }
    for (int j = threadIdx.x; j < NPY; j += NT) taus[j] = j < n ? taug[j] : 0.0;
    for (int c0 = 0; c0 < k; c0 += NT) {
        const int kc = min(NT, k - c0);
        const double *mine = top + (int64_t)c0 * ldtop;
        const double *theirs = partner_top + (int64_t)c0 * n;
        __syncthreads();
        for (int e = threadIdx.x; e < NPY * NT; e += NT) {
            const int r = e % NPY, cc = e / NPY;
            const bool ok = r < n && cc < kc;
            Ca[cc * LDY + r] = ok ? (is_lower ? mine[r + (int64_t)cc * ldtop] : theirs[r + (int64_t)cc * n]) : 0.0;
        }
        double cbh[NPY];
#pragma unroll
        for (int i = 0; i < NPY; ++i) {
            const bool ok = i < n && c < kc;
            cbh[i] = ok ? (is_lower ? theirs[i + (int64_t)c * n] : mine[i + (int64_t)c * ldtop]) : 0.0;
        }
        __syncthreads();
        team_node_apply<NPY, LDY1, LDY, true>(Y1, taus, Ca, cbh, n, c);
        __syncthreads();
        if (c < kc) {
#pragma unroll
            for (int i = 0; i < NPY; ++i)
                if (i < n) {
                    const double ra = Ca[c * LDY + i];
                    top[i + (int64_t)(c0 + c) * ldtop] = ra;
                    if (head_role == 1) C[i + (int64_t)(c0 + c) * ldc] = ra;
                    if (head_role == 2) C[i + (int64_t)(c0 + c) * ldc] = cbh[i];
                }
        }
    }
}

// Root X of this rank for form-Q: top-down over the butterfly nodes.
template <int NPY>
__global__ void __launch_bounds__(NPY)
k_cross_root_x(const double *Y1s, const double *taus_g, int rounds, int rank, int n, double *X0) {
    constexpr int LDY = NPY + 1, LDY1 = NPY + 2, NT = NPY;
    extern __shared__ __align__(16) double sm[];
    double *Y1 = sm, *Xa = sm + NPY * LDY1, *taus = Xa + NPY * LDY;
    const int c = threadIdx.x;
    for (int e = threadIdx.x; e < NPY * NPY; e += NT) {
        const int r = e % NPY, cc = e / NPY;
        Xa[cc * LDY + r] = (r == cc && r < n) ? 1.0 : 0.0;
    }
    double xb[NPY];
    for (int k = rounds; k >= 1; --k) {
        const double *Y1g = Y1s + (int64_t)(k - 1) * n * n;
        __syncthreads();
        for (int e = threadIdx.x; e < NPY * NPY; e += NT) {
            const int r = e % NPY, cc = e / NPY;
            Y1[cc * LDY1 + r] = (r < n && cc < n) ? Y1g[r + (int64_t)cc * n] : 0.0;
        }
        for (int j = threadIdx.x; j < NPY; j += NT) taus[j] = j < n ? taus_g[(k - 1) * n + j] : 0.0;
#pragma unroll
        for (int i = 0; i < NPY; ++i) xb[i] = 0.0;
        __syncthreads();
        team_node_apply<NPY, LDY1, LDY, false>(Y1, taus, Xa, xb, n, c);
        const bool lower = ((rank >> (k - 1)) & 1) == 0;
        __syncthreads();
        if (!lower) {
#pragma unroll
            for (int i = 0; i < NPY; ++i) Xa[c * LDY + i] = xb[i];
        }
    }
    __syncthreads();
    if (c < n)
        for (int i = 0; i < n; ++i) X0[i + (int64_t)c * n] = Xa[c * LDY + i];
}

// ================================================================= launchers
static cudaError_t set_smem(const void *fn, size_t bytes) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Tile shapes (rows a team holds): S = G * RT.
template <int CW, int S> struct TeamFor;
template <int CW> struct TeamFor<CW, 64> { using type = Team<CW, 1, 64>; };
template <int CW> struct TeamFor<CW, 96> { using type = Team<CW, 1, 96>; };
template <int CW> struct TeamFor<CW, 128> { using type = Team<CW, 2, 64>; };
template <int CW> struct TeamFor<CW, 192> { using type = Team<CW, 2, 96>; };

int team_rows_for(int64_t max_rows) {
    if (max_rows <= 64) return 64;
    if (max_rows <= 96) return 96;
    if (max_rows <= 128) return 128;
    return 192;
}

template <class T>
static cudaError_t launch_factor_t(const FactorArgs &f, cudaStream_t st) {
    const size_t sm = FactorSmem<T>::bytes;
    cudaError_t e = set_smem((const void *)k_factor<T>, sm);
    if (e != cudaSuccess) return e;
    k_factor<T><<<f.plan.L, T::NT, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile, f.tau_node, f.counters, f.R, f.ldr);
    return cudaGetLastError();
}

template <int CW>
static cudaError_t launch_factor_cw(const FactorArgs &f, cudaStream_t st) {
    switch (team_rows_for(f.max_rows)) {
        case 64: return launch_factor_t<typename TeamFor<CW, 64>::type>(f, st);
        case 96: return launch_factor_t<typename TeamFor<CW, 96>::type>(f, st);
        case 128: return launch_factor_t<typename TeamFor<CW, 128>::type>(f, st);
        default: return launch_factor_t<typename TeamFor<CW, 192>::type>(f, st);
    }
}

cudaError_t launch_factor(const FactorArgs &f, cudaStream_t st) {
    return f.NP <= 32 ? launch_factor_cw<1>(f, st) : launch_factor_cw<2>(f, st);
}

template <class T, int NPY>
static cudaError_t launch_apply_t(const ApplyArgs &f, cudaStream_t st) {
    const size_t sm = ApplySmem<T, NPY>::bytes;
    cudaError_t e;
    if (f.form_q) {
        e = set_smem((const void *)k_formq_leaf<T, NPY>, sm);
        if (e != cudaSuccess) return e;
        k_formq_leaf<T, NPY><<<f.plan.L, T::NT, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile, f.xbuf, f.C, f.ldc);
    } else {
        e = set_smem((const void *)k_apply_qt<T, NPY>, sm);
        if (e != cudaSuccess) return e;
        k_apply_qt<T, NPY><<<f.plan.L, T::NT, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile, f.tau_node, f.counters,
                                                         f.C, f.ldc, f.k);
    }
    return cudaGetLastError();
}

// Apply teams hold 64 columns of C (two column warps) per pass, in bands of at
// most 64 rows (a 96-row band of C plus the streamed reflector chunks would not
// fit the 255-register budget without spills).
template <int NPY>
static cudaError_t launch_apply_np(const ApplyArgs &f, cudaStream_t st) {
    switch (team_rows_for(f.max_rows)) {
        case 64: return launch_apply_t<Team<2, 1, 64>, NPY>(f, st);
        case 96: return launch_apply_t<Team<2, 2, 48>, NPY>(f, st);
        case 128: return launch_apply_t<Team<2, 2, 64>, NPY>(f, st);
        default: return launch_apply_t<Team<2, 4, 48>, NPY>(f, st);
    }
}

cudaError_t launch_apply(const ApplyArgs &f, cudaStream_t st) {
    return f.NP <= 32 ? launch_apply_np<32>(f, st) : launch_apply_np<64>(f, st);
}

template <int NPY>
static cudaError_t launch_formq_nodes_t(const double *A, int64_t lda, int n, const DevPlan &plan,
                                        const double *tau_node, const int *ids, int count, double *xbuf,
                                        cudaStream_t st) {
    const size_t sm = NodeSmem<NPY>::bytes;
    cudaError_t e = set_smem((const void *)k_formq_node<NPY>, sm);
    if (e != cudaSuccess) return e;
    k_formq_node<NPY><<<count, NPY, sm, st>>>(A, lda, n, plan, tau_node, ids, xbuf);
    return cudaGetLastError();
}

cudaError_t launch_formq_nodes(int NP, const double *A, int64_t lda, int n, const DevPlan &plan,
                               const double *tau_node, const int *ids, int count, double *xbuf, cudaStream_t st) {
    return NP <= 32 ? launch_formq_nodes_t<32>(A, lda, n, plan, tau_node, ids, count, xbuf, st)
                    : launch_formq_nodes_t<64>(A, lda, n, plan, tau_node, ids, count, xbuf, st);
}

cudaError_t launch_identity(double *X, int n, cudaStream_t st) {
    k_identity<<<(n * n + 255) / 256, 256, 0, st>>>(X, n);
    return cudaGetLastError();
}

cudaError_t launch_write_r(int, const double *A, int64_t lda, int n, double *R, int64_t ldr, cudaStream_t st) {
    k_write_r<<<(n * n + 255) / 256, 256, 0, st>>>(A, lda, n, R, ldr);
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

template <class T>
static cudaError_t launch_cross_factor_t(double *A, int64_t lda, int n, const double *pp, int is_lower, double *Y1,
                                         double *tau, double *R, int64_t ldr, cudaStream_t st) {
    const size_t sm = FactorSmem<T>::bytes;
    cudaError_t e = set_smem((const void *)k_cross_factor<T>, sm);
    if (e != cudaSuccess) return e;
    k_cross_factor<T><<<1, T::NT, sm, st>>>(A, lda, n, pp, is_lower, Y1, tau, R, ldr);
    return cudaGetLastError();
}

cudaError_t launch_cross_factor(int NP, double *A, int64_t lda, int n, const double *pp, int is_lower, double *Y1,
                                double *tau, double *R, int64_t ldr, cudaStream_t st) {
    return NP <= 32 ? launch_cross_factor_t<Team<1, 1, 64>>(A, lda, n, pp, is_lower, Y1, tau, R, ldr, st)
                    : launch_cross_factor_t<Team<2, 1, 64>>(A, lda, n, pp, is_lower, Y1, tau, R, ldr, st);
}

template <int NPY>
static cudaError_t launch_cross_apply_t(const double *Y1, const double *tau, double *top, int64_t ldtop,
                                        const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n,
                                        int k, cudaStream_t st) {
    const size_t sm = (size_t)(NPY * (NPY + 2) + 64 * (NPY + 1) + NPY + 2) * sizeof(double);
    cudaError_t e = set_smem((const void *)k_cross_apply<NPY>, sm);
    if (e != cudaSuccess) return e;
    k_cross_apply<NPY><<<1, 64, sm, st>>>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k);
    return cudaGetLastError();
}

cudaError_t launch_cross_apply(int NP, const double *Y1, const double *tau, double *top, int64_t ldtop,
                               const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n, int k,
                               cudaStream_t st) {
    return NP <= 32 ? launch_cross_apply_t<32>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, st)
                    : launch_cross_apply_t<64>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, st);
}

template <int NPY>
static cudaError_t launch_cross_root_x_t(const double *Y1s, const double *taus, int rounds, int rank, int n,
                                         double *X0, cudaStream_t st) {
    const size_t sm = (size_t)(NPY * (NPY + 2) + NPY * (NPY + 1) + NPY + 2) * sizeof(double);
    cudaError_t e = set_smem((const void *)k_cross_root_x<NPY>, sm);
    if (e != cudaSuccess) return e;
    k_cross_root_x<NPY><<<1, NPY, sm, st>>>(Y1s, taus, rounds, rank, n, X0);
    return cudaGetLastError();
}

cudaError_t launch_cross_root_x(int NP, const double *Y1s, const double *taus, int rounds, int rank, int n,
                                double *X0, cudaStream_t st) {
    return NP <= 32 ? launch_cross_root_x_t<32>(Y1s, taus, rounds, rank, n, X0, st)
                    : launch_cross_root_x_t<64>(Y1s, taus, rounds, rank, n, X0, st);
}

}  // namespace tsqr
