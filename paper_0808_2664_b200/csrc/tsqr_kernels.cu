// Kernels of the B200 TSQR hot path (sm_100a) and their host launchers.
// Product code; see tsqr_device.cuh for the register/smem layout.
//
//  k_factor      (a2)+(a4)+(a6): tile Householder QR, then the single-pass
//                ticketed tree: the second CTA to finish below a node runs the
//                structured combine (Alg. QR:qnxn) and climbs; the root writes R.
//  k_apply_qt    (a7)+(a8): tile reflectors on C (Q^T, forward), then the same
//                ticketed climb applying node reflectors to head rows.
//  k_formq_node  (a9): one tree step of the top-down pass [X_a; X_b] = Q_node [X; 0].
//  k_formq_leaf  (a10): Q_t = Q_tile [X_t; 0].
//  k_cross_*     (a5): butterfly round compute (stack by rank, combine / apply).
#include "tsqr_kernels.h"
#include "tsqr_device.cuh"

#include <cstdio>

namespace tsqr {

// ------------------------------------------------------------- shared pieces
template <int NP>
__device__ void combine_node(double *A, int64_t lda, int n, int64_t row_a, int64_t row_b,
                             double *tau_out, double *sm, double *red, double *taus) {
    double *Ra = sm, *Rb = sm + NP * (NP + 1);
    load_upper<NP, true>(Ra, A + row_a, lda, n);
    load_upper<NP, true>(Rb, A + row_b, lda, n);
    __syncthreads();
    node_qr<NP>(Ra, Rb, n, red, taus);
    store_upper<NP>(Ra, A + row_a, lda, n);          // R of the merged subtree
    store_upper<NP>(Rb, A + row_b, lda, n);          // Y1 of the node (eq. fact_2rs)
    for (int j = threadIdx.x; j < n; j += kThreads) tau_out[j] = taus[j];
    __syncthreads();
}

template <int NP>
__device__ void write_r_block(const double *A, int64_t lda, int n, double *R, int64_t ldr) {
    for (int e = threadIdx.x; e < n * n; e += kThreads) {
        const int r = e % n, c = e / n;
        R[r + (int64_t)c * ldr] = (r <= c) ? __ldcg(A + r + (int64_t)c * lda) : 0.0;
    }
}

// ============================================================== factor (a2,a4)
template <int NP, int RT>
struct FactorSmem {
    using Lt = Layout<NP, RT>;
    static constexpr int s0 = Lt::SLD * NP, s1 = 2 * NP * (NP + 1);
    static constexpr int stage = ((s0 > s1 ? s0 : s1) + 1) / 2 * 2;        // even: 16 B aligned
    static constexpr size_t doubles = (size_t)stage + Lt::S + 2 * kWarps * NP + 2 * NP + 3 * NP + 2;
};
template <int NP, int RT>
__global__ void __launch_bounds__(kThreads, (RT * Layout<NP, RT>::CPL <= 32) ? 2 : 1)
k_factor(double *A, int64_t lda, int n, DevPlan plan, double *tau_tile, double *tau_node,
         int *counters, double *R, int64_t ldr) {
    using Lt = Layout<NP, RT>;
    constexpr int STAGE = FactorSmem<NP, RT>::stage;
    extern __shared__ __align__(16) double smem[];
    double *stage = smem;                               // max(SLD * NP, 2 NP (NP+1))
    double *xs = stage + STAGE;
    double *red = xs + Lt::S;                           // 2 * kWarps * NP
    double *rowj = red + 2 * kWarps * NP;               // 2 * NP
    double *taus = rowj + 2 * NP;                       // NP
    double *betas = taus + NP, *scales = betas + NP;    // NP, NP
    int *flag = reinterpret_cast<int *>(scales + NP);

    const int t = blockIdx.x;
    const int64_t row0 = plan.tile_row0[t];
    const int rows = plan.tile_rows[t];
    double *At = A + row0;

    stage_in_async(stage, Lt::SLD, At, lda, rows, n, Lt::S, NP);
    cp_async_wait_all();
    __syncthreads();
    double a[RT][Lt::CPL];
    smem_to_regs<Lt>(stage, a);
    tile_qr<Lt>(a, n, xs, red, rowj, taus, betas, scales);
    __syncthreads();
    regs_to_smem<Lt>(stage, a);
    __syncthreads();
    stage_out(stage, Lt::SLD, At, lda, rows, n);
    for (int j = threadIdx.x; j < n; j += kThreads) tau_tile[(int64_t)t * n + j] = taus[j];

    // single-pass tree: climb while this CTA is the last arriver
    int p = plan.tile_parent[t];
    bool root = (p < 0);
    while (p >= 0) {
        if (!ticket(counters, p, flag)) return;
        const int a_t = plan.node_a[p];
        combine_node<NP>(A, lda, n, plan.tile_row0[a_t], plan.tile_row0[p],
                         tau_node + (int64_t)p * n, stage, red, taus);
        const int q = plan.node_parent[p];
        if (q < 0) root = true;
        p = q;
    }
    if (root && R != nullptr) {
        __threadfence();
        __syncthreads();
        write_r_block<NP>(A, lda, n, R, ldr);
    }
}

// ========================================================= apply Q^T (a7,a8)
// Y tile in smem with the unit diagonal and zeros above made explicit: the
// tile is staged with cp.async, then rows <= c of each column are overwritten.
template <int NP, int S>
__device__ void load_y_tile(double *Ys, int yld, const double *At, int64_t lda, int rows, int n) {
    stage_in_async(Ys, yld, At, lda, rows, n, S, NP);
    cp_async_wait_all();
    __syncthreads();
    for (int e = threadIdx.x; e < NP * NP; e += kThreads) {
        const int r = e % NP, c = e / NP;
        if (r <= c) Ys[c * yld + r] = (r == c && c < n) ? 1.0 : 0.0;
    }
}

template <int NP, int RT, int KC>
struct ApplyCfg {
    using Lt = Layout<NP, RT>;
    static constexpr int S = Lt::S;
    static constexpr int YLD = S + 2;                  // even: 16-byte vector reads
    static constexpr int LCC = KC < 32 ? KC : 32;
    static constexpr int RTC = S / (kWarps * (32 / LCC));
    using Ct = Layout<KC, RTC>;
    static_assert(Ct::S == S, "C tile must match the Y tile");
    static constexpr int REDW = NP > KC ? NP : KC;
    static constexpr int tile_area = YLD * NP + Ct::SLD * KC;
    static constexpr int node_area = 3 * NP * (NP + 1);
    static constexpr int base = ((tile_area > node_area ? tile_area : node_area) + 1) / 2 * 2;
    static constexpr size_t smem_doubles = (size_t)base + 2 * kWarps * REDW + NP + 4;
};

template <int NP, int RT, int KC>
__global__ void __launch_bounds__(kThreads, 1)
k_apply_qt(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_tile,
           const double *tau_node, int *counters, double *C, int64_t ldc, int k) {
    using Cfg = ApplyCfg<NP, RT, KC>;
    using Ct = typename Cfg::Ct;
    constexpr int S = Cfg::S, YLD = Cfg::YLD, REDW = Cfg::REDW;
    extern __shared__ __align__(16) double smem[];
    double *Ys = smem;                                   // YLD * NP
    double *Cs = Ys + YLD * NP;                          // Ct::SLD * KC
    double *red = smem + Cfg::base;                      // 2 * kWarps * REDW
    double *taus = red + 2 * kWarps * REDW;              // NP
    int *flag = reinterpret_cast<int *>(taus + NP);

    const int t = blockIdx.x;
    const int64_t row0 = plan.tile_row0[t];
    const int rows = plan.tile_rows[t];
    load_y_tile<NP, S>(Ys, YLD, A + row0, lda, rows, n);
    for (int j = threadIdx.x; j < NP; j += kThreads) taus[j] = j < n ? tau_tile[(int64_t)t * n + j] : 0.0;
    __syncthreads();
    double *Ct0 = C + row0;
    for (int c0 = 0; c0 < k; c0 += KC) {
        const int kc = min(KC, k - c0);
        stage_in_async(Cs, Ct::SLD, Ct0 + (int64_t)c0 * ldc, ldc, rows, kc, S, KC);
        cp_async_wait_all();
        __syncthreads();
        double c[Ct::RT][Ct::CPL];
        smem_to_regs<Ct>(Cs, c);
        tile_apply<Ct, true>(c, n, Ys, YLD, taus, red);
        regs_to_smem<Ct>(Cs, c);
        __syncthreads();
        stage_out(Cs, Ct::SLD, Ct0 + (int64_t)c0 * ldc, ldc, rows, kc);
        __syncthreads();
    }
    // node stage (eq. localQTupdate) on the head rows, climbing the tree
    int p = plan.tile_parent[t];
    double *Y1 = smem, *Ca = Y1 + NP * (NP + 1), *Cb = Ca + NP * (NP + 1);
    while (p >= 0) {
        if (!ticket(counters, p, flag)) return;
        const int a_t = plan.node_a[p];
        const int64_t ra = plan.tile_row0[a_t], rb = plan.tile_row0[p];
        load_upper<NP, true>(Y1, A + rb, lda, n);
        for (int j = threadIdx.x; j < NP; j += kThreads) taus[j] = j < n ? tau_node[(int64_t)p * n + j] : 0.0;
        for (int c0 = 0; c0 < k; c0 += NP) {
            const int kc = min(NP, k - c0);
            load_block<NP, true>(Ca, C + ra + (int64_t)c0 * ldc, ldc, n, kc);
            load_block<NP, true>(Cb, C + rb + (int64_t)c0 * ldc, ldc, n, kc);
            __syncthreads();
            node_apply<NP, true>(Y1, taus, Ca, Cb, n, red);
            store_block<NP>(Ca, C + ra + (int64_t)c0 * ldc, ldc, n, kc);
            store_block<NP>(Cb, C + rb + (int64_t)c0 * ldc, ldc, n, kc);
            __syncthreads();
        }
        p = plan.node_parent[p];
    }
}

template <int NP>
struct NodeSmem {
    static constexpr int red_off = (3 * NP * (NP + 1) + 1) / 2 * 2;
    static constexpr size_t doubles = (size_t)red_off + 2 * kWarps * NP + NP + 4;
};

// ============================================================ form Q (a9,a10)
// One top-down step: every node id in ids[] computes [X_a; X_b] = Q_node [X; 0]
// with X = xbuf[a] (n x n), storing X_a -> xbuf[a], X_b -> xbuf[b].
template <int NP>
__global__ void __launch_bounds__(kThreads)
k_formq_node(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_node,
             const int *ids, double *xbuf) {
    extern __shared__ __align__(16) double smem[];
    double *Y1 = smem, *Xa = Y1 + NP * (NP + 1), *Xb = Xa + NP * (NP + 1);
    double *red = smem + NodeSmem<NP>::red_off;
    double *taus = red + 2 * kWarps * NP;
    const int p = ids[blockIdx.x];
    const int a_t = plan.node_a[p];
    const int64_t nn = (int64_t)n * n;
    load_upper<NP, false>(Y1, A + plan.tile_row0[p], lda, n);
    load_block<NP, false>(Xa, xbuf + a_t * nn, n, n, n);
    for (int e = threadIdx.x; e < NP * (NP + 1); e += kThreads) Xb[e] = 0.0;
    for (int j = threadIdx.x; j < NP; j += kThreads) taus[j] = j < n ? tau_node[(int64_t)p * n + j] : 0.0;
    __syncthreads();
    node_apply<NP, false>(Y1, taus, Xa, Xb, n, red);
    store_block<NP>(Xa, xbuf + a_t * nn, n, n, n);
    store_block<NP>(Xb, xbuf + (int64_t)p * nn, n, n, n);
}

template <int NP, int RT, int KC>
__global__ void __launch_bounds__(kThreads, 1)
k_formq_leaf(const double *A, int64_t lda, int n, DevPlan plan, const double *tau_tile,
             const double *xbuf, double *Q, int64_t ldq) {
    using Cfg = ApplyCfg<NP, RT, KC>;
    using Ct = typename Cfg::Ct;
    constexpr int S = Cfg::S, YLD = Cfg::YLD, REDW = Cfg::REDW;
    extern __shared__ __align__(16) double smem[];
    double *Ys = smem;
    double *Cs = Ys + YLD * NP;
    double *red = smem + Cfg::base;
    double *taus = red + 2 * kWarps * REDW;

    const int t = blockIdx.x;
    const int64_t row0 = plan.tile_row0[t];
    const int rows = plan.tile_rows[t];
    load_y_tile<NP, S>(Ys, YLD, A + row0, lda, rows, n);
    for (int j = threadIdx.x; j < NP; j += kThreads) taus[j] = j < n ? tau_tile[(int64_t)t * n + j] : 0.0;
    const double *Xt = xbuf + (int64_t)t * n * n;
    for (int c0 = 0; c0 < n; c0 += KC) {
        const int kc = min(KC, n - c0);
        // [X_t; 0]: the first n rows from xbuf, zeros below
        stage_in_async(Cs, Ct::SLD, Xt + (int64_t)c0 * n, n, n, kc, S, KC);
        cp_async_wait_all();
        __syncthreads();
        double c[Ct::RT][Ct::CPL];
        smem_to_regs<Ct>(Cs, c);
        tile_apply<Ct, false>(c, n, Ys, YLD, taus, red);
        regs_to_smem<Ct>(Cs, c);
        __syncthreads();
        stage_out(Cs, Ct::SLD, Q + row0 + (int64_t)c0 * ldq, ldq, rows, kc);
        __syncthreads();
    }
}

__global__ void k_identity(double *X, int n) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x)
        X[e] = (e % n == e / n) ? 1.0 : 0.0;
}

// ================================================================ output / comm
template <int NP>
__global__ void k_write_r(const double *A, int64_t lda, int n, double *R, int64_t ldr) {
    write_r_block<NP>(A, lda, n, R, ldr);
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
template <int NP>
__global__ void __launch_bounds__(kThreads)
k_cross_factor(double *A, int64_t lda, int n, const double *partner_packed, int is_lower,
               double *Y1_out, double *tau_out, double *R, int64_t ldr) {
    extern __shared__ __align__(16) double smem[];
    double *Ra = smem, *Rb = Ra + NP * (NP + 1);
    double *red = smem + NodeSmem<NP>::red_off;
    double *taus = red + 2 * kWarps * NP;
    double *mine = is_lower ? Ra : Rb, *theirs = is_lower ? Rb : Ra;
    load_upper<NP, false>(mine, A, lda, n);
    for (int e = threadIdx.x; e < NP * NP; e += kThreads) {
        const int r = e % NP, c = e / NP;
        theirs[c * (NP + 1) + r] = (r <= c && c < n) ? partner_packed[(int64_t)c * (c + 1) / 2 + r] : 0.0;
    }
    __syncthreads();
    node_qr<NP>(Ra, Rb, n, red, taus);
    store_upper<NP>(Ra, A, lda, n);                   // the new current R (tile 0 head)
    for (int e = threadIdx.x; e < n * n; e += kThreads) {
        const int r = e % n, c = e / n;
        Y1_out[e] = (r <= c) ? Rb[c * (NP + 1) + r] : 0.0;
        if (R) R[r + (int64_t)c * ldr] = (r <= c) ? Ra[c * (NP + 1) + r] : 0.0;
    }
    for (int j = threadIdx.x; j < n; j += kThreads) tau_out[j] = taus[j];
}

// Butterfly round of apply Q^T on the R coordinates (n x k tops).
template <int NP>
__global__ void __launch_bounds__(kThreads)
k_cross_apply(const double *Y1g, const double *taug, double *top, int64_t ldtop,
              const double *partner_top, int is_lower, int head_role, double *C, int64_t ldc,
              int n, int k) {
    extern __shared__ __align__(16) double smem[];
    double *Y1 = smem, *Ca = Y1 + NP * (NP + 1), *Cb = Ca + NP * (NP + 1);
    double *red = smem + NodeSmem<NP>::red_off;
    double *taus = red + 2 * kWarps * NP;
    for (int e = threadIdx.x; e < NP * NP; e += kThreads) {
        const int r = e % NP, c = e / NP;
        Y1[c * (NP + 1) + r] = (r < n && c < n) ? Y1g[r + c * n] : 0.0;
    }
    for (int j = threadIdx.x; j < NP; j += kThreads) taus[j] = j < n ? taug[j] : 0.0;
    for (int c0 = 0; c0 < k; c0 += NP) {
        const int kc = min(NP, k - c0);
        double *mine = is_lower ? Ca : Cb, *theirs = is_lower ? Cb : Ca;
        load_block<NP, false>(mine, top + (int64_t)c0 * ldtop, ldtop, n, kc);
        load_block<NP, false>(theirs, partner_top + (int64_t)c0 * n, n, n, kc);
        __syncthreads();
        node_apply<NP, true>(Y1, taus, Ca, Cb, n, red);
        store_block<NP>(Ca, top + (int64_t)c0 * ldtop, ldtop, n, kc);
        if (head_role == 1) store_block<NP>(Ca, C + (int64_t)c0 * ldc, ldc, n, kc);
        if (head_role == 2) store_block<NP>(Cb, C + (int64_t)c0 * ldc, ldc, n, kc);
        __syncthreads();
    }
}

// Root X of this rank for form-Q: top-down over the butterfly nodes.
template <int NP>
__global__ void __launch_bounds__(kThreads)
k_cross_root_x(const double *Y1s, const double *taus_g, int rounds, int rank, int n, double *X0) {
    extern __shared__ __align__(16) double smem[];
    double *Y1 = smem, *Xa = Y1 + NP * (NP + 1), *Xb = Xa + NP * (NP + 1);
    double *red = smem + NodeSmem<NP>::red_off;
    double *taus = red + 2 * kWarps * NP;
    for (int e = threadIdx.x; e < NP * (NP + 1); e += kThreads) {
        const int r = e % (NP + 1), c = e / (NP + 1);
        Xa[e] = (r == c && r < n) ? 1.0 : 0.0;
    }
    for (int k = rounds; k >= 1; --k) {
        const double *Y1g = Y1s + (int64_t)(k - 1) * n * n;
        for (int e = threadIdx.x; e < NP * NP; e += kThreads) {
            const int r = e % NP, c = e / NP;
            Y1[c * (NP + 1) + r] = (r < n && c < n) ? Y1g[r + c * n] : 0.0;
            Xb[c * (NP + 1) + r] = 0.0;
        }
        for (int j = threadIdx.x; j < NP; j += kThreads) taus[j] = j < n ? taus_g[(k - 1) * n + j] : 0.0;
        __syncthreads();
        node_apply<NP, false>(Y1, taus, Xa, Xb, n, red);
        const bool lower = ((rank >> (k - 1)) & 1) == 0;
        if (!lower)
            for (int e = threadIdx.x; e < NP * (NP + 1); e += kThreads) Xa[e] = Xb[e];
        __syncthreads();
    }
    store_block<NP>(Xa, X0, n, n, n);
}

// ================================================================= launchers
static cudaError_t set_smem(const void *fn, size_t bytes) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int NP, int RT>
static size_t factor_smem() {
    return FactorSmem<NP, RT>::doubles * sizeof(double);
}

template <int NP, int RT>
static cudaError_t launch_factor_t(const FactorArgs &f, cudaStream_t st) {
    const size_t sm = factor_smem<NP, RT>();
    cudaError_t e = set_smem((const void *)k_factor<NP, RT>, sm);
    if (e != cudaSuccess) return e;
    k_factor<NP, RT><<<f.plan.L, kThreads, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile, f.tau_node,
                                                     f.counters, f.R, f.ldr);
    return cudaGetLastError();
}

template <int NP, int RT>
static size_t apply_smem() {
    constexpr int KC = ApplyKC<NP, RT>::value;
    return ApplyCfg<NP, RT, KC>::smem_doubles * sizeof(double);
}

template <int NP, int RT>
static cudaError_t launch_apply_t(const ApplyArgs &f, cudaStream_t st) {
    constexpr int KC = ApplyKC<NP, RT>::value;
    const size_t sm = apply_smem<NP, RT>();
    cudaError_t e;
    if (f.form_q) {
        e = set_smem((const void *)k_formq_leaf<NP, RT, KC>, sm);
        if (e != cudaSuccess) return e;
        k_formq_leaf<NP, RT, KC><<<f.plan.L, kThreads, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile,
                                                                 f.xbuf, f.C, f.ldc);
    } else {
        e = set_smem((const void *)k_apply_qt<NP, RT, KC>, sm);
        if (e != cudaSuccess) return e;
        k_apply_qt<NP, RT, KC><<<f.plan.L, kThreads, sm, st>>>(f.A, f.lda, f.n, f.plan, f.tau_tile,
                                                               f.tau_node, f.counters, f.C, f.ldc, f.k);
    }
    return cudaGetLastError();
}

template <int NP>
static size_t node_smem() {
    return NodeSmem<NP>::doubles * sizeof(double);
}

int tile_rt(int NP, int64_t max_rows) {
    // smallest of the two compiled capacities that holds the tallest tile
    const int64_t small = NP == 16 ? 512 : (NP == 32 ? 256 : 128);
    return max_rows <= small ? 0 : 1;
}

cudaError_t launch_factor(const FactorArgs &f, cudaStream_t st) {
    const int v = tile_rt(f.NP, f.max_rows);
    switch (f.NP) {
        case 16: return v ? launch_factor_t<16, 64>(f, st) : launch_factor_t<16, 32>(f, st);
        case 32: return v ? launch_factor_t<32, 64>(f, st) : launch_factor_t<32, 32>(f, st);
        default: return v ? launch_factor_t<64, 32>(f, st) : launch_factor_t<64, 16>(f, st);
    }
}

cudaError_t launch_apply(const ApplyArgs &f, cudaStream_t st) {
    const int v = tile_rt(f.NP, f.max_rows);
    switch (f.NP) {
        case 16: return v ? launch_apply_t<16, 64>(f, st) : launch_apply_t<16, 32>(f, st);
        case 32: return v ? launch_apply_t<32, 64>(f, st) : launch_apply_t<32, 32>(f, st);
        default: return v ? launch_apply_t<64, 32>(f, st) : launch_apply_t<64, 16>(f, st);
    }
}

template <int NP>
static cudaError_t launch_formq_nodes_t(const double *A, int64_t lda, int n, const DevPlan &plan,
                                        const double *tau_node, const int *ids, int count,
                                        double *xbuf, cudaStream_t st) {
    const size_t sm = node_smem<NP>();
    cudaError_t e = set_smem((const void *)k_formq_node<NP>, sm);
    if (e != cudaSuccess) return e;
    k_formq_node<NP><<<count, kThreads, sm, st>>>(A, lda, n, plan, tau_node, ids, xbuf);
    return cudaGetLastError();
}

cudaError_t launch_formq_nodes(int NP, const double *A, int64_t lda, int n, const DevPlan &plan,
                               const double *tau_node, const int *ids, int count, double *xbuf,
                               cudaStream_t st) {
    switch (NP) {
        case 16: return launch_formq_nodes_t<16>(A, lda, n, plan, tau_node, ids, count, xbuf, st);
        case 32: return launch_formq_nodes_t<32>(A, lda, n, plan, tau_node, ids, count, xbuf, st);
        default: return launch_formq_nodes_t<64>(A, lda, n, plan, tau_node, ids, count, xbuf, st);
    }
}

cudaError_t launch_identity(double *X, int n, cudaStream_t st) {
    k_identity<<<(n * n + 255) / 256, 256, 0, st>>>(X, n);
    return cudaGetLastError();
}

cudaError_t launch_write_r(int NP, const double *A, int64_t lda, int n, double *R, int64_t ldr,
                           cudaStream_t st) {
    switch (NP) {
        case 16: k_write_r<16><<<1, kThreads, 0, st>>>(A, lda, n, R, ldr); break;
        case 32: k_write_r<32><<<1, kThreads, 0, st>>>(A, lda, n, R, ldr); break;
        default: k_write_r<64><<<1, kThreads, 0, st>>>(A, lda, n, R, ldr); break;
    }
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

template <int NP>
static cudaError_t launch_cross_factor_t(double *A, int64_t lda, int n, const double *pp, int is_lower,
                                         double *Y1, double *tau, double *R, int64_t ldr, cudaStream_t st) {
    const size_t sm = node_smem<NP>();
    cudaError_t e = set_smem((const void *)k_cross_factor<NP>, sm);
    if (e != cudaSuccess) return e;
    k_cross_factor<NP><<<1, kThreads, sm, st>>>(A, lda, n, pp, is_lower, Y1, tau, R, ldr);
    return cudaGetLastError();
}

cudaError_t launch_cross_factor(int NP, double *A, int64_t lda, int n, const double *pp, int is_lower,
                                double *Y1, double *tau, double *R, int64_t ldr, cudaStream_t st) {
    switch (NP) {
        case 16: return launch_cross_factor_t<16>(A, lda, n, pp, is_lower, Y1, tau, R, ldr, st);
        case 32: return launch_cross_factor_t<32>(A, lda, n, pp, is_lower, Y1, tau, R, ldr, st);
        default: return launch_cross_factor_t<64>(A, lda, n, pp, is_lower, Y1, tau, R, ldr, st);
    }
}

template <int NP>
static cudaError_t launch_cross_apply_t(const double *Y1, const double *tau, double *top, int64_t ldtop,
                                        const double *ptop, int is_lower, int role, double *C, int64_t ldc,
                                        int n, int k, cudaStream_t st) {
    const size_t sm = node_smem<NP>();
    cudaError_t e = set_smem((const void *)k_cross_apply<NP>, sm);
    if (e != cudaSuccess) return e;
    k_cross_apply<NP><<<1, kThreads, sm, st>>>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k);
    return cudaGetLastError();
}

cudaError_t launch_cross_apply(int NP, const double *Y1, const double *tau, double *top, int64_t ldtop,
                               const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n,
                               int k, cudaStream_t st) {
    switch (NP) {
        case 16: return launch_cross_apply_t<16>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, st);
        case 32: return launch_cross_apply_t<32>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, st);
        default: return launch_cross_apply_t<64>(Y1, tau, top, ldtop, ptop, is_lower, role, C, ldc, n, k, st);
    }
}

template <int NP>
static cudaError_t launch_cross_root_x_t(const double *Y1s, const double *taus, int rounds, int rank, int n,
                                         double *X0, cudaStream_t st) {
    const size_t sm = node_smem<NP>();
    cudaError_t e = set_smem((const void *)k_cross_root_x<NP>, sm);
    if (e != cudaSuccess) return e;
    k_cross_root_x<NP><<<1, kThreads, sm, st>>>(Y1s, taus, rounds, rank, n, X0);
    return cudaGetLastError();
}

cudaError_t launch_cross_root_x(int NP, const double *Y1s, const double *taus, int rounds, int rank, int n,
                                double *X0, cudaStream_t st) {
    switch (NP) {
        case 16: return launch_cross_root_x_t<16>(Y1s, taus, rounds, rank, n, X0, st);
        case 32: return launch_cross_root_x_t<32>(Y1s, taus, rounds, rank, n, X0, st);
        default: return launch_cross_root_x_t<64>(Y1s, taus, rounds, rank, n, X0, st);
    }
}

}  // namespace tsqr
