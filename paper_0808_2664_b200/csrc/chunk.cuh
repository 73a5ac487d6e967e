// Register-resident chunk engine of the B200 TSQR leaf path (sm_100a).  Product code.
//
// A tile (the leaf of the binary tree) is factored as a
// flat chain ("sequential TSQR", flat tree P:954-993, [TR] Alg. P:1725-1753)
// over chunks of CH = 8 KM consecutive rows: for the chunk at tile row r0,
//     [R; A_k]  <-  Householder QR, column by column j = 0 .. n-1:
//   * j <  r0:            "structured" -- the pivot is row j of the running R
//                         (upper trapezoidal, min(r0, n) rows) and the tail is
//                         the whole chunk (Alg. QR:qnxn with a dense lower block);
//   * r0 <= j < r0 + CH:  "dense" -- the pivot is chunk row j - r0, the tail the
//                         chunk rows below it (ordinary Householder, DGEQR2);
//   * j >= r0 + CH:       the chunk lies above the pivot: nothing.
// One warp holds one chunk in registers as DMMA fragments (transposed
// accumulator layout): lane (q = lane & 3, l4 = lane >> 2) holds
//     a[k][cb][e] = A(chunk row 8k + 2q + e, column 8cb + l4).
// Columns are processed in panels of 8 (p = 0 .. NCB-1): the panel's Householder
// steps use warp shuffles only (x broadcast, 4-lane reductions); the panel's
// T (compact WY, Alg. YT:scaled P:2007-2028, LAPACK sign R3) comes from the
// Gram entries the steps compute anyway; the trailing update
//     W^T = C^T Y (+ R pivot rows),  W'^T = W^T T,  C^T -= W'^T Y^T
// runs on FP64 DMMA with the chunk registers as operands and accumulators.
// The running R lives in shared memory (row-major, ld LDR); row block p of R is
// the hand-off between consecutive chunks (a counter per row block).
#pragma once
#include <cstdint>
#include "wy.cuh"

#ifdef TSQR_PROBE
// Probe build only (tools/probe_chain.cu): lane 0 of each warp of CTA 0 logs
// (clock64 << 8 | event) into a per-warp shared-memory log, flushed to global
// memory at the end of the kernel.
__device__ unsigned long long *g_probe_buf;   // [warps][PROBE_N]
constexpr int PROBE_N = 512, PROBE_W = 8;
__device__ __forceinline__ unsigned long long *probe_log() {
    __shared__ unsigned long long log[PROBE_W][PROBE_N];
    return &log[0][0];
}
__device__ __forceinline__ void probe_mark(int id) {
    if ((threadIdx.x & 31) == 0) {
        unsigned long long *b = probe_log() + (threadIdx.x >> 5) * PROBE_N;
        const int i = (int)b[0] + 1;
        if (i < PROBE_N) {
            b[i] = ((unsigned long long)clock64() << 8) | (unsigned)id;
            b[0] = i;
        }
    }
}
__device__ __forceinline__ void probe_init() {
    if ((threadIdx.x & 31) == 0) probe_log()[(threadIdx.x >> 5) * PROBE_N] = 0;
}
__device__ __forceinline__ void probe_flush() {
    __syncthreads();
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < PROBE_W * PROBE_N; i += blockDim.x) g_probe_buf[i] = probe_log()[i];
}
#define PROBE(id) probe_mark(id)
#define PROBE_INIT() probe_init()
#define PROBE_FLUSH() probe_flush()
#else
#define PROBE(id)
#define PROBE_INIT()
#define PROBE_FLUSH()
#endif

namespace tsqr {
namespace chunk {

using wy::dmma;
using wy::House;
using wy::householder;

constexpr unsigned FULL = 0xffffffffu;

// Hand-off between consecutive chunks of one R buffer (a software pipeline
// over the warps of a CTA).  Every chunk of the buffer's sequence has a number
// s; counters hold "chunks done":
//   row[j] -- chunks that have finished Householder step j (R row j's panel
//             entries are final for them),
//   tr[p]  -- chunks that have finished panel p's update of R rows 8p..8p+7.
// Chunk s waits for row[j] >= s before step j and for tr[p] >= s before it
// touches R's trailing columns, and publishes s + 1 after each.  One writer at
// a time per counter, so every counter is monotonic.
struct Sync {
    int *row, *tr;
    int s;
};
// Hand-off ordering.  The publisher's lanes store the data, __syncwarp() orders
// those stores before lane 0's counter store; the waiter reads the counter and
// then the data.  Default build: the counter is a volatile access and the only
// fences are compiler barriers -- it relies on one warp's shared-memory
// accesses being performed in issue order by the SM's memory pipeline (the
// publisher's data stores reach shared memory before its counter store, and the
// waiter's data load issued after its counter load sees at least what the
// counter promised).  The PTX memory model does not promise that: a conforming
// build (-DTSQR_HANDOFF_ACQREL) makes the counter store a RELEASE and its load an
// ACQUIRE (release/acquire synchronisation at cta scope; __syncwarp gives the
// cumulativity over the publisher's lanes).  On sm_100a the release compiles to
// MEMBAR.ALL.CTA, which waits for the warp's outstanding global stores, and costs
// 6-16 % of the leaf kernel (C4 +16 % on the final code, profiles/r02j_house3_acqrel_ab.txt), so it is a variant; the
// jitter build (-DTSQR_HANDOFF_JITTER) injects pseudo-random __nanosleep delays
// between the data and the counter on both sides and is checked bitwise against
// the default build and against the oracle (tests/test_gpu_handoff.py).
#if defined(TSQR_HANDOFF_JITTER)
__device__ __forceinline__ void handoff_jitter() {
    unsigned t;
    asm volatile("mov.u32 %0, %%clock;" : "=r"(t));
    t = (t ^ (threadIdx.x * 2654435761u)) * 2246822519u;
    if (((t >> 13) & 7) == 0) __nanosleep(32 + ((t >> 17) & 511));
}
#else
__device__ __forceinline__ void handoff_jitter() {}
#endif
__device__ __forceinline__ int ld_acquire_cta(const int *c) {
#ifndef TSQR_HANDOFF_ACQREL
    const int v = *reinterpret_cast<const volatile int *>(c);
    asm volatile("" ::: "memory");
    handoff_jitter();
    return v;
#else
    int v;
    const unsigned a = (unsigned)__cvta_generic_to_shared(c);
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
#endif
}
__device__ __forceinline__ void st_release_cta(int *c, int v) {
#ifndef TSQR_HANDOFF_ACQREL
    asm volatile("" ::: "memory");
    handoff_jitter();
    *reinterpret_cast<volatile int *>(c) = v;
#else
    const unsigned a = (unsigned)__cvta_generic_to_shared(c);
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
#endif
}
__device__ __forceinline__ void sync_wait(const int *c, int v) {
    while (ld_acquire_cta(c) < v) {
    }
}
__device__ __forceinline__ void sync_publish(int *c, int v) {
    asm volatile("" ::: "memory");
    __syncwarp();
    if ((threadIdx.x & 31) == 0) st_release_cta(c, v);
}

// dlarfg scalars (readings R1/R2/R19), branch-free: beta = -sign(alpha) N with
// N = sqrt(alpha^2 + sigma2), tau = 1 + |alpha|/N, scale = 1/(alpha - beta);
// sigma2 == 0 gives H = I (tau = 0, beta = alpha).  1/sqrt(y) and 1/(|alpha| + N)
// from the MUFU seeds, each refined by one third-order correction (seed errors
// ~2^-22 -> O(2^-66) + rounding); the reciprocal is seeded from |alpha| + y r0
// so its MUFU runs while the root is refined.  (-DTSQR_HOUSE_NEWTON2: two Newton
// steps per seed, one dependent step longer: C4 leaf +0.5 %,
// profiles/r02j_house3_acqrel_ab.txt.)
// The plain sums and the flush-to-zero seeds need the input range of reading
// R23; the robust instantiation (kRobust) rescales outside it.
__device__ __forceinline__ House house_bf(double alpha, double s2) {
    const double y = fma(alpha, alpha, s2);
    const double aa = fabs(alpha);
    double r0, i0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(y));
    const double D0 = fma(y, r0, aa);
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(i0) : "d"(D0));
#ifdef TSQR_HOUSE_NEWTON2
    const double hy = 0.5 * y;
    double r = r0 * fma(-hy * r0, r0, 1.5);
    const double D1 = fma(y, r, aa);
    double i = fma(i0, fma(-D1, i0, 1.0), i0);
    r = r * fma(-hy * r, r, 1.5);
    const double N = y * r;
    const double D = aa + N;
    i = fma(i, fma(-D, i, 1.0), i);
#else
    // one third-order correction per seed: r = r0 (1 + e/2 + 3e^2/8), e = 1 - y r0^2;
    // i = i0 (1 + e' + e'^2), e' = 1 - D i0 (seed errors ~2^-20 -> O(2^-60))
    const double e = fma(-(y * r0), r0, 1.0);
    const double r = fma(r0 * e, fma(0.375, e, 0.5), r0);
    const double N = y * r;
    const double D = aa + N;
    const double ei = fma(-D, i0, 1.0);
    const double i = fma(i0 * ei, 1.0 + ei, i0);
#endif
    const bool z = (s2 == 0.0);
    House h;
    h.beta = z ? alpha : (alpha >= 0.0 ? -N : N);
    h.tau = z ? 0.0 : fma(aa, r, 1.0);
    h.scale = z ? 0.0 : (alpha >= 0.0 ? i : -i);
    return h;
}

// 16 < n <= 32 (variants: -DTSQR_KM32=<row blocks> -DTSQR_NW32=<warps>, plan.cpp TSQR_C32 = 8 KM)
#ifndef TSQR_KM32
#define TSQR_KM32 8
#endif
#ifndef TSQR_NW32
#define TSQR_NW32 8
#endif
#define TSQR_CFG32 4, TSQR_KM32, TSQR_NW32
template <int NCB_, int KM_, int NW_, int NBUF_ = 2>
struct Cfg {
    // NBUF: R buffers; with 2 the tiles of a CTA alternate and the next tile's head
    // chunk never waits for the previous tile; with 1 (to make room for taller
    // chunks) it follows the previous tile's last chunk panel by panel
    static constexpr int NCB = NCB_, KM = KM_, NW = NW_, NBUF = NBUF_;
    static constexpr int NP = 8 * NCB, CH = 8 * KM, NT = 32 * NW;
    static constexpr int LDR = NP + 2;                    // R buffer: R(i, c) at [i * LDR + c]
    static constexpr int RBUF = NP * LDR;
    // per-warp scratch: Y panel (CH x 8 row-major), Gram, T (row-major), taus
    static constexpr int YS = 0, GS = CH * 8, TS = GS + 64, T8 = TS + 64, XS = T8 + 8, WS = XS + 2 * CH;
    static constexpr int OFF_WS = NBUF * RBUF;            // after the R buffers
    static constexpr int OFF_SYNC = OFF_WS + NW * WS;     // per buffer: NP row + NCB panel counters
    static constexpr int SYNC_INTS = NP + NCB;
    // after the counters: one range-gate flag per buffer (NBUF ints)
    // per warp: the next chunk (col-major CH x NP), 128-byte aligned (TMA destination)
    static constexpr int OFF_STG = (OFF_SYNC + (NBUF * (SYNC_INTS + 1) + 1) / 2 + 15) & ~15;
    static constexpr int STG = CH * NP;
    static_assert((STG * 8) % 128 == 0, "TMA staging slots must stay 128-byte aligned");
    static constexpr int OFF_BAR = OFF_STG + NW * STG;    // one mbarrier per warp (TMA completion)
    static constexpr size_t BYTES = (size_t)(OFF_BAR + NW) * sizeof(double);
    static_assert(BYTES <= 232448, "exceeds 227 KB of shared memory per CTA");
};

// T (8x8, row-major) of one panel from its Gram entries G(l, c), l < c
// (row-major in Gs) and taus t: T(r,r) = t_r, T(r,c) = -t_c sum_l T(r,l) G(l,c).
__device__ __forceinline__ void build_t(const double *Gs, const double *t, double *Ts) {
    // straight-line for every lane (row lane & 7), so the compiler can overlap
    // it with the independent W^T DMMAs that follow; lanes 0..7 store
    const int r = threadIdx.x & 7;
    double row[8];
    const double tr = t[r];
#pragma unroll
    for (int c = 0; c < 8; ++c) row[c] = (c == r) ? tr : 0.0;
#pragma unroll
    for (int c = 1; c < 8; ++c) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < c; ++l) s = fma(row[l], Gs[l * 8 + c], s);
        row[c] = (r < c) ? -t[c] * s : row[c];
    }
    if ((threadIdx.x & 31) < 8) {
#pragma unroll
        for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2 *>(Ts + r * 8 + c) = make_double2(row[c], row[c + 1]);
    }
    __syncwarp();
}

// Sums of a value over the 4 lanes q of each column l4 (lane = 4 l4 + q), on
// the tensor pipe instead of two shuffle rounds: D = A 1 with A[l4][q] the
// lane's partial (one m8n8k4 DMMA per sum, both issued back to back); every
// lane of column l4 receives its column's sum.
__device__ __forceinline__ void quad_sums(double &d, double &s2, double pd, double ps) {
    double d1 = 0.0, s1 = 0.0;
    d = 0.0;
    s2 = 0.0;
    dmma(d, d1, pd, 1.0);
    dmma(s2, s1, ps, 1.0);
}

// Rescaled step (reading R23, wy::house_unsafe): the sums of a Householder step
// redone on s x for the register layouts in which every lane of a q group holds
// the same rows of the pivot column's tail (x[k][e] = row 8k + 2q + e) and
// a(k, e) is this lane's column l4 on those rows.  Every input is warp-uniform
// except a, so d (column l4's dot) and s2 are what the unscaled sums would be
// for s x; sc = s.  Taken only when y = alpha^2 + sigma^2 left [2^-900, 2^900].
template <int K, class AF>
__device__ __forceinline__ void rescaled_sums(const double (&x)[K][2], AF a, double alpha, double &d, double &s2,
                                              double &sc) {
    double mx = fabs(alpha);
#pragma unroll
    for (int k = 0; k < K; ++k) mx = fmax(mx, fmax(fabs(x[k][0]), fabs(x[k][1])));
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, 2));
    sc = wy::pow2_scale(mx);
    double d0 = 0.0, d1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double x0 = sc * x[k][0], x1 = sc * x[k][1];
        d0 = fma(x0, a(k, 0), d0);
        d1 = fma(x1, a(k, 1), d1);
        s0 = fma(x0, x0, s0);
        s1 = fma(x1, x1, s1);
    }
    d0 += d1;
    s0 += s1;
    d0 += __shfl_xor_sync(FULL, d0, 1);
    s0 += __shfl_xor_sync(FULL, s0, 1);
    d0 += __shfl_xor_sync(FULL, d0, 2);
    s0 += __shfl_xor_sync(FULL, s0, 2);
    d = d0;
    s2 = s0;
}

// Columns past n are padding: their Householder steps would be identities
// (tau = 0, zero reflector), so the panels stop after column n-1 and give the
// remaining columns tau = 0 and zero Gram entries, which makes their rows and
// columns of T zero exactly as the skipped steps would have.
__device__ __forceinline__ void pad_steps(double *Gs, double *t8, int jn) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    for (int c = jn; c < 8; ++c) {
        if (q == 0 && l4 < c) Gs[l4 * 8 + c] = 0.0;
        if (lane == 0) t8[c] = 0.0;
    }
}

template <class C>
struct Chunk {
    double a[C::KM][C::NCB][2];
};

// --------------------------------------------------------------- panel steps
// Structured panel P: pivots are R rows 8P .. 8P+7 (smem, Rb), the tail is the
// whole chunk.  On exit the panel registers hold v (the reflectors' chunk part,
// scale applied), R's pivot rows hold (beta, updated R entries) in the panel
// columns, Gs/t8 the Gram entries and taus.
template <class C, int P, bool kRobust>
__device__ __forceinline__ void panel_structured(Chunk<C> &ch, double *Rb, double *Gs, double *t8, double *xs,
                                                 double *tau_out, int n, const Sync &sy) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    // the pivot column is broadcast through a double-buffered row in smem: its
    // owners (l4 == jj) store it right after their update of the previous step
    if (l4 == 0) {
#pragma unroll
        for (int k = 0; k < C::KM; ++k)
            *reinterpret_cast<double2 *>(xs + 8 * k + 2 * q) = make_double2(ch.a[k][P][0], ch.a[k][P][1]);
    }
    __syncwarp();
    const int jn = (P + 1 < C::NCB) ? 8 : n - 8 * P;      // only the last panel has padding columns
    // A finished pivot column keeps x; its reflector v = scl x is formed once after
    // the panel (scl: this lane's column's scale), so each step updates with one
    // FMA per value: the pivot and finished columns get u = 0.
    double scl = 1.0;
#pragma unroll 1                  // unrolled, the kernel's code grows 1.5x and runs 27 % slower (C4)
    for (int jj = 0; jj < jn; ++jj) {
        const int j = 8 * P + jj;
        // Where R row j (released by the previous chunk) is read, measured per configuration:
        // for 56 < n <= 64 (one R buffer, 40-row chunks) counter and entries are read -- and
        // waited for -- at the top of the step, so their latency overlaps the dots (C4 leaf
        // 15.83 -> 15.27 ms); for the other configurations after the dots, where an early
        // wait costs more than it hides (C2 0.818 -> 0.836 ms, C5 10.47 -> 10.71 ms).
        constexpr bool kEarlyR = C::NCB == 8;
        const volatile double *rr = Rb + j * C::LDR;
        int c0 = 0;
        double alpha = 0.0, rj = 0.0;
        if constexpr (kEarlyR) {
            c0 = ld_acquire_cta(sy.row + j);
            alpha = rr[j];                                           // R(j, j)
            rj = rr[8 * P + l4];                                     // R(j, 8P + l4)
            if (c0 < sy.s) {
                sync_wait(sy.row + j, sy.s);
                alpha = rr[j];
                rj = rr[8 * P + l4];
            }
        }
        const double *xr = xs + (jj & 1) * C::CH;
        double x[C::KM][2];
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            const double2 v = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
            x[k][0] = v.x;
            x[k][1] = v.y;
        }
        // sigma^2 = the pivot column's own dot x^T x (its lanes hold x), read from
        // lane 4 jj: no separate sum of squares (half the step's FMAs)
        double dk[2][2] = {{0.0, 0.0}, {0.0, 0.0}};                 // four partial dots: shorter chains
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            dk[k & 1][0] = fma(x[k][0], ch.a[k][P][0], dk[k & 1][0]);
            dk[k & 1][1] = fma(x[k][1], ch.a[k][P][1], dk[k & 1][1]);
        }
        double d, s2, dz = 0.0;
        d = 0.0;
        dmma(d, dz, (dk[0][0] + dk[1][0]) + (dk[0][1] + dk[1][1]), 1.0);
        s2 = __shfl_sync(FULL, d, 4 * jj);
        PROBE(3);
        if constexpr (!kEarlyR) {
            // the counter and the row read together, the row again only if the counter was
            // short ("Hand-off ordering" above)
            c0 = ld_acquire_cta(sy.row + j);
            alpha = rr[j];
            rj = rr[8 * P + l4];
            if (c0 < sy.s) {
                sync_wait(sy.row + j, sy.s);
                alpha = rr[j];
                rj = rr[8 * P + l4];
            }
        }
        PROBE(4);
        House h = house_bf(alpha, s2);
        double sc = 1.0;
        double sx = h.scale;                                        // the scale of the unscaled x
        if (kRobust && __any_sync(FULL, wy::house_unsafe(alpha, s2))) {   // warp-uniform, R23
            rescaled_sums<C::KM>(x, [&](int k, int e) { return ch.a[k][P][e]; }, alpha, d, s2, sc);
            h = house_bf(sc * alpha, s2);
            h.beta = h.beta / sc;
            sx = h.scale * sc;
        }
        const double w = fma(h.scale, d, rj);                        // v^T [R(j,c); a_c]
        // a <- a - u x (u = tau scale w) for the trailing columns only
        const double u = (l4 > jj) ? h.tau * sx * w : 0.0;
        if (l4 == jj) scl = sx;
        // hand R row j to the next chunk first (its step j waits for it), then
        // update this chunk's panel
        const double rnew = (l4 == jj) ? h.beta : fma(-h.tau, w, rj);
        __syncwarp();                  // every lane has read R(j, .) before it is overwritten
        if (q == 0 && l4 >= jj) Rb[j * C::LDR + 8 * P + l4] = rnew;
        sync_publish(sy.row + j, sy.s + 1);
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            ch.a[k][P][0] = fma(-u, x[k][0], ch.a[k][P][0]);
            ch.a[k][P][1] = fma(-u, x[k][1], ch.a[k][P][1]);
        }
        if (l4 == jj + 1) {                                          // next pivot column -> the other row
            double *xw = xs + ((jj + 1) & 1) * C::CH;
#pragma unroll
            for (int k = 0; k < C::KM; ++k)
                *reinterpret_cast<double2 *>(xw + 8 * k + 2 * q) = make_double2(ch.a[k][P][0], ch.a[k][P][1]);
        }
        if (q == 0 && l4 < jj) Gs[l4 * 8 + jj] = scl * (h.scale * d);   // G(l, jj) = v_l^T v_jj, v_l = scl x_l
        if (lane == 0) t8[jj] = h.tau;
        __syncwarp();                                                // xs of the next step
        PROBE(2);
    }
#pragma unroll
    for (int k = 0; k < C::KM; ++k) {                                // v = scl x (exactly the former scale x + 0)
        ch.a[k][P][0] *= scl;
        ch.a[k][P][1] *= scl;
    }
    pad_steps(Gs, t8, jn);
    __syncwarp();
    if (lane < 8 && 8 * P + lane < n) tau_out[8 * P + lane] = t8[lane];
}

// Dense panel P: the pivots are chunk rows 8 kb .. 8 kb + 7 (kb = (8P - r0)/8).
// On exit the panel column holds R above/at the pivot (beta on the diagonal)
// and v below it, as DGEQR2 stores them.
template <class C, int P, bool kRobust>
__device__ __forceinline__ void panel_dense(Chunk<C> &ch, int kb, double *Gs, double *t8, double *tau_out, int n) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int jn = (P + 1 < C::NCB) ? 8 : n - 8 * P;      // only the last panel has padding columns
#pragma unroll 1
    for (int jj = 0; jj < jn; ++jj) {
        const int j = 8 * P + jj;
        const int qp = jj >> 1, ep = jj & 1;
        const int src = 4 * jj + q;
        double x[C::KM][2];
        double sel = 0.0;
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            x[k][0] = __shfl_sync(FULL, ch.a[k][P][0], src);
            x[k][1] = __shfl_sync(FULL, ch.a[k][P][1], src);
            const bool below0 = (k > kb) || (k == kb && 2 * q > jj);
            const bool below1 = (k > kb) || (k == kb && 2 * q + 1 > jj);
            x[k][0] = below0 ? x[k][0] : 0.0;
            x[k][1] = below1 ? x[k][1] : 0.0;
            if (k == kb) sel = ep ? ch.a[k][P][1] : ch.a[k][P][0];
        }
        const double rj = __shfl_sync(FULL, sel, 4 * l4 + qp);       // A(pivot row, 8P + l4)
        const double alpha = __shfl_sync(FULL, rj, 4 * jj);
        double d0 = 0.0, d1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            d0 = fma(x[k][0], ch.a[k][P][0], d0);
            d1 = fma(x[k][1], ch.a[k][P][1], d1);
            s0 = fma(x[k][0], x[k][0], s0);
            s1 = fma(x[k][1], x[k][1], s1);
        }
        double d, s2;
        quad_sums(d, s2, d0 + d1, s0 + s1);
        House h = house_bf(alpha, s2);
        double sc = 1.0;
        double sx = h.scale;                                        // the scale of the unscaled x
        if (kRobust && __any_sync(FULL, wy::house_unsafe(alpha, s2))) {   // warp-uniform, R23
            rescaled_sums<C::KM>(x, [&](int k, int e) { return ch.a[k][P][e]; }, alpha, d, s2, sc);
            h = house_bf(sc * alpha, s2);
            h.beta = h.beta / sc;
            sx = h.scale * sc;
        }
        const double w = fma(h.scale, d, rj);
        const double u = (l4 > jj) ? h.tau * sx * w : (l4 == jj ? 1.0 : 0.0);
        const double g = (l4 == jj) ? sx : 0.0;                      // pivot column: v = scale x exactly
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            ch.a[k][P][0] = fma(g, x[k][0], fma(-u, x[k][0], ch.a[k][P][0]));
            ch.a[k][P][1] = fma(g, x[k][1], fma(-u, x[k][1], ch.a[k][P][1]));
        }
        const double pnew = (l4 > jj) ? fma(-h.tau, w, rj) : (l4 == jj ? h.beta : rj);
        if (q == qp) {
#pragma unroll
            for (int k = 0; k < C::KM; ++k)
                if (k == kb) {
                    if (ep) ch.a[k][P][1] = pnew;
                    else ch.a[k][P][0] = pnew;
                }
        }
        if (q == 0 && l4 < jj) Gs[l4 * 8 + jj] = fma(h.scale, d, rj);    // G(l, jj) = y_l^T y_jj
        if (lane == 0) t8[jj] = h.tau;
    }
    pad_steps(Gs, t8, jn);
    __syncwarp();
    if (lane < 8 && 8 * P + lane < n) tau_out[8 * P + lane] = t8[lane];
}

// ------------------------------------------------------------ trailing update
// C <- (I - Y T^T Y^T) C for the chunk's column blocks cb > P (kStruct: with the
// R pivot rows 8P..8P+7 of Rb as the identity part of Y).  yv: the panel's Y
// (B operand of W^T = C^T Y); Ys: the same Y in smem (row-major, CH x 8).
// Order: W^T for every block (chunk registers only), then -- after the
// previous chunk has released R's rows -- the R part, W'^T = W^T T and R's
// update, publish, and only then the chunk's own update.
template <class C, int P, bool kStruct>
__device__ __forceinline__ void trailing(Chunk<C> &ch, const double (&yv)[C::KM][2], const double *Ys,
                                         const double *Gs, const double *t8, double *Ts, double *tg, double *Rb,
                                         const Sync &sy, bool defer) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    if constexpr (P + 1 < C::NCB) {
        double wt[C::NCB][2];
        // few trailing blocks (<= TSQR_WT_SPLIT, default 3): two accumulation chains per block,
        // which halves the dependent DMMA chain where it is not hidden by other blocks'
        // chains (C4 leaf 15.86 -> 15.69-15.76 ms; 0 disables)
#ifndef TSQR_WT_SPLIT
#define TSQR_WT_SPLIT 3
#endif
        constexpr bool kSplit = (C::NCB - 1 - P) <= TSQR_WT_SPLIT;
#pragma unroll
        for (int cb = P + 1; cb < C::NCB; ++cb) {
            wt[cb][0] = wt[cb][1] = 0.0;
            if constexpr (kSplit) {
                double u0 = 0.0, u1 = 0.0;
#pragma unroll
                for (int k = 0; k < C::KM; ++k) {
                    dmma(wt[cb][0], wt[cb][1], ch.a[k][cb][0], yv[k][0]);
                    dmma(u0, u1, ch.a[k][cb][1], yv[k][1]);
                }
                wt[cb][0] += u0;
                wt[cb][1] += u1;
            } else {
#pragma unroll
                for (int k = 0; k < C::KM; ++k) {
                    dmma(wt[cb][0], wt[cb][1], ch.a[k][cb][0], yv[k][0]);
                    dmma(wt[cb][0], wt[cb][1], ch.a[k][cb][1], yv[k][1]);
                }
            }
        }
        // T while the W^T DMMAs drain (it only needs the panel's Gram and taus; built before
        // them, or one column per step inside the steps, it measured slower)
        build_t(Gs, t8, Ts);
        if (tg != nullptr)
            *reinterpret_cast<double2 *>(tg + 8 * P * 8 + 2 * lane) = *reinterpret_cast<const double2 *>(Ts + 2 * lane);
        const double tb0 = Ts[(2 * q) * 8 + l4], tb1 = Ts[(2 * q + 1) * 8 + l4];
        PROBE(6);
        if (kStruct) sync_wait(sy.tr + P, sy.s);
        PROBE(9);
#pragma unroll
        for (int cb = P + 1; cb < C::NCB; ++cb) {
            double *r0p = Rb + (8 * P + 2 * q) * C::LDR + 8 * cb + l4;
            if (kStruct) {
                wt[cb][0] += r0p[0];
                wt[cb][1] += r0p[C::LDR];
            }
            double wp0 = 0.0, wp1 = 0.0;
            dmma(wp0, wp1, wt[cb][0], tb0);
            dmma(wp0, wp1, wt[cb][1], tb1);
            if (kStruct) {
                r0p[0] -= wp0;
                r0p[C::LDR] -= wp1;
            }
            wt[cb][0] = -wp0;
            wt[cb][1] = -wp1;
        }
        if (kStruct && !defer) sync_publish(sy.tr + P, sy.s + 1);
        PROBE(7);
        double yt[C::KM][2];
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            const double2 v = *reinterpret_cast<const double2 *>(Ys + (8 * k + l4) * 8 + 2 * q);
            yt[k][0] = v.x;
            yt[k][1] = v.y;
        }
#pragma unroll
        for (int cb = P + 1; cb < C::NCB; ++cb)
#pragma unroll
            for (int k = 0; k < C::KM; ++k) {
                dmma(ch.a[k][cb][0], ch.a[k][cb][1], wt[cb][0], yt[k][0]);
                dmma(ch.a[k][cb][0], ch.a[k][cb][1], wt[cb][1], yt[k][1]);
            }
    } else {
        build_t(Gs, t8, Ts);
        if (tg != nullptr)
            *reinterpret_cast<double2 *>(tg + 8 * P * 8 + 2 * lane) = *reinterpret_cast<const double2 *>(Ts + 2 * lane);
        if (kStruct) {
            sync_wait(sy.tr + P, sy.s);
            if (!defer) sync_publish(sy.tr + P, sy.s + 1);
        }
    }
}

// Panel P of the factorisation of one chunk (kind 0 structured, 1 dense, 2 none).
template <class C, int P, bool kRobust>
__device__ __forceinline__ void factor_panel(Chunk<C> &ch, int kind, int kb, double *Rb, double *ws,
                                             double *tau_out, int n, const Sync &sy, bool defer, double *tg,
                                             double *ydst = nullptr, int64_t ldy = 0) {
    // defer: the caller publishes tr[P] itself (after copying R rows out);
    // tg: this chunk's T cache (NCB x 8 x 8, row-major per panel) or null;
    // ydst: a full structured chunk whose rows and columns are all reflector entries, with
    // 16-byte aligned row pairs: the panel's reflectors are stored as soon as its steps end
    // (spread over the chunk instead of one burst after its last panel), or null
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    double *Ys = ws + C::YS, *Gs = ws + C::GS, *Ts = ws + C::TS, *t8 = ws + C::T8;
    if (kind != 0) {                  // the previous chunk must be done with R rows 8P..8P+7
        sync_wait(sy.tr + P, sy.s);
        if (kind == 2) {
            if (lane < 8 && 8 * P + lane < n) tau_out[8 * P + lane] = 0.0;
            if (lane < 8) st_release_cta(sy.row + 8 * P + lane, sy.s + 1);
            if (!defer) sync_publish(sy.tr + P, sy.s + 1);
            return;
        }
    }
    double yv[C::KM][2];
    PROBE(1);
    if (kind == 0) {
        panel_structured<C, P, kRobust>(ch, Rb, Gs, t8, ws + C::XS, tau_out, n, sy);
#pragma unroll
        for (int k = 0; k < C::KM; ++k) {
            yv[k][0] = ch.a[k][P][0];
            yv[k][1] = ch.a[k][P][1];
        }
        if (ydst != nullptr && 8 * P + l4 < n) {
#pragma unroll
            for (int k = 0; k < C::KM; ++k)
                *reinterpret_cast<double2 *>(ydst + 8 * k + 2 * q + (int64_t)(8 * P + l4) * ldy) =
                    make_double2(yv[k][0], yv[k][1]);
        }
    } else {
        panel_dense<C, P, kRobust>(ch, kb, Gs, t8, tau_out, n);
        const int piv = 8 * kb + l4;                      // chunk row of this lane's column's pivot
#pragma unroll
        for (int k = 0; k < C::KM; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = 8 * k + 2 * q + e;
                yv[k][e] = r > piv ? ch.a[k][P][e] : (r == piv ? 1.0 : 0.0);
            }
    }
#pragma unroll
    for (int k = 0; k < C::KM; ++k) {
        Ys[(8 * k + 2 * q) * 8 + l4] = yv[k][0];
        Ys[(8 * k + 2 * q + 1) * 8 + l4] = yv[k][1];
    }
    __syncwarp();
    PROBE(5);
    // T (compact WY of the panel; cached in tg for apply / form Q) is built
    // inside trailing(), overlapped with the W^T DMMAs
    if (kind == 0) trailing<C, P, true>(ch, yv, Ys, Gs, t8, Ts, tg, Rb, sy, defer);
    else {
        trailing<C, P, false>(ch, yv, Ys, Gs, t8, Ts, tg, Rb, sy, defer);
        // the pivot block rows are R rows 8P .. 8P+7 from here on
#pragma unroll
        for (int k = 0; k < C::KM; ++k)
            if (k == kb) {
#pragma unroll
                for (int cb = P; cb < C::NCB; ++cb) {
                    Rb[(8 * P + 2 * q) * C::LDR + 8 * cb + l4] = ch.a[k][cb][0];
                    Rb[(8 * P + 2 * q + 1) * C::LDR + 8 * cb + l4] = ch.a[k][cb][1];
                }
            }
        asm volatile("" ::: "memory");
        __syncwarp();
        if (lane < 8) st_release_cta(sy.row + 8 * P + lane, sy.s + 1);
        if (!defer) sync_publish(sy.tr + P, sy.s + 1);
    }
    __syncwarp();
}

}  // namespace chunk
}  // namespace tsqr
