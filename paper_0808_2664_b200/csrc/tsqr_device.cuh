// Device building blocks of the B200 TSQR path (sm_100a).  Product code.
//
// Layout ("column-owner teams"): a team is one CTA of
// CW x G warps.  Lane l of column-warp cw owns matrix column c = 32*cw + l for a
// band of RT consecutive rows; row-group g owns rows [g*RT, (g+1)*RT).  A
// column's band lives in that lane's registers for the whole sweep, so the
// inner products of a Householder step (x^T A(:,c)) are per-lane sums: no
// cross-lane reduction (G = 1), and the only synchronisation per column is the
// publication of the pivot column (warp-level for a one-warp team).  Many small
// teams per SM (registers, not barriers, bound the residency) hide each other's
// reflector latency.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsqr {

struct DevPlan {
    const int64_t *tile_row0;   // first local row of tile t
    const int *tile_rows;       // rows of tile t
    const int *tile_parent;     // node id of leaf t's first combine, -1: none
    const int *node_a;          // by node id b: leftmost tile of the left subtree
    const int *node_parent;     // by node id: next node, -1: local root
    int L;                      // tiles
};

template <int CW_, int G_, int RT_>
struct Team {
    static constexpr int CW = CW_;            // column warps (n <= 32*CW)
    static constexpr int G = G_;              // row groups
    static constexpr int RT = RT_;            // rows per lane band
    static constexpr int NW = CW * G;         // warps per team (= CTA)
    static constexpr int NT = NW * 32;
    static constexpr int NPAD = CW * 32;      // columns a team can hold
    static constexpr int S = G * RT;          // tile rows a team can hold
    static constexpr int LDR = NPAD + 1;      // ld of n x n node blocks in smem
    static_assert(RT % 16 == 0, "bands are processed in chunks of 16 rows");
    __device__ static int lane() { return threadIdx.x & 31; }
    __device__ static int warp() { return threadIdx.x >> 5; }
    __device__ static int grp() { return warp() / CW; }
    __device__ static int col() { return (warp() % CW) * 32 + lane(); }
    __device__ static int row0() { return grp() * RT; }
};

template <int NW>
__device__ __forceinline__ void team_sync() {
    if constexpr (NW == 1) __syncwarp();
    else __syncthreads();
}

// ----------------------------------------------------------- register access
// Runtime-indexed access to a register band on a warp-uniform index (the column
// step j): one switch over 8-row chunks, then branch-free selects inside the
// chunk (no per-row jump tables, no local memory).
template <int B, int N>
__device__ __forceinline__ double sel8(const double (&a)[N], int lo) {
    double r = a[B];
#pragma unroll
    for (int q = 1; q < 8; ++q)
        if (B + q < N) r = (lo == q) ? a[B + q < N ? B + q : 0] : r;
    return r;
}
template <int B, int N>
__device__ __forceinline__ void sub8(double (&a)[N], int lo, double v) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (B + q < N) a[B + q < N ? B + q : 0] -= (lo == q) ? v : 0.0;
}

#define TSQR_CHUNKS(OP)                                                                       \
    switch (i >> 3) {                                                                         \
        case 0: OP(0); case 1: OP(8); case 2: OP(16); case 3: OP(24); case 4: OP(32);         \
        case 5: OP(40); case 6: OP(48); case 7: OP(56); case 8: OP(64); case 9: OP(72);       \
        case 10: OP(80); case 11: OP(88); case 12: OP(96); case 13: OP(104); case 14: OP(112); \
        case 15: OP(120);                                                                     \
        default: break;                                                                       \
    }

template <int N>
__device__ __forceinline__ double reg_get(const double (&a)[N], int i) {
    static_assert(N <= 128, "covers 128 registers");
#define TSQR_G(b) if constexpr ((b) < N) return sel8<((b) < N ? (b) : 0), N>(a, i & 7); else return 0.0
    TSQR_CHUNKS(TSQR_G)
#undef TSQR_G
    return 0.0;
}

template <int N>
__device__ __forceinline__ void reg_sub(double (&a)[N], int i, double v) {
#define TSQR_S(b) if constexpr ((b) < N) { sub8<((b) < N ? (b) : 0), N>(a, i & 7, v); return; } else return
    TSQR_CHUNKS(TSQR_S)
#undef TSQR_S
}

// ------------------------------------------------------------------ staging
// Asynchronous global -> smem staging (cp.async, 8-byte elements, zero fill).
__device__ __forceinline__ void cp_async8(double *sm, const double *g, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// global (rows x ncols, ld) -> smem (cap_rows x cap_cols, sld), zero padded.
// The caller waits with cp_async_wait_all() and a barrier.
template <int NT>
__device__ __forceinline__ void stage_in_async(double *sm, int sld, const double *g, int64_t ldg, int rows,
                                               int ncols, int cap_rows, int cap_cols) {
    for (int c = 0; c < cap_cols; ++c) {
        const double *gc = g + (int64_t)(c < ncols ? c : 0) * ldg;
        for (int r = threadIdx.x; r < cap_rows; r += NT) {
            const bool ok = (c < ncols) && (r < rows);
            cp_async8(sm + c * sld + r, ok ? gc + r : g, ok);
        }
    }
}

template <int NT>
__device__ __forceinline__ void stage_out(const double *sm, int sld, double *g, int64_t ldg, int rows, int ncols) {
    for (int c = 0; c < ncols; ++c) {
        double *gc = g + (int64_t)c * ldg;
        for (int r = threadIdx.x; r < rows; r += NT) gc[r] = sm[c * sld + r];
    }
}

// ------------------------------------------------------------ Householder
// LAPACK dlarfg convention (readings R1/R2): beta = -sign(alpha) N,
// N = sqrt(alpha^2 + sigma2), tau = (beta - alpha)/beta = 1 + |alpha|/N,
// v = x / (alpha - beta), i.e. scale = sign(alpha) / (|alpha| + N).
// sigma2 == 0 -> H = I.  rsqrt / rcp use the hardware approximations refined by
// Newton steps (<= 2 ulp).
__device__ __forceinline__ double rcp_nr(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}

struct House {
    double beta, tau, scale;
};
__device__ __forceinline__ House householder(double alpha, double sigma2) {
    House h;
    if (sigma2 == 0.0) {
        h.beta = alpha;
        h.tau = 0.0;
        h.scale = 0.0;
    } else {
        const double y = fma(alpha, alpha, sigma2);
        const double r = rsqrt(y);
        const double N = y * r;
        const double aa = fabs(alpha);
        h.beta = alpha >= 0.0 ? -N : N;
        h.tau = fma(aa, r, 1.0);
        const double inv = rcp_nr(aa + N);
        h.scale = alpha >= 0.0 ? inv : -inv;
    }
    return h;
}

// -------------------------------------------------------------- band math
// p = sum_i x[i] a[i] over a band; x from smem in 16-row chunks (two rows per
// 16-byte broadcast load), 8 independent accumulators.
template <int RT>
__device__ __forceinline__ double band_dot(const double *x, const double (&a)[RT]) {
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const double2 *x2 = reinterpret_cast<const double2 *>(x);
#pragma unroll
    for (int k = 0; k < RT / 16; ++k) {
        double xv[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double2 v = x2[k * 8 + q];
            xv[2 * q] = v.x;
            xv[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) s[q & 7] = fma(xv[q], a[k * 16 + q], s[q & 7]);
    }
    return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

// a[i] -= x[i] u over a band.
template <int RT>
__device__ __forceinline__ void band_axpy(const double *x, double u, double (&a)[RT]) {
    const double2 *x2 = reinterpret_cast<const double2 *>(x);
#pragma unroll
    for (int k = 0; k < RT / 16; ++k) {
        double xv[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double2 v = x2[k * 8 + q];
            xv[2 * q] = v.x;
            xv[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) a[k * 16 + q] = fma(-xv[q], u, a[k * 16 + q]);
    }
}

// The same over rows 0..j only (structured node blocks): chunks of 8 rows; the
// loop stops at the first chunk past row j (warp-uniform branch).
template <int NR>
__device__ __forceinline__ double head_dot(const double *x, const double (&a)[NR], int j) {
    double s[4] = {0, 0, 0, 0};
    const double2 *x2 = reinterpret_cast<const double2 *>(x);
#pragma unroll
    for (int k = 0; k < NR / 8; ++k) {
        if (k * 8 > j) break;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 v = x2[k * 4 + q];
            s[q] = fma(v.x, a[k * 8 + 2 * q], s[q]);
            s[q] = fma(v.y, a[k * 8 + 2 * q + 1], s[q]);
        }
    }
    return (s[0] + s[1]) + (s[2] + s[3]);
}

template <int NR>
__device__ __forceinline__ void head_axpy(const double *x, double u, double (&a)[NR], int j) {
    const double2 *x2 = reinterpret_cast<const double2 *>(x);
#pragma unroll
    for (int k = 0; k < NR / 8; ++k) {
        if (k * 8 > j) break;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 v = x2[k * 4 + q];
            a[k * 8 + 2 * q] = fma(-v.x, u, a[k * 8 + 2 * q]);
            a[k * 8 + 2 * q + 1] = fma(-v.y, u, a[k * 8 + 2 * q + 1]);
        }
    }
}

// ============================================================== tile QR (a2)
// Unblocked Householder QR (DGEQR2: the leaf QR of Alg. TSQR:par line 1,
// P:1679-1680) of a team-resident tile.  Column j:
//  1. the owner lanes (column j, one per row group) publish x = A(:, j) with
//     rows <= j zeroed (double-buffered xs) and alpha = A(j, j);
//  2. sync; every lane forms p_c = x^T A(:, c) over its band (c = j gives
//     sigma^2 = ||A(j+1:, j)||^2); row groups add their partials (G > 1);
//  3. every lane forms beta, tau, scale (dlarfg) and w_c = A(j,c) + scale p_c
//     = v^T A(:, c), then A(:, c) -= x (tau scale w_c) and A(j, c) -= tau w_c.
// Column j stays in place and becomes (beta, v = scale x) once at the end.
// Smem: xs[2][S]; red[2][2][G][NPAD] (NW > 1); alph[2]; taus/betas/scales[NPAD].
struct NoProbe {
    __device__ static void mark(int, int) {}
};

template <class T, class Probe = NoProbe>
__device__ __forceinline__ void team_tile_qr(double (&a)[T::RT], int n, double *xs, double *red, double *alph,
                                             double *taus, double *betas, double *scales) {
    constexpr int RT = T::RT, S = T::S, G = T::G, NP = T::NPAD;
    const int c = T::col(), g = T::grp(), r0 = T::row0();
#pragma unroll 1
    for (int j = 0; j < n; ++j) {
        const int b = j & 1;
        double *xb = xs + b * S;
        const int gj = j / RT, ij = j - gj * RT;
        Probe::mark(j, 0);
        // 1. publish the pivot column: the owner lane stores its band unmasked
        //    (16-byte stores, no per-element predicates), then its warp zeroes
        //    rows <= j in parallel.  Warp-uniform branch: only the owner's warp.
        if ((T::warp() % T::CW) == (j >> 5)) {
            double *xg = xb + r0;
            if (T::lane() == (j & 31)) {
#pragma unroll
                for (int i = 0; i < RT; i += 2)
                    *reinterpret_cast<double2 *>(xg + i) = make_double2(a[i], a[i + 1]);
            }
            if (r0 <= j) {
                __syncwarp();
                const int hi = j - r0 < RT - 1 ? j - r0 : RT - 1;
                for (int r = T::lane(); r <= hi; r += 32) xg[r] = 0.0;
            }
        }
        Probe::mark(j, 1);
        team_sync<T::NW>();
        Probe::mark(j, 2);
        // 2. partial inner products over my band
        const double p = band_dot<RT>(xb + r0, a);
        const double rj = (g == gj) ? reg_get(a, ij) : 0.0;     // A(j, c)
        Probe::mark(j, 3);
        double P, RJ, sig2, alpha;
        if constexpr (T::NW == 1) {
            P = p;
            RJ = rj;
            sig2 = __shfl_sync(0xffffffffu, p, j);
            alpha = __shfl_sync(0xffffffffu, rj, j);
        } else {
            double *rp = red + (b * 2) * G * NP, *rr = rp + G * NP;
            rp[g * NP + c] = p;
            rr[g * NP + c] = rj;
            team_sync<T::NW>();
            P = 0.0;
            RJ = 0.0;
            sig2 = 0.0;
            alpha = 0.0;
#pragma unroll
            for (int q = 0; q < G; ++q) {
                P += rp[q * NP + c];
                RJ += rr[q * NP + c];
                sig2 += rp[q * NP + j];
                alpha += rr[q * NP + j];
            }
        }
        Probe::mark(j, 4);
        // 3. reflector and rank-1 update
        const House h = householder(alpha, sig2);
        const double w = fma(P, h.scale, RJ);                     // v^T A(:, c)
        const double u = (c > j && c < n) ? h.tau * h.scale * w : 0.0;
        Probe::mark(j, 5);
        band_axpy<RT>(xb + r0, u, a);
        Probe::mark(j, 6);
        if (g == gj) reg_sub(a, ij, (alpha - h.beta) * u);        // A(j,c) -= tau w_c
        Probe::mark(j, 7);
        if (threadIdx.x == 0) {
            taus[j] = h.tau;
            betas[j] = h.beta;
            scales[j] = h.scale;
        }
    }
    team_sync<T::NW>();
    if (c < n) {
        const double sc = scales[c], be = betas[c];
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            const int r = r0 + i;
            a[i] = r > c ? a[i] * sc : (r == c ? be : a[i]);
        }
    }
}

// ============================================================ node QR (a4)
// Structured QR of [Ra; Rb] (two n x n upper triangles), Alg. QR:qnxn with q = 2
// (P:1958-1979): reflector j acts on {row j of Ra} u {rows 0..j of Rb}.
// Ra: smem (ld LDR); lane c holds column c of Rb (rows 0..NPAD-1) in rb.
// On exit Ra = R (upper), rb = Y1(:, c) (eq. fact_2rs), taus[j].  Loops over Rb
// rows stop after row j: the triangular zeros are never touched.
template <class T>
__device__ __forceinline__ void team_node_qr(double *Ra, double (&rb)[T::NPAD], int n, double *xs, double *red,
                                             double *taus, double *betas, double *scales) {
    constexpr int NP = T::NPAD, LDR = T::LDR;
    const int c = T::col();
    const bool act = T::grp() == 0;          // row groups > 0 idle (they own the same columns)
#pragma unroll 1
    for (int j = 0; j < n; ++j) {
        const int b = j & 1;
        double *xb = xs + b * NP;
        if (act && c == j) {
#pragma unroll
            for (int k = 0; k < NP / 8; ++k) {
                if (k * 8 > j) break;
#pragma unroll
                for (int q = 0; q < 8; ++q) xb[k * 8 + q] = (k * 8 + q <= j) ? rb[k * 8 + q] : 0.0;
            }
        }
        team_sync<T::NW>();
        double p = 0.0, sig2 = 0.0;
        if (act) p = head_dot<NP>(xb, rb, j);
        if constexpr (T::NW == 1) {
            sig2 = __shfl_sync(0xffffffffu, p, j);
        } else {
            if (act && c == j) red[b] = p;
            team_sync<T::NW>();
            sig2 = red[b];
        }
        if (act) {
            const double alpha = Ra[j * LDR + j];
            const double RJ = Ra[c * LDR + j];
            const House h = householder(alpha, sig2);
            const double w = fma(p, h.scale, RJ);
            const bool trail = (c > j && c < n);
            const double u = trail ? h.tau * h.scale * w : 0.0;
            head_axpy<NP>(xb, u, rb, j);
            if (trail) Ra[c * LDR + j] = RJ - h.tau * w;
            if (threadIdx.x == 0) {
                taus[j] = h.tau;
                betas[j] = h.beta;
                scales[j] = h.scale;
            }
        }
    }
    team_sync<T::NW>();
    if (act && c < n) {
        const double sc = scales[c];
#pragma unroll
        for (int i = 0; i < NP; ++i)
            if (i <= c) rb[i] *= sc;
        Ra[c * LDR + c] = betas[c];
    }
    team_sync<T::NW>();
}

// ======================================================= reflector applies
// Tile reflectors on a team-resident band of C (lane = one C column),
// j = 0..n-1 (kForward: Q^T, [TR] P:1915-1938) or n-1..0 (Q, form-Q).
// Ys: smem, column-major (ld yld), unit diagonal and zeros above in place.
template <class T, bool kForward>
__device__ __forceinline__ void team_tile_apply(double (&cb)[T::RT], int n, const double *Ys, int yld, const double *tau,
                                double *red) {
    constexpr int RT = T::RT, G = T::G, NP = T::NPAD;
    const int c = T::col(), g = T::grp(), r0 = T::row0();
#pragma unroll 1
    for (int jj = 0; jj < n; ++jj) {
        const int j = kForward ? jj : n - 1 - jj;
        const double *x = Ys + j * yld + r0;
        double P = band_dot<RT>(x, cb);
        if constexpr (G > 1) {
            double *rp = red + (jj & 1) * G * NP;
            rp[g * NP + c] = P;
            team_sync<T::NW>();
            P = 0.0;
#pragma unroll
            for (int q = 0; q < G; ++q) P += rp[q * NP + c];
        }
        band_axpy<RT>(x, tau[j] * P, cb);
    }
}

// Node reflectors on the head rows [Ca; Cb] (eq. localQTupdate, P:2193-2212,
// one reflector [e_j; Y1(0:j, j)] at a time).  Y1: smem, column j at Y1 + j*LDY
// (LDY even: 16-byte aligned columns for the broadcast loads, zeros below the
// diagonal); Ca: smem, row j of column c at Ca[c*LDC + j] (LDC odd: conflict-free
// per-lane access); lane c holds column c of Cb (rows 0..NR-1) in cbh.  No
// synchronisation: every lane touches only its own column.
template <int NR, int LDY, int LDC, bool kForward>
__device__ __forceinline__ void team_node_apply(const double *Y1, const double *tau, double *Ca, double (&cbh)[NR],
                                                int n, int c) {
    static_assert(LDY % 2 == 0, "Y1 columns are read as double2");
#pragma unroll 1
    for (int jj = 0; jj < n; ++jj) {
        const int j = kForward ? jj : n - 1 - jj;
        const double *y = Y1 + j * LDY;
        const double caj = Ca[c * LDC + j];
        const double u = tau[j] * (caj + head_dot<NR>(y, cbh, j));
        head_axpy<NR>(y, u, cbh, j);
        Ca[c * LDC + j] = caj - u;
    }
}

// Ticket of the single-pass tree: true if this CTA is the second (last)
// arriver at node p and must run it.  Writers fence their global stores first.
template <int NW>
__device__ __forceinline__ bool ticket(int *counters, int p, int *flag_smem) {
    __threadfence();
    team_sync<NW>();
    if (threadIdx.x == 0) {
        const int old = atomicAdd(counters + p, 1);
        if (old == 1) counters[p] = 0;        // both arrived: reset for the next call
        *flag_smem = old;
    }
    team_sync<NW>();
    const bool last = (*flag_smem == 1);
    if (last) __threadfence();
    return last;
}

}  // namespace tsqr
