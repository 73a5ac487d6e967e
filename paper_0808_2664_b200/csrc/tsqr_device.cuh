// Device building blocks of the B200 TSQR path (sm_100a).  Product code.
//
// Data layout: fp64 column-major, element (i,j) at
// X[i + j*ld].  A tile of <= S rows x NP columns (NP = n padded to 16/32/64) is
// held in REGISTERS by a 256-thread CTA for the whole Householder sweep:
//   lane l of warp w owns columns  colbase(l) + 32*cc   (cc < CPL)
//                      and rows    w*RW + i*LPC + rph(l) (i < RT)
// so that every element is touched by exactly one thread and the per-column
// reductions are (warp partials in registers) -> (LPC-lane shuffle) -> (one
// __syncthreads on a double-buffered smem array).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsqr {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

struct DevPlan {
    const int64_t *tile_row0;   // first local row of tile t
    const int *tile_rows;       // rows of tile t
    const int *tile_parent;     // node id of leaf t's first combine, -1: none
    const int *node_a;          // by node id b: leftmost tile of the left subtree
    const int *node_parent;     // by node id: next node, -1: local root
    int L;                      // tiles
};

template <int NP_, int RT_>
struct Layout {
    static constexpr int NP = NP_;
    static constexpr int RT = RT_;                         // register rows per thread
    static constexpr int LC = NP < 32 ? NP : 32;           // lanes with distinct columns
    static constexpr int CPL = NP > 32 ? NP / 32 : 1;      // columns per lane
    static constexpr int LPC = 32 / LC;                    // lanes per column (row phases)
    static constexpr int RW = RT * LPC;                    // rows per warp
    static constexpr int S = RW * kWarps;                  // tile capacity (rows)
    static constexpr int SLD = S + 1;                      // odd smem ld: conflict-free
    __device__ static int lane() { return threadIdx.x & 31; }
    __device__ static int warp() { return threadIdx.x >> 5; }
    __device__ static int colbase() { return lane() % LC; }
    __device__ static int rph() { return lane() / LC; }
    __device__ static int col(int cc) { return colbase() + 32 * cc; }
    __device__ static int row(int i) { return warp() * RW + i * LPC + rph(); }
};

// ------------------------------------------------------------------ staging
__device__ __forceinline__ void stage_out(const double *sm, int sld, double *g, int64_t ldg,
                                          int rows, int ncols) {
    for (int c = 0; c < ncols; ++c) {
        double *gc = g + (int64_t)c * ldg;
        for (int r = threadIdx.x; r < rows; r += kThreads) gc[r] = sm[c * sld + r];
    }
}

// Asynchronous global -> smem staging (cp.async, 8-byte elements, zero fill):
// every element is in flight at once instead of one dependent load per column.
__device__ __forceinline__ void cp_async8(double *sm, const double *g, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// global (rows x ncols, ld) -> smem (cap_rows x cap_cols, sld), zero padded; the
// caller waits with cp_async_wait_all() + __syncthreads().
__device__ __forceinline__ void stage_in_async(double *sm, int sld, const double *g, int64_t ldg, int rows,
                                               int ncols, int cap_rows, int cap_cols) {
    for (int c = 0; c < cap_cols; ++c) {
        const double *gc = g + (int64_t)(c < ncols ? c : 0) * ldg;
        for (int r = threadIdx.x; r < cap_rows; r += kThreads) {
            const bool ok = (c < ncols) && (r < rows);
            cp_async8(sm + c * sld + r, ok ? gc + r : g, ok);
        }
    }
}

template <class Lt>
__device__ __forceinline__ void smem_to_regs(const double *sm, double (&a)[Lt::RT][Lt::CPL]) {
#pragma unroll
    for (int cc = 0; cc < Lt::CPL; ++cc)
#pragma unroll
        for (int i = 0; i < Lt::RT; ++i) a[i][cc] = sm[Lt::col(cc) * Lt::SLD + Lt::row(i)];
}

template <class Lt>
__device__ __forceinline__ void regs_to_smem(double *sm, const double (&a)[Lt::RT][Lt::CPL]) {
#pragma unroll
    for (int cc = 0; cc < Lt::CPL; ++cc)
#pragma unroll
        for (int i = 0; i < Lt::RT; ++i) sm[Lt::col(cc) * Lt::SLD + Lt::row(i)] = a[i][cc];
}

// Read this thread's RT values of a per-row vector xs[0..S) (same rows as the
// register tile).  LPC == 1: all lanes of a warp read the same addresses
// (broadcast), vectorised two rows per load.
template <class Lt>
__device__ __forceinline__ void load_rowvec(const double *xs, double (&x)[Lt::RT]) {
    if constexpr (Lt::LPC == 1 && (Lt::RT % 2) == 0) {
        const double2 *x2 = reinterpret_cast<const double2 *>(xs + Lt::warp() * Lt::RW);
#pragma unroll
        for (int i = 0; i < Lt::RT / 2; ++i) {
            double2 v = x2[i];
            x[2 * i] = v.x;
            x[2 * i + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < Lt::RT; ++i) x[i] = xs[Lt::row(i)];
    }
}

__device__ __forceinline__ double warp_sum_lpc(double v, int lc) {
    for (int o = lc; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Householder scalars in the LAPACK dlarfg convention (reading R1/R2):
// beta = -sign(alpha) N, N = sqrt(alpha^2 + sigma2), tau = (beta - alpha)/beta
// = 1 + |alpha|/N, v = x / (alpha - beta) below the pivot, i.e.
// scale = sign(alpha) / (|alpha| + N).  sigma2 == 0 -> H = I.
// The critical path avoids IEEE sqrt/div sequences: N = y * rsqrt(y) and the
// reciprocal use the hardware approximations refined by Newton steps
// (<= 2 ulp).
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
        const double r = rsqrt(y);                     // MUFU + Newton, ~1 ulp
        const double N = y * r;
        const double aa = fabs(alpha);
        h.beta = alpha >= 0.0 ? -N : N;
        h.tau = fma(aa, r, 1.0);                      // 1 + |alpha| / N
        const double inv = rcp_nr(aa + N);
        h.scale = alpha >= 0.0 ? inv : -inv;
    }
    return h;
}

// Sum of the kWarps partials of column c in a fixed tree order (every thread
// gets bit-identical results).
__device__ __forceinline__ double sum_warps(const double *redb, int stride, int c) {
    double v[kWarps];
#pragma unroll
    for (int q = 0; q < kWarps; ++q) v[q] = redb[q * stride + c];
#pragma unroll
    for (int h = kWarps / 2; h >= 1; h /= 2)
#pragma unroll
        for (int q = 0; q < h; ++q) v[q] = v[q] + v[q + h];
    return v[0];
}

// ============================================================== tile QR (a2)
// Fetch register row i (runtime index) of this thread's tile: a jump table,
// executed only by the one warp that holds the row (warp-uniform branch).
template <class Lt>
__device__ __forceinline__ double reg_row(const double (&a)[Lt::RT][Lt::CPL], int i, int cc) {
    static_assert(Lt::RT <= 64, "reg_row covers 64 register rows");
    switch (i) {
        case 0: return a[0 < Lt::RT ? 0 : 0][cc];
        case 1: return a[1 < Lt::RT ? 1 : 0][cc];
        case 2: return a[2 < Lt::RT ? 2 : 0][cc];
        case 3: return a[3 < Lt::RT ? 3 : 0][cc];
        case 4: return a[4 < Lt::RT ? 4 : 0][cc];
        case 5: return a[5 < Lt::RT ? 5 : 0][cc];
        case 6: return a[6 < Lt::RT ? 6 : 0][cc];
        case 7: return a[7 < Lt::RT ? 7 : 0][cc];
        case 8: return a[8 < Lt::RT ? 8 : 0][cc];
        case 9: return a[9 < Lt::RT ? 9 : 0][cc];
        case 10: return a[10 < Lt::RT ? 10 : 0][cc];
        case 11: return a[11 < Lt::RT ? 11 : 0][cc];
        case 12: return a[12 < Lt::RT ? 12 : 0][cc];
        case 13: return a[13 < Lt::RT ? 13 : 0][cc];
        case 14: return a[14 < Lt::RT ? 14 : 0][cc];
        case 15: return a[15 < Lt::RT ? 15 : 0][cc];
        case 16: return a[16 < Lt::RT ? 16 : 0][cc];
        case 17: return a[17 < Lt::RT ? 17 : 0][cc];
        case 18: return a[18 < Lt::RT ? 18 : 0][cc];
        case 19: return a[19 < Lt::RT ? 19 : 0][cc];
        case 20: return a[20 < Lt::RT ? 20 : 0][cc];
        case 21: return a[21 < Lt::RT ? 21 : 0][cc];
        case 22: return a[22 < Lt::RT ? 22 : 0][cc];
        case 23: return a[23 < Lt::RT ? 23 : 0][cc];
        case 24: return a[24 < Lt::RT ? 24 : 0][cc];
        case 25: return a[25 < Lt::RT ? 25 : 0][cc];
        case 26: return a[26 < Lt::RT ? 26 : 0][cc];
        case 27: return a[27 < Lt::RT ? 27 : 0][cc];
        case 28: return a[28 < Lt::RT ? 28 : 0][cc];
        case 29: return a[29 < Lt::RT ? 29 : 0][cc];
        case 30: return a[30 < Lt::RT ? 30 : 0][cc];
        case 31: return a[31 < Lt::RT ? 31 : 0][cc];
        case 32: return a[32 < Lt::RT ? 32 : 0][cc];
        case 33: return a[33 < Lt::RT ? 33 : 0][cc];
        case 34: return a[34 < Lt::RT ? 34 : 0][cc];
        case 35: return a[35 < Lt::RT ? 35 : 0][cc];
        case 36: return a[36 < Lt::RT ? 36 : 0][cc];
        case 37: return a[37 < Lt::RT ? 37 : 0][cc];
        case 38: return a[38 < Lt::RT ? 38 : 0][cc];
        case 39: return a[39 < Lt::RT ? 39 : 0][cc];
        case 40: return a[40 < Lt::RT ? 40 : 0][cc];
        case 41: return a[41 < Lt::RT ? 41 : 0][cc];
        case 42: return a[42 < Lt::RT ? 42 : 0][cc];
        case 43: return a[43 < Lt::RT ? 43 : 0][cc];
        case 44: return a[44 < Lt::RT ? 44 : 0][cc];
        case 45: return a[45 < Lt::RT ? 45 : 0][cc];
        case 46: return a[46 < Lt::RT ? 46 : 0][cc];
        case 47: return a[47 < Lt::RT ? 47 : 0][cc];
        case 48: return a[48 < Lt::RT ? 48 : 0][cc];
        case 49: return a[49 < Lt::RT ? 49 : 0][cc];
        case 50: return a[50 < Lt::RT ? 50 : 0][cc];
        case 51: return a[51 < Lt::RT ? 51 : 0][cc];
        case 52: return a[52 < Lt::RT ? 52 : 0][cc];
        case 53: return a[53 < Lt::RT ? 53 : 0][cc];
        case 54: return a[54 < Lt::RT ? 54 : 0][cc];
        case 55: return a[55 < Lt::RT ? 55 : 0][cc];
        case 56: return a[56 < Lt::RT ? 56 : 0][cc];
        case 57: return a[57 < Lt::RT ? 57 : 0][cc];
        case 58: return a[58 < Lt::RT ? 58 : 0][cc];
        case 59: return a[59 < Lt::RT ? 59 : 0][cc];
        case 60: return a[60 < Lt::RT ? 60 : 0][cc];
        case 61: return a[61 < Lt::RT ? 61 : 0][cc];
        case 62: return a[62 < Lt::RT ? 62 : 0][cc];
        case 63: return a[63 < Lt::RT ? 63 : 0][cc];
        default: return 0.0;
    }
}

// Unblocked Householder QR of the register tile a (rows x n, padded).  One
// __syncthreads per column.  Per column j:
//   1. the owner lane of column j publishes x = A(:, j) (rows > j; rows <= j
//      zeroed) in smem xs;
//   2. every thread forms partial dots x^T A(:, c) over its rows (c = j gives
//      sigma^2 = ||x(j+1:)||^2); the thread holding row j publishes A(j, :);
//   3. one barrier; every thread reduces the partials (same order: identical
//      scalars), forms beta, tau and scale = 1/(alpha - beta) (dlarfg), and
//      w_c = A(j,c) + scale x^T A(:,c) = v^T A(:,c);
//   4. xs[j] := alpha - beta, so one rank-1 update A(:,c) -= xs * (tau*scale*w_c)
//      also performs row j's update A(j,c) -= tau w_c, with no per-element masks.
// Column j itself is left untouched in the loop; its final form (beta on the
// diagonal, v = x * scale below) is applied once after the loop.
// Smem: xs[S], red[2][kWarps][NP], rowj[2][NP], taus/betas/scales[NP].
struct NoProbe {
    __device__ static void mark(int, int) {}
};

template <class Lt, class Probe = NoProbe>
__device__ void tile_qr(double (&a)[Lt::RT][Lt::CPL], int n, double *xs, double *red,
                        double *rowj, double *taus, double *betas, double *scales) {
    constexpr int RT = Lt::RT, CPL = Lt::CPL, NP = Lt::NP;
    const int w = Lt::warp(), l = Lt::lane(), rph = Lt::rph();
    for (int j = 0; j < n; ++j) {
        const int buf = j & 1;
        double *redb = red + buf * (kWarps * NP);
        double *rjb = rowj + buf * NP;
        const int wj = j / Lt::RW, ij = (j % Lt::RW) / Lt::LPC, pj = (j % Lt::RW) % Lt::LPC;
        Probe::mark(j, 0);
        // 1. publish the pivot column of my warp's rows
        __syncwarp();
        if (Lt::colbase() == (j & 31)) {
            double *xw = xs + w * Lt::RW;
            if (j < 32) {
#pragma unroll
                for (int i = 0; i < RT; ++i) xw[i * Lt::LPC + rph] = a[i][0];
            } else {
#pragma unroll
                for (int i = 0; i < RT; ++i) xw[i * Lt::LPC + rph] = a[i][CPL - 1];
            }
        }
        __syncwarp();
        if (w * Lt::RW <= j && l == 0) {                 // rows <= j of this warp are not in x
            const int hi = min(j, w * Lt::RW + Lt::RW - 1);
            for (int r = w * Lt::RW; r <= hi; ++r) xs[r] = 0.0;
        }
        __syncwarp();
        Probe::mark(j, 1);
        // 2. partial inner products x^T A(:, c) over my rows
        double p[CPL];
        {
            double x[RT];
            load_rowvec<Lt>(xs, x);
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) {
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
                for (int i = 0; i < RT; i += 4) {
                    s0 = fma(x[i], a[i][cc], s0);
                    if (i + 1 < RT) s1 = fma(x[i + 1], a[i + 1][cc], s1);
                    if (i + 2 < RT) s2 = fma(x[i + 2], a[i + 2][cc], s2);
                    if (i + 3 < RT) s3 = fma(x[i + 3], a[i + 3][cc], s3);
                }
                p[cc] = warp_sum_lpc((s0 + s1) + (s2 + s3), Lt::LC);
            }
        }
        if (rph == 0) {
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) redb[w * NP + Lt::col(cc)] = p[cc];
        }
        if (w == wj && rph == pj) {
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) rjb[Lt::col(cc)] = reg_row<Lt>(a, ij, cc);
        }
        Probe::mark(j, 2);
        __syncthreads();
        Probe::mark(j, 3);
        // 3. reduce across warps
        const double sig2 = sum_warps(redb, NP, j);
        const double alpha = rjb[j];
        const House h = householder(alpha, sig2);
        double u[CPL];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
            const int c = Lt::col(cc);
            const double P = sum_warps(redb, NP, c);
            const double wc = fma(P, h.scale, rjb[c]);        // v^T A(:, c)
            u[cc] = (c > j && c < n) ? h.tau * h.scale * wc : 0.0;
        }
        Probe::mark(j, 4);
        // 4. row j rides in the broadcast vector: xs[j] = alpha - beta (= 1/scale)
        if (w == wj && l == 0) xs[j] = alpha - h.beta;
        if (threadIdx.x == 0) {
            taus[j] = h.tau;
            betas[j] = h.beta;
            scales[j] = h.scale;
        }
        __syncwarp();
        double x[RT];
        load_rowvec<Lt>(xs, x);
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
            for (int i = 0; i < RT; ++i) a[i][cc] = fma(-x[i], u[cc], a[i][cc]);
        Probe::mark(j, 5);
    }
    __syncthreads();
    // the pivot columns become (beta, v = x * scale) in place
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
        const int c = Lt::col(cc);
        if (c < n) {
            const double sc = scales[c], be = betas[c];
#pragma unroll
            for (int i = 0; i < RT; ++i) {
                const int r = Lt::row(i);
                a[i][cc] = r > c ? a[i][cc] * sc : (r == c ? be : a[i][cc]);
            }
        }
    }
}

// ====================================================== tile reflector apply
// C (register tile, same rows as the Y tile in smem Ys[col*yld + row], with
// unit diagonal and zeros above it already in place) <- H_j C for
// j = 0..n-1 (kForward: Q^T, leaf stage of apply-Q^T, [TR] P:1915-1938) or
// j = n-1..0 (Q, leaf stage of form-Q).  One __syncthreads per reflector.
template <class Lt, bool kForward>
__device__ void tile_apply(double (&c)[Lt::RT][Lt::CPL], int n, const double *Ys, int yld,
                           const double *tau, double *red) {
    constexpr int RT = Lt::RT, CPL = Lt::CPL, NP = Lt::NP;
    const int w = Lt::warp(), rph = Lt::rph();
    for (int jj = 0; jj < n; ++jj) {
        const int j = kForward ? jj : n - 1 - jj;
        double *redb = red + (jj & 1) * (kWarps * NP);
        double p[CPL];
        {
            double x[RT];
            load_rowvec<Lt>(Ys + j * yld, x);
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) {
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
                for (int i = 0; i < RT; i += 4) {
                    s0 = fma(x[i], c[i][cc], s0);
                    if (i + 1 < RT) s1 = fma(x[i + 1], c[i + 1][cc], s1);
                    if (i + 2 < RT) s2 = fma(x[i + 2], c[i + 2][cc], s2);
                    if (i + 3 < RT) s3 = fma(x[i + 3], c[i + 3][cc], s3);
                }
                p[cc] = warp_sum_lpc((s0 + s1) + (s2 + s3), Lt::LC);
            }
        }
        if (rph == 0) {
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) redb[w * NP + Lt::col(cc)] = p[cc];
        }
        __syncthreads();
        const double t = tau[j];
        double x[RT];
        load_rowvec<Lt>(Ys + j * yld, x);
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
            const double P = sum_warps(redb, NP, Lt::col(cc));
            const double u = t * P;
#pragma unroll
            for (int i = 0; i < RT; ++i) c[i][cc] = fma(-x[i], u, c[i][cc]);
        }
    }
}

// ===================================================== node (structured) ops
// Thread mapping for n x n node work: lanes own columns as in Layout<NP,*>;
// row i of the lower block belongs to thread (w, rph) with
//   i = (k*kWarps + w)*LPC + rph,  k < KR = NP / (kWarps*LPC).
template <int NP>
struct NodeLayout {
    using Lt = Layout<NP, 1>;
    static constexpr int CPL = Lt::CPL, LPC = Lt::LPC, LC = Lt::LC;
    static constexpr int KR = NP / (kWarps * LPC) > 0 ? NP / (kWarps * LPC) : 1;
    static constexpr int LD = NP + 1;
    __device__ static int row(int k) { return (k * kWarps + Lt::warp()) * LPC + Lt::rph(); }
};

// Structured QR of [Ra; Rb] (two n x n upper triangles), Alg. QR:qnxn with q = 2
// (P:1958-1979): reflector j acts on {row j of Ra} u {rows 0..j of Rb}.
// Ra, Rb: smem n x n (ld NP+1), zero below the diagonal.  On exit Ra = R,
// Rb = Y1 (upper, eq. fact_2rs), taus[j].  One __syncthreads per column.
template <int NP>
__device__ void node_qr(double *Ra, double *Rb, int n, double *red, double *taus) {
    using NL = NodeLayout<NP>;
    using Lt = typename NL::Lt;
    constexpr int CPL = NL::CPL, KR = NL::KR, LD = NL::LD;
    const int w = Lt::warp(), rph = Lt::rph();
    double rb[KR][CPL];
#pragma unroll
    for (int k = 0; k < KR; ++k)
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) rb[k][cc] = Rb[Lt::col(cc) * LD + NL::row(k)];
    for (int j = 0; j < n; ++j) {
        double *redb = red + (j & 1) * (kWarps * NP);
        const int cj = j >> 5;
        const int src = (j & 31) % NL::LC + rph * NL::LC;     // lane owning (my rows, col j)
        double x[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const double v = __shfl_sync(0xffffffffu, (cj == 0) ? rb[k][0] : rb[k][CPL - 1], src);
            x[k] = NL::row(k) <= j ? v : 0.0;
        }
        double p[CPL], raj[CPL];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < KR; ++k) s = fma(x[k], rb[k][cc], s);
            p[cc] = warp_sum_lpc(s, NL::LC);
            raj[cc] = Ra[Lt::col(cc) * LD + j];
        }
        const double alpha = Ra[j * LD + j];
        if (rph == 0) {
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) redb[w * NP + Lt::col(cc)] = p[cc];
        }
        __syncthreads();
        const double sig2 = sum_warps(redb, NP, j);
        const House h = householder(alpha, sig2);
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
            const int c = Lt::col(cc);
            const double P = sum_warps(redb, NP, c);
            const double wc = fma(P, h.scale, raj[cc]);
            const bool trail = (c > j) && (c < n);
            const double u = trail ? h.tau * h.scale * wc : 0.0;
#pragma unroll
            for (int k = 0; k < KR; ++k) rb[k][cc] = fma(-x[k], u, rb[k][cc]);
            if (c == j) {
#pragma unroll
                for (int k = 0; k < KR; ++k) rb[k][cc] = x[k] * h.scale;   // Y1(:, j)
            }
            if (w == 0 && rph == 0) {
                if (trail) Ra[c * LD + j] = raj[cc] - h.tau * wc;
                else if (c == j) Ra[c * LD + j] = h.beta;
            }
        }
        if (threadIdx.x == 0) taus[j] = h.tau;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KR; ++k)
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) Rb[Lt::col(cc) * LD + NL::row(k)] = rb[k][cc];
    __syncthreads();
}

// Node reflectors applied to the head rows [Ca; Cb] (n x kc each, smem, ld NP+1,
// kc <= NP columns): eq. localQTupdate one reflector at a time,
// j ascending (kForward: Q^T, apply stage) or descending (Q, form-Q stage).
// Y1: smem n x n upper (ld NP+1).  One __syncthreads per reflector.
template <int NP, bool kForward>
__device__ void node_apply(const double *Y1, const double *tau, double *Ca, double *Cb, int n,
                           double *red) {
    using NL = NodeLayout<NP>;
    using Lt = typename NL::Lt;
    constexpr int CPL = NL::CPL, KR = NL::KR, LD = NL::LD;
    const int w = Lt::warp(), rph = Lt::rph();
    double cb[KR][CPL];
#pragma unroll
    for (int k = 0; k < KR; ++k)
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) cb[k][cc] = Cb[Lt::col(cc) * LD + NL::row(k)];
    for (int jj = 0; jj < n; ++jj) {
        const int j = kForward ? jj : n - 1 - jj;
        double *redb = red + (jj & 1) * (kWarps * NP);
        double y[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) y[k] = NL::row(k) <= j ? Y1[j * LD + NL::row(k)] : 0.0;
        double p[CPL], caj[CPL];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < KR; ++k) s = fma(y[k], cb[k][cc], s);
            p[cc] = warp_sum_lpc(s, NL::LC);
            caj[cc] = Ca[Lt::col(cc) * LD + j];
        }
        if (rph == 0) {
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) redb[w * NP + Lt::col(cc)] = p[cc];
        }
        __syncthreads();
        const double t = tau[j];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
            const int c = Lt::col(cc);
            const double P = sum_warps(redb, NP, c);
            const double u = t * (caj[cc] + P);
#pragma unroll
            for (int k = 0; k < KR; ++k) cb[k][cc] = fma(-y[k], u, cb[k][cc]);
            if (w == 0 && rph == 0) Ca[c * LD + j] = caj[cc] - u;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KR; ++k)
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) Cb[Lt::col(cc) * LD + NL::row(k)] = cb[k][cc];
    __syncthreads();
}

// Load / store an n x n upper triangle (head block of a tile) between global
// (ld) and smem (ld NP+1, zero elsewhere).  Loads are issued all at once
// (clamped addresses, select after the load) so they overlap.
template <int NP, bool kCG>
__device__ __forceinline__ void load_upper(double *sm, const double *g, int64_t ld, int n) {
    constexpr int PER = (NP * NP + kThreads - 1) / kThreads;
    double v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int e = threadIdx.x + q * kThreads;
        const int r = e % NP, c = e / NP;
        const bool ok = e < NP * NP && r <= c && c < n;
        const double *p = ok ? g + r + (int64_t)c * ld : g;
        v[q] = kCG ? __ldcg(p) : p[0];
        v[q] = ok ? v[q] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int e = threadIdx.x + q * kThreads;
        if (e < NP * NP) sm[(e / NP) * (NP + 1) + e % NP] = v[q];
    }
}

template <int NP>
__device__ __forceinline__ void store_upper(const double *sm, double *g, int64_t ld, int n) {
    for (int e = threadIdx.x; e < n * n; e += kThreads) {
        const int r = e % n, c = e / n;
        if (r <= c) g[r + (int64_t)c * ld] = sm[c * (NP + 1) + r];
    }
}

// Rectangular n x kc block between global and smem (ld NP+1).
template <int NP, bool kCG>
__device__ __forceinline__ void load_block(double *sm, const double *g, int64_t ld, int n, int kc) {
    constexpr int PER = (NP * NP + kThreads - 1) / kThreads;
    double v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int e = threadIdx.x + q * kThreads;
        const int r = e % NP, c = e / NP;
        const bool ok = e < NP * NP && r < n && c < kc;
        const double *p = ok ? g + r + (int64_t)c * ld : g;
        v[q] = kCG ? __ldcg(p) : p[0];
        v[q] = ok ? v[q] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int e = threadIdx.x + q * kThreads;
        if (e < NP * NP) sm[(e / NP) * (NP + 1) + e % NP] = v[q];
    }
}

template <int NP>
__device__ __forceinline__ void store_block(const double *sm, double *g, int64_t ld, int n, int kc) {
    for (int e = threadIdx.x; e < n * kc; e += kThreads) {
        const int r = e % n, c = e / n;
        g[r + (int64_t)c * ld] = sm[c * (NP + 1) + r];
    }
}

// Ticket of the single-pass tree: returns true if this CTA is the second (last)
// arriver at node p and must run it.  Writers fence their global stores first.
__device__ __forceinline__ bool ticket(int *counters, int p, int *flag_smem) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int old = atomicAdd(counters + p, 1);
        if (old == 1) counters[p] = 0;        // both arrived: reset for the next call
        *flag_smem = old;
    }
    __syncthreads();
    const bool last = (*flag_smem == 1);
    if (last) __threadfence();
    return last;
}

}  // namespace tsqr
