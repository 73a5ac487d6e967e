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
// global (rows x ncols, ld) -> smem (cap_rows x cap_cols, sld), zero padded.
template <bool kCG>
__device__ __forceinline__ void stage_in(double *sm, int sld, const double *g, int64_t ldg,
                                         int rows, int ncols, int cap_rows, int cap_cols) {
    for (int c = 0; c < cap_cols; ++c) {
        const double *gc = g + (int64_t)c * ldg;
        for (int r = threadIdx.x; r < cap_rows; r += kThreads) {
            double v = 0.0;
            if (c < ncols && r < rows) v = kCG ? __ldcg(gc + r) : gc[r];
            sm[c * sld + r] = v;
        }
    }
}

__device__ __forceinline__ void stage_out(const double *sm, int sld, double *g, int64_t ldg,
                                          int rows, int ncols) {
    for (int c = 0; c < ncols; ++c) {
        double *gc = g + (int64_t)c * ldg;
        for (int r = threadIdx.x; r < rows; r += kThreads) gc[r] = sm[c * sld + r];
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
// beta = -sign(alpha) sqrt(alpha^2 + sigma2), tau = (beta - alpha)/beta,
// v = x / (alpha - beta) below the pivot.  sigma2 == 0 -> H = I.
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
        const double nrm = sqrt(fma(alpha, alpha, sigma2));
        h.beta = alpha >= 0.0 ? -nrm : nrm;
        const double d = alpha - h.beta;      // |alpha| + |beta|: no cancellation
        h.tau = -d / h.beta;                  // (beta - alpha) / beta
        h.scale = 1.0 / d;
    }
    return h;
}

// ============================================================== tile QR (a2)
// Unblocked Householder QR of the register tile a (rows x n, padded).  One
// __syncthreads per column: partial inner products of the pivot column with
// every column (its own one gives sigma^2 = ||x(j+1:)||^2) are reduced once;
// w = v^T A_t follows from them by a scale (v = x/(alpha-beta)).
// Smem: xs[S] (pivot column broadcast), red[2][kWarps][NP], rowj[2][NP], taus[NP].
template <class Lt>
__device__ void tile_qr(double (&a)[Lt::RT][Lt::CPL], int n, double *xs, double *red,
                        double *rowj, double *taus) {
    constexpr int RT = Lt::RT, CPL = Lt::CPL, NP = Lt::NP;
    const int w = Lt::warp(), l = Lt::lane(), rph = Lt::rph();
    for (int j = 0; j < n; ++j) {
        const int buf = j & 1;
        double *redb = red + buf * (kWarps * NP);
        double *rjb = rowj + buf * NP;
        const int cj = j >> 5;                       // register column of j (CPL = 2)
        const bool owner = (Lt::colbase() == (j & 31)) && (cj < CPL);
        // 1. broadcast the pivot column (rows > j) inside each warp
        __syncwarp();
        if (owner) {
#pragma unroll
            for (int i = 0; i < RT; ++i) {
                const int r = Lt::row(i);
                const double v = (cj == 0) ? a[i][0] : a[i][CPL - 1];
                xs[r] = r > j ? v : 0.0;
            }
        }
        __syncwarp();
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
        // row j of every column (needed for w = A(j,:) + x^T A / (alpha - beta))
        const int wj = j / Lt::RW, ij = (j % Lt::RW) / Lt::LPC, pj = (j % Lt::RW) % Lt::LPC;
        if (w == wj && rph == pj) {
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) {
                double v = 0.0;
#pragma unroll
                for (int i = 0; i < RT; ++i) v = (i == ij) ? a[i][cc] : v;
                rjb[Lt::col(cc)] = v;
            }
        }
        __syncthreads();
        // 3. reduce across warps (same order in every thread: identical scalars)
        double sig2 = 0.0;
#pragma unroll
        for (int q = 0; q < kWarps; ++q) sig2 += redb[q * NP + j];
        const double alpha = rjb[j];
        const House h = householder(alpha, sig2);
        double u[CPL], ru[CPL];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
            const int c = Lt::col(cc);
            double P = 0.0;
#pragma unroll
            for (int q = 0; q < kWarps; ++q) P += redb[q * NP + c];
            const double wc = fma(P, h.scale, rjb[c]);   // v^T A(:, c)
            const bool trail = (c > j) && (c < n);
            u[cc] = trail ? h.tau * h.scale * wc : 0.0;  // A(r,c) -= x_r * u   (r > j)
            ru[cc] = trail ? h.tau * wc : 0.0;            // A(j,c) -= tau * w_c
        }
        // 4. rank-1 update of the trailing columns (x re-read: saves RT registers)
        double x[RT];
        load_rowvec<Lt>(xs, x);
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
            for (int i = 0; i < RT; ++i) a[i][cc] = fma(-x[i], u[cc], a[i][cc]);
        if (w == wj && rph == pj) {
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
                for (int i = 0; i < RT; ++i)
                    if (i == ij) a[i][cc] -= ru[cc];
        }
        // 5. the pivot column becomes (beta, v) in place
        if (owner) {
#pragma unroll
            for (int i = 0; i < RT; ++i) {
                const int r = Lt::row(i);
                double &aij = (cj == 0) ? a[i][0] : a[i][CPL - 1];
                if (r > j) aij = x[i] * h.scale;
                else if (r == j) aij = h.beta;
            }
        }
        if (threadIdx.x == 0) taus[j] = h.tau;
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
            double P = 0.0;
#pragma unroll
            for (int q = 0; q < kWarps; ++q) P += redb[q * NP + Lt::col(cc)];
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
        double sig2 = 0.0;
#pragma unroll
        for (int q = 0; q < kWarps; ++q) sig2 += redb[q * NP + j];
        const House h = householder(alpha, sig2);
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
            const int c = Lt::col(cc);
            double P = 0.0;
#pragma unroll
            for (int q = 0; q < kWarps; ++q) P += redb[q * NP + c];
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
            double P = 0.0;
#pragma unroll
            for (int q = 0; q < kWarps; ++q) P += redb[q * NP + c];
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
// (ld) and smem (ld NP+1, zero elsewhere).
template <int NP, bool kCG>
__device__ __forceinline__ void load_upper(double *sm, const double *g, int64_t ld, int n) {
    for (int e = threadIdx.x; e < NP * NP; e += kThreads) {
        const int r = e % NP, c = e / NP;
        double v = 0.0;
        if (r <= c && c < n) v = kCG ? __ldcg(g + r + (int64_t)c * ld) : g[r + (int64_t)c * ld];
        sm[c * (NP + 1) + r] = v;
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
    for (int e = threadIdx.x; e < NP * NP; e += kThreads) {
        const int r = e % NP, c = e / NP;
        double v = 0.0;
        if (r < n && c < kc) v = kCG ? __ldcg(g + r + (int64_t)c * ld) : g[r + (int64_t)c * ld];
        sm[c * (NP + 1) + r] = v;
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
