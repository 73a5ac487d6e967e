// Blocked compact-WY engine of the B200 TSQR path (sm_100a).  Product code.
//
// A "tile" is an S x NP fp64 block in shared memory, column-major with leading
// dimension ld (ld = 2 mod 16: conflict-free DMMA fragment loads).  Its columns
// are processed in panels of 8 (DMMA m8n8k4 granularity):
//
//  * panel_qr   one warp factors the panel (8 columns x the active rows) in
//               registers with unblocked Householder steps whose reductions are
//               warp shuffles only (Alg. QR:qnxn / DGEQR2 order, reflector by
//               reflector); it writes the panel's Y (unit diagonal, zeros above)
//               to Ys and taus/betas;
//  * build_t    T of the panel from its Gram matrix G = Y^T Y (one DMMA per 4
//               rows) and the recurrence of Alg. YT:scaled in the
//               LAPACK sign (reading R3): H_0...H_7 = I - Y T Y^T;
//  * wy_update  C <- (I - Y T^T Y^T) C (kTrans, applying Q^T) or
//               C <- (I - Y T Y^T) C (applying Q), as W = Y^T C, W <- T^(T) W,
//               C -= Y W on FP64 DMMA; each warp handles its own 8-column blocks
//               of C, so no cross-warp reduction is needed.
//
// Rows: the active rows of a panel are given as a list of 8-row blocks: a
// dense tile uses blocks p.. (rows below the panel's first pivot), a
// structured node [R_a; R_b] (Alg. QR:qnxn, eq. fact_2rs) uses block p of R_a
// and blocks 0..p of R_b, so the triangular zeros are never touched.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsqr {
namespace wy {

// D += A B for one 8x8x4 fp64 MMA (SASS DMMA.8x8x4).  Fragments (lane i):
// A[i/4][i%4], B[k=i%4][n=i/4], C/D[i/4][2(i%4)+{0,1}].
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double rcp_nr(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}

// dlarfg scalars (readings R1/R2): beta = -sign(alpha) N, N = sqrt(alpha^2 +
// sigma2), tau = 1 + |alpha|/N, scale = 1/(alpha - beta); sigma2 == 0 -> H = I.
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

// dlarfg's rescaling (LAPACK scales x by 1/safmin while |beta| < safmin; reading
// R23).  The unscaled step forms sigma^2 = sum x_i^2 and the dots x^T a in plain
// fp64 and takes 1/sqrt and 1/x from flush-to-zero MUFU seeds, so it needs
// y = alpha^2 + sigma^2 inside [2^-900, 2^900]: no square or dot under- or
// overflows there (entries of A around 1e-160 or 1e+155 leave it).  Outside it
// (a warp- or block-uniform branch, never taken on ordinary data) the step is
// redone on s x, s = 2^-e a power of two with s max(|alpha|, |x_i|) in [0.5, 1):
// the scalars of the scaled column are (s beta, tau, scale / s), so the caller
// keeps its formulas with
//     w = rj + scale_s d_s      (d_s = (s x)^T a: the dot recomputed on s x),
//     u = tau (s scale_s) w,    v = (s scale_s) x,    beta = beta_s / s.
__device__ __forceinline__ bool house_unsafe(double alpha, double s2) {
#ifdef TSQR_NO_RESCALE            // measurement variant only: the slow path compiled out
    return false;
#else
    const double y = fma(alpha, alpha, s2);
    return !(y >= 0x1p-900 && y <= 0x1p+900);
#endif
}
// s = 2^-e with s mx in [0.5, 1); 1 for mx = 0, inf or NaN (nothing to rescale);
// e clamped to [-1000, 1000] so that s and 1/s stay finite (a subnormal mx then
// lands near 2^-74, far inside the safe range)
__device__ __forceinline__ double pow2_scale(double mx) {
    if (!(mx > 0.0) || isinf(mx)) return 1.0;
    const int e = max(-1000, min(1000, ilogb(mx) + 1));
    return ldexp(1.0, -e);
}

// Active 8-row blocks of panel p: dense (blocks p .. nrb-1) or structured node
// (the pivot block piv holding row block p of R_a, then blocks na .. na+p of R_b).
struct Rows {
    int p, nrb, na, piv;      // na < 0: dense
    __device__ int count() const { return na < 0 ? nrb - p : p + 2; }
    __device__ int block(int k) const { return na < 0 ? p + k : (k == 0 ? piv : na + k - 1); }
};

// ------------------------------------------------------------------ panel QR
// The Householder column steps of one panel on KM register blocks, branch-free:
// blocks beyond the active count hold zeros and stay zero (x = 0 there).
//
// Gs (if not null) receives the panel's Gram entries G(l, jj) = y_l^T y_jj for
// l < jj (row-major 8x8): with y_c = (0.., 1, scl_c x_c) and d_l = x_jj^T x_l
// over the rows below pivot jj (the dot this step computes anyway),
// G(l, jj) = scl_l (x_l[jj] + scl_jj d_l).
template <int KM>
__device__ __forceinline__ void panel_steps(double (*pv)[2], int p, int n, double *taus, double *betas,
                                            double &scl, double *Gs) {
    const int lane = threadIdx.x & 31, cl = lane >> 2, q = lane & 3;
    const int col = 8 * p + cl;
    const int jend = min(8, n - 8 * p);
#pragma unroll 1
    for (int jj = 0; jj < jend; ++jj) {                      // rolled: keeps the loop in the I-cache
        const int src = 4 * jj + q;                          // owner of column 8p + jj, same rows
        // rows <= pivot of the pivot block are not part of the reflector's tail
        const bool m0 = 2 * q > jj, m1 = 2 * q + 1 > jj;
        double x[KM][2];
#pragma unroll
        for (int k = 0; k < KM; ++k) {
            x[k][0] = __shfl_sync(0xffffffffu, pv[k][0], src);
            x[k][1] = __shfl_sync(0xffffffffu, pv[k][1], src);
        }
        x[0][0] = m0 ? x[0][0] : 0.0;
        x[0][1] = m1 ? x[0][1] : 0.0;
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
        for (int k = 0; k < KM; k += 2) {
            d0 = fma(x[k][0], pv[k][0], d0);
            d1 = fma(x[k][1], pv[k][1], d1);
            if (k + 1 < KM) {
                d2 = fma(x[k + 1][0], pv[k + 1][0], d2);
                d3 = fma(x[k + 1][1], pv[k + 1][1], d3);
            }
        }
        double d = (d0 + d1) + (d2 + d3);
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        d += __shfl_xor_sync(0xffffffffu, d, 2);             // x^T A(:, col)
        const double pj = (jj & 1) ? pv[0][1] : pv[0][0];
        const double rj = __shfl_sync(0xffffffffu, pj, 4 * cl + (jj >> 1));   // A(8p + jj, col)
        const double sig2 = __shfl_sync(0xffffffffu, d, 4 * jj);
        const double alpha = __shfl_sync(0xffffffffu, rj, 4 * jj);
        House h = householder(alpha, sig2);
        double sx = h.scale;                                 // the scale that multiplies the unscaled x
        if (house_unsafe(alpha, sig2)) {                     // warp-uniform; rescaled step (R23)
            double mx = fabs(alpha);
#pragma unroll
            for (int k = 0; k < KM; ++k) mx = fmax(mx, fmax(fabs(x[k][0]), fabs(x[k][1])));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const double sc = pow2_scale(mx);
            double e0 = 0.0, e1 = 0.0;
#pragma unroll
            for (int k = 0; k < KM; ++k) {
                e0 = fma(sc * x[k][0], pv[k][0], e0);
                e1 = fma(sc * x[k][1], pv[k][1], e1);
            }
            d = e0 + e1;
            d += __shfl_xor_sync(0xffffffffu, d, 1);
            d += __shfl_xor_sync(0xffffffffu, d, 2);
            h = householder(sc * alpha, sc * __shfl_sync(0xffffffffu, d, 4 * jj));   // (s x)^T (s x)
            sx = h.scale * sc;
            h.beta = h.beta / sc;
        }
        const double w = fma(d, h.scale, rj);                // v^T A(:, col)
        const double u = (cl > jj && col < n) ? h.tau * sx * w : 0.0;
#pragma unroll
        for (int k = 0; k < KM; ++k) {
            pv[k][0] = fma(-x[k][0], u, pv[k][0]);
            pv[k][1] = fma(-x[k][1], u, pv[k][1]);
        }
        const double dr = (q == (jj >> 1)) ? (alpha - h.beta) * u : 0.0;   // A(j, col) -= tau w
        if (jj & 1) pv[0][1] -= dr;
        else pv[0][0] -= dr;
        if (Gs != nullptr && q == 0 && cl < jj) Gs[cl * 8 + jj] = scl * fma(h.scale, d, rj);
        scl = (cl == jj) ? sx : scl;
        if (lane == 0) {
            taus[8 * p + jj] = h.tau;
            betas[8 * p + jj] = h.beta;
        }
    }
}

// Factor columns 8p .. 8p+7 (those < n) of the tile over the active rows.
// Lane i = 4 cl + q holds column 8p + cl, rows 8 block(k) + 2q + {0,1}.
// On exit the tile holds R (rows <= pivot) and the reflector entries v (below)
// in place; Ys (ld ldy) holds Y of the panel (unit diagonal, zeros above,
// zeros outside the active rows); taus[8p..], betas[8p..] are set.
template <int KMAX>
__device__ __forceinline__ void panel_qr(double *tile, int ld, int n, const Rows &rows, double *Ys, int ldy,
                                         double *taus, double *betas, double *Gs = nullptr) {
    const int lane = threadIdx.x & 31, cl = lane >> 2, q = lane & 3;
    const int p = rows.p, cnt = rows.count();
    const int col = 8 * p + cl;
    double pv[KMAX][2];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        pv[k][0] = pv[k][1] = 0.0;
        if (k < cnt) {
            const double2 v = *reinterpret_cast<const double2 *>(tile + col * ld + 8 * rows.block(k) + 2 * q);
            pv[k][0] = v.x;
            pv[k][1] = v.y;
        }
    }
    double scl = 0.0;
    if (Gs != nullptr) {
        Gs[lane] = 0.0;
        Gs[lane + 32] = 0.0;
        __syncwarp();
    }
    constexpr int KH = (KMAX + 1) / 2;
    if (KH < KMAX && cnt <= KH) panel_steps<KH>(pv, p, n, taus, betas, scl, Gs);
    else panel_steps<KMAX>(pv, p, n, taus, betas, scl, Gs);
    __syncwarp();
    // the pivot column of each reflector becomes (beta, v = scale * x): rows > pivot
    if (col < n) {
        const double be = betas[col];
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (k < cnt) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    if (k == 0) {
                        const int r = 2 * q + e;              // row 8p + r of the pivot block
                        pv[0][e] = r > cl ? pv[0][e] * scl : (r == cl ? be : pv[0][e]);
                    } else {
                        pv[k][e] *= scl;
                    }
                }
            }
    }
    // back to the tile, and the panel's Y (unit lower, zeros above) to Ys
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
        if (k < cnt) {
            const int rb = rows.block(k);
            *reinterpret_cast<double2 *>(tile + col * ld + 8 * rb + 2 * q) = make_double2(pv[k][0], pv[k][1]);
            double y0 = pv[k][0], y1 = pv[k][1];
            if (k == 0) {
                const int r0 = 2 * q, r1 = 2 * q + 1;
                y0 = r0 > cl ? y0 : (r0 == cl ? 1.0 : 0.0);
                y1 = r1 > cl ? y1 : (r1 == cl ? 1.0 : 0.0);
            }
            if (col >= n) y0 = y1 = 0.0;
            *reinterpret_cast<double2 *>(Ys + cl * ldy + 8 * rb + 2 * q) = make_double2(y0, y1);
        }
}

// ------------------------------------------------------------------ T factor
// T (8x8, row-major Ts[r*8 + c]) of the panel whose Y is in Ys (rows given by
// `rows`) and taus t[0..8): G = Y^T Y by DMMA, then for c = 1..7, row r < c:
// T(r,c) = -tau_c sum_{l=r}^{c-1} T(r,l) G(l,c), T(c,c) = tau_c.  One warp.
__device__ __forceinline__ void build_t(const double *Ys, int ldy, const Rows &rows, const double *t, double *Gs,
                                        double *Ts) {
    const int lane = threadIdx.x & 31;
    double g0 = 0.0, g1 = 0.0;
    const int cnt = rows.count();
    for (int k = 0; k < cnt; ++k) {
        const int rb = rows.block(k);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const double a = Ys[(lane >> 2) * ldy + 8 * rb + 4 * e + (lane & 3)];
            dmma(g0, g1, a, a);
        }
    }
    Gs[(lane >> 2) * 8 + 2 * (lane & 3)] = g0;
    Gs[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = g1;
    __syncwarp();
    if (lane < 8) {
        const int r = lane;
        double row[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) row[c] = 0.0;
        row[r < 8 ? r : 0] = t[r];
#pragma unroll
        for (int c = 1; c < 8; ++c) {
            if (r < c) {
                double s = 0.0;
#pragma unroll
                for (int l = 0; l < c; ++l)
                    if (l >= r) s = fma(row[l], Gs[l * 8 + c], s);
                row[c] = -t[c] * s;
            }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) Ts[r * 8 + c] = row[c];
    }
    __syncwarp();
}

// T from the Gram entries panel_qr left in Gs (row-major, G(l, c) for l < c),
// same recurrence as build_t; lanes r < 8 own row r of T (static indexing:
// T(r, l) = 0 for l < r, so the sum may run over all l < c).
__device__ __forceinline__ void build_t_gram(const double *Gs, const double *t, double *Ts) {
    const int r = threadIdx.x & 31;
    if (r < 8) {
        double row[8];
        const double tr = t[r];
#pragma unroll
        for (int c = 0; c < 8; ++c) row[c] = (c == r) ? tr : 0.0;
#pragma unroll
        for (int c = 1; c < 8; ++c) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < c; ++l) s = fma(row[l], Gs[l * 8 + c], s);
            if (r < c) row[c] = -t[c] * s;
        }
#pragma unroll
        for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2 *>(Ts + r * 8 + c) = make_double2(row[c], row[c + 1]);
    }
    __syncwarp();
}

// ------------------------------------------------------------------ update
// For the calling warp's column block cb of C (columns 8cb..8cb+7, ld ldc):
// C <- (I - Y op(T) Y^T) C over the active rows, op(T) = T^T (kTrans: Q^T) or T.
// Wb: 8x8 per-warp scratch (row-major, stride 9).
template <bool kTrans>
__device__ __forceinline__ void wy_update_block(double *C, int ldc, int cb, const double *Ys, int ldy,
                                                const Rows &rows, const double *Ts, double *Wb) {
    const int lane = threadIdx.x & 31, lq = lane & 3, l4 = lane >> 2;
    const int cnt = rows.count();
    // W = Y^T C  (8 reflectors x 8 columns)
    double w0 = 0.0, w1 = 0.0;
    const double *cc = C + (8 * cb + l4) * ldc;
    for (int k = 0; k < cnt; ++k) {
        const int rb = rows.block(k);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int r = 8 * rb + 4 * e + lq;
            dmma(w0, w1, Ys[l4 * ldy + r], cc[r]);
        }
    }
    Wb[l4 * 9 + 2 * lq] = w0;
    Wb[l4 * 9 + 2 * lq + 1] = w1;
    __syncwarp();
    // W' = op(T) W
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int kk = 4 * e + lq;
        const double a = kTrans ? Ts[kk * 8 + l4] : Ts[l4 * 8 + kk];
        dmma(v0, v1, a, Wb[kk * 9 + l4]);
    }
    __syncwarp();
    Wb[l4 * 9 + 2 * lq] = v0;
    Wb[l4 * 9 + 2 * lq + 1] = v1;
    __syncwarp();
    // C -= Y W'   as  C^T -= W'^T Y^T  (accumulator = C^T block: lane holds
    // column 8cb + l4, rows 8rb + 2lq + {0,1})
    const double a0 = -Wb[(lq) * 9 + l4], a1 = -Wb[(4 + lq) * 9 + l4];
    double *cw = C + (8 * cb + l4) * ldc;
    for (int k = 0; k < cnt; ++k) {
        const int rb = rows.block(k);
        double2 c2 = *reinterpret_cast<const double2 *>(cw + 8 * rb + 2 * lq);
        dmma(c2.x, c2.y, a0, Ys[(lq)*ldy + 8 * rb + l4]);
        dmma(c2.x, c2.y, a1, Ys[(4 + lq) * ldy + 8 * rb + l4]);
        *reinterpret_cast<double2 *>(cw + 8 * rb + 2 * lq) = c2;
    }
    __syncwarp();
}

// wy_update_block on nb <= NB column blocks cb0, cb0+1, .. at once (one warp):
// the Y fragments are loaded once for all blocks and the NB DMMA chains
// interleave.  Wb: NB x 72 scratch.  nb is warp-uniform.
template <bool kTrans, int NB>
__device__ __forceinline__ void wy_update_multi(double *C, int ldc, int cb0, int nb, const double *Ys, int ldy,
                                                const Rows &rows, const double *Ts, double *Wb) {
    const int lane = threadIdx.x & 31, lq = lane & 3, l4 = lane >> 2;
    const int cnt = rows.count();
    double w[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) w[b][0] = w[b][1] = 0.0;
    const double *cc = C + (8 * cb0 + l4) * ldc;
    for (int k = 0; k < cnt; ++k) {
        const int rb = rows.block(k);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int r = 8 * rb + 4 * e + lq;
            const double a = Ys[l4 * ldy + r];
#pragma unroll
            for (int b = 0; b < NB; ++b)
                if (b < nb) dmma(w[b][0], w[b][1], a, cc[8 * b * ldc + r]);
        }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        Wb[72 * b + l4 * 9 + 2 * lq] = w[b][0];
        Wb[72 * b + l4 * 9 + 2 * lq + 1] = w[b][1];
    }
    __syncwarp();
    double a2[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int kk = 4 * e + lq;
        a2[e] = kTrans ? Ts[kk * 8 + l4] : Ts[l4 * 8 + kk];
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        w[b][0] = w[b][1] = 0.0;
        if (b < nb) {
#pragma unroll
            for (int e = 0; e < 2; ++e) dmma(w[b][0], w[b][1], a2[e], Wb[72 * b + (4 * e + lq) * 9 + l4]);
        }
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        Wb[72 * b + l4 * 9 + 2 * lq] = w[b][0];
        Wb[72 * b + l4 * 9 + 2 * lq + 1] = w[b][1];
    }
    __syncwarp();
    double a0[NB], a1[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        a0[b] = -Wb[72 * b + lq * 9 + l4];
        a1[b] = -Wb[72 * b + (4 + lq) * 9 + l4];
    }
    double *cw = C + (8 * cb0 + l4) * ldc;
    for (int k = 0; k < cnt; ++k) {
        const int rb = rows.block(k);
        const double y0 = Ys[lq * ldy + 8 * rb + l4], y1 = Ys[(4 + lq) * ldy + 8 * rb + l4];
#pragma unroll
        for (int b = 0; b < NB; ++b)
            if (b < nb) {
                double2 c2 = *reinterpret_cast<const double2 *>(cw + 8 * b * ldc + 8 * rb + 2 * lq);
                dmma(c2.x, c2.y, a0[b], y0);
                dmma(c2.x, c2.y, a1[b], y1);
                *reinterpret_cast<double2 *>(cw + 8 * b * ldc + 8 * rb + 2 * lq) = c2;
            }
    }
    __syncwarp();
}

}  // namespace wy
}  // namespace tsqr
