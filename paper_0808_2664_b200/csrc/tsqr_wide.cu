// Wide-n engine of the B200 TSQR path (64 < n <= 256, config 3's n = 200).  Product code.
//
// For wide n the running R of a flat chain (n x n, 320 KB at n = 200) does not
// fit on chip, so every leaf is factored by a blocked compact-WY Householder QR
// of the whole tile (the paper's leaf, DGEQR2 order, Alg. TSQR:par line 1
// P:1679-1680; compact WY Alg. YT:scaled P:2007-2028) by one CTA, with the tile
// in global memory (L2-resident):
//   panel p (8 columns): loaded row-split over the 8 warps (each warp a fixed
//       range of up to 288 logical rows, DMMA-fragment layout), Householder
//       steps with warp-shuffle + one __syncthreads cross-warp reduction per
//       column, written back (R above, v below the diagonal), T built;
//   trailing update, column-split: warp w owns column blocks w, w+8, ...; it
//       streams W^T = C^T Y over the rows (FP64 DMMA), W'^T = W^T T and
//       C -= Y W' -- no cross-warp reduction at all.
// A tree node (Alg. QR:qnxn, [R_a; R_b], eq. fact_2rs) is the same kernel on
// the stacked logical rows [R_a rows 0..n-1; R_b rows 0..n-1] with masks: R_a
// row i holds column c only for i <= c, R_b row r only for r <= c; everything
// else reads as zero and is never written.  The zeros are exact, so this is
// the structured combine itself (same beta, tau, v), touching only the
// upper triangles: R lands in R_a's, the node's Y1 in R_b's.
// k_wide_apply applies the stored reflectors (Q^T: panels forward with T^T;
// Q: backward with T) to C rows mapped the same way, column-split, no barriers.
#include "tsqr_kernels.h"

#include <cstdint>
#include "wy.cuh"
#include "chunk.cuh"

#include <cstdlib>
#include <type_traits>

namespace tsqr {
namespace wide {

using wy::dmma;
using wy::House;
constexpr unsigned FULL = 0xffffffffu;
constexpr int NW = 8, NT = 256, KMW = 36, RW = 8 * KMW;   // rows per warp (logical)
constexpr int MAXR = NW * RW;                               // 2304 logical rows

// branch-free dlarfg scalars (readings R1/R2/R19): chunk::house_bf (one
// third-order correction per MUFU seed)
__device__ __forceinline__ House house(double alpha, double s2) { return chunk::house_bf(alpha, s2); }

// A problem: logical rows [0, hA) -> segment A rows (the first nA exist),
// [hA, hA + hB) -> segment B rows.  A node pads its R_a segment to hA = NP
// rows so that R_b starts on an 8-row block; the padding rows never exist.
struct Prob {
    double *a;       // segment A (ld lda)
    double *b;       // segment B (ld ldb), may be null when hB = 0
    int64_t lda, ldb;
    int hA, hB, nA;
    int node;        // 1: [R_a; R_b] upper-triangle masks
};

__device__ __forceinline__ double *rowp(const Prob &P, int r, int c) {
    return r < P.hA ? P.a + r + (int64_t)c * P.lda : P.b + (r - P.hA) + (int64_t)c * P.ldb;
}
__device__ __forceinline__ bool row_exists(const Prob &P, int r) {
    return r < P.hA ? r < P.nA : r - P.hA < P.hB;
}
// Is logical element (r, c) part of the problem's matrix (else it reads as 0
// and is never written)?
__device__ __forceinline__ bool present(const Prob &P, int r, int c, int n) {
    if (c >= n || !row_exists(P, r)) return false;
    if (!P.node) return true;
    return r < P.hA ? r <= c : (r - P.hA) <= c;
}
// Y(r, j) of reflector j (pivot = logical row j) from the stored factor.
__device__ __forceinline__ double yval(const Prob &P, int r, int j, int n) {
    if (j >= n || r < j) return 0.0;
    if (r == j) return 1.0;
    return present(P, r, j, n) ? *rowp(P, r, j) : 0.0;
}

struct Smem {
    double part[2][NW][9];     // per-step partial dots (8 columns) + sigma^2, double-buffered
    double piv[2][8];          // the pivot row's panel values
    double Gs[64], Ts[64], t8[8];
    double xs[NW][2][RW];      // per-warp pivot-column broadcast (double-buffered)
};

// One problem: blocked Householder QR in place; tau[n], tcache[npan][64].
__device__ void wide_qr(const Prob &P, int n, double *tau, double *tcache, Smem &S) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int H = P.hA + P.hB;
    const int npan = (n + 7) / 8;
    const int rbase = warp * RW;
    for (int p = 0; p < npan; ++p) {
        const int c = 8 * p + l4;
        // ---- load the panel (this warp's logical rows)
        double a[KMW][2];
#pragma unroll
        for (int k = 0; k < KMW; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = rbase + 8 * k + 2 * q + e;
                a[k][e] = present(P, r, c, n) ? *rowp(P, r, c) : 0.0;
            }
        double *xs0 = S.xs[warp][0], *xs1 = S.xs[warp][1];
        if (l4 == 0) {
#pragma unroll
            for (int k = 0; k < KMW; ++k)
                *reinterpret_cast<double2 *>(xs0 + 8 * k + 2 * q) = make_double2(a[k][0], a[k][1]);
        }
        __syncwarp();
        const int jn = min(8, n - 8 * p);
#pragma unroll 1
        for (int jj = 0; jj < jn; ++jj) {
            const int j = 8 * p + jj;                         // pivot = logical row j
            const int par = jj & 1;
            const double *xr = par ? xs1 : xs0;
            double d[4] = {0.0, 0.0, 0.0, 0.0}, s[4] = {0.0, 0.0, 0.0, 0.0};
            double pv = 0.0;                                  // this lane's entry of the pivot row
            bool haspiv = false;
#pragma unroll
            for (int k = 0; k < KMW; ++k) {
                const double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                const int r = rbase + 8 * k + 2 * q;
                const double x0 = r > j ? xv.x : 0.0, x1 = r + 1 > j ? xv.y : 0.0;
                d[k & 3] = fma(x0, a[k][0], d[k & 3]);
                d[(k + 2) & 3] = fma(x1, a[k][1], d[(k + 2) & 3]);
                s[k & 3] = fma(x0, x0, s[k & 3]);
                s[(k + 2) & 3] = fma(x1, x1, s[(k + 2) & 3]);
                if (r == j) { pv = a[k][0]; haspiv = true; }
                if (r + 1 == j) { pv = a[k][1]; haspiv = true; }
            }
            double dd = (d[0] + d[1]) + (d[2] + d[3]), s2 = (s[0] + s[1]) + (s[2] + s[3]);
            dd += __shfl_xor_sync(FULL, dd, 1);
            s2 += __shfl_xor_sync(FULL, s2, 1);
            dd += __shfl_xor_sync(FULL, dd, 2);
            s2 += __shfl_xor_sync(FULL, s2, 2);
            if (q == 0) S.part[par][warp][l4] = dd;
            if (lane == 0) S.part[par][warp][8] = s2;
            if (haspiv) S.piv[par][l4] = pv;
            __syncthreads();
            dd = 0.0;
            s2 = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                dd += S.part[par][w][l4];
                s2 += S.part[par][w][8];
            }
            const double rj = S.piv[par][l4], alpha = S.piv[par][jj];
            House h = house(alpha, s2);
            double sc = 1.0;
            double sx = h.scale;
            if (wy::house_unsafe(alpha, s2)) {                      // block-uniform, rescaled step (R23)
                double mx = fabs(alpha);
#pragma unroll
                for (int k = 0; k < KMW; ++k) {
                    const double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                    const int r = rbase + 8 * k + 2 * q;
                    mx = fmax(mx, fmax(r > j ? fabs(xv.x) : 0.0, r + 1 > j ? fabs(xv.y) : 0.0));
                }
                mx = fmax(mx, __shfl_xor_sync(FULL, mx, 1));
                mx = fmax(mx, __shfl_xor_sync(FULL, mx, 2));
                // part[par ^ 1] is free: its last readers (step jj - 1) are past this step's barrier
                if (lane == 0) S.part[par ^ 1][warp][8] = mx;
                __syncthreads();
                for (int w = 0; w < NW; ++w) mx = fmax(mx, S.part[par ^ 1][w][8]);
                sc = wy::pow2_scale(mx);
                __syncthreads();
                double e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0;
#pragma unroll
                for (int k = 0; k < KMW; ++k) {
                    const double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                    const int r = rbase + 8 * k + 2 * q;
                    const double x0 = r > j ? sc * xv.x : 0.0, x1 = r + 1 > j ? sc * xv.y : 0.0;
                    e0 = fma(x0, a[k][0], e0);
                    e1 = fma(x1, a[k][1], e1);
                    f0 = fma(x0, x0, f0);
                    f1 = fma(x1, x1, f1);
                }
                dd = e0 + e1;
                s2 = f0 + f1;
                dd += __shfl_xor_sync(FULL, dd, 1);
                s2 += __shfl_xor_sync(FULL, s2, 1);
                dd += __shfl_xor_sync(FULL, dd, 2);
                s2 += __shfl_xor_sync(FULL, s2, 2);
                if (q == 0) S.part[par ^ 1][warp][l4] = dd;
                if (lane == 0) S.part[par ^ 1][warp][8] = s2;
                __syncthreads();
                dd = 0.0;
                s2 = 0.0;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    dd += S.part[par ^ 1][w][l4];
                    s2 += S.part[par ^ 1][w][8];
                }
                h = house(sc * alpha, s2);
                h.beta = h.beta / sc;
                sx = h.scale * sc;
            }
            const double wv = fma(h.scale, dd, rj);
            const double u = (l4 > jj) ? h.tau * sx * wv : (l4 == jj ? 1.0 : 0.0);
            const double g = (l4 == jj) ? sx : 0.0;             // pivot column: v = scale x exactly
            const double pnew = (l4 > jj) ? fma(-h.tau, wv, rj) : (l4 == jj ? h.beta : rj);
            double *xw = par ? xs0 : xs1;
#pragma unroll
            for (int k = 0; k < KMW; ++k) {
                const double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                const int r = rbase + 8 * k + 2 * q;
                const double x0 = r > j ? xv.x : 0.0, x1 = r + 1 > j ? xv.y : 0.0;
                double a0 = fma(g, x0, fma(-u, x0, a[k][0])), a1 = fma(g, x1, fma(-u, x1, a[k][1]));
                a0 = (r == j) ? pnew : a0;
                a1 = (r + 1 == j) ? pnew : a1;
                a[k][0] = a0;
                a[k][1] = a1;
                if (l4 == jj + 1) *reinterpret_cast<double2 *>(xw + 8 * k + 2 * q) = make_double2(a0, a1);
            }
            if (warp == 0 && q == 0 && l4 < jj) S.Gs[l4 * 8 + jj] = fma(h.scale, dd, rj);
            if (threadIdx.x == 0) S.t8[jj] = h.tau;
            __syncwarp();
        }
        if (warp == 0) {                         // padding columns past n: identity steps
            for (int c2 = jn; c2 < 8; ++c2) {
                if (q == 0 && l4 < c2) S.Gs[l4 * 8 + c2] = 0.0;
                if (lane == 0) S.t8[c2] = 0.0;
            }
        }
        // ---- write the panel back; T; taus
#pragma unroll
        for (int k = 0; k < KMW; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = rbase + 8 * k + 2 * q + e;
                if (present(P, r, c, n)) *rowp(P, r, c) = a[k][e];
            }
        __syncthreads();
        if (warp == 0) {
            const int rr = lane & 7;
            double row[8];
            const double tr = S.t8[rr];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) row[cc] = (cc == rr) ? tr : 0.0;
#pragma unroll
            for (int cc = 1; cc < 8; ++cc) {
                double sacc = 0.0;
#pragma unroll
                for (int l = 0; l < cc; ++l) sacc = fma(row[l], S.Gs[l * 8 + cc], sacc);
                row[cc] = (rr < cc) ? -S.t8[cc] * sacc : row[cc];
            }
            if (lane < 8) {
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    S.Ts[lane * 8 + cc] = row[cc];
                    tcache[p * 64 + lane * 8 + cc] = row[cc];
                }
                if (8 * p + lane < n) tau[8 * p + lane] = S.t8[lane];
            }
        }
        __syncthreads();
        // ---- trailing update, column-split over the warps
        const double tb0 = S.Ts[(2 * q) * 8 + l4], tb1 = S.Ts[(2 * q + 1) * 8 + l4];
        const int rb0 = P.node ? 0 : p;                        // first logical row block touched
        const int nrb = (H + 7) / 8;
        for (int cb = p + 1 + warp; cb < npan; cb += NW) {
            const int col = 8 * cb + l4;
            double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
            for (int k = rb0; k < nrb; ++k) {
                if (P.node && !(k == p || (k >= P.hA / 8 && k - P.hA / 8 <= p))) continue;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int r = 8 * k + 2 * q + e;
                    const double cv = present(P, r, col, n) ? *rowp(P, r, col) : 0.0;
                    const double yv = yval(P, r, 8 * p + l4, n);
                    dmma(w0[k & 1], w1[k & 1], cv, yv);
                }
            }
            double p0 = 0.0, p1 = 0.0;
            dmma(p0, p1, w0[0] + w0[1], tb0);
            dmma(p0, p1, w1[0] + w1[1], tb1);
            for (int k = rb0; k < nrb; ++k) {
                if (P.node && !(k == p || (k >= P.hA / 8 && k - P.hA / 8 <= p))) continue;
                const int r0 = 8 * k + 2 * q;
                const bool ok0 = present(P, r0, col, n), ok1 = present(P, r0 + 1, col, n);
                double c0 = ok0 ? *rowp(P, r0, col) : 0.0, c1 = ok1 ? *rowp(P, r0 + 1, col) : 0.0;
                const double y0 = yval(P, 8 * k + l4, 8 * p + 2 * q, n), y1 = yval(P, 8 * k + l4, 8 * p + 2 * q + 1, n);
                dmma(c0, c1, -p0, y0);
                dmma(c0, c1, -p1, y1);
                if (ok0) *rowp(P, r0, col) = c0;
                if (ok1) *rowp(P, r0 + 1, col) = c1;
            }
        }
        __syncthreads();
    }
}

// Apply the problem's stored reflectors to C (rows mapped like the problem's,
// every element present): Q^T (kFwd, panels forward, T^T) or Q (backward, T).
template <bool kFwd>
__device__ void wide_apply(const Prob &P, const Prob &Cp, int n, int k, const double *tcache) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int H = P.hA + P.hB;
    const int npan = (n + 7) / 8;
    const int nrb = (H + 7) / 8;
    auto cptr = [&](int r, int col) -> double * {
        return r < Cp.hA ? Cp.a + r + (int64_t)col * Cp.lda : Cp.b + (r - Cp.hA) + (int64_t)col * Cp.ldb;
    };
    for (int cb = warp; cb < (k + 7) / 8; cb += NW) {
        const int col = 8 * cb + l4;
        const bool okc = col < k;
        for (int pp = 0; pp < npan; ++pp) {
            const int p = kFwd ? pp : npan - 1 - pp;
            const double *Tg = tcache + p * 64;
            const double tb0 = kFwd ? Tg[(2 * q) * 8 + l4] : Tg[l4 * 8 + 2 * q];
            const double tb1 = kFwd ? Tg[(2 * q + 1) * 8 + l4] : Tg[l4 * 8 + 2 * q + 1];
            const int rb0 = P.node ? 0 : p;
            double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
            for (int kk = rb0; kk < nrb; ++kk) {
                if (P.node && !(kk == p || (kk >= P.hA / 8 && kk - P.hA / 8 <= p))) continue;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int r = 8 * kk + 2 * q + e;
                    const double cv = (okc && row_exists(Cp, r)) ? *cptr(r, col) : 0.0;
                    dmma(w0[kk & 1], w1[kk & 1], cv, yval(P, r, 8 * p + l4, n));
                }
            }
            double p0 = 0.0, p1 = 0.0;
            dmma(p0, p1, w0[0] + w0[1], tb0);
            dmma(p0, p1, w1[0] + w1[1], tb1);
            for (int kk = rb0; kk < nrb; ++kk) {
                if (P.node && !(kk == p || (kk >= P.hA / 8 && kk - P.hA / 8 <= p))) continue;
                const int r0 = 8 * kk + 2 * q;
                const bool e0 = okc && row_exists(Cp, r0), e1 = okc && row_exists(Cp, r0 + 1);
                double c0 = e0 ? *cptr(r0, col) : 0.0, c1 = e1 ? *cptr(r0 + 1, col) : 0.0;
                dmma(c0, c1, -p0, yval(P, 8 * kk + l4, 8 * p + 2 * q, n));
                dmma(c0, c1, -p1, yval(P, 8 * kk + l4, 8 * p + 2 * q + 1, n));
                if (e0) *cptr(r0, col) = c0;
                if (e1) *cptr(r0 + 1, col) = c1;
            }
        }
    }
}


// 8-byte global -> shared copy (zero-filled when !ok)
__device__ __forceinline__ void cp_async8(double *sm, const double *g, bool ok) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0) : "memory");
}

// ------------------------------------------------------------------ leaves
// The leaf path (plain tiles, no masks): the panel's Y is staged in shared
// memory (row-major H x 8, zero-padded to a whole row block), so the column-
// split trailing update / apply streams only C from global memory, with 8 row
// blocks of loads in flight per lane.
constexpr int UNR = 8;

// a lane's row pair (r, r+1) of a C column, r even: one 16-byte access when the column
// pointer is 16-byte aligned (even tile starts and an even ldc make every pair aligned)
#ifdef TSQR_WIDE_L2KEEP
// variant: the row pairs of C carry an L2 evict_last policy (a tile's trailing columns are
// re-streamed once per panel pair; keep them in L2 against the other tiles' traffic)
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
#endif
__device__ __forceinline__ void ld_pair(double &x0, double &x1, const double *cp, bool okc, int r, int H) {
    if (okc && r + 1 < H && !(reinterpret_cast<uintptr_t>(cp) & 15)) {
#ifdef TSQR_WIDE_L2KEEP
        asm("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
            : "=d"(x0), "=d"(x1) : "l"(cp + r), "l"(l2_keep_policy()) : "memory");
#else
        const double2 v = *reinterpret_cast<const double2 *>(cp + r);
        x0 = v.x;
        x1 = v.y;
#endif
    } else {
        x0 = (okc && r < H) ? cp[r] : 0.0;
        x1 = (okc && r + 1 < H) ? cp[r + 1] : 0.0;
    }
}
__device__ __forceinline__ void st_pair(double *cp, bool okc, int r, int H, double x0, double x1) {
    if (okc && r + 1 < H && !(reinterpret_cast<uintptr_t>(cp) & 15)) {
#ifdef TSQR_WIDE_L2KEEP
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;"
                     :: "l"(cp + r), "d"(x0), "d"(x1), "l"(l2_keep_policy()) : "memory");
#else
        *reinterpret_cast<double2 *>(cp + r) = make_double2(x0, x1);
#endif
    } else {
        if (okc && r < H) cp[r] = x0;
        if (okc && r + 1 < H) cp[r + 1] = x1;
    }
}

// one group of U row blocks of this lane's column of C (rows 8k+2q+{0,1})
template <int U>
__device__ __forceinline__ void load_grp(double (&cv)[U][2], const double *cp, bool okc, int H, int k0) {
    const int q = threadIdx.x & 3;
#pragma unroll
    for (int u = 0; u < U; ++u) ld_pair(cv[u][0], cv[u][1], cp, okc, 8 * (k0 + u) + 2 * q, H);
}
template <int U>
__device__ __forceinline__ void w_grp(double (&w0)[2], double (&w1)[2], const double (&cv)[U][2], const double *Ys,
                                      int nrb, int k0) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (k0 + u < nrb) {
            const int r = 8 * (k0 + u) + 2 * q;
            dmma(w0[u & 1], w1[u & 1], cv[u][0], Ys[r * 8 + l4]);
            dmma(w0[u & 1], w1[u & 1], cv[u][1], Ys[(r + 1) * 8 + l4]);
        }
    }
}
template <int U>
__device__ __forceinline__ void upd_grp(double (&cv)[U][2], double *cp, bool okc, int H, const double *Ys, int nrb,
                                        int k0, double p0, double p1) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (k0 + u < nrb) {
            const double2 y = *reinterpret_cast<const double2 *>(Ys + (8 * (k0 + u) + l4) * 8 + 2 * q);
            dmma(cv[u][0], cv[u][1], -p0, y.x);
            dmma(cv[u][0], cv[u][1], -p1, y.y);
            const int r = 8 * (k0 + u) + 2 * q;
            st_pair(cp, okc, r, H, cv[u][0], cv[u][1]);
        }
    }
}

// C <- (I - Y T' Y^T) C on columns [c_lo, c_hi) and rows [8 rb0, H) of C
// (T' = T^T for Q^T, kFwd; T for Q), Y = Ys (rows >= 8 rb0 valid, zero past H).
// Both passes over the rows are software-pipelined: the next group of UNR row
// blocks is loaded while the current one is consumed.
template <bool kFwd>
__device__ __forceinline__ void apply_panel_cols(const double *Ys, const double *Tg, double *C, int64_t ldc, int H,
                                                 int rb0, int c_lo, int c_hi) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const double tb0 = kFwd ? Tg[(2 * q) * 8 + l4] : Tg[l4 * 8 + 2 * q];
    const double tb1 = kFwd ? Tg[(2 * q + 1) * 8 + l4] : Tg[l4 * 8 + 2 * q + 1];
    const int nrb = (H + 7) / 8;
    for (int cb = c_lo / 8 + warp; 8 * cb < c_hi; cb += NW) {
        const int col = 8 * cb + l4;
        const bool okc = col < c_hi;
        double *cp = C + (int64_t)(okc ? col : c_lo) * ldc;
        double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
        double ca[UNR][2], cb2[UNR][2];
        load_grp<UNR>(ca, cp, okc, H, rb0);
        for (int k0 = rb0; k0 < nrb; k0 += 2 * UNR) {
            if (k0 + UNR < nrb) load_grp<UNR>(cb2, cp, okc, H, k0 + UNR);
            w_grp<UNR>(w0, w1, ca, Ys, nrb, k0);
            if (k0 + UNR >= nrb) break;
            if (k0 + 2 * UNR < nrb) load_grp<UNR>(ca, cp, okc, H, k0 + 2 * UNR);
            w_grp<UNR>(w0, w1, cb2, Ys, nrb, k0 + UNR);
        }
        double p0 = 0.0, p1 = 0.0;
        dmma(p0, p1, w0[0] + w0[1], tb0);
        dmma(p0, p1, w1[0] + w1[1], tb1);
        load_grp<UNR>(ca, cp, okc, H, rb0);
        for (int k0 = rb0; k0 < nrb; k0 += 2 * UNR) {
            if (k0 + UNR < nrb) load_grp<UNR>(cb2, cp, okc, H, k0 + UNR);
            upd_grp<UNR>(ca, cp, okc, H, Ys, nrb, k0, p0, p1);
            if (k0 + UNR >= nrb) break;
            if (k0 + 2 * UNR < nrb) load_grp<UNR>(ca, cp, okc, H, k0 + 2 * UNR);
            upd_grp<UNR>(cb2, cp, okc, H, Ys, nrb, k0 + UNR, p0, p1);
        }
    }
}

template <int KM>
struct LeafSmem {
    // KM <= 16: panels are applied to the trailing columns in pairs (16
    // reflectors per pass over C: half the passes); Y of a pair is H x 16
    static constexpr bool TWO = KM <= 16;
    static constexpr int YW = TWO ? 16 : 8;
    double part[2][NW][9];
    double piv[2][8];
    double Gs[64], Ts[3][64], t8[8];           // T of panel p (slot p & 1), T01 of a pair
    double gp[NW][64];                         // per-warp partial Gram Y0^T Y1 of a pair
    double xs[NW][2][8 * KM];
    double Ys[8];              // H_pad x YW (the launch sizes it to the tallest tile)
    static size_t bytes(int max_rows) { return sizeof(LeafSmem) + sizeof(double) * YW * ((max_rows + 7) / 8 * 8); }
};

// C <- (I - Y T16^T Y^T) C for a pair of panels (Y = [Y0 Y1], H x 16 in Ys,
// T16 = [T0 T01; 0 T1], LAPACK's forward compact WY of 16 reflectors) on the
// columns [c_lo, c_hi) and rows [8 rb0, H) of C: one W pass and one update
// pass over C for 16 reflectors, each software-pipelined like apply_panel_cols.
template <int U>
__device__ __forceinline__ void w_grp16(double (&w0)[2], double (&w1)[2], double (&v0)[2], double (&v1)[2],
                                        const double (&cv)[U][2], const double *Ys, int nrb, int k0) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (k0 + u < nrb) {
            const int r = 8 * (k0 + u) + 2 * q;
            dmma(w0[u & 1], w1[u & 1], cv[u][0], Ys[r * 16 + l4]);
            dmma(w0[u & 1], w1[u & 1], cv[u][1], Ys[(r + 1) * 16 + l4]);
            dmma(v0[u & 1], v1[u & 1], cv[u][0], Ys[r * 16 + 8 + l4]);
            dmma(v0[u & 1], v1[u & 1], cv[u][1], Ys[(r + 1) * 16 + 8 + l4]);
        }
    }
}
template <int U>
__device__ __forceinline__ void upd_grp16(double (&cv)[U][2], double *cp, bool okc, int H, const double *Ys,
                                          int nrb, int k0, double p0, double p1, double r0, double r1) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (k0 + u < nrb) {
            const double2 y = *reinterpret_cast<const double2 *>(Ys + (8 * (k0 + u) + l4) * 16 + 2 * q);
            const double2 z = *reinterpret_cast<const double2 *>(Ys + (8 * (k0 + u) + l4) * 16 + 8 + 2 * q);
            dmma(cv[u][0], cv[u][1], -p0, y.x);
            dmma(cv[u][0], cv[u][1], -p1, y.y);
            dmma(cv[u][0], cv[u][1], -r0, z.x);
            dmma(cv[u][0], cv[u][1], -r1, z.y);
            const int r = 8 * (k0 + u) + 2 * q;
            st_pair(cp, okc, r, H, cv[u][0], cv[u][1]);
        }
    }
}
template <bool kFwd = true>
__device__ __forceinline__ void apply_pair_cols(const double *Ys, const double *T0, const double *T1,
                                                const double *T01, double *C, int64_t ldc, int H, int rb0, int c_lo,
                                                int c_hi) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    // B operands: T(2q+e, l4) of the three 8x8 blocks for Q^T (P = W^T T16), T(l4, 2q+e) for Q
    // (P = W^T T16^T, T16^T = [T0^T 0; T01^T T1^T])
    auto tb = [&](const double *T, int e) { return kFwd ? T[(2 * q + e) * 8 + l4] : T[l4 * 8 + 2 * q + e]; };
    const double a0 = tb(T0, 0), a1 = tb(T0, 1), b0 = tb(T1, 0), b1 = tb(T1, 1), x0 = tb(T01, 0), x1 = tb(T01, 1);
    const int nrb = (H + 7) / 8;
    constexpr int U = 4;                       // row blocks per load group (register budget of 2 CTAs/SM)
    for (int cb = c_lo / 8 + warp; 8 * cb < c_hi; cb += NW) {
        const int col = 8 * cb + l4;
        const bool okc = col < c_hi;
        double *cp = C + (int64_t)(okc ? col : c_lo) * ldc;
        double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0}, v0[2] = {0.0, 0.0}, v1[2] = {0.0, 0.0};
        double ca[U][2], cb2[U][2];
        load_grp<U>(ca, cp, okc, H, rb0);
        for (int k0 = rb0; k0 < nrb; k0 += 2 * U) {
            if (k0 + U < nrb) load_grp<U>(cb2, cp, okc, H, k0 + U);
            w_grp16<U>(w0, w1, v0, v1, ca, Ys, nrb, k0);
            if (k0 + U >= nrb) break;
            if (k0 + 2 * U < nrb) load_grp<U>(ca, cp, okc, H, k0 + 2 * U);
            w_grp16<U>(w0, w1, v0, v1, cb2, Ys, nrb, k0 + U);
        }
        // P0 = W0^T T0, P1 = W0^T T01 + W1^T T1 (W^T = C^T [Y0 Y1], fragments of 8 columns)
        const double we = w0[0] + w0[1], wo = w1[0] + w1[1], ve = v0[0] + v0[1], vo = v1[0] + v1[1];
        double p0 = 0.0, p1 = 0.0, r0 = 0.0, r1 = 0.0;
        dmma(p0, p1, we, a0);
        dmma(p0, p1, wo, a1);
        if (kFwd) {                            // P1 = W0^T T01 + W1^T T1
            dmma(r0, r1, we, x0);
            dmma(r0, r1, wo, x1);
        } else {                               // P0 += W1^T T01^T
            dmma(p0, p1, ve, x0);
            dmma(p0, p1, vo, x1);
        }
        dmma(r0, r1, ve, b0);
        dmma(r0, r1, vo, b1);
        load_grp<U>(ca, cp, okc, H, rb0);
        for (int k0 = rb0; k0 < nrb; k0 += 2 * U) {
            if (k0 + U < nrb) load_grp<U>(cb2, cp, okc, H, k0 + U);
            upd_grp16<U>(ca, cp, okc, H, Ys, nrb, k0, p0, p1, r0, r1);
            if (k0 + U >= nrb) break;
            if (k0 + 2 * U < nrb) load_grp<U>(ca, cp, okc, H, k0 + 2 * U);
            upd_grp16<U>(cb2, cp, okc, H, Ys, nrb, k0 + U, p0, p1, r0, r1);
        }
    }
}

// The same for ONE column block [c_lo, c_hi) (c_hi <= c_lo + 8) of a tile whose rows fit
// KM row blocks per warp, split over the warps by rows instead of columns: warp w owns row
// blocks rb0 + w, rb0 + w + 8, ...; all of its loads are in flight at once and stay in
// registers for the update; the warps' partial W^T meet in gp (NW x 64, fixed summation
// order), every warp forms W'^T = W^T T^T itself.  Column-split, this block was one warp's
// work while the other seven waited at the panel's barrier (a lookahead step of a pair).
template <int KM, int YW>
__device__ __forceinline__ void apply_block_rows(const double *Ys, const double *Tg, double *C, int64_t ldc, int H,
                                                 int rb0, int c_lo, int c_hi, double (*gp)[64]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const double tb0 = Tg[(2 * q) * 8 + l4], tb1 = Tg[(2 * q + 1) * 8 + l4];
    const int nrb = (H + 7) / 8;
    const int col = c_lo + l4;
    const bool okc = col < c_hi;
    double *cp = C + (int64_t)(okc ? col : c_lo) * ldc;
    double cv[KM][2];
#pragma unroll
    for (int u = 0; u < KM; ++u) {
        const int k = rb0 + warp + NW * u;
        if (k < nrb) ld_pair(cv[u][0], cv[u][1], cp, okc, 8 * k + 2 * q, H);
        else cv[u][0] = cv[u][1] = 0.0;
    }
    double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < KM; ++u) {
        const int k = rb0 + warp + NW * u;
        if (k < nrb) {
            const int r = 8 * k + 2 * q;
            dmma(w0[u & 1], w1[u & 1], cv[u][0], Ys[r * YW + l4]);
            dmma(w0[u & 1], w1[u & 1], cv[u][1], Ys[(r + 1) * YW + l4]);
        }
    }
    *reinterpret_cast<double2 *>(&gp[warp][2 * lane]) = make_double2(w0[0] + w0[1], w1[0] + w1[1]);
    __syncthreads();
    double wt0 = 0.0, wt1 = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const double2 g = *reinterpret_cast<const double2 *>(&gp[w][2 * lane]);
        wt0 += g.x;
        wt1 += g.y;
    }
    double p0 = 0.0, p1 = 0.0;
    dmma(p0, p1, wt0, tb0);
    dmma(p0, p1, wt1, tb1);
#pragma unroll
    for (int u = 0; u < KM; ++u) {
        const int k = rb0 + warp + NW * u;
        if (k < nrb) {
            const int r8 = 8 * k + l4;
            dmma(cv[u][0], cv[u][1], -p0, Ys[r8 * YW + 2 * q]);
            dmma(cv[u][0], cv[u][1], -p1, Ys[r8 * YW + 2 * q + 1]);
            st_pair(cp, okc, 8 * k + 2 * q, H, cv[u][0], cv[u][1]);
        }
    }
}

// apply_panel_cols on a Y stored with row stride YW (one panel's 8 columns at Ys + off)
template <int YW, bool kFwd = true>
__device__ __forceinline__ void apply_one_cols(const double *Ys, const double *Tg, double *C, int64_t ldc, int H,
                                               int rb0, int c_lo, int c_hi) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const double tb0 = kFwd ? Tg[(2 * q) * 8 + l4] : Tg[l4 * 8 + 2 * q];
    const double tb1 = kFwd ? Tg[(2 * q + 1) * 8 + l4] : Tg[l4 * 8 + 2 * q + 1];
    const int nrb = (H + 7) / 8;
    for (int cb = c_lo / 8 + warp; 8 * cb < c_hi; cb += NW) {
        const int col = 8 * cb + l4;
        const bool okc = col < c_hi;
        double *cp = C + (int64_t)(okc ? col : c_lo) * ldc;
        double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
        for (int k0 = rb0; k0 < nrb; k0 += UNR) {
            double cv[UNR][2];
            load_grp<UNR>(cv, cp, okc, H, k0);
#pragma unroll
            for (int u = 0; u < UNR; ++u)
                if (k0 + u < nrb) {
                    const int r = 8 * (k0 + u) + 2 * q;
                    dmma(w0[u & 1], w1[u & 1], cv[u][0], Ys[r * YW + l4]);
                    dmma(w0[u & 1], w1[u & 1], cv[u][1], Ys[(r + 1) * YW + l4]);
                }
        }
        double p0 = 0.0, p1 = 0.0;
        dmma(p0, p1, w0[0] + w0[1], tb0);
        dmma(p0, p1, w1[0] + w1[1], tb1);
        for (int k0 = rb0; k0 < nrb; k0 += UNR) {
            double cv[UNR][2];
            load_grp<UNR>(cv, cp, okc, H, k0);
#pragma unroll
            for (int u = 0; u < UNR; ++u)
                if (k0 + u < nrb) {
                    const int r8 = 8 * (k0 + u) + l4;
                    dmma(cv[u][0], cv[u][1], -p0, Ys[r8 * YW + 2 * q]);
                    dmma(cv[u][0], cv[u][1], -p1, Ys[r8 * YW + 2 * q + 1]);
                    const int r = 8 * (k0 + u) + 2 * q;
                    st_pair(cp, okc, r, H, cv[u][0], cv[u][1]);
                }
        }
    }
}

// Blocked compact-WY QR of one tile (H rows, H <= 64 KM): the panel is
// row-split over the warps (warp w: rows [w 8KM, (w+1) 8KM)), one
// __syncthreads per Householder step for the cross-warp sums; T per panel;
// the trailing update column-split (apply_panel_cols).
template <int KM, bool kRobust>
__device__ void wide_leaf_qr(double *At, int64_t lda, int H, int n, double *tau, double *tcache, double *tpair,
                             LeafSmem<KM> &S) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int npan = (n + 7) / 8;
    const int rbase = warp * 8 * KM;
    const int Hp = 8 * ((H + 7) / 8);
    constexpr bool TWO = LeafSmem<KM>::TWO;
    constexpr int YW = LeafSmem<KM>::YW;
    for (int p = 0; p < npan; ++p) {
        const int c = 8 * p + l4;
        const int yo = TWO ? 8 * (p & 1) : 0;            // this panel's 8 columns of Ys
        double *Tp = S.Ts[TWO ? (p & 1) : 0];
        double *colp = At + (int64_t)(c < n ? c : 0) * lda;
        double a[KM][2];
#pragma unroll
        for (int k = 0; k < KM; ++k) ld_pair(a[k][0], a[k][1], colp, c < n, rbase + 8 * k + 2 * q, H);
        double *xs0 = S.xs[warp][0], *xs1 = S.xs[warp][1];
        if (l4 == 0) {
#pragma unroll
            for (int k = 0; k < KM; ++k)
                *reinterpret_cast<double2 *>(xs0 + 8 * k + 2 * q) = make_double2(a[k][0], a[k][1]);
        }
        __syncwarp();
        const int jn = min(8, n - 8 * p);
#pragma unroll 1
        for (int jj = 0; jj < jn; ++jj) {
            const int j = 8 * p + jj;
            const int par = jj & 1;
            const double *xr = par ? xs1 : xs0;
            double d[4] = {0.0, 0.0, 0.0, 0.0}, s[4] = {0.0, 0.0, 0.0, 0.0};
            double pv = 0.0;
            bool haspiv = false;
#pragma unroll
            for (int k = 0; k < KM; ++k) {
                const double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                const int r = rbase + 8 * k + 2 * q;
                const double x0 = r > j ? xv.x : 0.0, x1 = r + 1 > j ? xv.y : 0.0;
                d[k & 3] = fma(x0, a[k][0], d[k & 3]);
                d[(k + 2) & 3] = fma(x1, a[k][1], d[(k + 2) & 3]);
                s[k & 3] = fma(x0, x0, s[k & 3]);
                s[(k + 2) & 3] = fma(x1, x1, s[(k + 2) & 3]);
                if (r == j) { pv = a[k][0]; haspiv = true; }
                if (r + 1 == j) { pv = a[k][1]; haspiv = true; }
            }
            double dd = (d[0] + d[1]) + (d[2] + d[3]), s2 = (s[0] + s[1]) + (s[2] + s[3]);
            dd += __shfl_xor_sync(FULL, dd, 1);
            s2 += __shfl_xor_sync(FULL, s2, 1);
            dd += __shfl_xor_sync(FULL, dd, 2);
            s2 += __shfl_xor_sync(FULL, s2, 2);
            if (q == 0) S.part[par][warp][l4] = dd;
            if (lane == 0) S.part[par][warp][8] = s2;
            if (haspiv) S.piv[par][l4] = pv;
            __syncthreads();
            dd = 0.0;
            s2 = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                dd += S.part[par][w][l4];
                s2 += S.part[par][w][8];
            }
            const double rj = S.piv[par][l4], alpha = S.piv[par][jj];
            House h = house(alpha, s2);
            double sc = 1.0;
            double sx = h.scale;
            if (kRobust && wy::house_unsafe(alpha, s2)) {          // block-uniform, rescaled step (R23)
                double mx = fabs(alpha);
#pragma unroll
                for (int k = 0; k < KM; ++k) {
                    const double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                    const int r = rbase + 8 * k + 2 * q;
                    mx = fmax(mx, fmax(r > j ? fabs(xv.x) : 0.0, r + 1 > j ? fabs(xv.y) : 0.0));
                }
                mx = fmax(mx, __shfl_xor_sync(FULL, mx, 1));
                mx = fmax(mx, __shfl_xor_sync(FULL, mx, 2));
                // part[par ^ 1] is free: its last readers (step jj - 1) are past this step's barrier
                if (lane == 0) S.part[par ^ 1][warp][8] = mx;
                __syncthreads();
                for (int w = 0; w < NW; ++w) mx = fmax(mx, S.part[par ^ 1][w][8]);
                sc = wy::pow2_scale(mx);
                __syncthreads();
                double e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0;
#pragma unroll
                for (int k = 0; k < KM; ++k) {
                    const double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                    const int r = rbase + 8 * k + 2 * q;
                    const double x0 = r > j ? sc * xv.x : 0.0, x1 = r + 1 > j ? sc * xv.y : 0.0;
                    e0 = fma(x0, a[k][0], e0);
                    e1 = fma(x1, a[k][1], e1);
                    f0 = fma(x0, x0, f0);
                    f1 = fma(x1, x1, f1);
                }
                dd = e0 + e1;
                s2 = f0 + f1;
                dd += __shfl_xor_sync(FULL, dd, 1);
                s2 += __shfl_xor_sync(FULL, s2, 1);
                dd += __shfl_xor_sync(FULL, dd, 2);
                s2 += __shfl_xor_sync(FULL, s2, 2);
                if (q == 0) S.part[par ^ 1][warp][l4] = dd;
                if (lane == 0) S.part[par ^ 1][warp][8] = s2;
                __syncthreads();
                dd = 0.0;
                s2 = 0.0;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    dd += S.part[par ^ 1][w][l4];
                    s2 += S.part[par ^ 1][w][8];
                }
                h = house(sc * alpha, s2);
                h.beta = h.beta / sc;
                sx = h.scale * sc;
            }
            const double wv = fma(h.scale, dd, rj);
            const double u = (l4 > jj) ? h.tau * sx * wv : (l4 == jj ? 1.0 : 0.0);
            const double g = (l4 == jj) ? sx : 0.0;
            const double pnew = (l4 > jj) ? fma(-h.tau, wv, rj) : (l4 == jj ? h.beta : rj);
            double *xw = par ? xs0 : xs1;
#pragma unroll
            for (int k = 0; k < KM; ++k) {
                const double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
                const int r = rbase + 8 * k + 2 * q;
                const double x0 = r > j ? xv.x : 0.0, x1 = r + 1 > j ? xv.y : 0.0;
                double a0 = fma(g, x0, fma(-u, x0, a[k][0])), a1 = fma(g, x1, fma(-u, x1, a[k][1]));
                a0 = (r == j) ? pnew : a0;
                a1 = (r + 1 == j) ? pnew : a1;
                a[k][0] = a0;
                a[k][1] = a1;
                if (l4 == jj + 1) *reinterpret_cast<double2 *>(xw + 8 * k + 2 * q) = make_double2(a0, a1);
            }
            if (warp == 0 && q == 0 && l4 < jj) S.Gs[l4 * 8 + jj] = fma(h.scale, dd, rj);
            if (threadIdx.x == 0) S.t8[jj] = h.tau;
            __syncwarp();
        }
        if (warp == 0) {                         // padding columns past n: identity steps
            for (int c2 = jn; c2 < 8; ++c2) {
                if (q == 0 && l4 < c2) S.Gs[l4 * 8 + c2] = 0.0;
                if (lane == 0) S.t8[c2] = 0.0;
            }
        }
        // write the panel back; Y of the panel -> Ys (rows >= 8p, zero past H)
#pragma unroll
        for (int k = 0; k < KM; ++k) st_pair(colp, c < n, rbase + 8 * k + 2 * q, H, a[k][0], a[k][1]);
#pragma unroll
        for (int k = 0; k < KM; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = rbase + 8 * k + 2 * q + e;
                if (r >= 8 * (TWO ? (p & ~1) : p) && r < Hp)     // a pair's Y1 is zero on Y0's first rows
                    S.Ys[r * YW + yo + l4] = (c >= n || r < c || r >= H) ? 0.0 : (r == c ? 1.0 : a[k][e]);
            }
        __syncthreads();
        if (warp == 0) {
            const int rr = lane & 7;
            double row[8];
            const double tr = S.t8[rr];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) row[cc] = (cc == rr) ? tr : 0.0;
#pragma unroll
            for (int cc = 1; cc < 8; ++cc) {
                double sacc = 0.0;
#pragma unroll
                for (int l = 0; l < cc; ++l) sacc = fma(row[l], S.Gs[l * 8 + cc], sacc);
                row[cc] = (rr < cc) ? -S.t8[cc] * sacc : row[cc];
            }
            if (lane < 8) {
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    Tp[lane * 8 + cc] = row[cc];
                    tcache[p * 64 + lane * 8 + cc] = row[cc];
                }
                if (8 * p + lane < n) tau[8 * p + lane] = S.t8[lane];
            }
        }
        __syncthreads();
        if (!TWO) {
            if (p + 1 < npan) apply_one_cols<YW>(S.Ys, Tp, At, lda, H, p, 8 * (p + 1), n);
        } else if ((p & 1) == 0) {
            // first panel of a pair: update only the pair's second column block
            // (row-split over the warps: C3 leaf 0.953 -> 0.928 ms against one warp's column slab)
            if (p + 1 < npan) apply_block_rows<KM, YW>(S.Ys, Tp, At, lda, H, p, 8 * (p + 1), min(n, 8 * (p + 2)), S.gp);
        } else {
            // (also for the last pair: the apply / form-Q kernels use its T01)
            // second panel of a pair: T01 = -T0 (Y0^T Y1) T1, then the 16-reflector update
            {
                double g0 = 0.0, g1 = 0.0;
                for (int k = p + warp; k < Hp / 8; k += NW) {         // Y1 is zero above row 8p
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int r = 8 * k + 2 * q + e;
                        dmma(g0, g1, S.Ys[r * 16 + l4], S.Ys[r * 16 + 8 + l4]);
                    }
                }
                *reinterpret_cast<double2 *>(&S.gp[warp][8 * l4 + 2 * q]) = make_double2(g0, g1);
            }
            __syncthreads();
            if (warp == 0) {
                // lane (i, j0): T01(i, j0 + e) = -sum_a T0(i, a) sum_b G(a, b) T1(b, j0 + e),
                // G = Y0^T Y1 = sum of the warps' partials
                const int i = lane >> 2, j0 = 2 * (lane & 3);
                double t01[2] = {0.0, 0.0};
                // T01(i, j) = - sum_a T0(i, a) sum_b G(a, b) T1(b, j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = j0 + e;
                    double acc = 0.0;
#pragma unroll
                    for (int a = 0; a < 8; ++a) {
                        double gb = 0.0;
#pragma unroll
                        for (int bb = 0; bb < 8; ++bb) {
                            double gab = 0.0;
#pragma unroll
                            for (int w = 0; w < NW; ++w) gab += S.gp[w][8 * a + bb];
                            gb = fma(gab, S.Ts[1][bb * 8 + j], gb);
                        }
                        acc = fma(S.Ts[0][i * 8 + a], gb, acc);
                    }
                    t01[e] = -acc;
                }
                S.Ts[2][i * 8 + j0] = t01[0];
                S.Ts[2][i * 8 + j0 + 1] = t01[1];
                tpair[(p >> 1) * 64 + i * 8 + j0] = t01[0];     // for the paired apply / form Q
                tpair[(p >> 1) * 64 + i * 8 + j0 + 1] = t01[1];
            }
            __syncthreads();
            if (p + 1 < npan) apply_pair_cols(S.Ys, S.Ts[0], S.Ts[1], S.Ts[2], At, lda, H, p - 1, 8 * (p + 1), n);
        }
        __syncthreads();
    }
}
}  // namespace wide

using namespace wide;

// Leaves: tile t (one CTA each), row-split panels sized to the tile.
template <int KM, bool kRobust>
__global__ void __launch_bounds__(NT, KM <= 8 ? 2 : 1)
k_wide_leaves(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows, double *tau_tile,
              double *tcache_tile, double *tpair_tile) {
    extern __shared__ __align__(16) double smraw[];
    LeafSmem<KM> &S = *reinterpret_cast<LeafSmem<KM> *>(smraw);
    const int t = blockIdx.x;
    const int npan = (n + 7) / 8;
    wide_leaf_qr<KM, kRobust>(A + tile_row0[t], lda, tile_rows[t], n, tau_tile + (int64_t)t * n,
                     tcache_tile + (int64_t)t * npan * 64, tpair_tile + (int64_t)t * ((npan + 1) / 2) * 64, S);
}

// Tree nodes of one step: node ids[i] = b (right subtree's first tile), its
// left child's first tile node_a[b]; [R_a; R_b] in the tiles' head rows.
__global__ void __launch_bounds__(NT, 1)
k_wide_nodes(double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a, const int *ids,
             double *tau_node, double *tcache_node) {
    extern __shared__ __align__(16) double smraw[];
    Smem &S = *reinterpret_cast<Smem *>(smraw);
    const int b = ids[blockIdx.x];
    const int npan = (n + 7) / 8;
    Prob P{A + tile_row0[node_a[b]], A + tile_row0[b], lda, lda, 8 * npan, n, n, 1};
    wide_qr(P, n, tau_node + (int64_t)b * n, tcache_node + (int64_t)b * npan * 64, S);
}

// A single stacked node [Ra (ld lda); Rb (ld ldb)] (the cross-GPU rounds).
__global__ void __launch_bounds__(NT, 1)
k_wide_node1(double *Ra, int64_t lda, double *Rb, int64_t ldb, int n, double *tau, double *tcache) {
    extern __shared__ __align__(16) double smraw[];
    Smem &S = *reinterpret_cast<Smem *>(smraw);
    Prob P{Ra, Rb, lda, ldb, 8 * ((n + 7) / 8), n, n, 1};
    wide_qr(P, n, tau, tcache, S);
}

// Q^T C / Q C on the leaves (forward: all tiles; C rows = the tile's rows):
// panel by panel (forward for Q^T, backward for Q) the panel's Y is staged in
// shared memory from the stored factor, then the column-split update.
template <bool kFwd>
__global__ void __launch_bounds__(NT, 2)
k_wide_apply_leaves(const double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows,
                    const double *tcache_tile, const double *tpair_tile, int pairs, double *C, int64_t ldc, int k,
                    int two_slots) {
    // Panels are applied in the factor's pairs when it cached their T01 (pairs:
    // tiles <= 1024 rows): Y of a pair (H x 16, row stride 16) and its T0, T1,
    // T01 staged with cp.async, the next group's copy in flight in a second slot
    // when it fits; one 16-reflector pass over C per pair (apply_pair_cols).
    extern __shared__ __align__(16) double smraw[];
    const int t = blockIdx.x;
    const int npan = (n + 7) / 8;
    const int H = tile_rows[t];
    const int Hp = 8 * ((H + 7) / 8);
    double *Ts = smraw, *Ys = smraw + 2 * 192;                   // 2 slots: T0 T1 T01 | Y
    const double *At = A + tile_row0[t];
    const double *tc = tcache_tile + (int64_t)t * npan * 64;
    const double *tp = tpair_tile + (int64_t)t * ((npan + 1) / 2) * 64;
    const int gw = pairs ? 2 : 1;                               // panels per group
    const int yw = 8 * gw;                                      // Y's row stride
    const int ngrp = (npan + gw - 1) / gw;
    auto stage = [&](int g, int slot) {
        double *Y = Ys + slot * Hp * yw, *T = Ts + slot * 192;
        const int p0 = gw * g, np = min(gw, npan - p0), h0 = 8 * p0, hs = Hp - h0;
        for (int e = threadIdx.x; e < 8 * np * hs; e += NT) {
            const int r = h0 + e % hs, jj = e / hs, c = 8 * p0 + jj;
            const bool ok = c < n && r > c && r < H;
            cp_async8(Y + r * yw + jj, At + (ok ? r + (int64_t)c * lda : 0), ok);
        }
        if (threadIdx.x < 64 * np) cp_async8(T + threadIdx.x, tc + 64 * p0 + threadIdx.x, true);
        if (np == 2 && threadIdx.x < 64) cp_async8(T + 128 + threadIdx.x, tp + 64 * g + threadIdx.x, true);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    stage(kFwd ? 0 : ngrp - 1, 0);
    for (int gg = 0; gg < ngrp; ++gg) {
        const int g = kFwd ? gg : ngrp - 1 - gg, slot = two_slots ? (gg & 1) : 0;
        if (two_slots && gg + 1 < ngrp) {
            stage(kFwd ? g + 1 : g - 1, slot ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const int p0 = gw * g, np = min(gw, npan - p0);
        double *Y = Ys + slot * Hp * yw, *T = Ts + slot * 192;
        if (threadIdx.x < 8 * np) {                             // the unit diagonals
            const int c = 8 * p0 + threadIdx.x;
            if (c < n && c < H) Y[c * yw + threadIdx.x] = 1.0;
        }
        __syncthreads();
        if (np == 2) apply_pair_cols<kFwd>(Y, T, T + 64, T + 128, C + tile_row0[t], ldc, H, p0, 0, k);
        else if (pairs) apply_one_cols<16, kFwd>(Y, T, C + tile_row0[t], ldc, H, p0, 0, k);
        else apply_one_cols<8, kFwd>(Y, T, C + tile_row0[t], ldc, H, p0, 0, k);
        __syncthreads();
        if (!two_slots && gg + 1 < ngrp) stage(kFwd ? g + 1 : g - 1, 0);
    }
}

// The same with the warp's 8-column slab of C resident in registers for the whole tile
// (tiles of <= 8 MR rows, k <= 64: one slab per warp, pairs cached): C is read and written
// once per tile instead of streamed through L2 twice per panel pair, and every pair's W^T
// and update run on registers (the streamed version waited on L2 latency with 4-8 row blocks
// in flight).  One CTA per SM (the slab takes 2 MR registers per lane).
template <bool kFwd, int MR>
__global__ void __launch_bounds__(NT, 1)
k_wide_apply_leaves_reg(const double *A, int64_t lda, int n, const int64_t *tile_row0, const int *tile_rows,
                        const double *tcache_tile, const double *tpair_tile, double *C, int64_t ldc, int k) {
    extern __shared__ __align__(16) double smraw[];
    const int t = blockIdx.x;
    const int npan = (n + 7) / 8;
    const int H = tile_rows[t];
    const int Hp = 8 * ((H + 7) / 8);
    const int nrb = Hp / 8;
    double *Ts = smraw, *Ys = smraw + 2 * 192;                   // 2 slots: T0 T1 T01 | Y (H x 16)
    const double *At = A + tile_row0[t];
    const double *tc = tcache_tile + (int64_t)t * npan * 64;
    const double *tp = tpair_tile + (int64_t)t * ((npan + 1) / 2) * 64;
    const int ngrp = (npan + 1) / 2;
    auto stage = [&](int g, int slot) {
        double *Y = Ys + slot * Hp * 16, *T = Ts + slot * 192;
        const int p0 = 2 * g, np = min(2, npan - p0), h0 = 8 * p0, hs = Hp - h0;
        for (int e = threadIdx.x; e < 8 * np * hs; e += NT) {
            const int r = h0 + e % hs, jj = e / hs, c = 8 * p0 + jj;
            const bool ok = c < n && r > c && r < H;
            cp_async8(Y + r * 16 + jj, At + (ok ? r + (int64_t)c * lda : 0), ok);
        }
        if (threadIdx.x < 64 * np) cp_async8(T + threadIdx.x, tc + 64 * p0 + threadIdx.x, true);
        if (np == 2 && threadIdx.x < 64) cp_async8(T + 128 + threadIdx.x, tp + 64 * g + threadIdx.x, true);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int col = 8 * warp + l4;
    const bool okc = col < k;
    double *cp = C + tile_row0[t] + (int64_t)(okc ? col : 0) * ldc;
    stage(kFwd ? 0 : ngrp - 1, 0);
    double c[MR][2];
#pragma unroll
    for (int kk = 0; kk < MR; ++kk) {
        c[kk][0] = c[kk][1] = 0.0;
        if (kk < nrb) ld_pair(c[kk][0], c[kk][1], cp, okc, 8 * kk + 2 * q, H);
    }
    for (int gg = 0; gg < ngrp; ++gg) {
        const int g = kFwd ? gg : ngrp - 1 - gg, slot = gg & 1;
        if (gg + 1 < ngrp) {
            stage(kFwd ? g + 1 : g - 1, slot ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const int p0 = 2 * g, np = min(2, npan - p0);
        double *Y = Ys + slot * Hp * 16, *T = Ts + slot * 192;
        if (threadIdx.x < 8 * np) {                             // the unit diagonals
            const int cc = 8 * p0 + threadIdx.x;
            if (cc < n && cc < H) Y[cc * 16 + threadIdx.x] = 1.0;
        }
        __syncthreads();
        auto tb = [&](const double *Tm, int e) { return kFwd ? Tm[(2 * q + e) * 8 + l4] : Tm[l4 * 8 + 2 * q + e]; };
        if (np == 2) {
            const double a0 = tb(T, 0), a1 = tb(T, 1), b0 = tb(T + 64, 0), b1 = tb(T + 64, 1);
            const double x0 = tb(T + 128, 0), x1 = tb(T + 128, 1);
            double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0}, v0[2] = {0.0, 0.0}, v1[2] = {0.0, 0.0};
#pragma unroll
            for (int kk = 0; kk < MR; ++kk) {
                if (kk >= p0 && kk < nrb) {
                    const int r = 8 * kk + 2 * q;
                    dmma(w0[kk & 1], w1[kk & 1], c[kk][0], Y[r * 16 + l4]);
                    dmma(w0[kk & 1], w1[kk & 1], c[kk][1], Y[(r + 1) * 16 + l4]);
                    dmma(v0[kk & 1], v1[kk & 1], c[kk][0], Y[r * 16 + 8 + l4]);
                    dmma(v0[kk & 1], v1[kk & 1], c[kk][1], Y[(r + 1) * 16 + 8 + l4]);
                }
            }
            const double we = w0[0] + w0[1], wo = w1[0] + w1[1], ve = v0[0] + v0[1], vo = v1[0] + v1[1];
            double q0 = 0.0, q1 = 0.0, r0 = 0.0, r1 = 0.0;
            dmma(q0, q1, we, a0);
            dmma(q0, q1, wo, a1);
            if (kFwd) {                                         // P1 = W0^T T01 + W1^T T1
                dmma(r0, r1, we, x0);
                dmma(r0, r1, wo, x1);
            } else {                                            // P0 += W1^T T01^T
                dmma(q0, q1, ve, x0);
                dmma(q0, q1, vo, x1);
            }
            dmma(r0, r1, ve, b0);
            dmma(r0, r1, vo, b1);
#pragma unroll
            for (int kk = 0; kk < MR; ++kk) {
                if (kk >= p0 && kk < nrb) {
                    const double2 y = *reinterpret_cast<const double2 *>(Y + (8 * kk + l4) * 16 + 2 * q);
                    const double2 z = *reinterpret_cast<const double2 *>(Y + (8 * kk + l4) * 16 + 8 + 2 * q);
                    dmma(c[kk][0], c[kk][1], -q0, y.x);
                    dmma(c[kk][0], c[kk][1], -q1, y.y);
                    dmma(c[kk][0], c[kk][1], -r0, z.x);
                    dmma(c[kk][0], c[kk][1], -r1, z.y);
                }
            }
        } else {                                                // the last, unpaired panel
            const double t0 = tb(T, 0), t1 = tb(T, 1);
            double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
#pragma unroll
            for (int kk = 0; kk < MR; ++kk) {
                if (kk >= p0 && kk < nrb) {
                    const int r = 8 * kk + 2 * q;
                    dmma(w0[kk & 1], w1[kk & 1], c[kk][0], Y[r * 16 + l4]);
                    dmma(w0[kk & 1], w1[kk & 1], c[kk][1], Y[(r + 1) * 16 + l4]);
                }
            }
            double q0 = 0.0, q1 = 0.0;
            dmma(q0, q1, w0[0] + w0[1], t0);
            dmma(q0, q1, w1[0] + w1[1], t1);
#pragma unroll
            for (int kk = 0; kk < MR; ++kk) {
                if (kk >= p0 && kk < nrb) {
                    const int r8 = 8 * kk + l4;
                    dmma(c[kk][0], c[kk][1], -q0, Y[r8 * 16 + 2 * q]);
                    dmma(c[kk][0], c[kk][1], -q1, Y[r8 * 16 + 2 * q + 1]);
                }
            }
        }
        __syncthreads();                                        // the slot may be refilled
    }
#pragma unroll
    for (int kk = 0; kk < MR; ++kk)
        if (kk < nrb) st_pair(cp, okc, 8 * kk + 2 * q, H, c[kk][0], c[kk][1]);
}

// Q^T / Q of one tree step's nodes on C's head rows (or on xbuf blocks for form Q).
template <bool kFwd>
__global__ void __launch_bounds__(NT, 1)
k_wide_apply_nodes(const double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a,
                   const int *ids, const double *tcache_node, double *C, int64_t ldc, int k, int xbuf_mode) {
    const int b = ids[blockIdx.x];
    const int a = node_a[b];
    const int npan = (n + 7) / 8;
    const int hA = 8 * npan;
    Prob P{const_cast<double *>(A) + tile_row0[a], const_cast<double *>(A) + tile_row0[b], lda, lda, hA, n, n, 1};
    Prob Cp = xbuf_mode ? Prob{C + (int64_t)a * n * n, C + (int64_t)b * n * n, n, n, hA, n, n, 0}
                        : Prob{C + tile_row0[a], C + tile_row0[b], ldc, ldc, hA, n, n, 0};
    wide_apply<kFwd>(P, Cp, n, k, tcache_node + (int64_t)b * npan * 64);
}

// Q^T / Q of tree nodes for npan <= 28: the node's Y1 (upper block triangle of
// the right subtree's head, 8x8 column-major blocks) and its panels' T are
// staged in shared memory once; every warp then owns an 8-column slab of C and
// runs all panels alone: C_b's head rows (n x 8) in registers, C_a's row block P
// read and written back per panel (the identity part of the node's reflectors).
// No barrier after the staging.
// Launched either per tree step (ids = the step's nodes, one CTA each) or, with
// `flags`, once for the whole tree: ids is every node in dependency order
// (bottom-up for Q^T, top-down for Q), each CTA takes the next node from a ticket
// counter (flags[L]) when it starts -- so it only ever waits on nodes taken
// earlier, which are resident or done -- stages the node's factors, waits until
// the nodes it depends on (dep0/dep1: the producers of its two C head blocks
// bottom-up, its parent top-down; -1 none) have set their flags, applies the
// node and sets its own flag.  Levels overlap: the critical path is the tree's
// depth in node latencies instead of one launch per step.
constexpr int NPAN_NODE = 28;
template <bool kFwd, int NPAN_NODE>
__global__ void __launch_bounds__(NT, 1)
k_node_apply(const double *A, int64_t lda, int n, const int64_t *tile_row0, const int *node_a,
                       const int *ids, const double *tcache_node, double *C, int64_t ldc, int k, int xbuf_mode,
                       int *flags, int L, const int *dep0, const int *dep1, int *pflags) {
    extern __shared__ __align__(16) double smraw[];
    __shared__ int s_idx;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    if (flags) {
        if (threadIdx.x == 0) s_idx = atomicAdd(flags + L, 1);
        __syncthreads();
    }
    const int b = ids[flags ? s_idx : blockIdx.x], a = node_a[b];
    const int npan = (n + 7) / 8;
    const int nb = npan * (npan + 1) / 2;
    double *Yb = smraw, *Tn = smraw + 64 * nb;
    const double *Hb = A + tile_row0[b];
    // Y1 and the T's staged with cp.async: every copy of the CTA in flight at once
    for (int e = threadIdx.x; e < 64 * nb; e += NT) {
        const int bi = e >> 6, cl = (e >> 3) & 7, r = e & 7;
        int cb = (int)((sqrtf(8.0f * bi + 1.0f) - 1.0f) * 0.5f);   // bi = cb(cb+1)/2 + kk, kk <= cb
        cb += (cb + 1) * (cb + 2) / 2 <= bi;
        cb -= cb * (cb + 1) / 2 > bi;
        const int kk = bi - cb * (cb + 1) / 2;
        const int i = 8 * kk + r, c = 8 * cb + cl;
        const bool ok = i <= c && c < n;
        cp_async8(Yb + e, Hb + (ok ? i + (int64_t)c * lda : 0), ok);
    }
    const double *tc = tcache_node + (int64_t)b * npan * 64;
    for (int e = threadIdx.x; e < 64 * npan; e += NT) cp_async8(Tn + e, tc + e, true);
    const bool ppipe = flags && pflags;             // panel-level hand-offs (below)
    if (flags && !ppipe && threadIdx.x == 0) {       // the producers of this node's inputs
        const int d0 = dep0[b], d1 = dep1 ? dep1[b] : -1;
        if (d0 >= 0)
            while (*reinterpret_cast<volatile int *>(flags + d0) == 0) __nanosleep(64);
        if (d1 >= 0)
            while (*reinterpret_cast<volatile int *>(flags + d1) == 0) __nanosleep(64);
        __threadfence();
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    double *Ca, *Cb;
    int64_t ld;
    if (xbuf_mode) {
        Ca = C + (int64_t)a * n * n; Cb = C + (int64_t)b * n * n; ld = n;
    } else {
        Ca = C + tile_row0[a]; Cb = C + tile_row0[b]; ld = ldc;
    }
    if (ppipe) {
        // Whole tree in one launch, panel-level pipelining.  Q^T (bottom-up, panels forward):
        // this node's panel P needs only row block P of its two input head blocks (C_a: the
        // left child's output, C_b: the right child's), final once that child has applied its
        // own panel P; it publishes its output row block P (C_a's, read by its parent) with a
        // per-(node, 8-column slab, panel) flag right after computing it, and loads C_b's row
        // blocks as its panels first need them (panel P reads C_b row blocks <= P only).
        // Q / form Q (top-down, panels backward): C_b is ready at the start (the input's head
        // rows, or the zeroed X block); C_a's row block P comes from the parent, final once the
        // parent has applied its panel P, and so are both of this node's outputs' row blocks P
        // (C_a's at panel P, C_b's at its last update, panel P): they are stored and published
        // there.  The critical path is about depth + panels panel latencies instead of depth
        // whole nodes.
        const int nslab = (k + 7) / 8;
        const int d0 = dep0[b], d1 = dep1 ? dep1[b] : -1;
        for (int cbw = warp; cbw < nslab; cbw += NW) {
            const int col = 8 * cbw + l4;
            const bool okc = col < k;
            const int64_t co = (int64_t)(okc ? col : 0) * ld;
            const int *f0 = d0 >= 0 ? pflags + ((int64_t)d0 * nslab + cbw) * npan : nullptr;
            const int *f1 = d1 >= 0 ? pflags + ((int64_t)d1 * nslab + cbw) * npan : nullptr;
            int *fme = pflags + ((int64_t)b * nslab + cbw) * npan;
            double cb[NPAN_NODE][2];
#pragma unroll
            for (int kk = 0; kk < NPAN_NODE; ++kk)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int r = 8 * kk + 2 * q + e;
                    cb[kk][e] = (!kFwd && okc && kk < npan && r < n) ? Cb[r + co] : 0.0;
                }
            for (int pp = 0; pp < npan; ++pp) {
                const int P = kFwd ? pp : npan - 1 - pp;
                if (lane == 0) {
                    if (f1) while (*reinterpret_cast<const volatile int *>(f1 + P) == 0) __nanosleep(32);
                    if (f0) while (*reinterpret_cast<const volatile int *>(f0 + P) == 0) __nanosleep(32);
                }
                __syncwarp();
                __threadfence();
                const double *Tg = Tn + 64 * P;
                const double tb0 = kFwd ? Tg[(2 * q) * 8 + l4] : Tg[l4 * 8 + 2 * q];
                const double tb1 = kFwd ? Tg[(2 * q + 1) * 8 + l4] : Tg[l4 * 8 + 2 * q + 1];
                const int ra = 8 * P + 2 * q;
                const double ca0 = (okc && ra < n) ? __ldcg(Ca + ra + co) : 0.0;
                const double ca1 = (okc && ra + 1 < n) ? __ldcg(Ca + ra + 1 + co) : 0.0;
                if (kFwd) {
                    const double nb0 = (okc && ra < n) ? __ldcg(Cb + ra + co) : 0.0;
                    const double nb1 = (okc && ra + 1 < n) ? __ldcg(Cb + ra + 1 + co) : 0.0;
#pragma unroll
                    for (int kk = 0; kk < NPAN_NODE; ++kk)
                        if (kk == P) {
                            cb[kk][0] = nb0;
                            cb[kk][1] = nb1;
                        }
                }
                const double *yP = Yb + 64 * (P * (P + 1) / 2);
                double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
#pragma unroll
                for (int g = 0; g < NPAN_NODE; g += 4) {
                    if (g <= P) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int kk = g + u;
                            if (kk < NPAN_NODE) {
                                const bool ok = kk <= P;
                                double2 y = *reinterpret_cast<const double2 *>(yP + 64 * (ok ? kk : P) + 8 * l4 + 2 * q);
                                y.x = ok ? y.x : 0.0;
                                y.y = ok ? y.y : 0.0;
                                dmma(w0[u & 1], w1[u & 1], cb[kk][0], y.x);
                                dmma(w0[u & 1], w1[u & 1], cb[kk][1], y.y);
                            }
                        }
                    }
                }
                double p0 = 0.0, p1 = 0.0;
                dmma(p0, p1, w0[0] + w0[1] + ca0, tb0);
                dmma(p0, p1, w1[0] + w1[1] + ca1, tb1);
                if (okc && ra < n) Ca[ra + co] = ca0 - p0;
                if (okc && ra + 1 < n) Ca[ra + 1 + co] = ca1 - p1;
                if (kFwd) {
                    __threadfence();                  // this node's output row block P ...
                    __syncwarp();
                    if (lane == 0) *reinterpret_cast<volatile int *>(fme + P) = 1;   // ... is published
                }
#pragma unroll
                for (int g = 0; g < NPAN_NODE; g += 4) {
                    if (g <= P) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int kk = g + u;
                            if (kk < NPAN_NODE) {
                                const bool ok = kk <= P;
                                const double *yb = yP + 64 * (ok ? kk : P);
                                const double y0 = ok ? yb[8 * (2 * q) + l4] : 0.0, y1 = ok ? yb[8 * (2 * q + 1) + l4] : 0.0;
                                dmma(cb[kk][0], cb[kk][1], -p0, y0);
                                dmma(cb[kk][0], cb[kk][1], -p1, y1);
                            }
                        }
                    }
                }
                if (!kFwd) {                          // C_b's row block P had its last update
#pragma unroll
                    for (int kk = 0; kk < NPAN_NODE; ++kk)
                        if (kk == P) {
                            if (okc && ra < n) Cb[ra + co] = cb[kk][0];
                            if (okc && ra + 1 < n) Cb[ra + 1 + co] = cb[kk][1];
                        }
                    __threadfence();                  // both outputs' row blocks P ...
                    __syncwarp();
                    if (lane == 0) *reinterpret_cast<volatile int *>(fme + P) = 1;   // ... are published
                }
            }
            if (kFwd) {
#pragma unroll
                for (int kk = 0; kk < NPAN_NODE; ++kk)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int r = 8 * kk + 2 * q + e;
                        if (okc && kk < npan && r < n) Cb[r + co] = cb[kk][e];
                    }
            }
        }
    }
    for (int cbw = warp; !ppipe && 8 * cbw < k; cbw += NW) {
        const int col = 8 * cbw + l4;
        const bool okc = col < k;
        const int64_t co = (int64_t)(okc ? col : 0) * ld;
        double cb[NPAN_NODE][2];
#pragma unroll
        for (int kk = 0; kk < NPAN_NODE; ++kk)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = 8 * kk + 2 * q + e;
                cb[kk][e] = (okc && kk < npan && r < n) ? Cb[r + co] : 0.0;
            }
        // C_a's row block of the next panel is prefetched one panel ahead
        const int P0 = kFwd ? 0 : npan - 1;
        double na0 = (okc && 8 * P0 + 2 * q < n) ? Ca[8 * P0 + 2 * q + co] : 0.0;
        double na1 = (okc && 8 * P0 + 2 * q + 1 < n) ? Ca[8 * P0 + 2 * q + 1 + co] : 0.0;
        for (int pp = 0; pp < npan; ++pp) {
            const int P = kFwd ? pp : npan - 1 - pp;
            const double *Tg = Tn + 64 * P;
            const double tb0 = kFwd ? Tg[(2 * q) * 8 + l4] : Tg[l4 * 8 + 2 * q];
            const double tb1 = kFwd ? Tg[(2 * q + 1) * 8 + l4] : Tg[l4 * 8 + 2 * q + 1];
            const int ra = 8 * P + 2 * q;
            const double ca0 = na0, ca1 = na1;
            if (pp + 1 < npan) {
                const int rn = 8 * (kFwd ? P + 1 : P - 1) + 2 * q;
                na0 = (okc && rn < n) ? Ca[rn + co] : 0.0;
                na1 = (okc && rn + 1 < n) ? Ca[rn + 1 + co] : 0.0;
            }
            const double *yP = Yb + 64 * (P * (P + 1) / 2);           // block (0, P); block (kk, P) at + 64 kk
            // groups of 4 blocks behind one uniform branch each; inside a group the
            // blocks past P read block P (a valid address) and are zeroed by a
            // select, so there is no per-block branch (their DMMAs add exact zeros)
            double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
#pragma unroll
            for (int g = 0; g < NPAN_NODE; g += 4) {
                if (g <= P) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int kk = g + u;
                        if (kk < NPAN_NODE) {
                            const bool ok = kk <= P;
                            double2 y = *reinterpret_cast<const double2 *>(yP + 64 * (ok ? kk : P) + 8 * l4 + 2 * q);
                            y.x = ok ? y.x : 0.0;
                            y.y = ok ? y.y : 0.0;
                            dmma(w0[u & 1], w1[u & 1], cb[kk][0], y.x);
                            dmma(w0[u & 1], w1[u & 1], cb[kk][1], y.y);
                        }
                    }
                }
            }
            double p0 = 0.0, p1 = 0.0;
            dmma(p0, p1, w0[0] + w0[1] + ca0, tb0);
            dmma(p0, p1, w1[0] + w1[1] + ca1, tb1);
            if (okc && ra < n) Ca[ra + co] = ca0 - p0;
            if (okc && ra + 1 < n) Ca[ra + 1 + co] = ca1 - p1;
#pragma unroll
            for (int g = 0; g < NPAN_NODE; g += 4) {
                if (g <= P) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int kk = g + u;
                        if (kk < NPAN_NODE) {
                            const bool ok = kk <= P;
                            const double *yb = yP + 64 * (ok ? kk : P);
                            const double y0 = ok ? yb[8 * (2 * q) + l4] : 0.0, y1 = ok ? yb[8 * (2 * q + 1) + l4] : 0.0;
                            dmma(cb[kk][0], cb[kk][1], -p0, y0);
                            dmma(cb[kk][0], cb[kk][1], -p1, y1);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int kk = 0; kk < NPAN_NODE; ++kk)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = 8 * kk + 2 * q + e;
                if (okc && kk < npan && r < n) Cb[r + co] = cb[kk][e];
            }
    }
    if (flags) {                                      // this node's C blocks are final
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            *reinterpret_cast<volatile int *>(flags + b) = 1;
        }
    }
}

// One stacked node's reflectors (Y1 in Rb-storage, ld ldy) applied to [Ca; Cb].
template <bool kFwd>
__global__ void __launch_bounds__(NT, 1)
k_wide_apply_node1(const double *Ra_dummy, const double *Y1, int64_t ldy, int n, const double *tcache, double *Ca,
                   int64_t ldca, double *Cb, int64_t ldcb, int k) {
    const int hA = 8 * ((n + 7) / 8);
    Prob P{const_cast<double *>(Ra_dummy), const_cast<double *>(Y1), 1, ldy, hA, n, n, 1};
    Prob Cp{Ca, Cb, ldca, ldcb, hA, n, n, 0};
    wide_apply<kFwd>(P, Cp, n, k, tcache);
}

// [X; 0] for form Q: rows 0..n-1 of every tile's Q slab <- xbuf[t], the rest 0.
__global__ void k_wide_formq_init(const int64_t *tile_row0, const int *tile_rows, int n, const double *xbuf,
                                  double *Q, int64_t ldq) {
    const int t = blockIdx.x;
    const int h = tile_rows[t];
    for (int64_t e = threadIdx.x; e < (int64_t)h * n; e += blockDim.x) {
        const int r = (int)(e % h), c = (int)(e / h);
        Q[tile_row0[t] + r + (int64_t)c * ldq] = r < n ? xbuf[(int64_t)t * n * n + r + (int64_t)c * n] : 0.0;
    }
}

// ================================================================= launchers
static size_t wide_smem() { return sizeof(Smem); }
static cudaError_t wide_attr(const void *fn) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wide_smem());
}
int wide_max_rows() { return MAXR; }

static size_t apply_leaf_smem(int max_rows, int slots) {
    const int yw = max_rows <= 1024 ? 16 : 8;                // pairs of panels only for tiles <= 1024 rows
    return sizeof(double) * (slots * yw * ((max_rows + 7) / 8 * 8) + 2 * 192);
}

template <int KM, bool kRobust>
static cudaError_t launch_leaves_km(double *A, int64_t lda, int n, const int64_t *row0, const int *rows, int L,
                                   int max_rows, double *tau, double *tcache, double *tpair, cudaStream_t st) {
    size_t bytes = LeafSmem<KM>::bytes(max_rows);
#ifdef TSQR_WIDE_MIN_SMEM
    if (bytes < TSQR_WIDE_MIN_SMEM) bytes = TSQR_WIDE_MIN_SMEM;     // variant: cap resident CTAs per SM
#endif
    cudaError_t e = cudaFuncSetAttribute((const void *)k_wide_leaves<KM, kRobust>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    k_wide_leaves<KM, kRobust><<<L, NT, bytes, st>>>(A, lda, n, row0, rows, tau, tcache, tpair);
    return cudaGetLastError();
}

template <bool kRobust>
static cudaError_t launch_leaves_r(double *A, int64_t lda, int n, const int64_t *row0, const int *rows, int L,
                                   int max_rows, double *tau, double *tcache, double *tpair, cudaStream_t st) {
    // 48 / 56 rows per warp for tiles of <= 384 / 448 rows: the steps and the row-split
    // updates skip most of the padding of KM = 8 (C3's 342-row tiles at s = 400: leaf
    // 0.928 -> 0.878 ms with KM = 7, 0.851 ms with KM = 6)
    if (max_rows <= 384) return launch_leaves_km<6, kRobust>(A, lda, n, row0, rows, L, max_rows, tau, tcache, tpair, st);
    if (max_rows <= 448) return launch_leaves_km<7, kRobust>(A, lda, n, row0, rows, L, max_rows, tau, tcache, tpair, st);
    if (max_rows <= 512) return launch_leaves_km<8, kRobust>(A, lda, n, row0, rows, L, max_rows, tau, tcache, tpair, st);
    if (max_rows <= 1024) return launch_leaves_km<16, kRobust>(A, lda, n, row0, rows, L, max_rows, tau, tcache, tpair, st);
    if (max_rows <= 1536) return launch_leaves_km<24, kRobust>(A, lda, n, row0, rows, L, max_rows, tau, tcache, tpair, st);
    return launch_leaves_km<KMW, kRobust>(A, lda, n, row0, rows, L, max_rows, tau, tcache, tpair, st);
}

// max_rows: the tallest tile (selects the per-warp row range, 64 KM >= max_rows);
// robust: the rescaled steps of reading R23
cudaError_t launch_wide_leaves(double *A, int64_t lda, int n, const int64_t *row0, const int *rows, int L,
                               int max_rows, double *tau, double *tcache, double *tpair, bool robust, cudaStream_t st) {
    return robust ? launch_leaves_r<true>(A, lda, n, row0, rows, L, max_rows, tau, tcache, tpair, st)
                  : launch_leaves_r<false>(A, lda, n, row0, rows, L, max_rows, tau, tcache, tpair, st);
}

cudaError_t launch_wide_nodes(double *A, int64_t lda, int n, const int64_t *row0, const int *node_a, const int *ids,
                              int count, double *tau_node, double *tcache_node, cudaStream_t st) {
    cudaError_t e = wide_attr((const void *)k_wide_nodes);
    if (e != cudaSuccess) return e;
    k_wide_nodes<<<count, NT, wide_smem(), st>>>(A, lda, n, row0, node_a, ids, tau_node, tcache_node);
    return cudaGetLastError();
}

cudaError_t launch_wide_node1(double *Ra, int64_t lda, double *Rb, int64_t ldb, int n, double *tau, double *tcache,
                              cudaStream_t st) {
    cudaError_t e = wide_attr((const void *)k_wide_node1);
    if (e != cudaSuccess) return e;
    k_wide_node1<<<1, NT, wide_smem(), st>>>(Ra, lda, Rb, ldb, n, tau, tcache);
    return cudaGetLastError();
}

cudaError_t launch_wide_apply_leaves(const double *A, int64_t lda, int n, const int64_t *row0, const int *rows,
                                     int L, int max_rows, const double *tcache, const double *tpair, double *C,
                                     int64_t ldc, int k, int forward, cudaStream_t st) {
    const int pairs = max_rows <= 1024;                      // the factor cached T01 (wide_leaf_qr, KM <= 16)
#ifndef TSQR_NO_APPLY_REG
    constexpr int MR = 44;                                     // register-resident slab: tiles <= 352 rows
    if (pairs && k <= 64 && max_rows <= 8 * MR) {
        const size_t rb = sizeof(double) * (2 * 192 + 2 * (size_t)(8 * ((max_rows + 7) / 8)) * 16);
        const void *fr = forward ? (const void *)k_wide_apply_leaves_reg<true, MR>
                                 : (const void *)k_wide_apply_leaves_reg<false, MR>;
        cudaError_t er = cudaFuncSetAttribute(fr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rb);
        if (er != cudaSuccess) return er;
        if (forward)
            k_wide_apply_leaves_reg<true, MR><<<L, NT, rb, st>>>(A, lda, n, row0, rows, tcache, tpair, C, ldc, k);
        else
            k_wide_apply_leaves_reg<false, MR><<<L, NT, rb, st>>>(A, lda, n, row0, rows, tcache, tpair, C, ldc, k);
        return cudaGetLastError();
    }
#endif
    const int slots = apply_leaf_smem(max_rows, 2) <= 227 * 1024 ? 2 : 1;   // prefetch the next group if it fits
    const size_t bytes = apply_leaf_smem(max_rows, slots);
    const void *fn = forward ? (const void *)k_wide_apply_leaves<true> : (const void *)k_wide_apply_leaves<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    if (forward)
        k_wide_apply_leaves<true><<<L, NT, bytes, st>>>(A, lda, n, row0, rows, tcache, tpair, pairs, C, ldc, k,
                                                        slots == 2);
    else
        k_wide_apply_leaves<false><<<L, NT, bytes, st>>>(A, lda, n, row0, rows, tcache, tpair, pairs, C, ldc, k,
                                                         slots == 2);
    return cudaGetLastError();
}

cudaError_t launch_node_apply(const double *A, int64_t lda, int n, const int64_t *row0, const int *node_a,
                                    const int *ids, int count, const double *tcache_node, double *C, int64_t ldc,
                                    int k, int forward, int xbuf_mode, cudaStream_t st) {
    const int npan = (n + 7) / 8;
    if (npan <= NPAN_NODE) {
        const size_t bytes = sizeof(double) * 64 * (npan * (npan + 1) / 2 + npan);
        auto go = [&](auto kf, auto np) -> cudaError_t {
            constexpr bool F = decltype(kf)::value;
            constexpr int NPM = decltype(np)::value;
            cudaError_t e = cudaFuncSetAttribute((const void *)k_node_apply<F, NPM>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
            if (e != cudaSuccess) return e;
            k_node_apply<F, NPM><<<count, NT, bytes, st>>>(A, lda, n, row0, node_a, ids, tcache_node, C, ldc,
                                                                     k, xbuf_mode, nullptr, 0, nullptr, nullptr, nullptr);
            return cudaGetLastError();
        };
        using T8 = std::integral_constant<int, 8>;
        using T28 = std::integral_constant<int, NPAN_NODE>;
        if (forward) return npan <= 8 ? go(std::true_type(), T8()) : go(std::true_type(), T28());
        return npan <= 8 ? go(std::false_type(), T8()) : go(std::false_type(), T28());
    }
    if (forward)
        k_wide_apply_nodes<true><<<count, NT, 0, st>>>(A, lda, n, row0, node_a, ids, tcache_node, C, ldc, k, xbuf_mode);
    else
        k_wide_apply_nodes<false><<<count, NT, 0, st>>>(A, lda, n, row0, node_a, ids, tcache_node, C, ldc, k, xbuf_mode);
    return cudaGetLastError();
}

bool node_ppipe_disabled();

// The whole tree's node stage in one launch (k_node_apply with flags), npan <= 28:
// ids = every node in dependency order; flags[L + 1] scratch (zeroed here).
cudaError_t launch_node_apply_pipe(const double *A, int64_t lda, int n, const int64_t *row0, const int *node_a,
                                   const int *ids, int count, const int *dep0, const int *dep1, int *flags, int L,
                                   const double *tcache_node, double *C, int64_t ldc, int k, int forward,
                                   int xbuf_mode, cudaStream_t st) {
    const int npan = (n + 7) / 8;
    if (npan > NPAN_NODE) return cudaErrorNotSupported;
    if (count == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (L + 1), st);
    if (e != cudaSuccess) return e;
    // per-(node, 8-column slab, panel) flags of the panel-level pipeline, stream-ordered; for
    // npan > 8 only: C3 apply Q^T 0.852 -> 0.600 ms, form Q at n = 200 2.83 -> 1.96 ms, but
    // with <= 8 panels the per-panel publish costs more than the overlap gains (C5 apply Q^T
    // 23.9 -> 24.3 ms, C4 form Q 11.40 -> 11.68 ms, C2 0.816 -> 0.863 ms)
    int *pflags = nullptr;
    const bool pp_on = npan > 8 && (forward ? !xbuf_mode : true);
    const size_t pf_ints = pp_on ? (size_t)L * ((k + 7) / 8) * npan : 0;
    if (pf_ints > 0 && !node_ppipe_disabled()) {
        e = cudaMallocAsync((void **)&pflags, sizeof(int) * pf_ints, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(pflags, 0, sizeof(int) * pf_ints, st);
        if (e != cudaSuccess) return e;
    }
    const size_t bytes = sizeof(double) * 64 * (npan * (npan + 1) / 2 + npan);
    auto go = [&](auto kf, auto np) -> cudaError_t {
        constexpr bool F = decltype(kf)::value;
        constexpr int NPM = decltype(np)::value;
        cudaError_t r = cudaFuncSetAttribute((const void *)k_node_apply<F, NPM>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (r != cudaSuccess) return r;
        k_node_apply<F, NPM><<<count, NT, bytes, st>>>(A, lda, n, row0, node_a, ids, tcache_node, C, ldc, k,
                                                       xbuf_mode, flags, L, dep0, dep1, pflags);
        return cudaGetLastError();
    };
    using T8 = std::integral_constant<int, 8>;
    using T28 = std::integral_constant<int, NPAN_NODE>;
    if (forward) e = npan <= 8 ? go(std::true_type(), T8()) : go(std::true_type(), T28());
    else e = npan <= 8 ? go(std::false_type(), T8()) : go(std::false_type(), T28());
    if (pflags) {
        const cudaError_t f = cudaFreeAsync(pflags, st);
        if (e == cudaSuccess) e = f;
    }
    return e;
}

// TSQR_NO_NODE_PPIPE=1 in the environment: node-level hand-offs only (A/B)
bool node_ppipe_disabled() {
    const char *v = std::getenv("TSQR_NO_NODE_PPIPE");
    return v && *v == '1';
}

cudaError_t launch_wide_apply_node1(const double *Y1, int64_t ldy, int n, const double *tcache, double *Ca,
                                    int64_t ldca, double *Cb, int64_t ldcb, int k, int forward, cudaStream_t st) {
    if (forward) k_wide_apply_node1<true><<<1, NT, 0, st>>>(Y1, Y1, ldy, n, tcache, Ca, ldca, Cb, ldcb, k);
    else k_wide_apply_node1<false><<<1, NT, 0, st>>>(Y1, Y1, ldy, n, tcache, Ca, ldca, Cb, ldcb, k);
    return cudaGetLastError();
}

cudaError_t launch_wide_formq_init(const int64_t *row0, const int *rows, int L, int n, const double *xbuf, double *Q,
                                   int64_t ldq, cudaStream_t st) {
    k_wide_formq_init<<<L, 256, 0, st>>>(row0, rows, n, xbuf, Q, ldq);
    return cudaGetLastError();
}

}  // namespace tsqr

namespace tsqr {

// ------------------------------------------------------------ small helpers
// R (n x n, ldr) <- upper triangle of A's head rows, exact zeros below.
__global__ void k_extract_r(const double *A, int64_t lda, int n, double *R, int64_t ldr) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x) {
        const int r = e % n, c = e / n;
        R[r + (int64_t)c * ldr] = r <= c ? A[r + (int64_t)c * lda] : 0.0;
    }
}
cudaError_t launch_extract_r(const double *A, int64_t lda, int n, double *R, int64_t ldr, cudaStream_t st) {
    k_extract_r<<<(n * n + 255) / 256, 256, 0, st>>>(A, lda, n, R, ldr);
    return cudaGetLastError();
}

// Butterfly round, wide n: tmp (2n x n, ld 2n) <- [R_lower; R_upper] from this
// rank's head (upper triangle) and the partner's packed R.
__global__ void k_wide_stack(const double *Ahead, int64_t lda, const double *packed, int is_lower, int n,
                             double *tmp) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x) {
        const int r = e % n, c = e / n;
        const double mine = r <= c ? Ahead[r + (int64_t)c * lda] : 0.0;
        const double theirs = r <= c ? packed[(int64_t)c * (c + 1) / 2 + r] : 0.0;
        tmp[r + (int64_t)c * 2 * n] = is_lower ? mine : theirs;
        tmp[n + r + (int64_t)c * 2 * n] = is_lower ? theirs : mine;
    }
}
// After the node: this rank's head (upper) and R <- the new R; Y1 (ld n) <- the
// bottom's upper triangle.
__global__ void k_wide_unstack(const double *tmp, int n, double *Ahead, int64_t lda, double *R, int64_t ldr,
                               double *Y1) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x) {
        const int r = e % n, c = e / n;
        const double rv = r <= c ? tmp[r + (int64_t)c * 2 * n] : 0.0;
        if (r <= c) Ahead[r + (int64_t)c * lda] = rv;
        if (R) R[r + (int64_t)c * ldr] = rv;
        Y1[r + (int64_t)c * n] = r <= c ? tmp[n + r + (int64_t)c * 2 * n] : 0.0;
    }
}
cudaError_t launch_wide_cross_factor(double *A, int64_t lda, int n, const double *packed, int is_lower, double *tmp,
                                     double *Y1, double *tau, double *tcache, double *R, int64_t ldr,
                                     cudaStream_t st) {
    const int blocks = (n * n + 255) / 256;
    k_wide_stack<<<blocks, 256, 0, st>>>(A, lda, packed, is_lower, n, tmp);
    cudaError_t e = launch_wide_node1(tmp, 2 * n, tmp + n, 2 * n, n, tau, tcache, st);
    if (e != cudaSuccess) return e;
    k_wide_unstack<<<blocks, 256, 0, st>>>(tmp, n, A, lda, R, ldr, Y1);
    return cudaGetLastError();
}

// Butterfly round of Q^T C, wide n: tmp (2n x k, ld 2n) <- [top_lower; top_upper],
// the round's node reflectors applied, then top <- tmp's top half and C's head
// rows per head_role (1: the R coordinates, 2: the complement).
__global__ void k_wide_stack_c(const double *top, int64_t ldtop, const double *ptop, int is_lower, int n, int k,
                               double *tmp) {
    for (int64_t e = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; e < (int64_t)n * k; e += (int64_t)blockDim.x * gridDim.x) {
        const int r = (int)(e % n);
        const int64_t c = e / n;
        const double mine = top[r + c * ldtop], theirs = ptop[r + c * n];
        tmp[r + c * 2 * n] = is_lower ? mine : theirs;
        tmp[n + r + c * 2 * n] = is_lower ? theirs : mine;
    }
}
__global__ void k_wide_unstack_c(const double *tmp, int n, int k, double *top, int64_t ldtop, int role, double *C,
                                 int64_t ldc) {
    for (int64_t e = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; e < (int64_t)n * k; e += (int64_t)blockDim.x * gridDim.x) {
        const int r = (int)(e % n);
        const int64_t c = e / n;
        const double ra = tmp[(role == 3 ? n : 0) + r + c * 2 * n];     // role 3 (Q C): the upper half
        top[r + c * ldtop] = ra;
        if (role == 1 || role == 3) C[r + c * ldc] = ra;
        if (role == 2) C[r + c * ldc] = tmp[n + r + c * 2 * n];
    }
}
cudaError_t launch_wide_cross_apply(const double *Y1, const double *tcache, double *top, int64_t ldtop,
                                    const double *ptop, int is_lower, int role, double *C, int64_t ldc, int n, int k,
                                    double *tmp, int forward, cudaStream_t st) {
    const int64_t tot = (int64_t)n * k;
    const int blocks = (int)((tot + 255) / 256 < 4096 ? (tot + 255) / 256 : 4096);
    k_wide_stack_c<<<blocks, 256, 0, st>>>(top, ldtop, ptop, is_lower, n, k, tmp);
    cudaError_t e = launch_wide_apply_node1(Y1, n, n, tcache, tmp, 2 * n, tmp + n, 2 * n, k, forward, st);
    if (e != cudaSuccess) return e;
    if (!forward) role = is_lower ? 1 : 3;                  // Q C: keep this rank's half
    k_wide_unstack_c<<<blocks, 256, 0, st>>>(tmp, n, k, top, ldtop, role, C, ldc);
    return cudaGetLastError();
}

// Root X of this rank for form Q, wide n: top-down over the butterfly rounds,
// [X_lower; X_upper] = Q_round [X; 0], keep this rank's half.
__global__ void k_wide_x_init(double *tmp, int n) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < 2 * n * n; e += blockDim.x * gridDim.x) {
        const int r = e % (2 * n), c = e / (2 * n);
        tmp[e] = (r == c) ? 1.0 : 0.0;
    }
}
__global__ void k_wide_x_pick(double *tmp, int n, int upper, double *X0, int last) {
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < n * n; e += blockDim.x * gridDim.x) {
        const int r = e % n, c = e / n;
        const double v = tmp[(upper ? n : 0) + r + (int64_t)c * 2 * n];
        tmp[r + (int64_t)c * 2 * n] = v;
        tmp[n + r + (int64_t)c * 2 * n] = 0.0;
        if (last) X0[r + (int64_t)c * n] = v;
    }
}
cudaError_t launch_wide_cross_root_x(const double *Y1s, const double *tcaches, int64_t tstride, int rounds, int rank,
                                     int n, double *tmp, double *X0, cudaStream_t st) {
    const int blocks = (2 * n * n + 255) / 256;
    k_wide_x_init<<<blocks, 256, 0, st>>>(tmp, n);
    if (rounds == 0) {
        k_wide_x_pick<<<blocks, 256, 0, st>>>(tmp, n, 0, X0, 1);
        return cudaGetLastError();
    }
    for (int kr = rounds; kr >= 1; --kr) {
        cudaError_t e = launch_wide_apply_node1(Y1s + (int64_t)(kr - 1) * n * n, n, n, tcaches + (kr - 1) * tstride,
                                                tmp, 2 * n, tmp + n, 2 * n, n, 0, st);
        if (e != cudaSuccess) return e;
        const int upper = ((rank >> (kr - 1)) & 1) != 0;
        k_wide_x_pick<<<blocks, 256, 0, st>>>(tmp, n, upper, X0, kr == 1);
    }
    return cudaGetLastError();
}

}  // namespace tsqr
