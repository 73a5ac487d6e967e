// Column-split chunk engine of the B200 TSQR leaf path (sm_100a).  Product code.
//
// Same algorithm as chunk.cuh -- every tile is a flat chain ("sequential
// TSQR"; [TR] P:1725-1753) over chunks of CH rows, chunk k merged
// into the running R by qr([R; A_k]) -- but one chunk is held by a GROUP of NG
// warps that split its columns: warp wl owns the column blocks (8 columns
// each) of its slots (snake order over the group).  With one block per warp
// (NG = NCB, the configurations used) warp p owns column block p of every
// chunk, so the group is a systolic pipeline over panels: warp p applies the
// Y_0..Y_{p-1} of chunk s to its block, factors panel p, and moves on to chunk
// s+1 while warps p+1.. still work on chunk s.  A warp holds its block for
// all CH rows in registers as DMMA fragments:
//     a[k][j][e] = A(chunk row 8k + 2q + e, column 8 blk(wl, j) + l4),
// so one Householder step covers CH = 8 KM = 256 rows for the register budget
// that covers 32 rows when one warp owns all 64 columns.
//   panel p (its owner):  the Householder steps (warp shuffles + a
//       double-buffered smem row for the pivot column), T (compact WY,
//       Alg. YT:scaled P:2007-2028 in the LAPACK sign, reading R3), then Y_p
//       and T_p are published in the group's exchange slot for p;
//   every block b > p (its owner): W^T = C_b^T Y_p (+ R rows 8p..8p+7 of b),
//       W'^T = W^T T_p, R rows -= W', C_b -= Y_p W' on FP64 DMMA.
// R lives in shared memory (one buffer per group, row-major) and its columns
// are owned like the chunk's: only the owner of block b ever touches R(:, b),
// so consecutive chunks of a tile need no hand-off for R at all; the only
// cross-warp synchronisation is per panel: ready[p] (Y_p of chunk s is in the
// slot) and done[p] (applications of Y_p finished, so the slot may be reused).
#pragma once
#include <cstdint>
#include "chunk.cuh"

namespace tsqr {
namespace cs {

using chunk::build_t;
using chunk::House;
using chunk::house_bf;
using wy::dmma;
constexpr unsigned FULL = 0xffffffffu;

template <int NCB_, int KM_, int NG_, int NGRP_>
struct Cfg {
    static constexpr int NCB = NCB_, KM = KM_, NG = NG_, NGRP = NGRP_;
    static constexpr int NP = 8 * NCB, CH = 8 * KM, NW = NG * NGRP, NT = 32 * NW;
    static constexpr int NBW = (NCB + NG - 1) / NG;       // block slots per warp
    static constexpr int LDR = NP + 2;                     // R: R(i, c) at [i * LDR + c]
    static constexpr int RBUF = NP * LDR;
    static constexpr int YSLOT = CH * 8 + 64;              // Y_p (row-major CH x 8) + T_p (row-major 8x8)
    static constexpr int GS = 0, T8 = 64, TS = 72, XS = 136, WSCR = XS + 2 * CH;   // per warp
    static constexpr int OFF_R = 0;
    static constexpr int OFF_Y = OFF_R + NGRP * RBUF;
    static constexpr int OFF_W = OFF_Y + NGRP * NCB * YSLOT;
    static constexpr int OFF_SYNC = OFF_W + NW * WSCR;     // per group: ready[NCB], done[NCB]
    static constexpr size_t BYTES = (size_t)OFF_SYNC * sizeof(double) + (size_t)NGRP * 2 * NCB * sizeof(int);
    // block of slot j of warp wl (snake order), -1 if none
    __device__ static int blk(int wl, int j) {
        const int b = (j & 1) ? j * NG + NG - 1 - wl : j * NG + wl;
        return b < NCB ? b : -1;
    }
    // owner warp of block p (its slot is p / NG)
    __device__ static int owner(int p) {
        const int r = p / NG, pos = p % NG;
        return (r & 1) ? NG - 1 - pos : pos;
    }
};

template <class C>
struct Regs {
    double a[C::KM][C::NBW][2];
};

__device__ __forceinline__ void wait_ge(const int *c, int v) {
    while (*reinterpret_cast<const volatile int *>(c) < v) {
    }
    asm volatile("" ::: "memory");
}
__device__ __forceinline__ void publish(int *c, int v) {
    asm volatile("" ::: "memory");
    __syncwarp();
    if ((threadIdx.x & 31) == 0) *reinterpret_cast<volatile int *>(c) = v;
}
__device__ __forceinline__ void bump(int *c) {
    asm volatile("" ::: "memory");
    __syncwarp();
    if ((threadIdx.x & 31) == 0) atomicAdd(c, 1);
}

// ---------------------------------------------------------------- the panel
// Householder steps of panel P (runtime) on the warp's block (slot 0).
//   kDense = false: pivots are R rows 8P .. 8P+7 (smem Rb), the tail is the whole chunk;
//   kDense = true:  pivots are chunk rows 8P .. 8P+7 (head chunk, r0 = 0, row block P).
// On exit the block holds v below the pivots (dense: R at/above them), Gs the
// Gram entries, t8 the taus.  P is a runtime value so that one copy of the code
// serves every warp (I-cache); register arrays are only indexed by unrolled k.
template <class C, bool kDense>
__device__ __forceinline__ void panel_steps(Regs<C> &rg, int P, double *Rb, double *Gs, double *t8, double *xs) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    constexpr int KM = C::KM;
    if (l4 == 0) {
#pragma unroll
        for (int k = 0; k < KM; ++k)
            *reinterpret_cast<double2 *>(xs + 8 * k + 2 * q) = make_double2(rg.a[k][0][0], rg.a[k][0][1]);
    }
    __syncwarp();
#pragma unroll 1
    for (int jj = 0; jj < 8; ++jj) {
        const int j = 8 * P + jj;
        const double *xr = xs + (jj & 1) * C::CH;
        // partial dots over this lane's rows: d = x^T a(:, col), s2 = x^T x (x masked
        // to the rows below the pivot for a dense panel)
        double d[4] = {0.0, 0.0, 0.0, 0.0}, s[4] = {0.0, 0.0, 0.0, 0.0};
        double sel = 0.0;
#pragma unroll
        for (int k = 0; k < KM; ++k) {
            double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
            if (kDense) {
                xv.x = (k > P || (k == P && 2 * q > jj)) ? xv.x : 0.0;
                xv.y = (k > P || (k == P && 2 * q + 1 > jj)) ? xv.y : 0.0;
                sel = (k == P) ? ((jj & 1) ? rg.a[k][0][1] : rg.a[k][0][0]) : sel;
            }
            d[k & 3] = fma(xv.x, rg.a[k][0][0], d[k & 3]);
            d[(k + 2) & 3] = fma(xv.y, rg.a[k][0][1], d[(k + 2) & 3]);
            s[k & 3] = fma(xv.x, xv.x, s[k & 3]);
            s[(k + 2) & 3] = fma(xv.y, xv.y, s[(k + 2) & 3]);
        }
        double dd = (d[0] + d[1]) + (d[2] + d[3]), s2 = (s[0] + s[1]) + (s[2] + s[3]);
        dd += __shfl_xor_sync(FULL, dd, 1);
        s2 += __shfl_xor_sync(FULL, s2, 1);
        dd += __shfl_xor_sync(FULL, dd, 2);
        s2 += __shfl_xor_sync(FULL, s2, 2);
        double alpha, rj;
        if (kDense) {
            rj = __shfl_sync(FULL, sel, 4 * l4 + (jj >> 1));          // A(pivot row, 8P + l4)
            alpha = __shfl_sync(FULL, rj, 4 * jj);
        } else {
            alpha = Rb[j * C::LDR + j];
            rj = Rb[j * C::LDR + 8 * P + l4];                           // R(j, 8P + l4)
        }
        const House h = house_bf(alpha, s2);
        const double w = fma(h.scale, dd, rj);
        const double u = (l4 > jj) ? h.tau * h.scale * w : (l4 == jj ? 1.0 : 0.0);
        const double g = (l4 == jj) ? h.scale : 0.0;                 // pivot column: v = scale x exactly
        const double pnew = (l4 > jj) ? fma(-h.tau, w, rj) : (l4 == jj ? h.beta : rj);
        const bool nxt = (l4 == jj + 1);
        double *xw = xs + ((jj + 1) & 1) * C::CH;
        asm volatile("" ::: "memory");      // re-load x below rather than keep KM x 2 values live
#pragma unroll
        for (int k = 0; k < KM; ++k) {
            double2 xv = *reinterpret_cast<const double2 *>(xr + 8 * k + 2 * q);
            if (kDense) {
                xv.x = (k > P || (k == P && 2 * q > jj)) ? xv.x : 0.0;
                xv.y = (k > P || (k == P && 2 * q + 1 > jj)) ? xv.y : 0.0;
            }
            double a0 = fma(g, xv.x, fma(-u, xv.x, rg.a[k][0][0])), a1 = fma(g, xv.y, fma(-u, xv.y, rg.a[k][0][1]));
            if (kDense) {                                                // the pivot row
                const bool pr = (k == P) && (q == (jj >> 1));
                a0 = (pr && !(jj & 1)) ? pnew : a0;
                a1 = (pr && (jj & 1)) ? pnew : a1;
            }
            rg.a[k][0][0] = a0;
            rg.a[k][0][1] = a1;
            if (nxt) *reinterpret_cast<double2 *>(xw + 8 * k + 2 * q) = make_double2(a0, a1);
        }
        __syncwarp();                   // all lanes read R(j, .) / xs before they change
        if (!kDense) {
            if (q == 0 && l4 >= jj) Rb[j * C::LDR + 8 * P + l4] = pnew;
        }
        if (q == 0 && l4 < jj) Gs[l4 * 8 + jj] = kDense ? fma(h.scale, dd, rj) : h.scale * dd;
        if (lane == 0) t8[jj] = h.tau;
        __syncwarp();
    }
}

// Apply the panel P (runtime) whose Y (row-major CH x 8) and T follow in ys to
// the warp's block b: C_b <- (I - Y T^T Y^T) C_b, with the R rows 8P..8P+7 of
// columns b as the identity part when !kDense.
template <class C, bool kDense>
__device__ __forceinline__ void apply_block(Regs<C> &rg, int P, const double *ys, double *Rb, int b) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    constexpr int KM = C::KM;
    const double *Tg = ys + C::CH * 8;
    double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};     // two accumulation chains
#pragma unroll
    for (int k = 0; k < KM; ++k) {
        const double y0 = ys[(8 * k + 2 * q) * 8 + l4], y1 = ys[(8 * k + 2 * q + 1) * 8 + l4];
        dmma(w0[k & 1], w1[k & 1], rg.a[k][0][0], y0);
        dmma(w0[k & 1], w1[k & 1], rg.a[k][0][1], y1);
    }
    double wt0 = w0[0] + w0[1], wt1 = w1[0] + w1[1];      // W^T[col l4][refl 2q+{0,1}]
    double *r0p = Rb + (8 * P + 2 * q) * C::LDR + 8 * b + l4;
    if (!kDense) {
        wt0 += r0p[0];
        wt1 += r0p[C::LDR];
    }
    double p0 = 0.0, p1 = 0.0;
    dmma(p0, p1, wt0, Tg[(2 * q) * 8 + l4]);
    dmma(p0, p1, wt1, Tg[(2 * q + 1) * 8 + l4]);
    if (!kDense) {
        r0p[0] -= p0;
        r0p[C::LDR] -= p1;
    }
#pragma unroll
    for (int k = 0; k < KM; ++k) {
        const double2 yt = *reinterpret_cast<const double2 *>(ys + (8 * k + l4) * 8 + 2 * q);
        dmma(rg.a[k][0][0], rg.a[k][0][1], -p0, yt.x);
        dmma(rg.a[k][0][0], rg.a[k][0][1], -p1, yt.y);
    }
}

// Chunk row block P (runtime) of the warp's block b -> R rows 8P..8P+7 (dense head chunk).
template <class C>
__device__ __forceinline__ void rows_to_r(const Regs<C> &rg, int P, double *Rb, int b) {
    const int lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int k = 0; k < C::KM; ++k) {
        v0 = (k == P) ? rg.a[k][0][0] : v0;
        v1 = (k == P) ? rg.a[k][0][1] : v1;
    }
    Rb[(8 * P + 2 * q) * C::LDR + 8 * b + l4] = v0;
    Rb[(8 * P + 2 * q + 1) * C::LDR + 8 * b + l4] = v1;
}

}  // namespace cs
}  // namespace tsqr
