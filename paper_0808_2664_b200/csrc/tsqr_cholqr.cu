// CholeskyQR on the GPU: the comparison method of SURVEY 8(f) row 4, not the
// TSQR path.  Alg. CholeskyQR ([TR] P:1410-1419):
//     line 1  W := A^T A              (all-reduction across ranks: tsqr_ctx_cholqr)
//     line 2  W = L L^T  (R := L^T)
//     line 3  Q := A L^{-T} = A R^{-1}
// "the Q factor computed by CholeskyQR loses orthogonality proportionally to
// kappa_2(A)^2"; TSQR's does not -- the stability half of
// "only parallel TSQR is simultaneously fastest and stable".
//
// Kernels (sm_100a, FP64 DMMA for the two dense contractions):
//   k_gram_tile    partial W tiles (32 x 32) of a row range: each warp streams
//                  8-row groups, W_IJ += A_I^T A_J on DMMA.8x8x4 (the contraction
//                  runs over 4 rows), warps reduced through smem; grid = row
//                  splits x upper tile pairs (W is symmetric)
//   k_gram_reduce  W = sum of the splits' partials in split order (deterministic),
//                  mirrored to the full symmetric matrix
//   k_chol_inv     one CTA: right-looking Cholesky of W (smem for n <= 128),
//                  breakdown -> *info = j + 1; then R^{-1} row by row (a warp per
//                  column, lanes split the inner sum)
//   k_qmul         Q = A R^{-1} on DMMA (contraction over A's columns), R^{-1}'s
//                  column pass in smem (ld = 4 mod 16: conflict-free B fragments),
//                  persistent CTAs over 128-row blocks, the zero blocks of the
//                  triangle skipped.
// Product code (a comparison path beside the product TSQR).
#include "../../include/tsqr.h"
#include "tsqr_kernels.h"
#include "wy.cuh"

#include <cuda_runtime.h>

#include <algorithm>

namespace tsqr {
namespace {

using wy::dmma;

constexpr int GT = 32;          // W tile edge
constexpr int QLD = 68;         // smem ld of R^{-1}'s column pass (4 mod 16)

__device__ __forceinline__ void tile_pair(int p, int nt, int &ti, int &tj) {
    ti = 0;
    while (p >= nt - ti) {
        p -= nt - ti;
        ++ti;
    }
    tj = ti + p;
}

__global__ void __launch_bounds__(256) k_gram_tile(const double *A, int64_t lda, int64_t m, int n, int64_t rows_per_split,
                                                   double *part) {
    __shared__ double red[4][GT * GT];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int nt = (n + GT - 1) / GT, ntp = nt * (nt + 1) / 2;
    int ti, tj;
    tile_pair(blockIdx.y, nt, ti, tj);
    const int64_t lo = blockIdx.x * rows_per_split, hi = min(m, lo + rows_per_split);
    double acc[4][4][2];
#pragma unroll
    for (int I = 0; I < 4; ++I)
#pragma unroll
        for (int J = 0; J < 4; ++J) acc[I][J][0] = acc[I][J][1] = 0.0;
    int ci[4], cj[4];
#pragma unroll
    for (int X = 0; X < 4; ++X) {
        ci[X] = GT * ti + 8 * X + l4;
        cj[X] = GT * tj + 8 * X + l4;
    }
    for (int64_t g = lo + 8 * warp; g < hi; g += 64) {
        double aI[4][2], aJ[4][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int64_t r = g + 2 * q + e;
            const bool rok = r < hi;
#pragma unroll
            for (int X = 0; X < 4; ++X) {
                aI[X][e] = (rok && ci[X] < n) ? A[r + (int64_t)ci[X] * lda] : 0.0;
                aJ[X][e] = (rok && cj[X] < n) ? A[r + (int64_t)cj[X] * lda] : 0.0;
            }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int I = 0; I < 4; ++I)
#pragma unroll
                for (int J = 0; J < 4; ++J) dmma(acc[I][J][0], acc[I][J][1], aI[I][e], aJ[J][e]);
    }
    // D(l4, 2q + e) of block (I, J) = W(32 ti + 8I + l4, 32 tj + 8J + 2q + e); the 8 warps'
    // tiles summed as a fixed binary tree through smem (8 -> 4 -> 2 -> 1)
    for (int half = 4; half >= 1; half >>= 1) {
        if (warp >= half && warp < 2 * half) {
#pragma unroll
            for (int I = 0; I < 4; ++I)
#pragma unroll
                for (int J = 0; J < 4; ++J)
#pragma unroll
                    for (int e = 0; e < 2; ++e) red[warp - half][(8 * I + l4) * GT + 8 * J + 2 * q + e] = acc[I][J][e];
        }
        __syncthreads();
        if (warp < half) {
#pragma unroll
            for (int I = 0; I < 4; ++I)
#pragma unroll
                for (int J = 0; J < 4; ++J)
#pragma unroll
                    for (int e = 0; e < 2; ++e) acc[I][J][e] += red[warp][(8 * I + l4) * GT + 8 * J + 2 * q + e];
        }
        __syncthreads();
    }
    if (warp == 0) {
        double *out = part + ((int64_t)blockIdx.x * ntp + blockIdx.y) * (GT * GT);
#pragma unroll
        for (int I = 0; I < 4; ++I)
#pragma unroll
            for (int J = 0; J < 4; ++J)
#pragma unroll
                for (int e = 0; e < 2; ++e) out[(8 * I + l4) * GT + 8 * J + 2 * q + e] = acc[I][J][e];
    }
}

__global__ void k_gram_reduce(const double *part, int nsplit, int n, double *W) {
    const int nt = (n + GT - 1) / GT, ntp = nt * (nt + 1) / 2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx % n), j = (int)(idx / n);
        if (i > j) continue;
        const int ti = i / GT, tj = j / GT;
        const int tp = ti * nt - ti * (ti - 1) / 2 + (tj - ti);
        const int li = i - GT * ti, lj = j - GT * tj;
        double s = 0.0;
        for (int k = 0; k < nsplit; ++k) s += part[((int64_t)k * ntp + tp) * (GT * GT) + li * GT + lj];
        W[i + (int64_t)j * n] = s;
        W[j + (int64_t)i * n] = s;
    }
}

// Cholesky W = R^T R (upper R, positive diagonal) and R^{-1}.  S: the working
// copy of W (smem when it fits, else W itself in global memory), column-major ld n.
__global__ void __launch_bounds__(256) k_chol_inv(double *W, int n, double *R, int64_t ldr, double *Rinv, int *info,
                                                  int use_smem) {
    extern __shared__ double sm[];
    __shared__ double piv;
    __shared__ int bad;
    double *S = use_smem ? sm : W;
    const int tid = threadIdx.x, nth = blockDim.x;
    if (use_smem)
        for (int i = tid; i < n * n; i += nth) S[i] = W[i];
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        if (tid == 0) {
            const double d = S[j + (int64_t)j * n];
            if (!(d > 0.0)) bad = j + 1;                 // not positive definite (or NaN)
            else piv = sqrt(d);
        }
        __syncthreads();
        if (bad) break;
        const double r = piv;
        for (int c = j + 1 + tid; c < n; c += nth) S[j + (int64_t)c * n] /= r;
        if (tid == 0) S[j + (int64_t)j * n] = r;
        __syncthreads();
        const int w = n - j - 1;
        for (int idx = tid; idx < w * w; idx += nth) {
            const int i = j + 1 + idx / w, c = j + 1 + idx % w;
            if (i <= c) S[i + (int64_t)c * n] -= S[j + (int64_t)i * n] * S[j + (int64_t)c * n];
        }
        __syncthreads();
    }
    if (tid == 0) *info = bad;
    if (bad) return;
    for (int idx = tid; idx < n * n; idx += nth) {
        const int i = idx % n, c = idx / n;
        R[i + (int64_t)c * ldr] = i <= c ? S[i + (int64_t)c * n] : 0.0;
        Rinv[idx] = 0.0;
    }
    __syncthreads();
    // R^{-1} (upper): row i from the rows below it, i = n-1 .. 0:
    //   X(i,i) = 1/R(i,i),  X(i,j) = -X(i,i) sum_{k=i+1..j} R(i,k) X(k,j)
    const int warp = tid >> 5, lane = tid & 31, nw = nth >> 5;
    for (int i = n - 1; i >= 0; --i) {
        const double dinv = 1.0 / S[i + (int64_t)i * n];
        for (int j = i + warp; j < n; j += nw) {
            double s = 0.0;
            for (int k = i + 1 + lane; k <= j; k += 32) s = fma(S[i + (int64_t)k * n], Rinv[k + (int64_t)j * n], s);
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) Rinv[i + (int64_t)j * n] = (j == i) ? dinv : -dinv * s;
        }
        __syncthreads();
    }
}

// Q (m x n) = A R^{-1}: warp tile 16 rows x 64 columns (two 8-row groups x eight
// 8-column blocks); CTA = 8 warps = 128 rows; persistent over row blocks per pass.
__global__ void __launch_bounds__(256) k_qmul(const double *A, int64_t lda, int64_t m, int n, const double *Rinv,
                                              double *Q, int64_t ldq, const int *info) {
    extern __shared__ double sR[];               // (n rounded to 4) x 64 slice of R^{-1}, row-major ld QLD
    if (*info != 0) return;                      // Cholesky broke down: Q is not formed
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, l4 = lane >> 2;
    const int npass = (n + 63) / 64;
    const int64_t nblk = (m + 127) / 128;
    for (int pass = 0; pass < npass; ++pass) {
        const int j0 = 64 * pass;
        __syncthreads();
        const int n4 = (n + 3) & ~3;               // the K loop reads rows up to n rounded to 4
        for (int idx = threadIdx.x; idx < n4 * 64; idx += blockDim.x) {
            const int l = idx / 64, jj = idx % 64;
            sR[l * QLD + jj] = (l < n && j0 + jj < n) ? Rinv[l + (int64_t)(j0 + jj) * n] : 0.0;
        }
        __syncthreads();
        const int kend = min(n, j0 + 64);          // R^{-1}(l, j) = 0 for l > j
        for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
            const int64_t r0 = blk * 128 + 16 * warp;
            double acc[2][8][2];
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int J = 0; J < 8; ++J) acc[g][J][0] = acc[g][J][1] = 0.0;
            const int64_t ra = r0 + l4, rb = r0 + 8 + l4;
            const bool oka = ra < m, okb = rb < m;
#pragma unroll 4
            for (int l0 = 0; l0 < kend; l0 += 4) {
                const int l = l0 + q;
                const double a0 = (oka && l < n) ? A[ra + (int64_t)l * lda] : 0.0;
                const double a1 = (okb && l < n) ? A[rb + (int64_t)l * lda] : 0.0;
#pragma unroll
                for (int J = 0; J < 8; ++J) {
                    if (l0 <= j0 + 8 * J + 7) {
                        const double b = sR[l * QLD + 8 * J + l4];
                        dmma(acc[0][J][0], acc[0][J][1], a0, b);
                        dmma(acc[1][J][0], acc[1][J][1], a1, b);
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const int64_t r = r0 + 8 * g + l4;
                if (r >= m) continue;
#pragma unroll
                for (int J = 0; J < 8; ++J)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int c = j0 + 8 * J + 2 * q + e;
                        if (c < n) Q[r + (int64_t)c * ldq] = acc[g][J][e];
                    }
            }
        }
    }
}

// Butterfly all-reduction step: W <- lower + upper in rank order (both partners
// add the same operands in the same order: bitwise-identical W on every rank).
__global__ void k_add_ordered(double *W, const double *P, int64_t count, int is_lower) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        W[i] = is_lower ? W[i] + P[i] : P[i] + W[i];
}

int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

}  // namespace

// ---------------------------------------------------------------- host stages
CholqrWs::~CholqrWs() {}

cudaError_t cholqr_alloc(CholqrWs &w, int64_t m, int n, cudaStream_t st) {
    const int nt = (n + GT - 1) / GT, ntp = nt * (nt + 1) / 2;
    const int64_t groups = (m + 7) / 8;
    int ns = std::max(1, (4 * sm_count()) / ntp);
    ns = (int)std::min<int64_t>(ns, std::max<int64_t>(1, groups / 8));
    w.nsplit = ns;
    w.rows_per_split = ((m + ns - 1) / ns + 7) / 8 * 8;
    w.nsplit = (int)((m + w.rows_per_split - 1) / w.rows_per_split);
    const size_t bytes = sizeof(double) * ((size_t)2 * n * n + (size_t)w.nsplit * ntp * GT * GT) + 16;
    cudaError_t e = cudaMallocAsync((void **)&w.base, bytes, st);
    if (e != cudaSuccess) return e;
    w.W = w.base;
    w.Rinv = w.W + (size_t)n * n;
    w.part = w.Rinv + (size_t)n * n;
    return cudaSuccess;
}

void cholqr_free(CholqrWs &w, cudaStream_t st) {
    if (w.base) cudaFreeAsync(w.base, st);
    w.base = w.W = w.Rinv = w.part = nullptr;
}

cudaError_t cholqr_gram(const double *A, int64_t lda, int64_t m, int n, CholqrWs &w, cudaStream_t st) {
    const int nt = (n + GT - 1) / GT, ntp = nt * (nt + 1) / 2;
    k_gram_tile<<<dim3(w.nsplit, ntp), 256, 0, st>>>(A, lda, m, n, w.rows_per_split, w.part);
    k_gram_reduce<<<std::max(1, std::min(1024, (n * n + 255) / 256)), 256, 0, st>>>(w.part, w.nsplit, n, w.W);
    return cudaGetLastError();
}

cudaError_t cholqr_add_ordered(double *W, const double *P, int64_t count, int is_lower, cudaStream_t st) {
    k_add_ordered<<<(int)std::min<int64_t>(1024, (count + 255) / 256), 256, 0, st>>>(W, P, count, is_lower);
    return cudaGetLastError();
}

cudaError_t cholqr_finish(const double *A, int64_t lda, int64_t m, int n, CholqrWs &w, double *R, int64_t ldr,
                          double *Q, int64_t ldq, int *info, cudaStream_t st) {
    const int use_smem = n <= 128;
    const size_t sm1 = use_smem ? sizeof(double) * n * n : 0;
    cudaError_t e = cudaFuncSetAttribute((const void *)k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    if (e != cudaSuccess) return e;
    k_chol_inv<<<1, 256, sm1, st>>>(w.W, n, R, ldr, w.Rinv, info, use_smem);
    if ((e = cudaGetLastError()) != cudaSuccess || !Q) return e;
    const size_t sm2 = sizeof(double) * ((n + 3) & ~3) * QLD;
    e = cudaFuncSetAttribute((const void *)k_qmul, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    if (e != cudaSuccess) return e;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_qmul, 256, sm2);
    const int64_t nblk = (m + 127) / 128;
    const int grid = (int)std::min<int64_t>(nblk, (int64_t)sm_count() * std::max(1, occ));
    k_qmul<<<grid, 256, sm2, st>>>(A, lda, m, n, w.Rinv, Q, ldq, info);
    return cudaGetLastError();
}

}  // namespace tsqr

using namespace tsqr;

extern "C" {

tsqr_status_t tsqr_cholqr(int64_t m, int64_t n, const double *A, int64_t lda, double *R, int64_t ldr, double *Q,
                          int64_t ldq, int *info, void *stream) {
    if (!A || !R || !info) return TSQR_ERR_INVALID;
    if (n < 1 || m < n) return TSQR_ERR_SHAPE;
    if (n > TSQR_MAX_N) return TSQR_ERR_UNSUPPORTED;
    if (lda < m || ldr < n || (Q && ldq < m)) return TSQR_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    CholqrWs w;
    cudaError_t e = cholqr_alloc(w, m, (int)n, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return TSQR_ERR_ALLOC;
    }
    e = cholqr_gram(A, lda, m, (int)n, w, st);
    if (e == cudaSuccess) e = cholqr_finish(A, lda, m, (int)n, w, R, ldr, Q, ldq, info, st);
    cholqr_free(w, st);
    if (e != cudaSuccess) {
        set_last_error("tsqr_cholqr", e);
        return TSQR_ERR_CUDA;
    }
    return TSQR_OK;
}

}  // extern "C"
