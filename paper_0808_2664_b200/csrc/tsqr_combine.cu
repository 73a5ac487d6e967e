// q-ary structured combine: Alg. QR:qnxn ([TR] P:1957-1979),
// the Householder QR of q stacked n x n upper triangles [R_1; ...; R_q] that
// touches only the nonzero rows -- reflector j acts on I_j = {row j of R_1} U
// {rows 0..j of R_2..R_q}; (2/3)(q-1)n^3 flops.  The binary tree
// uses q = 2 inside its pipelined kernels; this entry point is the general node
// (a flat top of a tree, or the one-node alternative to the cross-GPU
// butterfly), one CTA, the triangles staged in shared memory when they fit.
// Product code.
#include "../../include/tsqr.h"
#include "tsqr_kernels.h"
#include "wy.cuh"

#include <cuda_runtime.h>

namespace {

constexpr int CT = 512;                 // threads of the combine CTA
constexpr int CW = CT / 32;

struct Packed {
    double *p;
    int64_t np;                         // n(n+1)/2
    __device__ double &at(int i, int r, int c) const { return p[(int64_t)i * np + (int64_t)c * (c + 1) / 2 + r]; }
};

__device__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < CW; ++w) s += red[w];
    __syncthreads();                    // red may be reused
    return s;
}

__device__ double block_max(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < CW; ++w) s = fmax(s, red[w]);
    __syncthreads();
    return s;
}

__global__ void __launch_bounds__(CT) k_combine_q(double *g, int q, int n, double *tau_out, int staged) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[CW];
    __shared__ double hh[3];            // tau, beta, 1/(alpha - beta)
    const int64_t np = (int64_t)n * (n + 1) / 2, tot = q * np;
    if (staged)
        for (int64_t e = threadIdx.x; e < tot; e += CT) sm[e] = g[e];
    __syncthreads();
    const Packed P{staged ? sm : g, np};
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = 0; j < n; ++j) {
        const int len = (q - 1) * (j + 1);          // the reflector's rows below its pivot
        double s = 0.0;
        for (int e = threadIdx.x; e < len; e += CT) {
            const double x = P.at(1 + e / (j + 1), e % (j + 1), j);
            s = fma(x, x, s);
        }
        double sigma2 = block_sum(s, red);
        double sc = 1.0;
        if (tsqr::wy::house_unsafe(P.at(0, j, j), sigma2)) {      // block-uniform: dlarfg's rescaling (R23)
            double mx = 0.0;
            for (int e = threadIdx.x; e < len; e += CT) mx = fmax(mx, fabs(P.at(1 + e / (j + 1), e % (j + 1), j)));
            sc = tsqr::wy::pow2_scale(fmax(block_max(mx, red), fabs(P.at(0, j, j))));
            s = 0.0;
            for (int e = threadIdx.x; e < len; e += CT) {
                const double x = sc * P.at(1 + e / (j + 1), e % (j + 1), j);
                s = fma(x, x, s);
            }
            sigma2 = block_sum(s, red);                        // of s w
        }
        if (threadIdx.x == 0) {
            // House(w), LAPACK dlarfg: beta = -sign(alpha)||w||, tau = (beta - alpha)/beta,
            // v = w / (alpha - beta), v(1) = 1; w with nothing to annihilate gives H = I;
            // computed on s w (s = 1 unless rescaled): beta = beta_s / s, 1/(alpha - beta) = s/(alpha_s - beta_s)
            const double alpha = sc * P.at(0, j, j);
            if (sigma2 == 0.0) {
                hh[0] = 0.0; hh[1] = alpha / sc; hh[2] = 0.0;
            } else {
                const double nrm = sqrt(fma(alpha, alpha, sigma2));
                const double beta = alpha >= 0.0 ? -nrm : nrm;
                hh[0] = (beta - alpha) / beta; hh[1] = beta / sc; hh[2] = sc / (alpha - beta);
            }
        }
        __syncthreads();
        const double t = hh[0], beta = hh[1], scale = hh[2];
        if (t != 0.0)
            for (int e = threadIdx.x; e < len; e += CT) P.at(1 + e / (j + 1), e % (j + 1), j) *= scale;
        __syncthreads();
        if (t != 0.0) {
            // columns j+1..n-1, one warp each: w = A(j, c) + v^T A(I_j minus {j}, c), then the update
            for (int c = j + 1 + warp; c < n; c += CW) {
                double w = 0.0;
                for (int e = lane; e < len; e += 32) {
                    const int i = 1 + e / (j + 1), r = e % (j + 1);
                    w = fma(P.at(i, r, j), P.at(i, r, c), w);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
                w += P.at(0, j, c);
                const double tw = t * w;
                if (lane == 0) P.at(0, j, c) -= tw;
                for (int e = lane; e < len; e += 32) {
                    const int i = 1 + e / (j + 1), r = e % (j + 1);
                    P.at(i, r, c) -= P.at(i, r, j) * tw;
                }
            }
        }
        if (threadIdx.x == 0) {
            P.at(0, j, j) = beta;
            tau_out[j] = t;
        }
        __syncthreads();
    }
    if (staged)
        for (int64_t e = threadIdx.x; e < tot; e += CT) g[e] = sm[e];
}

}  // namespace

extern "C" tsqr_status_t tsqr_combine_stacked(int32_t q, int64_t n, double *packed, double *tau, void *stream) {
    if (!packed || !tau) return TSQR_ERR_INVALID;
    if (q < 1 || n < 1) return TSQR_ERR_INVALID;
    if (n > TSQR_MAX_N) return TSQR_ERR_UNSUPPORTED;
    if ((int64_t)q * n > ((int64_t)1 << 24)) return TSQR_ERR_UNSUPPORTED;
    const size_t bytes = sizeof(double) * (size_t)q * (size_t)(n * (n + 1) / 2);
    const int staged = bytes <= 200 * 1024;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = staged ? cudaFuncSetAttribute((const void *)k_combine_q,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)
                           : cudaSuccess;
    if (e == cudaSuccess) {
        k_combine_q<<<1, CT, staged ? bytes : 0, st>>>(packed, q, (int)n, tau, staged);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) {
        tsqr::set_last_error("tsqr_combine_stacked", e);
        return TSQR_ERR_CUDA;
    }
    return TSQR_OK;
}
