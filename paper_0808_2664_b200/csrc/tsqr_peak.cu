// Measurement hook: the FP64 pipe peak of this GPU, measured in the same process as
// the bench numbers (the roofline denominator, SURVEY 8(d) "Peaks": max(DFMA, DMMA)
// on all SMs).  Not on the TSQR path.  Product code.
#include "../../include/tsqr.h"
#include "tsqr_kernels.h"

#include <cuda_runtime.h>

namespace {

// independent m8n8k4 FP64 MMA chains (SASS DMMA.8x8x4), 8 warps per CTA
__global__ void __launch_bounds__(256) k_peak_dmma(double *out, int iters) {
    double a = threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-7;
    double c[4][2] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[t][0]), "+d"(c[t][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
    if (s == 12345.678) out[0] = s;
}

// independent DFMA chains
__global__ void __launch_bounds__(256) k_peak_dfma(double *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" tsqr_status_t tsqr_measure_fp64_peak(double *dmma_tflops, double *dfma_tflops, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                   cudaSuccess) {
        tsqr::set_last_error("tsqr_measure_fp64_peak", cudaGetLastError());
        return TSQR_ERR_CUDA;
    }
    double *d = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&d, sizeof(double), st);
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    const int blocks = 4 * sms, thr = 256, iters = 20000;
    float best_mma = 0.f, best_fma = 0.f;
    for (int rep = 0; rep < 3 && e == cudaSuccess; ++rep) {
        k_peak_dmma<<<blocks, thr, 0, st>>>(d, 200);                 // warm-up (clocks up)
        cudaEventRecord(e0, st);
        k_peak_dmma<<<blocks, thr, 0, st>>>(d, iters);
        cudaEventRecord(e1, st);
        e = cudaEventSynchronize(e1);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 256.0 * 4.0 * iters * (thr / 32.0) * blocks;   // 256 FMA per DMMA
        if (e == cudaSuccess && ms > 0.f) best_mma = fmaxf(best_mma, (float)(fl / ms / 1e9));
        cudaEventRecord(e0, st);
        k_peak_dfma<<<blocks, thr, 0, st>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1, st);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        const double ff = 2.0 * 8.0 * iters * (double)thr * blocks;
        if (e == cudaSuccess && ms > 0.f) best_fma = fmaxf(best_fma, (float)(ff / ms / 1e9));
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (d) cudaFreeAsync(d, st);
    if (e != cudaSuccess) {
        tsqr::set_last_error("tsqr_measure_fp64_peak", e);
        return TSQR_ERR_CUDA;
    }
    if (dmma_tflops) *dmma_tflops = best_mma;
    if (dfma_tflops) *dfma_tflops = best_fma;
    return TSQR_OK;
}
