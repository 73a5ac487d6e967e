// Shared-memory / shuffle instruction throughput (tools only): cycles per
// warp-instruction seen by warp 0, with 1, 4 or 8 warps issuing the same mix.
#include <cstdio>
__global__ void k(double *out, long long *cyc, int mode, int iters) {
    __shared__ __align__(16) double sm[4096];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double acc = lane;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {            // STS.128 from lane 0 only (addresses vary per iteration)
        if (lane == 0)
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    { double *pp = sm + ((w * 256 + 2 * q + it * 32) & 4095); asm volatile("st.shared.v2.f64 [%0], {%1, %2};" :: "r"((unsigned)__cvta_generic_to_shared(pp)), "d"(acc + q), "d"(acc + it) : "memory"); }
            }
    } else if (mode == 1) {     // STS.128 full warp, distinct addresses
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
                *reinterpret_cast<double2 *>(sm + ((w * 32 + lane) * 2 + q * 512) % 4000) = make_double2(acc + q, acc);
        }
    } else if (mode == 2) {     // LDS.128 broadcast (all lanes same address), independent
        double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                double2 v = *reinterpret_cast<const double2 *>(sm + ((it * 32 + q * 2) & 2047));
                c[q & 7] += v.x + v.y;
            }
        }
        for (int q = 0; q < 8; ++q) acc += c[q];
    } else if (mode == 3) {     // LDS.64 broadcast
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 16; ++q) acc += sm[(it * 16 + q) & 2047];
        }
    } else if (mode == 4) {     // SHFL 64-bit, independent
        double c[8];
        for (int q = 0; q < 8; ++q) c[q] = acc + q;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 16; ++q) c[q & 7] = __shfl_sync(0xffffffffu, c[q & 7], (lane + q) & 31) + 1.0;
        }
        for (int q = 0; q < 8; ++q) acc += c[q];
    } else if (mode == 5) {     // DFMA independent (8 chains)
        double c[8];
        for (int q = 0; q < 8; ++q) c[q] = acc + q;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 16; ++q) c[q & 7] = fma(c[q & 7], 1.0000001, 1e-9);
        }
        for (int q = 0; q < 8; ++q) acc += c[q];
    }
    __syncwarp();
    long long t1 = clock64();
    if (lane == 0 && w == 0) cyc[mode] = t1 - t0;
    out[threadIdx.x] = acc + sm[threadIdx.x];
}
int main() {
    double *o;
    long long *c;
    cudaMalloc(&o, 8192 * 8);
    cudaMallocManaged(&c, 16 * 8);
    const char *names[] = {"STS.128 lane0", "STS.128 warp", "LDS.128 bcast", "LDS.64 bcast", "SHFL.64", "DFMA"};
    int iters = 256;
    for (int thr : {32, 128, 256}) {
        printf("warps/SM=%d (one CTA)\n", thr / 32);
        for (int m = 0; m < 6; ++m) {
            k<<<1, thr>>>(o, c, m, iters);
            k<<<1, thr>>>(o, c, m, iters);
            cudaDeviceSynchronize();
            printf("  %-14s %.2f cycles per warp-instruction (warp 0 view)\n", names[m], c[m] / double(iters * 16));
        }
    }
}
