// Dependent-chain latencies of FP64 ops on this GPU (tools only).
#include <cstdio>
#define N 1024
__global__ void k(double *out, long long *cyc, double a, double b) {
    double x = a + threadIdx.x;
    long long t0, t1;
    __shared__ double sm[64];
    sm[threadIdx.x & 63] = x;
    __syncthreads();
    // DFMA
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = fma(x, a, b);
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = x + b;
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) * a;
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) { sm[threadIdx.x & 63] = x; x = sm[(threadIdx.x + 1) & 63] * a; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N / 8; ++i) x = rsqrt(x * x + 1.0);
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) * 8;
    t0 = clock64();
    for (int i = 0; i < N / 8; ++i) x = sqrt(x * x + 1.0);
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) * 8;
    t0 = clock64();
    for (int i = 0; i < N / 8; ++i) x = 1.0 / (x + 2.0);
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) * 8;
    t0 = clock64();
    for (int i = 0; i < N / 8; ++i) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x + 2.0)); x = y; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) * 8;
    t0 = clock64();
    for (int i = 0; i < N / 8; ++i) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x * x + 1.0)); x = y; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0) * 8;
    t0 = clock64();
    for (int i = 0; i < N / 8; ++i) { __syncthreads(); x = x * a; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[9] = (t1 - t0) * 8;
    {
        double d0 = x, d1 = x * 0.5;
        t0 = clock64();
        for (int i = 0; i < N; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
        t1 = clock64(); if (threadIdx.x == 0) cyc[10] = t1 - t0;
        x += d0 + d1;
    }
    out[threadIdx.x] = x;
}
int main() {
    double *o; long long *c; cudaMalloc(&o, 4096 * 8); cudaMallocManaged(&c, 16 * 8);
    const char *names[] = {"dfma", "dadd", "shfl64+dmul", "sts+lds+dmul", "rsqrt(double)", "sqrt(double)", "div 1/x",
                           "rcp.approx.f64", "rsqrt.approx.f64", "bar.sync(256)+dmul", "dmma chain"};
    for (int thr : {32, 256}) {
        k<<<1, thr>>>(o, c, 1.0000001, 1e-9);
        k<<<1, thr>>>(o, c, 1.0000001, 1e-9);
        cudaDeviceSynchronize();
        printf("threads=%d\n", thr);
        for (int i = 0; i < 11; ++i) printf("  %-20s %.1f cycles/op\n", names[i], c[i] / double(N));
    }
}
