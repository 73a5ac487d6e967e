#include <cstdio>
__global__ void k(double *out, long long *cyc, double a, double b, int n) {
    double x = a + threadIdx.x, y = b;
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < n; ++i) {
        x = fma(x, y, 0.25);  x = fma(x, y, 0.25);  x = fma(x, y, 0.25);  x = fma(x, y, 0.25);
        x = fma(x, y, 0.25);  x = fma(x, y, 0.25);  x = fma(x, y, 0.25);  x = fma(x, y, 0.25);
    }
    long long t1 = clock64();
    double d0 = x, d1 = 0.0;
    #pragma unroll 1
    for (int i = 0; i < n; ++i) {
        #pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(y), "d"(y));
    }
    long long t2 = clock64();
    float f = (float)x, g = 1.0001f;
    #pragma unroll 1
    for (int i = 0; i < n; ++i) {
        f = fmaf(f, g, 0.25f); f = fmaf(f, g, 0.25f); f = fmaf(f, g, 0.25f); f = fmaf(f, g, 0.25f);
        f = fmaf(f, g, 0.25f); f = fmaf(f, g, 0.25f); f = fmaf(f, g, 0.25f); f = fmaf(f, g, 0.25f);
    }
    long long t3 = clock64();
    out[threadIdx.x] = x + d0 + d1 + f;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
    double *o; long long *c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
    for (int nw : {1, 2, 4, 8}) {
        k<<<1, 32 * nw>>>(o, c, 1.0, 0.999, 1000);
        cudaDeviceSynchronize();
        printf("warps/CTA %d: DFMA dep latency %.1f cycles, DMMA dep latency %.1f, FFMA %.1f\n", nw, c[0] / 8000.0, c[1] / 8000.0, c[2] / 8000.0);
    }
    return 0;
}
