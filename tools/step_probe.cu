// Cycle probe of the chunk engine's Householder step (not product code).
// Each warp keeps one chunk (KM x NCB DMMA fragments) in registers and a private R
// buffer in smem, and repeats panel P = 0 of the structured factorisation (8 steps,
// then optionally the trailing update) ITERS times; the hand-off counters are
// pre-set so no wait ever blocks.  Prints cycles per step with W warps per CTA
// (one CTA per SM), i.e. alone (W = 1) and with the SM's 8 warps interleaved.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_0808_2664_b200/csrc
//        -I <nccl>/include tools/step_probe.cu -o /tmp/step_probe
#include "chunk.cuh"

#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace tsqr;
using namespace tsqr::chunk;

template <class C, bool kTrail>
__global__ void __launch_bounds__(C::NT, 1) k_probe(int iters, int n, unsigned long long *out, double *sink) {
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *Rb = sm;                               // one R buffer for all warps (timing only)
    double *ws = sm + C::RBUF + warp * C::WS;
    int *cnt = reinterpret_cast<int *>(sm + C::RBUF + 16 * C::WS) + warp * C::SYNC_INTS;
    PROBE_INIT();
    for (int i = lane; i < C::RBUF; i += 32) Rb[i] = (i % (C::LDR + 1) == 0) ? 3.0 : 0.01 * (i % 7);
    for (int i = lane; i < C::SYNC_INTS; i += 32) cnt[i] = 1 << 30;
    __syncwarp();
    Chunk<C> ch;
#pragma unroll
    for (int k = 0; k < C::KM; ++k)
#pragma unroll
        for (int cb = 0; cb < C::NCB; ++cb) {
            ch.a[k][cb][0] = 0.1 + 0.001 * (lane + 7 * k + 13 * cb);
            ch.a[k][cb][1] = -0.2 + 0.0013 * (lane * 3 + k + cb);
        }
    const Sync sy{cnt, cnt + C::NP, 0};
    double tau[64];
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if constexpr (kTrail) factor_panel<C, 0, false>(ch, 0, 0, Rb, ws, tau, n, sy, true, nullptr);
        else panel_structured<C, 0, false>(ch, Rb, ws + C::GS, ws + C::T8, ws + C::XS, tau, n, sy);
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
    PROBE_FLUSH();
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < C::KM; ++k)
#pragma unroll
        for (int cb = 0; cb < C::NCB; ++cb) s += ch.a[k][cb][0] + ch.a[k][cb][1];
    if (s == 1234.5) sink[threadIdx.x] = s + tau[lane & 7];
}

template <class C, bool kTrail>
void run(const char *name, int warps) {
#ifdef TSQR_PROBE
    const int iters = 6;                         // the event log holds 512 entries per warp
#else
    const int iters = 200;
#endif
    const int n = 8 * C::NCB, sms = 148;
    unsigned long long *out;
    double *sink;
    cudaMalloc(&out, sizeof(unsigned long long) * sms * 16);
    cudaMalloc(&sink, 8 * 256);
    const size_t bytes = (size_t)(C::RBUF + 16 * C::WS + 16 * C::SYNC_INTS) * 8;
    cudaFuncSetAttribute((const void *)k_probe<C, kTrail>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
#ifdef TSQR_PROBE
    unsigned long long *pb;
    cudaMalloc(&pb, sizeof(unsigned long long) * PROBE_W * PROBE_N);
    cudaMemset(pb, 0, sizeof(unsigned long long) * PROBE_W * PROBE_N);
    cudaMemcpyToSymbol(g_probe_buf, &pb, sizeof(pb));
#endif
    k_probe<C, kTrail><<<sms, 32 * warps, bytes>>>(2, n, out, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_probe<C, kTrail><<<sms, 32 * warps, bytes>>>(iters, n, out, sink);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(sms * 16);
    cudaMemcpy(h.data(), out, 8 * h.size(), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int b = 0; b < sms; ++b)
        for (int w = 0; w < warps; ++w) avg += h[b * 16 + w];
    avg /= sms * warps;
    // per chunk-panel: useful FMAs of the panel's steps (+ trailing): c rows x 8 cols x 2 x 8 steps
    // (dots + updates), + trailing c x 8 x nt x 2 x 2 (W and C update)
    const double c = C::CH, nt = 8.0 * (C::NCB - 1);
    const double fl = 2.0 * (c * 8 * 8 * 2 + (kTrail ? c * 8 * nt * 2 * 2 : 0.0));
    const double tf = fl * iters * warps * sms / (ms * 1e-3) / 1e12;
    printf("%-22s warps=%d  %s  %8.0f cycles per panel  %6.0f cycles per step  %.2f TF/s useful (%.1f%% of 37.2)\n",
           name, warps, cudaGetErrorString(err), avg / iters, avg / iters / 8, tf, 100 * tf / 37.22);
#ifdef TSQR_PROBE
    {   // mean cycles between consecutive probe events of warp 0 of CTA 0
        std::vector<unsigned long long> hb(PROBE_W * PROBE_N);
        cudaMemcpy(hb.data(), pb, 8 * hb.size(), cudaMemcpyDeviceToHost);
        double acc[16][16] = {};
        long cnt[16][16] = {};
        for (int w = 0; w < warps; ++w) {
            const unsigned long long *b = hb.data() + (size_t)w * PROBE_N;
            const int c = (int)b[0];
            for (int i = 2; i <= c; ++i) {
                const int a = (int)(b[i - 1] & 255), z = (int)(b[i] & 255);
                acc[a][z] += (double)((b[i] >> 8) - (b[i - 1] >> 8));
                cnt[a][z]++;
            }
        }
        for (int a = 0; a < 16; ++a)
            for (int z = 0; z < 16; ++z)
                if (cnt[a][z]) printf("      event %d -> %d: %7.1f cycles (%ld)\n", a, z, acc[a][z] / cnt[a][z], cnt[a][z]);
    }
    cudaFree(pb);
#endif
    cudaFree(out);
    cudaFree(sink);
}

int main() {
    const char *only = std::getenv("PROBE_ONLY");
    if (only && only[0] == 'h') {     // half-chunk (32-column) chains at 8 and 12 warps vs the n64 chunk at 8
        run<Cfg<8, 5, 8, 1>, false>("n64 c40 steps", 8);
        run<Cfg<8, 5, 8, 1>, true>("n64 c40 steps+trail", 8);
        run<Cfg<4, 5, 12>, false>("n32 c40 steps", 8);
        run<Cfg<4, 5, 12>, true>("n32 c40 steps+trail", 8);
        run<Cfg<4, 5, 12>, false>("n32 c40 steps", 12);
        run<Cfg<4, 5, 12>, true>("n32 c40 steps+trail", 12);
        return 0;
    }
    for (int w : {1, 4, 8}) {
        run<Cfg<8, 5, 8, 1>, false>("n64 c40 steps", w);
        run<Cfg<8, 5, 8, 1>, true>("n64 c40 steps+trail", w);
        run<Cfg<7, 5, 8>, false>("n56 c40 steps", w);
        run<Cfg<7, 5, 8>, true>("n56 c40 steps+trail", w);
        run<Cfg<4, 8, 8>, false>("n32 c64 steps", w);
        run<Cfg<4, 8, 8>, true>("n32 c64 steps+trail", w);
    }
    return 0;
}

// dependent-latency microbenchmarks (one warp): DMMA accumulate chain, SHFL+DADD chain
__global__ void k_lat(int iters, unsigned long long *out, double *sink) {
    double a = threadIdx.x * 1e-3, b = 1.0, d0 = 0.0, d1 = 0.0, x = threadIdx.x;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) dmma(d0, d1, a, b);
    unsigned long long t1 = clock64();
    for (int i = 0; i < iters; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
    unsigned long long t2 = clock64();
    for (int i = 0; i < iters; ++i) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 1.0; }
    unsigned long long t3 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; }
    if (d0 + d1 + x == 1234.5) sink[0] = d0;
}

struct LatMain {
    LatMain() {
        unsigned long long *o; double *s;
        cudaMalloc(&o, 64); cudaMalloc(&s, 64);
        k_lat<<<1, 32>>>(10, o, s);
        k_lat<<<1, 32>>>(1000, o, s);
        unsigned long long h[3];
        cudaMemcpy(h, o, 24, cudaMemcpyDeviceToHost);
        printf("latency (cycles): DMMA chain %.1f  SHFL.64+DADD %.1f  rsqrt.approx+DADD %.1f\n", h[0] / 1000.0,
               h[1] / 1000.0, h[2] / 1000.0);
    }
} g_lat_main;
