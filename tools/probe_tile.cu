// Cycle probe of one column step of tile_qr (tools only, not product):
// one CTA factors one tile; warps 0 and 7, lane 0, record clock64 at phase marks.
#include "../paper_0808_2664_b200/csrc/tsqr_device.cuh"
#include <cstdio>
#include <vector>
using namespace tsqr;

__device__ long long g_marks[2][64][6];
struct ClockProbe {
    __device__ static void mark(int j, int ph) {
        const int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0 && (w == 0 || w == 7) && j < 64) g_marks[w ? 1 : 0][j][ph] = clock64();
    }
};

template <int NP, int RT>
__global__ void __launch_bounds__(256, 1) k_probe(double *A, int lda, int n, int rows) {
    using Lt = Layout<NP, RT>;
    extern __shared__ __align__(16) double sm[];
    double *stage = sm, *xs = stage + Lt::SLD * NP + 1;
    xs += ((size_t)xs / 8) % 2;
    double *red = xs + Lt::S, *rowj = red + 2 * kWarps * NP, *taus = rowj + 2 * NP;
    double *betas = taus + NP, *scales = betas + NP;
    stage_in_async(stage, Lt::SLD, A, lda, rows, n, Lt::S, NP);
    cp_async_wait_all();
    __syncthreads();
    double a[RT][Lt::CPL];
    smem_to_regs<Lt>(stage, a);
    long long t0 = clock64();
    tile_qr<Lt, ClockProbe>(a, n, xs, red, rowj, taus, betas, scales);
    long long t1 = clock64();
    regs_to_smem<Lt>(stage, a);
    __syncthreads();
    stage_out(stage, Lt::SLD, A, lda, rows, n);
    if (threadIdx.x == 0) printf("total tile_qr cycles %lld for n=%d rows=%d (%.0f per column)\n", t1 - t0, n, rows,
                                 double(t1 - t0) / n);
}

template <int NP, int RT>
void run(int n) {
    using Lt = Layout<NP, RT>;
    int rows = Lt::S;
    std::vector<double> h((size_t)rows * n);
    for (auto &x : h) x = (rand() / (double)RAND_MAX) - 0.5;
    double *d;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    size_t smem = (Lt::SLD * NP + Lt::S + 2 * kWarps * NP + 5 * NP + 8) * 8;
    cudaFuncSetAttribute(k_probe<NP, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        k_probe<NP, RT><<<1, 256, smem>>>(d, rows, n, rows);
        cudaDeviceSynchronize();
    }
    long long m[2][64][6];
    cudaMemcpyFromSymbol(m, g_marks, sizeof(m));
    printf("NP=%d RT=%d S=%d n=%d  (cycles per phase, warp0 | warp7), columns 1,10,30:\n", NP, RT, Lt::S, n);
    const char *names[] = {"publish", "dot+rowj", "barrier", "reduce+house", "update", "next"};
    for (int j : {1, 10, 30}) {
        if (j >= n - 1) continue;
        printf(" j=%2d", j);
        for (int ph = 0; ph < 5; ++ph)
            printf("  %s %4lld|%4lld", names[ph], m[0][j][ph + 1] - m[0][j][ph], m[1][j][ph + 1] - m[1][j][ph]);
        printf("  loop %lld|%lld\n", m[0][j + 1][0] - m[0][j][0], m[1][j + 1][0] - m[1][j][0]);
    }
    cudaFree(d);
}

int main() {
    run<64, 16>(50);
    run<64, 32>(64);
    run<32, 32>(32);
    run<16, 32>(16);
    return 0;
}
