// Cycle probe of the column steps of team_tile_qr (tools only, not product):
// one team factors one tile; lane 0 of warp 0 records clock64 at the phase marks.
#include "../paper_0808_2664_b200/csrc/tsqr_device.cuh"
#include <cstdio>
#include <vector>
using namespace tsqr;

__device__ long long g_marks[64][8];
struct ClockProbe {
    __device__ static void mark(int j, int ph) {
        if (threadIdx.x == 0 && j < 64) g_marks[j][ph] = clock64();
    }
};

template <class T>
__global__ void __launch_bounds__(T::NT) k_probe(double *A, int n, long long *tot) {
    extern __shared__ __align__(16) double sm[];
    double *xs = sm, *red = xs + 2 * T::S + 2, *alph = red + 4 * T::G * T::NPAD, *taus = alph + 2;
    double *betas = taus + T::NPAD, *scales = betas + T::NPAD;
    double a[T::RT];
#pragma unroll
    for (int i = 0; i < T::RT; ++i) a[i] = A[T::col() * T::S + T::row0() + i];
    __syncthreads();
    long long t0 = clock64();
    team_tile_qr<T, ClockProbe>(a, n, xs, red, alph, taus, betas, scales);
    long long t1 = clock64();
#pragma unroll
    for (int i = 0; i < T::RT; ++i) A[T::col() * T::S + T::row0() + i] = a[i];
    if (threadIdx.x == 0) *tot = t1 - t0;
}

template <class T>
void run(int n) {
    std::vector<double> h((size_t)T::S * T::NPAD);
    for (auto &x : h) x = (rand() / (double)RAND_MAX) - 0.5;
    double *d; long long *tot;
    cudaMalloc(&d, h.size() * 8); cudaMallocManaged(&tot, 8);
    size_t smem = (2 * T::S + 8 + 4 * T::G * T::NPAD + 3 * T::NPAD) * 8;
    cudaFuncSetAttribute(k_probe<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        k_probe<T><<<1, T::NT, smem>>>(d, n, tot);
        cudaDeviceSynchronize();
    }
    long long m[64][8];
    cudaMemcpyFromSymbol(m, g_marks, sizeof(m));
    printf("Team<%d,%d,%d> n=%d: %lld cycles (%.0f per column)\n", T::CW, T::G, T::RT, n, *tot, double(*tot) / n);
    const char *names[] = {"publish", "sync", "dot", "red", "house", "axpy", "regsub"};
    for (int j : {1, 10, 40}) {
        if (j >= n - 1) continue;
        printf("  j=%2d", j);
        for (int ph = 0; ph < 7; ++ph) printf(" %s %4lld", names[ph], m[j][ph + 1] - m[j][ph]);
        printf("  loop %lld\n", m[j + 1][0] - m[j][0]);
    }
    cudaFree(d);
}

int main() {
    run<Team<1, 1, 96>>(32);
    run<Team<2, 1, 96>>(64);
    run<Team<2, 1, 64>>(64);
    run<Team<1, 1, 64>>(32);
    run<Team<2, 2, 48>>(64);
    return 0;
}
