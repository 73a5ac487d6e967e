// Cycle probe of the blocked compact-WY engine (tools only, not product): one CTA
// runs panel_qr / build_t / wy_update_block on one tile; thread 0 records clock64.
#include "../paper_0808_2664_b200/csrc/wy.cuh"
#include <cstdio>
#include <vector>
using namespace tsqr;

template <int NCB, int NRB, int NW>
__global__ void k_probe(const double *A, int n, long long *out) {
    constexpr int S = 8 * NRB, NP = 8 * NCB;
    constexpr int NROWS = S > 2 * NP ? S : 2 * NP;
    constexpr int LD = ((NROWS + 13) / 16) * 16 + 2;
    constexpr int KMAX = NRB > NCB + 1 ? NRB : NCB + 1;
    extern __shared__ __align__(16) double sm[];
    double *tile = sm, *Ys = tile + NP * LD, *Ts = Ys + 8 * LD, *Gs = Ts + 64, *Wb = Gs + 64 * NW;
    double *taus = Wb + 72 * NW, *betas = taus + NP;
    const int warp = threadIdx.x >> 5;
    for (int e = threadIdx.x; e < NP * LD; e += 32 * NW) tile[e] = (e % LD) < S && (e / LD) < n ? A[e] : 0.0;
    for (int e = threadIdx.x; e < 8 * LD; e += 32 * NW) Ys[e] = 0.0;
    for (int e = threadIdx.x; e < NP; e += 32 * NW) taus[e] = 0.0;
    __syncthreads();
    __shared__ long long acc[2];
    if (threadIdx.x == 0) acc[0] = acc[1] = 0;
    __syncthreads();
    long long t_panel = 0, t_t = 0, t_upd = 0, t0, t1;
    const int npan = (n + 7) / 8;
    long long start = clock64();
    for (int p = 0; p < npan; ++p) {
        const wy::Rows R{p, NRB, -1, p};
        t0 = clock64();
        if (warp == p % NW) {
            wy::panel_qr<KMAX>(tile, LD, n, R, Ys, LD, taus, betas);
            __syncwarp();
            t1 = clock64();
            wy::build_t(Ys, LD, R, taus + 8 * p, Gs + 64 * warp, Ts);
            const long long t2 = clock64();
            if ((threadIdx.x & 31) == 0) {
                acc[0] += t1 - t0;
                acc[1] += t2 - t1;
            }
        }
        __syncthreads();
        t0 = clock64();
        for (int cb = warp; cb < npan; cb += NW)
            if (cb > p) wy::wy_update_block<true>(tile, LD, cb, Ys, LD, R, Ts, Wb + 72 * warp);
        if (threadIdx.x == 0) t_upd += clock64() - t0;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = acc[0];
        out[1] = acc[1];
        out[2] = t_upd;
        out[3] = clock64() - start;
    }
    (void)t_panel; (void)t_t;
}

template <int NCB, int NRB, int NW>
void run(int n) {
    constexpr int S = 8 * NRB, NP = 8 * NCB;
    constexpr int NROWS = S > 2 * NP ? S : 2 * NP;
    constexpr int LD = ((NROWS + 13) / 16) * 16 + 2;
    std::vector<double> h((size_t)NP * LD);
    for (auto &x : h) x = (rand() / (double)RAND_MAX) - 0.5;
    double *d; long long *o;
    cudaMalloc(&d, h.size() * 8); cudaMallocManaged(&o, 8 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    size_t smem = (NP * LD + 8 * LD + 64 + 64 * NW + 72 * NW + 2 * NP + 8) * 8;
    cudaFuncSetAttribute(k_probe<NCB, NRB, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
        for (int i = 0; i < 8; ++i) o[i] = 0;
        k_probe<NCB, NRB, NW><<<1, 32 * NW, smem>>>(d, n, o);
        cudaDeviceSynchronize();
    }
    const int npan = (n + 7) / 8;
    printf("NCB=%d NRB=%d NW=%d n=%d: total %lld cycles; per panel: panel_qr %.0f, build_t %.0f, update(warp0) %.0f\n", NCB,
           NRB, NW, n, o[3], o[0] / double(npan), o[1] / double(npan), o[2] / double(npan));
    cudaFree(d);
}

int main() {
    run<8, 8, 8>(64);
    run<8, 8, 1>(64);
    run<8, 16, 8>(64);
    run<8, 8, 8>(50);
    run<4, 16, 4>(32);
    run<4, 24, 4>(32);
    return 0;
}
