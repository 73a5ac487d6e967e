// Phase-cycle probe of the chunk-chain factor kernel (not product code).
// Builds k_chain_factor with TSQR_PROBE, runs one CTA on one tile of m rows,
// and prints the mean cycles of each phase per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTSQR_PROBE
//        -I paper_0808_2664_b200/csrc tools/probe_chain.cu -o tools/probe_chain
#include "../paper_0808_2664_b200/csrc/tsqr_chain.cu"
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

using namespace tsqr;

template <class C>
int run(int m, int n, int grid) {
    const int NWARP = PROBE_W;
    double *A; int64_t *row0; int *rows; int64_t *ch0; int *cta; double *tau; unsigned long long *pb;
    const int L = grid;
    cudaMalloc(&A, sizeof(double) * (size_t)m * n * L);
    std::vector<double> h((size_t)m * n * L);
    srand(1);
    for (auto &x : h) x = (rand() / (double)RAND_MAX) - 0.5;
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    std::vector<int64_t> r0(L), c0(L + 1);
    std::vector<int> rw(L), ct(L + 1);
    for (int t = 0; t < L; ++t) { r0[t] = (int64_t)t * m; rw[t] = m; c0[t] = (int64_t)t * ((m + C::CH - 1) / C::CH); ct[t] = t; }
    c0[L] = (int64_t)L * ((m + C::CH - 1) / C::CH); ct[L] = L;
    cudaMalloc(&row0, 8 * L); cudaMalloc(&rows, 4 * L); cudaMalloc(&ch0, 8 * (L + 1)); cudaMalloc(&cta, 4 * (L + 1));
    cudaMalloc(&tau, sizeof(double) * c0[L] * n);
    cudaMemcpy(row0, r0.data(), 8 * L, cudaMemcpyHostToDevice);
    cudaMemcpy(rows, rw.data(), 4 * L, cudaMemcpyHostToDevice);
    cudaMemcpy(ch0, c0.data(), 8 * (L + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(cta, ct.data(), 4 * (L + 1), cudaMemcpyHostToDevice);
    cudaMalloc(&pb, sizeof(unsigned long long) * NWARP * PROBE_N);
    cudaMemset(pb, 0, sizeof(unsigned long long) * NWARP * PROBE_N);
    cudaMemcpyToSymbol(g_probe_buf, &pb, sizeof(pb));
    cudaFuncSetAttribute((const void *)k_chain_factor<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
    int64_t lda = (int64_t)m * L;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_chain_factor<C><<<grid, C::NT, C::BYTES>>>(A, lda, n, row0, rows, ch0, cta, tau, nullptr);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("m=%d n=%d grid=%d: %s, %.3f ms (%.1f us per chunk-round)\n", m, n, grid, cudaGetErrorString(err), ms,
           1000.0 * ms / ((m / C::CH) / (double)NWARP));
    std::vector<unsigned long long> hb((size_t)NWARP * PROBE_N);
    cudaMemcpy(hb.data(), pb, hb.size() * 8, cudaMemcpyDeviceToHost);
    // per event pair (prev -> cur) accumulate cycles
    std::map<std::pair<int, int>, std::pair<double, long>> acc;
    for (int w = 0; w < NWARP; ++w) {
        const unsigned long long *b = hb.data() + (size_t)w * PROBE_N;
        int cnt = (int)b[0];
        for (int i = 2; i <= cnt; ++i) {
            int a = (int)(b[i - 1] & 255), c = (int)(b[i] & 255);
            double dt = (double)((b[i] >> 8) - (b[i - 1] >> 8));
            auto &x = acc[{a, c}];
            x.first += dt; x.second++;
        }
    }
    const char *nm[] = {"chunk0", "panel", "stepend", "pre-wait", "post-wait", "steps-done", "W^T done",
                        "R upd+pub", "trail-end", "tr-wait", "T built"};
    for (auto &kv : acc)
        printf("  %-10s -> %-10s : %8.1f cycles avg  (%ld)\n", nm[kv.first.first], nm[kv.first.second],
               kv.second.first / kv.second.second, kv.second.second);
    return 0;
}

int main(int argc, char **argv) {
    int m = argc > 1 ? atoi(argv[1]) : 2048;
    int n = argc > 2 ? atoi(argv[2]) : 64;
    int grid = argc > 3 ? atoi(argv[3]) : 1;
    int solo = argc > 4 ? atoi(argv[4]) : 0;
    if (solo) return run<chunk::Cfg<8, 4, 1>>(m, n, grid);
    if (n > 56) return run<chunk::Cfg<8, 4, 8>>(m, n, grid);
    if (n > 48) return run<chunk::Cfg<7, 4, 8>>(m, n, grid);
    return run<chunk::Cfg<4, 8, 8>>(m, n, grid);
}
