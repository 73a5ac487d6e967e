/* Plain C client of libtsqr.so (include/tsqr.h): no Python, no torch.
 * Factors a seeded m x n matrix on the GPU, forms Q, and checks ||A - QR||_F / ||A||_F and
 * ||Q^T Q - I||_F on the host.  Build: gcc -O2 -I include examples/c_abi_demo.c
 *   -L paper_0808_2664_b200 -ltsqr -L/usr/local/cuda/lib64 -lcudart -lm -o c_abi_demo
 * usage: c_abi_demo [m] [n]   (exit 0 when both checks pass) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "tsqr.h"

static double lcg(uint64_t *s) {                 /* uniform in [-1, 1) */
    *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
    return (double)(*s >> 11) / 4503599627370496.0 - 1.0;
}

#define CK(x)                                                                               \
    do {                                                                                    \
        tsqr_status_t s_ = (x);                                                             \
        if (s_ != TSQR_OK) {                                                                \
            fprintf(stderr, "%s: %s (%s)\n", #x, tsqr_status_string(s_), tsqr_last_error()); \
            return 1;                                                                       \
        }                                                                                   \
    } while (0)

int main(int argc, char **argv) {
    const int64_t m = argc > 1 ? atoll(argv[1]) : 20000, n = argc > 2 ? atoll(argv[2]) : 40;
    double *A = malloc(sizeof(double) * m * n), *Q = malloc(sizeof(double) * m * n), *R = malloc(sizeof(double) * n * n);
    uint64_t seed = 1;
    for (int64_t i = 0; i < m * n; ++i) A[i] = lcg(&seed);
    double *dA, *dQ, *dR;
    if (cudaMalloc((void **)&dA, sizeof(double) * m * n) || cudaMalloc((void **)&dQ, sizeof(double) * m * n) ||
        cudaMalloc((void **)&dR, sizeof(double) * n * n)) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    cudaMemcpy(dA, A, sizeof(double) * m * n, cudaMemcpyHostToDevice);
    tsqr_opts_t o = {4096, 0, 1, 0, 0, 0};          /* row blocks of 4096, default tiles, one rank */
    tsqr_tree_t tree = NULL;
    CK(tsqr_factor(m, n, dA, m, dR, n, &o, NULL, &tree));
    CK(tsqr_form_q(tree, dQ, m, NULL));
    cudaMemcpy(Q, dQ, sizeof(double) * m * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(R, dR, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
    CK(tsqr_tree_free(tree));
    double num = 0.0, den = 0.0, orth = 0.0;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double qr = 0.0;
            for (int64_t k = 0; k <= j; ++k) qr += Q[i + k * m] * R[k + j * n];
            const double d = A[i + j * m] - qr;
            num += d * d;
            den += A[i + j * m] * A[i + j * m];
        }
    for (int64_t a = 0; a < n; ++a)
        for (int64_t b = 0; b < n; ++b) {
            double g = 0.0;
            for (int64_t i = 0; i < m; ++i) g += Q[i + a * m] * Q[i + b * m];
            g -= (a == b);
            orth += g * g;
        }
    const double res = sqrt(num / den);
    orth = sqrt(orth);
    printf("c_abi_demo m=%lld n=%lld: ||A-QR||/||A|| = %.2e  ||Q^TQ-I|| = %.2e\n", (long long)m, (long long)n, res,
           orth);
    cudaFree(dA); cudaFree(dQ); cudaFree(dR);
    free(A); free(Q); free(R);
    return (res <= 1e-13 && orth <= 1e-13) ? 0 : 1;
}
