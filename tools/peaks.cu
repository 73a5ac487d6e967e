// FP64 / HBM peak microbenchmarks for the B200 roofline denominators.
// DFMA: register-resident independent FMA chains on every SM.
// DMMA: mma.sync.aligned.m8n8k4 f64 (SASS DMMA) chains on every SM.
// HBM : device copy kernel, read+write bytes.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
  #pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0; 
  #pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-7;
  double c[4][2];
  #pragma unroll
  for (int t = 0; t < 4; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  #pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

__global__ void bar_kernel(double* out, int iters) {
  __shared__ double s[1024];
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    s[threadIdx.x] = acc;
    __syncthreads();
    acc += s[(threadIdx.x + 1) % blockDim.x];
    __syncthreads();
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"name\":\"%s\",\"sms\":%d,\"smem_optin\":%zu,\"smem_per_sm\":%zu,\"regs_per_sm\":%d,\"l2\":%d,\"clock_khz\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor,
         p.regsPerMultiprocessor, p.l2CacheSize, p.clockRate);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int blocksPerSm : {1, 2, 4, 8}) {
    int iters = 20000; const int CH = 8; int thr = 256;
    dfma_kernel<CH><<<sms*blocksPerSm, thr>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<CH><<<sms*blocksPerSm, thr>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * CH * iters * (double)thr * sms * blocksPerSm;
    printf("{\"kind\":\"dfma\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", blocksPerSm, fl / ms / 1e9);
  }
  for (int blocksPerSm : {1, 2, 4, 8}) {
    int iters = 20000; int thr = 256;
    dmma_kernel<<<sms*blocksPerSm, thr>>>(d, 100);
    cudaEventRecord(e0);
    dmma_kernel<<<sms*blocksPerSm, thr>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 4 * (double)iters * (thr / 32) * sms * blocksPerSm;
    printf("{\"kind\":\"dmma\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", blocksPerSm, fl / ms / 1e9);
  }
  {
    size_t n = (size_t)1 << 30; // bytes 8 GiB per buffer? use 2 GiB
    n = ((size_t)2 << 30) / 16;
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    cudaMemset(a, 0, n * 16);
    float best = 1e30;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      copy_kernel<<<sms * 8, 512>>>(a, b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"kind\":\"hbm_copy\",\"gbs\":%.1f}\n", 2.0 * n * 16 / best / 1e6);
  }
  for (int thr : {256, 512}) {
    int iters = 20000;
    bar_kernel<<<sms, thr>>>(d, 100);
    cudaEventRecord(e0);
    bar_kernel<<<sms, thr>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kind\":\"bar_roundtrip\",\"threads\":%d,\"ns_per_iter\":%.2f}\n", thr, ms * 1e6 / iters);
  }
  return 0;
}
