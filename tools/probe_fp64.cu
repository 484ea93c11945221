// Probe: fp64 FMA throughput, DADD throughput, HBM copy, L2 size, SM count on the B200 box.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void copyk(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("name=%s sms=%d l2=%d smem_optin=%zu clock_khz=%d memclk_khz=%d buswidth=%d\n", p.name, p.multiProcessorCount,
         p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int bs : {256, 512}) for (int bpsm : {1, 2, 4, 8}) {
    int grid = p.multiProcessorCount * bpsm;
    if (bs * bpsm > 2048) continue;
    dfma_loop<<<grid, bs>>>(out, 100, 0.999999, 1e-7);
    cudaEventRecord(e0); dfma_loop<<<grid, bs>>>(out, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)grid * bs;
    printf("dfma bs=%d blocks/sm=%d : %.2f TFLOP/s (%.3f ms)\n", bs, bpsm, flops / ms / 1e9, ms);
  }
  size_t n = (size_t)1 << 28; double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  for (int bpsm : {2, 4, 8}) {
    int grid = p.multiProcessorCount * bpsm;
    copyk<<<grid, 512>>>(a, b, n);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) copyk<<<grid, 512>>>(a, b, n); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 4GiB blocks/sm=%d: %.1f GB/s\n", bpsm, 5.0 * 2 * n * 16 / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
