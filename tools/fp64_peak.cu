// FP64 FMA throughput probe: all SMs, independent DFMA chains per thread.
// Used to measure P_FP64 (the roofline's compute denominator) on the B200 box.
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-7 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}
int main() {
  int dev = 0; cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  printf("name=%s sms=%d l2=%d smem_optin=%zu clock_khz=%d\n", pr.name, pr.multiProcessorCount,
         pr.l2CacheSize, pr.sharedMemPerBlockOptin, pr.clockRate);
  double *d; cudaMalloc(&d, 8);
  const int iters = 20000, threads = 256;
  for (int rep = 0; rep < 2; ++rep)
  for (int bps : {4, 8}) {
    int blocks = pr.multiProcessorCount * bps;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dfma_kernel<8><<<blocks, threads>>>(d, 100, 0.999999, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("blocks/SM=%d  %.3f ms  %.2f TFLOP/s\n", bps, ms, flops / ms / 1e9);
  }
  // sustained: ~3 s loop
  {
    int blocks = pr.multiProcessorCount * 8;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    int n = 0; float ms = 0;
    while (ms < 3000) { dfma_kernel<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-9); ++n;
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); }
    double flops = 2.0 * 8 * iters * (double)blocks * threads * n;
    printf("sustained %.0f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  return 0;
}
