// FP64 throughput probe: DFMA (CUDA cores) vs DMMA m8n8k4 (tensor cores) vs both
// interleaved in one warp.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void k(double *out, int iters, double s) {
  double a[8], c[8][2];
  for (int i = 0; i < 8; ++i) {
    a[i] = s + i * 1e-3 + threadIdx.x * 1e-6;
    c[i][0] = c[i][1] = 0.0;
  }
  double f[16];
  for (int i = 0; i < 16; ++i) f[i] = s * i;
  for (int it = 0; it < iters; ++it) {
    if (MODE & 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = fma(f[i], 0.999999, 1e-7);
    }
    if (MODE & 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a[i], a[(i + 1) & 7]);
    }
  }
  double r = 0;
  for (int i = 0; i < 16; ++i) r += f[i];
  for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *o;
  cudaMalloc(&o, sizeof(double) * sms * 8 * 256);
  const int iters = 4000;
  for (int wpb : {4, 8, 16}) {
    const int grid = sms * 2, block = 32 * wpb;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 1; mode <= 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 1) k<1><<<grid, block>>>(o, iters, 1.0);
        if (mode == 2) k<2><<<grid, block>>>(o, iters, 1.0);
        if (mode == 3) k<3><<<grid, block>>>(o, iters, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double thr = (double)grid * block;
        const double dfma = (mode & 1) ? thr * iters * 16 * 2 : 0;           // flops
        const double dmma = (mode & 2) ? (thr / 32) * iters * 8 * 512.0 : 0;  // 8x8x4 x2 per mma
        if (rep == 1)
          printf("warps/CTA=%2d mode=%d  %.3f ms  DFMA %.2f TF/s  DMMA %.2f TF/s  total %.2f TF/s\n", wpb, mode, ms,
                 dfma / ms / 1e9, dmma / ms / 1e9, (dfma + dmma) / ms / 1e9);
      }
    }
  }
  return 0;
}
