// DFMA dependent latency and per-SM throughput vs (warps/SM, ILP) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double *out, long long *cyc, int iters) {
  double a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 0.999999, c = 1e-7;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, c);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int ILP>
void run(int warps, double *o, long long *cy) {
  int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<ILP><<<148, 32 * warps>>>(o, cy, iters);
  cudaEventRecord(e0);
  k<ILP><<<148, 32 * warps>>>(o, cy, iters);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cy, 8, cudaMemcpyDeviceToHost);
  double n = 148.0 * 32 * warps * iters * 16 * ILP;
  printf("warps/SM %2d ILP %d: %.2f cyc per dependent step (per warp), %.1f TFLOP/s\n", warps, ILP,
         double(c) / (iters * 16), 2 * n / (ms * 1e-3) / 1e12);
}
int main() {
  double *o;
  long long *cy;
  cudaMalloc(&o, 148 * 1024 * 8);
  cudaMalloc(&cy, 8);
  for (int w : {1, 4, 8, 16, 32}) {
    run<1>(w, o, cy);
    run<2>(w, o, cy);
    run<4>(w, o, cy);
    run<8>(w, o, cy);
  }
}
