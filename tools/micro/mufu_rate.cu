// Developer microbenchmark: MUFU.EX2 issue rate per SM vs resident warps (one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters, long long* cycles) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    int iters = 4096;
    k<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = double(iters) * 8 * warps * 32;
    printf("warps/SM %2d: %.2f ex2 lanes/clk/SM\n", warps, ops / c);
  }
  return 0;
}
