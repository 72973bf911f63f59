// Developer microbenchmark: MUFU exp2 throughput per SM, fp32 (ex2.approx.ftz.f32, one result per
// lane) vs packed half (ex2.approx.f16x2, two results per lane) — whether the softmax exponentials
// can be halved in MUFU issue by computing them as f16 pairs.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
__global__ void k32(float* out, int iters, long long* cycles) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = -(threadIdx.x * 1e-3f + j) * 0.01f;
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
__global__ void k16(float* out, int iters, long long* cycles) {
  unsigned x[8];
  for (int j = 0; j < 8; ++j) {
    __half2 h = __floats2half2_rn(-(threadIdx.x * 1e-3f + j) * 0.01f, -0.5f);
    x[j] = *reinterpret_cast<unsigned*>(&h);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[j]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += __low2float(*reinterpret_cast<__half2*>(&x[j]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  for (int warps : {4, 8, 16}) {
    int iters = 4096;
    long long c;
    k32<<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = double(iters) * 8 * warps * 32;
    printf("warps/SM %2d: f32   ex2 %.2f results/clk/SM\n", warps, ops / c);
    k16<<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("warps/SM %2d: f16x2 ex2 %.2f results/clk/SM (%s)\n", warps, 2 * ops / c,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
