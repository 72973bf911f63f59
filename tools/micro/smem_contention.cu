// Developer microbenchmark: how much shared-memory bandwidth is left to the threads while the
// tensor core streams SS operands.  One elected thread issues back-to-back 128 x N x 16
// tcgen05.mma (both operands in smem) while 8 warps time their own LDS.128 + STS.128 traffic over
// a separate smem region; compared with the same warps running alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2502_15349_b200/csrc
//        -o smem_contention smem_contention.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace af;

template <int N, bool kMma>
__global__ void __launch_bounds__(288, 1) kern(int iters, long long* cyc, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  uint8_t* opnd = smem;                        // A (32 KB) + B (N x 128 x 2)
  uint8_t* scratch = smem + (128 + 256) * 256;  // the warps' LDS / STS region (32 KB)
  for (int i = threadIdx.x; i < (128 + 256) * 256 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(opnd)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    stop = 0;
  }
  if (warp == 8) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 8) {
    if (kMma && elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
      const uint32_t a = smem_u32(opnd), b = smem_u32(opnd + 128 * 256);
      while (!stop) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem, make_sdesc(a + (kk / 4) * (128 * 128) + (kk % 4) * 32, 0, 1024),
                 make_sdesc(b + (kk / 4) * (N * 128) + (kk % 4) * 32, 0, 1024), idesc, 1);
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  } else {
    // 8 warps: each lane LDS.128 + STS.128 over its own 16-byte granules (conflict-free)
    uint4 acc = make_uint4(0, 0, 0, 0);
    uint4* base = reinterpret_cast<uint4*>(scratch) + warp * 256;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = base[(j * 32 + threadIdx.x % 32) & 255];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc.x ^= v[j].x + v[j].y;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        base[((j + 4) * 32 + threadIdx.x % 32) & 255] = make_uint4(acc.x, i, j, v[j].z);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc.x;
  }
  // stop the MMA thread once the timed warps are done
  __syncwarp();
  if (threadIdx.x == 0) stop = 1;
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int N, bool kMma>
void run(long long* cyc, float* sink) {
  const int iters = 4096;
  const int smem = (128 + 256) * 256 + 32 * 1024;
  cudaFuncSetAttribute(kern<N, kMma>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<N, kMma><<<148, 288, smem>>>(iters, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double bytes = double(iters) * 8 * 8 * 32 * 16;  // 4 LDS + 4 STS of 16 B, 8 warps
  printf("threads' LDS+STS %s (N=%d): %.1f B/clk/SM (%s)\n",
         kMma ? "while SS MMAs stream" : "alone               ", N, bytes / c,
         cudaGetErrorString(e));
}

int main() {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 288 * 4);
  run<128, false>(cyc, sink);
  run<64, true>(cyc, sink);
  run<128, true>(cyc, sink);
  run<256, true>(cyc, sink);
  return 0;
}
