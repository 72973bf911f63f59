// Developer microbenchmark: tcgen05.mma (kind::f16, bf16 in, fp32 accumulate, cta_group::1)
// issue-to-completion rate per SM for the tile shapes the attention kernels use — SS (both
// operands in shared memory) vs TS (A in TMEM) and N = 64 / 128 / 256 — to tell whether an SS MMA
// with a small N is bound by the shared-memory operand reads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2502_15349_b200/csrc
//        -o mma_rate mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace af;

template <int N, bool kTS>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (128 + 256) * 128 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 128 * 128 * 2);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = make_sdesc(b + (kk / 4) * (N * 128) + (kk % 4) * 32, 0, 1024);
        if constexpr (kTS)
          mma_ts(tmem + 256, tmem + kk * 8, bd, idesc, 1);
        else
          mma_ss(tmem + 256, make_sdesc(a + (kk / 4) * (128 * 128) + (kk % 4) * 32, 0, 1024), bd,
                 idesc, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int N, bool kTS>
void run(long long* cyc) {
  const int iters = 2000;
  const int smem = (128 + 256) * 128 * 2;
  cudaFuncSetAttribute(mma_kernel<N, kTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_kernel<N, kTS><<<148, 128, smem>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double ksteps = double(iters) * 8;
  printf("%s M=128 N=%3d K=16: %.1f clk per k-step (floor %d), %.0f%% of floor rate (%s)\n",
         kTS ? "TS" : "SS", N, c / ksteps, 128 * N / 256, 100.0 * (128 * N / 256) / (c / ksteps),
         cudaGetErrorString(e));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<64, false>(cyc);
  run<64, true>(cyc);
  run<128, false>(cyc);
  run<128, true>(cyc);
  run<256, false>(cyc);
  run<256, true>(cyc);
  return 0;
}
