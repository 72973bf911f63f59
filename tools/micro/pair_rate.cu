// Developer microbenchmark: issue-to-completion rate of tcgen05.mma.cta_group::2 (M = 256 over a
// CTA pair, N = 128, K = 16, bf16 -> fp32), SS and TS (A from TMEM), one issuing thread in the
// leader, against the floor of 64 cycles per instruction per SM (the cta_group::1 M = 128 rate).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2502_15349_b200/csrc
//        -o pair_rate pair_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace af;

template <bool kTS, bool kPair>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    rate_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if constexpr (kPair)
      tmem_alloc_pair<512>(&slot);
    else
      tmem_alloc<512>(&slot);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && (rank == 0 || !kPair) && elect_one()) {
    constexpr uint32_t id = make_idesc_bf16(kPair ? 256 : 128, 128, false, false);
    const uint32_t b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = make_sdesc(b + (kk / 4) * 8192 + (kk % 4) * 32, 0, 1024);
        if constexpr (kPair) {
          if constexpr (kTS)
            mma_ts_pair(tmem + 256, tmem + kk * 8, bd, id, 1);
          else
            mma_ss_pair(tmem + 256, make_sdesc(smem_u32(smem) + (kk / 4) * 16384 + (kk % 4) * 32, 0, 1024),
                        bd, id, 1);
        } else {
          if constexpr (kTS)
            mma_ts(tmem + 256, tmem + kk * 8, bd, id, 1);
          else
            mma_ss(tmem + 256, make_sdesc(smem_u32(smem) + (kk / 4) * 16384 + (kk % 4) * 32, 0, 1024),
                   bd, id, 1);
        }
      }
    }
    if constexpr (kPair)
      mma_commit_pair(&bar);
    else
      mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  } else if (warp == 0 && kPair && rank == 1) {
    // the peer's barrier receives the multicast commit
  }
  if (kPair && rank == 1 && threadIdx.x == 0) mbar_wait(&bar, 0);
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    if constexpr (kPair)
      tmem_dealloc_pair<512>(tmem);
    else
      tmem_dealloc<512>(tmem);
  }
}

template <bool kTS, bool kPair>
void run(long long* cyc) {
  const int iters = 2000;
  cudaFuncSetAttribute(rate_kernel<kTS, kPair>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  rate_kernel<kTS, kPair><<<148, 128, 65536>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%s %s M=%d N=128 K=16: %.1f clk per instruction (per-SM floor 64) (%s)\n",
         kPair ? "cta_group::2" : "cta_group::1", kTS ? "TS" : "SS", kPair ? 256 : 128,
         c / (iters * 8.0), cudaGetErrorString(e));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<false, false>(cyc);
  run<true, false>(cyc);
  run<false, true>(cyc);
  run<true, true>(cyc);
  return 0;
}
