// Developer check of the CTA-pair (cta_group::2) mechanics the paired MLA backward kernels use:
// a cluster of 2 CTAs computes D[256 x 128] = A[256 x 64] B[128 x 64]^T with
//   * A split by rows (each CTA its 128 rows; SS: smem, TS: TMEM), B split by rows of N (each CTA
//     64 of the 128 B rows), each CTA's TMA completing on the LEADER's mbarrier;
//   * tcgen05.alloc / dealloc .cta_group::2, the MMA issued by the leader only, and
//     tcgen05.commit .cta_group::2 multicast to both CTAs' barriers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I ../../paper_2502_15349_b200/csrc
//        -o pair_mma pair_mma.cu ../../paper_2502_15349_b200/csrc/host_common.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "host_common.h"
#include "sm100.cuh"

using namespace af;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

template <bool kTS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;            // [128][64] bf16, SW128 (16 KB)
  uint8_t* sB = smem + 16384;    // [64][64] bf16, SW128 (8 KB)
  __shared__ __align__(8) uint64_t full, done;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t full_leader = map_to_rank(smem_u32(&full), 0);
  if (threadIdx.x == 0) {
    if (rank == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full)),
                   "r"(2 * (16384 + 8192))
                   : "memory");
    // each CTA loads its own halves; the transaction bytes complete on the leader's barrier
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(sA)),
        "l"(reinterpret_cast<uint64_t>(&tm_a)), "r"(0), "r"(static_cast<int>(rank) * 128), "r"(0),
        "r"(0), "r"(full_leader)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(sB)),
        "l"(reinterpret_cast<uint64_t>(&tm_b)), "r"(0), "r"(static_cast<int>(rank) * 64), "r"(0),
        "r"(0), "r"(full_leader)
        : "memory");
  }
  if constexpr (kTS) {
    // A rows into TMEM columns [128, 160): each CTA its own 128 rows (needs the A bytes in smem:
    // wait for the leader's barrier from every thread of this CTA is not possible (remote), so
    // the leader signals "a_ready" below via a cluster barrier instead)
  }
  // both CTAs' data must be in smem before the TS copy / the MMA: leader waits its barrier,
  // then a cluster barrier publishes that to the peer
  if (rank == 0 && threadIdx.x == 0) mbar_wait(&full, 0);
  cluster_sync();
  if constexpr (kTS) {
    const int row = threadIdx.x;  // TMEM lane
    uint32_t v[32];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const uint4 q = *reinterpret_cast<const uint4*>(sA + row * 128 + ((g ^ (row & 7)) << 4));
      v[g * 4] = q.x;
      v[g * 4 + 1] = q.y;
      v[g * 4 + 2] = q.z;
      v[g * 4 + 3] = q.w;
    }
    tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 128, v);
    tmem_st_wait();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
  }
  if (rank == 0 && threadIdx.x == 0) {
    tc_fence_after();
    // M = 256 (both CTAs' A rows), N = 128 (both CTAs' B halves)
    constexpr uint32_t id = make_idesc_bf16(256, 128, false, false);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t bd = make_sdesc(smem_u32(sB) + kk * 32, 0, 1024);
      if constexpr (kTS)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
            "r"(tmem + 128 + kk * 8), "l"(bd), "r"(id), "r"(kk > 0 ? 1u : 0u)
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(make_sdesc(smem_u32(sA) + kk * 32, 0, 1024)), "l"(bd), "r"(id),
            "r"(kk > 0 ? 1u : 0u)
            : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(&done)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  {
    const int row = threadIdx.x;
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, v);
      tmem_ld_wait();
      for (int e = 0; e < 32; ++e)
        out[(rank * 128 + row) * 128 + c * 32 + e] = __uint_as_float(v[e]);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

int main() {
  const int M = 256, N = 128, K = 64;
  std::vector<__nv_bfloat16> a(M * K), b(N * K);
  std::vector<float> af(M * K), bf(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) {
    af[i] = __bfloat162float(__float2bfloat16((rand() % 200 - 100) / 64.0f));
    a[i] = __float2bfloat16(af[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    bf[i] = __bfloat162float(__float2bfloat16((rand() % 200 - 100) / 64.0f));
    b[i] = __float2bfloat16(bf[i]);
  }
  __nv_bfloat16 *da, *db;
  float* dout;
  cudaMalloc(&da, a.size() * 2);
  cudaMalloc(&db, b.size() * 2);
  cudaMalloc(&dout, M * N * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  const int64_t sa[4] = {0, 0, K, 1}, sb[4] = {0, 0, K, 1};
  if (!make_tmap_4d(&ta, da, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, M, 1, 1, sa, 64, 128, true) ||
      !make_tmap_4d(&tb, db, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, N, 1, 1, sb, 64, 64, true)) {
    printf("tmap failed\n");
    return 1;
  }
  for (int ts = 0; ts < 2; ++ts) {
    cudaMemset(dout, 0, M * N * 4);
    auto kern = ts ? pair_kernel<true> : pair_kernel<false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    kern<<<2, 128, 32768>>>(ta, tb, dout);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(M * N);
    cudaMemcpy(out.data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += double(af[i * K + k]) * bf[j * K + k];
        maxerr = std::max(maxerr, std::abs(s - out[i * N + j]));
      }
    printf("%s: %s, max abs err %.3e (out[0]=%f out[last]=%f)\n", ts ? "TS" : "SS",
           cudaGetErrorString(e), maxerr, out[0], out[M * N - 1]);
  }
  return 0;
}
