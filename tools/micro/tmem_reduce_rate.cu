// Developer microbenchmarks that size the fused (5-GEMM) backward:
//  (1) tcgen05.ld throughput per SM vs the number of warps reading TMEM concurrently;
//  (2) L2 fp32 reduce-add throughput chip-wide: TMA bulk reduce (cp.reduce.async.bulk .add.f32)
//      from shared memory, and red.global.add.v4.f32 from registers, to distinct addresses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_reduce_rate tmem_reduce_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kWarps>
__global__ void __launch_bounds__(kWarps * 32, 1) tmem_ld_kernel(int iters, long long* cycles,
                                                                 uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
  const uint32_t col0 = (warp / 4) * 32 % 512;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + lane_base + ((col0 + (i & 3) * 128) % 512)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 32; ++e) acc ^= r[e];
  }
  __syncthreads();
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Each CTA reduces `chunk` bytes from its smem buffer into a private slice of `dst`, `iters`
// times, cycling over `slices` distinct destinations (so L2 sees distinct lines).
__global__ void tma_reduce_kernel(float* dst, int chunk, int iters, int slices) {
  extern __shared__ __align__(128) float buf[];
  for (int i = threadIdx.x; i < chunk / 4; i += blockDim.x) buf[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      float* g = dst + (static_cast<int64_t>(blockIdx.x) * slices + (i % slices)) * (chunk / 4);
      asm volatile(
          "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(g),
          "r"(smem_u32(buf)), "r"(chunk)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void red_v4_kernel(float* dst, int iters, int slices) {
  // each warp writes 512 contiguous bytes per instruction (coalesced v4 reductions)
  const int64_t per_cta = static_cast<int64_t>(blockDim.x) * 4;
  for (int i = 0; i < iters; ++i) {
    float* g = dst + (static_cast<int64_t>(blockIdx.x) * slices + (i % slices)) * per_cta +
               threadIdx.x * 4;
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(g), "f"(1.0f), "f"(1.0f),
                 "f"(1.0f), "f"(1.0f)
                 : "memory");
  }
}

int main() {
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 4096;
  auto run_ld = [&](auto kern, int warps) {
    kern<<<148, warps * 32>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double bytes = double(iters) * warps * 32 * 32 * 4;
    printf("tmem_ld warps %2d: %.1f B/clk/SM (%s)\n", warps, bytes / c, cudaGetErrorString(e));
  };
  run_ld(tmem_ld_kernel<1>, 1);
  run_ld(tmem_ld_kernel<4>, 4);
  run_ld(tmem_ld_kernel<8>, 8);
  run_ld(tmem_ld_kernel<16>, 16);

  float* dst;
  const size_t bytes = size_t(2) << 30;
  cudaMalloc(&dst, bytes);
  cudaMemset(dst, 0, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t footprint : {size_t(32) << 20, size_t(96) << 20, bytes}) {
  for (int chunk : {8192, 32768}) {
    const int slices = static_cast<int>(footprint / (size_t(148 * 2) * chunk));
    cudaFuncSetAttribute(tma_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk);
    for (int ctas_per_sm : {1, 2}) {
      const int grid = 148 * ctas_per_sm;
      const int it = 2000;
      tma_reduce_kernel<<<grid, 128, chunk>>>(dst, chunk, 10, slices);
      cudaEventRecord(a);
      tma_reduce_kernel<<<grid, 128, chunk>>>(dst, chunk, it, slices);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("tma bulk reduce footprint %5zu MB chunk %6d B, %d CTA/SM: %.0f GB/s (%s)\n",
             footprint >> 20, chunk, ctas_per_sm,
             double(grid) * it * chunk / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
    }
  }
  }
  for (size_t footprint : {size_t(32) << 20, bytes})
  for (int threads : {256, 1024}) {
    const int grid = 148 * 2;
    const int it = 2000;
    const int slices = static_cast<int>(footprint / (size_t(grid) * threads * 16));
    red_v4_kernel<<<grid, threads>>>(dst, 10, slices);
    cudaEventRecord(a);
    red_v4_kernel<<<grid, threads>>>(dst, it, slices);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("red.global.add.v4.f32 footprint %5zu MB %4d thr x 2 CTA/SM: %.0f GB/s (%s)\n",
           footprint >> 20, threads,
           double(grid) * it * threads * 16 / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
  }
  return 0;
}
