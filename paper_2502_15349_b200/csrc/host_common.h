// Host-side helpers shared by the C-ABI translation units: error state, tensor maps, launch utils.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/attn_b200.h"

namespace af {

void set_error(const char* fmt, ...);
const char* last_error();

#define AF_REQUIRE(cond, code, ...) \
  do {                              \
    if (!(cond)) {                  \
      ::af::set_error(__VA_ARGS__); \
      return (code);                \
    }                               \
  } while (0)

#define AF_CUDA_CHECK(expr)                                                             \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::af::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                      __LINE__);                                                        \
      return AF_ERR_CUDA;                                                               \
    }                                                                                   \
  } while (0)

// 4-D bf16/fp32 tensor map over a [b, h, s, d] tensor given element strides (d stride 1).
// Box = {box_d, box_s, 1, 1}, swizzle 128B (box_d * elem == 128) or none.
bool make_tmap_4d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, int elem_bytes,
                  int d, int s, int h, int b, const int64_t* stride_bhsd, int box_d, int box_s,
                  bool swizzle128);

int sm_count();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device context: cache it per
// (current device, kernel) under a mutex, so a kernel first launched on one GPU still gets the
// attribute on the next GPU of the same process.
int ensure_max_smem(const void* func, int bytes);
#define AF_SMEM_ATTR(kern, bytes)                                                            \
  do {                                                                                       \
    if (::af::ensure_max_smem(reinterpret_cast<const void*>(kern), (bytes)) != AF_OK)        \
      return AF_ERR_CUDA;                                                                    \
  } while (0)

// Process-wide count of kernels this library launched (af_launch_count()).
void note_launch();
void ensure_context();

}  // namespace af
