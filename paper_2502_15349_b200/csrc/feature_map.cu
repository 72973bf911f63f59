// Elementwise feature maps of the templates' q_mod / k_mod / v_mod hooks (attnforge
// `AttentionSpec.q_mod/k_mod/v_mod`, attention.py:200-205; AttentionEngine's `feature_map`) and
// their VJPs, for the forms the planner recognises as a function of the tensor alone:
//   silu  x * sigmoid(x)   (the `silu-retention` variant, data/variants/silu-retention.json)
//   sigmoid, relu, tanh, exp
// Applied once per call ahead of the attention kernels (bf16 in, fp32 math, bf16 out), so every
// template kernel sees the mapped tensor; the backward maps dL/d(f(x)) to dL/dx.  The relu
// derivative at 0 routes to the first max operand (graph.py:517-527), i.e. 1.
#include <cuda_bf16.h>

#include <algorithm>

#include "host_common.h"

namespace af {
namespace {

enum FeatureMap : int { kFmNone = 0, kFmSilu = 1, kFmSigmoid = 2, kFmRelu = 3, kFmTanh = 4, kFmExp = 5 };

__device__ __forceinline__ float fm_sig(float x) { return 1.0f / (1.0f + __expf(-x)); }

__device__ __forceinline__ float fm_fwd(int kind, float x) {
  switch (kind) {
    case kFmSilu: return x * fm_sig(x);
    case kFmSigmoid: return fm_sig(x);
    case kFmRelu: return fmaxf(x, 0.0f);
    case kFmTanh: return tanhf(x);
    case kFmExp: return __expf(x);
    default: return x;
  }
}

__device__ __forceinline__ float fm_grad(int kind, float x) {
  switch (kind) {
    case kFmSilu: {
      const float s = fm_sig(x);
      return s * (1.0f + x * (1.0f - s));
    }
    case kFmSigmoid: {
      const float s = fm_sig(x);
      return s * (1.0f - s);
    }
    case kFmRelu: return x >= 0.0f ? 1.0f : 0.0f;
    case kFmTanh: {
      const float t = tanhf(x);
      return 1.0f - t * t;
    }
    case kFmExp: return __expf(x);
    default: return 1.0f;
  }
}

// 8 bf16 per thread (16-byte vectors); n is a multiple of 8 (checked on the host)
__global__ void feature_map_kernel(int kind, int backward, const uint4* __restrict__ x,
                                   const uint4* __restrict__ dy, uint4* __restrict__ y,
                                   int64_t n8) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 xv = x[i];
    const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv);
    uint4 out;
    __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&out);
    if (backward) {
      const uint4 gv = dy[i];
      const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gv);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 xf = __bfloat1622float2(xp[e]), gf = __bfloat1622float2(gp[e]);
        op[e] = __floats2bfloat162_rn(gf.x * fm_grad(kind, xf.x), gf.y * fm_grad(kind, xf.y));
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 xf = __bfloat1622float2(xp[e]);
        op[e] = __floats2bfloat162_rn(fm_fwd(kind, xf.x), fm_fwd(kind, xf.y));
      }
    }
    y[i] = out;
  }
}

}  // namespace
}  // namespace af

extern "C" int af_feature_map(int kind, int backward, const void* x, const void* dy, void* y,
                              int64_t n, void* stream) {
  using namespace af;
  AF_REQUIRE(kind >= kFmNone && kind <= kFmExp, AF_ERR_INPUT, "unknown feature map %d", kind);
  AF_REQUIRE(n >= 0 && n % 8 == 0, AF_ERR_INPUT, "feature map length %lld not a multiple of 8",
             static_cast<long long>(n));
  AF_REQUIRE(!backward || dy != nullptr, AF_ERR_INPUT, "feature map VJP needs dy");
  if (n == 0) return AF_OK;
  const int64_t n8 = n / 8;
  const int threads = 256;
  const int64_t want = (n8 + threads - 1) / threads;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(want, 16LL * sm_count()));
  ::af::note_launch();
  feature_map_kernel<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      kind, backward, static_cast<const uint4*>(x), static_cast<const uint4*>(dy),
      static_cast<uint4*>(y), n8);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}
