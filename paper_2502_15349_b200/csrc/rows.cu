// Row normalisation over materialised score rows — the generic (materialised) tier of the
// parallel template, for variants the fused kernels do not lower (hooks that read arbitrary
// materialised extras, head dims without a fused instantiation, ...).  This is
// attnforge `engine.run_naive_parallel` / `build_parallel` (engine.py:401-406,
// attention.py:389-449) restated on the GPU: S = Qm Km^T and O = P Vm are plain GEMMs, the score
// hooks run as af_hook_eval programs over [B, H, Sq, Sk], and these kernels apply the row
// normalisation (the rownorm families the planner recognises numerically) and its VJP:
//   softmax  p = e^{z - m} / l, stat = m + log l (-inf for fully-masked rows, whose p is 0)
//            (attention.py:556-572);   dz = p (dp - <dO, O>)
//   abssum   a = sum |z|, p = z / clamp(a, 1, inf), stat = a (attention.py:575-586);
//            dz = dp / c - [a >= 1] sign(z) <dO, O> / c, sign(0) = +1 (graph.py:554-557)
//   none     p = z;  dz = dp
// One CTA per row, fp32 throughout, row reductions in a fixed order (deterministic).
#include <cmath>
#include <cuda_bf16.h>

#include "host_common.h"

namespace af {
namespace {

constexpr int kRowThreads = 256;

template <bool kMax>
__device__ float block_reduce(float v, float* red) {
  for (int off = 16; off > 0; off >>= 1) {
    const float o = __shfl_xor_sync(0xffffffffu, v, off);
    v = kMax ? fmaxf(v, o) : v + o;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
  for (int i = 1; i < kRowThreads / 32; ++i) r = kMax ? fmaxf(r, red[i]) : r + red[i];
  return r;
}

__global__ void __launch_bounds__(kRowThreads) rownorm_fwd_kernel(int kind, const float* __restrict__ z,
                                                                  float* __restrict__ p,
                                                                  float* __restrict__ stat,
                                                                  int64_t n) {
  __shared__ float red[kRowThreads / 32];
  const int64_t row = blockIdx.x;
  const float* zr = z + row * n;
  float* pr = p + row * n;
  if (kind == AF_ROWNORM_SOFTMAX) {
    float m = -INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) m = fmaxf(m, zr[j]);
    m = block_reduce<true>(m, red);
    const bool empty = !(m > -INFINITY);
    float l = 0.0f;
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) {
      const float e = empty ? 0.0f : expf(zr[j] - m);
      pr[j] = e;
      l += e;
    }
    l = block_reduce<false>(l, red);
    const float inv = l > 0.0f ? 1.0f / l : 0.0f;
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) pr[j] *= inv;
    if (threadIdx.x == 0) stat[row] = l > 0.0f ? m + logf(l) : -INFINITY;
  } else if (kind == AF_ROWNORM_ABSSUM) {
    float a = 0.0f;
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) a += fabsf(zr[j]);
    a = block_reduce<false>(a, red);
    const float c = fmaxf(a, 1.0f);
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) pr[j] = zr[j] / c;
    if (threadIdx.x == 0) stat[row] = a;
  } else {
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) pr[j] = zr[j];
  }
}

__global__ void __launch_bounds__(kRowThreads) rownorm_bwd_kernel(
    int kind, const float* __restrict__ z, const float* __restrict__ p,
    const float* __restrict__ dp, const float* __restrict__ rowdot,
    const float* __restrict__ stat, float* __restrict__ dz, int64_t n) {
  const int64_t row = blockIdx.x;
  const float* zr = z + row * n;
  const float* pr = p + row * n;
  const float* dpr = dp + row * n;
  float* dzr = dz + row * n;
  if (kind == AF_ROWNORM_SOFTMAX) {
    const float d = rowdot[row];
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) dzr[j] = pr[j] * (dpr[j] - d);
  } else if (kind == AF_ROWNORM_ABSSUM) {
    const float a = stat[row], c = fmaxf(a, 1.0f), d = rowdot[row];
    const float clamp_live = a >= 1.0f ? 1.0f : 0.0f;
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) {
      const float sg = zr[j] >= 0.0f ? 1.0f : -1.0f;
      dzr[j] = dpr[j] / c - clamp_live * sg * d / c;
    }
  } else {
    for (int64_t j = threadIdx.x; j < n; j += kRowThreads) dzr[j] = dpr[j];
  }
}

// <a_r, b_r> over rows of two [R, D] tensors (bf16 or fp32, row strides given), fp32 out.
__global__ void __launch_bounds__(kRowThreads) rowdot_kernel(af_hook_operand a, af_hook_operand b,
                                                             int64_t d, int heads, int seq,
                                                             float* __restrict__ out) {
  __shared__ float red[kRowThreads / 32];
  const int64_t row = blockIdx.x;
  const int s = static_cast<int>(row % seq);
  const int h = static_cast<int>((row / seq) % heads);
  const int bb = static_cast<int>(row / (static_cast<int64_t>(seq) * heads));
  auto at = [&](const af_hook_operand& t, int64_t j) {
    const int64_t off = bb * t.stride[0] + h * t.stride[1] + s * t.stride[2] + j * t.stride[3];
    return t.dtype == AF_DTYPE_BF16
               ? __bfloat162float(static_cast<const __nv_bfloat16*>(t.ptr)[off])
               : static_cast<const float*>(t.ptr)[off];
  };
  float acc = 0.0f;
  for (int64_t j = threadIdx.x; j < d; j += kRowThreads) acc += at(a, j) * at(b, j);
  acc = block_reduce<false>(acc, red);
  if (threadIdx.x == 0) out[row] = acc;
}

}  // namespace
}  // namespace af

extern "C" int af_rownorm_fwd(int32_t kind, const float* z, float* p, float* stat, int64_t rows,
                              int64_t n, void* stream) {
  using namespace af;
  AF_REQUIRE(kind >= AF_ROWNORM_NONE && kind <= AF_ROWNORM_ABSSUM, AF_ERR_INPUT,
             "unknown rownorm kind %d", kind);
  AF_REQUIRE(z != nullptr && p != nullptr && (kind == AF_ROWNORM_NONE || stat != nullptr),
             AF_ERR_INPUT, "null rownorm buffer");
  AF_REQUIRE(rows >= 0 && n >= 1 && rows < (1LL << 31), AF_ERR_SHAPE, "bad rownorm extents");
  if (rows == 0) return AF_OK;
  ::af::note_launch();
  rownorm_fwd_kernel<<<static_cast<unsigned>(rows), kRowThreads, 0,
                       reinterpret_cast<cudaStream_t>(stream)>>>(kind, z, p, stat, n);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

extern "C" int af_rownorm_bwd(int32_t kind, const float* z, const float* p, const float* dp,
                              const float* rowdot, const float* stat, float* dz, int64_t rows,
                              int64_t n, void* stream) {
  using namespace af;
  AF_REQUIRE(kind >= AF_ROWNORM_NONE && kind <= AF_ROWNORM_ABSSUM, AF_ERR_INPUT,
             "unknown rownorm kind %d", kind);
  AF_REQUIRE(dp != nullptr && dz != nullptr, AF_ERR_INPUT, "null rownorm buffer");
  AF_REQUIRE(kind == AF_ROWNORM_NONE || (p != nullptr && rowdot != nullptr), AF_ERR_INPUT,
             "softmax / abssum VJP needs p and <dO, O>");
  AF_REQUIRE(kind != AF_ROWNORM_ABSSUM || (z != nullptr && stat != nullptr), AF_ERR_INPUT,
             "abssum VJP needs z and the row abs-sum");
  AF_REQUIRE(rows >= 0 && n >= 1 && rows < (1LL << 31), AF_ERR_SHAPE, "bad rownorm extents");
  if (rows == 0) return AF_OK;
  ::af::note_launch();
  rownorm_bwd_kernel<<<static_cast<unsigned>(rows), kRowThreads, 0,
                       reinterpret_cast<cudaStream_t>(stream)>>>(kind, z, p, dp, rowdot, stat, dz,
                                                                 n);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

extern "C" int af_rowdot(const af_hook_operand* a, const af_hook_operand* b, const int32_t* shape,
                         float* out, void* stream) {
  using namespace af;
  AF_REQUIRE(a != nullptr && b != nullptr && shape != nullptr && out != nullptr, AF_ERR_INPUT,
             "null rowdot argument");
  const int64_t rows = static_cast<int64_t>(shape[0]) * shape[1] * shape[2];
  AF_REQUIRE(rows >= 0 && rows < (1LL << 31) && shape[3] >= 1, AF_ERR_SHAPE,
             "bad rowdot extents");
  if (rows == 0) return AF_OK;
  ::af::note_launch();
  rowdot_kernel<<<static_cast<unsigned>(rows), kRowThreads, 0,
                  reinterpret_cast<cudaStream_t>(stream)>>>(*a, *b, shape[3], shape[1], shape[2],
                                                            out);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}
