// Error state, tensor-map encoding (driver entry point resolved through the runtime, so the
// library has no link-time dependency on libcuda) and device queries.
#include "host_common.h"

#include <atomic>
#include <mutex>
#include <set>
#include <utility>

namespace af {

namespace {
thread_local std::string g_last_error;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}
}  // namespace

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

const char* last_error() { return g_last_error.c_str(); }

int ensure_max_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  AF_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, func})) return AF_OK;
  AF_CUDA_CHECK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({dev, func});
  return AF_OK;
}

std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void ensure_context() {
  // The library links the CUDA runtime statically; a thread that has not touched CUDA through
  // *this* runtime (e.g. torch's autograd worker) may have no current driver context.
  using GetCurrentFn = CUresult (*)(CUcontext*);
  static GetCurrentFn get_current = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuCtxGetCurrent", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      get_current = reinterpret_cast<GetCurrentFn>(p);
  });
  CUcontext ctx = nullptr;
  if (get_current == nullptr || get_current(&ctx) != CUDA_SUCCESS || ctx == nullptr) cudaFree(0);
}

bool make_tmap_4d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, int elem_bytes,
                  int d, int s, int h, int b, const int64_t* st, int box_d, int box_s,
                  bool swizzle128) {
  ensure_context();
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old or no GPU)");
    return false;
  }
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(s),
                        static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(b)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(st[2] * elem_bytes),
                           static_cast<cuuint64_t>(st[1] * elem_bytes),
                           static_cast<cuuint64_t>(st[0] * elem_bytes)};
  // Broadcast / size-1 axes may carry any stride; TMA wants a positive multiple of 16.
  for (int i = 0; i < 3; ++i) {
    if (dims[i + 1] == 1 && strides[i] % 16 != 0) strides[i] = 16;
    if (strides[i] % 16 != 0) {
      set_error("tensor stride %llu bytes is not a multiple of 16 (TMA)",
                static_cast<unsigned long long>(strides[i]));
      return false;
    }
  }
  if (st[3] != 1) {
    set_error("innermost (feature) stride must be 1");
    return false;
  }
  cuuint32_t box[4] = {static_cast<cuuint32_t>(box_d), static_cast<cuuint32_t>(box_s), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, dtype, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) dims=[%d,%d,%d,%d]", static_cast<int>(r), d, s,
              h, b);
    return false;
  }
  return true;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace af

extern "C" {

const char* af_status_string(int status) {
  switch (status) {
    case AF_OK: return "ok";
    case AF_ERR_INPUT: return "input";
    case AF_ERR_SHAPE: return "shape-mismatch";
    case AF_ERR_UNSUPPORTED: return "unsupported";
    case AF_ERR_NAN: return "nan-in-output";
    case AF_ERR_CUDA: return "cuda";
    default: return "unknown";
  }
}

const char* af_last_error(void) { return af::last_error(); }

int af_device_sm_count(void) { return af::sm_count(); }

uint64_t af_launch_count(void) { return af::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
