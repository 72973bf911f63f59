// Entry points not yet implemented on sm_100a; they fail loudly with AF_ERR_UNSUPPORTED.
#include "host_common.h"

extern "C" {
int af_linear_fwd(const af_linear_desc*, const void*, const void*, const void*, const float*,
                  void*, float*, void*) {
  af::set_error("af_linear_fwd not built yet");
  return AF_ERR_UNSUPPORTED;
}
size_t af_linear_bwd_workspace(const af_linear_desc*) { return 0; }
int af_linear_bwd(const af_linear_desc*, const void*, const void*, const void*, const float*,
                  const void*, void*, void*, void*, float*, void*, size_t, void*) {
  af::set_error("af_linear_bwd not built yet");
  return AF_ERR_UNSUPPORTED;
}
size_t af_mla_decode_workspace(const af_mla_desc*) { return 0; }
int af_mla_decode(const af_mla_desc*, const void*, const void*, void*, float*, void*, size_t,
                  void*) {
  af::set_error("af_mla_decode not built yet");
  return AF_ERR_UNSUPPORTED;
}
}
