// Entry points not yet implemented on sm_100a; they fail loudly with AF_ERR_UNSUPPORTED.
#include "host_common.h"

extern "C" {
size_t af_mla_decode_workspace(const af_mla_desc*) { return 0; }
int af_mla_decode(const af_mla_desc*, const void*, const void*, void*, float*, void*, size_t,
                  void*) {
  af::set_error("af_mla_decode not built yet");
  return AF_ERR_UNSUPPORTED;
}
}
