// external.cu — the external path (pinned host in/out larger than the device budget). Placeholder.
#include "runtime.h"

namespace ley {
ley_status sort_external_host(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint32_t* perm_out, uint64_t n,
                              uint64_t budget, cudaStream_t s, Profiler& prof) {
  (void)ctx; (void)in; (void)out; (void)perm_out; (void)n; (void)budget; (void)s; (void)prof;
  set_error("external path: not available in this build");
  return LEY_ERR_UNSUPPORTED;
}
}  // namespace ley
