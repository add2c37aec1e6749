// dist.cpp — multi-GPU key-range sort over NCCL. Placeholder.
#include "runtime.h"

struct ley_comm {
  int nranks = 0, rank = 0, device = 0;
};

namespace ley {
ley_status comm_get_unique_id(uint8_t id_out[128]) {
  (void)id_out;
  set_error("dist: not available in this build");
  return LEY_ERR_UNSUPPORTED;
}
ley_status comm_init(ley_comm** comm, int nranks, int rank, const uint8_t id[128], int device) {
  (void)comm; (void)nranks; (void)rank; (void)id; (void)device;
  set_error("dist: not available in this build");
  return LEY_ERR_UNSUPPORTED;
}
ley_status dist_sort(ley_comm* comm, const void* in_local, uint64_t n_local, void* out_local, uint64_t out_capacity,
                     uint64_t* n_out_local, uint64_t* out_global_offset, uint64_t budget, cudaStream_t s) {
  (void)comm; (void)in_local; (void)n_local; (void)out_local; (void)out_capacity; (void)n_out_local;
  (void)out_global_offset; (void)budget; (void)s;
  set_error("dist: not available in this build");
  return LEY_ERR_UNSUPPORTED;
}
ley_status comm_destroy(ley_comm* comm) {
  (void)comm;
  return LEY_OK;
}
}  // namespace ley
