// k_exchange.cu — peer pointers of an NCCL symmetric-memory window, for the fused partition + exchange
// (§8a row a8): rank r's K-p stores records straight into rank d's receive window
// through the pointer ncclGetPeerPointer(win, 0, d), an NVLink/NVSwitch mapping of d's buffer that the
// NCCL device API (nccl_device.h, NCCL 2.28) resolves from the window registered collectively with
// NCCL_WIN_COLL_SYMMETRIC. The pointers are computed once per (re)registration and kept in a device array.
#include <nccl.h>
#include <nccl_device.h>

#include "kernels.cuh"

namespace ley {
namespace {

__global__ void kx_peer_pointers(ncclWindow_t win, int G, uint8_t** out) {
  const int d = threadIdx.x;
  if (d < G) out[d] = static_cast<uint8_t*>(ncclGetPeerPointer(win, 0, d));
}

// Fault-injection test hook (option dist_fault_stall): holds the stream the way a peer that never joins a
// collective would, until the library's abort path releases it through the mapped host flag. Bounded by
// the device clock (60 s), so a missed release can never wedge the GPU.
__global__ void kx_stall(const volatile uint32_t* release) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    if (*release) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60000000000ull) return;
    __nanosleep(10000);
  }
}

}  // namespace

cudaError_t launch_stall(const volatile uint32_t* release, cudaStream_t s) {
  kx_stall<<<1, 1, 0, s>>>(release);
  return cudaGetLastError();
}

cudaError_t launch_peer_pointers(ncclWindow_t win, int G, uint8_t** out, cudaStream_t s) {
  kx_peer_pointers<<<1, 32, 0, s>>>(win, G, out);
  return cudaGetLastError();
}

}  // namespace ley
