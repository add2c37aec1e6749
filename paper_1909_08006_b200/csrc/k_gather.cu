// k_gather.cu — K-e as a stand-alone kernel over one window of the sorted order, for the resident host
// path (resident.cu): out[j] = in[perm[j]] for j in [0, cnt) (§3.2: "scatter data
// records ... given the sorted (key, pointer) tuples"). The sort itself ran in
// perm-only mode; each window of the output is gathered into a device staging buffer and copied to the
// caller's pinned host memory while the next window is gathered.
//
// One warp per 32 consecutive output records: lane L owns perm[j0 + L]; the 32 x 25 words are copied as
// 25 rounds of 32 flattened words (record w / 25, word w % 25, the source ordinal taken from its owner
// lane by a shuffle), so every store instruction writes 128 contiguous bytes and the loads of one round
// touch at most two source records.
#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

constexpr int kGatherThreads = 256;

__global__ void __launch_bounds__(kGatherThreads) ke_gather(const uint8_t* __restrict__ in,
                                                            const uint32_t* __restrict__ perm, uint64_t cnt,
                                                            uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (kGatherThreads / 32);
  const uint32_t* in32 = reinterpret_cast<const uint32_t*>(in);
  uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
  for (uint64_t g = (uint64_t)blockIdx.x * (kGatherThreads / 32) + (threadIdx.x >> 5); g * 32 < cnt; g += warps) {
    const uint64_t j0 = g * 32;
    const uint32_t m = cnt - j0 < 32 ? (uint32_t)(cnt - j0) : 32u;
    const uint32_t p = (uint32_t)lane < m ? __ldg(perm + j0 + lane) : 0u;
    uint32_t v[kRecordWords];
#pragma unroll
    for (int q = 0; q < (int)kRecordWords; ++q) {  // all loads first
      const uint32_t w = (uint32_t)q * 32u + (uint32_t)lane;
      const uint32_t r = w / kRecordWords, c = w - r * kRecordWords;
      const uint32_t pr = __shfl_sync(0xffffffffu, p, r & 31u);
      v[q] = r < m ? __ldg(in32 + (uint64_t)pr * kRecordWords + c) : 0u;
    }
#pragma unroll
    for (int q = 0; q < (int)kRecordWords; ++q) {
      const uint32_t w = (uint32_t)q * 32u + (uint32_t)lane;
      if (w < m * kRecordWords) out32[j0 * kRecordWords + w] = v[q];
    }
  }
}

__global__ void ke_compose_perm(const uint32_t* __restrict__ prev, uint32_t* __restrict__ cur, uint64_t n) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    cur[j] = __ldg(prev + cur[j]);
}

}  // namespace

cudaError_t launch_compose_perm(const uint32_t* prev, uint32_t* cur, uint64_t n, int sms, cudaStream_t s) {
  if (!n) return cudaSuccess;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
  ke_compose_perm<<<(unsigned)blocks, 256, 0, s>>>(prev, cur, n);
  return cudaGetLastError();
}

cudaError_t launch_ke_gather(const uint8_t* in, const uint32_t* perm, uint64_t cnt, uint8_t* out, int sms,
                             cudaStream_t s) {
  if (!cnt) return cudaSuccess;
  const uint64_t groups = (cnt + 31) / 32, per_block = kGatherThreads / 32;
  uint64_t blocks = (groups + per_block - 1) / per_block;
  const uint64_t cap = (uint64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  ke_gather<<<(unsigned)blocks, kGatherThreads, 0, s>>>(in, perm, cnt, out);
  return cudaGetLastError();
}

}  // namespace ley
