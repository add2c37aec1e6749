// k_gather.cu — K-e: payload gather, out[j] = in[perm[j]] for the full 100-byte record.
//
// PAPER.md §3.2: "Leyenda is able to scatter data records directly to the page cache ...
// given the sorted (key, pointer) tuples" — here the destination is HBM instead of the page cache.
// §4.3 line 154 excludes this step from its sort times ("Excluding the time of scattering records"),
// a sign that it is the expensive one; SURVEY.md §8a row a6 and Appendix B (~72% of the bytes).
//
// Output-stationary, asynchronous copies: a warp owns a task of kTaskRecords consecutive output records.
// It reads their ordinals with one coalesced load, then the lanes issue 16-byte cp.async (LDGSTS, no
// register staging) for the 7 aligned chunks of each record's 112-byte window
// [floor(100 p / 16) * 16, +112), which always contains the record; every chunk starts inside the input
// buffer and, being 16-byte aligned, never crosses a page. With ~7 KB of copies in flight per warp the
// gather is not latency-bound. After cp.async.wait_all the warp re-aligns through shared memory and
// writes the task's output with 16-byte streaming stores (tasks start at multiples of 4 records, so the
// output is 16-byte aligned); a ragged final task ends with 4-byte stores.
#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

constexpr int kGatherWarps = 8;
constexpr int kGatherThreads = kGatherWarps * 32;
constexpr int kTaskRecords = 64;                      // records per warp task (multiple of 4)
constexpr int kWindow = 112;                          // 7 x 16 B
constexpr int kStageBytes = kTaskRecords * kWindow + kTaskRecords;  // windows + per-record offsets

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void stg_cs_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kGatherThreads)
    ke_gather(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm, uint8_t* __restrict__ out,
              uint64_t n) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* stage = smem + warp * kStageBytes;
  uint8_t* s_off = stage + kTaskRecords * kWindow;  // byte offset of record r inside its window
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
  const uint64_t ntasks = (n + kTaskRecords - 1) / kTaskRecords;
  const uint64_t nw = (uint64_t)gridDim.x * kGatherWarps;
  for (uint64_t task = (uint64_t)blockIdx.x * kGatherWarps + warp; task < ntasks; task += nw) {
    const uint64_t j0 = task * kTaskRecords;
    const int cnt = (int)(n - j0 < (uint64_t)kTaskRecords ? n - j0 : (uint64_t)kTaskRecords);
    const uint32_t pa = lane < cnt ? __ldg(perm + j0 + lane) : 0u;
    const uint32_t pb = lane + 32 < cnt ? __ldg(perm + j0 + lane + 32) : 0u;
    s_off[lane] = (uint8_t)((pa * 4u) & 15u);  // 100 p mod 16 == 4 p mod 16
    s_off[lane + 32] = (uint8_t)((pb * 4u) & 15u);
#pragma unroll
    for (int q = 0; q < kTaskRecords * 7 / 32; ++q) {
      const int cidx = q * 32 + lane;
      const int r = cidx / 7, c = cidx - r * 7;
      const uint32_t p = __shfl_sync(0xffffffffu, r < 32 ? pa : pb, r & 31);
      if (r < cnt) {
        const uint64_t ws = ((uint64_t)p * kRecordBytes) & ~uint64_t(15);
        cp_async16(stage_s + r * kWindow + c * 16, in + ws + c * 16);
      }
    }
    cp_async_wait_all();
    __syncwarp();
    uint8_t* obase = out + j0 * kRecordBytes;
    const int words = cnt * (int)kRecordWords;
    const int nchunks = words >> 2;
    for (int q = lane; q < nchunks; q += 32) {
      uint32_t wv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int wi = q * 4 + k;
        const int r = wi / 25, o = wi - r * 25;
        wv[k] = *reinterpret_cast<const uint32_t*>(stage + r * kWindow + s_off[r] + 4 * o);
      }
      stg_cs_v4(reinterpret_cast<uint4*>(obase) + q, make_uint4(wv[0], wv[1], wv[2], wv[3]));
    }
    for (int wi = nchunks * 4 + lane; wi < words; wi += 32) {
      const int r = wi / 25, o = wi - r * 25;
      stg_cs_u32(reinterpret_cast<uint32_t*>(obase) + wi,
                 *reinterpret_cast<const uint32_t*>(stage + r * kWindow + s_off[r] + 4 * o));
    }
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_ke_gather(const uint8_t* in, const uint32_t* perm, uint64_t n, uint8_t* out, int sms,
                             cudaStream_t s, int* launches) {
  if (n == 0) return cudaSuccess;
  const size_t smem = (size_t)kGatherWarps * kStageBytes;
  cudaError_t e = cudaFuncSetAttribute(ke_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ke_gather, kGatherThreads, smem);
  if (e != cudaSuccess) return e;
  const uint64_t ntasks = (n + kTaskRecords - 1) / kTaskRecords;
  uint64_t blocks = (ntasks + kGatherWarps - 1) / kGatherWarps;
  const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (blocks > cap) blocks = cap;
  ke_gather<<<(unsigned)blocks, kGatherThreads, smem, s>>>(in, perm, out, n);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  return cudaSuccess;
}

}  // namespace ley
