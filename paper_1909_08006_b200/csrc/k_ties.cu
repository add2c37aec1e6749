// k_ties.cu — keys longer than 10 bytes, hybrid form (§5: "make Leyenda hybrid between prefix
// sorting and comparison-based record sorting"). The radix sort orders the records by their first 10 key
// bytes (ties by input index); only records whose 10-byte prefixes tie need the rest of the key:
//   kt_tie_groups  one pass over the sorted records: maximal runs of equal 10-byte prefixes ("tie groups",
//                  >= 2 records) are reported as (first, last) positions (unordered lists; the host pairs
//                  them after sorting both, as groups never overlap)
//   kt_fix_small   one warp per tie group of <= 32 records: each lane ranks its record against the others
//                  by (key bytes [10, key_bytes), position) — a comparison sort on the records themselves —
//                  and the group is rewritten in place in that order
// Larger groups are sorted by the LSD window passes restricted to their slice (internal.cu).
#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

__device__ __forceinline__ bool prefix10_equal(const uint8_t* a, const uint8_t* b) {
  // records are 4-byte aligned: words 0, 1 and the low half of word 2
  const uint32_t* x = reinterpret_cast<const uint32_t*>(a);
  const uint32_t* y = reinterpret_cast<const uint32_t*>(b);
  return x[0] == y[0] && x[1] == y[1] && ((x[2] ^ y[2]) & 0xFFFFu) == 0;
}

// dg (nullable): the prefix digests K-e wrote beside the records (k_bucket.cu prefix_digest); equal
// prefixes have equal digests, so only adjacent records with equal digests are compared on the records.
__global__ void kt_tie_groups(const uint8_t* __restrict__ recs, const uint64_t* __restrict__ dg, uint64_t n,
                              uint32_t* __restrict__ firsts, uint32_t* __restrict__ lasts, uint32_t cap,
                              uint32_t* __restrict__ counts) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t* r = recs + j * kRecordBytes;
    bool cand_prev = j > 0, cand_next = j + 1 < n;
    if (dg) {
      const uint64_t d = dg[j];
      cand_prev = cand_prev && dg[j - 1] == d;
      cand_next = cand_next && dg[j + 1] == d;
    }
    const bool tie_prev = cand_prev && prefix10_equal(r - kRecordBytes, r);
    const bool tie_next = cand_next && prefix10_equal(r, r + kRecordBytes);
    if (tie_next && !tie_prev) {
      const uint32_t at = atomicAdd(&counts[0], 1u);
      if (at < cap) firsts[at] = (uint32_t)j;
    }
    if (tie_prev && !tie_next) {
      const uint32_t at = atomicAdd(&counts[1], 1u);
      if (at < cap) lasts[at] = (uint32_t)j;
    }
  }
}

// key bytes [10, kb) of records a and b (positions in `recs`), unsigned; ties by position
__device__ __forceinline__ bool tail_less(const uint8_t* recs, uint32_t a, uint32_t b, uint32_t kb) {
  const uint8_t* x = recs + (uint64_t)a * kRecordBytes;
  const uint8_t* y = recs + (uint64_t)b * kRecordBytes;
  for (uint32_t i = kKeyBytes; i < kb; ++i) {
    const uint32_t u = x[i], v = y[i];
    if (u != v) return u < v;
  }
  return a < b;
}

__global__ void kt_fix_small(uint8_t* __restrict__ recs, const uint2* __restrict__ groups, uint32_t ngroups,
                             uint32_t kb) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < ngroups; g += warps) {
    const uint2 grp = groups[g];  // (first, len), len in [2, 32]
    const bool active = (uint32_t)lane < grp.y;
    const uint32_t me = grp.x + lane;
    uint32_t rank = 0;
    if (active)
      for (uint32_t m = 0; m < grp.y; ++m)
        if (m != (uint32_t)lane && tail_less(recs, grp.x + m, me, kb)) ++rank;
    uint32_t w[kRecordWords];
    const uint32_t* src = reinterpret_cast<const uint32_t*>(recs + (uint64_t)me * kRecordBytes);
#pragma unroll
    for (int q = 0; q < (int)kRecordWords; ++q) w[q] = active ? src[q] : 0u;
    __syncwarp();  // every lane holds its record before any is overwritten
    if (active) {
      uint32_t* dst = reinterpret_cast<uint32_t*>(recs + (uint64_t)(grp.x + rank) * kRecordBytes);
#pragma unroll
      for (int q = 0; q < (int)kRecordWords; ++q) dst[q] = w[q];
    }
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_tie_groups(const uint8_t* recs, const uint64_t* dg, uint64_t n, uint32_t* firsts, uint32_t* lasts, uint32_t cap,
                              uint32_t* counts, int sms, cudaStream_t s) {
  if (n < 2) return cudaSuccess;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
  kt_tie_groups<<<(unsigned)blocks, 256, 0, s>>>(recs, dg, n, firsts, lasts, cap, counts);
  return cudaGetLastError();
}

cudaError_t launch_fix_small_groups(uint8_t* recs, const uint2* groups, uint32_t ngroups, uint32_t key_bytes, int sms,
                                    cudaStream_t s) {
  if (!ngroups) return cudaSuccess;
  uint64_t blocks = (ngroups + 7) / 8;
  if (blocks > (uint64_t)sms * 16) blocks = (uint64_t)sms * 16;
  kt_fix_small<<<(unsigned)blocks, 256, 0, s>>>(recs, groups, ngroups, key_bytes);
  return cudaGetLastError();
}

}  // namespace ley
