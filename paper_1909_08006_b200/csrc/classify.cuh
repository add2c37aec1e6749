// classify.cuh — route a finished MSD bucket to its tier (Algorithm 1, lines 60-85):
//   (depth counts consumed bytes of the composite key: key bytes 0..9, then the ordinal's 4 bytes, so
//    a bucket whose 10 key bytes are all equal keeps splitting on its ordinals — P:60/"radix < 10"
//    ends the key; SURVEY Q12 — and every bucket ends as a singleton at depth 14 at the latest)
//   len <= warp_tier_max        -> one-warp comparison network ("ComparisonSort(key)" for
//                                  k < tinyBucketThreshold)
//   len <= smem_tier_max        -> one CTA in shared memory ("SingleThreadRadixSort" of a small bucket,
//                                  P:74-75, load-balanced like smallBucketQueue)
//   otherwise                   -> big bucket: split again on the next byte by the whole device
//                                  ("if k > bigBucketThreshold then MSDRadixSort(key, radix+1, k)")
#pragma once
#include "common.cuh"

namespace ley {

__device__ __forceinline__ void classify_bucket(const Seg& s, const Tunables& tu, const ListSet& kd, Seg* big_out,
                                                uint32_t* big_count) {
  if (s.len == 0) return;
  int list;
  if (s.len <= tu.warp_tier_max) {
    list = kListWarp;
  } else if (s.len <= tu.smem_tier_max) {
    list = s.len <= 512    ? kListMed1
           : s.len <= 2048 ? kListMed2
           : s.len <= 8192 ? kListMed3
           : s.len <= 10240 ? kListMed4
                            : kListMed5;
  } else {
    uint32_t slot = atomicAdd(big_count, 1u);
    big_out[slot] = s;
    return;
  }
  uint32_t slot = atomicAdd(&kd.counts[list], 1u);
  kd.items[list][slot] = s;
}

}  // namespace ley
