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

__device__ __forceinline__ int tier_of(uint32_t len, const Tunables& tu) {
  if (len <= tu.warp_tier_max) return kListWarp;
  if (len <= tu.smem_tier_max)
    return len <= 512 ? kListMed1 : len <= 2048 ? kListMed2 : len <= 8192 ? kListMed3 : len <= 10240 ? kListMed4 : kListMed5;
  return kNumKdLists;  // big: recurse
}

// Block-wide classification (every thread of the CTA must call it; `valid` marks threads holding a bucket):
// list appends are aggregated per warp (match.any) and per CTA (shared counters), so each list costs one
// global atomic per CTA instead of one per bucket — buckets of one level number up to 256 x #segments.
// s_cnt: >= 16 u32 of shared memory.
__device__ __forceinline__ void classify_block(const Seg& s, bool valid, const Tunables& tu, const ListSet& kd,
                                               Seg* big_out, uint32_t* big_count, uint32_t* s_cnt) {
  const int list = (valid && s.len) ? tier_of(s.len, tu) : -1;
  if (threadIdx.x < 16) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t peers = __match_any_sync(0xffffffffu, list);
  const int leader = __ffs(peers) - 1;
  const uint32_t rank = __popc(peers & lanemask_lt());
  uint32_t wbase = 0;
  if (list >= 0 && rank == 0) wbase = atomicAdd(&s_cnt[list], (uint32_t)__popc(peers));
  wbase = __shfl_sync(0xffffffffu, wbase, leader);
  __syncthreads();
  if (threadIdx.x <= kNumKdLists && s_cnt[threadIdx.x])
    s_cnt[8 + threadIdx.x] =
        atomicAdd(threadIdx.x == kNumKdLists ? big_count : &kd.counts[threadIdx.x], s_cnt[threadIdx.x]);
  __syncthreads();
  if (list >= 0) {
    const uint32_t slot = s_cnt[8 + list] + wbase + rank;
    if (list == kNumKdLists) big_out[slot] = s;
    else kd.items[list][slot] = s;
  }
}

// Level-1 classification (run by extra CTAs of the K-c plan launch, k_split.cu): bucket p = key bytes
// 0..1 is Seg{B16[p], hist16[p], depth 2, buffer B}; 256 CTAs x 256 buckets. The last CTA to finish
// publishes the big-bucket count into mapped host memory (the host polls it; no separate publish launch).
struct ClassifyJob {
  Tunables tu;
  ListSet kd;
  const uint32_t* hist16;
  const uint32_t* B16;
  Seg* big_out;
  uint32_t* big_count;
  uint32_t* done;         // CTA-done counter (zeroed with the level-1 counters)
  uint32_t* host_mapped;  // device alias of the mapped pinned word the host polls
};
constexpr uint32_t kClassifyBlocks = 256;  // x 256 threads = 65536 buckets

__device__ __forceinline__ void classify_level1_block(const ClassifyJob& cj, uint32_t blk, uint32_t* s_cnt) {
  const uint32_t p = blk * 256 + threadIdx.x;
  const Seg s{cj.B16[p], cj.hist16[p], 2u, 1u};
  classify_block(s, true, cj.tu, cj.kd, cj.big_out, cj.big_count, s_cnt);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(cj.done, 1u) == kClassifyBlocks - 1) {
      __threadfence();
      *reinterpret_cast<volatile uint32_t*>(cj.host_mapped) = *reinterpret_cast<volatile uint32_t*>(cj.big_count);
    }
  }
}

}  // namespace ley
