// block_rank.cuh — stable block-wide ranking of one 8-bit digit per item (warp multi-split).
//
// The in-CTA counterpart of PAPER.md §3.1 line 96 ("compute a histogram based on the current radix to
// decide the size of each bucket and where each key should be placed"): items are ranked in element
// order e = warp * 32 * ITEMS + j * 32 + lane, so equal digits keep their input order (stability is
// the whole correctness contract).
#pragma once
#include "common.cuh"

namespace ley {

// Lanes of the warp holding the same 8-bit digit (and valid): 8 ballots, one per digit bit (warp
// multi-split), cheaper than match.any on sm_100a.
__device__ __forceinline__ uint32_t warp_peers8(uint32_t d, bool valid) {
#ifdef LEY_RANK_MATCH
  return __match_any_sync(0xffffffffu, valid ? d : (0x100u | (threadIdx.x & 31)));
#endif
  uint32_t peers = __ballot_sync(0xffffffffu, valid);
  if (!valid) peers = ~peers;
#pragma unroll
  for (int bit = 0; bit < 8; ++bit) {
    const bool set = (d >> bit) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, set);
    peers &= set ? bal : ~bal;
  }
  return peers;
}

// Unstable block-wide ranking by one 8-bit digit: a shared-memory atomic per item gives its position
// inside its digit group, a block scan of the 256 counts gives the group starts. The order inside a
// group is whatever the atomics produce — the sort's result does not depend on it, because every later
// comparison is on the composite (key, ordinal). s_hist: [256] u32; s_tmp: [32] u32.
// ZEROED = true: the caller zeroed s_hist before its last barrier (saves one barrier).
template <int THREADS, int ITEMS, bool ZEROED = false>
__device__ __forceinline__ void block_rank_atomic(const uint32_t (&dig)[ITEMS], uint32_t count, uint32_t (&pos)[ITEMS],
                                                  uint32_t* s_hist, uint32_t* s_tmp, uint32_t& total_d,
                                                  uint32_t& excl_d) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!ZEROED) {
    for (int i = threadIdx.x; i < kRadix; i += THREADS) s_hist[i] = 0;
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
    if (e < count) pos[j] = atomicAdd(&s_hist[dig[j]], 1u);
  }
  __syncthreads();
  const uint32_t total = threadIdx.x < kRadix ? s_hist[threadIdx.x] : 0u;
  const uint32_t excl = block_excl_scan<THREADS, false>(total, s_tmp, nullptr);  // (barrier below)
  if (threadIdx.x < kRadix) s_hist[threadIdx.x] = excl;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
    if (e < count) pos[j] += s_hist[dig[j]];
  }
  total_d = total;
  excl_d = excl;
}

// s_wh: [THREADS/32][256] u32 scratch; s_tmp: [32] u32.
// Output: pos[j] = position of item j in the block's digit-sorted order; for threads < 256,
// total_d / excl_d = count of digit d = threadIdx.x in the block and its exclusive offset.
template <int THREADS, int ITEMS>
__device__ __forceinline__ void block_rank_digits(const uint32_t (&dig)[ITEMS], uint32_t count, uint32_t (&pos)[ITEMS],
                                                  uint32_t* s_wh, uint32_t* s_tmp, uint32_t& total_d,
                                                  uint32_t& excl_d) {
  constexpr int WARPS = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < WARPS * kRadix; i += THREADS) s_wh[i] = 0;
  __syncthreads();
  uint32_t* wh = s_wh + warp * kRadix;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
    bool valid = e < count;
    uint32_t d = dig[j];
    uint32_t peers = warp_peers8(d, valid);
    uint32_t before = __popc(peers & lt);
    uint32_t cur = valid ? wh[d] : 0;
    __syncwarp();
    if (valid && before == 0) wh[d] = cur + __popc(peers);
    __syncwarp();
    pos[j] = cur + before;
  }
  __syncthreads();
  uint32_t total = 0;
  if (threadIdx.x < kRadix) {
    const int d = threadIdx.x;
#pragma unroll 4
    for (int w = 0; w < WARPS; ++w) {
      uint32_t v = s_wh[w * kRadix + d];
      s_wh[w * kRadix + d] = total;
      total += v;
    }
  }
  uint32_t excl = block_excl_scan<THREADS>(threadIdx.x < kRadix ? total : 0, s_tmp, nullptr);
  if (threadIdx.x < kRadix) {
    const int d = threadIdx.x;
#pragma unroll 4
    for (int w = 0; w < WARPS; ++w) s_wh[w * kRadix + d] += excl;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
    if (e < count) pos[j] += wh[dig[j]];
  }
  total_d = total;
  excl_d = excl;
}

// Decoupled look-back for digit d of chunk k whose segment starts at chunk k0, in two halves so the
// CTA can do useful work between them: publish the chunk's aggregate as soon as it is known, then
// later walk back to an inclusive prefix and publish it. Returns the exclusive prefix.
__device__ __forceinline__ void lookback_publish(uint64_t* status, uint64_t k, uint64_t k0, int d, uint32_t agg) {
  st_relaxed_u64(&status[k * kRadix + d], (k == k0 ? kFlagPrefix : kFlagAggregate) | agg);
}
__device__ __forceinline__ uint32_t lookback_wait(uint64_t* status, uint64_t k, uint64_t k0, int d, uint32_t agg) {
  if (k == k0) return 0;
  uint32_t excl = 0;
  uint64_t j = k - 1;
  while (true) {
    uint64_t s = ld_relaxed_u64(&status[j * kRadix + d]);
    uint32_t f = status_flag(s);
    if (f == 0) continue;
    excl += (uint32_t)s;
    if (f == 2) break;
    --j;
  }
  st_relaxed_u64(&status[k * kRadix + d], kFlagPrefix | (uint64_t)(excl + agg));
  return excl;
}
__device__ __forceinline__ uint32_t lookback_digit(uint64_t* status, uint64_t k, uint64_t k0, int d, uint32_t agg) {
  lookback_publish(status, k, k0, d, agg);
  return lookback_wait(status, k, k0, d, agg);
}

}  // namespace ley
