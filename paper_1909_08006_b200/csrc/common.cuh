// common.cuh — shared device helpers and data-structure definitions of the sm_100a sort path.
// Product code: shares nothing with oracle/ (SURVEY.md §8c).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "config.h"

namespace ley {

// A bucket still to be sorted: [start, start+len) of the pair buffer `parity` (0 = A, 1 = B),
// key bytes [0, depth) already equal across the bucket (consumed by MSD splits).
struct Seg {
  uint32_t start;
  uint32_t len;
  uint32_t depth;
  uint32_t parity;
};

// Work lists produced by classification (device-built; Alg. 1 smallBucketQueue).
enum ListId : int {
  kListWarp = 0,   // len <= warp_tier_max: one warp, register bitonic network
  kListMed1 = 1,   // len <= 512:   one CTA (128 threads), shared memory
  kListMed2 = 2,   // len <= 2048   (256 threads)
  kListMed3 = 3,   // len <= 8192   (512 threads)
  kListMed4 = 4,   // len <= 10240  (1024 threads, 1 CTA/SM; the C4 bucket size)
  kListMed5 = 5,   // len <= 16384  (512 threads, bucket re-read from L2)
  kNumKdLists = 6
};
static_assert(kNumKdLists == kNumKdListsHost, "host planning mirrors the K-d list count");

struct ListSet {
  Seg* items[kNumKdLists];
  uint32_t* counts;  // [kNumKdLists] device counters; counts[kTierTicket + l]: list l's claim ticket
  uint32_t cap;      // capacity of each list
};
constexpr int kTierTicket = 8;  // (counts and tickets are zeroed together: 2 * kTierTicket words)
static_assert(kNumKdLists <= kTierTicket, "tickets follow the counts");

// Runtime tunables (ley_set_option); copied by value into kernels that need them.
struct Tunables {
  uint32_t warp_tier_max = kWarpTierMax;
  uint32_t smem_tier_max = kSmemTierMax;
  int kd_digit_bits = kKdMaxBits;
  int kd_insert_max = 16;
  int kd_ws = 1;  // warp-specialised sort/gather tiers (kd_ws_sort) instead of the alternating kd_cta_sort
  int ws_tma = 0;  // kd_ws_sort: record windows by TMA tensor copies (64-B L2 fetches) or plain bulk copies
  int gather_l2_64 = 1;  // kd_cta_sort gathers: cp.async with .L2::64B (1) or without the hint (0)
  int kd_claim = 1;      // tier CTAs claim buckets by atomic ticket (1) or stride the list statically (0)
  int kc_corun = 0;      // the fused tier runs beside the level-1 K-c kernel (PDL, no entry wait; internal.cu)
  int pdl = 0;           // K-d/K-e tier kernels launched with programmatic dependent launch (launch_k): 0
                         // plain stream order; 1 every tier waits, then lets the next launch; 2 the first
                         // tier waits, later ones launch at once and wait only before exiting (overlap)
};

// Programmatic dependent launch (PDL): a kernel launched with the programmatic-serialization attribute
// may become resident while its predecessor in the stream still runs; it lets its own successor launch
// at once (pdl_trigger) and waits for the predecessor's completion and memory (pdl_wait) before touching
// anything the predecessor wrote. Without the attribute both are no-ops. The launch latency and empty
// grids of a chain of tier kernels then overlap the running one.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Kernel entry of a tier kernel under Tunables::pdl mode m; the returned guard waits at every exit in mode
// 2, so a tier never completes before its predecessor (stream order of completions is kept).
struct PdlExitWait {
  bool on;
  __device__ __forceinline__ ~PdlExitWait() {
    if (on) pdl_wait();
  }
};
__device__ __forceinline__ PdlExitWait pdl_enter(int m) {
  if (m != 2) pdl_wait();
  pdl_trigger();
  return PdlExitWait{m == 2};
}

// ------------------------------------------------------------------ device helpers
// Bulk L2 prefetch of [p, p + bytes) (widened to 16-byte bounds) with an evict-last policy: a K-d tier CTA
// fetches its next bucket's pairs while it gathers the current one, so the pair loads that start the next
// sort hit L2 instead of waiting on DRAM behind the gather traffic (C4 K-d+K-e 33.3 -> 32.7 ms).
__device__ __forceinline__ void prefetch_l2_last(const void* p, uint64_t bytes) {
  const uint64_t a = reinterpret_cast<uint64_t>(p) & ~uint64_t(15);
  const uint64_t e = (reinterpret_cast<uint64_t>(p) + bytes + 15) & ~uint64_t(15);
  if (e <= a) return;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a), "r"((uint32_t)(e - a)), "l"(pol)
               : "memory");
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ldg_nc_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void stg_cs_v4(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Decoupled look-back status word: [33:32] flag, [31:0] value.
constexpr uint64_t kFlagAggregate = 1ull << 32;
constexpr uint64_t kFlagPrefix = 2ull << 32;
__device__ __forceinline__ uint32_t status_flag(uint64_t s) { return (uint32_t)(s >> 32); }

// Block-wide exclusive scan of one u32 per thread (THREADS <= 1024). `tmp` holds >= 32 words.
// SYNC_AFTER = false: the caller guarantees a barrier before `tmp` is written again (saves one barrier).
template <int THREADS, bool SYNC_AFTER = true>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* tmp, uint32_t* total) {
  constexpr int WARPS = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < WARPS ? tmp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < WARPS) tmp[lane] = w;  // inclusive per-warp totals
  }
  __syncthreads();
  uint32_t warp_excl = warp ? tmp[warp - 1] : 0;
  if (total) *total = tmp[WARPS - 1];
  uint32_t r = warp_excl + x - v;
  if (SYNC_AFTER) __syncthreads();  // tmp reusable after return
  return r;
}

// Block-wide exclusive max-scan of one u32 per thread (identity 0). `tmp` holds >= 32 words.
template <int THREADS, bool SYNC_AFTER = true>
__device__ __forceinline__ uint32_t block_excl_max(uint32_t v, uint32_t* tmp) {
  constexpr int WARPS = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x = max(x, y);
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < WARPS ? tmp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w = max(w, y);
    }
    if (lane < WARPS) tmp[lane] = w;  // inclusive per-warp maxima
  }
  __syncthreads();
  uint32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
  uint32_t r = lane ? prev : 0u;
  if (warp) r = max(r, tmp[warp - 1]);
  if (SYNC_AFTER) __syncthreads();
  return r;
}

// Composite (key-tail, ordinal) order: the strict total order of the sort.
__device__ __forceinline__ bool pair_less(uint64_t ta, uint32_t ia, uint64_t tb, uint32_t ib) {
  return ta < tb || (ta == tb && ia < ib);
}

}  // namespace ley
