// kc_chunk.cuh — one level-1 K-c chunk as a device function any CTA (or a named-
// barrier thread group inside a CTA) can run, so the split can be fused into the K-d+K-e kernels.
//
// PAPER.md §3.1 line 96 (the scatter of the keys into their bucket offsets, "this scattering process takes
// the most time in radix sort"). Level-1 K-c (k_split.cu kc_split_level1) runs as its own persistent
// kernel; here the same chunk — gather the chunk's pairs from the tiles' byte-0 runs, rank by key byte 1,
// claim each digit's slice of its 16-bit bucket with one global atomic, stage in shared memory, write
// the runs — is a function, and after its stores the chunk is published in done[b], the count of
// finished chunks of byte-0 bucket b. A K-d+K-e kernel that owns the split (the fused form, internal.cu)
// sorts a 16-bit bucket of byte-0 bucket b once done[b] equals b's chunk count, and runs chunks itself
// while it waits: the split then executes in the sort's idle issue slots and spare DRAM bandwidth (the
// random record gather of K-e is bound by DRAM accesses, not bytes: profiles/r02_fetch_granularity.txt).
//
// Sync: the barrier of the participating threads (threadIdx.x in [0, THREADS)): __syncthreads() for a
// whole CTA, a named barrier for the sort group of the warp-specialised tier.
#pragma once
#include "block_rank.cuh"
#include "common.cuh"

namespace ley {

struct SyncCta {
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};
template <int ID, int N>
struct SyncGroup {
  __device__ __forceinline__ static void sync() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory"); }
};

// Everything a level-1 chunk needs (device pointers; see launch_kc_split_level1 for their meaning).
struct KcArgs {
  const uint64_t* k1_in;
  const uint32_t* w_in;
  uint32_t tiles;
  const uint32_t* off;      // [256 * tiles + 1] byte-0-major tile run starts (K-b)
  const uint32_t* lo;       // [tiles * 256] tile-local run offsets (K-a)
  const uint32_t* cstart;   // [257] first chunk of every byte-0 bucket
  const uint4* plan_a;      // per chunk: (b, v0, cnt, first chunk of b)
  const uint2* plan_b;      // per chunk: (t0, t1)
  const uint32_t* order;    // processing order of the chunks (null: identity)
  uint32_t* cursor;         // [65536] fill cursors of the 16-bit buckets (= B16 before the split)
  uint32_t* ticket;         // chunk ticket
  uint32_t* done;           // [256] finished chunks per byte-0 bucket
  uint32_t* kd_ticket;      // fused K-d: next 16-bit bucket to claim
  uint64_t* tail_out;
  uint32_t* idx_out;
  const uint32_t* hist16;   // [65536] level-1 bucket sizes (fused K-d: the items)
  const uint32_t* B16;      // [65536] level-1 bucket starts
};

constexpr uint32_t kKcRegion = kChunk * 13 + 16;                 // run table / staging (tail u64, idx u32, digit u8)
constexpr uint32_t kKcMaxRuns = kKcRegion / 8;
constexpr size_t kKcSmem = kKcRegion + 256 * 4 + 256 * 4 + 64 * 4;  // + s_hist, s_dst, s_misc

template <int THREADS, class Sync>
__device__ __forceinline__ uint32_t kc_excl_scan(uint32_t v, uint32_t* tmp) {
  constexpr int WARPS = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  Sync::sync();
  if (warp == 0) {
    uint32_t w = lane < WARPS ? tmp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < WARPS) tmp[lane] = w;
  }
  Sync::sync();
  return (warp ? tmp[warp - 1] : 0u) + x - v;  // (callers barrier before tmp is reused)
}

template <int THREADS, class Sync>
__device__ __forceinline__ uint32_t kc_excl_max(uint32_t v, uint32_t* tmp) {
  constexpr int WARPS = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x = max(x, y);
  }
  if (lane == 31) tmp[warp] = x;
  Sync::sync();
  if (warp == 0) {
    uint32_t w = lane < WARPS ? tmp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w = max(w, y);
    }
    if (lane < WARPS) tmp[lane] = w;
  }
  Sync::sync();
  const uint32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
  uint32_t r = lane ? prev : 0u;
  if (warp) r = max(r, tmp[warp - 1]);
  return r;
}

// Chunk k (a ticket value) of level 1 by THREADS threads (ITEMS * THREADS >= kChunk), shared memory `sm`
// (kKcSmem bytes, 16-byte aligned). On return the chunk's pairs are written and published in done[b].
template <int THREADS, int ITEMS, class Sync>
__device__ void kc_chunk(const KcArgs& a, uint32_t k, uint8_t* sm) {
  static_assert(THREADS * ITEMS >= (int)kChunk && THREADS >= kRadix, "chunk geometry");
  constexpr int PER = (kChunk + THREADS - 1) / THREADS;  // consecutive run marks per thread
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // load phase: run starts s_off [0, R), run-start marks (2 B per element) from a quarter of the region,
  // source bases s_lo from its half (R <= kKcMaxRuns / 2 keeps the three apart)
  uint32_t* s_off = reinterpret_cast<uint32_t*>(sm);
  uint16_t* s_mark = reinterpret_cast<uint16_t*>(s_off + kKcMaxRuns / 2);
  uint32_t* s_lo = s_off + kKcMaxRuns;
  uint64_t* s_tail = reinterpret_cast<uint64_t*>(sm);  // staging (scatter phase)
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_tail + kChunk);
  uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_idx + kChunk);
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(sm + kKcRegion);
  uint32_t* s_dst = s_hist + 256;
  uint32_t* s_misc = s_dst + 256;

  const uint32_t kk = a.order ? a.order[k] : k;
  const uint4 pa = a.plan_a[kk];
  const uint2 pb = a.plan_b[kk];
  const uint32_t b = pa.x, v0 = pa.y, cnt = pa.z, t0 = pb.x, t1 = pb.y;
  const uint32_t R = t1 - t0 + 1;
  const uint32_t* off_b = a.off + (uint64_t)b * a.tiles;
  const bool table = R <= kKcMaxRuns / 2;
  for (int q = threadIdx.x; q < kRadix; q += THREADS) s_hist[q] = 0;
  uint32_t src[ITEMS];
  if (table) {
    for (uint32_t e = threadIdx.x; e < cnt; e += THREADS) s_mark[e] = 0;
    for (uint32_t i = threadIdx.x; i < R; i += THREADS) {
      const uint32_t vs = off_b[t0 + i];
      s_off[i] = vs;
      s_lo[i] = ((t0 + i) << kTileLog2) + a.lo[(uint64_t)(t0 + i) * kRadix + b] - vs;
    }
    Sync::sync();
    for (uint32_t i = threadIdx.x; i < R; i += THREADS) {
      const uint32_t vs = s_off[i], ve = (i + 1 < R) ? s_off[i + 1] : off_b[t1 + 1];
      const uint32_t e = vs > v0 ? vs - v0 : 0u;
      if (ve > vs && e < cnt) s_mark[e] = (uint16_t)i;
    }
    Sync::sync();
    {
      const uint32_t e0 = threadIdx.x * PER;
      uint32_t m[PER], run = 0;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        m[q] = e0 + q < cnt ? s_mark[e0 + q] : 0u;
        run = max(run, m[q]);
        m[q] = run;
      }
      const uint32_t pre = kc_excl_max<THREADS, Sync>(run, s_misc);
#pragma unroll
      for (int q = 0; q < PER; ++q)
        if (e0 + q < cnt) s_mark[e0 + q] = (uint16_t)max(pre, m[q]);
    }
    Sync::sync();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
      src[j] = e < cnt ? s_lo[s_mark[e]] + v0 + e : 0u;
    }
  } else {  // very sparse bucket: search the global run table directly
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
      const uint32_t v = v0 + e;
      src[j] = 0;
      if (e < cnt) {
        uint64_t lo_t = t0, hi_t = (uint64_t)t1 + 1;
        while (hi_t - lo_t > 1) {
          const uint64_t mid = (lo_t + hi_t) >> 1;
          if (off_b[mid] <= v) lo_t = mid; else hi_t = mid;
        }
        const uint32_t t = (uint32_t)lo_t;
        src[j] = (t << kTileLog2) + a.lo[(uint64_t)t * kRadix + b] + (v - off_b[t]);
      }
    }
  }
  uint64_t k1[ITEMS];
  uint32_t w[ITEMS], dig[ITEMS], pos[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
    k1[j] = e < cnt ? a.k1_in[src[j]] : 0ull;
    w[j] = e < cnt ? a.w_in[src[j]] : 0u;
    dig[j] = (uint32_t)(k1[j] >> 56);
  }
  Sync::sync();  // run table dead; s_hist zeroed
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
    if (e < cnt) pos[j] = atomicAdd(&s_hist[dig[j]], 1u);
  }
  Sync::sync();
  const uint32_t total_d = threadIdx.x < kRadix ? s_hist[threadIdx.x] : 0u;
  const uint32_t excl_d = kc_excl_scan<THREADS, Sync>(total_d, s_misc);
  if (threadIdx.x < kRadix) {
    s_hist[threadIdx.x] = excl_d;
    const uint32_t base = total_d ? atomicAdd(&a.cursor[b * 256 + threadIdx.x], total_d) : 0u;
    s_dst[threadIdx.x] = base - excl_d;
  }
  Sync::sync();
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t e = warp * (32 * ITEMS) + j * 32 + lane;
    if (e < cnt) {
      const uint32_t p = pos[j] + s_hist[dig[j]];
      s_tail[p] = (k1[j] << 8) | (w[j] >> 24);
      s_idx[p] = (src[j] & ~(kTileRecords - 1)) | (w[j] & 0xFFFFFFu);
      s_dig[p] = (uint8_t)dig[j];
    }
  }
  Sync::sync();
  for (uint32_t i = threadIdx.x; i < cnt; i += THREADS) {
    const uint32_t g = s_dst[s_dig[i]] + i;
    a.tail_out[g] = s_tail[i];
    a.idx_out[g] = s_idx[i];
  }
  Sync::sync();  // every store of the chunk issued (and the staging free for the caller)
  if (threadIdx.x == 0) {
    __threadfence();  // cumulative over the group's stores ordered by the barrier above
    atomicAdd(&a.done[b], 1u);
  }
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Fused K-d driver step, by thread 0 of the group: the next 16-bit bucket of tier `tier` in ascending
// order (65536 = none left).
template <class TierOf>
__device__ __forceinline__ uint32_t kc_claim_bucket(const KcArgs& a, TierOf tier_match) {
  while (true) {
    const uint32_t p = atomicAdd(a.kd_ticket, 1u);
    if (p >= 65536u) return 65536u;
    const uint32_t len = a.hist16[p];
    if (len && tier_match(len)) return p;
  }
}

}  // namespace ley
