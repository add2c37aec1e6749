// k_tile.cu — K-a: key-prefix extraction + per-CTA byte-0 histogram + tile-local stable sort by byte 0.
//
// PAPER.md §3.1 Algorithm 1 line 59 "buckets[256][k] = ParallelRadixSort(key, radix, n)" with
// radix = 0, and the cache-aware scatter of line 96 ("we first compute a histogram based on the current
// radix ... aggregate the keys in the thread level CPU cache first, before scattering them"): here the
// "thread-level cache" is the CTA's shared memory. §3.2: "Leyenda extracts the (key, pointer)
// tuples from records during the read process" — K-a is that extraction. SURVEY.md §8a row a1.
//
// One CTA per tile of kTileRecords records:
//   1. load key bytes 0..9 of each record (three 4-byte loads; record i sits at byte 100 i, 4-aligned)
//   2. warp multi-split rank on byte 0 (8 ballots + popc of lanemask_lt; measured cheaper here than
//      shared-memory atomics, which win in K-c)
//   3. block scan of the 256 x WARPS counts -> tile-local offsets
//   4. scatter pairs into shared memory in byte-0 order, write them out coalesced:
//        k1 = key bytes 1..8 big-endian (u64)     w = key byte 9 << 24 | local index (u32)
//   5. cnt[b * tiles + t] = tile count of byte-0 value b (bucket-major, for K-b's scan)
//      lo[t * 256 + b]    = tile-local exclusive offset of b
//   6. hist16[key bytes 0..1] += 1 (warp-aggregated global reductions) — the level-1 bucket sizes
#include "block_rank.cuh"
#include "common.cuh"
#include "kernels.cuh"
#include "runtime.h"

namespace ley {
namespace {

__device__ __forceinline__ uint32_t ld_ef_u32(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// Flexible keys (§5). K-a sorts on a 10-byte key window at record byte
// key.off (a multiple of 10: words key.off/4 .. +2, shifted by 16 bits when key.off % 4 == 2); a key of
// more than 10 bytes is sorted LSD over its windows, last window first (internal.cu). A window of
// key.len < 10 bytes (a short key, or the last window of a long one) has its bytes [len, 10) replaced by
// the big-endian ordinal (its top bytes if fewer than 4 remain): (composite, ordinal) order is then
// (key, ordinal) order, and equal keys stop recursing as soon as the ordinal bytes are reached.
__device__ __forceinline__ void ka_window(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t w2, uint32_t sh) {
  // in: a, b, w2 = words key.off/4 .. +2; out: a, b = window bytes 0..7, c = window bytes 8..9 (low 16)
  if (sh) {
    a = __funnelshift_r(a, b, sh);
    b = __funnelshift_r(b, w2, sh);
    c = w2 >> sh;
  } else {
    c = w2;
  }
}

__device__ __forceinline__ void ka_compose(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t len, uint32_t ord) {
  unsigned __int128 K = ((unsigned __int128)bswap32(a) << 48) | ((unsigned __int128)bswap32(b) << 16) |
                        (((c & 0xFFu) << 8) | ((c >> 8) & 0xFFu));
  const uint32_t free_bits = 8u * (10u - len);  // 8 .. 72
  K = (K >> free_bits) << free_bits;
  K |= free_bits >= 32 ? ((unsigned __int128)ord << (free_bits - 32)) : (unsigned __int128)(ord >> (32 - free_bits));
  a = bswap32((uint32_t)(K >> 48));
  b = bswap32((uint32_t)(K >> 16));
  c = (c & 0xFFFF0000u) | (((uint32_t)K >> 8) & 0xFFu) | (((uint32_t)K & 0xFFu) << 8);
}

template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS, 2) ka_tile_sort(const uint8_t* __restrict__ in, uint64_t n, uint32_t tiles,
                                                         uint64_t* __restrict__ k1_out, uint32_t* __restrict__ w_out,
                                                         uint32_t* __restrict__ cnt, uint32_t* __restrict__ lo,
                                                         uint32_t* __restrict__ hist16, uint32_t copies, KeySpec key) {
  constexpr int T = THREADS * ITEMS;
  constexpr int WARPS = THREADS / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* s_k1 = reinterpret_cast<uint64_t*>(smem);                   // [T]
  uint32_t* s_w = reinterpret_cast<uint32_t*>(s_k1 + T);                // [T]
  uint32_t* s_wh = s_w + T;                                             // [WARPS][256]
  uint32_t* s_tmp = s_wh + WARPS * kRadix;                              // [32]

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t t = blockIdx.x;
  const uint64_t base = (uint64_t)t * T;
  const uint32_t cnt_t = (uint32_t)(n - base < (uint64_t)T ? n - base : (uint64_t)T);

  for (int i = threadIdx.x; i < WARPS * kRadix; i += THREADS) s_wh[i] = 0;
  uint32_t* hist_copy = hist16 + (size_t)(blockIdx.x % copies) * 65536;

  // L2 policies: the record lines are read once (evict first — measured: without it ~25% of them are
  // fetched twice, 128 vs 103 B/record of DRAM reads at C2); the hist16 copies are hot (evict last).
  uint64_t pol_ef, pol_el;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ef));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_el));
  // ---- 1. load keys (all loads issued before use)
  uint32_t a[ITEMS], b[ITEMS], c[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    uint32_t r = warp * (32 * ITEMS) + j * 32 + lane;
    if (r < cnt_t) {
      const uint32_t* p = reinterpret_cast<const uint32_t*>(in + (base + r) * kRecordBytes) + key.off / 4;
      a[j] = ld_ef_u32(p, pol_ef);
      b[j] = ld_ef_u32(p + 1, pol_ef);
      c[j] = ld_ef_u32(p + 2, pol_ef);
    } else {
      a[j] = b[j] = c[j] = 0;
    }
  }
  if (key.off | (key.len - 10u)) {  // (uniform) a key window other than the paper's bytes 0..9
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      ka_window(a[j], b[j], c[j], c[j], (key.off & 3u) * 8u);
      if (key.len < 10) ka_compose(a[j], b[j], c[j], key.len, (uint32_t)(base + warp * (32 * ITEMS) + j * 32 + lane));
    }
  }
  __syncthreads();

  // ---- 2. warp multi-split ranking on byte 0, in record order (stable)
  uint32_t rank[ITEMS];
  uint32_t* wh = s_wh + warp * kRadix;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    uint32_t r = warp * (32 * ITEMS) + j * 32 + lane;
    bool valid = r < cnt_t;
    uint32_t hi = bswap32(a[j]);            // key bytes 0..3, big-endian
    uint32_t d = hi >> 24;                  // byte 0
    uint32_t peers = warp_peers8(d, valid);
    uint32_t before = __popc(peers & lt);
    uint32_t cur = valid ? wh[d] : 0;
    __syncwarp();
    if (valid && before == 0) wh[d] = cur + __popc(peers);
    __syncwarp();
    rank[j] = cur + before;
    // level-1 bucket sizes: 16-bit prefix (bytes 0..1)
    uint32_t p16 = hi >> 16;
    uint32_t peers16 = peers & warp_peers8((hi >> 16) & 0xFFu, valid);
    if (valid && __popc(peers16 & lt) == 0)
      asm volatile("red.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(&hist_copy[p16]),
                   "r"((uint32_t)__popc(peers16)), "l"(pol_el) : "memory");
  }
  __syncthreads();

  // ---- 3. per-digit totals over warps, tile exclusive offsets
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
    cnt[(uint64_t)d * tiles + t] = total;
    lo[(uint64_t)t * kRadix + d] = excl;
  }
  __syncthreads();

  // ---- 4. scatter into shared memory in byte-0 order
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    uint32_t r = warp * (32 * ITEMS) + j * 32 + lane;
    if (r < cnt_t) {
      uint32_t hi = bswap32(a[j]);
      uint32_t d = hi >> 24;
      uint32_t pos = wh[d] + rank[j];
      uint64_t kk = ((uint64_t)hi << 32) | bswap32(b[j]);  // key bytes 0..7 big-endian
      s_k1[pos] = (kk << 8) | (c[j] & 0xFFu);               // bytes 1..8
      s_w[pos] = ((c[j] >> 8) & 0xFFu) << 24 | r;           // byte 9 | local index
    }
  }
  __syncthreads();

  // ---- 5. coalesced write-out
  for (uint32_t i = threadIdx.x; i < cnt_t; i += THREADS) {
    k1_out[base + i] = s_k1[i];
    w_out[base + i] = s_w[i];
  }
}

// ---------------------------------------------------------------------------- streaming K-a
// Same per-tile work as ka_tile_sort, restructured so the SM's record reads never wait for its compute:
// one persistent CTA per SM streams its tiles' records through a 3-slot shared-memory ring of 512-record
// pieces (51.2 KB each) with TMA bulk copies (cp.async.bulk + mbarrier); the key words of piece j of a
// tile land in item j of every thread (record r = j * 512 + tid), so while a tile is ranked, scattered
// and written, the first pieces of the next tile are already arriving.
constexpr int kPiece = kTileThreads;                        // records per piece (one per thread)
constexpr int kPieces = kTileRecords / kPiece;              // pieces per tile (= kTileItems)
constexpr int kRing = 3;
constexpr uint32_t kPieceBytes = kPiece * kRecordBytes;     // 51200
static_assert(kPieces == kTileItems, "one piece per item");

__device__ __forceinline__ void ka_mbar_init(uint32_t a, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void ka_mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ka_mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}"
               ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void ka_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar), "l"(pol) : "memory");
}

template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS, 1)
    ka_tile_stream(const uint8_t* __restrict__ in, uint64_t n, uint32_t tiles, uint64_t* __restrict__ k1_out,
                   uint32_t* __restrict__ w_out, uint32_t* __restrict__ cnt, uint32_t* __restrict__ lo,
                   uint32_t* __restrict__ hist16, uint32_t copies, uint32_t key_len) {
  constexpr int T = THREADS * ITEMS;
  constexpr int WARPS = THREADS / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* s_ring = smem;                                                        // [kRing][kPieceBytes]
  uint64_t* s_k1 = reinterpret_cast<uint64_t*>(smem + kRing * kPieceBytes);     // [T]
  uint32_t* s_w = reinterpret_cast<uint32_t*>(s_k1 + T);                        // [T]
  uint32_t* s_wh = s_w + T;                                                     // [WARPS][256]
  uint32_t* s_tmp = s_wh + WARPS * kRadix;                                      // [32]
  __shared__ __align__(8) uint64_t s_full[kRing];

  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t* hist_copy = hist16 + (size_t)(blockIdx.x % copies) * 65536;
  uint64_t pol_ef, pol_el;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ef));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_el));
  const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(&s_full[0]);
  const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(s_ring);
  if (tid < kRing) ka_mbar_init(full0 + 8 * tid, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  // global piece P of this CTA = (its tile i = P / kPieces, piece j = P % kPieces)
  const uint32_t my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t total_pieces = my_tiles * kPieces;
  auto issue = [&](uint32_t P) {  // thread 0 only
    const uint32_t t = blockIdx.x + (P / kPieces) * gridDim.x;
    const uint64_t r0 = (uint64_t)t * T + (uint64_t)(P % kPieces) * kPiece;
    const uint32_t slot = P % kRing;
    uint32_t bytes = 0;
    if (r0 < n) {
      const uint64_t c = n - r0 < (uint64_t)kPiece ? n - r0 : (uint64_t)kPiece;
      bytes = (uint32_t)((c * kRecordBytes) & ~uint64_t(15));  // keys of every record included (tail <= 12 B)
    }
    if (bytes) {
      ka_mbar_expect_tx(full0 + 8 * slot, bytes);
      ka_bulk_g2s(ring0 + slot * kPieceBytes, in + r0 * kRecordBytes, bytes, full0 + 8 * slot, pol_ef);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full0 + 8 * slot) : "memory");
    }
  };
  if (tid == 0)
    for (uint32_t P = 0; P < (uint32_t)kRing && P < total_pieces; ++P) issue(P);

  for (uint32_t i = 0; i < my_tiles; ++i) {
    const uint32_t t = blockIdx.x + i * gridDim.x;
    const uint64_t base = (uint64_t)t * T;
    const uint32_t cnt_t = (uint32_t)(n - base < (uint64_t)T ? n - base : (uint64_t)T);
    for (int q = tid; q < WARPS * kRadix; q += THREADS) s_wh[q] = 0;
    // ---- 1. keys of piece j -> item j (record r = j * THREADS + tid)
    uint32_t a[ITEMS], b[ITEMS], c[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t P = i * kPieces + j;
      const uint32_t slot = P % kRing;
      ka_mbar_wait(full0 + 8 * slot, (P / kRing) & 1u);
      const uint32_t r = j * THREADS + tid;
      if (r < cnt_t) {
        const uint32_t* kw = reinterpret_cast<const uint32_t*>(s_ring + slot * kPieceBytes + tid * kRecordBytes);
        a[j] = kw[0];
        b[j] = kw[1];
        c[j] = kw[2];
        if (key_len < 10) ka_compose(a[j], b[j], c[j], key_len, (uint32_t)(base + r));
      } else {
        a[j] = b[j] = c[j] = 0;
      }
      __syncthreads();  // every thread has its key words: the slot may be refilled
      if (tid == 0 && P + kRing < total_pieces) issue(P + kRing);
    }

    // ---- 2. warp multi-split ranking on byte 0
    uint32_t rank[ITEMS];
    uint32_t* wh = s_wh + warp * kRadix;
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t r = j * THREADS + tid;
      const bool valid = r < cnt_t;
      const uint32_t hi = bswap32(a[j]);
      const uint32_t d = hi >> 24;
      const uint32_t peers = warp_peers8(d, valid);
      const uint32_t before = __popc(peers & lt);
      const uint32_t cur = valid ? wh[d] : 0;
      __syncwarp();
      if (valid && before == 0) wh[d] = cur + __popc(peers);
      __syncwarp();
      rank[j] = cur + before;
      const uint32_t p16 = hi >> 16;
      const uint32_t peers16 = peers & warp_peers8((hi >> 16) & 0xFFu, valid);
      if (valid && __popc(peers16 & lt) == 0)
        asm volatile("red.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(&hist_copy[p16]),
                     "r"((uint32_t)__popc(peers16)), "l"(pol_el) : "memory");
    }
    __syncthreads();

    // ---- 3. per-digit totals over warps, tile exclusive offsets
    uint32_t total = 0;
    if (tid < kRadix) {
#pragma unroll 4
      for (int w = 0; w < WARPS; ++w) {
        const uint32_t v = s_wh[w * kRadix + tid];
        s_wh[w * kRadix + tid] = total;
        total += v;
      }
    }
    const uint32_t excl = block_excl_scan<THREADS>(tid < kRadix ? total : 0, s_tmp, nullptr);
    if (tid < kRadix) {
#pragma unroll 4
      for (int w = 0; w < WARPS; ++w) s_wh[w * kRadix + tid] += excl;
      cnt[(uint64_t)tid * tiles + t] = total;
      lo[(uint64_t)t * kRadix + tid] = excl;
    }
    __syncthreads();

    // ---- 4. scatter into shared memory in byte-0 order
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t r = j * THREADS + tid;
      if (r < cnt_t) {
        const uint32_t hi = bswap32(a[j]);
        const uint32_t d = hi >> 24;
        const uint32_t pos = wh[d] + rank[j];
        const uint64_t kk = ((uint64_t)hi << 32) | bswap32(b[j]);
        s_k1[pos] = (kk << 8) | (c[j] & 0xFFu);
        s_w[pos] = ((c[j] >> 8) & 0xFFu) << 24 | r;
      }
    }
    __syncthreads();

    // ---- 5. coalesced write-out
    for (uint32_t q = tid; q < cnt_t; q += THREADS) {
      k1_out[base + q] = s_k1[q];
      w_out[base + q] = s_w[q];
    }
    __syncthreads();  // staging and per-warp counters reused by the next tile
  }
}

// ---------------------------------------------------------------------------- key-row K-a (form 1)
// The streaming structure above, but the ring carries only the key rows, not whole records. A miss of
// the whole-record bulk copies (or of any plain load) fetches full 128-B lines: 100 B/record of DRAM
// reads for a 10-byte key. Here each 512-record piece arrives as four TMA tensor boxes over the record
// array viewed as [groups of 4][25 rows][16 B] (tmap.cu): rows {0}, {6}, {12,13}, {18,19} of 128
// consecutive groups hold the key bytes 0..11 of records 4g, 4g+1, 4g+2, 4g+3 at byte 0, 4, 8, 12 of
// their first row; the map's 64-B L2 promotion fetches 72 B/record (measured) into a 12 KB slot, so a
// deeper ring fits. The last n mod 4 records (outside the map) are read with plain loads.
constexpr int kKeyGroups = kPiece / 4;                   // 128 groups per piece
constexpr uint32_t kKeySlotBytes = kKeyGroups * 16 * 6;  // rows 0, 6 (16 B each), 12-13, 18-19 (32 B each)
static_assert(kPiece % 4 == 0, "pieces are whole 4-record groups");
int ka_ring_slots() { return (int)options_snapshot().ka_ring; }

__device__ __forceinline__ void ka_tma3(uint32_t dst, const CUtensorMap* m, int row, int grp, uint32_t mbar,
                                        uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(dst), "l"((uint64_t)m), "r"(0), "r"(row), "r"(grp), "r"(mbar), "l"(pol) : "memory");
}

// consumer-group barrier (named barrier 1: the THREADS consumer threads, not the producer warp)
template <int THREADS>
__device__ __forceinline__ void ka_csync() { asm volatile("bar.sync 1, %0;" ::"n"(THREADS) : "memory"); }

template <int THREADS>
__device__ __forceinline__ uint32_t ka_cscan(uint32_t v, uint32_t* tmp) {  // exclusive, consumers only
  constexpr int WARPS = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  ka_csync<THREADS>();
  if (warp == 0) {
    uint32_t w = lane < WARPS ? tmp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < WARPS) tmp[lane] = w;
  }
  ka_csync<THREADS>();
  const uint32_t r = (warp ? tmp[warp - 1] : 0u) + x - v;
  ka_csync<THREADS>();
  return r;
}

// THREADS consumer threads (one record of every piece each) + one producer warp that keeps the ring full:
// it refills a slot as soon as every consumer warp has arrived on the slot's "empty" mbarrier, so the
// consumers never stop at a block-wide barrier for the ring (only for the tile's rank/scan/scatter steps).
template <int THREADS, int ITEMS, int RING>
__global__ void __launch_bounds__(THREADS + 32, 1)
    ka_tile_keys(const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m2,
                 const uint8_t* __restrict__ in, uint64_t n, uint32_t tiles, uint64_t* __restrict__ k1_out,
                 uint32_t* __restrict__ w_out, uint32_t* __restrict__ cnt, uint32_t* __restrict__ lo,
                 uint32_t* __restrict__ hist16, uint32_t copies, uint32_t key_len) {
  constexpr int T = THREADS * ITEMS;
  constexpr int WARPS = THREADS / 32;
  static_assert(THREADS == kPiece, "one record of every piece per consumer thread");
  // (no static shared memory: the dynamic block starts the CTA's window, so the tensor-copy slots are
  // 128-byte aligned; the mbarriers live at its end)
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* s_ring = smem;                                                       // [RING][kKeySlotBytes]
  uint64_t* s_k1 = reinterpret_cast<uint64_t*>(smem + RING * kKeySlotBytes);    // [T]
  uint32_t* s_w = reinterpret_cast<uint32_t*>(s_k1 + T);                        // [T]
  uint32_t* s_wh = s_w + T;                                                     // [WARPS][256]
  uint32_t* s_tmp = s_wh + WARPS * kRadix;                                      // [32]
  uint64_t* s_full = reinterpret_cast<uint64_t*>(s_tmp + 32);                   // [RING]
  uint64_t* s_empty = s_full + RING;                                            // [RING]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(&s_full[0]);
  const uint32_t empty0 = (uint32_t)__cvta_generic_to_shared(&s_empty[0]);
  const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(s_ring);
  if (tid < RING) {
    ka_mbar_init(full0 + 8 * tid, 1);
    ka_mbar_init(empty0 + 8 * tid, WARPS);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  const uint64_t n4 = n & ~uint64_t(3);  // records inside the map
  const uint32_t my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t total_pieces = my_tiles * kPieces;

  if (tid >= THREADS) {
    // ================================================================ producer warp
    if (lane == 0) {
      uint64_t pol_ef;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ef));
      for (uint32_t P = 0; P < total_pieces; ++P) {
        const uint32_t slot = P % RING;
        if (P >= (uint32_t)RING) ka_mbar_wait(empty0 + 8 * slot, ((P / RING) - 1) & 1u);
        const uint32_t t = blockIdx.x + (P / kPieces) * gridDim.x;
        const uint64_t r0 = (uint64_t)t * T + (uint64_t)(P % kPieces) * kPiece;
        const uint32_t mb = full0 + 8 * slot;
        if (r0 < n4) {
          // boxes past the last group are zero-filled by the TMA and still count their full bytes
          const uint32_t dst = ring0 + slot * kKeySlotBytes;
          const int g0 = (int)(r0 >> 2);
          ka_mbar_expect_tx(mb, kKeySlotBytes);
          ka_tma3(dst, &m1, 0, g0, mb, pol_ef);
          ka_tma3(dst + kKeyGroups * 16, &m1, 6, g0, mb, pol_ef);
          ka_tma3(dst + kKeyGroups * 32, &m2, 12, g0, mb, pol_ef);
          ka_tma3(dst + kKeyGroups * 64, &m2, 18, g0, mb, pol_ef);
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
        }
      }
    }
    return;
  }

  // ================================================================ consumers
  uint32_t* hist_copy = hist16 + (size_t)(blockIdx.x % copies) * 65536;
  uint64_t pol_el;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_el));
  // where this thread's key words sit in a slot: record 4g + jj at byte 4 jj of its first row
  const uint32_t g = (uint32_t)tid >> 2, jj = (uint32_t)tid & 3u;
  const uint32_t key_off = jj == 0 ? g * 16 : jj == 1 ? kKeyGroups * 16 + g * 16 + 4
                         : jj == 2 ? kKeyGroups * 32 + g * 32 + 8 : kKeyGroups * 64 + g * 32 + 12;

  for (uint32_t i = 0; i < my_tiles; ++i) {
    const uint32_t t = blockIdx.x + i * gridDim.x;
    const uint64_t base = (uint64_t)t * T;
    const uint32_t cnt_t = (uint32_t)(n - base < (uint64_t)T ? n - base : (uint64_t)T);
    for (int q = tid; q < WARPS * kRadix; q += THREADS) s_wh[q] = 0;
    // ---- 1. keys of piece j -> item j (record r = j * THREADS + tid)
    uint32_t a[ITEMS], b[ITEMS], c[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t P = i * kPieces + j;
      const uint32_t slot = P % RING;
      ka_mbar_wait(full0 + 8 * slot, (P / RING) & 1u);
      const uint32_t r = j * THREADS + tid;
      if (r < cnt_t) {
        if (base + r < n4) {
          const uint32_t* kw = reinterpret_cast<const uint32_t*>(s_ring + slot * kKeySlotBytes + key_off);
          a[j] = kw[0];
          b[j] = kw[1];
          c[j] = kw[2];
        } else {  // one of the last n mod 4 records
          const uint32_t* kw = reinterpret_cast<const uint32_t*>(in + (base + r) * kRecordBytes);
          a[j] = kw[0];
          b[j] = kw[1];
          c[j] = kw[2];
        }
        if (key_len < 10) ka_compose(a[j], b[j], c[j], key_len, (uint32_t)(base + r));
      } else {
        a[j] = b[j] = c[j] = 0;
      }
      __syncwarp();
      if (lane == 0) {  // this warp is done with the slot (generic reads before the async-proxy refill)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * slot) : "memory");
      }
    }

    // ---- 2. warp multi-split ranking on byte 0
    uint32_t rank[ITEMS];
    uint32_t* wh = s_wh + warp * kRadix;
    const uint32_t lt = lanemask_lt();
    ka_csync<THREADS>();  // s_wh zeroed
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t r = j * THREADS + tid;
      const bool valid = r < cnt_t;
      const uint32_t hi = bswap32(a[j]);
      const uint32_t d = hi >> 24;
      const uint32_t peers = warp_peers8(d, valid);
      const uint32_t before = __popc(peers & lt);
      const uint32_t cur = valid ? wh[d] : 0;
      __syncwarp();
      if (valid && before == 0) wh[d] = cur + __popc(peers);
      __syncwarp();
      rank[j] = cur + before;
      const uint32_t p16 = hi >> 16;
      const uint32_t peers16 = peers & warp_peers8((hi >> 16) & 0xFFu, valid);
      if (valid && __popc(peers16 & lt) == 0)
        asm volatile("red.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(&hist_copy[p16]),
                     "r"((uint32_t)__popc(peers16)), "l"(pol_el) : "memory");
    }
    ka_csync<THREADS>();

    // ---- 3. per-digit totals over warps, tile exclusive offsets
    uint32_t total = 0;
    if (tid < kRadix) {
#pragma unroll 4
      for (int w = 0; w < WARPS; ++w) {
        const uint32_t v = s_wh[w * kRadix + tid];
        s_wh[w * kRadix + tid] = total;
        total += v;
      }
    }
    const uint32_t excl = ka_cscan<THREADS>(tid < kRadix ? total : 0, s_tmp);
    if (tid < kRadix) {
#pragma unroll 4
      for (int w = 0; w < WARPS; ++w) s_wh[w * kRadix + tid] += excl;
      cnt[(uint64_t)tid * tiles + t] = total;
      lo[(uint64_t)t * kRadix + tid] = excl;
    }
    ka_csync<THREADS>();

    // ---- 4. scatter into shared memory in byte-0 order
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t r = j * THREADS + tid;
      if (r < cnt_t) {
        const uint32_t hi = bswap32(a[j]);
        const uint32_t d = hi >> 24;
        const uint32_t pos = wh[d] + rank[j];
        const uint64_t kk = ((uint64_t)hi << 32) | bswap32(b[j]);
        s_k1[pos] = (kk << 8) | (c[j] & 0xFFu);
        s_w[pos] = ((c[j] >> 8) & 0xFFu) << 24 | r;
      }
    }
    ka_csync<THREADS>();

    // ---- 5. coalesced write-out
    for (uint32_t q = tid; q < cnt_t; q += THREADS) {
      k1_out[base + q] = s_k1[q];
      w_out[base + q] = s_w[q];
    }
    ka_csync<THREADS>();  // staging and per-warp counters reused by the next tile
  }
}

}  // namespace

size_t ka_smem_bytes() {
  return (size_t)kTileRecords * 12 + (size_t)(kTileThreads / 32) * kRadix * 4 + 32 * 4;
}

cudaError_t launch_ka_tile_sort(const uint8_t* in, uint64_t n, uint32_t tiles, uint64_t* k1_out, uint32_t* w_out,
                                uint32_t* cnt, uint32_t* lo, uint32_t* hist16, uint32_t copies, int form,
                                KeySpec key, cudaStream_t s) {
  auto kern = ka_tile_sort<kTileThreads, kTileItems>;
  size_t smem = ka_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (form != 0 && key.off == 0) {  // (the persistent forms read keys from record bytes 0..11 only)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t grid = tiles < (uint32_t)sms ? tiles : (uint32_t)sms;
    const size_t rest = (size_t)kTileRecords * 12 + (size_t)(kTileThreads / 32) * kRadix * 4 + 32 * 4;
    if (form == 1) {
      CUtensorMap m1, m2;  // boxes of 1 and 2 rows over kKeyGroups groups
      if ((e = record_group_map(&m1, in, n, 1, kKeyGroups)) != cudaSuccess) return e;
      if ((e = record_group_map(&m2, in, n, 2, kKeyGroups)) != cudaSuccess) return e;
      const int ring = ka_ring_slots();
      auto launch = [&](auto kk, int slots) {
        const size_t ksm = (size_t)slots * kKeySlotBytes + rest + 16 * slots;
        cudaError_t e2 = cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksm);
        if (e2 != cudaSuccess) return e2;
        kk<<<grid, kTileThreads + 32, ksm, s>>>(m1, m2, in, n, tiles, k1_out, w_out, cnt, lo, hist16, copies, key.len);
        return cudaGetLastError();
      };
      if (ring <= 4) return launch(ka_tile_keys<kTileThreads, kTileItems, 4>, 4);
      if (ring <= 6) return launch(ka_tile_keys<kTileThreads, kTileItems, 6>, 6);
      if (ring <= 8) return launch(ka_tile_keys<kTileThreads, kTileItems, 8>, 8);
      return launch(ka_tile_keys<kTileThreads, kTileItems, 11>, 11);
    }
    auto sk = ka_tile_stream<kTileThreads, kTileItems>;
    const size_t ssm = (size_t)kRing * kPieceBytes + rest;
    e = cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    if (e != cudaSuccess) return e;
    sk<<<grid, kTileThreads, ssm, s>>>(in, n, tiles, k1_out, w_out, cnt, lo, hist16, copies, key.len);
    return cudaGetLastError();
  }
  kern<<<tiles, kTileThreads, smem, s>>>(in, n, tiles, k1_out, w_out, cnt, lo, hist16, copies, key);
  return cudaGetLastError();
}

}  // namespace ley
