// k_bucket.cu — K-d + K-e fused: per-bucket sort of (key-tail, ordinal) pairs, then the record gather
// of that bucket, plus level-1 classification.
//
// PAPER.md §3.1 Algorithm 1 lines 65-85: buckets below bigBucketThreshold go to smallBucketQueue and
// are finished by one worker each — SingleThreadRadixSort on the next radix, then ComparisonSort for
// buckets under tinyBucketThreshold ("size is small enough for comparison-based sort to perform
// more efficient than Radix Sort"). On the GPU a "worker" is a warp (tiny buckets, register bitonic
// network over the composite (tail, ordinal)) or a CTA (shared-memory counting pass on the next 1..13
// unconsumed bits of the composite key, then an exact rank inside every tiny sub-bucket, or a warp
// bitonic network for larger ones). SURVEY.md §8a row a5.
//
// The same worker then performs the record scatter of its bucket (§3.2, "scatter
// data records ... given the sorted (key, pointer) tuples"): the bucket's output is
// the contiguous range out[start, start+len), so each warp takes groups of 32 output records, issues
// 16-byte cp.async copies of each record's 16-byte-aligned 112-byte window [floor(100 p/16)*16, +112)
// into its shared-memory staging, re-aligns and writes the group as a coalesced word stream. Fusing the
// two removes the perm round trip and hides the sort's shared-memory work under other
// CTAs' gather traffic. Every chunk copy starts inside the input buffer (the window starts at or below
// the record) and, being 16-byte aligned, never crosses a page.
//
// The comparison order is the composite (tail, ordinal) — the sort's strict total order — so the result
// does not depend on the order in which atomics place elements.
#include <stdio.h>
#include <stdlib.h>

#include "classify.cuh"
#include "common.cuh"
#include "kc_chunk.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

constexpr int kGroup = 32;                     // records per warp gather group
constexpr int kWindow = 112;                   // 7 x 16-byte chunks hold any 4-byte-aligned 100-byte record
constexpr int kStageBytes = kGroup * kWindow;  // 3584 B per gathering warp

// 16-byte chunk of a record window. .L2::64B caps the L2's DRAM fetch for the miss at 64 B: a plain miss
// is promoted to the whole 128-B line, so a random 100-B record cost 224 DRAM bytes instead of 162
// (profiles/r02_fetch_granularity.txt). src_bytes < 16 zero-fills the rest (the input's last chunk).
__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr, uint32_t src_bytes, bool l2_64) {
  if (l2_64)
    asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16, %2;" ::"r"(smem_addr), "l"(gptr), "r"(src_bytes)
                 : "memory");
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr), "l"(gptr), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void stg_cs_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Digest of a record's 10-byte key prefix (words 0, 1 and the low half of word 2): equal prefixes give
// equal digests, so the tie-group scan of the hybrid long-key form (k_ties.cu) reads 8 B per record
// instead of the records' lines and verifies only the candidates against the records.
__device__ __forceinline__ uint64_t prefix_digest(const uint32_t* w) {
  return ((uint64_t)w[1] << 32 | w[0]) ^ ((uint64_t)(w[2] & 0xFFFFu) * 0x9E3779B97F4A7C15ull);
}

// One group of cnt <= 32 records in[perm[g0 + r]] by one warp: group_issue starts the 16-byte cp.async
// copies of every record's window into `stage` (kStageBytes, 16-byte aligned); after cp_async_wait_all,
// group_store re-aligns the group and writes it as a coalesced word stream to dst (and, with dg, the
// records' prefix digests).
__device__ __forceinline__ void group_issue(const uint32_t* perm, uint32_t g0, uint32_t cnt, const uint8_t* __restrict__ in,
                                            uint64_t in_bytes, uint32_t stage_s, bool l2_64) {
  const int lane = threadIdx.x & 31;
  const uint32_t p = lane < (int)cnt ? perm[g0 + lane] : 0u;
  const uint32_t sl = stage_s + 16u * lane;  // chunk cidx -> stage byte r * 112 + c * 16 = 16 cidx
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const int cidx = q * 32 + lane;
    const int r = cidx / 7, c = cidx - r * 7;
    const uint32_t pr = __shfl_sync(0xffffffffu, p, r);
    const uint64_t a = (((uint64_t)pr * kRecordBytes) & ~uint64_t(15)) + (uint64_t)c * 16;
    if (r < (int)cnt && a < in_bytes)  // (chunks past the input's end hold no record byte)
      cp_async16(sl + 512u * q, in + a, in_bytes - a < 16 ? (uint32_t)(in_bytes - a) : 16u, l2_64);
  }
}
__device__ __forceinline__ void group_store(const uint32_t* perm, uint32_t g0, uint32_t cnt, const uint8_t* stage,
                                            uint32_t* __restrict__ dst, uint64_t* __restrict__ dg) {
  const int lane = threadIdx.x & 31;
  if (cnt == kGroup) {
    // a full group, unrolled: output word w = lane + 32 i of record r = w / 25 sits at stage byte
    // r * 112 + off_r + 4 (w - 25 r) = 4 w + X[r], X[r] = 12 r + off_r held by lane r (one shuffle per word
    // instead of a shared-memory load of perm[r] and the address arithmetic; the stores take immediate offsets)
    const uint32_t xl = 12u * lane + ((perm[g0 + lane] * 4u) & 15u);
    const uint8_t* sb = stage + 4 * lane;
    uint32_t* db = dst + lane;
#pragma unroll
    for (int i = 0; i < kRecordWords; ++i) {
      const uint32_t r = ((lane + 32u * i) * 1311u) >> 15;  // == (lane + 32 i) / 25 for all w < 800
      const uint32_t x = __shfl_sync(0xffffffffu, xl, r);
      stg_cs_u32(db + 32 * i, *reinterpret_cast<const uint32_t*>(sb + 128 * i + x));
    }
  } else {
    const uint32_t words = cnt * kRecordWords;
    for (uint32_t w = lane; w < words; w += 32) {
      const uint32_t r = w / kRecordWords, o = w - r * kRecordWords;
      const uint32_t off = (perm[g0 + r] * 4u) & 15u;  // 100 p mod 16 == 4 p mod 16
      stg_cs_u32(dst + w, *reinterpret_cast<const uint32_t*>(stage + r * kWindow + off + 4 * o));
    }
  }
  if (dg && lane < (int)cnt)
    dg[lane] = prefix_digest(reinterpret_cast<const uint32_t*>(stage + lane * kWindow + ((perm[g0 + lane] * 4u) & 15u)));
}

// Records in[perm[i]] -> out_base[i] for i in [0, s) by one warp, groups g0 = first, first + stride, ...
// of 32 records, through `stage`. perm lives in shared memory. With dg_base, also dg_base[i] =
// prefix_digest(record).
__device__ __forceinline__ void warp_gather(const uint32_t* perm, uint32_t s, uint32_t first, uint32_t stride,
                                            const uint8_t* __restrict__ in, uint64_t in_bytes,
                                            uint8_t* __restrict__ out_base, uint8_t* stage,
                                            uint64_t* __restrict__ dg_base, bool l2_64 = true) {
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
  for (uint32_t g0 = first; g0 < s; g0 += stride) {
    const uint32_t cnt = min((uint32_t)kGroup, s - g0);
    group_issue(perm, g0, cnt, in, in_bytes, stage_s, l2_64);
    cp_async_wait_all();
    __syncwarp();
    group_store(perm, g0, cnt, stage, reinterpret_cast<uint32_t*>(out_base + (uint64_t)g0 * kRecordBytes),
                dg_base ? dg_base + g0 : nullptr);
    __syncwarp();
  }
}

// Two groups in flight per warp (cp.async commit groups): group g's copies land while group g - stride is
// stored. stage0 / stage1: two kStageBytes slots (16-byte aligned, anywhere in shared memory).
__device__ __forceinline__ void warp_gather2(const uint32_t* perm, uint32_t s, uint32_t first, uint32_t stride,
                                             const uint8_t* __restrict__ in, uint64_t in_bytes,
                                             uint8_t* __restrict__ out_base, uint8_t* stage0, uint8_t* stage1,
                                             uint64_t* __restrict__ dg_base, bool l2_64) {
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(stage0), s1 = (uint32_t)__cvta_generic_to_shared(stage1);
  uint32_t ga = first, gb = first + stride;  // (two named slots, not an indexed pair: no local memory)
  auto issue = [&](uint32_t g, uint32_t ss) {
    if (g < s) group_issue(perm, g, min((uint32_t)kGroup, s - g), in, in_bytes, ss, l2_64);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto drain = [&](uint32_t g, const uint8_t* st) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // group g landed (the newer one may be in flight)
    __syncwarp();
    group_store(perm, g, min((uint32_t)kGroup, s - g), st, reinterpret_cast<uint32_t*>(out_base + (uint64_t)g * kRecordBytes),
                dg_base ? dg_base + g : nullptr);
    __syncwarp();
  };
  issue(ga, s0);
  issue(gb, s1);
  while (ga < s) {
    drain(ga, stage0);
    ga += 2 * stride;
    issue(ga, s0);
    if (gb >= s) break;
    drain(gb, stage1);
    gb += 2 * stride;
    issue(gb, s1);
  }
  cp_async_wait_all();
}

// LEY_KD_STAGES = 2 (build flag): the 1024-thread register tiers gather with warp_gather2 — measured slower
// (C4 K-d+K-e 40.8 vs 35.4 ms, C3 11.89 vs 11.65: 26 warps with two groups each lose to 32 with one;
// DESIGN.md §9)
#ifndef LEY_KD_STAGES
#define LEY_KD_STAGES 1
#endif
constexpr int kGatherStages = 1;  // groups in flight per gathering warp (one-stage tiers)

// ---------------------------------------------------------------------------- CTA tier
// In-smem all-ascending bitonic network over [b, e) by one warp; virtual +inf padding beyond e never
// moves, so compare-exchanges touching it are skipped.
__device__ void warp_bitonic_smem(uint64_t* st, uint32_t* si, uint32_t b, uint32_t e) {
  const uint32_t sz = e - b;
  uint32_t P = 1;
  while (P < sz) P <<= 1;
  const int lane = threadIdx.x & 31;
  for (uint32_t k = 2; k <= P; k <<= 1) {
    const uint32_t hk = k >> 1;
    for (uint32_t q = lane; q < P / 2; q += 32) {  // flip step: (blk*k + r, blk*k + k-1-r)
      uint32_t blk = q / hk, r = q % hk;
      uint32_t lo = blk * k + r, hi = blk * k + k - 1 - r;
      if (hi < sz) {
        uint64_t ta = st[b + lo], tb = st[b + hi];
        uint32_t xa = si[b + lo], xb = si[b + hi];
        if (pair_less(tb, xb, ta, xa)) {
          st[b + lo] = tb; st[b + hi] = ta;
          si[b + lo] = xb; si[b + hi] = xa;
        }
      }
    }
    __syncwarp();
    for (uint32_t j = hk >> 1; j > 0; j >>= 1) {
      for (uint32_t q = lane; q < P / 2; q += 32) {
        uint32_t lo = (q / j) * 2 * j + (q % j), hi = lo + j;
        if (hi < sz) {
          uint64_t ta = st[b + lo], tb = st[b + hi];
          uint32_t xa = si[b + lo], xb = si[b + hi];
          if (pair_less(tb, xb, ta, xa)) {
            st[b + lo] = tb; st[b + hi] = ta;
            si[b + lo] = xb; si[b + hi] = xa;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Counting bins of a tier: 2^14 for the register-form tiers of >= 8192 records, as two 16-bit counters
// per shared-memory word (C4's 10240 tier: sub-buckets of ~0.6 records; 13 bits gave C4 K-d+K-e -1 ms
// over 12), 2^12 otherwise.
template <uint32_t CAP, int THREADS>
__host__ __device__ constexpr uint32_t kd_bins() {
  return (CAP / THREADS <= 16 && CAP >= 8192) ? 16384u : CAP >= 4096 ? 4096u : CAP;
}
template <uint32_t CAP, int THREADS>
struct KdLayout {
  static constexpr uint32_t BINS = kd_bins<CAP, THREADS>();
  static constexpr int WARPS = THREADS / 32;
  static constexpr bool REGS = CAP / THREADS <= 16;  // bucket held in registers (else re-read from L2)
  // s_bigl: the sub-buckets of >= 2 records left for the warp network (<= CAP / 2 of them) in the register
  // form; the large-CAP form also uses it as a second per-bin counter array
  static constexpr uint32_t BIGL = REGS ? (BINS < CAP / 2 ? BINS : CAP / 2) : BINS;
  // counters packed two per 32-bit word (16 bits hold any count or start of a bucket of <= CAP < 2^16)
  static constexpr bool PACKED = REGS && BINS > 8192;
  static_assert(!PACKED || CAP < 65536, "16-bit counters");
  static constexpr uint32_t CNT_WORDS = PACKED ? BINS / 2 + 1 : BINS + 1;
  static_assert(!REGS || CAP % THREADS == 0, "the register form holds exactly CAP / THREADS items per thread");
  // [s_idx CAP x 4][s_perm CAP x 4 (REGS only)][reusable: s_tail CAP x 8 | s_cnt | s_bigl | s_tmp][stage]
  static constexpr size_t kIdx = 0;
  static constexpr size_t kPerm = kIdx + (size_t)CAP * 4;
  static constexpr size_t kTail = kPerm + (REGS ? (size_t)CAP * 4 : 0);
  static constexpr size_t kCnt = kTail + (size_t)CAP * 8;
  static constexpr size_t kBigl = kCnt + (size_t)CNT_WORDS * 4;
  static constexpr size_t kTmp = kBigl + (size_t)BIGL * 4;
  static constexpr size_t kReuseEnd = kTmp + 64 * 4;
  // gather staging: every warp gets kGatherStages groups, overlapping the sort area (free once the bucket
  // is sorted) and extending past it where the sort area is smaller
  static constexpr size_t kWarpStage = (size_t)kGatherStages * kStageBytes;
  static constexpr size_t kSmemMax = 227 * 1024 - 1024;  // dynamic; leaves room for the static mbarriers
  static constexpr int GWARPS_FIT = (int)((kSmemMax - kTail) / kWarpStage);
  static constexpr int GWARPS = GWARPS_FIT < WARPS ? GWARPS_FIT : WARPS;
  static constexpr size_t kStage = kTail;
  // Two-stage form (the one-CTA-per-SM register tiers, LEY_KD_STAGES = 2): slots in the dead s_idx area
  // [0, kPerm) and from kTail on; GW2 warps hold two slots each (C4's 10240 tier: 52 groups in flight per SM
  // instead of 32)
  static constexpr int SLOTS_A = REGS ? (int)(kPerm / kStageBytes) : 0;
  static constexpr int SLOTS_B = (int)((kSmemMax - kTail) / kStageBytes);
  static constexpr int GW2_FIT = (SLOTS_A + SLOTS_B) / 2;
  static constexpr int GW2 = GW2_FIT < WARPS ? GW2_FIT : WARPS;
  static constexpr bool TWO = LEY_KD_STAGES == 2 && REGS && THREADS >= 1024 && 2 * GW2 > GWARPS;
  static constexpr int SLOTS_B_USED = TWO ? (2 * GW2 - SLOTS_A > 0 ? 2 * GW2 - SLOTS_A : 0) : GWARPS;
  static constexpr size_t kStageEnd = kStage + (size_t)SLOTS_B_USED * kWarpStage;
  static constexpr size_t kBytes = kStageEnd > kReuseEnd ? kStageEnd : kReuseEnd;
  __host__ __device__ static constexpr size_t slot(int j) {
    return j < SLOTS_A ? (size_t)j * kStageBytes : kStage + (size_t)(j - SLOTS_A) * kStageBytes;
  }
  static_assert(kStage % 16 == 0, "gather staging must be 16-byte aligned");
  static_assert(GWARPS >= 1 && kBytes <= kSmemMax, "K-de tier does not fit shared memory");
};

// One CTA per bucket (len <= CAP), persistent over its list:
//   1. load the bucket's (tail, ordinal) pairs (coalesced; held in registers when CAP/THREADS <= 16,
//      else re-read from L2),
//   2. counting pass on the next `bits` unconsumed bits of the composite key (shared-memory atomics give
//      each item its rank inside its sub-bucket), block scan of the 2^bits counters, placement,
//   3. exact rank inside every tiny sub-bucket (count of smaller composites; <= kd_insert_max), a warp
//      bitonic network for larger ones — Alg. 1's ComparisonSort below tinyBucketThreshold,
//   4. the bucket's records gathered into out[start, start+len) by the CTA's warps (see file header).
// FUSED (level 1 only, THREADS >= 256): the kernel also owns the level-1 split, as kd_ws_sort's fused form
// (kc_chunk.cuh): its items are the 16-bit buckets of tier `tier` claimed in ascending order, each sorted
// once its byte-0 bucket is split; the CTA runs split chunks while it waits and after its last bucket.
template <uint32_t CAP, int THREADS, bool DG, bool FUSED = false>
__global__ void __launch_bounds__(THREADS, (THREADS >= 1024 || (CAP / THREADS) > 8) ? 1 : (CAP / THREADS) > 4 ? 4 : 8)
    kd_cta_sort(const Seg* __restrict__ list, const uint32_t* __restrict__ count, const uint64_t* __restrict__ t0,
                const uint32_t* __restrict__ i0, const uint64_t* __restrict__ t1, const uint32_t* __restrict__ i1,
                uint32_t* __restrict__ perm, Tunables tu, const uint8_t* __restrict__ in, uint64_t in_bytes,
                uint8_t* __restrict__ out, uint64_t* __restrict__ dg, KcArgs kc = KcArgs{}, int tier = -1) {
  using L = KdLayout<CAP, THREADS>;
  constexpr uint32_t BINS = L::BINS;
  constexpr int WARPS = L::WARPS;
  constexpr int ITEMS = CAP / THREADS;
  constexpr bool REGS = L::REGS;
  constexpr bool PACKED = L::PACKED;
  constexpr int RITEMS = REGS ? ITEMS : 1;
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(smem + L::kIdx);
  uint32_t* s_perm = REGS ? reinterpret_cast<uint32_t*>(smem + L::kPerm) : s_idx;  // sorted ordinals
  uint64_t* s_tail = reinterpret_cast<uint64_t*>(smem + L::kTail);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + L::kCnt);    // [BINS + 1]: counts, then starts
  auto cnt_get = [&](uint32_t g) -> uint32_t {                       // (PACKED: 16-bit halves)
    if constexpr (PACKED) return (s_cnt[g >> 1] >> (16u * (g & 1u))) & 0xFFFFu;
    else return s_cnt[g];
  };
  uint32_t* s_bigl = reinterpret_cast<uint32_t*>(smem + L::kBigl);  // [BINS]: sub-buckets for the network
  uint32_t* s_tmp = reinterpret_cast<uint32_t*>(smem + L::kTmp);    // [32] scan tmp, [32] = #big
  uint32_t* s_nbig = s_tmp + 32;
  uint8_t* s_stage = smem + L::kStage;                               // gather staging (reuses the sort area)

  const PdlExitWait pdl_exit = pdl_enter(tu.pdl);
  const uint32_t nitems = FUSED ? 0u : *count;
  const int warp = threadIdx.x >> 5;
  constexpr int KC_ITEMS = (kChunk + THREADS - 1) / THREADS;
  static_assert(!FUSED || (THREADS >= kRadix && L::kBytes >= kKcSmem), "fused split geometry");
  __shared__ uint32_t s_claim[4];
  const uint32_t kc_total = FUSED ? kc.cstart[256] : 0u;
  auto claim_chunk = [&]() -> uint32_t {  // next split chunk (~0u: none left)
    if (threadIdx.x == 0) {
      const uint32_t c = atomicAdd(kc.ticket, 1u);
      s_claim[2] = c < kc_total ? c : ~0u;
    }
    __syncthreads();
    const uint32_t c = s_claim[2];
    __syncthreads();
    return c;
  };
  uint32_t* const ticket = const_cast<uint32_t*>(count) + kTierTicket;
  uint32_t it = 0, nxt = tu.kd_claim ? 0u : blockIdx.x;
  __shared__ Seg s_next;  // the next bucket's descriptor, read early by the prefetch (s_next_it: its index)
  __shared__ uint32_t s_next_it;
  if (threadIdx.x == 0) s_next_it = ~0u;
  if (!FUSED && tu.kd_claim && threadIdx.x == 0) s_claim[3] = atomicAdd(ticket, 1u);
  while (true) {
    Seg sg;
    if constexpr (FUSED) {
      if (threadIdx.x == 0) s_claim[0] = kc_claim_bucket(kc, [&](uint32_t len) { return tier_of(len, tu) == tier; });
      __syncthreads();
      const uint32_t p = s_claim[0];
      __syncthreads();
      if (p >= 65536u) break;
      const uint32_t b0 = p >> 8, need = kc.cstart[b0 + 1] - kc.cstart[b0];
      while (true) {  // byte-0 bucket b0 must be split: run chunks while waiting
        if (threadIdx.x == 0) s_claim[1] = ld_acquire_u32(&kc.done[b0]) >= need;
        __syncthreads();
        const bool ready = s_claim[1] != 0;
        __syncthreads();
        if (ready) break;
        const uint32_t c = claim_chunk();
        if (c != ~0u) kc_chunk<THREADS, KC_ITEMS, SyncCta>(kc, c, smem);
        else __nanosleep(1000);  // the remaining chunks are being split by running CTAs
      }
      sg = Seg{kc.B16[p], kc.hist16[p], 2u, 1u};
    } else {  // buckets claimed dynamically (ticket kTierTicket words past the count), one bucket ahead so
              // the claim's round trip overlaps the current bucket: a CTA that becomes resident late (PDL
              // overlap with the previous tier) just takes fewer
      if (tu.kd_claim) {
        __syncthreads();
        it = s_claim[3];
        if (threadIdx.x == 0 && it < nitems) nxt = atomicAdd(ticket, 1u);
      } else {
        it = nxt;  // static: blockIdx.x, + gridDim.x, ...
        nxt = it + gridDim.x;
      }
      if (it >= nitems) break;
      // (claimed mode: the descriptor was read by the prefetch below during the last bucket, and the
      // barrier above orders that store before this read)
      sg = tu.kd_claim && s_next_it == it ? s_next : list[it];
    }
    for (uint32_t g = threadIdx.x; g < L::CNT_WORDS; g += THREADS) s_cnt[g] = 0;  // was gather staging
    __syncthreads();
    const uint32_t s = sg.len;
    // item j of this thread (index j THREADS + tid) exists iff j < nv: one register instead of the index
    // (which the compiler would otherwise rematerialise from %tid.x in every per-item loop)
    const uint32_t nv = s > threadIdx.x ? (s - threadIdx.x + THREADS - 1) / THREADS : 0u;
    const uint64_t* tp = (sg.parity ? t1 : t0) + sg.start;
    const uint32_t* ip = (sg.parity ? i1 : i0) + sg.start;
    // unconsumed bits of the composite key (tail = key bytes 2..9, then the 32-bit ordinal): key bits
    // while depth < 10, else ordinal bits (the key bytes are then all equal inside the bucket)
    const bool on_idx = sg.depth >= kKeyBytes;
    const uint32_t avail = on_idx ? 8u * (14u - sg.depth) : 8u * (kKeyBytes - sg.depth);
    uint32_t bits = s > 1 ? 32u - __clz(s - 1) : 0u;
    bits = min(bits, (uint32_t)tu.kd_digit_bits);
    bits = min(bits, avail);
    bits = min(bits, 31u - __clz(BINS));
    const uint32_t shift = avail - bits;
    const uint32_t nb = 1u << bits;
    const uint32_t mask = nb - 1;
    auto digit2 = [&](uint64_t t, uint32_t x) -> uint32_t {
      return bits ? (on_idx ? (x >> shift) & mask : (uint32_t)(t >> shift) & mask) : 0u;
    };

    uint64_t tr[RITEMS];
    uint32_t xr[RITEMS], rr[RITEMS];
    if (REGS) {
#pragma unroll
      for (int j = 0; j < RITEMS; ++j) {
        uint32_t i = j * THREADS + threadIdx.x;
        if (i < s) {
          tr[j] = __ldcg(tp + i);  // (L2 loads: in the fused form other SMs wrote these pairs during this kernel)
          xr[j] = __ldcg(ip + i);
        }
      }
#pragma unroll
      for (int j = 0; j < RITEMS; ++j) {
        if (j < nv) {
          const uint32_t d = digit2(tr[j], xr[j]);
          if constexpr (PACKED) {
            const uint32_t sh = 16u * (d & 1u);
            rr[j] = (atomicAdd(&s_cnt[d >> 1], 1u << sh) >> sh) & 0xFFFFu;
          } else {
            rr[j] = atomicAdd(&s_cnt[d], 1u);
          }
        }
      }
    } else {
      // batches of 8 independent loads per thread keep the bucket read latency-tolerant
      for (uint32_t i0b = threadIdx.x; i0b < s; i0b += 8 * THREADS) {
        uint64_t tb[8];
        uint32_t xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t i = i0b + u * THREADS;
          tb[u] = i < s ? __ldcg(tp + i) : 0;
          xb[u] = (i < s && on_idx) ? __ldcg(ip + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0b + u * THREADS < s) atomicAdd(&s_cnt[digit2(tb[u], xb[u])], 1u);
      }
    }
    if (threadIdx.x == 0) *s_nbig = 0;
    __syncthreads();
    // exclusive scan of the nb counters in place (contiguous slice per thread)
    if constexpr (PACKED) {  // slices of whole words (two counters each; an odd nb leaves a zero high half)
      const uint32_t nw = (nb + 1) >> 1;
      const uint32_t per = (nw + THREADS - 1) / THREADS;
      const uint32_t w0 = threadIdx.x * per;
      const uint32_t w1 = min(nw, w0 + per);
      uint32_t sum = 0;
      for (uint32_t w = w0; w < w1; ++w) sum += (s_cnt[w] & 0xFFFFu) + (s_cnt[w] >> 16);
      uint32_t run = block_excl_scan<THREADS>(sum, s_tmp, nullptr);
      for (uint32_t w = w0; w < w1; ++w) {
        const uint32_t c = s_cnt[w];
        const uint32_t lo = run;
        run += c & 0xFFFFu;
        s_cnt[w] = lo | (run << 16);
        run += c >> 16;
      }
      if (threadIdx.x == 0) {  // the sentinel start of bin nb (word nb/2 is no thread's slice unless nb = 1)
        const uint32_t w = nb >> 1, sh = 16u * (nb & 1u);
        s_cnt[w] = (s_cnt[w] & ~(0xFFFFu << sh)) | (s << sh);
      }
    } else {
      const uint32_t per = (nb + THREADS - 1) / THREADS;
      const uint32_t g0 = threadIdx.x * per;
      const uint32_t g1 = min(nb, g0 + per);
      uint32_t sum = 0;
      for (uint32_t g = g0; g < g1; ++g) sum += s_cnt[g];
      uint32_t run = block_excl_scan<THREADS>(sum, s_tmp, nullptr);
      for (uint32_t g = g0; g < g1; ++g) {
        uint32_t c = s_cnt[g];
        s_cnt[g] = run;
        run += c;
      }
      if (threadIdx.x == 0) s_cnt[nb] = s;
    }
    __syncthreads();
    if (REGS) {
      // place, then every item finds its final rank inside its (tiny) sub-bucket by counting the
      // smaller composites there
#pragma unroll
      for (int j = 0; j < RITEMS; ++j) {
        if (j < nv) {
          const uint32_t b = cnt_get(digit2(tr[j], xr[j]));
          s_tail[b + rr[j]] = tr[j];
          s_idx[b + rr[j]] = xr[j];
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < RITEMS; ++j) {
        if (j < nv) {
          const uint32_t d = digit2(tr[j], xr[j]);
          const uint32_t b = cnt_get(d), sz = cnt_get(d + 1) - b;
          if (sz == 1) {
            s_perm[b] = xr[j];
          } else if (sz <= (uint32_t)tu.kd_insert_max) {
            uint32_t rank = 0;
            const uint32_t self = b + rr[j];
            for (uint32_t m = b; m < b + sz; ++m)
              if (m != self) rank += pair_less(s_tail[m], s_idx[m], tr[j], xr[j]) ? 1u : 0u;
            s_perm[b + rank] = xr[j];
          } else if (rr[j] == 0) {
            s_bigl[atomicAdd(s_nbig, 1u)] = d;
          }
        }
      }
      __syncthreads();
      const uint32_t nbig = *s_nbig;
      for (uint32_t q = warp; q < nbig; q += WARPS) {
        const uint32_t g = s_bigl[q];
        const uint32_t b = cnt_get(g), e = cnt_get(g + 1);
        warp_bitonic_smem(s_tail, s_idx, b, e);
        for (uint32_t i = b + (threadIdx.x & 31); i < e; i += 32) s_perm[i] = s_idx[i];
      }
    } else {
      // ---- large-CAP path: elements re-read from L2, placed by a second counter pass
      for (uint32_t g = threadIdx.x; g < nb; g += THREADS) s_bigl[g] = 0;
      __syncthreads();
      for (uint32_t i0b = threadIdx.x; i0b < s; i0b += 8 * THREADS) {
        uint64_t tb[8];
        uint32_t xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t i = i0b + u * THREADS;
          if (i < s) {
            tb[u] = __ldcg(tp + i);
            xb[u] = __ldcg(ip + i);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (i0b + u * THREADS < s) {
            const uint32_t d = digit2(tb[u], xb[u]);
            const uint32_t p = s_cnt[d] + atomicAdd(&s_bigl[d], 1u);
            s_tail[p] = tb[u];
            s_idx[p] = xb[u];
          }
        }
      }
      __syncthreads();
      // comparison sort of every sub-bucket, in place
      for (uint32_t g = threadIdx.x; g < nb; g += THREADS) {
        uint32_t b = s_cnt[g], e = s_cnt[g + 1];
        uint32_t sz = e - b;
        if (sz <= 1) continue;
        if (sz <= (uint32_t)tu.kd_insert_max) {
          for (uint32_t i = b + 1; i < e; ++i) {
            uint64_t t = s_tail[i];
            uint32_t x = s_idx[i];
            uint32_t j = i;
            while (j > b && pair_less(t, x, s_tail[j - 1], s_idx[j - 1])) {
              s_tail[j] = s_tail[j - 1];
              s_idx[j] = s_idx[j - 1];
              --j;
            }
            s_tail[j] = t;
            s_idx[j] = x;
          }
        } else {
          s_bigl[atomicAdd(s_nbig, 1u)] = g;
        }
      }
      __syncthreads();
      const uint32_t nbig = *s_nbig;
      for (uint32_t q = warp; q < nbig; q += WARPS) {
        uint32_t g = s_bigl[q];
        warp_bitonic_smem(s_tail, s_idx, s_cnt[g], s_cnt[g + 1]);
      }
    }
    __syncthreads();  // sorted ordinals complete; the sort area is free for the gather staging
    if (!FUSED && threadIdx.x == 0 && nxt < nitems) {  // the next bucket's pairs, while this one is gathered
      const Seg ns = list[nxt];
      if (tu.kd_claim) {  // (published by the barriers that end this bucket)
        s_next = ns;
        s_next_it = nxt;
      }
      prefetch_l2_last((ns.parity ? t1 : t0) + ns.start, (uint64_t)ns.len * 8);
      prefetch_l2_last((ns.parity ? i1 : i0) + ns.start, (uint64_t)ns.len * 4);
    }
    if (perm)
      for (uint32_t i = threadIdx.x; i < s; i += THREADS) perm[sg.start + i] = s_perm[i];
    if constexpr (L::TWO) {
      if (out && warp < L::GW2)
        warp_gather2(s_perm, s, (uint32_t)warp * kGroup, (uint32_t)L::GW2 * kGroup, in, in_bytes,
                     out + (uint64_t)sg.start * kRecordBytes, smem + L::slot(2 * warp), smem + L::slot(2 * warp + 1),
                     DG ? dg + sg.start : nullptr, tu.gather_l2_64 != 0);
    } else {
      if (out && warp < L::GWARPS)
        warp_gather(s_perm, s, (uint32_t)warp * kGroup, (uint32_t)L::GWARPS * kGroup, in, in_bytes,
                    out + (uint64_t)sg.start * kRecordBytes, s_stage + (size_t)warp * kStageBytes,
                    DG ? dg + sg.start : nullptr, tu.gather_l2_64 != 0);
    }
    if (!FUSED && tu.kd_claim && threadIdx.x == 0) s_claim[3] = nxt;  // (every thread read this claim long ago)
    __syncthreads();  // staging (and s_perm) reused by the next bucket
  }
  if constexpr (FUSED)  // the split's remaining chunks: the other tiers' buckets (later kernels) need them
    for (uint32_t c = claim_chunk(); c != ~0u; c = claim_chunk()) kc_chunk<THREADS, KC_ITEMS, SyncCta>(kc, c, smem);
}

template <uint32_t CAP, int THREADS, bool DG>
cudaError_t launch_cta_sort(const Seg* list, const uint32_t* count, const uint64_t* t0, const uint32_t* i0,
                            const uint64_t* t1, const uint32_t* i1, uint32_t* perm, const Tunables& tu, int sms,
                            const uint8_t* in, uint64_t in_bytes, uint8_t* out, uint64_t* dg, cudaStream_t s,
                            const KcArgs* kc = nullptr, int tier = -1) {
  auto kern = kd_cta_sort<CAP, THREADS, DG, false>;
  if constexpr (THREADS >= kRadix && KdLayout<CAP, THREADS>::kBytes >= kKcSmem)
    if (kc) kern = kd_cta_sort<CAP, THREADS, DG, true>;
  const size_t smem = KdLayout<CAP, THREADS>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  e = launch_k(kern, sms * per_sm, THREADS, smem, s, tu.pdl != 0, list, count, t0, i0, t1, i1, perm, tu, in, in_bytes, out, dg,
               kc ? *kc : KcArgs{}, tier);
  if (e != cudaSuccess) return e;
  if (getenv("LEY_DEBUG_SYNC")) {
    fprintf(stderr, "[ley] kd_cta_sort<%u,%d> grid %d smem %zu\n", CAP, THREADS, sms * per_sm, smem);
    cudaError_t e2 = cudaStreamSynchronize(s);
    fprintf(stderr, "[ley]   done: %s\n", cudaGetErrorString(e2));
  }
  return cudaGetLastError();
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}"
               ::"r"(a), "r"(parity) : "memory");
}
// One record's 16-byte-aligned 112-byte window by a TMA tensor copy, completion counted in bytes on an
// mbarrier. The tensor map views the records as [n/4 groups][25 rows][16 B] (group pitch 400 B): record
// p = 4g + j starts in row floor(100 j / 16) = 0, 6, 12, 18 of group g and its window is the box of 7 rows
// there (never past row 24). The map's L2 promotion is 64 B: a plain bulk copy's misses fetch whole 128-B
// lines (224 DRAM bytes per random record instead of 162; profiles/r02_fetch_granularity.txt).
__device__ __forceinline__ void tma_window(uint32_t dst, const CUtensorMap* map, uint32_t p, uint32_t mbar) {
  const int row = (int)((100u * (p & 3u)) >> 4), grp = (int)(p >> 2);
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(dst), "l"((uint64_t)map), "r"(0), "r"(row), "r"(grp), "r"(mbar) : "memory");
}
// (A/B form: a plain bulk copy of the same window, whose misses fetch whole 128-B lines)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
constexpr int kWsSlot = 128;                     // tensor-copy destinations 128-byte aligned
constexpr int kWsStageBytes = kGroup * kWsSlot;  // 4096 B per gathering warp and stage

// ---------------------------------------------------------------------------- warp tier (len <= 32)
// One warp per bucket, software-pipelined: the next bucket's list entry and pairs are loaded and sorted in
// registers while the current bucket's record copies are in flight. The kernel is issue-bound at small n
// (C1: 56 M warp instructions for 1e6 records, ncu), so every step is cut to few instructions:
//  * the network sorts one 64-bit composite (tail >> 5, lane) per lane — 7 instructions per exchange
//    instead of ~25 for the (tail, ordinal) pair — then fetches each position's pair from its source lane.
//    It equals the (tail, ordinal) order unless two tails agree in their top 59 bits; that case (detected
//    on adjacent sorted tails) re-sorts the pairs with the full comparison;
//  * each record is one bulk copy of its 16-byte-aligned 112-byte window (the last n mod 4 records, whose
//    window may pass the input's end, by exact word loads), completion counted on the warp's mbarrier;
//  * the bucket's output is written in 16-byte stores (4-byte head and tail words at its unaligned ends).
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  return (uint64_t)__shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src) << 32 | __shfl_sync(0xffffffffu, (uint32_t)v, src);
}

__device__ __forceinline__ void warp_sort_pairs(uint64_t& t, uint32_t& x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      uint64_t ot = __shfl_xor_sync(0xffffffffu, t, j);
      uint32_t ox = __shfl_xor_sync(0xffffffffu, x, j);
      bool up = (lane & k) == 0;
      bool lower = (lane & j) == 0;
      bool take = (lower == up) ? pair_less(ot, ox, t, x) : pair_less(t, x, ot, ox);
      if (take) {
        t = ot;
        x = ox;
      }
    }
  }
}

// (t, x) of lane i < len -> lane i holds the i-th smallest pair; lanes >= len hold (~0, ~0) padding.
// Bitonic network over the composites of lanes [0, KMAX) (KMAX = 16: the lower half-warp ends ascending).
template <int KMAX>
__device__ __forceinline__ uint64_t warp_sort_composite(uint64_t c) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= KMAX; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t oc = shfl_u64(c, lane ^ j);
      const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
      c = ((oc < c) == keep_min) ? oc : c;  // (composites are distinct: their low 5 bits are the lanes)
    }
  }
  return c;
}

__device__ __forceinline__ void warp_sort_bucket(uint32_t len, uint64_t& t, uint32_t& x) {
  const int lane = threadIdx.x & 31;
  uint64_t c = (t & ~uint64_t(31)) | (uint64_t)lane;
  c = len <= 16 ? warp_sort_composite<16>(c) : warp_sort_composite<32>(c);  // (10 or 15 exchange steps)
  const int src = (int)(c & 31u);
  const uint64_t st = shfl_u64(t, src);
  const uint32_t sx = __shfl_sync(0xffffffffu, x, src);
  const uint64_t prev = shfl_u64(st >> 5, (lane + 31) & 31);
  if (__any_sync(0xffffffffu, lane > 0 && (uint32_t)lane < len && prev == (st >> 5))) {
    warp_sort_pairs(t, x);  // tails equal in their top 59 bits: the full (tail, ordinal) network
    return;
  }
  t = st;
  x = sx;
}

__device__ __forceinline__ void cp_async4(uint32_t smem_addr, const void* gptr) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr), "l"(gptr) : "memory");
}

template <bool DG>
__global__ void __launch_bounds__(256)
    kd_warp_sort(const Seg* __restrict__ list, const uint32_t* __restrict__ count, const uint64_t* __restrict__ t0,
                 const uint32_t* __restrict__ i0, const uint64_t* __restrict__ t1, const uint32_t* __restrict__ i1,
                 uint32_t* __restrict__ perm, const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                 uint64_t* __restrict__ dg, int pdl) {
  __shared__ __align__(128) uint8_t s_stage[8][kStageBytes];
  const PdlExitWait pdl_exit = pdl_enter(pdl);
  const uint32_t nitems = *count;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(s_stage[wib]);
  uint32_t it = blockIdx.x * (blockDim.x >> 5) + wib;
  if (it >= nitems) return;
  uint64_t pol = 0;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto load = [&](const Seg& sg, uint64_t& t, uint32_t& x) {
    const uint64_t* tp = (sg.parity ? t1 : t0) + sg.start;
    const uint32_t* ip = (sg.parity ? i1 : i0) + sg.start;
    t = ~0ull;
    x = ~0u;
    if ((uint32_t)lane < sg.len) {
      t = tp[lane];
      x = ip[lane];
    }
  };
  Seg sg = list[it];
  uint64_t t;
  uint32_t x;
  load(sg, t, x);
  warp_sort_bucket(sg.len, t, x);
  while (true) {
    const uint32_t len = sg.len;
    if (perm && (uint32_t)lane < len) perm[sg.start + lane] = x;
    const uint64_t obyte = (uint64_t)sg.start * kRecordBytes;
    // stage byte a + i holds bucket output byte i: the same phase mod 16 as its global address
    const uint32_t a = (uint32_t)(reinterpret_cast<uintptr_t>(out + obyte) & 15u);
    const uint32_t words = len * kRecordWords;
    if (out) {  // (perm-only mode: the resident host path gathers later, chunk by chunk)
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // previous store read the stage
      __syncwarp();
      // 8 lanes per record, 4 records per round: lane j of a record copies its words j, j+8, j+16 (and
      // j = 0 word 24), so each copy instruction reads 32 contiguous bytes of each of its 4 records
      const uint32_t j = lane & 7;
      for (uint32_t r0 = 0; r0 < len; r0 += 4) {
        const uint32_t r = r0 + (lane >> 3);
        const uint32_t p = __shfl_sync(0xffffffffu, x, r & 31);
        if (r < len) {
          const uint8_t* src = in + (uint64_t)p * kRecordBytes + 4 * j;
          const uint32_t dst = stage_s + a + r * kRecordBytes + 4 * j;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (j + 8 * i < (uint32_t)kRecordWords) cp_async4(dst + 32 * i, src + 32 * i);
        }
      }
    }
    const uint32_t nit = it + nwarps;
    Seg ns{};
    uint64_t nt = 0;
    uint32_t nx = 0;
    if (nit < nitems) {  // overlaps the copies in flight
      ns = list[nit];
      load(ns, nt, nx);
      warp_sort_bucket(ns.len, nt, nx);
    }
    if (out) {
      cp_async_wait_all();
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the copies, before the bulk store reads them
      __syncwarp();
      const uint32_t bytes = words * 4u;
      const uint32_t i0 = (16u - a) & 15u;                                // first 16-byte-aligned output byte
      const uint32_t mid = bytes > i0 ? (bytes - i0) & ~15u : 0u;         // aligned middle, one bulk store
      const uint32_t i1 = i0 + mid;
      uint32_t* o32 = reinterpret_cast<uint32_t*>(out + obyte);
      const uint32_t* s32 = reinterpret_cast<const uint32_t*>(s_stage[wib] + a);
      if (lane == 0 && mid) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(out + obyte + i0),
                     "r"(stage_s + a + i0), "r"(mid), "l"(pol)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      const uint32_t hw = (i0 < bytes ? i0 : bytes) >> 2, tw = (bytes - (i0 < bytes ? i1 : bytes)) >> 2;
      if ((uint32_t)lane < hw) stg_cs_u32(o32 + lane, s32[lane]);
      else if ((uint32_t)lane >= 4 && (uint32_t)lane < 4 + tw) stg_cs_u32(o32 + (i1 >> 2) + lane - 4, s32[(i1 >> 2) + lane - 4]);
      if (DG && (uint32_t)lane < len) dg[sg.start + lane] = prefix_digest(s32 + lane * kRecordWords);
    }
    __syncwarp();
    if (nit >= nitems) break;
    it = nit;
    sg = ns;
    t = nt;
    x = nx;
  }
  if (out && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------- warp-specialised tier
// The fused kernel above alternates: all warps sort a bucket, then all warps gather it, so a CTA issues no
// record reads while it sorts. Here a CTA splits into a sort group (ST threads) and a gather group (GW
// warps) that run concurrently on consecutive buckets of the CTA's list through a two-slot ring of sorted
// ordinals: the sort group sorts bucket k+1 while the gather warps stream bucket k, each warp keeping two
// 32-record groups in flight (cp.async double buffering). Hand-off by named barriers (bar.arrive /
// bar.sync, producer/consumer counts): FULL[q] sort -> gather, EMPTY[q] gather -> sort.
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int kBarSort = 1, kBarFull = 2, kBarEmpty = 4;  // ids 1, 2-3, 4-5 (0 is __syncthreads)

// exclusive scan over a group of THREADS threads (tid = group-local index) synchronised by barrier `bar`
template <int THREADS>
__device__ __forceinline__ uint32_t group_excl_scan(uint32_t v, uint32_t* tmp, int tid, int bar) {
  constexpr int WARPS = THREADS / 32;
  const int lane = tid & 31, warp = tid >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  nbar_sync(bar, THREADS);
  if (warp == 0) {
    uint32_t w = lane < WARPS ? tmp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < WARPS) tmp[lane] = w;
  }
  nbar_sync(bar, THREADS);
  const uint32_t r = (warp ? tmp[warp - 1] : 0u) + x - v;
  nbar_sync(bar, THREADS);
  return r;
}

template <uint32_t CAP, int ST, int GW>
struct WsLayout {
  static constexpr uint32_t BINS = CAP < 1024 ? CAP : 1024;
  static constexpr size_t kIdx = 0;                                   // u32[CAP]
  static constexpr size_t kTail = kIdx + (size_t)CAP * 4;             // u64[CAP]
  static constexpr size_t kCnt = kTail + (size_t)CAP * 8;             // u32[BINS + 1]
  static constexpr size_t kBigl = kCnt + (size_t)(BINS + 1) * 4;      // u32[BINS]
  static constexpr size_t kTmp = kBigl + (size_t)BINS * 4;            // u32[64]
  static constexpr size_t kRing = (kTmp + 64 * 4 + 15) & ~size_t(15);  // u32[2][CAP]
  static constexpr size_t kDesc = kRing + 2 * (size_t)CAP * 4;        // uint2[2]
  static constexpr size_t kMbar = kDesc + 16;                          // u64[GW][2] gather-stage mbarriers
  static constexpr size_t kStage = (kMbar + (size_t)GW * 16 + 127) & ~size_t(127);  // [GW][2][kWsStageBytes]
  static constexpr size_t kBytes = kStage + (size_t)GW * 2 * kWsStageBytes;
};

constexpr uint32_t kEndDesc = 0xFFFFFFFFu;  // ring descriptor length that ends the gather group's loop

// FUSED (level 1 only): the kernel also owns the level-1 split K-c (kc_chunk.cuh). Its items are the 16-bit
// buckets of this tier claimed in ascending order from kc.kd_ticket instead of a list; before sorting a
// bucket of byte-0 bucket b the sort group waits for done[b], running split chunks itself meanwhile, and
// when no bucket is left it runs the split's remaining chunks (the other tiers' buckets need them).
template <uint32_t CAP, int ST, int GW, bool DG, bool FUSED>
__global__ void __launch_bounds__(ST + 32 * GW, 2)
    kd_ws_sort(const Seg* __restrict__ list, const uint32_t* __restrict__ count, const uint64_t* __restrict__ t0,
               const uint32_t* __restrict__ i0, const uint64_t* __restrict__ t1, const uint32_t* __restrict__ i1,
               uint32_t* __restrict__ perm, Tunables tu, const __grid_constant__ CUtensorMap in_map,
               const uint8_t* __restrict__ in, uint64_t n4, uint8_t* __restrict__ out, uint64_t* __restrict__ dg,
               KcArgs kc) {
  using L = WsLayout<CAP, ST, GW>;
  constexpr uint32_t BINS = L::BINS;
  constexpr int ITEMS = CAP / ST;
  constexpr int NT = ST + 32 * GW;
  constexpr int SW = ST / 32;
  // (no static shared memory: the dynamic block starts the CTA's window, so the 128-byte-aligned stage
  // offsets are 128-byte-aligned addresses, as the tensor copies need)
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(smem + L::kIdx);
  uint64_t* s_tail = reinterpret_cast<uint64_t*>(smem + L::kTail);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + L::kCnt);
  uint32_t* s_bigl = reinterpret_cast<uint32_t*>(smem + L::kBigl);
  uint32_t* s_tmp = reinterpret_cast<uint32_t*>(smem + L::kTmp);
  uint32_t* s_nbig = s_tmp + 32;
  uint32_t* s_ring = reinterpret_cast<uint32_t*>(smem + L::kRing);
  uint2* s_desc = reinterpret_cast<uint2*>(smem + L::kDesc);
  const PdlExitWait pdl_exit = pdl_enter(tu.pdl);
  const uint32_t nitems = FUSED ? 0u : *count;
  const int tid = threadIdx.x;
  static_assert(!FUSED || kKcSmem <= L::kTmp, "the split's staging reuses the sort area");

  if (tid < ST) {
    // ================================================================ sort group
    const int warp = tid >> 5;
    using Group = SyncGroup<kBarSort, ST>;
    uint32_t* s_claim = s_tmp + 40;  // (past the scan words and s_nbig; outside the split's staging)
    const uint32_t kc_total = FUSED ? kc.cstart[256] : 0u;
    // the next split chunk to run (thread 0 claims, the group reads; ~0u: none left)
    auto claim_chunk = [&]() -> uint32_t {
      if (tid == 0) {
        const uint32_t c = atomicAdd(kc.ticket, 1u);
        s_claim[2] = c < kc_total ? c : ~0u;
      }
      nbar_sync(kBarSort, ST);
      const uint32_t c = s_claim[2];
      nbar_sync(kBarSort, ST);  // (read by all before thread 0 writes it again)
      return c;
    };
    uint32_t k = 0;
    uint32_t* const ticket = const_cast<uint32_t*>(count) + kTierTicket;
    uint32_t it = 0, nxt = tu.kd_claim ? 0u : blockIdx.x;
    if (!FUSED && tu.kd_claim && tid == 0) s_claim[3] = atomicAdd(ticket, 1u);
    for (;; ++k) {
      Seg sg;
      if constexpr (FUSED) {
        if (tid == 0)
          s_claim[0] = kc_claim_bucket(kc, [&](uint32_t len) { return tier_of(len, tu) == kListMed2; });
        nbar_sync(kBarSort, ST);
        const uint32_t p = s_claim[0];
        nbar_sync(kBarSort, ST);
        if (p >= 65536u) break;
        const uint32_t b0 = p >> 8, need = kc.cstart[b0 + 1] - kc.cstart[b0];
        while (true) {  // byte-0 bucket b0 must be split: run chunks while waiting
          if (tid == 0) s_claim[1] = ld_acquire_u32(&kc.done[b0]) >= need;
          nbar_sync(kBarSort, ST);
          const bool ready = s_claim[1] != 0;
          nbar_sync(kBarSort, ST);
          if (ready) break;
          const uint32_t c = tu.kc_corun ? ~0u : claim_chunk();  // (co-run: the split kernel runs them all)
          if (c != ~0u) kc_chunk<ST, (kChunk + ST - 1) / ST, Group>(kc, c, smem);
          else __nanosleep(tu.kc_corun ? 256 : 1000);  // the remaining chunks are being split by running CTAs
        }
        sg = Seg{kc.B16[p], kc.hist16[p], 2u, 1u};
      } else {  // (dynamic claims one bucket ahead, or static, as in kd_cta_sort)
        if (tu.kd_claim) {
          nbar_sync(kBarSort, ST);
          it = s_claim[3];
          if (tid == 0 && it < nitems) nxt = atomicAdd(ticket, 1u);
        } else {
          it = nxt;
          nxt = it + gridDim.x;
        }
        if (it >= nitems) break;
        sg = list[it];
      }
      const int q = k & 1;
      uint32_t* s_perm = s_ring + q * CAP;
      if (k >= 2) nbar_sync(kBarEmpty + q, NT);  // the gather warps released slot q (bucket k-2)
      for (uint32_t g = tid; g <= BINS; g += ST) s_cnt[g] = 0;
      if (tid == 0) *s_nbig = 0;
      nbar_sync(kBarSort, ST);
      const uint32_t s = sg.len;
      const uint32_t nv = s > (uint32_t)tid ? (s - tid + ST - 1) / ST : 0u;  // (item j exists iff j < nv)
      const uint64_t* tp = (sg.parity ? t1 : t0) + sg.start;
      const uint32_t* ip = (sg.parity ? i1 : i0) + sg.start;
      const bool on_idx = sg.depth >= kKeyBytes;
      const uint32_t avail = on_idx ? 8u * (14u - sg.depth) : 8u * (kKeyBytes - sg.depth);
      uint32_t bits = s > 1 ? 32u - __clz(s - 1) : 0u;
      bits = min(bits, (uint32_t)tu.kd_digit_bits);
      bits = min(bits, avail);
      bits = min(bits, 31u - __clz(BINS));
      const uint32_t shift = avail - bits;
      const uint32_t nb = 1u << bits;
      const uint32_t mask = nb - 1;
      auto digit2 = [&](uint64_t t, uint32_t x) -> uint32_t {
        return bits ? (on_idx ? (x >> shift) & mask : (uint32_t)(t >> shift) & mask) : 0u;
      };
      uint64_t tr[ITEMS];
      uint32_t xr[ITEMS], rr[ITEMS];
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const uint32_t i = j * ST + tid;
        if (i < s) {  // (L2 loads: in the fused form other SMs wrote these pairs during this kernel)
          tr[j] = __ldcg(tp + i);
          xr[j] = __ldcg(ip + i);
        }
      }
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if (j < nv) rr[j] = atomicAdd(&s_cnt[digit2(tr[j], xr[j])], 1u);
      }
      nbar_sync(kBarSort, ST);
      {
        const uint32_t per = (nb + ST - 1) / ST;
        const uint32_t g0 = tid * per, g1 = min(nb, g0 + per);
        uint32_t sum = 0;
        for (uint32_t g = g0; g < g1; ++g) sum += s_cnt[g];
        uint32_t run = group_excl_scan<ST>(sum, s_tmp, tid, kBarSort);
        for (uint32_t g = g0; g < g1; ++g) {
          const uint32_t c = s_cnt[g];
          s_cnt[g] = run;
          run += c;
        }
        if (tid == 0) s_cnt[nb] = s;
      }
      nbar_sync(kBarSort, ST);
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if (j < nv) {
          const uint32_t b = s_cnt[digit2(tr[j], xr[j])];
          s_tail[b + rr[j]] = tr[j];
          s_idx[b + rr[j]] = xr[j];
        }
      }
      nbar_sync(kBarSort, ST);
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if (j < nv) {
          const uint32_t d = digit2(tr[j], xr[j]);
          const uint32_t b = s_cnt[d], sz = s_cnt[d + 1] - b;
          if (sz == 1) {
            s_perm[b] = xr[j];
          } else if (sz <= (uint32_t)tu.kd_insert_max) {
            uint32_t rank = 0;
            const uint32_t self = b + rr[j];
            for (uint32_t m = b; m < b + sz; ++m)
              if (m != self) rank += pair_less(s_tail[m], s_idx[m], tr[j], xr[j]) ? 1u : 0u;
            s_perm[b + rank] = xr[j];
          } else if (rr[j] == 0) {
            s_bigl[atomicAdd(s_nbig, 1u)] = d;
          }
        }
      }
      nbar_sync(kBarSort, ST);
      const uint32_t nbig = *s_nbig;
      for (uint32_t qq = warp; qq < nbig; qq += SW) {
        const uint32_t g = s_bigl[qq];
        const uint32_t b = s_cnt[g], e = s_cnt[g + 1];
        warp_bitonic_smem(s_tail, s_idx, b, e);
        for (uint32_t i = b + (tid & 31); i < e; i += 32) s_perm[i] = s_idx[i];
      }
      if (!FUSED && tu.kd_claim && tid == 0) s_claim[3] = nxt;
      nbar_sync(kBarSort, ST);
      if (perm)
        for (uint32_t i = tid; i < s; i += ST) perm[sg.start + i] = s_perm[i];
      if (tid == 0) s_desc[q] = make_uint2(sg.start, s);
      __threadfence_block();
      nbar_arrive(kBarFull + q, NT);  // bucket k is in slot q
    }
    if constexpr (FUSED) {  // the split's remaining chunks: the other tiers' buckets (later kernels) need them
      if (!tu.kc_corun)
        for (uint32_t c = claim_chunk(); c != ~0u; c = claim_chunk()) kc_chunk<ST, (kChunk + ST - 1) / ST, Group>(kc, c, smem);
    }
    // end marker for the gather group, then consume its last releases so no barrier keeps pending arrivals
    {
      const int q = k & 1;
      if (k >= 2) nbar_sync(kBarEmpty + q, NT);
      if (tid == 0) s_desc[q] = make_uint2(0u, kEndDesc);
      __threadfence_block();
      nbar_arrive(kBarFull + q, NT);
      for (uint32_t kk = k >= 2 ? k - 1 : 0; kk < k; ++kk) nbar_sync(kBarEmpty + (kk & 1), NT);
    }
  } else {
    // ================================================================ gather group
    const int gw = (tid - ST) >> 5, lane = tid & 31;
    uint8_t* stage = smem + L::kStage + (size_t)gw * 2 * kWsStageBytes;
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
    const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(smem + L::kMbar + (size_t)gw * 16);
    if (lane < 2) mbar_init(mb0 + 8 * lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t phases = 0;
    for (uint32_t k = 0;; ++k) {
      const int q = k & 1;
      nbar_sync(kBarFull + q, NT);
      const uint2 d = s_desc[q];
      if (d.y == kEndDesc) break;
      const uint32_t* pr = s_ring + q * CAP;
      const uint32_t len = d.y;
      uint8_t* ob = out + (uint64_t)d.x * kRecordBytes;
      auto issue = [&](uint32_t g0, int st) {
        const uint32_t cnt = min((uint32_t)kGroup, len - g0);
        const uint32_t p = lane < (int)cnt ? pr[g0 + lane] : 0u;
        const bool tma = lane < (int)cnt && p < n4;
        const uint32_t ntma = __popc(__ballot_sync(0xffffffffu, tma));
        if (lane == 0) mbar_expect_tx(mb0 + 8 * st, ntma * kWindow);
        __syncwarp();
        if (tma && !tu.ws_tma) {
          bulk_g2s(stage_s + st * kWsStageBytes + lane * kWsSlot, in + (((uint64_t)p * kRecordBytes) & ~uint64_t(15)),
                   kWindow, mb0 + 8 * st);
        } else if (tma) {
          tma_window(stage_s + st * kWsStageBytes + lane * kWsSlot, &in_map, p, mb0 + 8 * st);
        } else if (lane < (int)cnt) {  // one of the last n mod 4 records (outside the map): exact word loads
          const uint32_t* src = reinterpret_cast<const uint32_t*>(in + (uint64_t)p * kRecordBytes);
          uint32_t* dst = reinterpret_cast<uint32_t*>(stage + st * kWsStageBytes + lane * kWsSlot + ((p * 4u) & 15u));
#pragma unroll 5
          for (int o = 0; o < kRecordWords; ++o) dst[o] = src[o];
        }
      };
      const uint32_t first = (uint32_t)gw * kGroup, stride = (uint32_t)GW * kGroup;
      int st = 0;
      if (first < len) issue(first, 0);
      for (uint32_t g0 = first; g0 < len; g0 += stride) {
        const uint32_t gn = g0 + stride;
        if (gn < len) issue(gn, st ^ 1);
        mbar_wait(mb0 + 8 * st, (phases >> st) & 1u);
        phases ^= 1u << st;
        __syncwarp();
        const uint32_t cnt = min((uint32_t)kGroup, len - g0);
        const uint8_t* sb = stage + st * kWsStageBytes;
        uint32_t* dst = reinterpret_cast<uint32_t*>(ob + (uint64_t)g0 * kRecordBytes);
        if (cnt == (uint32_t)kGroup) {  // unrolled, as group_store: word w of record r at 4 w + 28 r + off_r
          const uint32_t xl = (uint32_t)(kWsSlot - kRecordBytes) * lane + ((pr[g0 + lane] * 4u) & 15u);
          const uint8_t* sbl = sb + 4 * lane;
          uint32_t* dl = dst + lane;
#pragma unroll
          for (int i = 0; i < kRecordWords; ++i) {
            const uint32_t r = ((lane + 32u * i) * 1311u) >> 15;  // == (lane + 32 i) / 25 for all w < 800
            const uint32_t x = __shfl_sync(0xffffffffu, xl, r);
            stg_cs_u32(dl + 32 * i, *reinterpret_cast<const uint32_t*>(sbl + 128 * i + x));
          }
        } else {
          const uint32_t words = cnt * kRecordWords;
          for (uint32_t w = lane; w < words; w += 32) {
            const uint32_t r = w / kRecordWords, o = w - r * kRecordWords;
            const uint32_t off = (pr[g0 + r] * 4u) & 15u;
            stg_cs_u32(dst + w, *reinterpret_cast<const uint32_t*>(sb + r * kWsSlot + off + 4 * o));
          }
        }
        if (DG && lane < (int)cnt)
          dg[d.x + g0 + lane] =
              prefix_digest(reinterpret_cast<const uint32_t*>(sb + lane * kWsSlot + ((pr[g0 + lane] * 4u) & 15u)));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        st ^= 1;
      }
      nbar_arrive(kBarEmpty + q, NT);  // slot q may be refilled
    }
  }
}

template <uint32_t CAP, int ST, int GW, bool DG>
cudaError_t launch_ws_sort(const Seg* list, const uint32_t* count, const uint64_t* t0, const uint32_t* i0,
                           const uint64_t* t1, const uint32_t* i1, uint32_t* perm, const Tunables& tu, int sms,
                           const uint8_t* in, uint64_t n_in, uint8_t* out, uint64_t* dg, cudaStream_t s,
                           const KcArgs* kc = nullptr) {
  CUtensorMap map;  // the record windows of tma_window: boxes of 7 rows x 1 group (tmap.cu)
  cudaError_t me = record_group_map(&map, in, n_in, 7, 1);
  if (me != cudaSuccess) return me;
  auto kern = kc ? kd_ws_sort<CAP, ST, GW, DG, true> : kd_ws_sort<CAP, ST, GW, DG, false>;
  const size_t smem = WsLayout<CAP, ST, GW>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ST + 32 * GW, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  return launch_k(kern, sms * per_sm, ST + 32 * GW, smem, s, tu.pdl != 0, list, count, t0, i0, t1, i1, perm, tu, map, in,
                  n_in & ~uint64_t(3), out, dg, kc ? *kc : KcArgs{});
}

}  // namespace

namespace {
// All K-d/K-e tiers for the lists of one level (counts are read on the device; no host sync).
template <bool DG>
cudaError_t kd_all(const ListSet& kd, const uint64_t* t0, const uint32_t* i0, const uint64_t* t1, const uint32_t* i1,
                   uint32_t* perm, const Tunables& tu0, int sms, const uint8_t* in, uint64_t n_in, uint8_t* out,
                   uint64_t* dg, cudaStream_t s, int* launches, const KcArgs* kc, int fused_tier) {
  const uint64_t in_bytes = n_in * kRecordBytes;
  static int warp_per_sm = 0;  // resident CTAs per SM (registers bound it: 5 at 46 registers)
  if (!warp_per_sm && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&warp_per_sm, kd_warp_sort<DG>, 256, 0) != cudaSuccess ||
                       warp_per_sm < 1))
    warp_per_sm = 4;
  // tier t's kernel; with split != nullptr the fused form (it also runs the level-1 split, and claims its
  // buckets itself instead of reading list t)
  // PDL modes (common.cuh): the first tier waits for the split/classification, later ones overlap it (their
  // lists, pairs and output ranges are disjoint) — except around a fused tier, whose split the others need.
  int nlaunched = 0;
  auto tier_launch = [&](int t, const KcArgs* split) -> cudaError_t {
    Tunables tu = tu0;
    tu.pdl = !tu0.pdl ? 0 : (nlaunched++ == 0 || kc || tu0.pdl == 1) ? 1 : 2;
    // co-run: the fused tier becomes resident beside the running split kernel (launched with PDL, no entry
    // wait: its bucket waits on done[] order it after the split; it waits for the split's completion only
    // at exit, so the tiers after it still find the split complete)
    if (split && tu0.kc_corun) tu.pdl = 2;
    switch (t) {
      case kListWarp:
        return launch_k(kd_warp_sort<DG>, sms * warp_per_sm, 256, 0, s, tu.pdl != 0, kd.items[kListWarp],
                        kd.counts + kListWarp, t0, i0, t1, i1, perm, in, out, dg, tu.pdl);
      // (the warp-specialised form loses on small buckets: a ~100-record bucket keeps only 3 of its gather
      // warps busy and the ring hand-off dominates — measured C3 level 3: 17.0 vs 12.3 ms)
      case kListMed1:
        return launch_cta_sort<512, 128, DG>(kd.items[kListMed1], kd.counts + kListMed1, t0, i0, t1, i1, perm, tu, sms, in,
                                             in_bytes, out, dg, s);
      case kListMed2:
        if (tu.kd_ws && out)  // (no gather warps to feed in perm-only mode)
          return launch_ws_sort<2048, 256, 8, DG>(kd.items[kListMed2], kd.counts + kListMed2, t0, i0, t1, i1, perm, tu, sms,
                                                  in, n_in, out, dg, s, split);
        return launch_cta_sort<2048, 256, DG>(kd.items[kListMed2], kd.counts + kListMed2, t0, i0, t1, i1, perm, tu, sms, in,
                                              in_bytes, out, dg, s, split, kListMed2);
      case kListMed3:
        return launch_cta_sort<8192, 1024, DG>(kd.items[kListMed3], kd.counts + kListMed3, t0, i0, t1, i1, perm, tu, sms, in,
                                               in_bytes, out, dg, s, split, kListMed3);
      case kListMed4:
        return launch_cta_sort<10240, 1024, DG>(kd.items[kListMed4], kd.counts + kListMed4, t0, i0, t1, i1, perm, tu, sms,
                                                in, in_bytes, out, dg, s, split, kListMed4);
      default:
        return launch_cta_sort<16384, 768, DG>(kd.items[kListMed5], kd.counts + kListMed5, t0, i0, t1, i1, perm, tu, sms,
                                               in, in_bytes, out, dg, s, split, kListMed5);
    }
  };
  cudaError_t e;
  const bool fused = kc && fused_tier >= kListMed2 && fused_tier < kNumKdLists;
  if (fused && (e = tier_launch(fused_tier, kc)) != cudaSuccess) return e;  // first: the split is done when it ends
  for (int t = 0; t < kNumKdLists; ++t)
    if (!(fused && t == fused_tier) && (e = tier_launch(t, nullptr)) != cudaSuccess) return e;
  if (launches) *launches += 6;
  return cudaSuccess;
}
}  // namespace

cudaError_t launch_kd_all(const ListSet& kd, const uint64_t* t0, const uint32_t* i0, const uint64_t* t1,
                          const uint32_t* i1, uint32_t* perm, const Tunables& tu, int sms, const uint8_t* in,
                          uint64_t n_in, uint8_t* out, uint64_t* dg, cudaStream_t s, int* launches, const KcArgs* kc,
                          int fused_tier) {
  return dg && out ? kd_all<true>(kd, t0, i0, t1, i1, perm, tu, sms, in, n_in, out, dg, s, launches, kc, fused_tier)
                   : kd_all<false>(kd, t0, i0, t1, i1, perm, tu, sms, in, n_in, out, nullptr, s, launches, kc, fused_tier);
}

}  // namespace ley
