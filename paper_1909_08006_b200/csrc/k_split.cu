// k_split.cu — K-c / K-c': stable segmented scatter of (key-tail, index) pairs into MSB buckets.
//
// PAPER.md §3.1 line 96 (cache-aware scattering: "we then scatter the keys to their bucket offsets by
// copying from the key to the tmp array ... this scattering process takes the most time in radix sort")
// and Algorithm 1 lines 59-63 (after the first round every bucket is split again on the next radix;
// "if k > bigBucketThreshold then MSDRadixSort(key, radix + 1, k)"). SURVEY.md §8a rows a3 and a4.
//
// K-c (level 1): byte-0 bucket b is the concatenation of the byte-0 runs K-a left in every tile. Each
// CTA takes kChunk-pair chunks of one bucket (persistent, ticketed), gathers a chunk from the runs, ranks
// it by key byte 1 (shared-memory atomics), claims each digit's slice of its 16-bit bucket with one global
// atomic on that bucket's fill cursor (initialised to B16), stages the pairs in shared memory in digit
// order and writes them out as coalesced runs. Output pair: tail = key bytes 2..9 big-endian (u64),
// idx = global ordinal (u32).
//
// The order inside a bucket is whatever the atomics produce: it does not matter, because every later
// step orders by the composite (key bytes, ordinal) — the ordinal is the least significant part of the
// sort key, which is what makes the result the stable sort. No look-back is needed.
//
// K-c' (level >= 2): the same on contiguous big buckets, digit = key byte `depth` (depth 10..13: byte
// depth-10 of the big-endian ordinal, for buckets whose 10 key bytes are all equal); the bucket's
// digit histogram comes from kr_hist and its children are classified by kr_plan before the split.
#include "block_rank.cuh"
#include "classify.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

constexpr int kThreads = kSplitThreads;
constexpr int kItems = kSplitItems;
constexpr int kWarps = kThreads / 32;

struct SplitSmem {
  static constexpr size_t kRegionA = (size_t)kChunk * 13 + 16;          // tails u64 + idx u32 + digit u8
  static constexpr size_t kRuns = (size_t)(kChunk + 1) * 8;              // run_v u32 + run_src u32
  static constexpr size_t kRegion = kRegionA > kRuns ? kRegionA : kRuns;
  static constexpr size_t kWh = (size_t)kWarps * kRadix * 4;
  static constexpr size_t kBytes = kRegion + kWh + 256 * 4 + 64 * 4;
};

// largest i in [lo, hi) with a[i] <= v (a non-decreasing, a[lo] <= v)
__device__ __forceinline__ uint64_t search_le_g(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t v) {
  while (hi - lo > 1) {
    uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid; else hi = mid;
  }
  return lo;
}

// Largest t in [lo, hi) with a[t] <= v (a non-decreasing, a[lo] <= v), galloping out from the guess g: a
// good guess (the tiles are equal-sized, so a byte-0 run's start grows about linearly in t) costs 2-4
// dependent loads instead of log2(hi - lo).
__device__ __forceinline__ uint64_t search_le_guess(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t v, uint64_t g) {
  g = g < lo ? lo : (g >= hi ? hi - 1 : g);
  uint64_t l, h;  // invariant target: a[l] <= v, (h == hi or a[h] > v)
  if (a[g] <= v) {
    l = g;
    uint64_t step = 1;
    h = l + step;
    while (h < hi && a[h] <= v) {
      l = h;
      step <<= 1;
      h = l + step;
    }
    if (h > hi) h = hi;
  } else {
    h = g;
    uint64_t step = 1;
    l = h > lo + step ? h - step : lo;
    while (l > lo && a[l] > v) {
      h = l;
      step <<= 1;
      l = h > lo + step ? h - step : lo;
    }
  }
  return search_le_g(a, l, h, v);
}

// Per-chunk decomposition of level 1, one thread per chunk: segment b, virtual range [v0, v0+cnt), the
// tile range [t0, t1] whose byte-0 runs cover it, and the segment's first chunk k0. Parallel searches
// here keep them off the K-c critical path. Every CTA first derives the chunk starts itself (byte-0
// segment b = [B16[256 b], B16[256 (b+1)]) is cut into ceil(len / kChunk) chunks; cstart = exclusive
// scan of the chunk counts; CTA 0 publishes them). With `order` non-null it also writes the chunks'
// processing order (kOrderGroup, below). (The split's fill cursors = B16 are written by the K-b scan.)
// 256 threads per CTA.
constexpr int kOrderGroup = 4;
__global__ void __launch_bounds__(256)
    kc_plan_level1(const uint32_t* __restrict__ off, uint32_t tiles, const uint32_t* __restrict__ B16, uint64_t n,
                   uint32_t* __restrict__ cstart, uint32_t grid_ub, uint4* __restrict__ plan_a,
                   uint2* __restrict__ plan_b, uint32_t* __restrict__ order, const ClassifyJob cj, uint32_t pblocks) {
  __shared__ uint32_t s_cst[257];
  __shared__ uint32_t s_tmp[32];
  if (blockIdx.x >= pblocks) {  // the classification CTAs (they run beside the planning ones)
    classify_level1_block(cj, blockIdx.x - pblocks, s_tmp);
    return;
  }
  {
    const uint32_t b = threadIdx.x;
    const uint64_t beg = B16[b * 256], end = (b < 255) ? B16[(b + 1) * 256] : n;
    const uint32_t nch = (uint32_t)((end - beg + kChunk - 1) / kChunk);
    uint32_t total;
    const uint32_t ex = block_excl_scan<256>(nch, s_tmp, &total);
    s_cst[b] = ex;
    if (b == 0) s_cst[256] = total;
    if (blockIdx.x == 0) {
      cstart[b] = ex;
      if (b == 0) cstart[256] = total;
    }
  }
  const uint32_t nth = pblocks * blockDim.x;
  __syncthreads();
  const uint32_t kend = min(s_cst[256], grid_ub);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < kend; k += nth) {
    uint32_t b = 0, hi = 256;
    while (hi - b > 1) {
      uint32_t mid = (b + hi) >> 1;
      if (s_cst[mid] <= k) b = mid; else hi = mid;
    }
    const uint32_t c = k - s_cst[b];
    const uint32_t seg_beg = B16[b * 256];
    const uint64_t seg_end = (b < 255) ? B16[(b + 1) * 256] : n;
    const uint32_t v0 = seg_beg + c * kChunk;
    const uint32_t cnt = (uint32_t)(seg_end - v0 < kChunk ? seg_end - v0 : kChunk);
    const uint32_t* off_b = off + (uint64_t)b * tiles;
    const uint64_t len = seg_end - seg_beg;
    // (two independent searches, so their load chains overlap)
    const uint32_t t0 = (uint32_t)search_le_guess(off_b, 0, tiles, v0, (uint64_t)(v0 - seg_beg) * tiles / len);
    const uint32_t t1 =
        (uint32_t)search_le_guess(off_b, 0, tiles, v0 + cnt - 1, (uint64_t)(v0 + cnt - 1 - seg_beg) * tiles / len);
    plan_a[k] = make_uint4(b, v0, cnt, k - c);
    plan_b[k] = make_uint2(t0, t1);
    if (order) {  // position of chunk c of bucket j of its group in the interleaved order
      const uint32_t g0 = b & ~(uint32_t)(kOrderGroup - 1), j = b - g0;
      uint32_t pos = s_cst[g0];
#pragma unroll
      for (uint32_t q = 0; q < (uint32_t)kOrderGroup; ++q) {
        const uint32_t nq = s_cst[g0 + q + 1] - s_cst[g0 + q];
        pos += min(c, nq) + (q < j && nq > c ? 1u : 0u);
      }
      order[pos] = k;
    }
  }
}

// Processing order of the level-1 chunks (written by kc_plan_level1): bucket-major, but the chunks of
// kOrderGroup = 4 neighbouring byte-0 buckets interleaved (chunk c of buckets 4g..4g+3, then chunk c+1,
// ...). A tile's runs of neighbouring buckets share their boundary lines; interleaving reads both sides of
// most boundaries while the line is still in L2 once K-a's output outgrows the L2 (C4: a boundary line
// would otherwise be fetched twice, ~1/256 of the pass apart), and keeps the writes to 1024 active 16-bit
// buckets.
constexpr uint64_t kInterleaveMinRecords = 300000000;

constexpr uint32_t kMaxRuns = (uint32_t)((kChunk * 13 + 16) / 8);  // run table fits the staging region

__global__ void __launch_bounds__(kThreads, kSplitMinBlocks)
    kc_split_level1(const uint64_t* __restrict__ k1_in, const uint32_t* __restrict__ w_in, uint32_t tiles,
                    const uint32_t* __restrict__ off /*[256*tiles+1]*/, const uint32_t* __restrict__ lo,
                    const uint32_t* __restrict__ B16, const uint32_t* __restrict__ cstart,
                    const uint4* __restrict__ plan_a, const uint2* __restrict__ plan_b,
                    const uint32_t* __restrict__ order, uint32_t* __restrict__ cursor, uint32_t* __restrict__ ticket,
                    uint64_t* __restrict__ tail_out, uint32_t* __restrict__ idx_out, uint32_t* __restrict__ done) {
  extern __shared__ __align__(16) uint8_t smem[];
  // co-run form (done != null, internal.cu): every CTA is resident before the fused K-d+K-e tier launches
  // beside it (PDL); each finished chunk is published in done[b] for that kernel's bucket waits
  if (done) pdl_trigger();
  uint8_t* region = smem;
  uint32_t* s_wh = reinterpret_cast<uint32_t*>(smem + SplitSmem::kRegion);
  uint32_t* s_dst = s_wh + kWarps * kRadix;
  uint32_t* s_misc = s_dst + 256;  // [0..31] scan tmp, [32..] scalars
  uint32_t* s_off = reinterpret_cast<uint32_t*>(region);  // run table (load phase)
  uint32_t* s_lo = s_off + kMaxRuns;
  uint64_t* s_tail = reinterpret_cast<uint64_t*>(region);  // staging (scatter phase)
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_tail + kChunk);
  uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_idx + kChunk);
  const uint32_t total = cstart[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  // persistent: chunks are claimed by ticket (thread 0), one chunk ahead — the next ticket and its plan are
  // fetched while the current chunk is processed, and every thread prefetches its entry of the next chunk's
  // run table during the write-out, so neither latency sits between chunks (no look-back: any order works).
  for (int q = threadIdx.x; q < kRadix; q += kThreads) s_wh[q] = 0;  // (block_rank_atomic: pre-zeroed)
  if (threadIdx.x == 0) {  // the first chunk
    const uint32_t k = atomicAdd(ticket, 1u);
    s_misc[40] = k;
    if (k < total) {
      const uint32_t kk = order ? order[k] : k;
      const uint4 pa = plan_a[kk];
      const uint2 pb = plan_b[kk];
      s_misc[41] = pa.x;
      s_misc[42] = pa.y;
      s_misc[43] = pa.z;
      s_misc[46] = pa.w;
      s_misc[44] = pb.x;
      s_misc[45] = pb.y;
    }
  }
  __syncthreads();
  uint32_t pf_vs = 0, pf_lo = 0;  // this thread's run-table entry of the current chunk, if prefetched
  bool pf = false;
  while (true) {
    const uint32_t k = s_misc[40];
    if (k >= total) return;
    const uint32_t b = s_misc[41], v0 = s_misc[42], cnt = s_misc[43], t0 = s_misc[44], t1 = s_misc[45];
    const uint32_t R = t1 - t0 + 1;
    const uint32_t* off_b = off + (uint64_t)b * tiles;
    const bool table = R <= kMaxRuns / 2;
    __syncthreads();  // everyone has the plan: thread 0 may fetch the next one into s_misc[40..46]
    uint32_t nxt[7];
    if (threadIdx.x == 0) {  // issued now, stored to shared memory once the chunk's run table is dead
      nxt[0] = atomicAdd(ticket, 1u);
      if (nxt[0] < total) {
        const uint32_t kk = order ? order[nxt[0]] : nxt[0];
        const uint4 pa = plan_a[kk];
        const uint2 pb = plan_b[kk];
        nxt[1] = pa.x;
        nxt[2] = pa.y;
        nxt[3] = pa.z;
        nxt[6] = pa.w;
        nxt[4] = pb.x;
        nxt[5] = pb.y;
      }
    }
    uint32_t src[kItems];  // position of each element in K-a's output
    if (table) {
      // run table (virtual start, source base: src = base + v) and run-start marks; an inclusive
      // max-scan of the marks gives every element of the chunk its run without any search
      uint16_t* s_mark = reinterpret_cast<uint16_t*>(s_off + kMaxRuns / 2);
      for (uint32_t e = threadIdx.x; e < cnt; e += kThreads) s_mark[e] = 0;
      for (uint32_t i = threadIdx.x; i < R; i += kThreads) {
        uint32_t vs, lv;
        if (pf && i == threadIdx.x) {
          vs = pf_vs;
          lv = pf_lo;
        } else {
          vs = off_b[t0 + i];
          lv = lo[(uint64_t)(t0 + i) * kRadix + b];
        }
        s_off[i] = vs;
        s_lo[i] = ((t0 + i) << kTileLog2) + lv - vs;
      }
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < R; i += kThreads) {
        const uint32_t vs = s_off[i], ve = (i + 1 < R) ? s_off[i + 1] : off_b[t1 + 1];
        const uint32_t e = vs > v0 ? vs - v0 : 0u;
        if (ve > vs && e < cnt) s_mark[e] = (uint16_t)i;
      }
      __syncthreads();
      {
        constexpr int PER = kChunk / kThreads;  // 8 consecutive marks per thread
        const uint32_t e0 = threadIdx.x * PER;
        uint32_t m[PER], run = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          m[q] = e0 + q < cnt ? s_mark[e0 + q] : 0u;
          run = max(run, m[q]);
          m[q] = run;
        }
        const uint32_t pre = block_excl_max<kThreads, false>(run, s_misc);  // (barrier below)
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (e0 + q < cnt) s_mark[e0 + q] = (uint16_t)max(pre, m[q]);
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        uint32_t e = warp * (32 * kItems) + j * 32 + lane;
        src[j] = e < cnt ? s_lo[s_mark[e]] + v0 + e : 0u;
      }
    } else {  // very sparse bucket: search the global run table directly
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        uint32_t e = warp * (32 * kItems) + j * 32 + lane;
        uint32_t v = v0 + e;
        src[j] = 0;
        if (e < cnt) {
          uint32_t t = (uint32_t)search_le_g(off_b, t0, (uint64_t)t1 + 1, v);
          src[j] = (t << kTileLog2) + lo[(uint64_t)t * kRadix + b] + (v - off_b[t]);
        }
      }
    }
    uint64_t k1[kItems];
    uint32_t w[kItems], dig[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      uint32_t e = warp * (32 * kItems) + j * 32 + lane;
      if (e < cnt) {
        k1[j] = k1_in[src[j]];
        w[j] = w_in[src[j]];
      } else {
        k1[j] = 0;
        w[j] = 0;
      }
      dig[j] = (uint32_t)(k1[j] >> 56);
    }
    __syncthreads();  // run tables dead from here on
    if (threadIdx.x == 0) {
      s_misc[40] = nxt[0];
      if (nxt[0] < total)
        for (int q = 1; q < 7; ++q) s_misc[40 + q] = nxt[q];
    }

    uint32_t pos[kItems], total_d, excl_d;
        block_rank_atomic<kThreads, kItems, true>(dig, cnt, pos, s_wh, s_misc, total_d, excl_d);
    // each digit's slice of its 16-bit bucket: the atomic's round trip overlaps the staging scatter below
    static_assert(kThreads == kRadix, "one digit per thread");
    const uint32_t dbase = total_d ? atomicAdd(&cursor[b * 256 + threadIdx.x], total_d) : 0u;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      uint32_t e = warp * (32 * kItems) + j * 32 + lane;
      if (e < cnt) {
        uint32_t p = pos[j];
        s_tail[p] = (k1[j] << 8) | (w[j] >> 24);
        s_idx[p] = (src[j] & ~(kTileRecords - 1)) | (w[j] & 0xFFFFFFu);
        s_dig[p] = (uint8_t)dig[j];
      }
    }
    s_dst[threadIdx.x] = dbase - excl_d;
    __syncthreads();
    // the next chunk's plan is in s_misc[40..46]: prefetch this thread's run-table entry while writing
    pf = false;
    {
      const uint32_t kn = s_misc[40];
      if (kn < total) {
        const uint32_t bn = s_misc[41], tn0 = s_misc[44], Rn = s_misc[45] - tn0 + 1;
        if (Rn <= kMaxRuns / 2 && threadIdx.x < Rn) {
          pf_vs = off[(uint64_t)bn * tiles + tn0 + threadIdx.x];
          pf_lo = lo[(uint64_t)(tn0 + threadIdx.x) * kRadix + bn];
          pf = true;
        }
      }
    }
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
      uint32_t g = s_dst[s_dig[i]] + i;
      tail_out[g] = s_tail[i];
      idx_out[g] = s_idx[i];
    }
    for (int q = threadIdx.x; q < kRadix; q += kThreads) s_wh[q] = 0;  // the next chunk's rank histogram
    __syncthreads();  // staging reused by the next chunk; every store of this chunk issued
    if (done && threadIdx.x == 0) {
      __threadfence();  // cumulative over the CTA's stores ordered by the barrier above
      atomicAdd(&done[b], 1u);
    }
  }
}

// ------------------------------------------------------------------------------------ level >= 2
// chunk -> segment of the current big list
__device__ __forceinline__ uint32_t chunk_segment(const uint32_t* cstart, uint32_t nseg, uint32_t k) {
  uint32_t s = 0, hi = nseg;
  while (hi - s > 1) {
    uint32_t mid = (s + hi) >> 1;
    if (cstart[mid] <= k) s = mid; else hi = mid;
  }
  return s;
}

// Digit `depth` of the composite sort key (key bytes 0..9, then the big-endian ordinal as bytes 10..13):
// tail = key bytes 2..9, so byte d < 10 is (tail >> 8 (9 - d)); bytes 10..13 come from the ordinal.
__device__ __forceinline__ uint32_t digit_at(uint64_t tail, uint32_t idx, uint32_t depth) {
  return depth < 10 ? (uint32_t)(tail >> (8 * (9 - depth))) & 0xFFu : (idx >> (8 * (13 - depth))) & 0xFFu;
}

__global__ void kr_nchunks(const Seg* __restrict__ segs, uint32_t nseg, uint32_t* __restrict__ nch) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) nch[s] = (segs[s].len + kChunk - 1) / kChunk;
}

// chunk -> (segment, chunk inside it), one thread per chunk: the binary searches run in parallel here
// instead of one dependent chain of global loads per chunk inside kr_hist / kr_split
__global__ void kr_chunk_map(const uint32_t* __restrict__ cstart, uint32_t nseg, uint32_t ub, uint2* __restrict__ map) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ub || k >= cstart[nseg]) return;
  const uint32_t s = chunk_segment(cstart, nseg, k);
  map[k] = make_uint2(s, k - cstart[s]);
}

__global__ void __launch_bounds__(256)
    kr_hist(const Seg* __restrict__ segs, uint32_t nseg, const uint32_t* __restrict__ cstart, uint32_t nchunks_total_ub,
            const uint64_t* __restrict__ tails0, const uint32_t* __restrict__ idx0, const uint64_t* __restrict__ tails1,
            const uint32_t* __restrict__ idx1, uint32_t* __restrict__ seg_hist, const uint2* __restrict__ map) {
  __shared__ uint32_t h[kRadix];
  const uint32_t total = cstart[nseg];
  for (uint32_t k = blockIdx.x; k < total; k += gridDim.x) {
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint2 m = map[k];
    const uint32_t s = m.x, c = m.y;
    Seg sg = segs[s];
    uint32_t beg = c * kChunk, end = min(sg.len, beg + kChunk);
    if (sg.depth < 10) {
      const uint64_t* t = (sg.parity ? tails1 : tails0) + sg.start;
      for (uint32_t i = beg + threadIdx.x; i < end; i += 256) atomicAdd(&h[digit_at(t[i], 0, sg.depth)], 1u);
    } else {
      const uint32_t* x = (sg.parity ? idx1 : idx0) + sg.start;
      for (uint32_t i = beg + threadIdx.x; i < end; i += 256) atomicAdd(&h[digit_at(0, x[i], sg.depth)], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&seg_hist[(uint64_t)s * kRadix + threadIdx.x], h[threadIdx.x]);
    __syncthreads();
  }
  (void)nchunks_total_ub;
}

// One CTA (256 threads) per big segment: bucket offsets (also the fill cursors of kr_split), children,
// constant-digit skip.
__global__ void __launch_bounds__(256)
    kr_plan(const Seg* __restrict__ segs, uint32_t nseg, const uint32_t* __restrict__ seg_hist,
            uint32_t* __restrict__ seg_excl, uint8_t* __restrict__ noscatter, Tunables tu, ListSet kd,
            Seg* __restrict__ big_out, uint32_t* __restrict__ big_count) {
  __shared__ uint32_t s_tmp[32];
  __shared__ uint32_t s_cnt[16];
  __shared__ uint32_t s_single;
  const uint32_t s = blockIdx.x;
  const Seg sg = segs[s];
  const int d = threadIdx.x;
  uint32_t h = seg_hist[(uint64_t)s * kRadix + d];
  if (d == 0) s_single = 0;
  __syncthreads();
  if (h == sg.len) s_single = 1;  // one digit holds the whole bucket: nothing to move
  uint32_t ex = block_excl_scan<256>(h, s_tmp, nullptr);
  seg_excl[(uint64_t)s * kRadix + d] = ex;
  const bool single = s_single != 0;
  if (d == 0) noscatter[s] = single ? 1 : 0;
  const Seg ch = single ? Seg{sg.start, sg.len, sg.depth + 1, sg.parity}
                        : Seg{sg.start + ex, h, sg.depth + 1, sg.parity ^ 1u};
  classify_block(ch, single ? d == 0 : h != 0, tu, kd, big_out, big_count, s_cnt);
}

__global__ void __launch_bounds__(kThreads, kSplitMinBlocks)
    kr_split(const Seg* __restrict__ segs, uint32_t nseg, const uint32_t* __restrict__ cstart,
             uint32_t* __restrict__ cursor, const uint8_t* __restrict__ noscatter, uint64_t* tails0, uint32_t* idx0,
             uint64_t* tails1, uint32_t* idx1, uint32_t* __restrict__ ticket, const uint2* __restrict__ map) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* s_tail = reinterpret_cast<uint64_t*>(smem);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_tail + kChunk);
  uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_idx + kChunk);
  uint32_t* s_wh = reinterpret_cast<uint32_t*>(smem + SplitSmem::kRegion);
  uint32_t* s_dst = s_wh + kWarps * kRadix;
  uint32_t* s_misc = s_dst + 256;
  const uint32_t total = cstart[nseg];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // chunks claimed one ahead (as in kc_split_level1): thread 0 fetches the next ticket and its map entry
  // while this chunk is processed
  for (int q = threadIdx.x; q < kRadix; q += kThreads) s_wh[q] = 0;  // (block_rank_atomic: pre-zeroed)
  if (threadIdx.x == 0) {
    const uint32_t k = atomicAdd(ticket, 1u);
    s_misc[40] = k;
    if (k < total) {
      const uint2 m = map[k];
      s_misc[41] = m.x;
      s_misc[42] = m.y;
    }
  }
  __syncthreads();
  while (true) {
    const uint32_t k = s_misc[40];
    if (k >= total) return;
    const uint32_t s = s_misc[41], c = s_misc[42];
    __syncthreads();  // everyone has the chunk: thread 0 may claim the next
    uint32_t nk = 0;
    uint2 nm = make_uint2(0, 0);
    if (threadIdx.x == 0) {
      nk = atomicAdd(ticket, 1u);
      if (nk < total) nm = map[nk];
    }
    auto publish_next = [&]() {
      if (threadIdx.x == 0) {
        s_misc[40] = nk;
        s_misc[41] = nm.x;
        s_misc[42] = nm.y;
      }
    };
    if (noscatter[s]) {
      publish_next();
      __syncthreads();
      continue;
    }
    const Seg sg = segs[s];
    const uint32_t beg = c * kChunk;
    const uint32_t cnt = min(kChunk, sg.len - beg);
    const uint64_t* tin = (sg.parity ? tails1 : tails0) + sg.start + beg;
    const uint32_t* iin = (sg.parity ? idx1 : idx0) + sg.start + beg;
    uint64_t* tout = (sg.parity ? tails0 : tails1) + sg.start;
    uint32_t* iout = (sg.parity ? idx0 : idx1) + sg.start;

    uint64_t tv[kItems];
    uint32_t iv[kItems], dig[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      uint32_t e = warp * (32 * kItems) + j * 32 + lane;
      if (e < cnt) {
        tv[j] = tin[e];
        iv[j] = iin[e];
      } else {
        tv[j] = 0;
        iv[j] = 0;
      }
      dig[j] = digit_at(tv[j], iv[j], sg.depth);
    }
    uint32_t pos[kItems], total_d, excl_d;
        block_rank_atomic<kThreads, kItems, true>(dig, cnt, pos, s_wh, s_misc, total_d, excl_d);
    publish_next();  // (read after the barrier below, at the top of the next iteration)
    if (threadIdx.x < kRadix) {
      const int d = threadIdx.x;
      const uint32_t base = total_d ? atomicAdd(&cursor[(uint64_t)s * kRadix + d], total_d) : 0u;
      s_dst[d] = base - excl_d;
    }
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      uint32_t e = warp * (32 * kItems) + j * 32 + lane;
      if (e < cnt) {
        uint32_t p = pos[j];
        s_tail[p] = tv[j];
        s_idx[p] = iv[j];
        s_dig[p] = (uint8_t)dig[j];
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
      uint32_t g = s_dst[s_dig[i]] + i;
      tout[g] = s_tail[i];
      iout[g] = s_idx[i];
    }
    for (int q = threadIdx.x; q < kRadix; q += kThreads) s_wh[q] = 0;  // the next chunk's rank histogram
    __syncthreads();
  }
}

}  // namespace

size_t split_smem_bytes() { return SplitSmem::kBytes; }

cudaError_t launch_kc_split_level1(const uint64_t* k1_in, const uint32_t* w_in, uint32_t tiles, const uint32_t* off,
                                   const uint32_t* lo, const uint32_t* B16, uint64_t n, uint32_t* cstart,
                                   uint4* plan_a, uint2* plan_b, uint32_t* order, uint32_t* cursor, uint32_t* ticket,
                                   uint64_t* tail_out, uint32_t* idx_out, uint32_t grid_ub, cudaStream_t s,
                                   const ClassifyJob& cls, bool run_split, const uint32_t** order_used,
                                   uint32_t* done, int corun_per_sm) {
  // the interleaved order pays only once K-a's output is many times the L2 (C4: 30.6 -> ~18 B/pair of
  // reads, K-c 6.7 -> 6.1 ms); below that the plain bucket-major order is as fast or faster (C3 skew)
  if (n < kInterleaveMinRecords) order = nullptr;
  const uint32_t pblocks = std::max<uint32_t>((grid_ub + 255) / 256, 1);
  kc_plan_level1<<<pblocks + kClassifyBlocks, 256, 0, s>>>(off, tiles, B16, n, cstart, grid_ub, plan_a, plan_b, order,
                                                            cls, pblocks);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (order_used) *order_used = order;
  if (!run_split) return cudaSuccess;  // (the fused K-d+K-e kernel runs the chunks: kc_chunk.cuh)
  size_t smem = SplitSmem::kBytes;
  e = cudaFuncSetAttribute(kc_split_level1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 2, dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kc_split_level1, kThreads, smem);
  if (e != cudaSuccess) return e;
  // (co-run: corun_per_sm CTAs per SM leave room for a K-d+K-e tier CTA beside them; the SMs must be
  // configured for the largest shared-memory carveout while the split runs, else the tier's CTAs cannot
  // join them until they drain)
  const bool corun = done && corun_per_sm > 0;
  if (corun && corun_per_sm < per_sm) per_sm = corun_per_sm;
  e = cudaFuncSetAttribute(kc_split_level1, cudaFuncAttributePreferredSharedMemoryCarveout,
                           corun ? (int)cudaSharedmemCarveoutMaxShared : (int)cudaSharedmemCarveoutDefault);
  if (e != cudaSuccess) return e;
  uint32_t grid = (uint32_t)sms * (uint32_t)(per_sm > 0 ? per_sm : 1);
  if (grid > grid_ub) grid = grid_ub;
  kc_split_level1<<<grid, kThreads, smem, s>>>(k1_in, w_in, tiles, off, lo, B16, cstart, plan_a, plan_b, order,
                                               cursor, ticket, tail_out, idx_out, done);
  return cudaGetLastError();
}

cudaError_t launch_kr_nchunks(const Seg* segs, uint32_t nseg, uint32_t* nch, cudaStream_t s) {
  kr_nchunks<<<(nseg + 255) / 256, 256, 0, s>>>(segs, nseg, nch);
  return cudaGetLastError();
}

cudaError_t launch_kr_chunk_map(const uint32_t* cstart, uint32_t nseg, uint32_t ub, uint2* map, cudaStream_t s) {
  kr_chunk_map<<<(ub + 255) / 256, 256, 0, s>>>(cstart, nseg, ub, map);
  return cudaGetLastError();
}

cudaError_t launch_kr_hist(const Seg* segs, uint32_t nseg, const uint32_t* cstart, uint32_t grid,
                           const uint64_t* tails0, const uint32_t* idx0, const uint64_t* tails1, const uint32_t* idx1,
                           uint32_t* seg_hist, const uint2* map, cudaStream_t s) {
  kr_hist<<<grid, 256, 0, s>>>(segs, nseg, cstart, grid, tails0, idx0, tails1, idx1, seg_hist, map);
  return cudaGetLastError();
}

cudaError_t launch_kr_plan(const Seg* segs, uint32_t nseg, const uint32_t* seg_hist, uint32_t* seg_excl,
                           uint8_t* noscatter, const Tunables& tu, const ListSet& kd, Seg* big_out,
                           uint32_t* big_count, cudaStream_t s) {
  kr_plan<<<nseg, 256, 0, s>>>(segs, nseg, seg_hist, seg_excl, noscatter, tu, kd, big_out, big_count);
  return cudaGetLastError();
}

cudaError_t launch_kr_split(const Seg* segs, uint32_t nseg, const uint32_t* cstart, uint32_t* cursor,
                            const uint8_t* noscatter, uint64_t* tails0, uint32_t* idx0, uint64_t* tails1,
                            uint32_t* idx1, uint32_t* ticket, const uint2* map, uint32_t grid_ub, cudaStream_t s) {
  size_t smem = SplitSmem::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kr_split, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 2, dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kr_split, kThreads, smem);
  if (e != cudaSuccess) return e;
  uint32_t grid = (uint32_t)sms * (uint32_t)(per_sm > 0 ? per_sm : 1);
  if (grid > grid_ub) grid = grid_ub;
  kr_split<<<grid, kThreads, smem, s>>>(segs, nseg, cstart, cursor, noscatter, tails0, idx0, tails1, idx1, ticket,
                                        map);
  return cudaGetLastError();
}

}  // namespace ley
