// k_dist.cu — kernels of the multi-GPU key-range sort.
//
// BASELINE.json north_star: "Each GPU histograms the leading key bytes, all GPUs agree on range
// splitters, and records move to their owning GPU by an NCCL all-to-all over NVLink; each GPU then sorts
// its range locally, and the output is the concatenation of the ranges." The paper itself is single-node
// (§3, P:70 threads[40]); this is the B200 extension the north star names.
//
//   K-s0  ks_hist16       per-rank histogram of key bytes 0..1 (65536 bins, warp-aggregated atomics)
//   K-s1  ks_candidates   stable compaction of the records whose 16-bit prefix is a boundary bin
//                         (full records + global ordinals), single pass with decoupled look-back
//   K-s2  ks_dest_counts  per-destination counts of the local candidates against the exact splitters
//   K-p   kp_partition    stable partition of full records into G destination segments: a 256-record
//                         tile is staged in shared memory, ranked by destination (ballots), offset by a
//                         per-destination decoupled look-back over tiles, and written back in
//                         destination order as coalesced word streams. Each destination run goes to
//                         dst_base[d] + dst_off[d]: the local send buffer (then an NCCL all-to-all), or
//                         — the fused exchange — straight into rank d's receive window
//                         over NVLink (NCCL symmetric memory, k_exchange.cu), so the exchange overlaps the
//                         partition tile by tile and the 200 B/record send-buffer round trip disappears
// Destination of a record = number of splitters s_k (k = 1..G-1) with s_k <= (key, global ordinal):
// the exact splitter s_k is the element of global sorted rank floor(k N / G).
#include "block_rank.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace ley {

namespace {

__device__ __forceinline__ void load_key(const uint8_t* in, uint64_t i, uint32_t& hi, uint32_t& mid, uint32_t& lo16,
                                         const DistKeyMask& km) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(in + i * kRecordBytes);
  hi = bswap32(__ldg(p)) & km.hi;        // key bytes 0..3
  mid = bswap32(__ldg(p + 1)) & km.mid;  // 4..7
  const uint32_t c = __ldg(p + 2);
  lo16 = (((c & 0xFFu) << 8) | ((c >> 8) & 0xFFu)) & km.lo16;  // bytes 8..9
}

__device__ __forceinline__ int splitter_cmp(uint32_t hi, uint32_t mid, uint32_t lo16, uint32_t gidx,
                                            const DistSplitter& s) {
  if (hi != s.hi) return hi < s.hi ? -1 : 1;
  if (mid != s.mid) return mid < s.mid ? -1 : 1;
  if (lo16 != s.lo16) return lo16 < s.lo16 ? -1 : 1;
  if (gidx != s.gidx) return gidx < s.gidx ? -1 : 1;
  return 0;
}

__device__ __forceinline__ uint32_t dest_of(uint32_t hi, uint32_t mid, uint32_t lo16, uint32_t gidx,
                                            const DistSplitter* spl, int nspl) {
  uint32_t d = 0;
  const uint32_t p16 = hi >> 16;
  for (int k = 0; k < nspl; ++k) {
    const uint32_t b = spl[k].hi >> 16;
    if (p16 > b) ++d;
    else if (p16 == b && splitter_cmp(hi, mid, lo16, gidx, spl[k]) >= 0) ++d;
  }
  return d;
}

// ------------------------------------------------------------------------------------------ K-s0
// Also keeps every record's 16-bit prefix (2 B/record, coalesced) so that K-s1 finds the boundary-bin
// records from the prefixes instead of reading every record's key line again (~100 B/record).
// (the 4 key bytes of a record sit in one 64-byte block: .L2::64B fetches that block instead of the whole
// 128-byte line a plain miss brings, 64 instead of 100 DRAM bytes per record; profiles/r02_fetch_granularity.txt)
__device__ __forceinline__ uint32_t ld_key_word(const uint8_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(256) ks_hist16(const uint8_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ hist,
                                                 uint16_t* __restrict__ pref, uint32_t mask_hi) {
  const uint32_t lt = lanemask_lt();
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    const bool valid = i < n;
    uint32_t hi = 0;
    if (valid) hi = bswap32(ld_key_word(in + i * kRecordBytes)) & mask_hi;
    const uint32_t p16 = hi >> 16;
    if (valid) pref[i] = (uint16_t)p16;
    const uint32_t peers = warp_peers8(p16 & 0xFFu, valid) & warp_peers8(p16 >> 8, valid);
    if (valid && __popc(peers & lt) == 0) atomicAdd(&hist[p16], (uint32_t)__popc(peers));
  }
}

// ------------------------------------------------------------------------------------------ K-s1
constexpr int kCandThreads = 256;
constexpr int kCandItems = 8;
constexpr uint32_t kCandTile = kCandThreads * kCandItems;

__global__ void __launch_bounds__(kCandThreads)
    ks_candidates(const uint8_t* __restrict__ in, const uint16_t* __restrict__ pref16, uint64_t n, uint32_t gbase,
                  const uint32_t* __restrict__ bins,
                  int nbins, uint64_t* __restrict__ status, uint32_t* __restrict__ ticket, uint8_t* __restrict__ cand,
                  uint32_t* __restrict__ cand_gidx, uint32_t* __restrict__ cand_count) {
  __shared__ uint32_t s_tmp[32];
  __shared__ uint32_t s_t, s_pre;
  __shared__ uint32_t s_bins[8];
  if (threadIdx.x < 8) s_bins[threadIdx.x] = threadIdx.x < (unsigned)nbins ? bins[threadIdx.x] : 0xFFFFFFFFu;
  if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t t = s_t;
  const uint64_t base = (uint64_t)t * kCandTile;
  if (base >= n) return;
  // blocked: thread owns items [tid*ITEMS, +ITEMS) so the block order is the input order
  uint32_t flags = 0, cnt = 0;
#pragma unroll
  for (int j = 0; j < kCandItems; ++j) {
    const uint64_t i = base + threadIdx.x * kCandItems + j;
    if (i < n) {
      const uint32_t pref = __ldg(pref16 + i);
      bool f = false;
#pragma unroll
      for (int k = 0; k < 8; ++k) f |= (pref == s_bins[k]);
      if (f) {
        flags |= 1u << j;
        ++cnt;
      }
    }
  }
  uint32_t agg;
  const uint32_t ex = block_excl_scan<kCandThreads>(cnt, s_tmp, &agg);
  if (threadIdx.x == 0) {
    uint32_t pre = 0;
    if (t == 0) {
      st_relaxed_u64(&status[0], kFlagPrefix | agg);
    } else {
      st_relaxed_u64(&status[t], kFlagAggregate | agg);
      int64_t j = (int64_t)t - 1;
      while (true) {
        const uint64_t sv = ld_relaxed_u64(&status[j]);
        const uint32_t f = status_flag(sv);
        if (f == 0) continue;
        pre += (uint32_t)sv;
        if (f == 2) break;
        --j;
      }
      st_relaxed_u64(&status[t], kFlagPrefix | (uint64_t)(pre + agg));
    }
    s_pre = pre;
    if (base + kCandTile >= n) *cand_count = pre + agg;
  }
  __syncthreads();
  uint32_t pos = s_pre + ex;
#pragma unroll
  for (int j = 0; j < kCandItems; ++j) {
    if (flags & (1u << j)) {
      const uint64_t i = base + threadIdx.x * kCandItems + j;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(in + i * kRecordBytes);
      uint32_t* dst = reinterpret_cast<uint32_t*>(cand + (uint64_t)pos * kRecordBytes);
#pragma unroll
      for (int w = 0; w < (int)kRecordWords; ++w) dst[w] = __ldg(src + w);
      cand_gidx[pos] = gbase + (uint32_t)i;
      ++pos;
    }
  }
}

// ------------------------------------------------------------------------------------------ K-s2
__global__ void ks_dest_counts(const uint8_t* __restrict__ cand, const uint32_t* __restrict__ cand_gidx,
                               uint32_t ncand, const DistSplitter* __restrict__ spl, int nspl,
                               unsigned long long* __restrict__ counts, DistKeyMask km) {
  __shared__ unsigned long long s_c[kMaxRanks];
  if (threadIdx.x < kMaxRanks) s_c[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ncand; i += gridDim.x * blockDim.x) {
    uint32_t hi, mid, lo16;
    load_key(cand, i, hi, mid, lo16, km);
    atomicAdd(&s_c[dest_of(hi, mid, lo16, cand_gidx[i], spl, nspl)], 1ull);
  }
  __syncthreads();
  if (threadIdx.x < kMaxRanks && s_c[threadIdx.x]) atomicAdd(&counts[threadIdx.x], s_c[threadIdx.x]);
}

// ------------------------------------------------------------------------------------------ K-p
constexpr int kPartThreads = 256;
constexpr uint32_t kPartTile = 256;  // records per tile (one per thread)

__global__ void __launch_bounds__(kPartThreads)
    kp_partition(const uint8_t* __restrict__ in, uint64_t n, uint32_t gbase, const DistSplitter* __restrict__ spl,
                 int nspl, uint8_t* const* __restrict__ dst_base, const uint64_t* __restrict__ dst_off,
                 uint64_t* __restrict__ status, uint32_t* __restrict__ ticket, int remote, DistKeyMask km) {
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t* s_rec = s_dyn;                                 // tile in input order
  __shared__ uint16_t s_inv[kPartTile];                    // destination-ordered slot p holds record s_inv[p]
  __shared__ uint8_t s_slot_d[kPartTile];                  // and goes to destination s_slot_d[p]
  __shared__ DistSplitter s_spl[kMaxRanks - 1];
  __shared__ uint32_t s_wc[kPartThreads / 32][kMaxRanks];
  __shared__ uint32_t s_dcnt[kMaxRanks], s_dex[kMaxRanks];
  __shared__ uint64_t s_dst[kMaxRanks];
  __shared__ uint8_t* s_dptr[kMaxRanks];
  __shared__ uint32_t s_t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < (unsigned)nspl) s_spl[threadIdx.x] = spl[threadIdx.x];
  if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t t = s_t;
  const uint64_t base = (uint64_t)t * kPartTile;
  if (base >= n) return;
  const uint32_t cnt = (uint32_t)(n - base < kPartTile ? n - base : kPartTile);
  // coalesced tile load (the tile starts at a multiple of 256 records -> 16-byte aligned)
  {
    const uint4* src = reinterpret_cast<const uint4*>(in + base * kRecordBytes);
    const uint32_t nvec = cnt * kRecordBytes / 16;
    uint4* dst = reinterpret_cast<uint4*>(s_rec);
    for (uint32_t v = threadIdx.x; v < nvec; v += kPartThreads) dst[v] = __ldg(src + v);
    const uint32_t done = nvec * 4, words = cnt * kRecordWords;
    const uint32_t* srcw = reinterpret_cast<const uint32_t*>(in + base * kRecordBytes);
    for (uint32_t w = done + threadIdx.x; w < words; w += kPartThreads) s_rec[w] = __ldg(srcw + w);
  }
  __syncthreads();
  const uint32_t i = threadIdx.x;
  const bool valid = i < cnt;
  uint32_t d = 0;
  if (valid) {
    const uint32_t* r = s_rec + i * kRecordWords;
    const uint32_t c = r[2];
    d = dest_of(bswap32(r[0]) & km.hi, bswap32(r[1]) & km.mid, (((c & 0xFFu) << 8) | ((c >> 8) & 0xFFu)) & km.lo16,
                gbase + (uint32_t)(base + i), s_spl, nspl);
  }
  // stable rank by destination (3 ballots: destinations < 8)
  uint32_t peers = __ballot_sync(0xffffffffu, valid);
  if (!valid) peers = ~peers;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const bool set = (d >> b) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, set);
    peers &= set ? bal : ~bal;
  }
  const uint32_t before = __popc(peers & lanemask_lt());
  if (threadIdx.x < kMaxRanks * (kPartThreads / 32)) (&s_wc[0][0])[threadIdx.x] = 0;
  __syncthreads();
  if (valid && before == 0) s_wc[warp][d] = __popc(peers);
  __syncthreads();
  if (threadIdx.x < kMaxRanks) {
    uint32_t run = 0;
    for (int w = 0; w < kPartThreads / 32; ++w) {
      const uint32_t v = s_wc[w][threadIdx.x];
      s_wc[w][threadIdx.x] = run;
      run += v;
    }
    s_dcnt[threadIdx.x] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int k = 0; k < kMaxRanks; ++k) {
      s_dex[k] = run;
      run += s_dcnt[k];
    }
  }
  __syncthreads();
  // per-destination look-back over tiles (threads 0..G-1)
  if (threadIdx.x < (unsigned)(nspl + 1)) {
    const int k = threadIdx.x;
    const uint32_t agg = s_dcnt[k];
    uint64_t* st = status + (uint64_t)t * kMaxRanks + k;
    uint32_t pre = 0;
    if (t == 0) {
      st_relaxed_u64(st, kFlagPrefix | agg);
    } else {
      st_relaxed_u64(st, kFlagAggregate | agg);
      int64_t j = (int64_t)t - 1;
      while (true) {
        const uint64_t sv = ld_relaxed_u64(status + (uint64_t)j * kMaxRanks + k);
        const uint32_t f = status_flag(sv);
        if (f == 0) continue;
        pre += (uint32_t)sv;
        if (f == 2) break;
        --j;
      }
      st_relaxed_u64(st, kFlagPrefix | (uint64_t)(pre + agg));
    }
    s_dst[k] = dst_off[k] + pre;
    s_dptr[k] = dst_base[k];
  }
  // destination order as a slot map (no second copy of the tile: half the shared memory, twice the CTAs
  // per SM), then every destination run written as a coalesced word stream straight from the input tile
  if (valid) {
    const uint32_t p = s_dex[d] + s_wc[warp][d] + before;
    s_inv[p] = (uint16_t)i;
    s_slot_d[p] = (uint8_t)d;
  }
  __syncthreads();
  for (uint32_t w = threadIdx.x; w < cnt * kRecordWords; w += kPartThreads) {
    const uint32_t p = w / kRecordWords, c = w - p * kRecordWords;
    const uint32_t k = s_slot_d[p];
    uint32_t* dst = reinterpret_cast<uint32_t*>(s_dptr[k] + (s_dst[k] + p - s_dex[k]) * kRecordBytes);
    dst[c] = s_rec[(uint32_t)s_inv[p] * kRecordWords + c];
  }
  // fused exchange: the stores above went to peers' receive windows over NVLink. One system-scope fence
  // per CTA, after the barrier that orders every thread's stores before it (fences are cumulative), so
  // they are performed before the grid completes and the host's ordering collective runs (a fence per
  // thread cost ~30% of the kernel: membar stalls)
  if (remote) {
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
  (void)lane;
}

unsigned grid_cap(uint64_t items, int per_block, int sms, int per_sm) {
  uint64_t b = (items + per_block - 1) / per_block;
  uint64_t cap = (uint64_t)sms * per_sm;
  if (b > cap) b = cap;
  return (unsigned)(b ? b : 1);
}

}  // namespace

cudaError_t launch_ks_hist16(const uint8_t* in, uint64_t n, uint32_t* hist, uint16_t* pref, DistKeyMask km, int sms,
                             cudaStream_t s) {
  if (!n) return cudaSuccess;
  ks_hist16<<<grid_cap(n, 256, sms, 8), 256, 0, s>>>(in, n, hist, pref, km.hi);
  return cudaGetLastError();
}

uint64_t ks_candidate_tiles(uint64_t n) { return (n + kCandTile - 1) / kCandTile; }

cudaError_t launch_ks_candidates(const uint8_t* in, const uint16_t* pref, uint64_t n, uint32_t gbase,
                                 const uint32_t* bins, int nbins,
                                 uint64_t* status, uint32_t* ticket, uint8_t* cand, uint32_t* cand_gidx,
                                 uint32_t* cand_count, cudaStream_t s) {
  if (!n) return cudaSuccess;
  ks_candidates<<<(unsigned)ks_candidate_tiles(n), kCandThreads, 0, s>>>(in, pref, n, gbase, bins, nbins, status, ticket,
                                                                          cand, cand_gidx, cand_count);
  return cudaGetLastError();
}

cudaError_t launch_ks_dest_counts(const uint8_t* cand, const uint32_t* cand_gidx, uint32_t ncand,
                                  const DistSplitter* spl, int nspl, unsigned long long* counts, DistKeyMask km,
                                  int sms, cudaStream_t s) {
  if (!ncand) return cudaSuccess;
  ks_dest_counts<<<grid_cap(ncand, 256, sms, 4), 256, 0, s>>>(cand, cand_gidx, ncand, spl, nspl, counts, km);
  return cudaGetLastError();
}

uint64_t kp_tiles(uint64_t n) { return (n + kPartTile - 1) / kPartTile; }

cudaError_t launch_kp_partition(const uint8_t* in, uint64_t n, uint32_t gbase, const DistSplitter* spl, int nspl,
                                uint8_t* const* dst_base, const uint64_t* dst_off, uint64_t* status, uint32_t* ticket,
                                bool remote, DistKeyMask km, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const size_t smem = (size_t)kPartTile * kRecordBytes;
  cudaError_t e = cudaFuncSetAttribute(kp_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kp_partition<<<(unsigned)kp_tiles(n), kPartThreads, smem, s>>>(in, n, gbase, spl, nspl, dst_base, dst_off, status,
                                                                  ticket, remote ? 1 : 0, km);
  return cudaGetLastError();
}

}  // namespace ley
