// k_bucket.cu — K-d: per-bucket sort of (key-tail, index) pairs, plus level-1 classification.
//
// PAPER.md §3.1 Algorithm 1 lines 65-85: buckets below bigBucketThreshold go to smallBucketQueue and
// are finished by one worker each — SingleThreadRadixSort on the next radix, then ComparisonSort for
// buckets under tinyBucketThreshold ("size is small enough for comparison-based sort to perform
// more efficient than Radix Sort"). On the GPU a "worker" is a warp (tiny buckets, register bitonic
// network over the composite (tail, index)) or a CTA (shared-memory counting pass on the next 1..12 key
// bits, then per-sub-bucket comparison sort). SURVEY.md §8a row a5.
//
// Every bucket writes perm[start .. start+len) = input ordinals in sorted order. The comparison order is
// the composite (tail, index), which is the sort's strict total order, so the result does not depend on
// the (non-deterministic) atomics used to place elements inside a CTA.
#include <stdio.h>
#include <stdlib.h>

#include "classify.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

__global__ void kd_classify_level1(const uint32_t* __restrict__ hist16, const uint32_t* __restrict__ B16,
                                   Tunables tu, ListSet kd, Seg* __restrict__ big_out, uint32_t* __restrict__ big_count) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= 65536) return;
  Seg s{B16[p], hist16[p], 2u, 1u};
  classify_bucket(s, tu, kd, big_out, big_count);
}

// ---------------------------------------------------------------------------- warp tier (len <= 32)
__global__ void __launch_bounds__(256)
    kd_warp_sort(const Seg* __restrict__ list, const uint32_t* __restrict__ count, const uint64_t* __restrict__ t0,
                 const uint32_t* __restrict__ i0, const uint64_t* __restrict__ t1, const uint32_t* __restrict__ i1,
                 uint32_t* __restrict__ perm) {
  const uint32_t nitems = *count;
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t it = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < nitems; it += nwarps) {
    const Seg sg = list[it];
    const uint64_t* tp = (sg.parity ? t1 : t0) + sg.start;
    const uint32_t* ip = (sg.parity ? i1 : i0) + sg.start;
    uint64_t t = ~0ull;
    uint32_t x = ~0u;
    if ((uint32_t)lane < sg.len) {
      t = tp[lane];
      x = ip[lane];
    }
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
    if ((uint32_t)lane < sg.len) perm[sg.start + lane] = x;
  }
}

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

template <uint32_t CAP>
__host__ __device__ constexpr uint32_t kd_bins() {
  return CAP >= 4096 ? 4096u : CAP;  // <= 2^12 counting bins
}
template <uint32_t CAP>
__host__ __device__ constexpr size_t kd_smem() {
  return (size_t)CAP * 12 + (size_t)(2 * kd_bins<CAP>() + 1) * 4 + 64 * 4 + 16;
}

// One CTA per bucket (len <= CAP), persistent over its list:
//   1. load the bucket's (tail, idx) pairs (coalesced; kept in registers when CAP/THREADS <= 16,
//      else re-read from L2),
//   2. counting pass on the next `bits` unconsumed key bits (shared-memory atomics give each item its
//      rank inside its sub-bucket), block scan of the 2^bits counters, placement into shared memory,
//   3. comparison sort of every sub-bucket on the composite (tail, idx): insertion sort by one thread
//      (tiny) or a warp bitonic network (larger) — Alg. 1's ComparisonSort below tinyBucketThreshold,
//   4. perm[start + i] = idx of the i-th smallest, coalesced.
template <uint32_t CAP, int THREADS>
__global__ void __launch_bounds__(THREADS, (THREADS >= 1024 || (CAP / THREADS) > 8) ? 1 : (CAP / THREADS) > 4 ? 4 : 6)
    kd_cta_sort(const Seg* __restrict__ list, const uint32_t* __restrict__ count, const uint64_t* __restrict__ t0,
                const uint32_t* __restrict__ i0, const uint64_t* __restrict__ t1, const uint32_t* __restrict__ i1,
                uint32_t* __restrict__ perm, Tunables tu) {
  constexpr uint32_t BINS = kd_bins<CAP>();
  constexpr int WARPS = THREADS / 32;
  constexpr int ITEMS = CAP / THREADS;
  constexpr bool REGS = ITEMS <= 16;
  constexpr int RITEMS = REGS ? ITEMS : 1;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* s_tail = reinterpret_cast<uint64_t*>(smem);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_tail + CAP);
  uint32_t* s_cnt = s_idx + CAP;            // [BINS + 1]: counts, then exclusive starts
  uint32_t* s_bigl = s_cnt + BINS + 1;      // [BINS]: sub-buckets needing the warp network
  uint32_t* s_tmp = s_bigl + BINS;          // [32] scan tmp, [32] = number of big sub-buckets
  uint32_t* s_nbig = s_tmp + 32;

  for (uint32_t g = threadIdx.x; g <= BINS; g += THREADS) s_cnt[g] = 0;
  __syncthreads();
  const uint32_t nitems = *count;
  const int warp = threadIdx.x >> 5;
  for (uint32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const Seg sg = list[it];
    const uint32_t s = sg.len;
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
          tr[j] = tp[i];
          xr[j] = ip[i];
        }
      }
#pragma unroll
      for (int j = 0; j < RITEMS; ++j) {
        uint32_t i = j * THREADS + threadIdx.x;
        if (i < s) {
          rr[j] = atomicAdd(&s_cnt[digit2(tr[j], xr[j])], 1u);
        }
      }
    } else {
      // batches of 8 independent loads per thread keep the bucket read latency-tolerant
      for (uint32_t i0 = threadIdx.x; i0 < s; i0 += 8 * THREADS) {
        uint64_t tb[8];
        uint32_t xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t i = i0 + u * THREADS;
          tb[u] = i < s ? tp[i] : 0;
          xb[u] = (i < s && on_idx) ? ip[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u * THREADS < s) atomicAdd(&s_cnt[digit2(tb[u], xb[u])], 1u);
      }
    }
    if (threadIdx.x == 0) *s_nbig = 0;
    __syncthreads();
    // exclusive scan of the nb counters in place (contiguous slice per thread)
    {
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
      // smaller composites there, and writes its ordinal straight to perm.
#pragma unroll
      for (int j = 0; j < RITEMS; ++j) {
        uint32_t i = j * THREADS + threadIdx.x;
        if (i < s) {
          const uint32_t b = s_cnt[digit2(tr[j], xr[j])];
          s_tail[b + rr[j]] = tr[j];
          s_idx[b + rr[j]] = xr[j];
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < RITEMS; ++j) {
        uint32_t i = j * THREADS + threadIdx.x;
        if (i < s) {
          const uint32_t d = digit2(tr[j], xr[j]);
          const uint32_t b = s_cnt[d], sz = s_cnt[d + 1] - b;
          if (sz == 1) {
            perm[sg.start + b] = xr[j];
          } else if (sz <= (uint32_t)tu.kd_insert_max) {
            uint32_t rank = 0;
            for (uint32_t m = b; m < b + sz; ++m) rank += pair_less(s_tail[m], s_idx[m], tr[j], xr[j]) ? 1u : 0u;
            perm[sg.start + b + rank] = xr[j];
          } else if (rr[j] == 0) {
            s_bigl[atomicAdd(s_nbig, 1u)] = digit2(tr[j], xr[j]);
          }
        }
      }
      __syncthreads();
      const uint32_t nbig = *s_nbig;
      for (uint32_t q = warp; q < nbig; q += WARPS) {
        const uint32_t g = s_bigl[q];
        const uint32_t b = s_cnt[g], e = s_cnt[g + 1];
        warp_bitonic_smem(s_tail, s_idx, b, e);
        for (uint32_t i = b + (threadIdx.x & 31); i < e; i += 32) perm[sg.start + i] = s_idx[i];
      }
      __syncthreads();  // every warp is done reading the sub-bucket bounds before they are cleared
      for (uint32_t g = threadIdx.x; g <= nb; g += THREADS) s_cnt[g] = 0;
      __syncthreads();
      continue;
    }
    // ---- large-CAP path: elements re-read from L2, placed by a second counter pass
    for (uint32_t g = threadIdx.x; g < nb; g += THREADS) s_bigl[g] = 0;
    __syncthreads();
    for (uint32_t i0 = threadIdx.x; i0 < s; i0 += 8 * THREADS) {
      uint64_t tb[8];
      uint32_t xb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t i = i0 + u * THREADS;
        if (i < s) {
          tb[u] = tp[i];
          xb[u] = ip[i];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (i0 + u * THREADS < s) {
          const uint32_t d = digit2(tb[u], xb[u]);
          const uint32_t p = s_cnt[d] + atomicAdd(&s_bigl[d], 1u);
          s_tail[p] = tb[u];
          s_idx[p] = xb[u];
        }
      }
    }
    __syncthreads();
    // comparison sort of every sub-bucket
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
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < s; i += THREADS) perm[sg.start + i] = s_idx[i];
    for (uint32_t g = threadIdx.x; g <= nb; g += THREADS) s_cnt[g] = 0;
    __syncthreads();
  }
}

template <uint32_t CAP, int THREADS>
cudaError_t launch_cta_sort(const Seg* list, const uint32_t* count, const uint64_t* t0, const uint32_t* i0,
                            const uint64_t* t1, const uint32_t* i1, uint32_t* perm, const Tunables& tu, int sms,
                            cudaStream_t s) {
  auto kern = kd_cta_sort<CAP, THREADS>;
  const size_t smem = kd_smem<CAP>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  kern<<<sms * per_sm, THREADS, smem, s>>>(list, count, t0, i0, t1, i1, perm, tu);
  if (getenv("LEY_DEBUG_SYNC")) {
    fprintf(stderr, "[ley] kd_cta_sort<%u,%d> grid %d smem %zu\n", CAP, THREADS, sms * per_sm, smem);
    cudaError_t e2 = cudaStreamSynchronize(s);
    fprintf(stderr, "[ley]   done: %s\n", cudaGetErrorString(e2));
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_kd_classify_level1(const uint32_t* hist16, const uint32_t* B16, const Tunables& tu,
                                      const ListSet& kd, Seg* big_out, uint32_t* big_count, cudaStream_t s) {
  kd_classify_level1<<<256, 256, 0, s>>>(hist16, B16, tu, kd, big_out, big_count);
  return cudaGetLastError();
}

// All K-d tiers for the lists of one level (counts are read on the device; no host sync).
cudaError_t launch_kd_all(const ListSet& kd, const uint64_t* t0, const uint32_t* i0, const uint64_t* t1,
                          const uint32_t* i1, uint32_t* perm, const Tunables& tu, int sms, cudaStream_t s,
                          int* launches) {
  cudaError_t e;
  kd_warp_sort<<<sms * 8, 256, 0, s>>>(kd.items[kListWarp], kd.counts + kListWarp, t0, i0, t1, i1, perm);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = launch_cta_sort<512, 128>(kd.items[kListMed1], kd.counts + kListMed1, t0, i0, t1, i1, perm, tu, sms, s)))
    return e;
  if ((e = launch_cta_sort<2048, 256>(kd.items[kListMed2], kd.counts + kListMed2, t0, i0, t1, i1, perm, tu, sms, s)))
    return e;
  if ((e = launch_cta_sort<8192, 512>(kd.items[kListMed3], kd.counts + kListMed3, t0, i0, t1, i1, perm, tu, sms, s)))
    return e;
  if ((e = launch_cta_sort<10240, 1024>(kd.items[kListMed4], kd.counts + kListMed4, t0, i0, t1, i1, perm, tu, sms, s)))
    return e;
  if ((e = launch_cta_sort<16384, 512>(kd.items[kListMed5], kd.counts + kListMed5, t0, i0, t1, i1, perm, tu, sms, s)))
    return e;
  if (launches) *launches += 6;
  return cudaSuccess;
}

}  // namespace ley
