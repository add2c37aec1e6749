// k_ties.cu — keys longer than 10 bytes, hybrid form (§5: "make Leyenda hybrid between prefix
// sorting and comparison-based record sorting"). The radix sort orders the records by their first 10 key
// bytes (ties by input index); only records whose 10-byte prefixes tie need the rest of the key:
//   kt_tie_groups  one pass over the sorted records: maximal runs of equal 10-byte prefixes ("tie groups",
//                  >= 2 records) are reported as first and last positions (two unordered lists)
//   kt_large_lasts the "large lasts" list (a group is large, > kCtaGroup records, iff the record kCtaGroup
//                  before its last ties)
//   kt_fix_tiny    eight lanes per group first: the lanes find the group's length themselves (a ballot of
//                  prefix equality over the next 8 records — the run is contiguous and maximal); a group of
//                  <= 7 records is ranked lane by lane by (key bytes [10, key_bytes), position) — a
//                  comparison sort on the records themselves — and rewritten in place in that order; a
//                  longer one goes to the "mid" list (written over the lasts, no longer needed)
//   kt_fix_small   the same with a whole warp per mid group for groups of <= 32 records; a longer one goes
//                  to the "big" list (written over the firsts)
//   kt_fix_cta     one CTA per big group, staged in shared memory and ordered there: groups of <= 128
//                  records by small CTAs (many per SM), longer ones passed on to CTAs with 100 KB staging for
//                  <= kCtaGroup records; longer still: appended to the short "large firsts" list
// No list is ever sorted or shipped to the host except the two large lists (<= 65 entries read); large
// groups are sorted by the LSD window passes restricted to their slice (internal.cu).
#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

constexpr uint32_t kCtaGroup = 1024;  // largest group kt_fix_cta sorts (100 KB of shared memory staging)

__device__ __forceinline__ bool prefix10_equal(const uint8_t* a, const uint8_t* b) {
  // records are 4-byte aligned: words 0, 1 and the low half of word 2
  const uint32_t* x = reinterpret_cast<const uint32_t*>(a);
  const uint32_t* y = reinterpret_cast<const uint32_t*>(b);
  return x[0] == y[0] && x[1] == y[1] && ((x[2] ^ y[2]) & 0xFFFFu) == 0;
}

// Appends v to list[counts[c]++] for the lanes with `take` (one atomic per warp; all 32 lanes call it).
__device__ __forceinline__ void warp_append(bool take, uint32_t v, uint32_t* list, uint32_t* counter, uint32_t cap) {
  const uint32_t m = __ballot_sync(0xffffffffu, take);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(counter, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (take) {
    const uint32_t at = base + __popc(m & ((1u << lane) - 1u));
    if (at < cap) list[at] = v;
  }
}

// dg (nullable): the prefix digests K-e wrote beside the records (k_bucket.cu prefix_digest); equal
// prefixes have equal digests, so only adjacent records with equal digests are compared on the records.
__global__ void kt_tie_groups(const uint8_t* __restrict__ recs, const uint64_t* __restrict__ dg, uint64_t n,
                              uint32_t* __restrict__ firsts, uint32_t* __restrict__ lasts, uint32_t cap,
                              uint32_t* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count: every lane takes part in the appends' ballots
  for (uint64_t j0 = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); j0 < n; j0 += stride) {
    const uint64_t j = j0 + (threadIdx.x & 31);
    bool tie_prev = false, tie_next = false;
    if (j < n) {
      const uint8_t* r = recs + j * kRecordBytes;
      bool cand_prev = j > 0, cand_next = j + 1 < n;
      if (dg) {
        const uint64_t d = dg[j];
        cand_prev = cand_prev && dg[j - 1] == d;
        cand_next = cand_next && dg[j + 1] == d;
      }
      tie_prev = cand_prev && prefix10_equal(r - kRecordBytes, r);
      tie_next = cand_next && prefix10_equal(r, r + kRecordBytes);
    }
    warp_append(tie_next && !tie_prev, (uint32_t)j, firsts, &counts[0], cap);
    warp_append(tie_prev && !tie_next, (uint32_t)j, lasts, &counts[1], cap);
  }
}

// key bytes [10, kb) of records a and b (positions in `recs`), unsigned; ties by position
__device__ __forceinline__ bool tail_less(const uint8_t* recs, uint32_t a, uint32_t b, uint32_t kb) {
  const uint8_t* x = recs + (uint64_t)a * kRecordBytes;
  const uint8_t* y = recs + (uint64_t)b * kRecordBytes;
  for (uint32_t i = kKeyBytes; i < kb; ++i) {
    const uint32_t u = x[i], v = y[i];
    if (u != v) return u < v;
  }
  return a < b;
}

// (prefix comparisons go to the records only where the digests dg already match)
__device__ __forceinline__ bool same_prefix(const uint8_t* recs, const uint64_t* dg, uint64_t a, uint64_t b) {
  return dg[a] == dg[b] && prefix10_equal(recs + a * kRecordBytes, recs + b * kRecordBytes);
}

// Lanes [0, len) of a group of len records starting at f (all lanes of the warp call it): rank by
// (key bytes [10, kb), position), then rewrite the group in place in that order.
__device__ __forceinline__ void rank_and_rewrite(uint8_t* recs, uint32_t f, uint32_t len, bool active, uint32_t idx,
                                                 uint32_t kb) {
  const uint32_t me = f + idx;
  uint32_t rank = 0;
  if (active)
    for (uint32_t m = 0; m < len; ++m)
      if (m != idx && tail_less(recs, f + m, me, kb)) ++rank;
  uint32_t w[kRecordWords];
  const uint32_t* src = reinterpret_cast<const uint32_t*>(recs + (uint64_t)me * kRecordBytes);
#pragma unroll
  for (int q = 0; q < (int)kRecordWords; ++q) w[q] = active ? src[q] : 0u;
  __syncwarp();  // every lane holds its record before any is overwritten
  if (active) {
    uint32_t* dst = reinterpret_cast<uint32_t*>(recs + (uint64_t)(f + rank) * kRecordBytes);
#pragma unroll
    for (int q = 0; q < (int)kRecordWords; ++q) dst[q] = w[q];
  }
  __syncwarp();
}

__global__ void kt_fix_tiny(uint8_t* __restrict__ recs, const uint64_t* __restrict__ dg, uint64_t n,
                            const uint32_t* __restrict__ firsts, uint32_t* __restrict__ counts, uint32_t kb,
                            uint32_t* __restrict__ mid, uint32_t cap) {
  const int lane = threadIdx.x & 31, sub = lane >> 3, sl = lane & 7;
  const uint32_t step = gridDim.x * (blockDim.x >> 3);  // four groups per warp per iteration
  const uint32_t ngroups = counts[0];
  for (uint32_t g0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4; g0 < ngroups; g0 += step) {
    const uint32_t g = g0 + sub;
    const bool valid = g < ngroups;
    const uint32_t f = valid ? firsts[g] : 0u;
    const bool eq = valid && (uint64_t)f + sl < n && same_prefix(recs, dg, f, (uint64_t)f + sl);
    const uint32_t len = __popc((__ballot_sync(0xffffffffu, eq) >> (sub * 8)) & 0xFFu);
    const bool tiny = valid && len < 8;  // the record after the run was seen (or is past n)
    warp_append(valid && !tiny && sl == 0, f, mid, &counts[4], cap);
    rank_and_rewrite(recs, f, len, tiny && (uint32_t)sl < len, (uint32_t)sl, kb);
  }
}

__global__ void kt_fix_small(uint8_t* __restrict__ recs, const uint64_t* __restrict__ dg, uint64_t n,
                             const uint32_t* __restrict__ firsts, const uint32_t* __restrict__ count, uint32_t kb,
                             uint32_t* __restrict__ counts, uint32_t* __restrict__ big) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const uint32_t ngroups = *count;
  for (uint32_t g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < ngroups; g += warps) {
    const uint32_t f = firsts[g];
    const bool eq = (uint64_t)f + lane < n && same_prefix(recs, dg, f, (uint64_t)f + lane);
    const uint32_t len = __popc(__ballot_sync(0xffffffffu, eq));  // the run from f is contiguous
    if (len == 32 && (uint64_t)f + 32 < n && same_prefix(recs, dg, f, (uint64_t)f + 32)) {
      if (lane == 0) big[atomicAdd(&counts[5], 1u)] = f;  // (one per warp-group: no aggregation needed)
      continue;
    }
    rank_and_rewrite(recs, f, len, (uint32_t)lane < len, (uint32_t)lane, kb);
  }
}

// One CTA per listed group known to be longer than LO records: a group of <= CAPG records is staged in
// shared memory, ordered there (rank by pairs up to 128 records, else a bitonic network) and written back
// in place; a longer one goes to `next` (entries past next_cap dropped). Two tiers: <= 128 records with
// 12.8 KB of staging (many CTAs per SM), <= 1024 with 100 KB.
template <uint32_t LO, uint32_t CAPG, int THREADS>
__global__ void __launch_bounds__(THREADS)
    kt_fix_cta(uint8_t* __restrict__ recs, const uint64_t* __restrict__ dg, uint64_t n,
               const uint32_t* __restrict__ big, const uint32_t* __restrict__ count, uint32_t kb,
               uint32_t* __restrict__ next, uint32_t* __restrict__ next_count, uint32_t next_cap) {
  constexpr int kCtaThreads = THREADS;
  extern __shared__ __align__(16) uint32_t s_rec[];  // [CAPG * kRecordWords]
  __shared__ uint32_t s_len;
  __shared__ uint32_t s_rank[CAPG];
  const uint8_t* sb = reinterpret_cast<const uint8_t*>(s_rec);
  const uint32_t nbig = *count;
  for (uint32_t g = blockIdx.x; g < nbig; g += gridDim.x) {
    const uint32_t f = big[g];
    if (threadIdx.x == 0) s_len = CAPG + 1;
    __syncthreads();
    // the run from f is contiguous: its length is the first position that does not tie with f (scanned
    // THREADS positions at a time, stopping at the first window that holds it). The stop decision is the
    // barrier's own OR, so every warp leaves the loop at the same window (reading s_len after a plain
    // barrier could see a faster warp's atomicMin from the next window and break one window early).
    for (uint32_t t0 = LO + 1; t0 <= CAPG; t0 += kCtaThreads) {
      const uint32_t t = t0 + threadIdx.x;
      const bool end = t <= CAPG && ((uint64_t)f + t >= n || !same_prefix(recs, dg, f, (uint64_t)f + t));
      if (end) atomicMin(&s_len, t);
      if (__syncthreads_or(end)) break;
    }
    const uint32_t len = s_len;
    if (len > CAPG) {
      if (threadIdx.x == 0) {
        const uint32_t at = atomicAdd(next_count, 1u);
        if (at < next_cap) next[at] = f;
      }
      __syncthreads();  // s_len is rewritten by the next group
      continue;
    }
    const uint32_t* src = reinterpret_cast<const uint32_t*>(recs + (uint64_t)f * kRecordBytes);
    for (uint32_t w = threadIdx.x; w < len * kRecordWords; w += kCtaThreads) s_rec[w] = src[w];
    // (group records y before x by (key bytes [10, kb), position); indices >= len are +infinity)
    auto before = [&](uint32_t y, uint32_t x) -> bool {
      if (y >= len) return false;
      if (x >= len) return true;
      const uint8_t* px = sb + (size_t)x * kRecordBytes;
      const uint8_t* py = sb + (size_t)y * kRecordBytes;
      uint32_t b = kKeyBytes;
      while (b < kb && px[b] == py[b]) ++b;
      return b < kb ? py[b] < px[b] : y < x;
    };
    uint32_t* dst = reinterpret_cast<uint32_t*>(recs + (uint64_t)f * kRecordBytes);
    if (CAPG <= 128 || len <= 128) {
      // small: rank of record i = how many records precede it; every ordered pair (i, m) with m before i
      // adds one (a warp: 32 different i, one m)
      for (uint32_t i = threadIdx.x; i < len; i += kCtaThreads) s_rank[i] = 0;
      __syncthreads();
      for (uint32_t p = threadIdx.x; p < len * len; p += kCtaThreads) {
        const uint32_t m = p / len, i = p - m * len;
        if (m != i && before(m, i)) atomicAdd(&s_rank[i], 1u);
      }
      __syncthreads();
      for (uint32_t w = threadIdx.x; w < len * kRecordWords; w += kCtaThreads) {
        const uint32_t i = w / kRecordWords, q = w - i * kRecordWords;
        dst[(size_t)s_rank[i] * kRecordWords + q] = s_rec[w];
      }
    } else {
      // larger: bitonic network over the record indices, padded to a power of two with +infinity
      uint32_t P = 256;
      while (P < len) P <<= 1;
      for (uint32_t i = threadIdx.x; i < P; i += kCtaThreads) s_rank[i] = i;
      __syncthreads();
      for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t t = threadIdx.x; t < P / 2; t += kCtaThreads) {
            const uint32_t i = (t / j) * 2 * j + (t % j), l = i + j;
            const uint32_t a = s_rank[i], b = s_rank[l];
            if (((i & k) == 0) ? before(b, a) : before(a, b)) {
              s_rank[i] = b;
              s_rank[l] = a;
            }
          }
          __syncthreads();
        }
      for (uint32_t w = threadIdx.x; w < len * kRecordWords; w += kCtaThreads) {
        const uint32_t r = w / kRecordWords, q = w - r * kRecordWords;
        dst[w] = s_rec[(size_t)s_rank[r] * kRecordWords + q];
      }
    }
    __syncthreads();  // staging reused by the next group
  }
}

__global__ void kt_large_lasts(const uint8_t* __restrict__ recs, const uint64_t* __restrict__ dg,
                               const uint32_t* __restrict__ lasts, uint32_t* __restrict__ counts,
                               uint32_t* __restrict__ large_l, uint32_t large_cap) {
  const uint32_t nl = counts[1];
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < nl; g += gridDim.x * blockDim.x) {
    const uint32_t l = lasts[g];
    if (l >= kCtaGroup && same_prefix(recs, dg, l - kCtaGroup, l)) {
      const uint32_t at = atomicAdd(&counts[3], 1u);  // (rare: at most a few large groups)
      if (at < large_cap) large_l[at] = l;
    }
  }
}

}  // namespace

cudaError_t launch_tie_groups(const uint8_t* recs, const uint64_t* dg, uint64_t n, uint32_t* firsts, uint32_t* lasts, uint32_t cap,
                              uint32_t* counts, int sms, cudaStream_t s) {
  if (n < 2) return cudaSuccess;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
  kt_tie_groups<<<(unsigned)blocks, 256, 0, s>>>(recs, dg, n, firsts, lasts, cap, counts);
  return cudaGetLastError();
}

cudaError_t launch_fix_small_groups(uint8_t* recs, const uint64_t* dg, uint64_t n, uint32_t* firsts,
                                    uint32_t* lasts, uint32_t* counts, uint32_t key_bytes, uint32_t* large_f,
                                    uint32_t* large_l, uint32_t large_cap, int sms, cudaStream_t s) {
  if (n < 2) return cudaSuccess;
  // group counts live on the device: persistent grids, grid-stride over the counts. The large lasts first:
  // the tiny pass then reuses the lasts array for its mid list (counts[4]).
  kt_large_lasts<<<sms * 4, 256, 0, s>>>(recs, dg, lasts, counts, large_l, large_cap);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  uint32_t* mid = lasts;
  kt_fix_tiny<<<sms * 8, 256, 0, s>>>(recs, dg, n, firsts, counts, key_bytes, mid, (uint32_t)(n / 2 + 1));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // the firsts are no longer needed once kt_fix_tiny is done: the big list goes there (counts[5]); the
  // mid list is free again after kt_fix_small: groups over 128 records go there (counts[6])
  kt_fix_small<<<sms * 8, 256, 0, s>>>(recs, dg, n, mid, counts + 4, key_bytes, counts, firsts);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  kt_fix_cta<32, 128, 128><<<sms * 16, 128, 128 * kRecordBytes, s>>>(recs, dg, n, firsts, counts + 5, key_bytes, mid,
                                                                      counts + 6, (uint32_t)(n / 2 + 1));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t smem = (size_t)kCtaGroup * kRecordBytes;
  auto k2 = kt_fix_cta<128, kCtaGroup, 512>;
  if ((e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
  k2<<<sms * 2, 512, smem, s>>>(recs, dg, n, mid, counts + 6, key_bytes, large_f, counts + 2, large_cap);
  return cudaGetLastError();
}

}  // namespace ley
