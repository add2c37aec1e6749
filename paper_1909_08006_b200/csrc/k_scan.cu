// k_scan.cu — K-b: single-pass decoupled-lookback device-wide exclusive scan,
// plus the small planning kernels that turn scanned histograms into work decompositions.
//
// PAPER.md §3.1 line 96: "we first compute a histogram based on the current radix to decide the size of
// each bucket and where each key should be placed" — the "where" is an exclusive prefix sum over the
// histogram. Over the bucket-major count matrix cnt[b * tiles + t] written by K-a it yields, for every
// (byte-0 value b, tile t), the global position of tile t's run of b in the byte-0-ordered sequence.
// Over hist16 it yields the level-1 bucket bases B16[p] (p = key bytes 0..1).
//
// Block tiles are claimed with an atomic ticket, so every block a block waits on is already resident
// (forward progress). Status words pack [flag | value] in 64 bits and are read/written with relaxed
// gpu-scope 64-bit accesses (single-copy atomic), so no torn reads.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

struct ScanJob {
  const uint32_t* in;
  uint32_t* out;
  uint64_t m;
  uint64_t* status;
  uint32_t* total_out;
  uint32_t copies = 1;     // in = `copies` arrays `stride` words apart: the scan is over their sum ...
  uint64_t stride = 0;
  uint32_t* sum_out = nullptr;  // ... written back here (copy 0; level-1 hist16), if given
  uint32_t* out2 = nullptr;     // a second copy of the exclusive prefix (level 1: the split's fill cursors)
};

// Exclusive prefix of block blk's predecessors by warp 0: a window of 32 predecessor status words per
// step (one per lane), summed up to the nearest published inclusive prefix — one round trip per 32 blocks
// instead of one per block.
__device__ __forceinline__ uint32_t lookback(uint64_t* status, uint32_t blk) {
  const int lane = threadIdx.x & 31;
  uint32_t excl = 0;
  for (int64_t end = (int64_t)blk - 1;; end -= 32) {
    const int64_t j = end - lane;
    uint64_t s = j >= 0 ? ld_relaxed_u64(&status[j]) : kFlagPrefix;  // (before block 0: prefix 0)
    while (__any_sync(0xffffffffu, status_flag(s) == 0))
      if (status_flag(s) == 0) s = ld_relaxed_u64(&status[j]);
    const uint32_t pre = __ballot_sync(0xffffffffu, status_flag(s) == 2);
    const int stop = pre ? __ffs(pre) - 1 : 31;  // lanes 0..stop: the nearest prefix and the aggregates after it
    uint32_t v = lane <= stop ? (uint32_t)s : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (pre) return excl;
  }
}

__device__ __forceinline__ void scan_block(const ScanJob& jb, uint32_t blk, uint32_t* s_tmp, uint32_t* s_prefix) {
  const uint32_t* __restrict__ in = jb.in;
  uint32_t* __restrict__ out = jb.out;
  const uint64_t m = jb.m;
  const uint64_t base = (uint64_t)blk * kScanTile + (uint64_t)threadIdx.x * kScanItems;

  // each thread's kScanItems consecutive words as 16-byte vectors (base is a multiple of 16 words)
  static_assert(kScanItems % 4 == 0, "vector loads");
  uint32_t v[kScanItems];
  uint32_t sum = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out) |
                     reinterpret_cast<uintptr_t>(jb.sum_out) | (jb.stride * 4)) & 15) == 0 &&
                   base + kScanItems <= m;
  if (vec) {
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      uint4 x = __ldg(reinterpret_cast<const uint4*>(in + base) + q);
      for (uint32_t c = 1; c < jb.copies; ++c) {
        const uint4 y = __ldg(reinterpret_cast<const uint4*>(in + c * jb.stride + base) + q);
        x.x += y.x;
        x.y += y.y;
        x.z += y.z;
        x.w += y.w;
      }
      if (jb.sum_out) reinterpret_cast<uint4*>(jb.sum_out + base)[q] = x;
      v[4 * q] = x.x;
      v[4 * q + 1] = x.y;
      v[4 * q + 2] = x.z;
      v[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      v[i] = 0;
      if (base + i < m) {
        for (uint32_t c = 0; c < jb.copies; ++c) v[i] += in[c * jb.stride + base + i];
        if (jb.sum_out) jb.sum_out[base + i] = v[i];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) sum += v[i];
  uint32_t agg;
  uint32_t texcl = block_excl_scan<kScanThreads>(sum, s_tmp, &agg);

  if (threadIdx.x < 32) {
    uint32_t excl = 0;
    if (blk == 0) {
      if (threadIdx.x == 0) st_relaxed_u64(&jb.status[0], kFlagPrefix | agg);
    } else {
      if (threadIdx.x == 0) st_relaxed_u64(&jb.status[blk], kFlagAggregate | agg);
      excl = lookback(jb.status, blk);
      if (threadIdx.x == 0) st_relaxed_u64(&jb.status[blk], kFlagPrefix | (uint64_t)(excl + agg));
    }
    if (threadIdx.x == 0) {
      *s_prefix = excl;
      if (jb.total_out && (uint64_t)(blk + 1) * kScanTile >= m) *jb.total_out = excl + agg;
    }
  }
  __syncthreads();
  uint32_t run = *s_prefix + texcl;
  if (vec) {
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      uint4 x;
      x.x = run;
      run += v[4 * q];
      x.y = run;
      run += v[4 * q + 1];
      x.z = run;
      run += v[4 * q + 2];
      x.w = run;
      run += v[4 * q + 3];
      reinterpret_cast<uint4*>(out + base)[q] = x;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (base + i < m) out[base + i] = run;
      run += v[i];
    }
  }
  if (jb.out2) {  // (same layout and alignment as out: 65536 words)
    uint32_t r = *s_prefix + texcl;
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      uint4 x;
      x.x = r;
      r += v[4 * q];
      x.y = r;
      r += v[4 * q + 1];
      x.z = r;
      r += v[4 * q + 2];
      x.w = r;
      r += v[4 * q + 3];
      reinterpret_cast<uint4*>(jb.out2 + base)[q] = x;
    }
  }
}

// Two independent scans in one launch: tickets [0, blocks_a) scan job a, the rest job b (claimed in
// order, so every block a block waits on is resident). blocks_b may be 0 (one scan).
__global__ void __launch_bounds__(kScanThreads)
    kb_scan_excl(ScanJob ja, uint32_t blocks_a, ScanJob jb, uint32_t* __restrict__ ticket) {
  __shared__ uint32_t s_tmp[32];
  __shared__ uint32_t s_blk;
  __shared__ uint32_t s_prefix;
  if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t t = s_blk;
  if (t < blocks_a) scan_block(ja, t, s_tmp, &s_prefix);
  else scan_block(jb, t - blocks_a, s_tmp, &s_prefix);
}

// Copy one device counter into mapped pinned host memory with a store from the SM: the host reads a
// recursion level's big-bucket count without a copy-engine transfer, which would queue behind a large
// D2H on the copy engine (the streaming and external paths overlap sorts with such copies).
__global__ void kb_publish_u32(const uint32_t* __restrict__ src, volatile uint32_t* dst) { *dst = *src; }

// Zero up to three 16-byte-aligned ranges (sizes multiples of 16) in one launch: the level-1 counters
// (hist16 copies, tickets / list counters, look-back status words) instead of three memset nodes.
__global__ void kb_zero3(uint4* a, uint64_t na, uint4* b, uint64_t nb, uint4* c, uint64_t nc) {
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < na + nb + nc; i += nth) {
    if (i < na) a[i] = z;
    else if (i < na + nb) b[i - na] = z;
    else c[i - na - nb] = z;
  }
}

}  // namespace

cudaError_t launch_zero3(void* a, uint64_t a_bytes, void* b, uint64_t b_bytes, void* c, uint64_t c_bytes, int sms,
                         cudaStream_t s) {
  const uint64_t words = (a_bytes + b_bytes + c_bytes) / 16;
  const uint64_t blocks = std::min<uint64_t>((words + 255) / 256, (uint64_t)sms * 4);
  if (!blocks) return cudaSuccess;
  kb_zero3<<<(unsigned)blocks, 256, 0, s>>>(static_cast<uint4*>(a), a_bytes / 16, static_cast<uint4*>(b), b_bytes / 16,
                                            static_cast<uint4*>(c), c_bytes / 16);
  return cudaGetLastError();
}

cudaError_t launch_publish_u32(const uint32_t* src, uint32_t* host_mapped_dev, cudaStream_t s) {
  kb_publish_u32<<<1, 1, 0, s>>>(src, host_mapped_dev);
  return cudaGetLastError();
}


cudaError_t launch_scan_excl(const uint32_t* in, uint32_t* out, uint64_t m, uint64_t* status, uint32_t* ticket,
                             uint32_t* total_out, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const uint64_t blocks = (m + kScanTile - 1) / kScanTile;
  kb_scan_excl<<<(unsigned)blocks, kScanThreads, 0, s>>>(ScanJob{in, out, m, status, total_out}, (uint32_t)blocks,
                                                         ScanJob{}, ticket);
  return cudaGetLastError();
}

cudaError_t launch_scan_excl2(const uint32_t* in_a, uint32_t* out_a, uint64_t m_a, uint64_t* status_a,
                              uint32_t* total_a, uint32_t* in_b, uint32_t* out_b, uint64_t m_b,
                              uint64_t* status_b, uint32_t* total_b, uint32_t copies_b, uint64_t stride_b,
                              uint32_t* ticket, cudaStream_t s, uint32_t* out2_b) {
  const uint64_t ba = (m_a + kScanTile - 1) / kScanTile, bb = (m_b + kScanTile - 1) / kScanTile;
  if (ba + bb == 0) return cudaSuccess;
  ScanJob jb{in_b, out_b, m_b, status_b, total_b, copies_b, stride_b, copies_b > 1 ? in_b : nullptr, out2_b};
  kb_scan_excl<<<(unsigned)(ba + bb), kScanThreads, 0, s>>>(ScanJob{in_a, out_a, m_a, status_a, total_a}, (uint32_t)ba,
                                                            jb, ticket);
  return cudaGetLastError();
}

uint64_t scan_status_words(uint64_t m) { return (m + kScanTile - 1) / kScanTile; }


}  // namespace ley
