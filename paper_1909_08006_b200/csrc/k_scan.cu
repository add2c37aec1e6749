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
#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

__global__ void __launch_bounds__(kScanThreads)
    kb_scan_excl(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t m,
                 uint64_t* __restrict__ status, uint32_t* __restrict__ ticket, uint32_t* __restrict__ total_out) {
  __shared__ uint32_t s_tmp[32];
  __shared__ uint32_t s_blk;
  __shared__ uint32_t s_prefix;
  if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t blk = s_blk;
  const uint64_t base = (uint64_t)blk * kScanTile + (uint64_t)threadIdx.x * kScanItems;

  // each thread's kScanItems consecutive words as 16-byte vectors (base is a multiple of 16 words)
  static_assert(kScanItems % 4 == 0, "vector loads");
  uint32_t v[kScanItems];
  uint32_t sum = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0 &&
                   base + kScanItems <= m;
  if (vec) {
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(in + base) + q);
      v[4 * q] = x.x;
      v[4 * q + 1] = x.y;
      v[4 * q + 2] = x.z;
      v[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) v[i] = (base + i < m) ? in[base + i] : 0u;
  }
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) sum += v[i];
  uint32_t agg;
  uint32_t texcl = block_excl_scan<kScanThreads>(sum, s_tmp, &agg);

  if (threadIdx.x == 0) {
    uint32_t excl = 0;
    if (blk == 0) {
      st_relaxed_u64(&status[0], kFlagPrefix | agg);
    } else {
      st_relaxed_u64(&status[blk], kFlagAggregate | agg);
      int64_t j = (int64_t)blk - 1;
      while (true) {
        uint64_t s = ld_relaxed_u64(&status[j]);
        uint32_t f = status_flag(s);
        if (f == 0) continue;
        excl += (uint32_t)s;
        if (f == 2) break;
        --j;
      }
      st_relaxed_u64(&status[blk], kFlagPrefix | (uint64_t)(excl + agg));
    }
    s_prefix = excl;
    if (total_out && (uint64_t)(blk + 1) * kScanTile >= m) *total_out = excl + agg;
  }
  __syncthreads();
  uint32_t run = s_prefix + texcl;
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
}

// Level-1 decomposition (K-c): byte-0 segment b = [B16[256 b], B16[256 (b+1)]) of the byte-0-ordered
// sequence; it is cut into ceil(len / chunk) chunks; cstart = exclusive scan of the chunk counts.
__global__ void kc_plan_chunks(const uint32_t* __restrict__ B16, uint64_t n, uint32_t chunk,
                               uint32_t* __restrict__ cstart) {
  __shared__ uint32_t s_tmp[32];
  const int b = threadIdx.x;  // 256 threads
  uint64_t beg = B16[b * 256];
  uint64_t end = (b < 255) ? B16[(b + 1) * 256] : n;
  uint32_t nch = (uint32_t)((end - beg + chunk - 1) / chunk);
  uint32_t total;
  uint32_t ex = block_excl_scan<256>(nch, s_tmp, &total);
  cstart[b] = ex;
  if (b == 0) cstart[256] = total;
}

// hist16[b] = sum of the kHistCopies copies (copy 0 is overwritten in place).
__global__ void kb_hist_reduce(uint32_t* __restrict__ hist, uint32_t copies) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= 65536) return;
  uint32_t s = 0;
  for (uint32_t c = 0; c < copies; ++c) s += hist[(size_t)c * 65536 + b];
  hist[b] = s;
}

// Copy one device counter into mapped pinned host memory with a store from the SM: the host reads a
// recursion level's big-bucket count without a copy-engine transfer, which would queue behind a large
// D2H on the copy engine (the streaming and external paths overlap sorts with such copies).
__global__ void kb_publish_u32(const uint32_t* __restrict__ src, volatile uint32_t* dst) { *dst = *src; }

}  // namespace

cudaError_t launch_publish_u32(const uint32_t* src, uint32_t* host_mapped_dev, cudaStream_t s) {
  kb_publish_u32<<<1, 1, 0, s>>>(src, host_mapped_dev);
  return cudaGetLastError();
}

cudaError_t launch_hist_reduce(uint32_t* hist, uint32_t copies, cudaStream_t s) {
  if (copies <= 1) return cudaSuccess;
  kb_hist_reduce<<<256, 256, 0, s>>>(hist, copies);
  return cudaGetLastError();
}

cudaError_t launch_scan_excl(const uint32_t* in, uint32_t* out, uint64_t m, uint64_t* status, uint32_t* ticket,
                             uint32_t* total_out, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  uint64_t blocks = (m + kScanTile - 1) / kScanTile;
  kb_scan_excl<<<(unsigned)blocks, kScanThreads, 0, s>>>(in, out, m, status, ticket, total_out);
  return cudaGetLastError();
}

uint64_t scan_status_words(uint64_t m) { return (m + kScanTile - 1) / kScanTile; }

cudaError_t launch_kc_plan_chunks(const uint32_t* B16, uint64_t n, uint32_t chunk, uint32_t* cstart,
                                  cudaStream_t s) {
  kc_plan_chunks<<<1, 256, 0, s>>>(B16, n, chunk, cstart);
  return cudaGetLastError();
}

}  // namespace ley
