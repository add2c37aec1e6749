// external.cu — the external path: pinned-host records larger than the device budget (SURVEY.md §8a
// rows a10-a12; BASELINE.json configs[4]).
//
// PAPER.md §3.2 lines 114-118 (Figure 1, "External Sort-Merge-Write Routine"): "in the sort stage,
// Leyenda reads and sorts records in small trunks and writes them down ... creating several sorted
// intermediate files. In the merge stage ... a reader thread pool [reads] one partition at a time ...
// merged by the merger thread to a globally sorted partition, using a K-way merge algorithm. Then the
// writer thread will write it to the final output file. The partitioning, in other words - load
// balancing process, makes it possible for read/merge/write threads to work simultaneously."
//
// B200 mapping (device memory capped by device_budget_bytes, P:19's memory limit):
//   a10 run generation: run r = input records [r C, (r+1) C) -> H2D -> internal sort (K-a..K-e) -> D2H
//       into pinned host run scratch; every S-th record of each sorted run is kept on the device as a
//       sample. Two device slots: while run r sorts, run r+1 streams in and run r-1 streams out (two
//       copy streams, full-duplex PCIe), so each direction of the host link stays busy.
//   a11 partition location: the samples are sorted (the internal sort again: sample order = (key, run,
//       pos)), every q-th one becomes a splitter, and K-loc binary-searches every sorted run for every
//       splitter directly in pinned host memory (zero-copy) -> exact slice bounds split[p][r].
//   a12 merge: partition p's R slices are copied H2D (concatenated in run order), turned into 16-byte
//       composite keys (key bytes 0..9, position in the concatenation = (run, pos) order), merged by a
//       ceil(log2 R)-level tree of 2-way merge-path merges (K-m), gathered (K-e style, device-local) and
//       copied D2H to out at the partition's offset. Two slots again: partition p+1's slices stream in
//       while p merges and p-1 streams out.
// Ties: records with equal keys from different runs come out in run order, within a run in position
// order — i.e. by global input index, which is the stable order.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "runtime.h"

namespace ley {
namespace {

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

// ---------------------------------------------------------------------------------------- kernels
// samples[base + s] = run[s * S] (full 100-byte records, 4-byte words)
__global__ void ext_take_samples(const uint32_t* __restrict__ run, uint64_t run_len, uint32_t S,
                                 uint32_t* __restrict__ samples, uint64_t base) {
  const uint64_t nsamp = (run_len + S - 1) / S;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nsamp * kRecordWords;
       w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = w / kRecordWords, o = w - s * kRecordWords;
    samples[(base + s) * kRecordWords + o] = run[s * S * kRecordWords + o];
  }
}

// perm of a run -> global ordinals (run base added)
__global__ void ext_add_base(uint32_t* __restrict__ p, uint64_t n, uint32_t base) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] += base;
}

struct Splitter {
  uint8_t key[12];   // key bytes 0..9 (+2 pad)
  uint32_t run;      // run of the splitter record
  uint64_t pos;      // its position in that run
};

// keys of kb <= 10 bytes (P:164 flexible key sizes): bytes [kb, 10) never decide
__device__ __forceinline__ int cmp_key(const uint8_t* a, const uint8_t* b, uint32_t kb) {
  for (uint32_t i = 0; i < kb; ++i) {
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  }
  return 0;
}

// split[p * R + r] = number of records of run r that precede splitter p in (key, run, pos) order.
// Binary search over the sorted run, reading keys from pinned host scratch (zero-copy).
__global__ void ext_locate(const uint8_t* __restrict__ scratch_dev, const uint64_t* __restrict__ run_off,
                           const uint64_t* __restrict__ run_len, uint32_t R, const Splitter* __restrict__ spl,
                           uint32_t nspl, uint32_t kb, uint64_t* __restrict__ split) {
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (uint64_t)nspl * R) return;
  const uint32_t p = (uint32_t)(id / R), r = (uint32_t)(id % R);
  const Splitter sp = spl[p];
  const uint8_t* base = scratch_dev + run_off[r] * kRecordBytes;
  uint64_t lo = 0, hi = run_len[r];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    uint8_t k[10];
    const uint8_t* rec = base + mid * kRecordBytes;
#pragma unroll
    for (int i = 0; i < 10; ++i) k[i] = rec[i];
    const int c = cmp_key(k, sp.key, kb);
    const bool before = c < 0 || (c == 0 && (r < sp.run || (r == sp.run && mid < sp.pos)));
    if (before) lo = mid + 1; else hi = mid;
  }
  split[id] = lo;
}

// composite key of element i of the concatenated slice buffer: (key bytes 0..7 BE, bytes 8..9 << 48 | i),
// key bytes [kb, 10) zeroed (keys shorter than 10 bytes: ties then fall to (run, pos) = the slice order)
__global__ void ext_make_comp(const uint8_t* __restrict__ recs, uint64_t m, uint32_t kb, uint64_t* __restrict__ hi,
                              uint64_t* __restrict__ lo) {
  const uint64_t mhi = kb >= 8 ? ~0ull : ~(~0ull >> (8 * kb));
  const uint64_t mlo = kb >= 10 ? 0xFFFFull : (kb == 9 ? 0xFF00ull : 0ull);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(recs + i * kRecordBytes);
    const uint32_t a = w[0], b = w[1], c = w[2];
    hi[i] = (((uint64_t)bswap32(a) << 32) | bswap32(b)) & mhi;
    lo[i] = ((uint64_t)(((c & 0xFFu) << 8) | ((c >> 8) & 0xFFu)) & mlo) << 48 | i;
  }
}

__device__ __forceinline__ bool comp_less(uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl) {
  return ah < bh || (ah == bh && al < bl);
}

// One level of the K-m merge tree: adjacent sequence pairs (bnd[2q], bnd[2q+1], bnd[2q+2]) are merged
// into the same output range. Each thread owns kMergeItems consecutive outputs: one merge-path binary
// search on its start diagonal, then a sequential merge.
constexpr int kMergeItems = 16;
__global__ void ext_merge_level(const uint64_t* __restrict__ ih, const uint64_t* __restrict__ il,
                                uint64_t* __restrict__ oh, uint64_t* __restrict__ ol, uint64_t m,
                                const uint64_t* __restrict__ bnd, uint32_t K) {
  const uint64_t j0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kMergeItems;
  if (j0 >= m) return;
  const uint64_t j1 = min(m, j0 + kMergeItems);
  uint64_t j = j0;
  while (j < j1) {
    // pair q containing output j: largest q with bnd[2q] <= j
    uint32_t qlo = 0, qhi = (K + 1) / 2;
    while (qhi - qlo > 1) {
      uint32_t mid = (qlo + qhi) >> 1;
      if (bnd[2 * mid] <= j) qlo = mid; else qhi = mid;
    }
    const uint32_t q = qlo;
    const uint64_t a0 = bnd[2 * q];
    const uint64_t a1 = (2 * q + 1 <= K) ? bnd[min(2 * q + 1, K)] : a0;
    const uint64_t b1 = (2 * q + 2 <= K) ? bnd[2 * q + 2] : a1;
    const uint64_t lenA = a1 - a0, lenB = b1 - a1;
    const uint64_t diag = j - a0;
    uint64_t lo = diag > lenB ? diag - lenB : 0, hi = min(diag, lenA);
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      const uint64_t bi = a1 + diag - 1 - mid;
      if (comp_less(ih[a0 + mid], il[a0 + mid], ih[bi], il[bi])) lo = mid + 1; else hi = mid;
    }
    uint64_t ia = a0 + lo, ib = a1 + (diag - lo);
    const uint64_t jend = min(j1, b1);
    for (; j < jend; ++j) {
      bool takeA;
      if (ia >= a1) takeA = false;
      else if (ib >= b1) takeA = true;
      else takeA = comp_less(ih[ia], il[ia], ih[ib], il[ib]);
      if (takeA) {
        oh[j] = ih[ia];
        ol[j] = il[ia];
        ++ia;
      } else {
        oh[j] = ih[ib];
        ol[j] = il[ib];
        ++ib;
      }
    }
  }
}

// out[j] = slice[pos_j], pos_j = low 48 bits of the merged composite (device-local gather, word stream)
__global__ void ext_gather(const uint32_t* __restrict__ slice, const uint64_t* __restrict__ lo, uint64_t m,
                           uint32_t* __restrict__ out, const uint32_t* __restrict__ pslice, uint32_t* __restrict__ pout) {
  const uint64_t words = m * kRecordWords;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = w / kRecordWords, o = w - j * kRecordWords;
    const uint64_t p = lo[j] & 0xFFFFFFFFFFFFull;
    out[w] = slice[p * kRecordWords + o];
    if (pout && o == 0) pout[j] = pslice[p];
  }
}

// ------------------------------------------------------------------ key-pointer form (option ext_keyptr)
// SURVEY §8f NEXT 3, the paper's own §3.2 pattern ("radix sort ... on key-pointer tuples only";
// P:104-106 the records are then scattered given the sorted tuples): runs hold 16-byte (key, ordinal)
// tuples instead of 100-byte records, and the merge gathers every output record from the caller's pinned
// input by its ordinal. Tuple: x,y = key bytes 0..7 big-endian (y = high word), z = key bytes 8..9
// big-endian (bytes [kb, 10) zeroed), w = global ordinal.
__device__ __forceinline__ void key_masks(uint32_t kb, uint64_t& mhi, uint32_t& m89) {
  mhi = kb >= 8 ? ~0ull : ~(~0ull >> (8 * kb));
  m89 = kb >= 10 ? 0xFFFFu : (kb == 9 ? 0xFF00u : 0u);
}

// tuples of a sorted run: t[j] = (key of run record perm[j], base + perm[j])
__global__ void ext_make_tuples(const uint8_t* __restrict__ recs, const uint32_t* __restrict__ perm, uint64_t len,
                                uint32_t base, uint32_t kb, uint4* __restrict__ t) {
  uint64_t mhi;
  uint32_t m89;
  key_masks(kb, mhi, m89);
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[j];
    const uint32_t* w = reinterpret_cast<const uint32_t*>(recs + (uint64_t)p * kRecordBytes);
    const uint32_t a = w[0], b = w[1], c = w[2];
    const uint64_t hi = (((uint64_t)bswap32(a) << 32) | bswap32(b)) & mhi;
    t[j] = make_uint4((uint32_t)hi, (uint32_t)(hi >> 32), ((((c & 0xFFu) << 8) | ((c >> 8) & 0xFFu)) & m89), base + p);
  }
}

// samples[base + s] = a 100-byte pseudo-record carrying the key of tuple s * S (the sample sort orders by
// key, then sample index = (run, pos) order)
__global__ void ext_take_tuple_samples(const uint4* __restrict__ t, uint64_t run_len, uint32_t S,
                                       uint8_t* __restrict__ samples, uint64_t base) {
  const uint64_t nsamp = (run_len + S - 1) / S;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nsamp; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = t[s * S];
    uint32_t* r = reinterpret_cast<uint32_t*>(samples + (base + s) * kRecordBytes);
    r[0] = bswap32(v.y);
    r[1] = bswap32(v.x);
    r[2] = ((v.z >> 8) & 0xFFu) | ((v.z & 0xFFu) << 8);
  }
}

// ext_locate over tuple runs (16-byte stride in the zero-copy scratch)
__global__ void ext_locate_tuples(const uint4* __restrict__ scratch_dev, const uint64_t* __restrict__ run_off,
                                  const uint64_t* __restrict__ run_len, uint32_t R, const Splitter* __restrict__ spl,
                                  uint32_t nspl, uint32_t kb, uint64_t* __restrict__ split) {
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (uint64_t)nspl * R) return;
  const uint32_t p = (uint32_t)(id / R), r = (uint32_t)(id % R);
  const Splitter sp = spl[p];
  const uint4* base = scratch_dev + run_off[r];
  uint64_t lo = 0, hi = run_len[r];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    const uint4 v = base[mid];
    uint8_t k[10];
    const uint64_t h = ((uint64_t)v.y << 32) | v.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) k[i] = (uint8_t)(h >> (56 - 8 * i));
    k[8] = (uint8_t)(v.z >> 8);
    k[9] = (uint8_t)v.z;
    const int c = cmp_key(k, sp.key, kb);
    const bool before = c < 0 || (c == 0 && (r < sp.run || (r == sp.run && mid < sp.pos)));
    if (before) lo = mid + 1; else hi = mid;
  }
  split[id] = lo;
}

// merge composites of a concatenated tuple slice: (key bytes 0..7, bytes 8..9 << 48 | position)
__global__ void ext_make_comp_tuples(const uint4* __restrict__ t, uint64_t m, uint64_t* __restrict__ hi,
                                     uint64_t* __restrict__ lo) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = t[i];
    hi[i] = ((uint64_t)v.y << 32) | v.x;
    lo[i] = (uint64_t)v.z << 48 | i;
  }
}

// out[j] = in[ordinal of the merged tuple j], read from the caller's pinned input through its device
// mapping (zero-copy over the host link). Random 100-byte reads over PCIe need few, large requests: one TMA
// bulk copy of the record's 16-byte-aligned 112-byte window per record (16-byte pieces were 2-3x slower),
// two groups of 32 records in flight per warp (mbarrier completion); a window that would pass the input's
// end (the last record or two) is read with exact 4-byte loads instead.
__device__ __forceinline__ void xg_mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}"
               ::"r"(a), "r"(parity) : "memory");
}
__global__ void __launch_bounds__(128) ext_gather_host(const uint8_t* __restrict__ in, uint64_t in_bytes,
                                                       const uint4* __restrict__ t, const uint64_t* __restrict__ lo,
                                                       uint64_t m, uint8_t* __restrict__ out, uint32_t* __restrict__ pout) {
  constexpr int kWin = 112, kSlot = 128;
  __shared__ __align__(128) uint8_t stage[4][2][32 * kSlot];  // 4 warps per CTA
  __shared__ uint32_t s_p[4][2][32];
  __shared__ __align__(8) uint64_t s_mb[4][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&s_mb[w][0]);
  if (lane < 2) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8 * lane) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t ngroups = (m + 31) / 32, nw = (uint64_t)gridDim.x * 4;
  auto issue = [&](uint64_t g, int st) {
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, m - j0);
    const uint32_t p = lane < (int)cnt ? t[lo[j0 + lane] & 0xFFFFFFFFFFFFull].w : 0u;
    s_p[w][st][lane] = p;
    if (pout && lane < (int)cnt) pout[j0 + lane] = p;
    const uint64_t a = ((uint64_t)p * kRecordBytes) & ~uint64_t(15);
    const bool bulk = lane < (int)cnt && a + kWin <= in_bytes;
    const uint32_t nbulk = __popc(__ballot_sync(0xffffffffu, bulk));
    const uint32_t mb = mb0 + 8 * st;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(nbulk * kWin) : "memory");
    __syncwarp();
    uint8_t* slot = stage[w][st] + lane * kSlot;
    if (bulk) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"((uint32_t)__cvta_generic_to_shared(slot)), "l"(in + a), "r"(kWin), "r"(mb) : "memory");
    } else if (lane < (int)cnt) {  // the input's last record(s): exact loads
      const uint32_t* src = reinterpret_cast<const uint32_t*>(in + (uint64_t)p * kRecordBytes);
      uint32_t* dst = reinterpret_cast<uint32_t*>(slot + ((p * 4u) & 15u));
      for (int o = 0; o < (int)kRecordWords; ++o) dst[o] = src[o];
    }
  };
  const uint64_t g_first = (uint64_t)blockIdx.x * 4 + w;
  if (g_first < ngroups) issue(g_first, 0);
  uint32_t phases = 0;
  int st = 0;
  for (uint64_t g = g_first; g < ngroups; g += nw) {
    if (g + nw < ngroups) issue(g + nw, st ^ 1);
    xg_mbar_wait(mb0 + 8 * st, (phases >> st) & 1u);
    phases ^= 1u << st;
    __syncwarp();
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, m - j0);
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + j0 * kRecordBytes);
    for (uint32_t x = lane; x < cnt * kRecordWords; x += 32) {
      const uint32_t r = x / kRecordWords, o = x - r * kRecordWords;
      dst[x] = *reinterpret_cast<const uint32_t*>(stage[w][st] + r * kSlot + ((s_p[w][st][r] * 4u) & 15u) + 4 * o);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    st ^= 1;
  }
}

// LEY_TRACE_EXT=1: events around every copy / sort of the external path; per-category busy time and
// span printed to stderr at the end (diagnostics only; never on by default).
struct ExtTrace {
  bool on = getenv("LEY_TRACE_EXT") != nullptr;
  cudaEvent_t origin = nullptr;
  struct Span { const char* cat; cudaEvent_t a, b; };
  std::vector<Span> spans;
  void start(cudaStream_t st) {
    if (!on) return;
    cudaEventCreate(&origin);
    cudaEventRecord(origin, st);
  }
  size_t begin(const char* cat, cudaStream_t st) {
    if (!on) return 0;
    Span sp{cat, nullptr, nullptr};
    cudaEventCreate(&sp.a);
    cudaEventCreate(&sp.b);
    cudaEventRecord(sp.a, st);
    spans.push_back(sp);
    return spans.size() - 1;
  }
  void end(size_t i, cudaStream_t st) {
    if (on) cudaEventRecord(spans[i].b, st);
  }
  void report() {
    if (!on) return;
    cudaDeviceSynchronize();
    std::vector<std::string> cats;
    for (auto& sp : spans) {
      bool seen = false;
      for (auto& c : cats) seen |= c == sp.cat;
      if (!seen) cats.push_back(sp.cat);
    }
    for (auto& c : cats) {
      float busy = 0, first = 1e30f, last = 0;
      int cnt = 0;
      for (auto& sp : spans) {
        if (c != sp.cat) continue;
        float a = 0, b = 0, d = 0;
        cudaEventElapsedTime(&a, origin, sp.a);
        cudaEventElapsedTime(&b, origin, sp.b);
        cudaEventElapsedTime(&d, sp.a, sp.b);
        busy += d;
        first = std::min(first, a);
        last = std::max(last, b);
        ++cnt;
      }
      fprintf(stderr, "[ext trace] %-12s n=%4d busy %8.2f ms  span [%8.2f, %8.2f] ms\n", c.c_str(), cnt, busy, first,
              last);
    }
    for (auto& sp : spans) {
      cudaEventDestroy(sp.a);
      cudaEventDestroy(sp.b);
    }
    cudaEventDestroy(origin);
  }
};

unsigned grid_for(uint64_t work, int sms, int per_sm = 8) {
  uint64_t b = (work + 255) / 256;
  uint64_t cap = (uint64_t)sms * per_sm;
  return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

// ---------------------------------------------------------------------------------------- phases
// Sorted runs in a pinned (mapped) host scratch. Record j of the global layout sits at h_runs + 100 j; run
// k covers [off[k], off[k] + len[k]) and was sampled every S[k]-th record (its first sample is sample
// number samp_base[k] of the run-ordered sample set). With one GPU the layout is the input's; with G ranks
// the runs of rank r sit at its global offset (ranks' runs in rank order = global input order).
struct RunSet {
  uint8_t* h_runs = nullptr;
  uint8_t* h_runs_dev = nullptr;
  uint32_t* h_perm = nullptr;  // global ordinals of the run records (perm requested)
  bool kp = false;             // key-pointer form: runs of 16-byte tuples (option ext_keyptr)
  const uint8_t* in_dev = nullptr;  // kp: the caller's pinned input through its device mapping
  uint64_t in_bytes = 0;
  std::vector<uint64_t> off, len, S, samp_base;
  uint64_t nsamp = 0;
};

// Phase-1 device buffers: two run slots (in | out), the inner sort's workspace, two run perms, and the
// sample area (samples, sorted samples, sample perm, sample-sort workspace) for up to `nsamp_cap` samples.
struct Phase1 {
  uint8_t* d_in[2];
  uint8_t* d_out[2];
  uint8_t* d_work;
  uint32_t* d_run_perm[2];
  uint8_t* d_samp;
  uint8_t* d_samp_sorted;
  uint32_t* d_samp_perm;
  uint8_t* d_work2;
  size_t work_bytes, work2_bytes;
};

size_t phase1_bytes(uint64_t C, uint64_t nsamp_cap) {
  return 4 * a256(C * kRecordBytes) + a256(plan_internal(C).bytes) + 2 * a256(nsamp_cap * kRecordBytes) +
         a256(4 * nsamp_cap) + 2 * a256(4 * C) + a256(plan_internal(nsamp_cap).bytes);
}

Phase1 phase1_layout(uint8_t* eb, uint64_t C, uint64_t nsamp_cap) {
  Phase1 b;
  const size_t sz_run = a256(C * kRecordBytes), sz_samples = a256(nsamp_cap * kRecordBytes);
  b.d_in[0] = eb;
  b.d_in[1] = eb + sz_run;
  b.d_out[0] = eb + 2 * sz_run;
  b.d_out[1] = eb + 3 * sz_run;
  b.d_work = eb + 4 * sz_run;
  b.work_bytes = plan_internal(C).bytes;
  b.d_samp = b.d_work + a256(b.work_bytes);
  b.d_samp_sorted = b.d_samp + sz_samples;
  b.d_samp_perm = reinterpret_cast<uint32_t*>(b.d_samp_sorted + sz_samples);
  b.d_run_perm[0] = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(b.d_samp_perm) + a256(4 * nsamp_cap));
  b.d_run_perm[1] = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(b.d_run_perm[0]) + a256(4 * C));
  b.d_work2 = reinterpret_cast<uint8_t*>(b.d_run_perm[1]) + a256(4 * C);
  b.work2_bytes = plan_internal(nsamp_cap).bytes;
  return b;
}

// a10: input records [0, n) of `in` (global records [gbase, gbase + n)) -> sorted runs of C records in
// rs.h_runs at their global offsets; samples appended to b.d_samp at rs.nsamp.
ley_status ext_generate(DeviceContext& ctx, const uint8_t* in, uint64_t n, uint64_t gbase, uint64_t C, uint64_t S,
                        RunSet& rs, const Phase1& b, bool want_perm, uint32_t key_bytes, cudaStream_t s,
                        Profiler& prof, ExtTrace& tr) {
  ley_status st;
  const int sms = ctx.sms;
  const size_t first = rs.off.size();
  for (uint64_t at = 0; at < n; at += C) {
    rs.off.push_back(gbase + at);
    rs.len.push_back(std::min<uint64_t>(C, n - at));
    rs.S.push_back(S);
    rs.samp_base.push_back(rs.nsamp);
    rs.nsamp += (rs.len.back() + S - 1) / S;
  }
  const uint32_t R = (uint32_t)(rs.off.size() - first);
  cudaStream_t h2d = ctx.copy_stream[0], d2h = ctx.copy_stream[1];
  // per slot: input landed, slot sorted (input free, output ready), output copied out (output free)
  cudaEvent_t ev_start = ctx.ev[0];
  cudaEvent_t ev_in[2] = {ctx.ev[1], ctx.ev[2]}, ev_sorted[2] = {ctx.ev[3], ctx.ev[4]},
              ev_out[2] = {ctx.ev[5], ctx.ev[6]};
  LEY_CUDA("ext runs", cudaEventRecord(ev_start, s));
  LEY_CUDA("ext runs", cudaStreamWaitEvent(h2d, ev_start, 0));
  LEY_CUDA("ext runs", cudaStreamWaitEvent(d2h, ev_start, 0));
  Profiler quiet;  // inner sorts are not profiled stage by stage
  quiet.ctx = &ctx;
  quiet.stream = s;
  // H2D of run r into slot r & 1, once run r-2 (same slot) has been sorted
  auto issue_run_h2d = [&](uint32_t r) -> ley_status {
    const int sl = r & 1;
    if (r >= 2) LEY_CUDA("ext runs", cudaStreamWaitEvent(h2d, ev_sorted[sl], 0));
    const size_t t_h = tr.begin("run H2D", h2d);
    LEY_CUDA("ext H2D", cudaMemcpyAsync(b.d_in[sl], in + (rs.off[first + r] - gbase) * kRecordBytes,
                                        rs.len[first + r] * kRecordBytes, cudaMemcpyHostToDevice, h2d));
    tr.end(t_h, h2d);
    LEY_CUDA("ext runs", cudaEventRecord(ev_in[sl], h2d));
    return LEY_OK;
  };
  if (R && (st = issue_run_h2d(0))) return st;
  for (uint32_t r = 0; r < R; ++r) {
    const size_t k = first + r;
    const uint64_t len = rs.len[k];
    const int sl = r & 1;
    // queue the next run's input before this run's sort blocks the host on its own stream
    if (r + 1 < R && (st = issue_run_h2d(r + 1))) return st;
    LEY_CUDA("ext runs", cudaStreamWaitEvent(s, ev_in[sl], 0));
    if (r >= 2) LEY_CUDA("ext runs", cudaStreamWaitEvent(s, ev_out[sl], 0));  // d_out[sl] copied out
    const size_t t_s = tr.begin("run sort", s);
    if (rs.kp) {  // key-pointer form: perm-only sort (no gather), then the run's sorted (key, ordinal) tuples
      st = sort_internal_device(ctx, b.d_in[sl], nullptr, b.d_run_perm[sl], len, s, quiet, b.d_work, b.work_bytes,
                                key_bytes);
      if (st) return st;
      ext_make_tuples<<<grid_for(len, sms), 256, 0, s>>>(b.d_in[sl], b.d_run_perm[sl], len, (uint32_t)rs.off[k],
                                                         key_bytes, reinterpret_cast<uint4*>(b.d_out[sl]));
      LEY_CUDA("ext tuples", cudaGetLastError());
      ext_take_tuple_samples<<<grid_for((len + S - 1) / S, sms), 256, 0, s>>>(
          reinterpret_cast<const uint4*>(b.d_out[sl]), len, (uint32_t)S, b.d_samp, rs.samp_base[k]);
      LEY_CUDA("ext samples", cudaGetLastError());
      prof.launches += quiet.launches + 2;
      quiet.launches = 0;
      tr.end(t_s, s);
      LEY_CUDA("ext runs", cudaEventRecord(ev_sorted[sl], s));
      LEY_CUDA("ext runs", cudaStreamWaitEvent(d2h, ev_sorted[sl], 0));
      const size_t t_d = tr.begin("run D2H", d2h);
      LEY_CUDA("ext D2H", cudaMemcpyAsync(rs.h_runs + rs.off[k] * 16, b.d_out[sl], len * 16, cudaMemcpyDeviceToHost, d2h));
      tr.end(t_d, d2h);
      LEY_CUDA("ext runs", cudaEventRecord(ev_out[sl], d2h));
      continue;
    }
    st = sort_internal_device(ctx, b.d_in[sl], b.d_out[sl], want_perm ? b.d_run_perm[sl] : nullptr, len, s, quiet,
                              b.d_work, b.work_bytes, key_bytes);
    if (st) return st;
    tr.end(t_s, s);
    prof.launches += quiet.launches;
    quiet.launches = 0;
    ext_take_samples<<<grid_for((len + S - 1) / S * kRecordWords, sms), 256, 0, s>>>(
        reinterpret_cast<const uint32_t*>(b.d_out[sl]), len, (uint32_t)S, reinterpret_cast<uint32_t*>(b.d_samp),
        rs.samp_base[k]);
    LEY_CUDA("ext samples", cudaGetLastError());
    prof.launches += 1;
    if (want_perm) {
      ext_add_base<<<grid_for(len, sms), 256, 0, s>>>(b.d_run_perm[sl], len, (uint32_t)rs.off[k]);
      LEY_CUDA("ext perm", cudaGetLastError());
      prof.launches += 1;
    }
    LEY_CUDA("ext runs", cudaEventRecord(ev_sorted[sl], s));
    LEY_CUDA("ext runs", cudaStreamWaitEvent(d2h, ev_sorted[sl], 0));
    const size_t t_d = tr.begin("run D2H", d2h);
    LEY_CUDA("ext D2H", cudaMemcpyAsync(rs.h_runs + rs.off[k] * kRecordBytes, b.d_out[sl], len * kRecordBytes,
                                        cudaMemcpyDeviceToHost, d2h));
    tr.end(t_d, d2h);
    if (want_perm)
      LEY_CUDA("ext D2H", cudaMemcpyAsync(rs.h_perm + rs.off[k], b.d_run_perm[sl], len * 4, cudaMemcpyDeviceToHost, d2h));
    LEY_CUDA("ext runs", cudaEventRecord(ev_out[sl], d2h));
  }
  LEY_CUDA("ext runs", cudaEventRecord(ev_start, d2h));  // every run copied out
  LEY_CUDA("ext runs", cudaStreamWaitEvent(s, ev_start, 0));
  return LEY_OK;
}

// a11: splitters from the run-ordered samples b.d_samp[0, rs.nsamp) (sorted: order = (key, run, pos)),
// every q-th one a splitter; exact slice bounds split[p * R + k] of every run by K-loc. part_off[p] =
// first global output position of partition p.
ley_status ext_partition(DeviceContext& ctx, const RunSet& rs, const Phase1& b, uint64_t q, uint32_t key_bytes,
                         cudaStream_t s, Profiler& prof, uint32_t* P_out, std::vector<uint64_t>& split,
                         std::vector<uint64_t>& part_off) {
  const uint32_t R = (uint32_t)rs.off.size();
  const uint32_t P = (uint32_t)std::max<uint64_t>(1, (rs.nsamp + q - 1) / q);
  std::vector<Splitter> spl(P > 1 ? P - 1 : 0);
  split.assign((size_t)(P + 1) * R, 0);
  for (uint32_t r = 0; r < R; ++r) split[(size_t)P * R + r] = rs.len[r];
  if (P > 1) {
    Profiler quiet;
    quiet.ctx = &ctx;
    quiet.stream = s;
    ley_status st = sort_internal_device(ctx, b.d_samp, b.d_samp_sorted, b.d_samp_perm, rs.nsamp, s, quiet, b.d_work2,
                                         b.work2_bytes, key_bytes);
    if (st) return st;
    prof.launches += quiet.launches;
    std::vector<uint32_t> sidx(P - 1);
    for (uint32_t p = 1; p < P; ++p) {
      const uint64_t at = (uint64_t)p * q;
      LEY_CUDA("ext splitters", cudaMemcpyAsync(&sidx[p - 1], b.d_samp_perm + at, 4, cudaMemcpyDeviceToHost, s));
      LEY_CUDA("ext splitters", cudaMemcpyAsync(spl[p - 1].key, b.d_samp_sorted + at * kRecordBytes, 10,
                                                cudaMemcpyDeviceToHost, s));
    }
    LEY_CUDA("ext splitters", cudaStreamSynchronize(s));
    for (uint32_t p = 1; p < P; ++p) {
      const uint32_t r = (uint32_t)(std::upper_bound(rs.samp_base.begin(), rs.samp_base.end(), (uint64_t)sidx[p - 1]) -
                                    rs.samp_base.begin() - 1);
      spl[p - 1].run = r;
      spl[p - 1].pos = (sidx[p - 1] - rs.samp_base[r]) * rs.S[r];
    }
    // the run offsets relative to the scratch base: ext_locate reads run r at h_runs_dev + 100 off[r]
    Splitter* d_spl = reinterpret_cast<Splitter*>(b.d_work);
    uint64_t* d_runoff = reinterpret_cast<uint64_t*>(b.d_work + a256(sizeof(Splitter) * spl.size()));
    uint64_t* d_runlen = d_runoff + R;
    uint64_t* d_split = d_runlen + R;
    LEY_CUDA("ext locate", cudaMemcpyAsync(d_spl, spl.data(), sizeof(Splitter) * spl.size(), cudaMemcpyHostToDevice, s));
    LEY_CUDA("ext locate", cudaMemcpyAsync(d_runoff, rs.off.data(), 8 * R, cudaMemcpyHostToDevice, s));
    LEY_CUDA("ext locate", cudaMemcpyAsync(d_runlen, rs.len.data(), 8 * R, cudaMemcpyHostToDevice, s));
    const uint64_t nthreads = (uint64_t)(P - 1) * R;
    if (rs.kp)
      ext_locate_tuples<<<(unsigned)((nthreads + 127) / 128), 128, 0, s>>>(reinterpret_cast<const uint4*>(rs.h_runs_dev),
                                                                           d_runoff, d_runlen, R, d_spl, P - 1, key_bytes,
                                                                           d_split);
    else
      ext_locate<<<(unsigned)((nthreads + 127) / 128), 128, 0, s>>>(rs.h_runs_dev, d_runoff, d_runlen, R, d_spl, P - 1,
                                                                    key_bytes, d_split);
    LEY_CUDA("ext locate", cudaGetLastError());
    prof.launches += 1;
    LEY_CUDA("ext locate", cudaMemcpyAsync(split.data() + R, d_split, 8 * nthreads, cudaMemcpyDeviceToHost, s));
    LEY_CUDA("ext locate", cudaStreamSynchronize(s));
  }
  part_off.assign(P + 1, 0);
  for (uint32_t p = 0; p < P; ++p) {
    uint64_t m = 0;
    for (uint32_t r = 0; r < R; ++r) m += split[(size_t)(p + 1) * R + r] - split[(size_t)p * R + r];
    part_off[p + 1] = part_off[p] + m;
  }
  *P_out = P;
  return LEY_OK;
}

// a12: K-way merge of partitions [p_begin, p_end); partition p lands at out + 100 (part_off[p] -
// part_off[p_begin]) (perm_out likewise).
ley_status ext_merge(DeviceContext& ctx, const RunSet& rs, const std::vector<uint64_t>& split,
                     const std::vector<uint64_t>& part_off, uint32_t p_begin, uint32_t p_end, uint8_t* out,
                     uint32_t* perm_out, uint32_t key_bytes, cudaStream_t s, Profiler& prof, ExtTrace& tr,
                     uint64_t clip_lo = 0, uint64_t clip_hi = ~0ull) {
  // only global output positions [clip_lo, clip_hi) are written, at out + 100 (pos - max(clip_lo,
  // part_off[p_begin])) — a rank of the multi-GPU external sort keeps its exact share of the boundary
  // partitions it merges
  ley_status st;
  const uint32_t R = (uint32_t)rs.off.size();
  const int sms = ctx.sms;
  cudaStream_t h2d = ctx.copy_stream[0], d2h = ctx.copy_stream[1];
  cudaEvent_t ev_start = ctx.ev[0];
  cudaEvent_t ev_in[2] = {ctx.ev[1], ctx.ev[2]}, ev_sorted[2] = {ctx.ev[3], ctx.ev[4]},
              ev_out[2] = {ctx.ev[5], ctx.ev[6]};
  uint64_t m_max = 0;
  std::vector<uint32_t> parts;  // non-empty partitions, merged in order
  for (uint32_t p = p_begin; p < p_end; ++p) {
    m_max = std::max(m_max, part_off[p + 1] - part_off[p]);
    if (part_off[p + 1] > part_off[p]) parts.push_back(p);
  }
  const size_t elem = rs.kp ? 16 : kRecordBytes;  // a run element: a tuple or a record
  const size_t sz_slice = a256(m_max * elem);
  const size_t sz_mout = a256(m_max * kRecordBytes);
  const size_t sz_comp = a256(m_max * 8);
  const size_t sz_p = perm_out ? a256(m_max * 4) : 0;
  // merge-tree boundaries of every level of every partition, computed once on the host and copied to the
  // device in one transfer (no host round trip between levels): level 0 = the R slice starts in the
  // concatenation; level l+1 keeps every other boundary of level l (adjacent pairs merged)
  const size_t bstride = 2 * (size_t)(R + 1) + 64;
  std::vector<uint64_t> hb(parts.size() * bstride, 0);
  std::vector<std::vector<std::pair<size_t, uint32_t>>> levels(parts.size());  // (offset in hb, K)
  for (size_t i = 0; i < parts.size(); ++i) {
    const uint32_t p = parts[i];
    std::vector<uint64_t> cur(R + 1);
    uint64_t at = 0;
    for (uint32_t r = 0; r < R; ++r) {
      cur[r] = at;
      at += split[(size_t)(p + 1) * R + r] - split[(size_t)p * R + r];
    }
    cur[R] = at;
    size_t o = i * bstride;
    std::copy(cur.begin(), cur.end(), hb.begin() + o);  // level 0 also gives the slice offsets
    while (cur.size() > 2) {
      std::copy(cur.begin(), cur.end(), hb.begin() + o);
      levels[i].push_back({o, (uint32_t)cur.size() - 1});
      o += cur.size();
      std::vector<uint64_t> nxt;
      for (size_t k = 0; k < cur.size(); k += 2) nxt.push_back(cur[k]);
      if (nxt.back() != cur.back()) nxt.push_back(cur.back());
      cur.swap(nxt);
    }
  }
  const size_t phase2 = 2 * sz_slice + 2 * sz_mout + 4 * sz_comp + 4 * sz_p + a256(8 * hb.size());
  if (phase2 > ctx.ext.cap) {
    if ((st = ensure_buffer(ctx.ext, phase2, "external merge buffers", s))) return st;
  }
  uint8_t* eb = static_cast<uint8_t*>(ctx.ext.ptr);
  uint8_t* d_slice[2] = {eb, eb + sz_slice};
  uint8_t* d_mout[2] = {eb + 2 * sz_slice, eb + 2 * sz_slice + sz_mout};
  uint8_t* cb = eb + 2 * sz_slice + 2 * sz_mout;
  uint64_t* c_h[2] = {reinterpret_cast<uint64_t*>(cb), reinterpret_cast<uint64_t*>(cb + 2 * sz_comp)};
  uint64_t* c_l[2] = {reinterpret_cast<uint64_t*>(cb + sz_comp), reinterpret_cast<uint64_t*>(cb + 3 * sz_comp)};
  uint8_t* pb = cb + 4 * sz_comp;
  uint32_t* d_pslice[2] = {nullptr, nullptr};
  uint32_t* d_pout[2] = {nullptr, nullptr};
  if (perm_out) {
    for (int i = 0; i < 2; ++i) {
      d_pslice[i] = reinterpret_cast<uint32_t*>(pb + i * sz_p);
      d_pout[i] = reinterpret_cast<uint32_t*>(pb + (2 + i) * sz_p);
    }
  }
  uint64_t* d_bnd = reinterpret_cast<uint64_t*>(pb + 4 * sz_p);
  LEY_CUDA("ext merge", cudaMemcpyAsync(d_bnd, hb.data(), 8 * hb.size(), cudaMemcpyHostToDevice, s));
  LEY_CUDA("ext merge", cudaStreamSynchronize(s));
  // H2D of the i-th partition's R slices into slot i & 1, once partition i-2 (same slot) is gathered
  auto issue_slices = [&](size_t i) -> ley_status {
    const uint32_t p = parts[i];
    const int sl = i & 1;
    if (i >= 2) LEY_CUDA("ext merge", cudaStreamWaitEvent(h2d, ev_sorted[sl], 0));
    const uint64_t* off0 = hb.data() + i * bstride;  // slice r lands at off0[r]
    const size_t t_mh = tr.begin("merge H2D", h2d);
    for (uint32_t r = 0; r < R; ++r) {
      const uint64_t lo = split[(size_t)p * R + r], hi = split[(size_t)(p + 1) * R + r];
      const uint64_t at = off0[r];
      if (hi > lo) {
        LEY_CUDA("ext merge H2D", cudaMemcpyAsync(d_slice[sl] + at * elem, rs.h_runs + (rs.off[r] + lo) * elem,
                                                  (hi - lo) * elem, cudaMemcpyHostToDevice, h2d));
        if (perm_out && !rs.kp)
          LEY_CUDA("ext merge H2D", cudaMemcpyAsync(d_pslice[sl] + at, rs.h_perm + rs.off[r] + lo, (hi - lo) * 4,
                                                    cudaMemcpyHostToDevice, h2d));
      }
    }
    tr.end(t_mh, h2d);
    LEY_CUDA("ext merge", cudaEventRecord(ev_in[sl], h2d));
    return LEY_OK;
  };
  // the slices are read from the host run scratch: every run's D2H (which s has waited for) comes first
  LEY_CUDA("ext merge", cudaEventRecord(ctx.ev[7], s));
  LEY_CUDA("ext merge", cudaStreamWaitEvent(h2d, ctx.ev[7], 0));
  LEY_CUDA("ext merge", cudaStreamWaitEvent(d2h, ctx.ev[7], 0));
  if (!parts.empty() && (st = issue_slices(0))) return st;
  for (size_t i = 0; i < parts.size(); ++i) {
    const uint32_t p = parts[i];
    const int sl = i & 1;
    const uint64_t m = part_off[p + 1] - part_off[p];
    if (i + 1 < parts.size() && (st = issue_slices(i + 1))) return st;  // queued ahead of this merge
    LEY_CUDA("ext merge", cudaStreamWaitEvent(s, ev_in[sl], 0));
    if (i >= 2) LEY_CUDA("ext merge", cudaStreamWaitEvent(s, ev_out[sl], 0));  // d_mout[sl] copied out
    const size_t t_mm = tr.begin("merge K-m", s);
    if (rs.kp)
      ext_make_comp_tuples<<<grid_for(m, sms), 256, 0, s>>>(reinterpret_cast<const uint4*>(d_slice[sl]), m, c_h[0], c_l[0]);
    else
      ext_make_comp<<<grid_for(m, sms), 256, 0, s>>>(d_slice[sl], m, key_bytes, c_h[0], c_l[0]);
    LEY_CUDA("K-m merge", cudaGetLastError());
    prof.launches += 1;
    // merge tree over the R run slices: one launch per level, boundaries already on the device
    int src = 0;
    for (const auto& lv : levels[i]) {
      const uint64_t threads = (m + kMergeItems - 1) / kMergeItems;
      ext_merge_level<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(c_h[src], c_l[src], c_h[src ^ 1], c_l[src ^ 1],
                                                                        m, d_bnd + lv.first, lv.second);
      LEY_CUDA("K-m merge", cudaGetLastError());
      prof.launches += 1;
      src ^= 1;
    }
    if (rs.kp)  // the records come from the caller's pinned input, by the merged tuples' ordinals
      ext_gather_host<<<(unsigned)std::max<uint64_t>(1, std::min<uint64_t>((m + 127) / 128, (uint64_t)sms * 6)), 128, 0,
                        s>>>(rs.in_dev, rs.in_bytes, reinterpret_cast<const uint4*>(d_slice[sl]), c_l[src], m, d_mout[sl],
                             d_pout[sl]);
    else
      ext_gather<<<grid_for(m * kRecordWords, sms), 256, 0, s>>>(reinterpret_cast<const uint32_t*>(d_slice[sl]), c_l[src],
                                                                 m, reinterpret_cast<uint32_t*>(d_mout[sl]), d_pslice[sl],
                                                                 d_pout[sl]);
    LEY_CUDA("K-e gather", cudaGetLastError());
    prof.launches += 1;
    LEY_CUDA("ext merge", cudaEventRecord(ev_sorted[sl], s));
    LEY_CUDA("ext merge", cudaStreamWaitEvent(d2h, ev_sorted[sl], 0));
    tr.end(t_mm, s);
    const uint64_t base = std::max(clip_lo, part_off[p_begin]);
    const uint64_t w0 = std::max(part_off[p], clip_lo), w1 = std::min(part_off[p + 1], clip_hi);
    const size_t t_md = tr.begin("merge D2H", d2h);
    if (w1 > w0) {
      const uint64_t o = w0 - base, from = w0 - part_off[p], cnt = w1 - w0;
      LEY_CUDA("ext merge D2H", cudaMemcpyAsync(out + o * kRecordBytes, d_mout[sl] + from * kRecordBytes,
                                                cnt * kRecordBytes, cudaMemcpyDeviceToHost, d2h));
      if (perm_out)
        LEY_CUDA("ext merge D2H", cudaMemcpyAsync(perm_out + o, d_pout[sl] + from, cnt * 4, cudaMemcpyDeviceToHost, d2h));
    }
    tr.end(t_md, d2h);
    LEY_CUDA("ext merge", cudaEventRecord(ev_out[sl], d2h));
  }
  LEY_CUDA("ext merge", cudaEventRecord(ev_start, d2h));
  LEY_CUDA("ext merge", cudaStreamWaitEvent(s, ev_start, 0));
  return LEY_OK;
}

// partitions of about m_target records: every q-th sample (a partition holds at most (q + R) S records)
uint64_t ext_sample_q(uint64_t m_target, uint64_t S, uint64_t R) {
  uint64_t q = m_target / S > 2ull * R ? m_target / S - R : std::max<uint64_t>(1, m_target / (2 * S));
  return q ? q : 1;
}

}  // namespace

// Pinned, mapped host run scratch of the external paths (grow-only; freed by ley_release_cache).
ley_status ensure_host_scratch(DeviceContext& ctx, size_t bytes) {
  if (ctx.host_scratch_cap >= bytes) return LEY_OK;
  if (ctx.host_scratch) cudaFreeHost(ctx.host_scratch);
  ctx.host_scratch = nullptr;
  ctx.host_scratch_cap = 0;
  LEY_CUDA("external scratch", cudaHostAlloc(&ctx.host_scratch, bytes, cudaHostAllocMapped));
  ctx.host_scratch_cap = bytes;
  return LEY_OK;
}

// ---------------------------------------------------------------------------------------- driver
ley_status sort_external_host(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint32_t* perm_out, uint64_t n,
                              uint64_t budget, uint32_t key_bytes, cudaStream_t s, Profiler& prof) {
  ley_status st;
  if (key_bytes > kKeyBytes) {  // the merge compares 10-byte composites (K-m)
    set_error("external: keys longer than 10 bytes are not supported on the external path (raise the budget "
              "to the staged path's ley_plan_query().staged_bytes)");
    return LEY_ERR_UNSUPPORTED;
  }
  const uint64_t C = external_run_records(n, budget);
  if (C < 1024 && C < n) {
    set_error("external: device_budget_bytes " + std::to_string(budget) +
              " is below the minimum working set (runs of >= 1024 records)");
    return LEY_ERR_BUDGET;
  }
  const uint64_t R = (n + C - 1) / C;
  const uint64_t S = external_sample_stride(n, C, budget);  // sample stride (bounds every partition)
  const uint64_t nsamp_cap = R * ((C + S - 1) / S);
  if ((st = ensure_buffer(ctx.ext, phase1_bytes(C, nsamp_cap), "external buffers", s))) return st;
  const Phase1 b = phase1_layout(static_cast<uint8_t*>(ctx.ext.ptr), C, nsamp_cap);
  // pinned host run scratch (records, and global ordinals when perm is requested)
  RunSet rs;
  rs.kp = options_snapshot().ext_keyptr != 0;
  if (rs.kp) {  // key-pointer form: the records are gathered from the input itself, through its device mapping
    if (cudaHostGetDevicePointer((void**)&rs.in_dev, const_cast<uint8_t*>(in), 0) != cudaSuccess || !rs.in_dev) {
      cudaGetLastError();
      set_error("external (ext_keyptr): the input is not mapped pinned memory (cudaHostGetDevicePointer failed)");
      return LEY_ERR_UNSUPPORTED;
    }
    rs.in_bytes = n * kRecordBytes;
  }
  // pinned host run scratch: records (+ global ordinals when perm is requested), or 16-byte tuples
  if ((st = ensure_host_scratch(ctx, rs.kp ? (size_t)n * 16
                                           : (size_t)n * kRecordBytes + (perm_out ? (size_t)n * 4 : 0))))
    return st;
  rs.h_runs = static_cast<uint8_t*>(ctx.host_scratch);
  rs.h_perm = perm_out && !rs.kp ? reinterpret_cast<uint32_t*>(rs.h_runs + (size_t)n * kRecordBytes) : nullptr;
  LEY_CUDA("external scratch", cudaHostGetDevicePointer((void**)&rs.h_runs_dev, rs.h_runs, 0));
  if ((st = ensure_copy_streams(ctx))) return st;
  ExtTrace tr;
  tr.start(s);

  if ((st = prof.begin("ext run generation"))) return st;
  if ((st = ext_generate(ctx, in, n, 0, C, S, rs, b, perm_out != nullptr, key_bytes, s, prof, tr))) return st;
  if ((st = prof.end())) return st;

  if ((st = prof.begin("ext partition"))) return st;
  // merge-phase device plan: a partition of m records needs two slots of slice (100 m) + out (100 m)
  // (partition p+1 streams in and p-1 streams out while p merges) + 2 x 16 m composites (+ 16 m perm);
  // keep it inside the same budget as phase 1.
  const uint64_t q = ext_sample_q(external_merge_target(C, budget), S, R);
  uint32_t P = 1;
  std::vector<uint64_t> split, part_off;
  if ((st = ext_partition(ctx, rs, b, q, key_bytes, s, prof, &P, split, part_off))) return st;
  if ((st = prof.end())) return st;

  if ((st = prof.begin("ext merge"))) return st;
  if ((st = ext_merge(ctx, rs, split, part_off, 0, P, out, perm_out, key_bytes, s, prof, tr))) return st;
  tr.report();
  return prof.end();
}

// ------------------------------------------------------------------------------- multi-GPU external
// SURVEY.md §8e "External at 8 GPUs" (BASELINE.json configs[4] at 8 GPUs): every rank generates sorted runs
// of its pinned host slice into a host run scratch that every rank can read (global record layout), the
// samples of all runs are shared, every rank derives the same splitters and slice bounds, and rank r merges
// the partitions that cover global sorted positions [floor(r N / G), floor((r+1) N / G)) — the boundary
// partitions by both neighbours, each keeping its exact share — into its own output. No NVLink traffic:
// the host link (and host DRAM) is the bound.
ExtDistPlan ext_dist_plan(const std::vector<uint64_t>& n_local, uint64_t budget) {
  ExtDistPlan P;
  const int G = (int)n_local.size();
  P.N = 0;
  for (uint64_t v : n_local) P.N += v;
  P.C = std::max<uint64_t>(1, external_run_records(P.N, budget));
  P.S = external_sample_stride(P.N, P.C, budget);
  P.gbase.assign(G, 0);
  P.samp_off.assign(G + 1, 0);
  uint64_t runs = 0;
  for (int r = 0; r < G; ++r) {
    P.gbase[r] = r ? P.gbase[r - 1] + n_local[r - 1] : 0;
    uint64_t ns = 0;
    for (uint64_t at = 0; at < n_local[r]; at += P.C) {
      ns += (std::min<uint64_t>(P.C, n_local[r] - at) + P.S - 1) / P.S;
      ++runs;
    }
    P.samp_off[r + 1] = P.samp_off[r] + ns;
  }
  P.n_local = n_local;
  P.runs = runs;
  P.q = ext_sample_q(external_merge_target(P.C, budget), P.S, std::max<uint64_t>(1, runs));
  return P;
}

size_t ext_dist_device_bytes(const ExtDistPlan& P) { return phase1_bytes(P.C, std::max<uint64_t>(1, P.samp_off.back())); }

namespace {
RunSet ext_dist_runset(const ExtDistPlan& P, uint8_t* h_runs) {
  RunSet rs;
  rs.h_runs = h_runs;
  for (size_t r = 0; r < P.n_local.size(); ++r)
    for (uint64_t at = 0; at < P.n_local[r]; at += P.C) {
      rs.off.push_back(P.gbase[r] + at);
      rs.len.push_back(std::min<uint64_t>(P.C, P.n_local[r] - at));
      rs.S.push_back(P.S);
      rs.samp_base.push_back(rs.nsamp);
      rs.nsamp += (rs.len.back() + P.S - 1) / P.S;
    }
  return rs;
}
}  // namespace

uint8_t* ext_dist_samples(DeviceContext& ctx, const ExtDistPlan& P) {
  return phase1_layout(static_cast<uint8_t*>(ctx.ext.ptr), P.C, std::max<uint64_t>(1, P.samp_off.back())).d_samp;
}

ley_status ext_dist_runs(DeviceContext& ctx, const ExtDistPlan& P, int rank, const uint8_t* in, uint8_t* h_runs,
                         uint32_t key_bytes, cudaStream_t s, Profiler& prof) {
  ley_status st;
  const uint64_t cap = std::max<uint64_t>(1, P.samp_off.back());
  if ((st = ensure_buffer(ctx.ext, phase1_bytes(P.C, cap), "external buffers", s))) return st;
  if ((st = ensure_copy_streams(ctx))) return st;
  const Phase1 b = phase1_layout(static_cast<uint8_t*>(ctx.ext.ptr), P.C, cap);
  RunSet rs;
  rs.h_runs = h_runs;
  rs.nsamp = P.samp_off[rank];  // this rank's samples land at their place in the run-ordered sample set
  ExtTrace tr;
  return ext_generate(ctx, in, P.n_local[rank], P.gbase[rank], P.C, P.S, rs, b, false, key_bytes, s, prof, tr);
}

ley_status ext_dist_partition(DeviceContext& ctx, const ExtDistPlan& P, uint8_t* h_runs, uint32_t key_bytes,
                              cudaStream_t s, Profiler& prof, ExtDistParts& parts) {
  RunSet rs = ext_dist_runset(P, h_runs);
  LEY_CUDA("external scratch", cudaHostGetDevicePointer((void**)&rs.h_runs_dev, h_runs, 0));
  const Phase1 b = phase1_layout(static_cast<uint8_t*>(ctx.ext.ptr), P.C, std::max<uint64_t>(1, P.samp_off.back()));
  return ext_partition(ctx, rs, b, P.q, key_bytes, s, prof, &parts.P, parts.split, parts.part_off);
}

ley_status ext_dist_merge(DeviceContext& ctx, const ExtDistPlan& P, const ExtDistParts& parts, int rank,
                          uint8_t* h_runs, uint8_t* out, uint64_t cap, uint64_t* n_out, uint64_t* out_off,
                          uint32_t key_bytes, cudaStream_t s, Profiler& prof) {
  const int G = (int)P.n_local.size();
  const uint64_t lo = (uint64_t)((unsigned __int128)rank * P.N / (unsigned)G);
  const uint64_t hi = (uint64_t)((unsigned __int128)(rank + 1) * P.N / (unsigned)G);
  *n_out = hi - lo;
  *out_off = lo;
  if (hi - lo > cap) {
    set_error("dist external: rank " + std::to_string(rank) + " must hold " + std::to_string(hi - lo) +
              " records but out_capacity_records is " + std::to_string(cap));
    return LEY_ERR_CAPACITY;
  }
  if (hi == lo) return LEY_OK;
  // partitions overlapping [lo, hi)
  const auto& po = parts.part_off;
  const uint32_t pb = (uint32_t)(std::upper_bound(po.begin(), po.end(), lo) - po.begin() - 1);
  const uint32_t pe = (uint32_t)(std::lower_bound(po.begin(), po.end(), hi) - po.begin());
  RunSet rs = ext_dist_runset(P, h_runs);
  ley_status st = ensure_copy_streams(ctx);
  if (st) return st;
  ExtTrace tr;
  return ext_merge(ctx, rs, parts.split, po, pb, std::min<uint32_t>(pe, parts.P), out, nullptr, key_bytes, s, prof, tr,
                   lo, hi);
}

}  // namespace ley
