// k_gather.cu — K-e: payload gather, out[j] = in[perm[j]] for the full 100-byte record.
//
// PAPER.md §3.2: "Leyenda is able to scatter data records directly to the page cache ...
// given the sorted (key, pointer) tuples" — here the destination is HBM instead of the page cache.
// §4.3 line 154 excludes this step from its sort times ("Excluding the time of scattering records"),
// a sign that it is the expensive one; SURVEY.md §8a row a6 and Appendix B (~72% of the bytes).
//
// Output-stationary: one thread per 16-byte output chunk, written with one 16-byte streaming store,
// so every warp stores 512 contiguous bytes. The chunk's four 4-byte words come from at most two source
// records (record offsets are multiples of 4 bytes, never of 16 in general), each loaded with a
// read-only, L1-no-allocate 4-byte load; 4 x UNROLL independent loads per thread are in flight.
#include "common.cuh"
#include "kernels.cuh"

namespace ley {
namespace {

constexpr int kGatherThreads = 256;
constexpr int kGatherUnroll = 4;

__global__ void __launch_bounds__(kGatherThreads)
    ke_gather(const uint32_t* __restrict__ in32, const uint32_t* __restrict__ perm, uint64_t n,
              uint4* __restrict__ out16, uint64_t nchunks) {
  const uint64_t stride = (uint64_t)gridDim.x * kGatherThreads * kGatherUnroll;
  for (uint64_t q0 = (uint64_t)blockIdx.x * kGatherThreads * kGatherUnroll + threadIdx.x; q0 < nchunks;
       q0 += stride) {
    uint4 v[kGatherUnroll];
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      uint64_t q = q0 + (uint64_t)u * kGatherThreads;
      if (q < nchunks) {
        uint64_t word = q * 4;                // output word index
        uint64_t j = word / kRecordWords;     // output record
        uint32_t o = (uint32_t)(word - j * kRecordWords);  // word offset inside it (0..24)
        uint64_t s0 = (uint64_t)perm[j] * kRecordWords;
        uint64_t s1 = (o + 3 >= kRecordWords) ? (uint64_t)perm[j + 1] * kRecordWords : 0;
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t ok = o + k;
          const uint32_t* p = (ok < kRecordWords) ? in32 + s0 + ok : in32 + s1 + (ok - kRecordWords);
          w[k] = ldg_nc_u32(p);
        }
        v[u] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      uint64_t q = q0 + (uint64_t)u * kGatherThreads;
      if (q < nchunks) stg_cs_v4(out16 + q, v[u]);
    }
  }
}

// Trailing 1..3 words when 100 n is not a multiple of 16.
__global__ void ke_gather_tail(const uint32_t* __restrict__ in32, const uint32_t* __restrict__ perm, uint64_t n,
                               uint32_t* __restrict__ out32, uint64_t first_word) {
  uint64_t word = first_word + threadIdx.x;
  if (word >= n * kRecordWords) return;
  uint64_t j = word / kRecordWords;
  uint32_t o = (uint32_t)(word - j * kRecordWords);
  out32[word] = in32[(uint64_t)perm[j] * kRecordWords + o];
}

}  // namespace

cudaError_t launch_ke_gather(const uint8_t* in, const uint32_t* perm, uint64_t n, uint8_t* out, int sms,
                             cudaStream_t s, int* launches) {
  if (n == 0) return cudaSuccess;
  const uint64_t words = n * kRecordWords;
  const uint64_t nchunks = words / 4;
  if (nchunks) {
    uint64_t blocks = (nchunks + kGatherThreads * kGatherUnroll - 1) / (kGatherThreads * kGatherUnroll);
    uint64_t cap = (uint64_t)sms * 64;
    if (blocks > cap) blocks = cap;
    ke_gather<<<(unsigned)blocks, kGatherThreads, 0, s>>>(reinterpret_cast<const uint32_t*>(in), perm, n,
                                                          reinterpret_cast<uint4*>(out), nchunks);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
  }
  if (words % 4) {
    ke_gather_tail<<<1, 32, 0, s>>>(reinterpret_cast<const uint32_t*>(in), perm, n, reinterpret_cast<uint32_t*>(out),
                                    nchunks * 4);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
  }
  return cudaSuccess;
}

}  // namespace ley
