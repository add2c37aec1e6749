// mb_l2.cu — can an L2-resident region make the random record gather cheap? (design probe, not product)
// For a region of W records: (A) read it sequentially with an L2 evict_last policy so its lines stay
// resident, then (B) gather its records in a random order (sequential 100-B-record writes elsewhere).
// Compare B's time and DRAM reads with and without A. Build: nvcc -shared (see tools/mb_build.sh).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
__global__ void l2_load(const uint4* __restrict__ p, uint64_t nv, uint32_t* sink) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  uint32_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i), "l"(pol));
    acc ^= v.x + v.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// one warp per 32 output records: lane = record, 7 x 16-B loads of its window, transpose via smem
__global__ void __launch_bounds__(256) gather(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm,
                                              uint8_t* __restrict__ out, uint64_t n) {
  __shared__ __align__(16) uint32_t tb[8][32 * 25];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t ngroups = n / 32, nw = (uint64_t)gridDim.x * 8;
  for (uint64_t g = (uint64_t)blockIdx.x * 8 + w; g < ngroups; g += nw) {
    const uint32_t p = perm[g * 32 + lane];
    const uint4* s = reinterpret_cast<const uint4*>(in + (((uint64_t)p * 100) & ~15ull));
    uint32_t wd[28];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const uint4 v = s[q];
      wd[4 * q] = v.x; wd[4 * q + 1] = v.y; wd[4 * q + 2] = v.z; wd[4 * q + 3] = v.w;
    }
    const uint32_t sh = p & 3u;
#pragma unroll
    for (int o = 0; o < 25; ++o) tb[w][lane * 25 + o] = sh == 0 ? wd[o] : sh == 1 ? wd[o + 1] : sh == 2 ? wd[o + 2] : wd[o + 3];
    __syncwarp();
    uint4* dst = reinterpret_cast<uint4*>(out + g * 3200);
    const uint4* src = reinterpret_cast<const uint4*>(tb[w]);
    for (int x = lane; x < 200; x += 32) __stcs(dst + x, src[x]);
    __syncwarp();
  }
}
}  // namespace

extern "C" int l2_run(int which, const void* in, void* out, const uint32_t* perm, uint32_t* sink, uint64_t n, int grid,
                      cudaStream_t s) {
  if (which == 0) l2_load<<<grid, 256, 0, s>>>((const uint4*)in, n * 100 / 16, sink);
  else gather<<<grid, 256, 0, s>>>((const uint8_t*)in, perm, (uint8_t*)out, n);
  return (int)cudaGetLastError();
}
