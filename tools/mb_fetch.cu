// mb_fetch.cu — does the L2 fetch granularity (cudaLimitMaxL2FetchGranularity, load qualifiers) change
// what DRAM charges for the two access patterns that set the sort's byte floor:
//   keys  : 12 B read per 100-B record (K-a's key extraction)
//   gather: random 100-B records, 16-B-aligned 112-B windows (K-e), sequential 100-B writes
// Not product code. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared
//   -o tools/libmb_fetch.so tools/mb_fetch.cu ; driven by tools/mb_fetch.py (timing, and ncu for bytes).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

template <int MODE>
__device__ __forceinline__ uint32_t ld32(const uint32_t* p) {
  uint32_t v;
  if (MODE == 0) asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (MODE == 1) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (MODE == 3) asm volatile("ld.global.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else asm volatile("ld.global.L2::128B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) mbf_keys(const uint8_t* __restrict__ in, uint32_t* __restrict__ sink, uint64_t n) {
  uint32_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(in + i * 100);
    acc ^= ld32<MODE>(p) + ld32<MODE>(p + 1) * 3 + ld32<MODE>(p + 2) * 7;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int MODE>
__device__ __forceinline__ uint4 ld128(const void* p) {
  uint4 v;
  if (MODE == 0) asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (MODE == 1) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (MODE == 3) asm volatile("ld.global.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else asm volatile("ld.global.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// random gather: lane = one record; 7 x 16-B loads of its aligned 112-B window into registers, realign,
// transpose through shared memory, 4-B coalesced stores (the output side is sequential)
template <int MODE>
__global__ void __launch_bounds__(256) mbf_gather(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm,
                                                  uint8_t* __restrict__ out, uint64_t n) {
  __shared__ uint32_t tb[8][32 * 25];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t ngroups = (n + 31) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  for (uint64_t g = (uint64_t)blockIdx.x * 8 + w; g < ngroups; g += nw) {
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
    uint32_t wd[28];
    uint32_t sh = 0;
    if (lane < (int)cnt) {
      const uint32_t p = perm[j0 + lane];
      const uint8_t* s = in + (((uint64_t)p * 100) & ~15ull);
      sh = p & 3u;
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const uint4 v = ld128<MODE>(s + 16 * q);
        wd[4 * q] = v.x; wd[4 * q + 1] = v.y; wd[4 * q + 2] = v.z; wd[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int o = 0; o < 25; ++o)
        tb[w][lane * 25 + o] = sh == 0 ? wd[o] : sh == 1 ? wd[o + 1] : sh == 2 ? wd[o + 2] : wd[o + 3];
    }
    __syncwarp();
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + j0 * 100);
    for (uint32_t x = lane; x < cnt * 25; x += 32) __stcs(dst + x, tb[w][x]);
    __syncwarp();
  }
}

// exact-sector gather: each lane fetches only the 32-B sectors its record touches (4 x 32 B = the 128-B
// aligned span [100p & ~31, +128) always covers the record: 100p mod 32 <= 28, 28 + 100 = 128)
template <int MODE>
__global__ void __launch_bounds__(256) mbf_gather_sec(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm,
                                                      uint8_t* __restrict__ out, uint64_t n) {
  __shared__ uint32_t tb[8][32 * 25];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t ngroups = (n + 31) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  for (uint64_t g = (uint64_t)blockIdx.x * 8 + w; g < ngroups; g += nw) {
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
    if (lane < (int)cnt) {
      const uint32_t p = perm[j0 + lane];
      const uint64_t b = (uint64_t)p * 100;
      const uint8_t* s = in + (b & ~31ull);
      const uint32_t sh = (uint32_t)(b & 31) >> 2;  // words to skip: 0, 1, ..., 7
      uint32_t wd[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        // window words [4q, 4q+4) needed iff they overlap [sh, sh + 25)
        uint4 v = make_uint4(0, 0, 0, 0);
        if (4 * q + 3 >= (int)sh && 4 * q < (int)sh + 25) v = ld128<MODE>(s + 16 * q);
        wd[4 * q] = v.x; wd[4 * q + 1] = v.y; wd[4 * q + 2] = v.z; wd[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int o = 0; o < 25; ++o) {
        uint32_t x = wd[o];
#pragma unroll
        for (int k = 1; k < 8; ++k) x = sh == (uint32_t)k ? wd[o + k] : x;
        tb[w][lane * 25 + o] = x;
      }
    }
    __syncwarp();
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + j0 * 100);
    for (uint32_t x = lane; x < cnt * 25; x += 32) __stcs(dst + x, tb[w][x]);
    __syncwarp();
  }
}

__global__ void mbf_copy(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t nv) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (uint64_t)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

// 32-B-strided single-word reads: one u32 per 32-B sector of every other 128-B line half (a pure
// granularity probe: reads 4 B out of each 64 B; DRAM bytes / useful sectors tells the fetch atom)
template <int MODE>
__global__ void mbf_probe(const uint8_t* __restrict__ in, uint32_t* __restrict__ sink, uint64_t nbytes, uint32_t stride) {
  uint32_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i * stride < nbytes; i += (uint64_t)gridDim.x * blockDim.x)
    acc += ld32<MODE>(reinterpret_cast<const uint32_t*>(in + i * stride));
  if (acc == 0x12345678u) sink[0] = acc;
}

}  // namespace

extern "C" {
int mbf_set_fetch(int bytes) {
  if (bytes < 0) return 0;
  return (int)cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
}
int mbf_get_fetch() {
  size_t v = 0;
  cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
  return (int)v;
}
// which: 0 keys, 1 gather (7 x 16 B window), 2 gather exact sectors, 3 copy, 4 probe (stride = extra)
int mbf_run(int which, int mode, const void* in, void* out, const uint32_t* perm, uint32_t* sink, uint64_t n, int grid,
            uint32_t extra, cudaStream_t s) {
#define MBF_DISPATCH(K, ...)                                  \
  switch (mode) {                                             \
    case 0: K<0><<<grid, 256, 0, s>>>(__VA_ARGS__); break;    \
    case 1: K<1><<<grid, 256, 0, s>>>(__VA_ARGS__); break;    \
    case 2: K<2><<<grid, 256, 0, s>>>(__VA_ARGS__); break;    \
    case 3: K<3><<<grid, 256, 0, s>>>(__VA_ARGS__); break;    \
    default: K<4><<<grid, 256, 0, s>>>(__VA_ARGS__); break;   \
  }
  switch (which) {
    case 0: MBF_DISPATCH(mbf_keys, (const uint8_t*)in, sink, n); break;
    case 1: MBF_DISPATCH(mbf_gather, (const uint8_t*)in, perm, (uint8_t*)out, n); break;
    case 2: MBF_DISPATCH(mbf_gather_sec, (const uint8_t*)in, perm, (uint8_t*)out, n); break;
    case 3: mbf_copy<<<grid, 256, 0, s>>>((const uint4*)in, (uint4*)out, n * 100 / 16); break;
    default: MBF_DISPATCH(mbf_probe, (const uint8_t*)in, sink, n * 100, extra); break;
  }
#undef MBF_DISPATCH
  return (int)cudaGetLastError();
}
}
