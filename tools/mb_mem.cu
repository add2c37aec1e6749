// mb_mem.cu — memory-system microbenchmarks for the record-permutation design (not product code).
// Measures what a 100-byte-record permutation costs on B200 DRAM in its two forms:
//   gather : out[j] = in[perm[j]]   (random 100-B reads, sequential writes)  — today's K-e
//   scatter: out[rank[i]] = in[i]   (sequential reads, random 100-B writes)
// plus the 4-B index scatter rank[perm[j]] = j, a key-only read, and a plain copy.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

constexpr int kWin = 112;

__global__ void __launch_bounds__(256) mb_gather(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm,
                                                 uint8_t* __restrict__ out, uint64_t n) {
  __shared__ __align__(16) uint8_t stage[8][32 * kWin];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t ss = (uint32_t)__cvta_generic_to_shared(stage[w]);
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  for (uint64_t g = (uint64_t)blockIdx.x * 8 + w; g * 32 < n; g += nw) {
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
    const uint32_t p = lane < (int)cnt ? perm[j0 + lane] : 0u;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const int ci = q * 32 + lane, r = ci / 7, c = ci - r * 7;
      const uint32_t pr = __shfl_sync(0xffffffffu, p, r);
      if (r < (int)cnt) cp_async16(ss + r * kWin + c * 16, in + (((uint64_t)pr * 100) & ~15ull) + c * 16);
    }
    cp_async_wait_all();
    __syncwarp();
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + j0 * 100);
    for (uint32_t x = lane; x < cnt * 25; x += 32) {
      const uint32_t r = x / 25, o = x - r * 25;
      const uint32_t pr = __shfl_sync(__activemask(), p, r);
      dst[x] = *reinterpret_cast<const uint32_t*>(stage[w] + r * kWin + ((pr * 4u) & 15u) + 4 * o);
    }
    __syncwarp();
  }
}

// sequential 16-B loads of 32 records per warp into smem, then 4-B stores to out + 100 rank[i]
__global__ void __launch_bounds__(256) mb_scatter(const uint8_t* __restrict__ in, const uint32_t* __restrict__ rank,
                                                  uint8_t* __restrict__ out, uint64_t n) {
  __shared__ __align__(16) uint32_t stage[8][800];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  for (uint64_t g = (uint64_t)blockIdx.x * 8 + w; g * 32 < n; g += nw) {
    const uint64_t i0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - i0);
    const uint4* src = reinterpret_cast<const uint4*>(in + i0 * 100);
    const uint32_t vecs = cnt * 100 / 16;  // cnt multiple of 4 except the tail (n % 4 == 0 in the bench)
    uint4 v[7];
#pragma unroll
    for (int q = 0; q < 7; ++q)
      if (q * 32 + lane < (int)vecs) v[q] = __ldcs(src + q * 32 + lane);
#pragma unroll
    for (int q = 0; q < 7; ++q)
      if (q * 32 + lane < (int)vecs) reinterpret_cast<uint4*>(stage[w])[q * 32 + lane] = v[q];
    const uint32_t rk = lane < (int)cnt ? rank[i0 + lane] : 0u;
    __syncwarp();
    for (uint32_t x = lane; x < cnt * 25; x += 32) {
      const uint32_t r = x / 25, o = x - r * 25;
      const uint32_t d = __shfl_sync(__activemask(), rk, r);
      reinterpret_cast<uint32_t*>(out + (uint64_t)d * 100)[o] = stage[w][x];
    }
    __syncwarp();
  }
}

__global__ void mb_scatter_idx(const uint32_t* __restrict__ perm, uint32_t* __restrict__ rank, uint64_t n) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    rank[perm[j]] = (uint32_t)j;
}

__global__ void mb_keys(const uint8_t* __restrict__ in, uint32_t* __restrict__ sink, uint64_t n) {
  uint32_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(in + i * 100);
    acc ^= __ldg(p) + __ldg(p + 1) * 3 + __ldg(p + 2) * 7;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void mb_copy(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t nv) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (uint64_t)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}


// gather variant: mode bit0 = L1-cached 16-B loads (ld.global.v4) instead of cp.async.cg;
// bit1 = blocked assignment (CTA c handles output groups [c*chunk_groups, (c+1)*chunk_groups) per round)
__global__ void __launch_bounds__(256) mb_gather2(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm,
                                                  uint8_t* __restrict__ out, uint64_t n, int mode, uint32_t chunk_groups) {
  __shared__ __align__(16) uint8_t stage[8][32 * kWin];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t ss = (uint32_t)__cvta_generic_to_shared(stage[w]);
  const uint64_t ngroups = (n + 31) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  for (uint64_t it = (uint64_t)blockIdx.x * 8 + w;; it += nw) {
    uint64_t g;
    if (mode & 2) {
      // blocked: round r = it / nw covers gridDim.x * chunk_groups groups; CTA c its chunk
      const uint64_t r = it / nw, c = blockIdx.x;
      const uint64_t k = (it % nw) - c * 8;  // 0..7 : warp index in CTA
      (void)k;
      const uint64_t base = r * gridDim.x * (uint64_t)chunk_groups + c * chunk_groups;
      // each warp loops over its share of the CTA chunk inside this round
      bool any = false;
      for (uint32_t q = w; q < chunk_groups; q += 8) {
        g = base + q;
        if (g >= ngroups) break;
        any = true;
        const uint64_t j0 = g * 32;
        const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
        const uint32_t p = lane < (int)cnt ? perm[j0 + lane] : 0u;
        if (mode & 1) {
          for (int qq = 0; qq < 7; ++qq) {
            const int ci = qq * 32 + lane, rr = ci / 7, cc = ci - rr * 7;
            const uint32_t pr = __shfl_sync(0xffffffffu, p, rr);
            if (rr < (int)cnt)
              *reinterpret_cast<uint4*>(stage[w] + rr * kWin + cc * 16) =
                  *reinterpret_cast<const uint4*>(in + (((uint64_t)pr * 100) & ~15ull) + cc * 16);
          }
        } else {
          for (int qq = 0; qq < 7; ++qq) {
            const int ci = qq * 32 + lane, rr = ci / 7, cc = ci - rr * 7;
            const uint32_t pr = __shfl_sync(0xffffffffu, p, rr);
            if (rr < (int)cnt) cp_async16(ss + rr * kWin + cc * 16, in + (((uint64_t)pr * 100) & ~15ull) + cc * 16);
          }
          cp_async_wait_all();
        }
        __syncwarp();
        uint32_t* dst = reinterpret_cast<uint32_t*>(out + j0 * 100);
        for (uint32_t x = lane; x < cnt * 25; x += 32) {
          const uint32_t r2 = x / 25, o = x - r2 * 25;
          const uint32_t pr = __shfl_sync(__activemask(), p, r2);
          dst[x] = *reinterpret_cast<const uint32_t*>(stage[w] + r2 * kWin + ((pr * 4u) & 15u) + 4 * o);
        }
        __syncwarp();
      }
      if (!any) return;
      continue;
    }
    g = it;
    if (g >= ngroups) return;
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
    const uint32_t p = lane < (int)cnt ? perm[j0 + lane] : 0u;
    if (mode & 1) {
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const int ci = q * 32 + lane, r = ci / 7, c = ci - r * 7;
        const uint32_t pr = __shfl_sync(0xffffffffu, p, r);
        if (r < (int)cnt)
          *reinterpret_cast<uint4*>(stage[w] + r * kWin + c * 16) =
              *reinterpret_cast<const uint4*>(in + (((uint64_t)pr * 100) & ~15ull) + c * 16);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const int ci = q * 32 + lane, r = ci / 7, c = ci - r * 7;
        const uint32_t pr = __shfl_sync(0xffffffffu, p, r);
        if (r < (int)cnt) cp_async16(ss + r * kWin + c * 16, in + (((uint64_t)pr * 100) & ~15ull) + c * 16);
      }
      cp_async_wait_all();
    }
    __syncwarp();
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + j0 * 100);
    for (uint32_t x = lane; x < cnt * 25; x += 32) {
      const uint32_t r = x / 25, o = x - r * 25;
      const uint32_t pr = __shfl_sync(__activemask(), p, r);
      dst[x] = *reinterpret_cast<const uint32_t*>(stage[w] + r * kWin + ((pr * 4u) & 15u) + 4 * o);
    }
    __syncwarp();
  }
}

}  // namespace

extern "C" {
int mb_run(int which, const void* in, void* out, const uint32_t* idx, uint32_t* idx_out, uint64_t n, int grid,
           cudaStream_t s) {
  switch (which) {
    case 0: mb_gather<<<grid, 256, 0, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); break;
    case 1: mb_scatter<<<grid, 256, 0, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); break;
    case 2: mb_scatter_idx<<<grid, 256, 0, s>>>(idx, idx_out, n); break;
    case 3: mb_keys<<<grid, 256, 0, s>>>((const uint8_t*)in, idx_out, n); break;
    case 4: mb_copy<<<grid, 256, 0, s>>>((const uint4*)in, (uint4*)out, n * 100 / 16); break;
    default: mb_gather2<<<grid, 256, 0, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n, (which - 10) & 3, (uint32_t)((which - 10) >> 2)); break;
  }
  return (int)cudaGetLastError();
}
}
