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


// ---- gather via TMA bulk copies (one cp.async.bulk of the 112-B window per record), STAGES groups in
// flight per warp, mbarrier completion
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}"
               ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(256) mb_gather_bulk(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm,
                                                      uint8_t* __restrict__ out, uint64_t n) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(8) uint64_t bars[8][STAGES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* stage0 = dsm + (size_t)w * STAGES * 32 * kWin;
  if (lane < STAGES) mbar_init((uint32_t)__cvta_generic_to_shared(&bars[w][lane]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t ngroups = (n + 31) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  const uint64_t g_first = (uint64_t)blockIdx.x * 8 + w;
  auto issue = [&](uint64_t g, int st) {
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bars[w][st]);
    if (lane == 0) mbar_expect(mb, cnt * kWin);
    __syncwarp();
    if (lane < (int)cnt) {
      const uint32_t p = perm[j0 + lane];
      bulk_g2s((uint32_t)__cvta_generic_to_shared(stage0 + (st * 32 + lane) * kWin),
               in + (((uint64_t)p * 100) & ~15ull), kWin, mb);
    }
  };
  // prologue
  for (int st = 0; st < STAGES; ++st) {
    const uint64_t g = g_first + (uint64_t)st * nw;
    if (g < ngroups) issue(g, st);
  }
  uint32_t phase = 0;
  int st = 0;
  for (uint64_t g = g_first; g < ngroups; g += nw) {
    mbar_wait((uint32_t)__cvta_generic_to_shared(&bars[w][st]), phase);
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
    const uint32_t p = lane < (int)cnt ? perm[j0 + lane] : 0u;  // (re-read; L1/L2 hit)
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + j0 * 100);
    const uint8_t* sb = stage0 + st * 32 * kWin;
    for (uint32_t x = lane; x < cnt * 25; x += 32) {
      const uint32_t r = x / 25, o = x - r * 25;
      const uint32_t pr = __shfl_sync(__activemask(), p, r);
      dst[x] = *reinterpret_cast<const uint32_t*>(sb + r * kWin + ((pr * 4u) & 15u) + 4 * o);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const uint64_t gn = g + (uint64_t)STAGES * nw;
    if (gn < ngroups) issue(gn, st);
    if (++st == STAGES) { st = 0; phase ^= 1; }
  }
}

// ---- gather into registers (7 x 16-B loads per lane = its record's window), transpose through smem
__global__ void __launch_bounds__(256) mb_gather_reg(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm,
                                                     uint8_t* __restrict__ out, uint64_t n) {
  __shared__ uint32_t tb[8][32 * 25];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t ngroups = (n + 31) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  for (uint64_t g = (uint64_t)blockIdx.x * 8 + w; g < ngroups; g += nw) {
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
    uint4 v[7];
    uint32_t sh = 0;
    if (lane < (int)cnt) {
      const uint32_t p = perm[j0 + lane];
      const uint4* s = reinterpret_cast<const uint4*>(in + (((uint64_t)p * 100) & ~15ull));
      sh = (p & 3u);  // word shift = (100 p mod 16) / 4 = p mod 4
#pragma unroll
      for (int q = 0; q < 7; ++q) v[q] = __ldcs(s + q);
    }
    uint32_t wd[28];
#pragma unroll
    for (int q = 0; q < 7; ++q) { wd[4*q] = v[q].x; wd[4*q+1] = v[q].y; wd[4*q+2] = v[q].z; wd[4*q+3] = v[q].w; }
    if (lane < (int)cnt) {
#pragma unroll
      for (int o = 0; o < 25; ++o) {
        const uint32_t a0 = wd[o], a1 = wd[o + 1], a2 = wd[o + 2], a3 = wd[o + 3];
        tb[w][lane * 25 + o] = sh == 0 ? a0 : sh == 1 ? a1 : sh == 2 ? a2 : a3;
      }
    }
    __syncwarp();
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + j0 * 100);
    for (uint32_t x = lane; x < cnt * 25; x += 32) __stcs(dst + x, tb[w][x]);
    __syncwarp();
  }
}


// ---- bulk gather + in-register realign + packed smem tile + one bulk store per group (D)
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes) : "memory");
}
template <int STAGES>
__global__ void __launch_bounds__(256) mb_gather_tma(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm,
                                                     uint8_t* __restrict__ out, uint64_t n) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(8) uint64_t bars[8][STAGES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* stage0 = dsm + (size_t)w * (STAGES * 32 * kWin + 2 * 3200);
  uint8_t* pack0 = stage0 + STAGES * 32 * kWin;
  if (lane < STAGES) mbar_init((uint32_t)__cvta_generic_to_shared(&bars[w][lane]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t ngroups = (n + 31) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  const uint64_t g_first = (uint64_t)blockIdx.x * 8 + w;
  uint32_t pr[STAGES];
  auto issue = [&](uint64_t g, int st) {
    const uint64_t j0 = g * 32;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bars[w][st]);
    if (lane == 0) mbar_expect(mb, cnt * kWin);
    __syncwarp();
    uint32_t p = 0;
    if (lane < (int)cnt) {
      p = perm[j0 + lane];
      bulk_g2s((uint32_t)__cvta_generic_to_shared(stage0 + (st * 32 + lane) * kWin),
               in + (((uint64_t)p * 100) & ~15ull), kWin, mb);
    }
    return p;
  };
#pragma unroll
  for (int st = 0; st < STAGES; ++st) {
    const uint64_t g = g_first + (uint64_t)st * nw;
    pr[st] = g < ngroups ? issue(g, st) : 0u;
  }
  uint32_t phase = 0, pk = 0;
  for (uint64_t g0 = g_first; g0 < ngroups; g0 += (uint64_t)STAGES * nw) {
#pragma unroll
    for (int st = 0; st < STAGES; ++st) {
      const uint64_t g = g0 + (uint64_t)st * nw;
      if (g >= ngroups) break;
      mbar_wait((uint32_t)__cvta_generic_to_shared(&bars[w][st]), phase);
      const uint64_t j0 = g * 32;
      const uint32_t cnt = (uint32_t)min((uint64_t)32, n - j0);
      // packed tile pk must be free: its previous bulk store has finished reading
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      uint32_t* pack = reinterpret_cast<uint32_t*>(pack0 + pk * 3200);
      if (lane < (int)cnt) {
        const uint4* win = reinterpret_cast<const uint4*>(stage0 + (st * 32 + lane) * kWin);
        uint32_t wd[28];
#pragma unroll
        for (int q = 0; q < 7; ++q) { uint4 v = win[q]; wd[4*q] = v.x; wd[4*q+1] = v.y; wd[4*q+2] = v.z; wd[4*q+3] = v.w; }
        const uint32_t sh = pr[st] & 3u;
#pragma unroll
        for (int o = 0; o < 25; ++o)
          pack[lane * 25 + o] = sh == 0 ? wd[o] : sh == 1 ? wd[o + 1] : sh == 2 ? wd[o + 2] : wd[o + 3];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        bulk_s2g(out + j0 * 100, (uint32_t)__cvta_generic_to_shared(pack), cnt * 100);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      pk ^= 1;
      const uint64_t gn = g + (uint64_t)STAGES * nw;
      pr[st] = gn < ngroups ? issue(gn, st) : 0u;
    }
    phase ^= 1;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
    case 5: mb_gather_reg<<<grid, 256, 0, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); break;
    case 6: case 7: case 8: {
      const int st = which == 6 ? 2 : which == 7 ? 4 : 3;
      const size_t sm = (size_t)8 * st * 32 * kWin;
      if (st == 2) { cudaFuncSetAttribute(mb_gather_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); mb_gather_bulk<2><<<grid, 256, sm, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); }
      if (st == 3) { cudaFuncSetAttribute(mb_gather_bulk<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); mb_gather_bulk<3><<<grid, 256, sm, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); }
      if (st == 4) { cudaFuncSetAttribute(mb_gather_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); mb_gather_bulk<4><<<grid, 256, sm, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); }
      break;
    }
    case 20: case 21: case 22: {
      const int st = which - 19;
      const size_t sm = (size_t)8 * (st * 32 * kWin + 2 * 3200);
      if (st == 1) { cudaFuncSetAttribute(mb_gather_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); mb_gather_tma<1><<<grid, 256, sm, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); }
      if (st == 2) { cudaFuncSetAttribute(mb_gather_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); mb_gather_tma<2><<<grid, 256, sm, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); }
      if (st == 3) { cudaFuncSetAttribute(mb_gather_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); mb_gather_tma<3><<<grid, 256, sm, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n); }
      break;
    }
    default: mb_gather2<<<grid, 256, 0, s>>>((const uint8_t*)in, idx, (uint8_t*)out, n, (which - 10) & 3, (uint32_t)((which - 10) >> 2)); break;
  }
  return (int)cudaGetLastError();
}
}
