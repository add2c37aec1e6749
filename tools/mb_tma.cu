// mb_tma.cu — TMA tensor copies with an explicit L2 promotion setting (CUtensorMap l2Promotion) as the way
// to fetch only the DRAM sectors a record access needs (follow-up of tools/mb_fetch.cu: plain loads and
// bulk copies promote every L2 miss to the whole 128-B line; ld.global.L2::64B limits it to 64 B).
//   keys  : the 12 key bytes of every record through a 3-D view of the record array (16-B rows, 25 rows
//           per 4-record group, 400-B group pitch): 4 boxes per 256 groups fetch rows {0}, {6}, {12,13},
//           {18,19} — one 32-B sector per record under L2_PROMOTION_NONE.
//   gather: out[j] = in[perm[j]] with one 2-D box of 7 rows x 16 B per record (the record's 16-B-aligned
//           112-B window): 4 sectors = 128 B per record under L2_PROMOTION_NONE.
// Not product code. Build: tools/mb_build.sh-style nvcc -shared; driven by tools/mb_tma.py.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
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
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint32_t mbar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(dst), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(mbar) : "memory");
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t mbar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(dst), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(mbar) : "memory");
}

constexpr int kG = 256;                 // groups (of 4 records) per tile
constexpr int kTileBytes = kG * 16 * 6;  // rows 0, 6 (1 row each), 12-13, 18-19 (2 rows each)
constexpr int kStages = 4;

// one CTA per SM; thread 0 issues 4 boxes per tile into a kStages ring; all threads fold the keys
__global__ void __launch_bounds__(256) mbt_keys(const __grid_constant__ CUtensorMap m1,
                                                const __grid_constant__ CUtensorMap m2, uint32_t ngroups,
                                                uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[kStages];
  const uint32_t ntiles = (ngroups + kG - 1) / kG;
  if (threadIdx.x < kStages) mbar_init(sa(&bar[threadIdx.x]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](uint32_t t, int st) {
    const uint32_t dst = sa(sm + st * kTileBytes);
    const uint32_t mb = sa(&bar[st]);
    mbar_expect(mb, kTileBytes);
    const int g0 = (int)(t * kG);
    tma3(dst, &m1, 0, 0, g0, mb);
    tma3(dst + kG * 16, &m1, 0, 6, g0, mb);
    tma3(dst + kG * 32, &m2, 0, 12, g0, mb);
    tma3(dst + kG * 64, &m2, 0, 18, g0, mb);
  };
  uint32_t acc = 0;
  int st = 0;
  uint32_t ph = 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < kStages; ++k)
      if (blockIdx.x + k * gridDim.x < ntiles) issue(blockIdx.x + k * gridDim.x, k);
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(sa(&bar[st]), ph);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(sm + st * kTileBytes);
    for (uint32_t i = threadIdx.x; i < kTileBytes / 4; i += blockDim.x) acc += w[i] * (i | 1);
    __syncthreads();
    if (threadIdx.x == 0 && t + kStages * gridDim.x < ntiles) issue(t + kStages * gridDim.x, st);
    if (++st == kStages) { st = 0; ph ^= 1; }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// gather: each warp keeps STAGES groups of 32 records in flight; lane = record; one 2-D box per record
template <int STAGES>
__global__ void __launch_bounds__(256) mbt_gather(const __grid_constant__ CUtensorMap gm, const uint32_t* __restrict__ perm,
                                                  uint8_t* __restrict__ out, uint64_t n) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(8) uint64_t bars[8][STAGES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* stage0 = dsm + (size_t)w * STAGES * 32 * 128;
  if (lane < STAGES) mbar_init(sa(&bars[w][lane]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t ngroups = n / 32;  // (full groups only: the bench uses n % 32 == 0)
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  const uint64_t g_first = (uint64_t)blockIdx.x * 8 + w;
  auto issue = [&](uint64_t g, int st) {
    const uint32_t mb = sa(&bars[w][st]);
    if (lane == 0) mbar_expect(mb, 32 * 112);
    __syncwarp();
    const uint32_t p = perm[g * 32 + lane];
    tma2(sa(stage0 + (st * 32 + lane) * 128), &gm, 0, (int)(((uint64_t)p * 100) >> 4), mb);
    return p;
  };
  uint32_t pr[STAGES];
#pragma unroll
  for (int st = 0; st < STAGES; ++st) {
    const uint64_t g = g_first + (uint64_t)st * nw;
    pr[st] = g < ngroups ? issue(g, st) : 0u;
  }
  __shared__ __align__(16) uint32_t tb[8][32 * 25];
  uint32_t phase = 0;
  for (uint64_t g0 = g_first; g0 < ngroups; g0 += (uint64_t)STAGES * nw) {
#pragma unroll
    for (int st = 0; st < STAGES; ++st) {
      const uint64_t g = g0 + (uint64_t)st * nw;
      if (g >= ngroups) break;
      mbar_wait(sa(&bars[w][st]), phase);
      const uint4* win = reinterpret_cast<const uint4*>(stage0 + (st * 32 + lane) * 128);
      uint32_t wd[28];
#pragma unroll
      for (int q = 0; q < 7; ++q) { uint4 v = win[q]; wd[4*q] = v.x; wd[4*q+1] = v.y; wd[4*q+2] = v.z; wd[4*q+3] = v.w; }
      const uint32_t sh = pr[st] & 3u;
#pragma unroll
      for (int o = 0; o < 25; ++o)
        tb[w][lane * 25 + o] = sh == 0 ? wd[o] : sh == 1 ? wd[o + 1] : sh == 2 ? wd[o + 2] : wd[o + 3];
      __syncwarp();
      uint4* dst = reinterpret_cast<uint4*>(out + g * 3200);
      const uint4* src = reinterpret_cast<const uint4*>(tb[w]);
      for (int x = lane; x < 200; x += 32) __stcs(dst + x, src[x]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      const uint64_t gn = g + (uint64_t)STAGES * nw;
      pr[st] = gn < ngroups ? issue(gn, st) : 0u;
    }
    phase ^= 1;
  }
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

CUtensorMapL2promotion promo(int p) {
  return p == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : p == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : p == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

}  // namespace

extern "C" {
// which: 0 keys, 1 gather (2 stages), 2 gather (3 stages), 3 gather (4 stages); p = promotion bytes (0 = none)
int mbt_run(int which, int p, const void* in, void* out, const uint32_t* perm, uint32_t* sink, uint64_t n, int grid,
            cudaStream_t s) {
  EncodeTiled enc = encode();
  if (!enc) return 1000;
  CUresult r;
  if (which == 0) {
    CUtensorMap m1, m2;
    const uint64_t ngroups = n / 4;
    cuuint64_t dims[3] = {16, 25, ngroups};
    cuuint64_t strides[2] = {16, 400};
    cuuint32_t box1[3] = {16, 1, kG}, box2[3] = {16, 2, kG}, es[3] = {1, 1, 1};
    r = enc(&m1, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(in), dims, strides, box1, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo(p), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) return 2000 + (int)r;
    r = enc(&m2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(in), dims, strides, box2, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo(p), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) return 3000 + (int)r;
    const int smem = kStages * kTileBytes;
    cudaFuncSetAttribute(mbt_keys, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mbt_keys<<<grid, 256, smem, s>>>(m1, m2, (uint32_t)ngroups, sink);
  } else {
    CUtensorMap gm;
    cuuint64_t dims[2] = {16, n * 100 / 16};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {16, 7}, es[2] = {1, 1};
    r = enc(&gm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(in), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo(p), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) return 4000 + (int)r;
    if (which == 1) {
      const int smem = 8 * 2 * 32 * 128;
      cudaFuncSetAttribute(mbt_gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      mbt_gather<2><<<grid, 256, smem, s>>>(gm, perm, (uint8_t*)out, n);
    } else if (which == 2) {
      const int smem = 8 * 3 * 32 * 128;
      cudaFuncSetAttribute(mbt_gather<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      mbt_gather<3><<<grid, 256, smem, s>>>(gm, perm, (uint8_t*)out, n);
    } else {
      const int smem = 8 * 4 * 32 * 128;
      cudaFuncSetAttribute(mbt_gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      mbt_gather<4><<<grid, 256, smem, s>>>(gm, perm, (uint8_t*)out, n);
    }
  }
  return (int)cudaGetLastError();
}
}

// ---- gather variants in the structure of tools/mb_mem.cu's mb_gather_bulk (STAGES groups of 32 records
// in flight per warp, 8 warps per CTA, 4-B stores straight from the staging): what fetches a random
// record's window fastest. mode 0: one bulk copy of the 112-B window; 1: one 3-D tensor box (7 rows, map
// promotion as built); 2: 7 x cp.async 16 B with .L2::64B; 3: 7 x cp.async 16 B, no hint.
namespace {
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
template <int STAGES>
__global__ void __launch_bounds__(256) mbt_gv(const __grid_constant__ CUtensorMap gm, const uint8_t* __restrict__ in,
                                              const uint32_t* __restrict__ perm, uint8_t* __restrict__ out, uint64_t n,
                                              int mode) {
  extern __shared__ __align__(128) uint8_t dsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + 8 * STAGES * 32 * 128);
  uint8_t* stage0 = dsm + (size_t)w * STAGES * 32 * 128;
  if (lane < STAGES) mbar_init(sa(&bars[w * STAGES + lane]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t ngroups = n / 32;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  const uint64_t g_first = (uint64_t)blockIdx.x * 8 + w;
  auto issue = [&](uint64_t g, int st) {
    const uint32_t mb = sa(&bars[w * STAGES + st]);
    const uint32_t p = perm[g * 32 + lane];
    const uint32_t dst = sa(stage0 + (st * 32 + lane) * 128);
    const uint8_t* src = mode == 7 ? in + (uint64_t)p * 128 : in + (((uint64_t)p * 100) & ~15ull);  // 7: line-aligned
    if (mode <= 1 || mode >= 4) {
      if (lane == 0) mbar_expect(mb, 32 * 112);  // (mode 7 copies 112 B of a 128-B-aligned slot)
      __syncwarp();
      if (mode == 0 || mode >= 4) bulk_g2s(dst, src, 112, mb);
      else asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                        ::"r"(dst), "l"((uint64_t)&gm), "r"(0), "r"((int)((100u * (p & 3u)) >> 4)), "r"((int)(p >> 2)), "r"(mb) : "memory");
    } else {
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        if (mode == 2) asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(dst + 16 * c), "l"(src + 16 * c) : "memory");
        else asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * c), "l"(src + 16 * c) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(mb) : "memory");
    }
  };
  if ((mode == 2 || mode == 3) && lane < STAGES) {  // cp.async completion: 32 arrivals (one per lane) per phase
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bars[w * STAGES + lane])), "r"(32) : "memory");
  }
  __syncwarp();
  uint32_t pr[STAGES];
#pragma unroll
  for (int st = 0; st < STAGES; ++st) {
    const uint64_t g = g_first + (uint64_t)st * nw;
    if (g < ngroups) { issue(g, st); pr[st] = perm[g * 32 + lane]; }
  }
  uint32_t phase = 0;
  for (uint64_t g0 = g_first; g0 < ngroups; g0 += (uint64_t)STAGES * nw) {
#pragma unroll
    for (int st = 0; st < STAGES; ++st) {
      const uint64_t g = g0 + (uint64_t)st * nw;
      if (g >= ngroups) break;
      mbar_wait(sa(&bars[w * STAGES + st]), phase);
      uint32_t* dst = reinterpret_cast<uint32_t*>(out + g * 3200);
      const uint8_t* sb = stage0 + st * 32 * 128;
      for (uint32_t x = lane; x < 800; x += 32) {
        const uint32_t r = x / 25, o = x - r * 25;
        const uint32_t q = __shfl_sync(0xffffffffu, pr[st], r);
        asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(dst + x), "r"(*reinterpret_cast<const uint32_t*>(sb + r * 128 + ((q * 4u) & 15u) + 4 * o)) : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      const uint64_t gn = g + (uint64_t)STAGES * nw;
      if (gn < ngroups) { issue(gn, st); pr[st] = perm[gn * 32 + lane]; }
      if (mode >= 4) {  // L2 prefetch of the window PF groups beyond the next issue (no shared memory used)
        const uint64_t pf = gn + (uint64_t)(mode == 4 ? 2 : mode == 5 ? 4 : 8) * nw;
        if (pf < ngroups) {
          const uint32_t q = perm[pf * 32 + lane];
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], 112;" ::"l"(in + (((uint64_t)q * 100) & ~15ull)) : "memory");
        }
      }
    }
    phase ^= 1;
  }
}
}  // namespace

extern "C" int mbt_gv_run(int mode, int stages, int prom, const void* in, void* out, const uint32_t* perm, uint64_t n,
                          int grid, cudaStream_t s) {
  EncodeTiled enc = encode();
  CUtensorMap gm;
  cuuint64_t dims[3] = {16, 25, n / 4};
  cuuint64_t strides[2] = {16, 400};
  cuuint32_t box[3] = {16, 7, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&gm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(in), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo(prom), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) return 5000 + (int)r;
  const int smem = 8 * stages * 32 * 128 + 8 * 8 * stages;
#define GV(S) if (stages == S) { cudaFuncSetAttribute(mbt_gv<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
                                 mbt_gv<S><<<grid, 256, smem, s>>>(gm, (const uint8_t*)in, perm, (uint8_t*)out, n, mode); }
  GV(1) GV(2) GV(3) GV(4)
#undef GV
  return (int)cudaGetLastError();
}
