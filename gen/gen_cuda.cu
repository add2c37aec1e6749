/* gen_cuda.cu — CUDA twin of the seeded record generator (gen_core.h), so the bench and the GPU tests
 * can create multi-GB inputs directly in HBM. Input generation only; it is not part of libleyenda and
 * holds none of the sort's arithmetic. Byte-identical to gen.cpp by construction (same header) and by
 * test (tests/test_gpu_parity.py::test_generator_twin). */
#include <cuda_runtime.h>
#include <stdint.h>

#include "gen_core.h"

extern "C" void gen_build_zipf(uint64_t zt[256]);

namespace {

__global__ void gen_records_kernel(uint32_t* __restrict__ out, uint64_t i0, uint64_t count, uint64_t seed,
                                   int dist, const uint64_t* __restrict__ zt_g) {
  __shared__ uint64_t zt[256];
  for (int v = threadIdx.x; v < 256; v += blockDim.x) zt[v] = zt_g[v];
  __syncthreads();
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride) {
    union {
      uint8_t b[100];
      uint32_t w[25];
    } rec;
    gen_record(rec.b, seed, i0 + k, dist, zt);
    uint32_t* dst = out + 25 * k;
#pragma unroll
    for (int q = 0; q < 25; ++q) dst[q] = rec.w[q];
  }
}

}  // namespace

extern "C" int gen_records_cuda(void* dev_out, uint64_t i0, uint64_t count, uint64_t seed, int dist,
                                void* stream) {
  if (count == 0) return 0;
  if (((uintptr_t)dev_out & 3) != 0) return 1;
  uint64_t zt[256];
  gen_build_zipf(zt);
  uint64_t* zt_d = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMallocAsync((void**)&zt_d, sizeof(zt), s) != cudaSuccess) return 2;
  cudaMemcpyAsync(zt_d, zt, sizeof(zt), cudaMemcpyHostToDevice, s);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (count + 255) / 256;
  uint64_t cap = (uint64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  gen_records_kernel<<<(unsigned)blocks, 256, 0, s>>>((uint32_t*)dev_out, i0, count, seed, dist, zt_d);
  cudaFreeAsync(zt_d, s);
  cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? 0 : 3;
}
