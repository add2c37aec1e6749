// testhooks.cpp — per-kernel verification entry points (kernel unit tests against
// CPU models). They run single kernels of the path on caller-provided device buffers; the tests compare
// each output with a plain CPU model (a naive tally, a sequential prefix sum). Not performance paths.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "leyenda.h"
#include "runtime.h"

using namespace ley;

extern "C" {

ley_status ley_test_scan_excl(const uint32_t* in, uint32_t* out, uint64_t m, void* stream) {
  clear_error();
  if (m == 0) return LEY_OK;
  if (!in || !out) {
    set_error("ley_test_scan_excl: NULL");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t words = scan_status_words(m);
  uint64_t* status = nullptr;
  uint32_t* scratch = nullptr;
  LEY_CUDA("test scan", cudaMallocAsync(&status, 8 * words + 8, s));
  LEY_CUDA("test scan", cudaMallocAsync(&scratch, 16, s));
  LEY_CUDA("test scan", cudaMemsetAsync(status, 0, 8 * words + 8, s));
  LEY_CUDA("test scan", cudaMemsetAsync(scratch, 0, 16, s));
  // out[m] receives the total
  LEY_CUDA("test scan", launch_scan_excl(in, out, m, status, scratch, out + m, s));
  LEY_CUDA("test scan", cudaFreeAsync(status, s));
  LEY_CUDA("test scan", cudaFreeAsync(scratch, s));
  LEY_CUDA("test scan", cudaStreamSynchronize(s));
  return LEY_OK;
}

ley_status ley_test_tile_sort(const void* in, uint64_t n, uint64_t* k1, uint32_t* w, uint32_t* cnt, uint32_t* lo,
                              uint32_t* hist16, int stream_form, void* stream) {
  clear_error();
  if (n == 0) return LEY_OK;
  if (!in || !k1 || !w || !cnt || !lo || !hist16) {
    set_error("ley_test_tile_sort: NULL");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t tiles = (uint32_t)((n + kTileRecords - 1) / kTileRecords);
  LEY_CUDA("test K-a", cudaMemsetAsync(hist16, 0, 4 * 65536, s));
  LEY_CUDA("test K-a", launch_ka_tile_sort(static_cast<const uint8_t*>(in), n, tiles, k1, w, cnt, lo, hist16, 1,
                                           stream_form, KeySpec{}, s));
  LEY_CUDA("test K-a", cudaStreamSynchronize(s));
  return LEY_OK;
}

}  // extern "C"
