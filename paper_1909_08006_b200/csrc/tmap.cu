// tmap.cu — TMA tensor maps over the record array (host side).
//
// Why tensor maps for 100-byte records: a plain load, cp.async or bulk copy that misses in L2 makes the
// L2 fetch the whole 128-byte line from DRAM, so reading a 10-byte key costs 100 B/record and gathering a
// random 100-byte record 224 B; a tensor map carries an L2 promotion setting, and with
// CU_TENSOR_MAP_L2_PROMOTION_L2_64B the misses fetch 64 B: 72 B/record for the keys, 162 B for a random
// record (profiles/r02_fetch_granularity.txt; "none" behaves like 128 B on this part). The record array is
// viewed as [groups of 4 records][25 rows][16 B] with a 400-B group pitch (a record pitch of 100 B is not
// a legal tensor stride, 400 is): record 4g + j starts in row floor(100 j / 16) = 0, 6, 12, 18 of group g,
// 16-byte aligned at byte offset 0, 4, 8, 12 of that row.
#include "kernels.cuh"
#include "runtime.h"

#include <cuda.h>

namespace ley {

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encoder() {
  // from the driver through the runtime's entry-point query (no link-time libcuda dependency)
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (EncodeTiledFn) nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
}  // namespace

cudaError_t record_group_map(CUtensorMap* map, const uint8_t* in, uint64_t n, uint32_t box_rows,
                             uint32_t box_groups) {
  EncodeTiledFn enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  const uint64_t groups = n / 4 ? n / 4 : 1;  // (with n < 4 the map is never used: every record is a tail record)
  if (groups > 0xFFFFFFFFull) return cudaErrorInvalidValue;
  const cuuint64_t dims[3] = {16, 25, groups};
  const cuuint64_t strides[2] = {16, 400};
  const cuuint32_t box[3] = {16, box_rows, box_groups}, es[3] = {1, 1, 1};
  const int64_t pr = options_snapshot().tma_l2_promo;  // (an A/B knob; 64 is the measured best)
  const CUtensorMapL2promotion promo = pr == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                       : pr <= 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                       : pr <= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(in), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace ley
