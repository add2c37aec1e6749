// resident.cu — host path 2, "resident input, streamed output": the paper's partial in-memory regime
// (§4.1 P:126 — the 20 GB data set against Table 2's 30 GB of memory, P:130 — and §3.2 P:102-106,
// sort the (key, pointer) tuples, then "scatter data records ... given the sorted tuples").
//
// For pinned host in/out whose input fits the device budget but whose input AND output do not:
//   1. H2D of the whole input into a device staging buffer;
//   2. the internal sort (K-a .. K-d) in perm-only mode: K-d writes the sorted ordinals instead of
//      gathering records (no device output buffer);
//   3. K-e by windows of C records (ke_gather, k_gather.cu) into two device staging windows, each copied
//      to the caller's pinned output on a copy stream while the next window is gathered.
// Device bytes: internal scratch + 100 n (input) + 4 n (perm) + 2 x 100 C, i.e. about half of the staged
// internal path (resident_bytes in runtime.cpp). Both directions of the host link carry exactly 100 B per
// record, as on the staged path, and ~half the external path's 4 crossings.
#include <cuda_runtime.h>

#include "config.h"
#include "kernels.cuh"
#include "runtime.h"

namespace ley {
namespace {
inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

ley_status sort_resident_host(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint32_t* perm_out, uint64_t n,
                              uint32_t key_bytes, cudaStream_t s, Profiler& prof) {
  const uint64_t C = resident_chunk_records(n);
  const size_t a_in = a256((size_t)n * kRecordBytes), a_perm = a256(4 * (size_t)n), a_win = a256(C * kRecordBytes);
  ley_status st = ensure_buffer(ctx.stage, a_in + a_perm + 2 * a_win, "resident staging", s);
  if (st) return st;
  if ((st = ensure_copy_streams(ctx))) return st;
  uint8_t* din = static_cast<uint8_t*>(ctx.stage.ptr);
  uint32_t* dperm = reinterpret_cast<uint32_t*>(din + a_in);
  uint8_t* win[2] = {din + a_in + a_perm, din + a_in + a_perm + a_win};
  cudaStream_t d2h = ctx.copy_stream[1];
  cudaEvent_t gathered[2] = {ctx.ev[1], ctx.ev[2]}, copied[2] = {ctx.ev[3], ctx.ev[4]}, done = ctx.ev[5];

  if ((st = prof.begin("H2D"))) return st;
  LEY_CUDA("resident H2D", cudaMemcpyAsync(din, in, (size_t)n * kRecordBytes, cudaMemcpyHostToDevice, s));
  if ((st = prof.end())) return st;
  if ((st = sort_internal_device(ctx, din, nullptr, dperm, n, s, prof, nullptr, 0, key_bytes))) return st;
  if (perm_out) LEY_CUDA("resident perm", cudaMemcpyAsync(perm_out, dperm, 4 * n, cudaMemcpyDeviceToHost, s));

  if ((st = prof.begin("K-e gather+D2H"))) return st;
  uint64_t k = 0;
  for (uint64_t j0 = 0; j0 < n; j0 += C, ++k) {
    const int b = (int)(k & 1);
    const uint64_t m = n - j0 < C ? n - j0 : C;
    if (k >= 2) LEY_CUDA("resident gather", cudaStreamWaitEvent(s, copied[b], 0));  // window b copied out
    LEY_CUDA("resident gather", launch_ke_gather(din, dperm + j0, m, win[b], ctx.sms, s));
    ++prof.launches;
    LEY_CUDA("resident gather", cudaEventRecord(gathered[b], s));
    LEY_CUDA("resident D2H", cudaStreamWaitEvent(d2h, gathered[b], 0));
    LEY_CUDA("resident D2H", cudaMemcpyAsync(out + j0 * kRecordBytes, win[b], m * kRecordBytes,
                                             cudaMemcpyDeviceToHost, d2h));
    LEY_CUDA("resident D2H", cudaEventRecord(copied[b], d2h));
  }
  LEY_CUDA("resident D2H", cudaEventRecord(done, d2h));
  LEY_CUDA("resident D2H", cudaStreamWaitEvent(s, done, 0));  // the caller's stream completes with the copies
  return prof.end();
}

}  // namespace ley
