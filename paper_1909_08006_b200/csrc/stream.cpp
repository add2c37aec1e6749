// stream.cpp — streaming host sort (ley_sort_submit / ley_sort_drain): the staged-internal path of
// ley_sort (H2D -> K-a..K-e -> D2H) as a three-stage pipeline across calls.
//
// A sort of host-resident records is bound by the host link twice (P:116-118 describe the same
// reader / sorter / writer overlap for the paper's disk path: "reads and sorts records in small trunks
// and writes them down to disk at the same time"). One call cannot overlap its own H2D with its own
// D2H (every output record depends on every input record), but consecutive calls can: call k+1's input
// crosses the link on one copy engine while call k's output returns on the other, and the device sorts
// in between. Two device slots (input | output) alternate; events order every reuse:
//   h2d  : wait(user work) wait(sorted[s]: slot input free)  H2D in -> slot s      record copied_in[s]
//   comp : wait(copied_in[s]) wait(copied_out[s]: slot output free)  sort          record sorted[s]
//   d2h  : wait(sorted[s])  D2H slot s -> out                                     record copied_out[s]
// The caller's stream only orders the start (the H2D waits for work already on it); completion is
// observed with ley_sort_drain — making the caller's stream wait for the D2H would chain call k+1's H2D
// behind call k's D2H and undo the overlap.
// The internal sort blocks the host only on its own compute stream (one 4-byte read per MSD level),
// while the copy engines keep running.
#include <cuda_runtime.h>

#include "config.h"
#include "runtime.h"

namespace ley {

void pipe_release(DeviceContext& c) {
  auto& P = c.pipe;
  if (!P.init) return;
  for (cudaStream_t st : {P.h2d, P.comp, P.d2h})
    if (st) cudaStreamSynchronize(st);
  for (int i = 0; i < 2; ++i) {
    if (P.slot[i].ptr) cudaFree(P.slot[i].ptr);
    P.slot[i] = DeviceBuffer{};
    for (cudaEvent_t* e : {&P.copied_in[i], &P.sorted[i], &P.copied_out[i]}) {
      if (*e) cudaEventDestroy(*e);
      *e = nullptr;
    }
    P.used[i] = false;
  }
  if (P.user) cudaEventDestroy(P.user);
  for (cudaStream_t* st : {&P.h2d, &P.comp, &P.d2h}) {
    if (*st) cudaStreamDestroy(*st);
    *st = nullptr;
  }
  P.user = nullptr;
  P.next = 0;
  P.init = false;
}

ley_status sort_submit(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint64_t n, cudaStream_t user) {
  auto& P = ctx.pipe;
  if (!P.init) {
    for (cudaStream_t* st : {&P.h2d, &P.comp, &P.d2h})
      LEY_CUDA("submit", cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    LEY_CUDA("submit", cudaEventCreateWithFlags(&P.user, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t* e : {&P.copied_in[i], &P.sorted[i], &P.copied_out[i]})
        LEY_CUDA("submit", cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    P.init = true;
  }
  const size_t bytes = (size_t)n * kRecordBytes;
  const size_t a = (bytes + 255) & ~size_t(255);
  const int s = P.next;
  P.next ^= 1;
  if (P.slot[s].cap < 2 * a) {  // growth: nothing may still use the old slot
    for (cudaStream_t st : {P.h2d, P.comp, P.d2h}) LEY_CUDA("submit", cudaStreamSynchronize(st));
    ley_status st = ensure_buffer(P.slot[s], 2 * a, "stream slot", P.comp);
    if (st) return st;
  }
  uint8_t* din = static_cast<uint8_t*>(P.slot[s].ptr);
  uint8_t* dout = din + a;
  LEY_CUDA("submit H2D", cudaEventRecord(P.user, user));
  LEY_CUDA("submit H2D", cudaStreamWaitEvent(P.h2d, P.user, 0));
  if (P.used[s]) LEY_CUDA("submit H2D", cudaStreamWaitEvent(P.h2d, P.sorted[s], 0));
  LEY_CUDA("submit H2D", cudaMemcpyAsync(din, in, bytes, cudaMemcpyHostToDevice, P.h2d));
  LEY_CUDA("submit H2D", cudaEventRecord(P.copied_in[s], P.h2d));
  LEY_CUDA("submit sort", cudaStreamWaitEvent(P.comp, P.copied_in[s], 0));
  if (P.used[s]) LEY_CUDA("submit sort", cudaStreamWaitEvent(P.comp, P.copied_out[s], 0));
  Profiler prof;  // stage timing is not recorded on the streaming path
  ley_status st = sort_internal_device(ctx, din, dout, nullptr, n, P.comp, prof);
  if (st) return st;
  LEY_CUDA("submit sort", cudaEventRecord(P.sorted[s], P.comp));
  LEY_CUDA("submit D2H", cudaStreamWaitEvent(P.d2h, P.sorted[s], 0));
  LEY_CUDA("submit D2H", cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, P.d2h));
  LEY_CUDA("submit D2H", cudaEventRecord(P.copied_out[s], P.d2h));
  P.used[s] = true;
  return LEY_OK;
}

ley_status sort_drain(DeviceContext& ctx) {
  auto& P = ctx.pipe;
  if (!P.init) return LEY_OK;
  for (cudaStream_t st : {P.h2d, P.comp, P.d2h}) LEY_CUDA("drain", cudaStreamSynchronize(st));
  LEY_CUDA("drain", cudaGetLastError());
  return LEY_OK;
}

}  // namespace ley
