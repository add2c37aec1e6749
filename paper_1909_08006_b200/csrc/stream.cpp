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
// The caller's thread enqueues the H2D and returns; a worker thread (one per device) runs each call's
// sort — which blocks the host on its own stream once per MSD level — and enqueues its D2H, so the next
// call's H2D is already queued while this call sorts. The caller's stream only orders the start;
// completion is observed with ley_sort_drain.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "config.h"
#include "runtime.h"

namespace ley {

namespace {

// LEY_TRACE_PIPE=1: per-call start/end of H2D, sort and D2H (ms from the first event), printed by drain.
// Events are created on the caller's thread (tag = 6 k + {0,1: H2D, 2,3: sort, 4,5: D2H}).
struct PipeTrace {
  bool on = getenv("LEY_TRACE_PIPE") != nullptr;
  std::mutex mu;
  std::vector<cudaEvent_t> ev;  // indexed by tag
  void reserve(uint64_t k) {
    if (!on) return;
    std::lock_guard<std::mutex> g(mu);
    while (ev.size() < 6 * (k + 1)) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
  }
  void mark(uint64_t tag, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    {
      std::lock_guard<std::mutex> g(mu);
      e = ev[tag];
    }
    cudaEventRecord(e, s);
  }
  void dump() {
    if (!on || ev.empty()) return;
    std::lock_guard<std::mutex> g(mu);
    for (size_t t = 0; t < ev.size(); ++t) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[0], ev[t]);
      fprintf(stderr, "[pipe] call %zu %s %s %8.2f\n", t / 6, (t % 6) < 2 ? "H2D " : (t % 6) < 4 ? "sort" : "D2H ",
              (t & 1) ? "end  " : "begin", ms);
    }
    cudaGetLastError();
  }
};
PipeTrace g_trace;

void worker_main(DeviceContext* ctx) {
  auto& P = ctx->pipe;
  cudaSetDevice(ctx->device);
  while (true) {
    DeviceContext::Pipe::Job job;
    {
      std::unique_lock<std::mutex> lk(P.mu);
      P.cv.wait(lk, [&] { return P.stop || !P.q.empty(); });
      if (P.q.empty()) return;  // stop requested and nothing left
      job = P.q.front();
      P.q.pop_front();
      P.busy = true;
    }
    const int s = (int)(job.k & 1);
    ley_status st = LEY_OK;
    std::string msg;
    {
      std::lock_guard<std::mutex> g(ctx->mu);  // the sort uses the device's shared workspace
      auto fail = [&](const char* what, cudaError_t e) {
        st = LEY_ERR_CUDA;
        msg = std::string(what) + ": " + cudaGetErrorString(e);
      };
      cudaError_t e = cudaSuccess;
      if (ctx->async_pending) {  // (a stream-ordered ley_sort may still use the workspace: async_join)
        ctx->async_pending = false;
        if (P.comp != ctx->async_stream) e = cudaStreamWaitEvent(P.comp, ctx->async_ev, 0);
      }
      if (e == cudaSuccess) e = cudaStreamWaitEvent(P.comp, P.copied_in[s], 0);
      if (e == cudaSuccess && job.k >= 2) e = cudaStreamWaitEvent(P.comp, P.copied_out[s], 0);
      if (e != cudaSuccess) fail("submit sort", e);
      g_trace.mark((uint64_t)(6 * job.k + 2), P.comp);
      if (!st) {
        Profiler prof;  // stage timing is not recorded on the streaming path
        st = sort_internal_device(*ctx, job.din, job.dout, nullptr, job.n, P.comp, prof, nullptr, 0, job.key_bytes);
        if (st) msg = last_error();
      }
      g_trace.mark((uint64_t)(6 * job.k + 3), P.comp);
      if (!st && (e = cudaEventRecord(P.sorted[s], P.comp)) != cudaSuccess) fail("submit sort", e);
      if (!st && (e = cudaStreamWaitEvent(P.d2h, P.sorted[s], 0)) != cudaSuccess) fail("submit D2H", e);
      g_trace.mark((uint64_t)(6 * job.k + 4), P.d2h);
      // the output in job.parts pieces, piece q > 0 on its own stream, all joined back into d2h
      const size_t bytes = job.n * kRecordBytes;
      const size_t piece = job.parts > 1 ? (bytes / job.parts) & ~size_t(255) : bytes;
      for (int q = 1; q < job.parts && !st; ++q) {
        const size_t o = q * piece, len = q + 1 < job.parts ? piece : bytes - o;
        if ((e = cudaStreamWaitEvent(P.d2h_x[q - 1], P.sorted[s], 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(job.out + o, job.dout + o, len, cudaMemcpyDeviceToHost, P.d2h_x[q - 1])) != cudaSuccess ||
            (e = cudaEventRecord(P.part_out[q - 1], P.d2h_x[q - 1])) != cudaSuccess)
          fail("submit D2H", e);
      }
      if (!st && (e = cudaMemcpyAsync(job.out, job.dout, piece, cudaMemcpyDeviceToHost, P.d2h)) != cudaSuccess)
        fail("submit D2H", e);
      for (int q = 1; q < job.parts && !st; ++q)
        if ((e = cudaStreamWaitEvent(P.d2h, P.part_out[q - 1], 0)) != cudaSuccess) fail("submit D2H", e);
      g_trace.mark((uint64_t)(6 * job.k + 5), P.d2h);
      if (!st && (e = cudaEventRecord(P.copied_out[s], P.d2h)) != cudaSuccess) fail("submit D2H", e);
    }
    {
      std::lock_guard<std::mutex> lk(P.mu);
      ++P.sort_done;
      P.busy = false;
      if (st && !P.err) {
        P.err = st;
        P.err_msg = msg;
      }
    }
    P.cv.notify_all();
  }
}

ley_status take_error(DeviceContext::Pipe& P) {  // with P.mu held
  if (!P.err) return LEY_OK;
  const ley_status st = P.err;
  set_error(P.err_msg);
  P.err = LEY_OK;
  P.err_msg.clear();
  return st;
}

}  // namespace

void pipe_release(DeviceContext& c) {
  auto& P = c.pipe;
  if (!P.init) return;
  {
    std::lock_guard<std::mutex> lk(P.mu);
    P.stop = true;
  }
  P.cv.notify_all();
  if (P.worker.joinable()) P.worker.join();
  for (cudaStream_t st : {P.h2d, P.comp, P.d2h})
    if (st) cudaStreamSynchronize(st);
  for (int q = 0; q < DeviceContext::Pipe::kParts - 1; ++q)
    for (cudaStream_t st : {P.h2d_x[q], P.d2h_x[q]})
      if (st) cudaStreamSynchronize(st);
  for (int i = 0; i < 2; ++i) {
    if (P.slot[i].ptr) {
      cudaFree(P.slot[i].ptr);
      track_device_bytes(-(int64_t)P.slot[i].cap);
    }
    P.slot[i] = DeviceBuffer{};
    for (cudaEvent_t* e : {&P.copied_in[i], &P.sorted[i], &P.copied_out[i]}) {
      if (*e) cudaEventDestroy(*e);
      *e = nullptr;
    }
  }
  if (P.user) cudaEventDestroy(P.user);
  P.user = nullptr;
  for (cudaStream_t* st : {&P.h2d, &P.comp, &P.d2h}) {
    if (*st) cudaStreamDestroy(*st);
    *st = nullptr;
  }
  for (int q = 0; q < DeviceContext::Pipe::kParts - 1; ++q) {
    for (cudaStream_t* st : {&P.h2d_x[q], &P.d2h_x[q]}) {
      if (*st) cudaStreamDestroy(*st);
      *st = nullptr;
    }
    for (cudaEvent_t* e : {&P.part_in[q], &P.part_out[q]}) {
      if (*e) cudaEventDestroy(*e);
      *e = nullptr;
    }
  }
  P.submitted = P.sort_done = 0;
  P.q.clear();
  P.stop = P.busy = false;
  P.err = LEY_OK;
  P.err_msg.clear();
  P.init = false;
}

ley_status sort_submit(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint64_t n, uint32_t key_bytes,
                       cudaStream_t user) {
  auto& P = ctx.pipe;
  std::unique_lock<std::mutex> lk(P.mu);
  if (ley_status st = take_error(P)) return st;
  if (!P.init) {
    for (cudaStream_t* st : {&P.h2d, &P.comp, &P.d2h})
      LEY_CUDA("submit", cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    for (int q = 0; q < DeviceContext::Pipe::kParts - 1; ++q) {
      LEY_CUDA("submit", cudaStreamCreateWithFlags(&P.h2d_x[q], cudaStreamNonBlocking));
      LEY_CUDA("submit", cudaStreamCreateWithFlags(&P.d2h_x[q], cudaStreamNonBlocking));
      LEY_CUDA("submit", cudaEventCreateWithFlags(&P.part_in[q], cudaEventDisableTiming));
      LEY_CUDA("submit", cudaEventCreateWithFlags(&P.part_out[q], cudaEventDisableTiming));
    }
    LEY_CUDA("submit", cudaEventCreateWithFlags(&P.user, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t* e : {&P.copied_in[i], &P.sorted[i], &P.copied_out[i]})
        LEY_CUDA("submit", cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    P.stop = false;
    P.worker = std::thread(worker_main, &ctx);
    P.init = true;
  }
  const uint64_t k = P.submitted;
  const int s = (int)(k & 1);
  // slot s was last used by call k-2: its sort must be enqueued (sorted[s] then refers to it)
  if (k >= 2) P.cv.wait(lk, [&] { return P.sort_done + 1 >= k || P.err; });
  if (ley_status st = take_error(P)) return st;
  const size_t bytes = (size_t)n * kRecordBytes;
  const size_t a = (bytes + 255) & ~size_t(255);
  if (P.slot[s].cap < 2 * a) {  // growth: call k-2's D2H (the last user of slot s) must be complete
    if (k >= 2) LEY_CUDA("submit", cudaEventSynchronize(P.copied_out[s]));
    LEY_CUDA("submit", cudaStreamSynchronize(P.h2d));
    ley_status st = ensure_buffer(P.slot[s], 2 * a, "stream slot", P.h2d);
    if (st) return st;
  }
  uint8_t* din = static_cast<uint8_t*>(P.slot[s].ptr);
  uint8_t* dout = din + a;
  LEY_CUDA("submit H2D", cudaEventRecord(P.user, user));
  LEY_CUDA("submit H2D", cudaStreamWaitEvent(P.h2d, P.user, 0));
  if (k >= 2) LEY_CUDA("submit H2D", cudaStreamWaitEvent(P.h2d, P.sorted[s], 0));
  g_trace.reserve(k);
  g_trace.mark((uint64_t)(6 * k + 0), P.h2d);
  // the input in `parts` pieces, piece q > 0 on its own stream, all joined back into h2d
  const int parts = (int)options_snapshot().pipe_split;
  const size_t piece = parts > 1 ? (bytes / parts) & ~size_t(255) : bytes;
  for (int q = 1; q < parts; ++q) {
    const size_t o = q * piece, len = q + 1 < parts ? piece : bytes - o;
    LEY_CUDA("submit H2D", cudaStreamWaitEvent(P.h2d_x[q - 1], P.user, 0));
    if (k >= 2) LEY_CUDA("submit H2D", cudaStreamWaitEvent(P.h2d_x[q - 1], P.sorted[s], 0));
    LEY_CUDA("submit H2D", cudaMemcpyAsync(din + o, in + o, len, cudaMemcpyHostToDevice, P.h2d_x[q - 1]));
    LEY_CUDA("submit H2D", cudaEventRecord(P.part_in[q - 1], P.h2d_x[q - 1]));
  }
  LEY_CUDA("submit H2D", cudaMemcpyAsync(din, in, piece, cudaMemcpyHostToDevice, P.h2d));
  for (int q = 1; q < parts; ++q) LEY_CUDA("submit H2D", cudaStreamWaitEvent(P.h2d, P.part_in[q - 1], 0));
  g_trace.mark((uint64_t)(6 * k + 1), P.h2d);
  LEY_CUDA("submit H2D", cudaEventRecord(P.copied_in[s], P.h2d));
  P.q.push_back(DeviceContext::Pipe::Job{k, din, dout, out, n, key_bytes, parts});
  P.submitted = k + 1;
  lk.unlock();
  P.cv.notify_all();
  return LEY_OK;
}

ley_status sort_drain(DeviceContext& ctx) {
  auto& P = ctx.pipe;
  std::unique_lock<std::mutex> lk(P.mu);
  if (!P.init) return LEY_OK;
  P.cv.wait(lk, [&] { return P.q.empty() && !P.busy; });
  for (cudaStream_t st : {P.h2d, P.comp, P.d2h}) LEY_CUDA("drain", cudaStreamSynchronize(st));
  for (int q = 0; q < DeviceContext::Pipe::kParts - 1; ++q) {
    LEY_CUDA("drain", cudaStreamSynchronize(P.h2d_x[q]));
    LEY_CUDA("drain", cudaStreamSynchronize(P.d2h_x[q]));
  }
  LEY_CUDA("drain", cudaGetLastError());
  g_trace.dump();
  return take_error(P);
}

}  // namespace ley
