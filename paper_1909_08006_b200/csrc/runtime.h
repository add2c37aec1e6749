// runtime.h — host-side runtime of libleyenda: status/error plumbing, options, plan, device arena,
// per-call profiling. Plain C++ (no device code) so the plan logic is testable without a GPU.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "leyenda.h"

namespace ley {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
void clear_error();
const char* last_error();

struct Status {
  ley_status code = LEY_OK;
  bool ok() const { return code == LEY_OK; }
};

// CUDA call wrapper: returns LEY_ERR_CUDA with a stage-tagged message on failure.
#define LEY_CUDA(stage, expr)                                                                          \
  do {                                                                                                 \
    cudaError_t _e = (expr);                                                                           \
    if (_e != cudaSuccess) {                                                                           \
      ::ley::set_error(std::string(stage) + ": " + cudaGetErrorName(_e) + " (" + cudaGetErrorString(_e) + \
                       ") at " #expr);                                                                 \
      return LEY_ERR_CUDA;                                                                             \
    }                                                                                                  \
  } while (0)

// ------------------------------------------------------------------ options
struct Options {
  int64_t warp_tier_max = 32;
  int64_t smem_tier_max = 16384;
  int64_t kd_digit_bits = 14;
  int64_t kd_insert_max = 16;
  int64_t kd_ws = 1;
  int64_t ka_stream = 1;
  int64_t key_hybrid = 1;         // keys > 10 bytes: 10-byte sort + tie-group fix-up (0: LSD windows always)
  int64_t resident_path = 1;        // host pointers: allow path 2 (resident input, streamed output)
  int64_t resident_chunk_records = 0;  // path 2 output window (records; 0 = 2^21)
  int64_t pipe_split = 2;          // ley_sort_submit: each copy in this many pieces on their own streams
  int64_t dist_fused = 1;        // K-p stores into peers' NCCL symmetric windows (0: send buffer + all-to-all)
  int64_t dist_exchange_g1 = 0;  // run splitters/partition/exchange even when G == 1 (test hook)
  int64_t profile = 0;
  int64_t ext_run_records = 0;
  int64_t l2_fetch_bytes = 0;  // 0 = leave the device default; else cudaLimitMaxL2FetchGranularity
  int64_t nccl_timeout_ms = 120000;  // multi-GPU: a collective not complete after this long aborts the comm
  int64_t dist_fault_stall = 0;      // test hook: stall the stream after the k-th collective of a call
  int64_t tma_l2_promo = 64;  // L2 promotion of the record tensor maps (0 = none, 64, 128, 256)
  int64_t ws_gather_tma = 0;  // kd_ws_sort gathers by tensor copies (1) or by plain bulk copies (0)
  int64_t gather_l2_64 = 1;   // K-d CTA-tier gathers with cp.async .L2::64B (1) or without the hint (0)
  int64_t ext_keyptr = 0;  // external path: runs of (key, ordinal) tuples, records gathered from the input
  int64_t async = 0;     // ley_sort on device pointers returns once enqueued (stream-ordered), see leyenda.h
  int64_t kd_claim = 1;  // K-d/K-e tier CTAs claim buckets dynamically (1) or stride their list (0)
  int64_t pdl = 3;      // PDL of the K-d/K-e tier kernels: 0 off, 1 wait-first, 2 overlap, 3 overlap below 1e7 records
  int64_t graphs = 1;   // replay level 1 of the internal sort from a cached CUDA graph (0: launch directly)
  int64_t kc_corun = 0;  // level-1 K-c kernel co-resident with the fused 2048 tier: K-c CTAs per SM (0 off)
  int64_t kc_fuse = 0;  // level-1 split fused into a K-d+K-e tier (0 off, 1 auto, 2..5 force tier 2048..16384):
                        // measured slower (C2 K-c+K-de 7.49 vs 6.40 ms, C4 54.5 vs 38.8 ms)
  int64_t ka_ring = 6;        // K-a key-row form: ring slots (4, 6, 8 or 11 pieces in flight)
};
Options options_snapshot();
ley_status option_set(const char* name, int64_t value);
ley_status option_get(const char* name, int64_t* value);

// ------------------------------------------------------------------ plan (host-only arithmetic)
// small counters of one sort (zeroed per call): [0, 16) tickets, [16, 16 + kNumKdLists) K-d list counts,
// [32] big-bucket count, [64, 320) done chunks per byte-0 bucket (fused split), [320] fused K-d ticket
constexpr uint32_t kSmallWords = 64 + 256 + 16;
static_assert(kSmallWords % 4 == 0, "zeroed in 16-byte words (launch_zero3)");
struct InternalLayout {
  uint64_t n = 0, tiles = 0, m = 0;  // m = 256 * tiles
  uint64_t split_chunks_ub = 0;      // level-1 chunk upper bound
  // byte offsets inside the workspace
  size_t off_At = 0, off_Ai = 0, off_Bt = 0, off_Bi = 0, off_perm = 0;
  size_t off_cnt = 0, off_off = 0, off_lo = 0, off_hist16 = 0, off_B16 = 0, off_cstart = 0;
  size_t off_scan_status = 0, off_cursor = 0, off_small = 0, off_plan_a = 0, off_plan_b = 0, off_order = 0;
  size_t scan_status_words = 0;
  uint32_t hist_copies = 1;  // K-a hist16 copies (contention relief under skew)
  size_t bytes = 0;  // total
};
InternalLayout plan_internal(uint64_t n);
uint64_t internal_aux_bytes(uint64_t n);
ley_status plan_query(uint64_t n, uint64_t budget, ley_plan_info* info);
uint64_t external_run_records(uint64_t n, uint64_t budget);
uint64_t resident_chunk_records(uint64_t n);  // path 2 output window
uint64_t resident_bytes(uint64_t n);          // path 2 device bytes (scratch + input + perm + 2 windows)
uint64_t external_merge_target(uint64_t C, uint64_t budget);
uint64_t external_sample_stride(uint64_t n, uint64_t C, uint64_t budget);

// ------------------------------------------------------------------ device arena
// A growable cached buffer per (device, slot). Growth frees and reallocates (stream synchronised first).
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t cap = 0;
};

struct DeviceContext {
  std::mutex mu;
  int device = -1;
  int sms = 148;
  DeviceBuffer work;      // internal workspace (InternalLayout)
  DeviceBuffer lists;     // K-d work lists (kNumKdLists x cap)
  DeviceBuffer big[2];    // big-bucket lists, ping-pong across recursion levels
  DeviceBuffer rec;       // recursion-level arrays (chunk starts, histograms, look-back status)
  DeviceBuffer stage;     // staged input/output for host pointers
  DeviceBuffer ext;       // external path device buffers
  DeviceBuffer keypass;   // keys > 10 bytes: the other record buffer of the LSD window passes (+ perms)
  void* host_pinned = nullptr;  // small pinned host scratch (counters)
  // a stream-ordered ley_sort (option async) may still run on async_stream when its call returns: the next
  // user of this context's buffers orders itself after async_ev (async_join / async_drain)
  bool async_pending = false;
  cudaStream_t async_stream = nullptr;
  cudaEvent_t async_ev = nullptr;
  void* host_scratch = nullptr;  // external path: pinned (mapped) host run scratch
  size_t host_scratch_cap = 0;
  cudaStream_t copy_stream[2] = {nullptr, nullptr};  // external path: H2D / D2H copy streams
  static constexpr int kExtEvents = 8;
  cudaEvent_t ev[kExtEvents] = {};
  std::vector<cudaEvent_t> events;
  // cached CUDA graphs of the internal sort's level 1 (internal.cu), replayed on their own stream
  struct Graph {
    uint64_t key[13] = {};
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
    uint64_t used = 0;
    // profiler ranges recorded inside the graph (event record nodes): names and event indices
    std::vector<const char*> names;
    std::vector<int> ev_begin, ev_end;
    int events = 0;
  };
  std::vector<Graph> graphs;
  uint64_t graph_clock = 0;
  cudaStream_t graph_stream = nullptr;
  // one large host-link copy split into pieces on their own streams (copy_split)
  static constexpr int kSplitParts = 4;
  cudaStream_t split_stream[kSplitParts] = {};
  cudaEvent_t split_ev[kSplitParts + 1] = {};
  // streaming host sort (ley_sort_submit): two device staging slots (in | out), three streams and a
  // worker thread, so the H2D of call k+1, the sort of call k and the D2H of call k-1 all overlap
  struct Pipe {
    struct Job {
      uint64_t k;
      uint8_t* din;
      uint8_t* dout;
      uint8_t* out;
      uint64_t n;
      uint32_t key_bytes;
      int parts;
    };
    bool init = false;
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    static constexpr int kParts = 4;  // copies split into up to kParts pieces on their own streams
    cudaStream_t h2d_x[kParts - 1] = {}, d2h_x[kParts - 1] = {};
    cudaEvent_t part_in[kParts - 1] = {}, part_out[kParts - 1] = {};
    DeviceBuffer slot[2];
    cudaEvent_t user = nullptr;
    cudaEvent_t copied_in[2] = {nullptr, nullptr}, sorted[2] = {nullptr, nullptr}, copied_out[2] = {nullptr, nullptr};
    uint64_t submitted = 0;   // calls whose H2D is enqueued (call k uses slot k & 1)
    uint64_t sort_done = 0;   // calls whose sort + D2H the worker has enqueued (in order)
    std::mutex mu;
    std::condition_variable cv;
    std::deque<Job> q;
    std::thread worker;
    bool stop = false, busy = false;
    ley_status err = LEY_OK;
    std::string err_msg;
    ~Pipe() {  // process exit: stop the worker (no CUDA calls here)
      if (worker.joinable()) {
        {
          std::lock_guard<std::mutex> lk(mu);
          stop = true;
          q.clear();
        }
        cv.notify_all();
        worker.join();
      }
    }
  } pipe;
};
DeviceContext& device_context(int device);
ley_status ensure_buffer(DeviceBuffer& b, size_t bytes, const char* what, cudaStream_t s);
// Runs fn (a fixed sequence of stream work) as a CUDA graph cached under key: on the first call fn is
// captured on the context's graph stream (falling back to running fn(s) directly if capture fails), then
// the graph is launched on the graph stream ordered after s, and s after it. prof's launch count grows by
// the kernel launches fn made while captured, and the profiler ranges fn opened (their events are record
// nodes of the graph, so stage times stay live) are replayed into prof.
struct GraphKey {
  uint64_t w[12];
};
uint64_t options_fingerprint(const Options& o);
struct Profiler;
ley_status graph_run(DeviceContext& ctx, const GraphKey& key, cudaStream_t s,
                     const std::function<ley_status(cudaStream_t)>& fn, Profiler& prof);
void graphs_release(DeviceContext& ctx);
// library device-memory accounting (ensure_buffer and the few direct allocations report here)
void track_device_bytes(int64_t delta);
void device_bytes(uint64_t* current, uint64_t* peak, bool reset_peak);
void release_device(int device);

// ------------------------------------------------------------------ profiling
struct Profiler {
  bool on = false;
  cudaStream_t stream = nullptr;
  DeviceContext* ctx = nullptr;
  std::vector<const char*> names;
  std::vector<int> ev_begin, ev_end;
  int next_event = 0;
  int launches = 0;
  int nvtx_depth = 0;  // open NVTX ranges (closed by end(); an early error return leaves them to ~Profiler)
  ~Profiler();
  ley_status begin(const char* name);
  ley_status end();
  void finish();  // after stream sync: compute times into the thread-local record
};
void record_launches(int launches);
int stage_times(const char** names, float* ms, int max, int* launches);

// ------------------------------------------------------------------ drivers
// Internal sort of device-resident records (K-a .. K-e). perm_out may be null.
// `work` (optional) is a caller-provided workspace of >= plan_internal(n).bytes; else ctx.work is used.
// key_bytes (1..100): the key is record bytes [0, key_bytes) (> 10: LSD passes over 10-byte windows,
// scratch keypass_bytes from ctx.keypass; perm-only mode (out == nullptr) needs key_bytes <= 10).
// allow_async: with no big buckets after level 1, return without waiting for the tier kernels and set
// ctx.async_pending (the ABI's stream-ordered mode; the caller records ctx.async_ev).
ley_status sort_internal_device(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint32_t* perm_out, uint64_t n,
                                cudaStream_t s, Profiler& prof, void* work = nullptr, size_t work_bytes = 0,
                                uint32_t key_bytes = 10, bool allow_async = false);
// Order work on this context after a stream-ordered sort still in flight: stream s waits for it
// (async_join) or the host does (async_drain). Call with ctx.mu held.
ley_status async_join(DeviceContext& ctx, cudaStream_t s);
ley_status async_drain(DeviceContext& ctx);
uint64_t keypass_bytes(uint64_t n, uint32_t key_bytes, bool perm);
// Streaming staged-internal sort of pinned host records (ley_sort_submit / ley_sort_drain).
// Host path 2 (resident.cu): input staged whole on the device, sorted in perm-only mode, output gathered
// window by window into two device staging buffers and copied to the caller's pinned memory.
ley_status sort_resident_host(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint32_t* perm_out, uint64_t n,
                              uint32_t key_bytes, cudaStream_t s, Profiler& prof);
ley_status ensure_copy_streams(DeviceContext& ctx);  // ctx.copy_stream[2] + ctx.ev (external / resident)
// cudaMemcpyAsync of `bytes` as `parts` pieces on the context's split streams, ordered after s and joined
// back into s (a single D2H copy engine stream reaches ~52 GB/s on this link, four ~55: profiles/r02_*)
ley_status copy_split(DeviceContext& ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                      cudaStream_t s, int parts);
ley_status ensure_host_scratch(DeviceContext& ctx, size_t bytes);  // ctx.host_scratch (external.cu)

// Multi-GPU external sort (external.cu): the plan every rank derives alike from the ranks'
// slice sizes and the budget, the phases, and the partition set they share.
struct ExtDistPlan {
  uint64_t N = 0, C = 0, S = 1, q = 1, runs = 0;
  std::vector<uint64_t> n_local, gbase, samp_off;  // samp_off[r]: rank r's first sample (run order)
};
struct ExtDistParts {
  uint32_t P = 1;
  std::vector<uint64_t> split, part_off;
};
ExtDistPlan ext_dist_plan(const std::vector<uint64_t>& n_local, uint64_t budget);
size_t ext_dist_device_bytes(const ExtDistPlan& P);
// a10 for one rank: its runs into h_runs (global layout, pinned + mapped), its samples into the ctx.ext
// sample area at samp_off[rank]
ley_status ext_dist_runs(DeviceContext& ctx, const ExtDistPlan& P, int rank, const uint8_t* in, uint8_t* h_runs,
                         uint32_t key_bytes, cudaStream_t s, Profiler& prof);
uint8_t* ext_dist_samples(DeviceContext& ctx, const ExtDistPlan& P);  // the sample area (all ranks' samples)
// a11 once all runs are in h_runs and all samples in the sample area (identical on every rank)
ley_status ext_dist_partition(DeviceContext& ctx, const ExtDistPlan& P, uint8_t* h_runs, uint32_t key_bytes,
                              cudaStream_t s, Profiler& prof, ExtDistParts& parts);
// a12 for one rank: global sorted positions [floor(r N/G), floor((r+1) N/G)) into out
ley_status ext_dist_merge(DeviceContext& ctx, const ExtDistPlan& P, const ExtDistParts& parts, int rank,
                          uint8_t* h_runs, uint8_t* out, uint64_t cap, uint64_t* n_out, uint64_t* out_off,
                          uint32_t key_bytes, cudaStream_t s, Profiler& prof);
ley_status sort_submit(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint64_t n, uint32_t key_bytes,
                       cudaStream_t user);
ley_status sort_drain(DeviceContext& ctx);
void pipe_release(DeviceContext& ctx);

}  // namespace ley
