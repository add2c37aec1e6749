// runtime.cpp — errors, options, planning, device arena and profiling for libleyenda (host C++).
#include "runtime.h"

#include <nvtx3/nvToolsExt.h>

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <memory>

#include "config.h"

namespace ley {

// ------------------------------------------------------------------ errors
static thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }
void clear_error() { g_error.clear(); }
const char* last_error() { return g_error.c_str(); }

// ------------------------------------------------------------------ options
namespace {
std::mutex g_opt_mu;
Options g_opt;

struct OptDesc {
  const char* name;
  int64_t Options::*field;
  int64_t lo, hi;
};
const OptDesc kOpts[] = {
    {"warp_tier_max", &Options::warp_tier_max, 1, 32},
    {"smem_tier_max", &Options::smem_tier_max, 0, 16384},
    {"kd_digit_bits", &Options::kd_digit_bits, 0, 14},
    {"kd_insert_max", &Options::kd_insert_max, 1, 64},
    {"kd_ws", &Options::kd_ws, 0, 1},
    {"ka_stream", &Options::ka_stream, 0, 2},
    {"key_hybrid", &Options::key_hybrid, 0, 1},
    {"resident_path", &Options::resident_path, 0, 1},
    {"resident_chunk_records", &Options::resident_chunk_records, 0, (int64_t)0xFFFFFFFEll},
    {"pipe_split", &Options::pipe_split, 1, DeviceContext::Pipe::kParts},
    {"dist_fused", &Options::dist_fused, 0, 1},
    {"dist_exchange_g1", &Options::dist_exchange_g1, 0, 1},
    {"profile", &Options::profile, 0, 1},
    {"ext_run_records", &Options::ext_run_records, 0, (int64_t)0xFFFFFFFEll},
    {"l2_fetch_bytes", &Options::l2_fetch_bytes, 0, 128},
    {"nccl_timeout_ms", &Options::nccl_timeout_ms, 50, 3600000},
    {"dist_fault_stall", &Options::dist_fault_stall, 0, 1000},
    {"tma_l2_promo", &Options::tma_l2_promo, 0, 256},
    {"ws_gather_tma", &Options::ws_gather_tma, 0, 1},
    {"ka_ring", &Options::ka_ring, 1, 11},
    {"gather_l2_64", &Options::gather_l2_64, 0, 1},
    {"kc_fuse", &Options::kc_fuse, 0, 5},
    {"kc_corun", &Options::kc_corun, 0, 3},
    {"graphs", &Options::graphs, 0, 1},
    {"pdl", &Options::pdl, 0, 3},
    {"kd_claim", &Options::kd_claim, 0, 1},
    {"async", &Options::async, 0, 1},
    {"ext_keyptr", &Options::ext_keyptr, 0, 1},
};
}  // namespace

Options options_snapshot() {
  std::lock_guard<std::mutex> g(g_opt_mu);
  return g_opt;
}

ley_status option_set(const char* name, int64_t value) {
  if (!name) {
    set_error("ley_set_option: NULL name");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  for (const OptDesc& d : kOpts) {
    if (strcmp(d.name, name) == 0) {
      if (value < d.lo || value > d.hi) {
        set_error(std::string("ley_set_option: ") + name + " out of range [" + std::to_string(d.lo) + ", " +
                  std::to_string(d.hi) + "]");
        return LEY_ERR_INVALID_ARGUMENT;
      }
      std::lock_guard<std::mutex> g(g_opt_mu);
      g_opt.*(d.field) = value;
      return LEY_OK;
    }
  }
  set_error(std::string("ley_set_option: unknown option '") + name + "'");
  return LEY_ERR_INVALID_ARGUMENT;
}

ley_status option_get(const char* name, int64_t* value) {
  if (!name || !value) {
    set_error("ley_get_option: NULL argument");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  for (const OptDesc& d : kOpts) {
    if (strcmp(d.name, name) == 0) {
      std::lock_guard<std::mutex> g(g_opt_mu);
      *value = g_opt.*(d.field);
      return LEY_OK;
    }
  }
  set_error(std::string("ley_get_option: unknown option '") + name + "'");
  return LEY_ERR_INVALID_ARGUMENT;
}

// ------------------------------------------------------------------ plan
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

InternalLayout plan_internal(uint64_t n) {
  InternalLayout L;
  L.n = n;
  L.tiles = (n + kTileRecords - 1) / kTileRecords;
  L.m = (uint64_t)kRadix * L.tiles;
  L.split_chunks_ub = n / kChunk + kRadix + 1;
  L.scan_status_words = (std::max<uint64_t>(L.m, 65536) + kScanTile - 1) / kScanTile;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += align256(bytes);
    return at;
  };
  L.off_At = take(8 * n);
  L.off_Ai = take(4 * n);
  L.off_Bt = take(8 * n);
  L.off_Bi = take(4 * n);
  L.off_perm = take(4 * n);
  L.off_cnt = take(4 * L.m);
  L.off_off = take(4 * (L.m + 1));
  L.off_lo = take(4 * L.m);
  L.hist_copies = (uint32_t)std::min<uint64_t>(kHistCopies, std::max<uint64_t>(1, L.tiles / 64));
  L.off_hist16 = take(4ull * 65536 * L.hist_copies);
  L.off_B16 = take(4 * (65536 + 1));
  L.off_cstart = take(4 * 260);
  L.off_scan_status = take(8 * 2 * L.scan_status_words);
  L.off_cursor = take(4 * 65536);
  L.off_small = take(4 * kSmallWords);  // tickets, list counters, the fused split's done[256] + K-d ticket
  L.off_plan_a = take(16 * L.split_chunks_ub);
  L.off_plan_b = take(8 * L.split_chunks_ub);
  L.off_order = take(4 * L.split_chunks_ub);  // K-c chunk processing order
  L.bytes = o;
  return L;
}

// External path planning, shared by the planner and the driver.
// Phase 2 (merge): a partition of m records needs two slots of slice + output (400 m), composites (32 m)
// and perms (16 m, when requested): m_target = (budget - K-d lists - 2 MB) / 448.
// Sample stride S: every S-th record of every sorted run is a sample; a partition between two splitters
// holds at most (q + R) S records (q samples apart, plus up to one sample interval from each of the R
// runs), so S <= m_target / (2 R) keeps every partition within m_target.
uint64_t external_merge_target(uint64_t C, uint64_t budget) {
  const uint64_t lists = 7ull * 16 * std::min<uint64_t>(65536, C) + (2ull << 20);
  const uint64_t per_rec = 4 * kRecordBytes + 32 + 16;
  const uint64_t avail = std::max<uint64_t>(budget > lists ? budget - lists : 0, per_rec * 1024);
  return std::max<uint64_t>(1024, avail / per_rec);
}
uint64_t external_sample_stride(uint64_t n, uint64_t C, uint64_t budget) {
  if (C == 0) return 1;
  const uint64_t R = (n + C - 1) / C;
  uint64_t S = std::min<uint64_t>(4096, C / 16);
  if (budget) S = std::min<uint64_t>(S, external_merge_target(C, budget) / (2 * R));
  return std::max<uint64_t>(1, S);
}
// Phase 1 (runs): the largest run C (records) whose run-generation working set fits the budget: two
// slots of run in + run out (400 C; run r+1 streams in and run r-1 streams out while run r sorts) + the
// internal sort's workspace and K-d lists for C records + two runs' perms (8 C) + the samples and their
// sort + 2 MB slack.
uint64_t external_run_need(uint64_t n, uint64_t C, uint64_t budget) {
  if (C == 0) return 0;
  const uint64_t S = external_sample_stride(n, C, budget);
  const uint64_t runs = (n + C - 1) / C;
  const uint64_t nsamp = runs * ((C + S - 1) / S);
  const uint64_t lists = 6ull * 16 * std::min<uint64_t>(65536, C) + 16ull * std::min<uint64_t>(65536, C);
  return 408 * C + plan_internal(C).bytes + lists + 2 * 100 * nsamp + 4 * nsamp + plan_internal(nsamp).bytes +
         (2ull << 20);
}

uint64_t external_run_records(uint64_t n, uint64_t budget) {
  Options o = options_snapshot();
  if (o.ext_run_records > 0) return std::min<uint64_t>(n, (uint64_t)o.ext_run_records);
  uint64_t lo = 0, hi = std::min<uint64_t>(n, 0xFFFFFFFEull);
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo + 1) / 2;
    if (external_run_need(n, mid, budget) <= budget) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Device bytes the internal path holds outside its workspace: the K-d work lists (6 tiers of 16-byte
// bucket descriptors, level 1: one per 16-bit bucket; deeper levels: at most 256 children of each of the
// <= n / 16385 big buckets), the big-bucket lists and the recursion arrays (each at least 1 MB): per big
// bucket 2 x 256 u32 histograms/cursors (<= n / 8 bytes) plus per-chunk and per-bucket words (<= n / 256).
uint64_t internal_aux_bytes(uint64_t n) {
  const uint64_t buckets = std::max<uint64_t>(std::min<uint64_t>(65536, n), n / 64 + 1);
  return (uint64_t)kNumKdListsHost * align256(16 * buckets) + 2 * std::max<uint64_t>(1 << 20, 16 * (n / 16385 + 1)) +
         std::max<uint64_t>(1 << 20, n / 8 + n / 256 + (64 << 10));
}

ley_status ensure_copy_streams(DeviceContext& ctx) {
  if (ctx.copy_stream[0]) return LEY_OK;
  for (int i = 0; i < 2; ++i) LEY_CUDA("copy streams", cudaStreamCreateWithFlags(&ctx.copy_stream[i], cudaStreamNonBlocking));
  for (int i = 0; i < DeviceContext::kExtEvents; ++i)
    LEY_CUDA("copy streams", cudaEventCreateWithFlags(&ctx.ev[i], cudaEventDisableTiming));
  return LEY_OK;
}

ley_status copy_split(DeviceContext& ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                      cudaStream_t s, int parts) {
  parts = std::max(1, std::min(parts, DeviceContext::kSplitParts));
  if (parts == 1 || bytes < ((size_t)256 << 20)) {
    LEY_CUDA("copy", cudaMemcpyAsync(dst, src, bytes, kind, s));
    return LEY_OK;
  }
  if (!ctx.split_stream[0]) {
    for (auto& st : ctx.split_stream) LEY_CUDA("copy streams", cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& e : ctx.split_ev) LEY_CUDA("copy streams", cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  LEY_CUDA("copy", cudaEventRecord(ctx.split_ev[0], s));
  const size_t piece = ((bytes / parts) + 255) & ~size_t(255);
  for (int i = 0; i < parts; ++i) {
    const size_t a = std::min(bytes, (size_t)i * piece), b = i == parts - 1 ? bytes : std::min(bytes, a + piece);
    LEY_CUDA("copy", cudaStreamWaitEvent(ctx.split_stream[i], ctx.split_ev[0], 0));
    if (b > a)
      LEY_CUDA("copy", cudaMemcpyAsync(static_cast<uint8_t*>(dst) + a, static_cast<const uint8_t*>(src) + a, b - a, kind,
                                       ctx.split_stream[i]));
    LEY_CUDA("copy", cudaEventRecord(ctx.split_ev[i + 1], ctx.split_stream[i]));
    LEY_CUDA("copy", cudaStreamWaitEvent(s, ctx.split_ev[i + 1], 0));
  }
  return LEY_OK;
}

uint64_t resident_chunk_records(uint64_t n) {
  const int64_t o = options_snapshot().resident_chunk_records;
  const uint64_t c = o > 0 ? (uint64_t)o : (uint64_t)1 << 21;  // 210 MB windows: full-speed D2H copies
  // at most a quarter of n, so the two windows stay below the output buffer the staged path would need
  return std::max<uint64_t>(1, std::min<uint64_t>((n + 3) / 4, c));
}

uint64_t resident_bytes(uint64_t n) {
  return plan_internal(n).bytes + internal_aux_bytes(n) + align256(100 * n) + align256(4 * n) +
         2 * align256(100 * resident_chunk_records(n));
}

ley_status plan_query(uint64_t n, uint64_t budget, ley_plan_info* info) {
  if (!info) {
    set_error("ley_plan_query: NULL info");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  if (n > LEY_MAX_RECORDS) {
    set_error("ley_plan_query: n_records > 2^32-2");
    return LEY_ERR_TOO_LARGE;
  }
  memset(info, 0, sizeof(*info));
  InternalLayout L = plan_internal(n);
  info->n_records = n;
  info->tile_records = kTileRecords;
  info->tiles = L.tiles;
  info->chunk_records = kChunk;
  info->internal_scratch = L.bytes + internal_aux_bytes(n);
  info->staged_bytes = info->internal_scratch + 2 * align256(100 * n);
  info->resident_bytes = resident_bytes(n);
  if (budget == 0 || info->staged_bytes <= budget)
    info->host_path = 0;
  else if (options_snapshot().resident_path && info->resident_bytes <= budget)
    info->host_path = 2;
  else
    info->host_path = 1;
  if (info->host_path == 1) {
    info->run_records = external_run_records(n, budget);
    info->runs = info->run_records ? (n + info->run_records - 1) / info->run_records : 0;
  } else {
    info->run_records = n;
    info->runs = n ? 1 : 0;
  }
  return LEY_OK;
}

// ------------------------------------------------------------------ arena
namespace {
std::mutex g_ctx_mu;
std::unique_ptr<DeviceContext> g_ctx[64];
}  // namespace

DeviceContext& device_context(int device) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  if (!g_ctx[device]) {
    g_ctx[device].reset(new DeviceContext());
    g_ctx[device]->device = device;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
      g_ctx[device]->sms = sms;
    else
      cudaGetLastError();
  }
  return *g_ctx[device];
}

// Device bytes held by the library's cached buffers (all devices) and their high-water mark.
namespace {
std::atomic<uint64_t> g_dev_bytes{0}, g_dev_peak{0};
}
void track_device_bytes(int64_t delta) {
  const uint64_t now = g_dev_bytes.fetch_add((uint64_t)delta) + (uint64_t)delta;
  uint64_t pk = g_dev_peak.load();
  while (now > pk && !g_dev_peak.compare_exchange_weak(pk, now)) {
  }
}
void device_bytes(uint64_t* current, uint64_t* peak, bool reset_peak) {
  if (current) *current = g_dev_bytes.load();
  if (peak) *peak = g_dev_peak.load();
  if (reset_peak) g_dev_peak.store(g_dev_bytes.load());
}

ley_status ensure_buffer(DeviceBuffer& b, size_t bytes, const char* what, cudaStream_t s) {
  if (b.cap >= bytes && b.ptr) return LEY_OK;
  if (b.ptr) {
    LEY_CUDA(what, cudaStreamSynchronize(s));
    LEY_CUDA(what, cudaFree(b.ptr));
    track_device_bytes(-(int64_t)b.cap);
    b.ptr = nullptr;
    b.cap = 0;
  }
  size_t want = std::max<size_t>(bytes, 1 << 20);
  cudaError_t e = cudaMalloc(&b.ptr, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    b.ptr = nullptr;
    set_error(std::string(what) + ": cudaMalloc of " + std::to_string(want) + " bytes failed (" +
              cudaGetErrorString(e) + ")");
    return LEY_ERR_CUDA;
  }
  b.cap = want;
  track_device_bytes((int64_t)want);
  if (getenv("LEY_DEBUG_ALLOC")) fprintf(stderr, "[ley alloc] %s: %zu bytes (held %llu)\n", what, want,
                                         (unsigned long long)g_dev_bytes.load());
  return LEY_OK;
}

uint64_t options_fingerprint(const Options& o) {
  uint64_t h = 1469598103934665603ull;
  for (const OptDesc& d : kOpts)
    if (d.field != &Options::async)  // (host-side only: the captured level-1 sequence does not depend on it)
      h = (h ^ (uint64_t)(o.*(d.field))) * 1099511628211ull;
  return h;
}

ley_status async_join(DeviceContext& c, cudaStream_t s) {
  if (!c.async_pending) return LEY_OK;
  c.async_pending = false;
  if (s != c.async_stream) LEY_CUDA("async join", cudaStreamWaitEvent(s, c.async_ev, 0));
  return LEY_OK;
}

ley_status async_drain(DeviceContext& c) {
  if (!c.async_pending) return LEY_OK;
  c.async_pending = false;
  LEY_CUDA("async drain", cudaEventSynchronize(c.async_ev));
  return LEY_OK;
}

void graphs_release(DeviceContext& c) {
  for (auto& g : c.graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  c.graphs.clear();
}

ley_status graph_run(DeviceContext& ctx, const GraphKey& key, cudaStream_t s,
                     const std::function<ley_status(cudaStream_t)>& fn, Profiler& prof) {
  if (!ctx.graph_stream) {
    LEY_CUDA("graph", cudaStreamCreateWithFlags(&ctx.graph_stream, cudaStreamNonBlocking));
  }
  uint64_t k[13];
  memcpy(k, key.w, sizeof(key.w));
  k[12] = ((uint64_t)(prof.on ? 1 : 0) << 32) | (uint32_t)prof.next_event;  // (event indices are baked in)
  DeviceContext::Graph* g = nullptr;
  for (auto& e : ctx.graphs)
    if (memcmp(e.key, k, sizeof(k)) == 0) g = &e;
  const cudaStream_t prof_stream = prof.stream;
  if (!g) {
    const int launches0 = prof.launches, event0 = prof.next_event;
    const size_t names0 = prof.names.size(), b0 = prof.ev_begin.size(), e0 = prof.ev_end.size();
    cudaGraph_t graph = nullptr;
    LEY_CUDA("graph capture", cudaStreamBeginCapture(ctx.graph_stream, cudaStreamCaptureModeThreadLocal));
    prof.stream = ctx.graph_stream;
    const ley_status st = fn(ctx.graph_stream);
    prof.stream = prof_stream;
    const cudaError_t ce = cudaStreamEndCapture(ctx.graph_stream, &graph);
    cudaGraphExec_t exec = nullptr;
    DeviceContext::Graph ng;
    ng.names.assign(prof.names.begin() + names0, prof.names.end());
    ng.ev_begin.assign(prof.ev_begin.begin() + b0, prof.ev_begin.end());
    ng.ev_end.assign(prof.ev_end.begin() + e0, prof.ev_end.end());
    ng.events = prof.next_event - event0;
    ng.launches = prof.launches - launches0;
    prof.names.resize(names0);  // (the replay below adds them back)
    prof.ev_begin.resize(b0);
    prof.ev_end.resize(e0);
    prof.next_event = event0;
    prof.launches = launches0;
    const cudaError_t ie = (st || ce != cudaSuccess || !graph) ? cudaErrorUnknown : cudaGraphInstantiate(&exec, graph, 0);
    if (ie != cudaSuccess) {
      if (getenv("LEY_DEBUG_GRAPH"))
        fprintf(stderr, "[ley] graph capture failed: fn %d (%s), end %s, instantiate %s\n", (int)st, last_error(),
                cudaGetErrorString(ce), cudaGetErrorString(ie));
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      return fn(s);  // (capture is an optimisation: run the sequence directly)
    }
    cudaGraphDestroy(graph);
    if (ctx.graphs.size() >= 8) {  // evict the least recently used
      auto lru = std::min_element(ctx.graphs.begin(), ctx.graphs.end(),
                                  [](const auto& x, const auto& y) { return x.used < y.used; });
      cudaGraphExecDestroy(lru->exec);
      ctx.graphs.erase(lru);
    }
    memcpy(ng.key, k, sizeof(k));
    ng.exec = exec;
    ctx.graphs.push_back(std::move(ng));
    g = &ctx.graphs.back();
  }
  g->used = ++ctx.graph_clock;
  LEY_CUDA("graph", cudaGraphLaunch(g->exec, s));  // (captured on graph_stream; replayed in the caller's stream order)
  prof.launches += g->launches;
  prof.names.insert(prof.names.end(), g->names.begin(), g->names.end());
  prof.ev_begin.insert(prof.ev_begin.end(), g->ev_begin.begin(), g->ev_begin.end());
  prof.ev_end.insert(prof.ev_end.end(), g->ev_end.begin(), g->ev_end.end());
  prof.next_event += g->events;
  return LEY_OK;
}

void release_device(int device) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  for (int d = 0; d < 64; ++d) {
    if (device >= 0 && d != device) continue;
    if (!g_ctx[d]) continue;
    DeviceContext& c = *g_ctx[d];
    pipe_release(c);  // stops the streaming worker first (it takes c.mu for its sorts)
    std::lock_guard<std::mutex> g2(c.mu);
    async_drain(c);     // (a stream-ordered sort may still use the buffers)
    graphs_release(c);  // (they hold this context's buffer and pinned-counter addresses)
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(d);
    for (DeviceBuffer* b : {&c.work, &c.lists, &c.big[0], &c.big[1], &c.rec, &c.stage, &c.ext, &c.keypass}) {
      if (b->ptr) {
        cudaFree(b->ptr);
        track_device_bytes(-(int64_t)b->cap);
      }
      b->ptr = nullptr;
      b->cap = 0;
    }
    if (c.host_pinned) cudaFreeHost(c.host_pinned);
    c.host_pinned = nullptr;
    if (c.host_scratch) cudaFreeHost(c.host_scratch);
    c.host_scratch = nullptr;
    c.host_scratch_cap = 0;
    for (int i = 0; i < 2; ++i) {
      if (c.copy_stream[i]) cudaStreamDestroy(c.copy_stream[i]);
      c.copy_stream[i] = nullptr;
    }
    for (int i = 0; i < DeviceContext::kExtEvents; ++i) {
      if (c.ev[i]) cudaEventDestroy(c.ev[i]);
      c.ev[i] = nullptr;
    }
    for (cudaEvent_t e : c.events) cudaEventDestroy(e);
    c.events.clear();
    cudaSetDevice(prev);
  }
}

// ------------------------------------------------------------------ profiling
namespace {
struct StageRecord {
  std::vector<const char*> names;
  std::vector<float> ms;
  int launches = 0;
};
thread_local StageRecord g_stages;
}  // namespace

// Every stage is also an NVTX range (header-only NVTX3: a no-op unless a tool such as Nsight Systems
// is attached), so the sort's stages show up on a profiler timeline without the "profile" option.
ley_status Profiler::begin(const char* name) {
  nvtxRangePushA(name);
  ++nvtx_depth;
  if (!on) return LEY_OK;
  int need = next_event + 2;
  while ((int)ctx->events.size() < need) {
    cudaEvent_t e;
    LEY_CUDA("profiler", cudaEventCreate(&e));
    ctx->events.push_back(e);
  }
  names.push_back(name);
  ev_begin.push_back(next_event);
  LEY_CUDA("profiler", cudaEventRecord(ctx->events[next_event++], stream));
  return LEY_OK;
}

ley_status Profiler::end() {
  if (nvtx_depth > 0) {
    nvtxRangePop();
    --nvtx_depth;
  }
  if (!on) return LEY_OK;
  ev_end.push_back(next_event);
  LEY_CUDA("profiler", cudaEventRecord(ctx->events[next_event++], stream));
  return LEY_OK;
}

Profiler::~Profiler() {
  while (nvtx_depth-- > 0) nvtxRangePop();
}

void Profiler::finish() {
  g_stages.names.clear();
  g_stages.ms.clear();
  g_stages.launches = launches;
  if (!on) return;
  // stages that recur (one per MSD recursion level) are summed under their name, in first-use order
  for (size_t i = 0; i < names.size() && i < ev_end.size(); ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->events[ev_begin[i]], ctx->events[ev_end[i]]) != cudaSuccess) {
      cudaGetLastError();  // (a stage without a valid pair of events reports 0 rather than poisoning the next call)
      ms = 0.f;
    }
    size_t k = 0;
    while (k < g_stages.names.size() && strcmp(g_stages.names[k], names[i]) != 0) ++k;
    if (k == g_stages.names.size()) {
      g_stages.names.push_back(names[i]);
      g_stages.ms.push_back(0.f);
    }
    g_stages.ms[k] += ms;
  }
}

void record_launches(int launches) {  // a call without stage profiling: no stale stage list
  g_stages.names.clear();
  g_stages.ms.clear();
  g_stages.launches = launches;
}

int stage_times(const char** names, float* ms, int max, int* launches) {
  int k = 0;
  for (size_t i = 0; i < g_stages.names.size() && k < max; ++i, ++k) {
    if (names) names[k] = g_stages.names[i];
    if (ms) ms[k] = g_stages.ms[i];
  }
  if (launches) *launches = g_stages.launches;
  return k;
}

}  // namespace ley
