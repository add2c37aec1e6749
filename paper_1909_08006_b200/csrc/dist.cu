// dist.cpp — multi-GPU key-range sort: host orchestration over NCCL, and
// a loopback transport that runs the same G-rank algorithm on one device.
//
// BASELINE.json north_star: "Each GPU histograms the leading key bytes, all GPUs agree on range
// splitters, and records move to their owning GPU by an NCCL all-to-all over NVLink; each GPU then sorts
// its range locally, and the output is the concatenation of the ranges."
//
// Phases of one rank (collectives between them):
//   P1  K-s0 local hist16 of key bytes 0..1                       C1 allreduce(hist16), allgather(n_local)
//   P2  plan: split ranks q_k = floor(k N / G), k = 1..G-1 -> boundary bin b_k and rank rho_k inside it
//       (ley_dist_plan_splitters); K-s1 compacts this rank's records of the boundary bins (with global
//       ordinals)                                                 C2 allgather(candidate counts, candidates)
//   P3  sort all candidates (the internal sort: order = (key, global ordinal)), splitter s_k = candidate
//       at (first candidate of bin b_k) + rho_k -> exact (key, ordinal) splitters, identical on all ranks
//   P4  send counts per destination: whole bins from the local hist16 (ley_dist_bin_dest_counts) +
//       K-s2 over the local candidates                             C3 allgather(send counts G x G)
//   P5  exchange plan (ley_dist_plan_exchange); K-p stable partition into the send buffer
//                                                                  C4 all-to-all-v (grouped send/recv)
//   P6  internal sort of the received records (K-a..K-e); receive order = global ordinal order.
// With exact splitters rank r ends up with global sorted positions [floor(r N/G), floor((r+1) N/G)).
#include <fcntl.h>
#include <nccl.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/statvfs.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <thread>
#include <vector>

#include "kernels.cuh"
#include "runtime.h"

namespace ley {

// ------------------------------------------------------------------------------- host planning (pure)
// For k = 1..G-1: q_k = floor(k N / G); bin b_k = the 16-bit prefix bin holding global sorted rank q_k;
// rho_k = q_k - (records in bins < b_k). bin_first_k = records in bins < b_k.
int dist_plan_splitters(const uint64_t* hist, uint64_t N, int G, uint32_t* bins, uint64_t* rho, uint64_t* first) {
  if (G < 1 || G > kMaxRanks) return 1;
  uint64_t cum = 0;
  uint32_t b = 0;
  for (int k = 1; k < G; ++k) {
    const uint64_t q = (uint64_t)((unsigned __int128)k * N / (unsigned)G);
    while (b < 65536 && cum + hist[b] <= q) {
      cum += hist[b];
      ++b;
    }
    if (b >= 65536) return 2;  // q >= N: impossible for k < G and N > 0
    bins[k - 1] = b;
    rho[k - 1] = q - cum;
    first[k - 1] = cum;
  }
  return 0;
}

// Destination counts of the whole (non-boundary) bins of a local histogram: bin b goes to rank
// #{k : b_k < b}; the boundary bins themselves are counted from the candidates (K-s2).
void dist_bin_dest_counts(const uint64_t* local_hist, const uint32_t* bins, int nspl, uint64_t* counts) {
  for (int d = 0; d <= nspl; ++d) counts[d] = 0;
  for (uint32_t b = 0; b < 65536; ++b) {
    if (!local_hist[b]) continue;
    bool boundary = false;
    int d = 0;
    for (int k = 0; k < nspl; ++k) {
      if (bins[k] == b) boundary = true;
      if (bins[k] < b) ++d;
    }
    if (!boundary) counts[d] += local_hist[b];
  }
}

// send_counts[src * G + dst] (records). Receive order = source rank order (= global ordinal order).
void dist_plan_exchange(const uint64_t* send_counts, int G, int rank, uint64_t* recv_counts, uint64_t* recv_off,
                        uint64_t* send_off, uint64_t* n_out, uint64_t* out_off) {
  uint64_t acc = 0;
  for (int s = 0; s < G; ++s) {
    recv_counts[s] = send_counts[(size_t)s * G + rank];
    recv_off[s] = acc;
    acc += recv_counts[s];
  }
  *n_out = acc;
  uint64_t so = 0;
  for (int d = 0; d < G; ++d) {
    send_off[d] = so;
    so += send_counts[(size_t)rank * G + d];
  }
  uint64_t before = 0;
  for (int r = 0; r < rank; ++r)
    for (int s = 0; s < G; ++s) before += send_counts[(size_t)s * G + r];
  *out_off = before;
}

// Fused exchange: where source rank `rank`'s run starts inside each destination's receive buffer
// (records) = what lower source ranks send to that destination (receive order = source rank order).
void dist_dest_offsets(const uint64_t* send_counts, int G, int rank, uint64_t* dst_off) {
  for (int d = 0; d < G; ++d) {
    uint64_t acc = 0;
    for (int s = 0; s < rank; ++s) acc += send_counts[(size_t)s * G + d];
    dst_off[d] = acc;
  }
}

namespace {

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

#define LEY_NCCL(stage, expr)                                                                   \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess) {                                                                    \
      ::ley::set_error(std::string(stage) + ": " + ncclGetErrorString(_r) + " at " #expr);     \
      return LEY_ERR_NCCL;                                                                      \
    }                                                                                           \
  } while (0)

// Per-rank state of one distributed sort.
struct RankState {
  int rank = 0;
  DeviceContext* ctx = nullptr;
  cudaStream_t s = nullptr;
  const uint8_t* in = nullptr;
  uint64_t n = 0;
  uint8_t* out = nullptr;
  uint64_t cap = 0;
  uint64_t gbase = 0;
  uint32_t key_bytes = 10;  // keys = record bytes [0, key_bytes), 1..10
  DistKeyMask km;
  // device scratch (one buffer)
  DeviceBuffer buf;
  uint32_t* d_hist = nullptr;        // [65536]
  uint64_t* d_status = nullptr;      // look-back status (candidates / partition)
  uint32_t* d_small = nullptr;       // tickets, counts
  uint8_t* d_cand = nullptr;         // local candidates (records)
  uint32_t* d_cand_gidx = nullptr;
  unsigned long long* d_dcount = nullptr;  // [kMaxRanks]
  uint64_t* d_doff = nullptr;        // [kMaxRanks] K-p: start of this rank's run at each destination
  uint8_t** d_dptr = nullptr;        // [kMaxRanks] K-p: destination bases (send buffer or receive windows)
  DistSplitter* d_spl = nullptr;     // [kMaxRanks]
  uint32_t* d_bins = nullptr;        // [kMaxRanks]
  uint16_t* d_pref = nullptr;        // n 16-bit key prefixes (K-s0 -> K-s1)
  uint8_t* d_recv = nullptr;         // received records
  uint64_t recv_cap = 0;
  // host side
  std::vector<uint64_t> hist;        // local hist16 (u64)
  uint32_t ncand = 0;
  uint64_t send_counts[kMaxRanks] = {0};
  uint64_t recv_counts[kMaxRanks], recv_off[kMaxRanks], send_off[kMaxRanks];
  uint64_t n_out = 0, out_off = 0;
  int launches = 0;  // kernels this rank launched in the current sort (reported by ley_stage_times)
  // grow-only caches, so repeated sorts allocate nothing on the hot path
  DeviceBuffer cand_buf, split_buf, recv_buf, send_buf;
  uint32_t* h_hist = nullptr;  // pinned: [0, 65536) local hist16, [65536, 131072) the global one
  ~RankState() {
    if (h_hist) cudaFreeHost(h_hist);
    for (DeviceBuffer* b : {&buf, &cand_buf, &split_buf, &recv_buf, &send_buf})
      if (b->ptr) {
        cudaFree(b->ptr);
        track_device_bytes(-(int64_t)b->cap);
      }
  }
};

// Shared (replicated) plan of the sort.
struct Plan {
  int G = 1;
  uint64_t N = 0;
  std::vector<uint64_t> n_local, ghist;
  uint32_t bins[kMaxRanks] = {0};
  uint64_t rho[kMaxRanks] = {0}, first[kMaxRanks] = {0};
  DistSplitter spl[kMaxRanks];
  std::vector<uint64_t> send_matrix;  // G x G
  int launches = 0;                   // replicated-phase kernels (the candidate sort)
};

ley_status rank_alloc(RankState& r) {
  const uint64_t n = std::max<uint64_t>(r.n, 1);
  const uint64_t cand_cap = n;  // worst case: every record in a boundary bin
  const uint64_t status_words = std::max<uint64_t>(std::max<uint64_t>(ks_candidate_tiles(n), kp_tiles(n) * kMaxRanks), 128) + 16;
  size_t o = 0;
  auto take = [&](size_t b) { size_t at = o; o += a256(b); return at; };
  const size_t o_hist = take(4 * 65536), o_status = take(8 * status_words), o_small = take(256),
               o_cand = take(cand_cap * kRecordBytes), o_cgidx = take(4 * cand_cap), o_dcount = take(8 * kMaxRanks),
               o_doff = take(8 * kMaxRanks), o_dptr = take(8 * kMaxRanks),
               o_spl = take(sizeof(DistSplitter) * kMaxRanks), o_bins = take(4 * kMaxRanks), o_pref = take(2 * n);
  if (r.buf.cap < o) {
    if (r.buf.ptr) {
      cudaFree(r.buf.ptr);
      track_device_bytes(-(int64_t)r.buf.cap);
    }
    r.buf.ptr = nullptr;
    r.buf.cap = 0;
    LEY_CUDA("dist alloc", cudaMalloc(&r.buf.ptr, o));
    r.buf.cap = o;
    track_device_bytes((int64_t)o);
  }
  uint8_t* b = static_cast<uint8_t*>(r.buf.ptr);
  r.d_hist = reinterpret_cast<uint32_t*>(b + o_hist);
  r.d_status = reinterpret_cast<uint64_t*>(b + o_status);
  r.d_small = reinterpret_cast<uint32_t*>(b + o_small);
  r.d_cand = b + o_cand;
  r.d_cand_gidx = reinterpret_cast<uint32_t*>(b + o_cgidx);
  r.d_dcount = reinterpret_cast<unsigned long long*>(b + o_dcount);
  r.d_doff = reinterpret_cast<uint64_t*>(b + o_doff);
  r.d_dptr = reinterpret_cast<uint8_t**>(b + o_dptr);
  r.d_spl = reinterpret_cast<DistSplitter*>(b + o_spl);
  r.d_bins = reinterpret_cast<uint32_t*>(b + o_bins);
  r.d_pref = reinterpret_cast<uint16_t*>(b + o_pref);
  return LEY_OK;
}

// ---------------------------------------------------------------------------- phases (one rank)
ley_status phase1_hist(RankState& r) {
  LEY_CUDA("K-s0 hist", cudaMemsetAsync(r.d_hist, 0, 4 * 65536, r.s));
  LEY_CUDA("K-s0 hist", launch_ks_hist16(r.in, r.n, r.d_hist, r.d_pref, r.km, r.ctx->sms, r.s));
  r.launches += 1;
  return LEY_OK;
}

ley_status phase2_candidates(RankState& r, const Plan& P) {
  const int nspl = P.G - 1;
  LEY_CUDA("K-s1 candidates", cudaMemcpyAsync(r.d_bins, P.bins, 4 * std::max(nspl, 1), cudaMemcpyHostToDevice, r.s));
  LEY_CUDA("K-s1 candidates", cudaMemsetAsync(r.d_small, 0, 256, r.s));
  LEY_CUDA("K-s1 candidates", cudaMemsetAsync(r.d_status, 0, 8 * (ks_candidate_tiles(r.n) + 1), r.s));
  r.launches += 1;
  LEY_CUDA("K-s1 candidates", launch_ks_candidates(r.in, r.d_pref, r.n, (uint32_t)r.gbase, r.d_bins, nspl, r.d_status,
                                                   r.d_small + 0, r.d_cand, r.d_cand_gidx, r.d_small + 1, r.s));
  uint32_t* h = static_cast<uint32_t*>(r.ctx->host_pinned);
  LEY_CUDA("K-s1 candidates", cudaMemcpyAsync(h, r.d_small + 1, 4, cudaMemcpyDeviceToHost, r.s));
  LEY_CUDA("K-s1 candidates", cudaStreamSynchronize(r.s));
  r.ncand = r.n ? h[0] : 0;
  return LEY_OK;
}

// Given all candidates concatenated in rank order (device records + ordinals), find the exact splitters.
ley_status phase3_splitters(DeviceContext& ctx, cudaStream_t s, const uint8_t* all_cand, const uint32_t* all_gidx,
                            uint64_t total_cand, Plan& P, DeviceBuffer& tmp, uint32_t key_bytes) {
  const int nspl = P.G - 1;
  if (nspl == 0) return LEY_OK;
  const InternalLayout L = plan_internal(total_cand);
  const size_t bytes = a256(total_cand * kRecordBytes) + a256(4 * total_cand) + a256(L.bytes);
  ley_status est = ensure_buffer(tmp, bytes, "K-s splitters", s);
  if (est) return est;
  uint8_t* sorted = static_cast<uint8_t*>(tmp.ptr);
  uint32_t* perm = reinterpret_cast<uint32_t*>(sorted + a256(total_cand * kRecordBytes));
  uint8_t* work = reinterpret_cast<uint8_t*>(perm) + a256(4 * total_cand);
  Profiler quiet;
  quiet.ctx = &ctx;
  quiet.stream = s;
  ley_status st = sort_internal_device(ctx, all_cand, sorted, perm, total_cand, s, quiet, work, L.bytes, key_bytes);
  if (st) return st;
  P.launches += quiet.launches;
  // first sorted index of each boundary bin = candidates in smaller boundary bins; all splitters' key
  // bytes and sorted positions are read back in one batch, then their global ordinals in a second
  std::vector<uint64_t> at(nspl);
  for (int k = 0; k < nspl; ++k) {
    uint64_t start = 0;
    std::vector<uint32_t> seen;
    for (int j = 0; j < nspl; ++j) {
      if (P.bins[j] < P.bins[k] && std::find(seen.begin(), seen.end(), P.bins[j]) == seen.end()) {
        start += P.ghist[P.bins[j]];
        seen.push_back(P.bins[j]);
      }
    }
    at[k] = start + P.rho[k];
  }
  uint8_t keys[kMaxRanks][12] = {};
  uint32_t pidx[kMaxRanks] = {}, gidx[kMaxRanks] = {};
  for (int k = 0; k < nspl; ++k) {
    LEY_CUDA("K-s splitters", cudaMemcpyAsync(keys[k], sorted + at[k] * kRecordBytes, 10, cudaMemcpyDeviceToHost, s));
    LEY_CUDA("K-s splitters", cudaMemcpyAsync(&pidx[k], perm + at[k], 4, cudaMemcpyDeviceToHost, s));
  }
  LEY_CUDA("K-s splitters", cudaStreamSynchronize(s));
  for (int k = 0; k < nspl; ++k)
    LEY_CUDA("K-s splitters", cudaMemcpyAsync(&gidx[k], all_gidx + pidx[k], 4, cudaMemcpyDeviceToHost, s));
  LEY_CUDA("K-s splitters", cudaStreamSynchronize(s));
  for (int k = 0; k < nspl; ++k) {
    const uint8_t* key = keys[k];
    DistSplitter& d = P.spl[k];
    d.hi = ((uint32_t)key[0] << 24) | ((uint32_t)key[1] << 16) | ((uint32_t)key[2] << 8) | key[3];
    d.mid = ((uint32_t)key[4] << 24) | ((uint32_t)key[5] << 16) | ((uint32_t)key[6] << 8) | key[7];
    d.lo16 = ((uint32_t)key[8] << 8) | key[9];
    const DistKeyMask km = dist_key_mask(key_bytes);
    d.hi &= km.hi;
    d.mid &= km.mid;
    d.lo16 &= km.lo16;
    d.gidx = gidx[k];
  }
  return LEY_OK;
}

// K-s2 on the device, accumulated onto the whole-bin counts in r.d_dcount (left there for the all-gather;
// nothing is read back here).
ley_status phase4_counts_device(RankState& r, const Plan& P) {
  const int nspl = P.G - 1;
  dist_bin_dest_counts(r.hist.data(), P.bins, nspl, r.send_counts);
  LEY_CUDA("K-s2 counts", cudaMemcpyAsync(r.d_dcount, r.send_counts, 8 * P.G, cudaMemcpyHostToDevice, r.s));
  if (nspl == 0) return LEY_OK;
  LEY_CUDA("K-s2 counts", cudaMemcpyAsync(r.d_spl, P.spl, sizeof(DistSplitter) * nspl, cudaMemcpyHostToDevice, r.s));
  r.launches += 1;
  LEY_CUDA("K-s2 counts", launch_ks_dest_counts(r.d_cand, r.d_cand_gidx, r.ncand, r.d_spl, nspl, r.d_dcount,
                                                r.km, r.ctx->sms, r.s));
  return LEY_OK;
}

ley_status phase4_counts(RankState& r, const Plan& P) {
  const int nspl = P.G - 1;
  dist_bin_dest_counts(r.hist.data(), P.bins, nspl, r.send_counts);
  if (nspl == 0) return LEY_OK;
  LEY_CUDA("K-s2 counts", cudaMemcpyAsync(r.d_spl, P.spl, sizeof(DistSplitter) * nspl, cudaMemcpyHostToDevice, r.s));
  LEY_CUDA("K-s2 counts", cudaMemsetAsync(r.d_dcount, 0, 8 * kMaxRanks, r.s));
  r.launches += 1;
  LEY_CUDA("K-s2 counts", launch_ks_dest_counts(r.d_cand, r.d_cand_gidx, r.ncand, r.d_spl, nspl, r.d_dcount,
                                                r.km, r.ctx->sms, r.s));
  unsigned long long c[kMaxRanks];
  LEY_CUDA("K-s2 counts", cudaMemcpyAsync(c, r.d_dcount, 8 * kMaxRanks, cudaMemcpyDeviceToHost, r.s));
  LEY_CUDA("K-s2 counts", cudaStreamSynchronize(r.s));
  for (int d = 0; d <= nspl; ++d) r.send_counts[d] += c[d];
  return LEY_OK;
}

// P5a: the exchange plan of this rank (receive layout, send segments, its output range).
ley_status phase5_plan(RankState& r, const Plan& P) {
  dist_plan_exchange(P.send_matrix.data(), P.G, r.rank, r.recv_counts, r.recv_off, r.send_off, &r.n_out, &r.out_off);
  if (r.n_out > r.cap) {
    set_error("dist: rank " + std::to_string(r.rank) + " must hold " + std::to_string(r.n_out) +
              " records but out_capacity_records is " + std::to_string(r.cap));
    return LEY_ERR_CAPACITY;
  }
  return LEY_OK;
}

// P5b: K-p. Destination d's run of this rank starts at record off[d] of base d: bases come either as a
// host array (copied into r.d_dptr) or as a device array already filled (peer window pointers).
ley_status phase5_partition(RankState& r, const Plan& P, uint8_t* const* host_bases, uint8_t* const* dev_bases,
                            const uint64_t* off, bool remote) {
  const int G = P.G;
  if (host_bases) {
    LEY_CUDA("K-p partition", cudaMemcpyAsync(r.d_dptr, host_bases, 8 * G, cudaMemcpyHostToDevice, r.s));
    dev_bases = r.d_dptr;
  }
  LEY_CUDA("K-p partition", cudaMemcpyAsync(r.d_doff, off, 8 * G, cudaMemcpyHostToDevice, r.s));
  LEY_CUDA("K-p partition", cudaMemsetAsync(r.d_small, 0, 256, r.s));
  LEY_CUDA("K-p partition", cudaMemsetAsync(r.d_status, 0, 8 * (kp_tiles(r.n) * kMaxRanks + 1), r.s));
  r.launches += 1;
  LEY_CUDA("K-p partition", launch_kp_partition(r.in, r.n, (uint32_t)r.gbase, r.d_spl, G - 1, dev_bases, r.d_doff,
                                                r.d_status, r.d_small + 2, remote, r.km, r.s));
  return LEY_OK;
}

// K-p into this rank's own send buffer (segments at send_off), for the all-to-all-v transports.
ley_status phase5_partition_send(RankState& r, const Plan& P) {
  if (!r.n) return LEY_OK;
  ley_status st = ensure_buffer(r.send_buf, r.n * kRecordBytes, "dist send buffer", r.s);
  if (st) return st;
  uint8_t* bases[kMaxRanks];
  for (int d = 0; d < P.G; ++d) bases[d] = static_cast<uint8_t*>(r.send_buf.ptr);
  return phase5_partition(r, P, bases, nullptr, r.send_off, false);
}

ley_status phase6_local_sort(RankState& r, const uint8_t* recv) {
  Profiler quiet;
  quiet.ctx = r.ctx;
  quiet.stream = r.s;
  if (r.n_out == 0) return LEY_OK;
  const ley_status st = sort_internal_device(*r.ctx, recv, r.out, nullptr, r.n_out, r.s, quiet, nullptr, 0, r.key_bytes);
  r.launches += quiet.launches;
  return st;
}

// The local histogram into pinned host memory on the rank's stream (queued; read after the next sync).
ley_status host_hist_async(RankState& r) {
  if (!r.h_hist) LEY_CUDA("dist hist", cudaHostAlloc(&r.h_hist, 2 * 4 * 65536, cudaHostAllocDefault));
  LEY_CUDA("dist hist", cudaMemcpyAsync(r.h_hist, r.d_hist, 4 * 65536, cudaMemcpyDeviceToHost, r.s));
  return LEY_OK;
}
void host_hist_take(RankState& r) {
  r.hist.assign(r.h_hist, r.h_hist + 65536);
}

}  // namespace
}  // namespace ley

// ------------------------------------------------------------------------------------ NCCL comm
struct ley_comm {
  int nranks = 0, rank = 0, device = 0;
  ncclComm_t nccl = nullptr;
  ley::RankState state;
  // fused exchange: this rank's receive window (ncclMemAlloc + symmetric registration; same size on every
  // rank) and the device array of every rank's window pointer as seen from this GPU
  void* win_buf = nullptr;
  size_t win_cap = 0;
  ncclWindow_t win = nullptr;
  uint8_t** d_peers = nullptr;
  ley::DeviceBuffer stage;  // pinned host slices: the device copy of this rank's input and output
  int fused_ok = -1;        // fused exchange usable on this communicator (-1: not checked yet)
  uint64_t uid_hash = 0;    // names this communicator's shared host run scratch (external path)
  uint64_t ext_calls = 0;   // (the same count on every rank: calls are collective)
  // fault handling ("any stage failure aborts the pipeline, reports the stage")
  bool aborted = false;                      // ncclCommAbort ran: the communicator refuses further work
  volatile uint32_t* stall_flag = nullptr;  // mapped pinned word releasing the fault-injection stall
  int colls = 0;                             // collectives enqueued by the current call (test hook)
};

namespace ley {

cudaError_t launch_peer_pointers(ncclWindow_t win, int G, uint8_t** out, cudaStream_t s);  // k_exchange.cu
cudaError_t launch_stall(const volatile uint32_t* release, cudaStream_t s);                // k_exchange.cu

namespace {

// ------------------------------------------------------------------ NCCL fault handling
// Every NCCL call goes through comm_wait (an error aborts; ncclInProgress, which only a nonblocking
// communicator returns, is polled through ncclCommGetAsyncError with the timeout), and every host wait on
// a stream that carries a collective goes through comm_sync, which polls the stream and the
// communicator's asynchronous error instead of blocking in cudaStreamSynchronize. An NCCL error, or a
// collective still incomplete after the "nccl_timeout_ms" option (a peer that failed before it, or died),
// aborts the communicator (ncclCommAbort: in-flight NCCL kernels exit) and returns LEY_ERR_NCCL naming the
// stage. Communicator creation and window registration are blocking NCCL calls; the library reaches the
// registration only after an all-rank agreement, so every rank is alive when it starts.
using Clock = std::chrono::steady_clock;

int64_t elapsed_ms(Clock::time_point t0) {
  return std::chrono::duration_cast<std::chrono::milliseconds>(Clock::now() - t0).count();
}

void comm_abort(ley_comm* c, cudaStream_t s) {
  if (c->stall_flag) *c->stall_flag = 1u;
  if (c->nccl && !c->aborted) ncclCommAbort(c->nccl);
  c->aborted = true;
  if (!s) return;
  // let what the aborted kernels leave on the stream drain (bounded), so no buffer is still in use
  const auto t0 = Clock::now();
  while (cudaStreamQuery(s) == cudaErrorNotReady && elapsed_ms(t0) < 10000)
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  cudaGetLastError();
}

ley_status comm_fail(ley_comm* c, cudaStream_t s, const std::string& stage, const std::string& why) {
  comm_abort(c, s);
  set_error(stage + ": " + why + " (rank " + std::to_string(c->rank) + " of " + std::to_string(c->nranks) +
            "; communicator aborted)");
  return LEY_ERR_NCCL;
}

// Completes one NCCL call on the communicator.
ley_status comm_wait(ley_comm* c, cudaStream_t s, ncclResult_t r, const char* stage, const char* what) {
  if (r == ncclSuccess) return LEY_OK;
  if (r != ncclInProgress) return comm_fail(c, s, stage, std::string(ncclGetErrorString(r)) + " at " + what);
  const auto t0 = Clock::now();
  const int64_t to = options_snapshot().nccl_timeout_ms;
  for (;;) {
    ncclResult_t a = ncclInProgress;
    const ncclResult_t q = ncclCommGetAsyncError(c->nccl, &a);
    if (q != ncclSuccess) a = q;
    if (a == ncclSuccess) return LEY_OK;
    if (a != ncclInProgress) return comm_fail(c, s, stage, std::string(ncclGetErrorString(a)) + " at " + what);
    if (elapsed_ms(t0) > to)
      return comm_fail(c, s, stage, std::string("no completion after ") + std::to_string(to) + " ms at " + what);
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// Host wait for stream s, which carries collectives of c.
ley_status comm_sync(ley_comm* c, cudaStream_t s, const char* stage) {
  const auto t0 = Clock::now();
  const int64_t to = options_snapshot().nccl_timeout_ms;
  for (uint32_t spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return LEY_OK;
    if (e != cudaErrorNotReady) {
      set_error(std::string(stage) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") while waiting on the stream");
      return LEY_ERR_CUDA;
    }
    ncclResult_t a = ncclSuccess;
    if (ncclCommGetAsyncError(c->nccl, &a) == ncclSuccess && a != ncclSuccess && a != ncclInProgress)
      return comm_fail(c, s, stage, std::string("NCCL asynchronous error: ") + ncclGetErrorString(a));
    const int64_t ms = elapsed_ms(t0);
    if (ms > to)
      return comm_fail(c, s, stage, "collective not complete after " + std::to_string(to) +
                                        " ms (a peer failed before it or died)");
    // poll tightly for the first millisecond (the usual wait: a sync must not add sleep latency to every
    // phase of a 2-ms sort), then back off
    if (ms < 1) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(20));
    (void)spin;
  }
}

// After each collective: the fault-injection hook (option dist_fault_stall = k holds the stream after the
// k-th collective of the call, as a peer that never completes it would).
ley_status comm_after_collective(ley_comm* c, cudaStream_t s) {
  const int64_t k = options_snapshot().dist_fault_stall;
  if (++c->colls != k) return LEY_OK;
  if (!c->stall_flag) {
    void* p = nullptr;
    LEY_CUDA("dist fault hook", cudaHostAlloc(&p, 64, cudaHostAllocMapped));
    c->stall_flag = static_cast<volatile uint32_t*>(p);
  }
  *c->stall_flag = 0u;
  LEY_CUDA("dist fault hook", launch_stall(c->stall_flag, s));
  return LEY_OK;
}

#define LEY_NCCLC(c, s, stage, expr)                                                   \
  do {                                                                                  \
    if (ley_status _st = ::ley::comm_wait((c), (s), (expr), (stage), #expr)) return _st; \
  } while (0)
#define LEY_COLL(c, s, stage, expr)                                                     \
  do {                                                                                  \
    LEY_NCCLC(c, s, stage, expr);                                                       \
    if (ley_status _st = ::ley::comm_after_collective((c), (s))) return _st;            \
  } while (0)
#define LEY_CSYNC(c, s, stage)                                                          \
  do {                                                                                  \
    if (ley_status _st = ::ley::comm_sync((c), (s), (stage))) return _st;               \
  } while (0)

// All ranks' outcomes summed (NCCL, on s): *any = number of ranks that reported !ok.
ley_status agree(ley_comm* comm, bool ok, cudaStream_t s, uint64_t* any) {
  uint64_t* flag = reinterpret_cast<uint64_t*>(comm->state.d_status);
  const uint64_t bad = ok ? 0 : 1;
  LEY_CUDA("dist agree", cudaMemcpyAsync(flag, &bad, 8, cudaMemcpyHostToDevice, s));
  LEY_COLL(comm, s, "dist agree", ncclAllReduce(flag, flag, 1, ncclUint64, ncclSum, comm->nccl, s));
  LEY_CSYNC(comm, s, "dist agree");  // (a D2H into pageable memory would block in the copy)
  LEY_CUDA("dist agree", cudaMemcpyAsync(any, flag, 8, cudaMemcpyDeviceToHost, s));
  LEY_CSYNC(comm, s, "dist agree");
  return LEY_OK;
}

ley_status window_release(ley_comm* c, cudaStream_t s) {
  ley_status st = LEY_OK;
  if (c->win && !c->aborted) st = comm_wait(c, s, ncclCommWindowDeregister(c->nccl, c->win), "dist window", "deregister");
  if (c->win_buf) {
    ncclMemFree(c->win_buf);
    track_device_bytes(-(int64_t)c->win_cap);
  }
  c->win = nullptr;
  c->win_buf = nullptr;
  c->win_cap = 0;
  return st;
}

// Collective: every rank calls it with the same `bytes` (derived from the replicated send matrix), so
// they all (re)register together. Grow-only with 25% headroom, so repeated sorts register once. The steps
// a rank could fail alone (the allocation, the peer mapping) are each agreed before the next collective
// step, so either every rank ends with a usable window (fused_ok = 1) or every rank falls back to the
// all-to-all transport (fused_ok = 0) together; a failing collective registration is an NCCL error
// (timeout + abort on the ranks left waiting).
ley_status window_ensure(ley_comm* c, size_t bytes, cudaStream_t s) {
  if (c->win && c->win_cap >= bytes) return LEY_OK;
  LEY_CSYNC(c, s, "dist window");  // nothing may still use the old window
  if (ley_status st = window_release(c, s)) return st;
  size_t cap = bytes + bytes / 4;
  cap = (cap + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
  const bool alloc_ok = ncclMemAlloc(&c->win_buf, cap) == ncclSuccess && c->win_buf;
  if (alloc_ok) {
    c->win_cap = cap;
    track_device_bytes((int64_t)cap);
  } else {
    c->win_buf = nullptr;
  }
  uint64_t any = 0;
  if (ley_status st = agree(c, alloc_ok, s, &any)) return st;
  if (any) {  // some rank could not allocate: nobody registers, everybody uses the all-to-all
    window_release(c, s);
    c->fused_ok = 0;
    return LEY_OK;
  }
  LEY_NCCLC(c, s, "dist window", ncclCommWindowRegister(c->nccl, c->win_buf, cap, &c->win, NCCL_WIN_COLL_SYMMETRIC));
  // every peer must be reachable through the window (one NVLink/NVSwitch domain)
  bool peers_ok = true;
  if (!c->d_peers && cudaMalloc(&c->d_peers, 8 * kMaxRanks) != cudaSuccess) {
    cudaGetLastError();
    c->d_peers = nullptr;
    peers_ok = false;
  }
  if (peers_ok) {
    LEY_CUDA("dist window", launch_peer_pointers(c->win, c->nranks, c->d_peers, s));
    uint8_t* hp[kMaxRanks] = {};
    LEY_CUDA("dist window", cudaMemcpyAsync(hp, c->d_peers, 8 * c->nranks, cudaMemcpyDeviceToHost, s));
    LEY_CSYNC(c, s, "dist window");
    for (int d = 0; d < c->nranks; ++d) peers_ok = peers_ok && hp[d] != nullptr;
    // this rank's own run goes through its local mapping: stores through the window's flat (LSA) mapping
    // of local memory measured slower (C2 at G=1: K-p 9.0 vs 7.3 ms)
    LEY_CUDA("dist window", cudaMemcpyAsync(c->d_peers + c->rank, &c->win_buf, 8, cudaMemcpyHostToDevice, s));
  }
  if (ley_status st = agree(c, peers_ok, s, &any)) return st;
  if (any) {
    if (ley_status st = window_release(c, s)) return st;
    c->fused_ok = 0;
    return LEY_OK;
  }
  c->fused_ok = 1;
  return LEY_OK;
}

}  // namespace

ley_status comm_get_unique_id(uint8_t id_out[128]) {
  if (!id_out) {
    set_error("ley_comm_get_unique_id: NULL");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  ncclUniqueId id;
  LEY_NCCL("comm", ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id_out, &id, 128);
  return LEY_OK;
}

ley_status comm_init(ley_comm** comm, int nranks, int rank, const uint8_t id[128], int device) {
  if (!comm || !id || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) {
    set_error("ley_comm_init: invalid arguments (1 <= nranks <= 8, 0 <= rank < nranks)");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  LEY_CUDA("comm", cudaSetDevice(device));
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  std::unique_ptr<ley_comm> c(new ley_comm());
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  // blocking communicator (a nonblocking one sets up symmetric windows asynchronously: the peer-pointer
  // kernel then read an unfinished window, measured); the waits that can hang on a dead peer are the stream
  // waits after collectives, and those go through comm_sync's timeout
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 1;
  const ncclResult_t ir = ncclCommInitRankConfig(&c->nccl, nranks, uid, rank, &cfg);
  if (ir != ncclSuccess && ir != ncclInProgress) {
    set_error(std::string("comm: ") + ncclGetErrorString(ir) + " at ncclCommInitRankConfig");
    return LEY_ERR_NCCL;
  }
  if (ley_status st = comm_wait(c.get(), nullptr, ir, "comm", "ncclCommInitRankConfig")) return st;  // aborted
  uint64_t h = 1469598103934665603ull;  // FNV-1a of the unique id
  for (int i = 0; i < 128; ++i) h = (h ^ id[i]) * 1099511628211ull;
  c->uid_hash = h;
  *comm = c.release();
  return LEY_OK;
}

ley_status comm_destroy(ley_comm* comm) {
  if (!comm) return LEY_OK;
  cudaSetDevice(comm->device);
  cudaDeviceSynchronize();
  ley_status st = window_release(comm, nullptr);
  if (comm->d_peers) cudaFree(comm->d_peers);
  if (comm->stage.ptr) {
    cudaFree(comm->stage.ptr);
    track_device_bytes(-(int64_t)comm->stage.cap);
  }
  if (comm->nccl && !comm->aborted) {
    // finalize (collective; bounded by the timeout, which aborts instead), then free
    const ley_status fst = comm_wait(comm, nullptr, ncclCommFinalize(comm->nccl), "comm destroy", "ncclCommFinalize");
    if (!st) st = fst;
    if (!comm->aborted) ncclCommDestroy(comm->nccl);
  }
  if (comm->stall_flag) cudaFreeHost(const_cast<uint32_t*>(comm->stall_flag));
  delete comm;
  return st;
}

namespace {
ley_status dist_sort_device(ley_comm* comm, const void* in_local, uint64_t n_local, void* out_local,
                            uint64_t out_capacity, uint64_t* n_out_local, uint64_t* out_global_offset,
                            uint32_t key_bytes, cudaStream_t s) {
  const int G = comm->nranks;
  LEY_CUDA("dist", cudaSetDevice(comm->device));
  DeviceContext& ctx = device_context(comm->device);
  std::lock_guard<std::mutex> guard(ctx.mu);
  if (ley_status ast = async_drain(ctx)) return ast;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, comm->device);
  if (sms > 0) ctx.sms = sms;
  if (!ctx.host_pinned) LEY_CUDA("dist", cudaHostAlloc(&ctx.host_pinned, 4096, cudaHostAllocMapped));
  if (n_local && (!in_local || !out_local)) {
    set_error("dist: NULL in/out with n_local > 0");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  RankState& r = comm->state;
  r.launches = 0;
  r.rank = comm->rank;
  r.ctx = &ctx;
  r.s = s;
  r.in = static_cast<const uint8_t*>(in_local);
  r.n = n_local;
  r.out = static_cast<uint8_t*>(out_local);
  r.cap = out_capacity;
  r.key_bytes = key_bytes;
  r.km = dist_key_mask(key_bytes);
  ley_status st = rank_alloc(r);
  if (st) return st;
  Plan P;
  P.G = G;
  const Options opts = options_snapshot();
  Profiler prof;  // per-phase device times when the "profile" option is on (ley_stage_times)
  prof.on = opts.profile != 0;
  prof.stream = s;
  prof.ctx = &ctx;
  // C1: allgather n_local, allreduce hist16
  uint64_t* d_tmp = reinterpret_cast<uint64_t*>(r.d_status);  // status area reused as collective scratch
  {
    uint64_t* d_nl = d_tmp;
    LEY_CUDA("dist", cudaMemcpyAsync(d_nl + G, &n_local, 8, cudaMemcpyHostToDevice, s));
    LEY_COLL(comm, s, "dist allgather n", ncclAllGather(d_nl + G, d_nl, 1, ncclUint64, comm->nccl, s));
    P.n_local.resize(G);
    LEY_CSYNC(comm, s, "dist");  // (a D2H into pageable memory would block in the copy)
    LEY_CUDA("dist", cudaMemcpyAsync(P.n_local.data(), d_nl, 8 * G, cudaMemcpyDeviceToHost, s));
    LEY_CSYNC(comm, s, "dist");
  }
  P.N = 0;
  r.gbase = 0;
  for (int i = 0; i < G; ++i) {
    if (i < r.rank) r.gbase += P.n_local[i];
    P.N += P.n_local[i];
  }
  if (P.N > LEY_MAX_RECORDS) {
    set_error("dist: total records > 2^32-2");
    return LEY_ERR_TOO_LARGE;
  }
  const bool exchange = G > 1 || opts.dist_exchange_g1;
  if (!exchange) {  // one rank owns every key: no histogram, splitters or exchange, just the local sort
    r.n_out = n_local;
    r.out_off = 0;
    if (r.n_out > r.cap) {
      set_error("dist: out_capacity_records is smaller than n_local");
      return LEY_ERR_CAPACITY;
    }
    if ((st = prof.begin("D5 local sort")) || (st = phase6_local_sort(r, r.in)) || (st = prof.end())) return st;
    LEY_CSYNC(comm, s, "dist");
    *n_out_local = r.n_out;
    *out_global_offset = 0;
    prof.launches = r.launches;
    prof.finish();
    return LEY_OK;
  }
  if ((st = prof.begin("D1 hist16+allreduce"))) return st;
  if ((st = phase1_hist(r)) || (st = host_hist_async(r))) return st;
  // global histogram (u32 sums: N < 2^32), in place once the local copy is queued; one host sync for both
  LEY_COLL(comm, s, "dist allreduce hist16", ncclAllReduce(r.d_hist, r.d_hist, 65536, ncclUint32, ncclSum, comm->nccl, s));
  LEY_CUDA("dist", cudaMemcpyAsync(r.h_hist + 65536, r.d_hist, 4 * 65536, cudaMemcpyDeviceToHost, s));
  LEY_CSYNC(comm, s, "dist");
  host_hist_take(r);
  P.ghist.assign(r.h_hist + 65536, r.h_hist + 2 * 65536);
  if ((st = prof.end()) || (st = prof.begin("D2 splitters"))) return st;
  if (P.N && dist_plan_splitters(P.ghist.data(), P.N, G, P.bins, P.rho, P.first)) {
    set_error("dist: splitter planning failed");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  // P2 + C2: candidates
  if (G > 1 && P.N) {
    if ((st = phase2_candidates(r, P))) return st;
    std::vector<uint64_t> counts(G);
    {
      uint64_t* d_c = d_tmp;
      uint64_t mine = r.ncand;
      LEY_CUDA("dist", cudaMemcpyAsync(d_c + G, &mine, 8, cudaMemcpyHostToDevice, s));
      LEY_COLL(comm, s, "dist allgather cand", ncclAllGather(d_c + G, d_c, 1, ncclUint64, comm->nccl, s));
      LEY_CSYNC(comm, s, "dist");  // (a D2H into pageable memory would block in the copy)
      LEY_CUDA("dist", cudaMemcpyAsync(counts.data(), d_c, 8 * G, cudaMemcpyDeviceToHost, s));
      LEY_CSYNC(comm, s, "dist");
    }
    uint64_t maxc = 0, total = 0;
    for (int i = 0; i < G; ++i) {
      maxc = std::max(maxc, counts[i]);
      total += counts[i];
    }
    // padded allgather of candidate records and ordinals, then compaction into rank order
    const size_t rec_b = a256(maxc * kRecordBytes), gid_b = a256(4 * maxc);
    const size_t bytes = (size_t)G * (rec_b + gid_b) + rec_b + gid_b + a256(total * kRecordBytes) + a256(4 * total);
    if ((st = ensure_buffer(r.cand_buf, std::max<size_t>(bytes, 256), "dist cand", s))) return st;
    uint8_t* base = static_cast<uint8_t*>(r.cand_buf.ptr);
    uint8_t* all_rec = base;                                   // G x rec_b
    uint8_t* all_gid = all_rec + (size_t)G * rec_b;            // G x gid_b
    uint8_t* my_rec = all_gid + (size_t)G * gid_b;
    uint8_t* my_gid = my_rec + rec_b;
    uint8_t* cat_rec = my_gid + gid_b;
    uint32_t* cat_gid = reinterpret_cast<uint32_t*>(cat_rec + a256(total * kRecordBytes));
    if (r.ncand) {
      LEY_CUDA("dist cand", cudaMemcpyAsync(my_rec, r.d_cand, r.ncand * kRecordBytes, cudaMemcpyDeviceToDevice, s));
      LEY_CUDA("dist cand", cudaMemcpyAsync(my_gid, r.d_cand_gidx, 4ull * r.ncand, cudaMemcpyDeviceToDevice, s));
    }
    LEY_COLL(comm, s, "dist allgather cand", ncclAllGather(my_rec, all_rec, rec_b, ncclUint8, comm->nccl, s));
    LEY_COLL(comm, s, "dist allgather cand", ncclAllGather(my_gid, all_gid, gid_b, ncclUint8, comm->nccl, s));
    uint64_t at = 0;
    for (int i = 0; i < G; ++i) {
      if (counts[i]) {
        LEY_CUDA("dist cand", cudaMemcpyAsync(cat_rec + at * kRecordBytes, all_rec + (size_t)i * rec_b,
                                              counts[i] * kRecordBytes, cudaMemcpyDeviceToDevice, s));
        LEY_CUDA("dist cand", cudaMemcpyAsync(cat_gid + at, all_gid + (size_t)i * gid_b, 4 * counts[i],
                                              cudaMemcpyDeviceToDevice, s));
      }
      at += counts[i];
    }
    LEY_CSYNC(comm, s, "dist allgather cand");  // the candidate sort below waits on the host
    if ((st = phase3_splitters(ctx, s, cat_rec, cat_gid, total, P, r.split_buf, key_bytes))) return st;
    LEY_CSYNC(comm, s, "dist cand");
  }
  // P4 + C3: send counts
  if ((st = prof.end()) || (st = prof.begin("D3 send counts"))) return st;
  if ((st = phase4_counts_device(r, P))) return st;
  P.send_matrix.assign((size_t)G * G, 0);
  {  // the counts stay on the device: all-gathered from d_dcount, one host sync for the matrix
    uint64_t* d_m = d_tmp;
    LEY_COLL(comm, s, "dist allgather counts", ncclAllGather(r.d_dcount, d_m, G, ncclUint64, comm->nccl, s));
    LEY_CSYNC(comm, s, "dist");  // (a D2H into pageable memory would block in the copy)
    LEY_CUDA("dist", cudaMemcpyAsync(P.send_matrix.data(), d_m, 8ull * G * G, cudaMemcpyDeviceToHost, s));
    LEY_CSYNC(comm, s, "dist");
    for (int d = 0; d < G; ++d) r.send_counts[d] = P.send_matrix[(size_t)r.rank * G + d];
  }
  // P5 + C4: partition and exchange
  if ((st = prof.end()) || (st = prof.begin("D4 partition"))) return st;
  if ((st = phase5_plan(r, P))) return st;
  const uint8_t* recv = nullptr;
  bool fused = opts.dist_fused && comm->fused_ok != 0;
  if (fused) {
    uint64_t most = 0;
    for (int d = 0; d < G; ++d) {
      uint64_t in_d = 0;
      for (int src = 0; src < G; ++src) in_d += P.send_matrix[(size_t)src * G + d];
      most = std::max(most, in_d);
    }
    // every rank computes the same size from the replicated matrix, so all ranks (re)register together
    // and all reach the same fused_ok
    if ((st = window_ensure(comm, std::max<size_t>(most * kRecordBytes, 4096), s))) return st;
    fused = comm->fused_ok == 1;
  }
  if (fused) {
    // fused: K-p stores each destination run straight into its owner's symmetric
    // window over NVLink; one tiny all-reduce afterwards orders every rank's stores before any local sort
    uint64_t dst_off[kMaxRanks];
    dist_dest_offsets(P.send_matrix.data(), G, r.rank, dst_off);
    if (r.n && (st = phase5_partition(r, P, nullptr, comm->d_peers, dst_off, G > 1))) return st;
    if ((st = prof.end()) || (st = prof.begin("D4b exchange"))) return st;
    LEY_COLL(comm, s, "dist exchange", ncclAllReduce(d_tmp, d_tmp, 1, ncclUint64, ncclSum, comm->nccl, s));
    LEY_CSYNC(comm, s, "dist exchange");  // the local sort below waits on the host
    recv = static_cast<const uint8_t*>(comm->win_buf);
  } else {
    if ((st = phase5_partition_send(r, P))) return st;
    if ((st = prof.end()) || (st = prof.begin("D4b exchange"))) return st;
    if ((st = ensure_buffer(r.recv_buf, std::max<size_t>(r.n_out * kRecordBytes, 256), "dist exchange", s))) return st;
    DeviceBuffer& rb = r.recv_buf;
    const uint8_t* send = static_cast<const uint8_t*>(r.send_buf.ptr);
    LEY_NCCLC(comm, s, "dist exchange", ncclGroupStart());
    for (int peer = 0; peer < G; ++peer) {
      const uint64_t sc = P.send_matrix[(size_t)r.rank * G + peer];
      if (sc)
        LEY_NCCLC(comm, s, "dist exchange", ncclSend(send + r.send_off[peer] * kRecordBytes, sc * kRecordBytes, ncclUint8,
                                           peer, comm->nccl, s));
      if (r.recv_counts[peer])
        LEY_NCCLC(comm, s, "dist exchange", ncclRecv(static_cast<uint8_t*>(rb.ptr) + r.recv_off[peer] * kRecordBytes,
                                           r.recv_counts[peer] * kRecordBytes, ncclUint8, peer, comm->nccl, s));
    }
    LEY_COLL(comm, s, "dist exchange", ncclGroupEnd());
    LEY_CSYNC(comm, s, "dist exchange");
    recv = static_cast<uint8_t*>(rb.ptr);
  }
  // P6: local sort of the received range
  if ((st = prof.end()) || (st = prof.begin("D5 local sort"))) return st;
  if ((st = phase6_local_sort(r, recv))) return st;
  if ((st = prof.end())) return st;
  LEY_CSYNC(comm, s, "dist");
  *n_out_local = r.n_out;
  *out_global_offset = r.out_off;
  prof.launches = r.launches + P.launches;
  prof.finish();
  return LEY_OK;
}

}  // namespace

// ------------------------------------------------------------------------- multi-GPU external path
// Host run scratch every rank can read: POSIX shared memory (rank 0 creates it, every rank maps it and
// registers it with CUDA as mapped pinned memory); with one rank the library's own pinned scratch.
struct SharedScratch {
  void* p = nullptr;
  size_t bytes = 0;
  bool registered = false;
};

void shared_scratch_close(SharedScratch& sh) {
  if (sh.registered) cudaHostUnregister(sh.p);
  if (sh.p) munmap(sh.p, sh.bytes);
  sh = SharedScratch{};
}

// 0 on success; else an error message (the caller turns every rank's outcome into one agreement)
std::string shared_scratch_open(const std::string& name, size_t bytes, bool create, SharedScratch& sh,
                                bool cuda_register = true) {
  if (create) {
    struct statvfs v{};
    if (statvfs("/dev/shm", &v) == 0 && (uint64_t)v.f_bavail * v.f_frsize < bytes)
      return "dist external: /dev/shm has " + std::to_string((uint64_t)v.f_bavail * v.f_frsize) +
             " bytes free, the shared run scratch needs " + std::to_string(bytes);
    shm_unlink(name.c_str());  // a stale segment of a crashed run
  }
  const int fd = shm_open(name.c_str(), create ? (O_CREAT | O_RDWR | O_EXCL) : O_RDWR, 0600);
  if (fd < 0) return "dist external: shm_open(" + name + ") failed: " + strerror(errno);
  if (create && ftruncate(fd, (off_t)bytes) != 0) {
    const std::string e = strerror(errno);
    close(fd);
    return "dist external: ftruncate of the shared run scratch failed: " + e;
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return std::string("dist external: mmap failed: ") + strerror(errno);
  sh.p = p;
  sh.bytes = bytes;
  if (!cuda_register) return "";
  if (cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
    cudaGetLastError();
    return "dist external: cudaHostRegister of the shared run scratch failed";
  }
  sh.registered = true;
  return "";
}

// SURVEY §8e "External at 8 GPUs": runs of every rank's pinned host slice into the shared scratch (global
// layout), samples broadcast to every rank, identical splitters and slice bounds everywhere, and rank r
// merging global sorted positions [floor(r N/G), floor((r+1) N/G)) into its out_local (external.cu).
ley_status dist_sort_external(ley_comm* comm, const uint8_t* in, uint64_t n_local, uint8_t* out, uint64_t cap,
                              uint64_t* n_out_local, uint64_t* out_global_offset, uint64_t budget, uint32_t key_bytes,
                              cudaStream_t s) {
  const int G = comm->nranks, rank = comm->rank;
  if (key_bytes > kKeyBytes) {
    set_error("dist external: keys longer than 10 bytes are not supported on the external path");
    return LEY_ERR_UNSUPPORTED;
  }
  DeviceContext& ctx = device_context(comm->device);
  std::lock_guard<std::mutex> guard(ctx.mu);
  if (ley_status ast = async_drain(ctx)) return ast;
  if (!ctx.host_pinned) LEY_CUDA("dist", cudaHostAlloc(&ctx.host_pinned, 4096, cudaHostAllocMapped));
  // slice sizes -> the plan every rank derives alike
  std::vector<uint64_t> nl(G);
  {
    uint64_t* d = reinterpret_cast<uint64_t*>(comm->state.d_status);
    LEY_CUDA("dist external", cudaMemcpyAsync(d + G, &n_local, 8, cudaMemcpyHostToDevice, s));
    LEY_COLL(comm, s, "dist external", ncclAllGather(d + G, d, 1, ncclUint64, comm->nccl, s));
    LEY_CSYNC(comm, s, "dist external");  // (a D2H into pageable memory would block in the copy)
    LEY_CUDA("dist external", cudaMemcpyAsync(nl.data(), d, 8 * G, cudaMemcpyDeviceToHost, s));
    LEY_CSYNC(comm, s, "dist external");
  }
  const ExtDistPlan P = ext_dist_plan(nl, budget);
  if (P.N > LEY_MAX_RECORDS) {
    set_error("dist external: total records > 2^32-2");
    return LEY_ERR_TOO_LARGE;
  }
  const bool dev_ok = !budget || ext_dist_device_bytes(P) <= budget;
  // shared host run scratch
  const size_t bytes = std::max<size_t>((size_t)P.N * kRecordBytes, 4096);
  SharedScratch sh;
  std::string err;
  const std::string name = "/ley-" + std::to_string(comm->uid_hash) + "-" + std::to_string(comm->ext_calls++);
  uint8_t* h_runs = nullptr;
  if (G == 1) {
    if (ley_status hs = ensure_host_scratch(ctx, bytes)) return hs;
    h_runs = static_cast<uint8_t*>(ctx.host_scratch);
  } else if (rank == 0) {
    err = shared_scratch_open(name, bytes, true, sh);
  }
  uint64_t any = 0;
  ley_status st = agree(comm, err.empty() && dev_ok, s, &any);
  if (!st && !any && G > 1 && rank != 0) err = shared_scratch_open(name, bytes, false, sh);
  if (!st && !any && G > 1) st = agree(comm, err.empty(), s, &any);
  if (G > 1 && rank == 0 && !st) shm_unlink(name.c_str());  // every rank has it mapped (or gave up)
  auto fail = [&](ley_status code) {
    shared_scratch_close(sh);
    return code;
  };
  if (st) return fail(st);
  if (any) {
    set_error(!err.empty() ? err : !dev_ok ? "dist external: device_budget_bytes below the external working set ("
                                                 + std::to_string(ext_dist_device_bytes(P)) + " bytes)"
                                           : "dist external: another rank could not set up the shared run scratch");
    return fail(dev_ok ? LEY_ERR_UNSUPPORTED : LEY_ERR_BUDGET);
  }
  if (G > 1) h_runs = static_cast<uint8_t*>(sh.p);
  Profiler quiet;
  quiet.ctx = &ctx;
  quiet.stream = s;
  // a10: this rank's runs; then every rank's runs must be in the scratch before anyone reads them
  // (agreed: a rank whose run generation failed must not leave the others in the broadcasts below)
  ley_status rst = ext_dist_runs(ctx, P, rank, in, h_runs, key_bytes, s, quiet);
  if (!rst) rst = comm_sync(comm, s, "dist external runs");
  if (comm->aborted) return fail(rst);
  if ((st = agree(comm, rst == LEY_OK, s, &any))) return fail(st);
  if (rst) return fail(rst);
  if (any) {
    set_error("dist external: another rank failed its run generation");
    return fail(LEY_ERR_NCCL);
  }
  // samples: rank r's block of the run-ordered sample set broadcast from rank r (the all-reduce inside
  // the group also orders every rank's run D2H before the partition phase reads the scratch)
  uint8_t* samp = ext_dist_samples(ctx, P);
  LEY_NCCLC(comm, s, "dist external", ncclGroupStart());
  for (int r = 0; r < G; ++r) {
    const uint64_t c = (P.samp_off[r + 1] - P.samp_off[r]) * kRecordBytes;
    if (c) {
      uint8_t* blk = samp + P.samp_off[r] * kRecordBytes;
      LEY_COLL(comm, s, "dist external", ncclBroadcast(blk, blk, c, ncclUint8, r, comm->nccl, s));
    }
  }
  LEY_COLL(comm, s, "dist external", ncclGroupEnd());
  if ((st = agree(comm, true, s, &any))) return fail(st);
  // a11 (identical on every rank) and a12 (this rank's range); every rank checks its capacity first
  const uint64_t lo = (uint64_t)((unsigned __int128)rank * P.N / (unsigned)G);
  const uint64_t hi = (uint64_t)((unsigned __int128)(rank + 1) * P.N / (unsigned)G);
  if ((st = agree(comm, hi - lo <= cap, s, &any))) return fail(st);
  if (any) {
    set_error("dist external: out_capacity_records below the rank's share floor((r+1) N/G) - floor(r N/G) on some rank");
    return fail(LEY_ERR_CAPACITY);
  }
  ExtDistParts parts;
  if ((st = ext_dist_partition(ctx, P, h_runs, key_bytes, s, quiet, parts))) return fail(st);
  if ((st = ext_dist_merge(ctx, P, parts, rank, h_runs, out, cap, n_out_local, out_global_offset, key_bytes, s, quiet)))
    return fail(st);
  LEY_CSYNC(comm, s, "dist external");
  // nobody may unmap a scratch another rank still reads: one last agreement
  if ((st = agree(comm, true, s, &any))) return fail(st);
  record_launches(quiet.launches);
  shared_scratch_close(sh);
  return LEY_OK;
}

// Pointer kinds: both device pointers (the NCCL path proper), or both pinned host pointers — staged: this
// rank's slice is copied into a comm-owned device buffer, sorted by the device path, and its output range
// copied back. Every rank first agrees (one all-reduce) that its staging fits its budget, so a rank that
// cannot proceed never leaves the others waiting in a collective.
ley_status dist_sort(ley_comm* comm, const void* in_local, uint64_t n_local, void* out_local, uint64_t out_capacity,
                     uint64_t* n_out_local, uint64_t* out_global_offset, uint64_t budget, uint32_t key_bytes,
                     cudaStream_t s) {
  if (comm->aborted) {
    set_error("dist: the communicator was aborted by an earlier failure (destroy it and create a new one)");
    return LEY_ERR_NCCL;
  }
  comm->colls = 0;
  LEY_CUDA("dist", cudaSetDevice(comm->device));
  int kind = -1;  // 0 device, 1 pinned host
  const void* ptrs[2] = {n_local ? in_local : nullptr, out_capacity ? out_local : nullptr};
  for (const void* p : ptrs) {
    if (!p) continue;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      set_error("dist: cudaPointerGetAttributes failed");
      return LEY_ERR_CUDA;
    }
    int k = a.type == cudaMemoryTypeDevice && a.device == comm->device ? 0 : (a.type == cudaMemoryTypeHost ? 1 : 2);
    if (k == 2 || (kind >= 0 && k != kind)) {
      set_error("dist: in_local/out_local must both be device memory on the comm's device or both pinned host memory");
      return LEY_ERR_UNSUPPORTED;
    }
    kind = k;
  }
  if (kind != 1)
    return dist_sort_device(comm, in_local, n_local, out_local, out_capacity, n_out_local, out_global_offset,
                            key_bytes, s);
  const size_t a_in = a256(n_local * kRecordBytes), a_out = a256(out_capacity * kRecordBytes);
  const bool fits = !budget || a_in + a_out <= budget;
  bool external = false;
  ley_status st_ = LEY_OK;
  {
    DeviceContext& ctx = device_context(comm->device);
    std::lock_guard<std::mutex> guard(ctx.mu);
    if (ley_status ast = async_drain(ctx)) return ast;
    uint64_t* flag = reinterpret_cast<uint64_t*>(comm->state.d_status);
    if (!flag) {  // first call on this comm: scratch for the agreement
      if (ley_status st = rank_alloc(comm->state)) return st;
      flag = reinterpret_cast<uint64_t*>(comm->state.d_status);
    }
    const uint64_t bad = fits ? 0 : 1;
    LEY_CUDA("dist staging", cudaMemcpyAsync(flag, &bad, 8, cudaMemcpyHostToDevice, s));
    LEY_COLL(comm, s, "dist staging", ncclAllReduce(flag, flag, 1, ncclUint64, ncclSum, comm->nccl, s));
    uint64_t any = 0;
    LEY_CSYNC(comm, s, "dist staging");  // (a D2H into pageable memory would block in the copy)
    LEY_CUDA("dist staging", cudaMemcpyAsync(&any, flag, 8, cudaMemcpyDeviceToHost, s));
    LEY_CSYNC(comm, s, "dist staging");
    if (!any && (st_ = ensure_buffer(comm->stage, std::max<size_t>(a_in + a_out, 256), "dist staging", s))) return st_;
    if (any) external = true;
  }
  if (external)
    return dist_sort_external(comm, static_cast<const uint8_t*>(in_local), n_local, static_cast<uint8_t*>(out_local),
                              out_capacity, n_out_local, out_global_offset, budget, key_bytes, s);
  uint8_t* din = static_cast<uint8_t*>(comm->stage.ptr);
  uint8_t* dout = din + a_in;
  if (n_local)
    LEY_CUDA("dist H2D", cudaMemcpyAsync(din, in_local, n_local * kRecordBytes, cudaMemcpyHostToDevice, s));
  ley_status st = dist_sort_device(comm, din, n_local, dout, out_capacity, n_out_local, out_global_offset, key_bytes, s);
  if (st) return st;
  if (*n_out_local)
    LEY_CUDA("dist D2H", cudaMemcpyAsync(out_local, dout, *n_out_local * kRecordBytes, cudaMemcpyDeviceToHost, s));
  LEY_CSYNC(comm, s, "dist D2H");
  return LEY_OK;
}

// ------------------------------------------------------------------------------ loopback transport
// All G ranks on the current device in one process; collectives are host-side reductions and device
// copies. Exercises exactly the kernels and plans of dist_sort (test hook).
// Loopback of the multi-GPU external path: the G ranks' phases run one after another on this device
// (run generation of every rank, one partition, each rank's merge); the library's pinned scratch stands in
// for the shared memory segment.
ley_status dist_external_loopback(int G, const void* const* in, const uint64_t* n_local, void* const* out,
                                  const uint64_t* caps, uint64_t* n_out, uint64_t* out_off, uint64_t budget,
                                  uint32_t key_bytes, cudaStream_t s) {
  if (key_bytes > kKeyBytes) {
    set_error("dist external: keys longer than 10 bytes are not supported on the external path");
    return LEY_ERR_UNSUPPORTED;
  }
  int dev = 0;
  LEY_CUDA("loopback", cudaGetDevice(&dev));
  DeviceContext& ctx = device_context(dev);
  std::lock_guard<std::mutex> guard(ctx.mu);
  if (ley_status ast = async_drain(ctx)) return ast;
  if (!ctx.host_pinned) LEY_CUDA("loopback", cudaHostAlloc(&ctx.host_pinned, 4096, cudaHostAllocMapped));
  const ExtDistPlan P = ext_dist_plan(std::vector<uint64_t>(n_local, n_local + G), budget);
  if (budget && ext_dist_device_bytes(P) > budget) {
    set_error("dist external: device_budget_bytes below the external working set");
    return LEY_ERR_BUDGET;
  }
  const size_t bytes = std::max<size_t>((size_t)P.N * kRecordBytes, 4096);
  ley_status st = ensure_host_scratch(ctx, bytes);
  if (st) return st;
  uint8_t* h_runs = static_cast<uint8_t*>(ctx.host_scratch);
  Profiler quiet;
  quiet.ctx = &ctx;
  quiet.stream = s;
  for (int r = 0; r < G; ++r)
    if ((st = ext_dist_runs(ctx, P, r, static_cast<const uint8_t*>(in[r]), h_runs, key_bytes, s, quiet))) return st;
  LEY_CUDA("loopback", cudaStreamSynchronize(s));
  ExtDistParts parts;
  if ((st = ext_dist_partition(ctx, P, h_runs, key_bytes, s, quiet, parts))) return st;
  for (int r = 0; r < G; ++r)
    if ((st = ext_dist_merge(ctx, P, parts, r, h_runs, static_cast<uint8_t*>(out[r]), caps[r], &n_out[r], &out_off[r],
                             key_bytes, s, quiet)))
      return st;
  LEY_CUDA("loopback", cudaStreamSynchronize(s));
  record_launches(quiet.launches);
  return LEY_OK;
}

ley_status dist_sort_loopback(int G, const void* const* in, const uint64_t* n_local, void* const* out,
                              const uint64_t* caps, uint64_t* n_out, uint64_t* out_off, uint64_t budget,
                              uint32_t key_bytes, cudaStream_t s) {
  if (G < 1 || G > kMaxRanks) {
    set_error("loopback: 1 <= G <= 8");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  {  // pinned host slices: the multi-GPU external path
    cudaPointerAttributes a{};
    const void* probe = nullptr;
    for (int i = 0; i < G && !probe; ++i)
      if (n_local[i]) probe = in[i];
    if (probe && cudaPointerGetAttributes(&a, probe) == cudaSuccess && a.type == cudaMemoryTypeHost)
      return dist_external_loopback(G, in, n_local, out, caps, n_out, out_off, budget, key_bytes, s);
    cudaGetLastError();
  }
  int dev = 0;
  LEY_CUDA("loopback", cudaGetDevice(&dev));
  DeviceContext& ctx = device_context(dev);
  std::lock_guard<std::mutex> guard(ctx.mu);
  if (ley_status ast = async_drain(ctx)) return ast;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms > 0) ctx.sms = sms;
  if (!ctx.host_pinned) LEY_CUDA("loopback", cudaHostAlloc(&ctx.host_pinned, 4096, cudaHostAllocMapped));
  std::vector<std::unique_ptr<RankState>> R(G);
  Plan P;
  P.G = G;
  P.n_local.assign(n_local, n_local + G);
  ley_status st;
  for (int i = 0; i < G; ++i) {
    R[i].reset(new RankState());
    RankState& r = *R[i];
    r.rank = i;
    r.ctx = &ctx;
    r.s = s;
    r.in = static_cast<const uint8_t*>(in[i]);
    r.n = n_local[i];
    r.out = static_cast<uint8_t*>(out[i]);
    r.cap = caps[i];
    r.key_bytes = key_bytes;
    r.km = dist_key_mask(key_bytes);
    r.gbase = P.N;
    P.N += n_local[i];
    if ((st = rank_alloc(r))) return st;
  }
  if (P.N > LEY_MAX_RECORDS) {
    set_error("loopback: total records > 2^32-2");
    return LEY_ERR_TOO_LARGE;
  }
  // P1 + C1
  P.ghist.assign(65536, 0);
  for (int i = 0; i < G; ++i) {
    if ((st = phase1_hist(*R[i])) || (st = host_hist_async(*R[i]))) return st;
    LEY_CUDA("loopback", cudaStreamSynchronize(s));
    host_hist_take(*R[i]);
    for (int b = 0; b < 65536; ++b) P.ghist[b] += R[i]->hist[b];
  }
  if (P.N && dist_plan_splitters(P.ghist.data(), P.N, G, P.bins, P.rho, P.first)) {
    set_error("loopback: splitter planning failed");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  // P2 + C2 + P3
  if (G > 1 && P.N) {
    uint64_t total = 0;
    for (int i = 0; i < G; ++i) {
      if ((st = phase2_candidates(*R[i], P))) return st;
      total += R[i]->ncand;
    }
    DeviceBuffer cb;
    LEY_CUDA("loopback", cudaMalloc(&cb.ptr, a256(total * kRecordBytes) + a256(4 * total) + 256));
    std::unique_ptr<void, decltype(&cudaFree)> g(cb.ptr, &cudaFree);
    uint8_t* cat = static_cast<uint8_t*>(cb.ptr);
    uint32_t* gid = reinterpret_cast<uint32_t*>(cat + a256(total * kRecordBytes));
    uint64_t at = 0;
    for (int i = 0; i < G; ++i) {
      const uint64_t c = R[i]->ncand;
      if (c) {
        LEY_CUDA("loopback", cudaMemcpyAsync(cat + at * kRecordBytes, R[i]->d_cand, c * kRecordBytes,
                                             cudaMemcpyDeviceToDevice, s));
        LEY_CUDA("loopback", cudaMemcpyAsync(gid + at, R[i]->d_cand_gidx, 4 * c, cudaMemcpyDeviceToDevice, s));
      }
      at += c;
    }
    if ((st = phase3_splitters(ctx, s, cat, gid, total, P, R[0]->split_buf, key_bytes))) return st;
  }
  // P4 + C3
  P.send_matrix.assign((size_t)G * G, 0);
  for (int i = 0; i < G; ++i) {
    if ((st = phase4_counts(*R[i], P))) return st;
    for (int d = 0; d < G; ++d) P.send_matrix[(size_t)i * G + d] = R[i]->send_counts[d];
  }
  // P5 + C4: every rank's receive buffer exists before any K-p runs; fused: K-p of rank i writes its
  // runs straight into the receivers' buffers (the kernels never wait on one another); else K-p into a
  // send buffer and device copies stand in for the all-to-all-v
  const Options opts = options_snapshot();
  std::vector<std::unique_ptr<void, decltype(&cudaFree)>> recvs;
  std::vector<uint8_t*> rbuf(G);
  for (int i = 0; i < G; ++i) {
    if ((st = phase5_plan(*R[i], P))) return st;
    void* p = nullptr;
    LEY_CUDA("loopback exchange", cudaMalloc(&p, std::max<size_t>(R[i]->n_out * kRecordBytes, 256)));
    recvs.emplace_back(p, &cudaFree);
    rbuf[i] = static_cast<uint8_t*>(p);
  }
  for (int i = 0; i < G; ++i) {
    RankState& r = *R[i];
    if (!r.n) continue;
    if (opts.dist_fused) {
      uint64_t dst_off[kMaxRanks];
      dist_dest_offsets(P.send_matrix.data(), G, i, dst_off);
      // remote = G > 1, exactly as the NCCL path launches it: the per-CTA system-scope fence form runs
      if ((st = phase5_partition(r, P, rbuf.data(), nullptr, dst_off, G > 1))) return st;
    } else {
      if ((st = phase5_partition_send(r, P))) return st;
      for (int d = 0; d < G; ++d) {
        const uint64_t c = P.send_matrix[(size_t)i * G + d];
        if (c)
          LEY_CUDA("loopback exchange",
                   cudaMemcpyAsync(rbuf[d] + R[d]->recv_off[i] * kRecordBytes,
                                   static_cast<uint8_t*>(r.send_buf.ptr) + r.send_off[d] * kRecordBytes,
                                   c * kRecordBytes, cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  for (int i = 0; i < G; ++i) {
    RankState& r = *R[i];
    if ((st = phase6_local_sort(r, rbuf[i]))) return st;
    LEY_CUDA("loopback", cudaStreamSynchronize(s));
    n_out[i] = r.n_out;
    out_off[i] = r.out_off;
  }
  return LEY_OK;
}

// Test hooks of the shared host run scratch (host logic only: no CUDA registration), so two CPU
// processes can check creation, opening, sizing and unlinking (tests/test_dist.py, gloo).
ley_status test_shared_scratch(const char* name, uint64_t bytes, int create, void** ptr) {
  SharedScratch sh;
  const std::string err = shared_scratch_open(name, bytes, create != 0, sh, false);
  if (!err.empty()) {
    set_error(err);
    shared_scratch_close(sh);
    return LEY_ERR_UNSUPPORTED;
  }
  *ptr = sh.p;
  return LEY_OK;
}
void test_shared_scratch_close(void* p, uint64_t bytes, const char* unlink_name) {
  if (p) munmap(p, bytes);
  if (unlink_name) shm_unlink(unlink_name);
}

}  // namespace ley
