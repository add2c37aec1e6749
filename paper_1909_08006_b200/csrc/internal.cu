// internal.cu — the 1-GPU internal sort driver: Algorithm 1 (§3.1, lines 54-90) on the device.
//
//   K-a  tile-local sort by byte 0 + hist16            (ParallelRadixSort, radix 0; P:102 extraction)
//   K-b  scans: tile runs -> global byte-0 positions; hist16 -> level-1 bucket bases
//   K-c  split every byte-0 bucket on byte 1           (the next round of ParallelRadixSort)
//   classify level-1 buckets                           (big -> recurse P:62-63; small -> queue P:65-66)
//   K-d  sort the queued buckets (warp / CTA tiers)    (SingleThreadRadixSort + ComparisonSort)
//   K-e  ... and, in the same kernels, gather each sorted bucket's records (record scatter)
//   loop while big buckets remain: K-c' on byte depth (MSDRadixSort(key, radix+1, k)) + K-d/K-e
//
// All work is on the caller's stream. The only host synchronisations are one 4-byte read of the
// big-bucket count per recursion level (usually exactly one per call) and the final completion wait.
#include <algorithm>
#include <vector>

#include "classify.cuh"
#include "kc_chunk.cuh"
#include "kernels.cuh"
#include "runtime.h"

namespace ley {

namespace {
inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr uint64_t kPdlMaxRecords = 10000000;  // (option pdl = 3: tier overlap below this size)
}  // namespace

namespace {
// One pass of the internal sort (K-a .. K-e) ordered by the key window `key`.
ley_status sort_pass(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint32_t* perm_out, uint64_t n,
                     cudaStream_t s, Profiler& prof, void* work, size_t work_bytes, KeySpec key,
                     uint64_t* digest = nullptr, bool allow_async = false) {
  const InternalLayout L = plan_internal(n);
  ley_status st;
  if (!out && !perm_out) {  // out == nullptr is the perm-only mode (K-d without the fused gather)
    set_error("internal: neither out nor perm requested");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  if (!work) {
    if ((st = ensure_buffer(ctx.work, L.bytes, "workspace", s))) return st;
    work = ctx.work.ptr;
  } else if (work_bytes < L.bytes) {
    set_error("internal: caller workspace too small");
    return LEY_ERR_BUDGET;
  }
  if (!ctx.host_pinned) LEY_CUDA("setup", cudaHostAlloc(&ctx.host_pinned, 4096, cudaHostAllocMapped));
  uint8_t* base = static_cast<uint8_t*>(work);
  uint64_t* At = reinterpret_cast<uint64_t*>(base + L.off_At);
  uint32_t* Ai = reinterpret_cast<uint32_t*>(base + L.off_Ai);
  uint64_t* Bt = reinterpret_cast<uint64_t*>(base + L.off_Bt);
  uint32_t* Bi = reinterpret_cast<uint32_t*>(base + L.off_Bi);
  uint32_t* perm = reinterpret_cast<uint32_t*>(base + L.off_perm);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(base + L.off_cnt);
  uint32_t* off = reinterpret_cast<uint32_t*>(base + L.off_off);
  uint32_t* lo = reinterpret_cast<uint32_t*>(base + L.off_lo);
  uint32_t* hist16 = reinterpret_cast<uint32_t*>(base + L.off_hist16);
  uint32_t* B16 = reinterpret_cast<uint32_t*>(base + L.off_B16);
  uint32_t* cstart = reinterpret_cast<uint32_t*>(base + L.off_cstart);
  uint64_t* scan_status = reinterpret_cast<uint64_t*>(base + L.off_scan_status);
  uint32_t* cursor = reinterpret_cast<uint32_t*>(base + L.off_cursor);
  uint32_t* small = reinterpret_cast<uint32_t*>(base + L.off_small);
  uint32_t* tickets = small;          // [0..15]
  uint32_t* kd_counts = small + 16;   // [kNumKdLists] counts, [kTierTicket + l] claim tickets
  uint32_t* big_count = small + 32;   // [1]; small[33]: classify's CTA-done counter
  volatile uint32_t* host_cnt = static_cast<volatile uint32_t*>(ctx.host_pinned);
  uint32_t* host_cnt_dev = nullptr;  // its device alias: counters are published by a kernel store
  LEY_CUDA("setup", cudaHostGetDevicePointer((void**)&host_cnt_dev, ctx.host_pinned, 0));

  const Options o = options_snapshot();
  Tunables tu;
  tu.warp_tier_max = (uint32_t)o.warp_tier_max;
  tu.smem_tier_max = (uint32_t)o.smem_tier_max;
  tu.kd_digit_bits = (int)o.kd_digit_bits;
  tu.kd_insert_max = (int)o.kd_insert_max;
  tu.kd_ws = (int)o.kd_ws;
  tu.ws_tma = (int)o.ws_gather_tma;
  tu.gather_l2_64 = (int)o.gather_l2_64;
  // PDL of the tier kernels (k_bucket.cu kd_all): overlapping the tiers pays for small sorts, where their
  // launch latency and empty grids are a visible share (C1 0.148 -> 0.141 ms), and costs at large ones (C4
  // +2.3 ms, C2 +0.1 ms: measured, tools/ab_opts.py); option 3 (default) picks by n
  tu.pdl = o.pdl == 3 ? (n < kPdlMaxRecords ? 2 : 0) : (int)o.pdl;
  tu.kd_claim = (int)o.kd_claim;
  const uint32_t tiles = (uint32_t)L.tiles;
  const int sms = ctx.sms;
  int& launches = prof.launches;
  uint64_t tier = std::max<uint64_t>(tu.smem_tier_max, tu.warp_tier_max);
  uint64_t big_cap = std::min<uint64_t>(65536, n / (tier + 1) + 1);
  uint32_t kd_cap = (uint32_t)std::min<uint64_t>(65536, n);  // level-1 buckets: at most min(2^16, n) non-empty
  if ((st = ensure_buffer(ctx.lists, (size_t)kNumKdLists * a256((size_t)kd_cap * sizeof(Seg)), "K-d lists", s)))
    return st;
  if ((st = ensure_buffer(ctx.big[0], big_cap * sizeof(Seg), "big-bucket list", s))) return st;
  ListSet kd;
  auto bind_lists = [&](uint32_t cap) {
    for (int l = 0; l < kNumKdLists; ++l)
      kd.items[l] = reinterpret_cast<Seg*>(static_cast<uint8_t*>(ctx.lists.ptr) + l * a256((size_t)cap * sizeof(Seg)));
    kd.counts = kd_counts;
    kd.cap = cap;
  };
  bind_lists(kd_cap);

  // Level 1 (init .. K-a .. K-b .. K-c .. classify .. K-d+K-e of every tier .. publish of the big-bucket
  // count) is a fixed sequence for a given (buffers, n, options): ~16 launches whose launch overhead
  // dominates small sorts (C1). It is captured once into a CUDA graph and replayed (option "graphs"), on
  // the library's own stream joined to the caller's by events (the caller's stream may be the legacy
  // default stream, which cannot be captured). With stage profiling on it runs directly.
  auto level1 = [&](cudaStream_t s) -> ley_status {
    ley_status st;

    // ---------------------------------------------------------------- zero counters / look-back state
    if ((st = prof.begin("init"))) return st;
    LEY_CUDA("init", launch_zero3(hist16, 4ull * 65536 * L.hist_copies, small, 4 * kSmallWords, scan_status,
                                  8 * 2 * L.scan_status_words, sms, s));
    ++launches;
    if ((st = prof.end())) return st;

    // ---------------------------------------------------------------- K-a
    if ((st = prof.begin("K-a tile sort"))) return st;
    LEY_CUDA("K-a tile sort", launch_ka_tile_sort(in, n, tiles, At, Ai, cnt, lo, hist16, L.hist_copies, (int)o.ka_stream,
                                                  key, s));
    ++launches;
    if ((st = prof.end())) return st;

    // ---------------------------------------------------------------- K-b
    if ((st = prof.begin("K-b scan"))) return st;
    // (the hist16 copies are summed by the scan itself, which writes the sum back over copy 0)
    // (the hist16 blocks also write the split's fill cursors = B16)
    LEY_CUDA("K-b scan", launch_scan_excl2(cnt, off, L.m, scan_status, off + L.m, hist16, B16, 65536,
                                           scan_status + L.scan_status_words, B16 + 65536, L.hist_copies, 65536,
                                           tickets + 0, s, cursor));
    ++launches;
    if ((st = prof.end())) return st;

    // ---------------------------------------------------------------- K-c (byte 1)
    // Fused form (option kc_fuse, off by default: measured slower): the split runs inside the
    // level-1 K-d+K-e kernel of the tier the average 16-bit bucket falls in (kc_chunk.cuh), meant for the idle
    // issue slots of its DRAM-bound record gather; the tier is a guess (n / 65536), any choice gives the same
    // bytes. Not for tiers of small buckets (warp /
    // 128-thread kernels) unless forced (kc_fuse = 2..5: the 2048 / 8192 / 10240 / 16384 tier; tests), nor in
    // perm-only mode.
    int fused_tier = -1;
    if (o.kc_fuse >= 2 && out) {
      fused_tier = kListMed2 + (int)(o.kc_fuse - 2);
    } else if (o.kc_fuse && out) {
      const uint64_t avg = n / 65536;
      const int t = avg <= tu.warp_tier_max ? kListWarp : avg > tu.smem_tier_max ? kNumKdLists
                  : avg <= 512 ? kListMed1 : avg <= 2048 ? kListMed2 : avg <= 8192 ? kListMed3 : avg <= 10240 ? kListMed4
                                                                                                     : kListMed5;
      if (t >= kListMed2 && t < kNumKdLists) fused_tier = t;
    }
    // Co-run form (option kc_corun = K-c CTAs per SM): the split keeps its own persistent kernel, narrowed to
    // leave room on every SM for a warp-specialised 2048-tier CTA, and that tier (the fused form: buckets
    // claimed in ascending order, each sorted once done[] shows its byte-0 bucket split) is PDL-launched
    // beside it, so the issue-bound split overlaps the DRAM-bound gather. Only where the average bucket
    // falls in that tier (whose CTAs fit beside a split CTA; C2), or with kc_fuse = 2 (forced: tests).
    bool corun = false;
    if (o.kc_corun && (!o.kc_fuse || o.kc_fuse == 2) && out && tu.kd_ws) {
      const uint64_t avg = n / 65536;
      if (o.kc_fuse == 2 || (avg > 512 && avg <= 2048 && avg > tu.warp_tier_max && 2048 <= tu.smem_tier_max)) {
        fused_tier = kListMed2;
        corun = true;
        tu.kc_corun = 1;
      }
    }
    // (the plan launch also classifies the level-1 buckets: Alg. 1's queues, classify.cuh)
    ClassifyJob cj{};
    cj.tu = tu;
    cj.kd = kd;
    cj.hist16 = hist16;
    cj.B16 = B16;
    cj.big_out = static_cast<Seg*>(ctx.big[0].ptr);
    cj.big_count = big_count;
    cj.done = small + 33;
    cj.host_mapped = host_cnt_dev;
    const uint32_t* order_used = nullptr;
    if ((st = prof.begin(corun ? "K-c+K-de co-run" : fused_tier >= 0 ? "K-c plan" : "K-c split"))) return st;
    LEY_CUDA("K-c split", launch_kc_split_level1(At, Ai, tiles, off, lo, B16, n, cstart,
                                                 reinterpret_cast<uint4*>(base + L.off_plan_a),
                                                 reinterpret_cast<uint2*>(base + L.off_plan_b),
                                                 reinterpret_cast<uint32_t*>(base + L.off_order), cursor,
                                                 tickets + 2, Bt, Bi, (uint32_t)L.split_chunks_ub, s, cj,
                                                 fused_tier < 0 || corun, &order_used, corun ? small + 64 : nullptr,
                                                 corun ? (int)o.kc_corun : 0));
    launches += fused_tier < 0 || corun ? 2 : 1;  // plan (+ split)
    // (co-run: no stage boundary between the split and the tier kernel, whose launch must follow it directly)
    if (!corun && (st = prof.end())) return st;

    // ---------------------------------------------------------------- classify level 1, K-d
    if (!corun && (st = prof.begin(fused_tier >= 0 ? "K-c+K-de fused" : "K-de sort+gather"))) return st;
    KcArgs kc;
    if (fused_tier >= 0) {
      kc.k1_in = At;
      kc.w_in = Ai;
      kc.tiles = tiles;
      kc.off = off;
      kc.lo = lo;
      kc.cstart = cstart;
      kc.plan_a = reinterpret_cast<const uint4*>(base + L.off_plan_a);
      kc.plan_b = reinterpret_cast<const uint2*>(base + L.off_plan_b);
      kc.order = order_used;
      kc.cursor = cursor;
      kc.ticket = tickets + 2;
      kc.done = small + 64;
      kc.kd_ticket = small + 320;
      kc.tail_out = Bt;
      kc.idx_out = Bi;
      kc.hist16 = hist16;
      kc.B16 = B16;
    }
    LEY_CUDA("K-de sort+gather", launch_kd_all(kd, At, Ai, Bt, Bi, perm_out ? perm : nullptr, tu, sms, in, n, out, digest, s,
                                               &launches, fused_tier >= 0 ? &kc : nullptr, fused_tier));
    return LEY_OK;
  };
  auto copy_perm = [&]() -> ley_status {  // the workspace permutation to the caller's (stream-ordered)
    if (perm_out) {
      cudaPointerAttributes pa{};
      LEY_CUDA("perm", cudaPointerGetAttributes(&pa, perm_out));
      cudaMemcpyKind kind = pa.type == cudaMemoryTypeDevice ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
      LEY_CUDA("perm", cudaMemcpyAsync(perm_out, perm, 4 * n, kind, s));
    }
    return LEY_OK;
  };
  // Stream-ordered mode (option async, device pointers, keys <= 10 bytes): the host waits only for the
  // classification's big-bucket count, published from the SM into mapped memory over a sentinel it wrote
  // before the launch; with no big buckets it returns while the tier kernels still run.
  constexpr uint32_t kPending = 0xFFFFFFFFu;
  const bool async_ok = allow_async && !prof.on;
  if (async_ok) host_cnt[0] = kPending;
  // (not while profiling: elapsed times between event-record nodes of a graph are refused, measured)
  const bool graphs = o.graphs && !prof.on && !getenv("LEY_DEBUG_SYNC");
  if (!graphs) {
    if ((st = level1(s))) return st;
  } else {
    const GraphKey gk{{(uint64_t)in, (uint64_t)out, (uint64_t)perm_out, (uint64_t)digest, (uint64_t)work,
                       (uint64_t)ctx.lists.ptr, (uint64_t)ctx.big[0].ptr, (uint64_t)ctx.host_pinned, n,
                       ((uint64_t)key.off << 32) | key.len, options_fingerprint(o), (uint64_t)ctx.sms}};
    if ((st = graph_run(ctx, gk, s, [&](cudaStream_t cs) { return level1(cs); }, prof))) return st;
  }
  uint32_t nbig;
  if (async_ok) {
    for (uint32_t spin = 1; (nbig = host_cnt[0]) == kPending; ++spin) {
      if (spin % 1024) continue;
      const cudaError_t q = cudaStreamQuery(s);  // (a failed launch never publishes)
      if (q == cudaSuccess && (nbig = host_cnt[0]) == kPending) {
        set_error("internal: level 1 completed without publishing its big-bucket count");
        return LEY_ERR_CUDA;
      }
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) LEY_CUDA("K-de sort+gather", q);
    }
    if (!nbig) {  // done once the stream gets there
      if ((st = copy_perm())) return st;
      if (!ctx.async_ev) LEY_CUDA("async", cudaEventCreateWithFlags(&ctx.async_ev, cudaEventDisableTiming));
      LEY_CUDA("async", cudaEventRecord(ctx.async_ev, s));
      ctx.async_pending = true;
      ctx.async_stream = s;
      return LEY_OK;
    }
  }
  LEY_CUDA("K-de sort+gather", cudaStreamSynchronize(s));
  nbig = host_cnt[0];
  if ((st = prof.end())) return st;

  // ---------------------------------------------------------------- recursion on big buckets
  int cur = 0;
  while (nbig) {
    const uint64_t chunks_ub = n / kChunk + nbig + 1;
    const uint64_t child_cap = std::min<uint64_t>((uint64_t)nbig * kRadix, n + 1);
    const uint64_t next_big_cap = std::min<uint64_t>(child_cap, n / (tier + 1) + 1);
    const size_t scan_words = scan_status_words(nbig);
    // rec layout: nch | cstart2 | seg_hist | seg_excl (= fill cursors) | noscatter | scan status | tickets
    size_t r_nch = 0, r_cst = a256(4ull * (nbig + 1)), r_hist = r_cst + a256(4ull * (nbig + 1));
    size_t r_excl = r_hist + a256(4ull * nbig * kRadix), r_nos = r_excl + a256(4ull * nbig * kRadix);
    size_t r_scan = r_nos + a256(nbig);
    size_t r_tick = r_scan + a256(8 * scan_words), r_map = r_tick + 256, r_end = r_map + a256(8 * chunks_ub);
    if ((st = ensure_buffer(ctx.rec, r_end, "recursion arrays", s))) return st;
    if (child_cap > kd.cap) {
      if ((st = ensure_buffer(ctx.lists, (size_t)kNumKdLists * a256(child_cap * sizeof(Seg)), "K-d lists", s)))
        return st;
      bind_lists((uint32_t)child_cap);
    }
    if ((st = ensure_buffer(ctx.big[cur ^ 1], std::max<uint64_t>(next_big_cap, 1) * sizeof(Seg), "big-bucket list",
                            s)))
      return st;
    uint8_t* rb = static_cast<uint8_t*>(ctx.rec.ptr);
    uint32_t* nch = reinterpret_cast<uint32_t*>(rb + r_nch);
    uint32_t* cst = reinterpret_cast<uint32_t*>(rb + r_cst);
    uint32_t* seg_hist = reinterpret_cast<uint32_t*>(rb + r_hist);
    uint32_t* seg_excl = reinterpret_cast<uint32_t*>(rb + r_excl);
    uint8_t* noscatter = rb + r_nos;
    uint64_t* rscan = reinterpret_cast<uint64_t*>(rb + r_scan);
    uint32_t* rtick = reinterpret_cast<uint32_t*>(rb + r_tick);
    uint2* cmap = reinterpret_cast<uint2*>(rb + r_map);
    const Seg* segs = static_cast<const Seg*>(ctx.big[cur].ptr);
    Seg* next_big = static_cast<Seg*>(ctx.big[cur ^ 1].ptr);

    if ((st = prof.begin("K-c' split"))) return st;
    LEY_CUDA("K-c' recursion", cudaMemsetAsync(seg_hist, 0, 4ull * nbig * kRadix, s));
    LEY_CUDA("K-c' recursion", cudaMemsetAsync(rscan, 0, 8 * scan_words, s));
    LEY_CUDA("K-c' recursion", cudaMemsetAsync(rtick, 0, 256, s));
    LEY_CUDA("K-c' recursion", cudaMemsetAsync(kd_counts, 0, 4 * 2 * kTierTicket, s));  // counts + tickets
    LEY_CUDA("K-c' recursion", cudaMemsetAsync(big_count, 0, 4, s));
    LEY_CUDA("K-c' recursion", launch_kr_nchunks(segs, nbig, nch, s));
    LEY_CUDA("K-c' recursion", launch_scan_excl(nch, cst, nbig, rscan, rtick + 0, cst + nbig, s));
    uint32_t hist_grid = (uint32_t)std::min<uint64_t>(chunks_ub, (uint64_t)sms * 8);
    LEY_CUDA("K-c' recursion", launch_kr_chunk_map(cst, nbig, (uint32_t)chunks_ub, cmap, s));
    LEY_CUDA("K-c' recursion", launch_kr_hist(segs, nbig, cst, hist_grid, At, Ai, Bt, Bi, seg_hist, cmap, s));
    LEY_CUDA("K-c' recursion",
             launch_kr_plan(segs, nbig, seg_hist, seg_excl, noscatter, tu, kd, next_big, big_count, s));
    LEY_CUDA("K-c' recursion", launch_kr_split(segs, nbig, cst, seg_excl, noscatter, At, Ai, Bt, Bi, rtick + 1, cmap,
                                              (uint32_t)chunks_ub, s));
    launches += 6;
    if ((st = prof.end())) return st;
    if ((st = prof.begin("K-de sort+gather"))) return st;
    LEY_CUDA("K-c' recursion", launch_kd_all(kd, At, Ai, Bt, Bi, perm_out ? perm : nullptr, tu, sms, in, n, out, digest, s, &launches));
    LEY_CUDA("K-c' recursion", launch_publish_u32(big_count, host_cnt_dev, s));
    LEY_CUDA("K-c' recursion", cudaStreamSynchronize(s));
    nbig = host_cnt[0];
    cur ^= 1;
    if ((st = prof.end())) return st;
  }

  return copy_perm();
}

}  // namespace

uint64_t keypass_bytes(uint64_t n, uint32_t key_bytes, bool perm) {
  if (key_bytes <= kKeyBytes) return 0;
  // the other record buffer of the window passes; with perm two permutation arrays, else the tie-group
  // lists of the hybrid form (first/last positions, <= n/2 groups each, the two large-group lists and
  // the counts)
  return a256(n * kRecordBytes) + (perm ? 2 * a256(4 * n) : 2 * a256(4 * (n / 2 + 1)) + 1024);
}

namespace {
// tie groups of <= 1024 records are sorted on the device (k_ties.cu: eight lanes for <= 7 records, a warp
// for <= 32, one CTA for <= 128 / <= 1024); only longer ones get window passes on their slice, unless
// there are more than this many
constexpr size_t kMaxLargeGroups = 64;
constexpr uint32_t kLargeCap = kMaxLargeGroups + 1;  // large-group list entries read back

// LSD passes over windows W-1 .. first_window of records [0, n) of `data` (in place, via tmp), ordinals =
// current positions.
ley_status window_passes(DeviceContext& ctx, uint8_t* data, uint8_t* tmp, uint64_t n, uint32_t key_bytes,
                         uint32_t first_window, cudaStream_t s, Profiler& prof, void* work, size_t work_bytes) {
  const uint32_t W = (key_bytes + kKeyBytes - 1) / kKeyBytes;
  const uint8_t* src = data;
  uint8_t* dst = tmp;
  for (uint32_t w = W; w-- > first_window;) {
    const KeySpec ks{kKeyBytes * w, std::min<uint32_t>(kKeyBytes, key_bytes - kKeyBytes * w)};
    if (ley_status st = sort_pass(ctx, src, dst, nullptr, n, s, prof, work, work_bytes, ks)) return st;
    src = dst;
    dst = dst == tmp ? data : tmp;
  }
  if (src != data) LEY_CUDA("tie groups", cudaMemcpyAsync(data, src, n * kRecordBytes, cudaMemcpyDeviceToDevice, s));
  return LEY_OK;
}
}  // namespace

// Keys of up to 10 bytes: one pass. Longer keys (§5, flexible key sizes): LSD over the
// 10-byte windows, the last (possibly partial) window first. Each pass is stable with respect to its own
// input order (the ordinal is the position in that input), so after the pass on window 0 the records
// are in (window 0, window 1, ..., original index) order. Passes alternate between out and a scratch
// buffer so the last one lands in out; with perm, the passes' permutations are composed on the device.
ley_status sort_internal_device(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint32_t* perm_out, uint64_t n,
                                cudaStream_t s, Profiler& prof, void* work, size_t work_bytes, uint32_t key_bytes,
                                bool allow_async) {
  if (key_bytes < 1 || key_bytes > kRecordBytes) {
    set_error("internal: key_bytes must be in [1, 100]");
    return LEY_ERR_UNSUPPORTED;
  }
  if (key_bytes <= kKeyBytes)
    return sort_pass(ctx, in, out, perm_out, n, s, prof, work, work_bytes, KeySpec{0, key_bytes}, nullptr, allow_async);
  if (!out) {
    set_error("internal: keys longer than 10 bytes need an output buffer (multi-pass)");
    return LEY_ERR_UNSUPPORTED;
  }
  const uint32_t W = (key_bytes + kKeyBytes - 1) / kKeyBytes;
  ley_status st = ensure_buffer(ctx.keypass, keypass_bytes(n, key_bytes, perm_out != nullptr), "key passes", s);
  if (st) return st;
  uint8_t* tmp = static_cast<uint8_t*>(ctx.keypass.ptr);
  if (!perm_out && options_snapshot().key_hybrid) {
    // Hybrid ("hybrid between prefix sorting and comparison-based record sorting"): sort by the first
    // 10 key bytes, then only the runs of equal 10-byte prefixes need the rest of the key — tiny ones by a
    // warp comparison sort, a few large ones by the window passes on their slice. Random keys: no ties,
    // one pass + one read of the output.
    // K-e writes each output record's prefix digest into the (not yet used) scratch record buffer, so the
    // tie-group scan reads 8 B per record instead of the records' lines
    uint64_t* digest = reinterpret_cast<uint64_t*>(tmp);
    if ((st = sort_pass(ctx, in, out, nullptr, n, s, prof, work, work_bytes, KeySpec{0, kKeyBytes}, digest))) return st;
    const uint32_t cap = (uint32_t)(n / 2 + 1);
    uint32_t* firsts = reinterpret_cast<uint32_t*>(tmp + a256(n * kRecordBytes));
    uint32_t* lasts = firsts + a256(4ull * cap) / 4;
    uint32_t* large_f = lasts + a256(4ull * cap) / 4;  // [kLargeCap] each, then the 4 counts
    uint32_t* large_l = large_f + kLargeCap;
    uint32_t* counts = large_l + kLargeCap;  // [8]
    if ((st = prof.begin("tie groups"))) return st;
    LEY_CUDA("tie groups", cudaMemsetAsync(counts, 0, 32, s));
    LEY_CUDA("tie groups", launch_tie_groups(out, digest, n, firsts, lasts, cap, counts, ctx.sms, s));
    ++prof.launches;
    // no tie groups (random keys): done after one small read-back, without the fixers' launches
    uint32_t h[2 * kLargeCap + 4];
    const uint32_t* hc = h + 2 * kLargeCap;
    LEY_CUDA("tie groups", cudaMemcpyAsync(h + 2 * kLargeCap, counts, 16, cudaMemcpyDeviceToHost, s));
    LEY_CUDA("tie groups", cudaStreamSynchronize(s));
    if (hc[0] || hc[1]) {
      LEY_CUDA("tie groups", launch_fix_small_groups(out, digest, n, firsts, lasts, counts, key_bytes, large_f,
                                                     large_l, kLargeCap, ctx.sms, s));
      prof.launches += 5;
      // one read-back: the counts and the two short large-group lists
      LEY_CUDA("tie groups", cudaMemcpyAsync(h, large_f, sizeof(h), cudaMemcpyDeviceToHost, s));
      LEY_CUDA("tie groups", cudaStreamSynchronize(s));
    }
    bool fallback = hc[0] != hc[1] || hc[0] > cap || hc[2] != hc[3] || hc[2] > kMaxLargeGroups;
    if (!fallback && hc[2]) {
      std::vector<uint32_t> f(h, h + hc[2]), l(h + kLargeCap, h + kLargeCap + hc[3]);
      std::sort(f.begin(), f.end());
      std::sort(l.begin(), l.end());
      // the passes open their own profiler ranges: close "tie groups" first (ranges do not nest)
      if ((st = prof.end()) || (st = prof.begin("tie group passes"))) return st;
      for (size_t g = 0; g < f.size() && !st; ++g) {
        // the passes need a 16-byte-aligned slice: start at the record index rounded down to a multiple
        // of 4 and sort by the whole key (window 0 too), so the up to 3 records before the group — already
        // in their final order, all with a smaller or equal-and-earlier full key — stay where they are
        const uint64_t x0 = f[g] & ~3u, len = l[g] + 1 - x0;
        st = window_passes(ctx, out + x0 * kRecordBytes, tmp, len, key_bytes, 0, s, prof, work, work_bytes);
      }
      if (st) return st;
    }
    if ((st = prof.end())) return st;
    if (!fallback) return LEY_OK;
    // many large tie groups: the plain LSD window passes from the input (below)
  }
  uint32_t* pa = perm_out ? reinterpret_cast<uint32_t*>(tmp + a256(n * kRecordBytes)) : nullptr;
  uint32_t* pb = perm_out ? pa + a256(4 * n) / 4 : nullptr;
  const uint8_t* src = in;
  for (uint32_t p = 0; p < W; ++p) {
    const uint32_t w = W - 1 - p;
    const KeySpec ks{kKeyBytes * w, std::min<uint32_t>(kKeyBytes, key_bytes - kKeyBytes * w)};
    uint8_t* dst = (w % 2 == 0) ? out : tmp;
    uint32_t* pcur = perm_out ? (p == 0 ? pa : pb) : nullptr;
    if ((st = sort_pass(ctx, src, dst, pcur, n, s, prof, work, work_bytes, ks))) return st;
    if (perm_out && p > 0) {  // total order so far: pb[j] = pa[pb[j]]
      LEY_CUDA("key passes", launch_compose_perm(pa, pb, n, ctx.sms, s));
      ++prof.launches;
      std::swap(pa, pb);
    }
    src = dst;
  }
  if (perm_out) {
    cudaPointerAttributes pa_attr{};
    LEY_CUDA("perm", cudaPointerGetAttributes(&pa_attr, perm_out));
    const cudaMemcpyKind kind = pa_attr.type == cudaMemoryTypeDevice ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    LEY_CUDA("perm", cudaMemcpyAsync(perm_out, pa, 4 * n, kind, s));
  }
  return LEY_OK;
}

}  // namespace ley
