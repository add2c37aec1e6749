/* leyenda.h — C ABI of libleyenda.so: a B200-native (sm_100a) stable MSB radix sort of fixed 100-byte
 * records, the hot path of Leyenda (arXiv 1909.08006).
 *
 * Citations: P:n = PAPER.md line n (the paper text), S:n = SPEC.md line n, BJ = BASELINE.json.
 *   Problem statement: sort records of "a 10-byte key and 90-byte value" under a memory limit
 *   ("only 30 GB of memory is allowed"), internally or externally ("able to adaptively
 *   sort divergent workloads that may or may not fit into memory"). Signature: BJ north_star
 *   "ley_sort(in, out, n_records, record_bytes=100, key_bytes=10, device_budget_bytes, stream)".
 *
 * RESULT (all entry points): the unique stable ascending arrangement out[j] = in[pi(j)] where pi orders
 * record ordinals by (key bytes [0, key_bytes) compared as unsigned bytes, most significant first; then
 * ordinal). key_bytes = 10 is the paper's record format; 1..100 are its "flexible key sizes".
 * Ties keep input order (BJ north_star "stable tie order"). Output is bit-identical
 * across runs, budgets, paths, thresholds/options and GPU counts.
 *
 * THREADING: calls on different devices may run concurrently; calls on the same device are serialised
 * by a per-device mutex. ley_last_error() is thread-local.
 *
 * OWNERSHIP: the caller owns in, out, perm and the stream. The library owns a per-device cached device
 * arena (allocated on first use, grown on demand, released by ley_release_cache), pinned host staging
 * for the external path, internal events, and NCCL communicators created by ley_comm_init.
 *
 * ERRORS: every entry point returns a ley_status. On any error `out` (and `perm`) are unspecified,
 * nothing the caller owns is freed, and ley_last_error() holds a stage-tagged message
 * ("K-c split: an illegal memory access ..."). n_records == 0 returns LEY_OK without touching memory.
 */
#ifndef LEYENDA_H_
#define LEYENDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LEY_OK = 0,
  LEY_ERR_INVALID_ARGUMENT = 1, /* NULL with n>0; in/out (or perm) overlap; base not 16-byte aligned;
                                   pointer on another device; unknown option name                      */
  LEY_ERR_UNSUPPORTED = 2,      /* record_bytes != 100; key_bytes outside 1..100 (1..10 on the external
                                   and multi-GPU paths, see ley_sort); pageable or managed memory;
                                   in/out of different kinds (one host, one device)                   */
  LEY_ERR_BUDGET = 3,           /* device_budget_bytes below the minimum working set of every path   */
  LEY_ERR_TOO_LARGE = 4,        /* n_records > 2^32 - 2 (u32 ordinals plus one sentinel) */
  LEY_ERR_CAPACITY = 5,         /* dist: out_capacity_records < records this rank must hold          */
  LEY_ERR_CUDA = 6,             /* a CUDA runtime error; text in ley_last_error()                     */
  LEY_ERR_NCCL = 7              /* an NCCL error; text in ley_last_error()                            */
} ley_status;

#define LEY_RECORD_BYTES 100u
#define LEY_KEY_BYTES 10u
#define LEY_MAX_RECORDS 0xFFFFFFFEull

/* ley_sort — stable ascending sort of n_records fixed-size records by key bytes [0, key_bytes).
 *   in, out       : both DEVICE pointers on the current device (internal path: K-a .. K-e, §8a rows
 *                   a1-a6), or both PINNED HOST pointers (cudaHostAlloc / cudaHostRegister). Host
 *                   pointers take the staged-internal path when the working set fits
 *                   device_budget_bytes, else the resident path (input staged, output streamed out;
 *                   the paper's partial in-memory regime) when the input fits, else the external path
 *                   (run generation + merge-path K-way merge). ley_plan_query tells which.
 *                   Layout: n_records * record_bytes contiguous bytes, record i at
 *                   byte offset i*record_bytes, key = its first key_bytes bytes. 16-byte aligned bases.
 *                   Out-of-place only ("from the key to the tmp array"); `in` is never written.
 *   n_records     : 0 .. 2^32-2.
 *   record_bytes  : must be 100.
 *   key_bytes     : the key is record bytes [0, key_bytes), 1..100: the paper's 10 and its
 *                   "flexible key sizes". <= 10: one pass; bytes [key_bytes, 10) of the sort
 *                   key carry the ordinal, so equal keys keep input order. > 10: LSD passes over the
 *                   10-byte windows (last window first), each stable, so the result is the same
 *                   stable order; they need an extra n_records x 100-byte device buffer (+ 8 bytes per
 *                   record with perm), device pointers or the staged host path (else
 *                   LEY_ERR_UNSUPPORTED: the external and resident paths take keys of <= 10 bytes).
 *   device_budget_bytes : cap on device memory the LIBRARY allocates for this call (caller buffers
 *                   excluded); 0 = no cap (P:19's memory limit; BJ configs[4] "4 GB per GPU").
 *   stream        : a cudaStream_t (0 = legacy default stream). Work is ordered after prior work on
 *                   `stream`; returns when `out` is complete (host-synchronous) — unless option "async"
 *                   is 1, the pointers are device pointers, key_bytes <= 10 and no bucket needs the
 *                   byte-2 recursion: then it returns once the sort is enqueued and `out` (and perm) are
 *                   complete when `stream` gets there (stream-ordered, like cudaMemcpyAsync). Later
 *                   library calls on the same device order themselves after it. */
ley_status ley_sort(const void* in, void* out, uint64_t n_records, uint32_t record_bytes,
                    uint32_t key_bytes, uint64_t device_budget_bytes, void* stream);

/* ley_sort_perm — ley_sort that also writes perm[j] = input ordinal of output record j (u32, n_records
 * entries, same memory kind as out). Verification hook; not the timed path. */
ley_status ley_sort_perm(const void* in, void* out, uint32_t* perm, uint64_t n_records,
                         uint32_t record_bytes, uint32_t key_bytes, uint64_t device_budget_bytes,
                         void* stream);

/* ---------------------------------------------------------------- streaming host sort
 * ley_sort_submit — enqueue the staged-internal sort of PINNED HOST records (in -> out, same layout and
 *   result as ley_sort) and return once the sort itself is done, WITHOUT waiting for the output's
 *   device->host copy. Consecutive submits on the current device form a pipeline over two device
 *   staging slots and three internal streams: the H2D of call k+1 overlaps the D2H of call k (the two
 *   copy engines), so a stream of sorts is bound by max(H2D, D2H) per call instead of their sum (the
 *   reader/sorter/writer overlap of P:116-118).
 *   in, out, n_records, record_bytes, key_bytes: as ley_sort; both pointers must be pinned host memory
 *     (else LEY_ERR_UNSUPPORTED). `in` must stay unmodified, and `out` is complete, only after
 *     ley_sort_drain(). `stream` orders the start: the H2D waits for work already enqueued on it; the
 *     caller's stream is NOT made to wait for the output (that would serialise consecutive calls).
 *   device_budget_bytes: 0 = no cap. If two slots (4 x n_records x 100 bytes) plus the internal scratch
 *     do not fit the cap, the call runs the blocking ley_sort instead (which may take the external path).
 *   Ownership: the library owns the slots (freed by ley_release_cache). Errors as ley_sort; on error the
 *   pipeline state of earlier calls is unaffected.
 * ley_sort_drain — block until every submitted sort on the current device has landed in its `out`. */
ley_status ley_sort_submit(const void* in, void* out, uint64_t n_records, uint32_t record_bytes,
                           uint32_t key_bytes, uint64_t device_budget_bytes, void* stream);
ley_status ley_sort_drain(void);

/* Stage-tagged message for the last failing call on this thread ("" if none). Valid until the next
 * call on this thread. */
const char* ley_last_error(void);

/* ---------------------------------------------------------------- multi-GPU (one process per GPU)
 * BJ north_star: "Each GPU histograms the leading key bytes, all GPUs agree on range splitters, and
 * records move to their owning GPU by an NCCL all-to-all over NVLink; each GPU then sorts its range
 * locally, and the output is the concatenation of the ranges."
 * Rank r passes its contiguous input slice (device memory); the global ordinal of local record i is
 * (sum of n_local over ranks < r) + i. On return rank r holds global sorted positions
 * [*out_global_offset, *out_global_offset + *n_out_local) with exact splitters:
 * n_out_local(r) = floor((r+1) n / G) - floor(r n / G). Concatenating ranks 0..G-1 equals ley_sort of
 * the concatenated input. key_bytes: 1..10 (shorter keys compare as their prefix).
 * in_local/out_local: device memory on the comm's device, or pinned host memory on EVERY rank — then each
 * rank's slice and output capacity are staged on its device (H2D, the device path, D2H of its range) if
 * they fit device_budget_bytes on every rank, else the multi-GPU EXTERNAL path runs: every
 * rank writes sorted runs of its slice into a host run scratch shared by all ranks (POSIX shared memory
 * under /dev/shm, N x 100 bytes; LEY_ERR_UNSUPPORTED if it cannot be created), all ranks derive the same
 * splitters from the shared samples, and rank r merges global sorted positions
 * [floor(r N/G), floor((r+1) N/G)) into out_local (key_bytes <= 10). */
typedef struct ley_comm ley_comm;
ley_status ley_comm_get_unique_id(uint8_t id_out[128]);  /* rank 0; broadcast it (e.g. torch PG)  */
ley_status ley_comm_init(ley_comm** comm, int nranks, int rank, const uint8_t id[128], int device);
ley_status ley_sort_dist(ley_comm* comm, const void* in_local, uint64_t n_local, void* out_local,
                         uint64_t out_capacity_records, uint64_t* n_out_local,
                         uint64_t* out_global_offset, uint32_t record_bytes, uint32_t key_bytes,
                         uint64_t device_budget_bytes, void* stream);
ley_status ley_comm_destroy(ley_comm* comm);

/* Loopback verification hook: the same G-rank algorithm (kernels K-s0/K-s1/
 * K-s2/K-p, plans, local sort) with all G ranks' slices on the CURRENT device; K-p stores into every
 * receiver's buffer (dist_fused) or device copies stand in for the all-to-all. Arrays have nranks
 * entries. in_local[r]/out_local[r]: device pointers, or pinned host pointers — then the multi-GPU
 * EXTERNAL algorithm runs (every rank's runs, one shared partition, each rank's merge of its exact share;
 * device_budget_bytes as in ley_sort_dist). Same results as ley_sort_dist on G GPUs. Not a performance
 * path. */
ley_status ley_sort_dist_loopback(int nranks, const void* const* in_local, const uint64_t* n_local,
                                  void* const* out_local, const uint64_t* out_capacity_records,
                                  uint64_t* n_out_local, uint64_t* out_global_offset, uint32_t record_bytes,
                                  uint32_t key_bytes, uint64_t device_budget_bytes, void* stream);

/* Host-only planning steps of the distributed sort (pure functions, no CUDA; exposed so the multi-rank
 * logic is testable on CPU with any transport):
 *  ley_dist_plan_splitters: global 65536-bin histogram of key bytes 0..1 (u64) and N -> for k = 1..G-1
 *    the bin holding global sorted rank floor(k N / G) (bins[k-1]), that rank's offset inside the bin
 *    (rank_in_bin[k-1]) and the number of records in smaller bins (bin_first[k-1]). 0 on success.
 *  ley_dist_bin_dest_counts: per-destination record counts of a rank's WHOLE bins (bins that hold no
 *    splitter); boundary-bin records are counted separately against the exact splitters.
 *  ley_dist_plan_exchange: G x G send-count matrix [src][dst] -> this rank's receive counts/offsets (in
 *    source-rank order), send offsets, output size and global output offset.
 *  ley_dist_dest_offsets: the same matrix -> for every destination d, the record offset inside d's
 *    receive buffer where this (source) rank's run starts; the fused exchange (option "dist_fused") has
 *    K-p store there directly. Equals ley_dist_plan_exchange(d).recv_offsets[rank]. */
int ley_dist_plan_splitters(const uint64_t* global_hist16, uint64_t n_total, int nranks, uint32_t* bins,
                            uint64_t* rank_in_bin, uint64_t* bin_first);
void ley_dist_bin_dest_counts(const uint64_t* local_hist16, const uint32_t* bins, int nranks, uint64_t* counts);
void ley_dist_plan_exchange(const uint64_t* send_counts, int nranks, int rank, uint64_t* recv_counts,
                            uint64_t* recv_offsets, uint64_t* send_offsets, uint64_t* n_out, uint64_t* out_offset);
void ley_dist_dest_offsets(const uint64_t* send_counts, int nranks, int rank, uint64_t* dst_offsets);

/* Test hooks of the multi-GPU external path's shared host run scratch (host logic only, no CUDA): create
 * (create=1: checks /dev/shm free space, replaces a stale segment) or open a POSIX shared memory segment
 * of `bytes` and map it (*ptr); close unmaps it and, if unlink_name is non-NULL, removes the name. */
ley_status ley_test_shared_scratch(const char* name, uint64_t bytes, int create, void** ptr);
void ley_test_shared_scratch_close(void* ptr, uint64_t bytes, const char* unlink_name);

/* ---------------------------------------------------------------- introspection and tuning */

/* Host-only plan query (no CUDA calls): device bytes the library allocates to sort n_records on one
 * GPU in-core (internal path), and the path ley_sort would choose for host pointers under `budget`:
 * 0 = staged internal (in and out both staged on the device: staged_bytes), else 2 = resident input,
 * streamed output (the paper's "partial in-memory" regime: the input staged whole, sorted in
 * perm-only mode, the output gathered window by window and copied out: resident_bytes), else
 * 1 = external. Lets tests and callers size budgets. */
typedef struct {
  uint64_t n_records;
  uint64_t tile_records;        /* K-a tile (records)                                    */
  uint64_t tiles;               /* ceil(n / tile)                                        */
  uint64_t chunk_records;       /* K-c / K-c' chunk (pairs)                              */
  uint64_t internal_scratch;    /* bytes of library device memory for the internal path  */
  uint64_t staged_bytes;        /* internal_scratch + in/out staging (host pointers)     */
  int32_t host_path;            /* 0 = staged internal, 1 = external, 2 = resident      */
  uint64_t run_records;         /* external: records per sorted run                      */
  uint64_t runs;                /* external: number of runs                              */
  uint64_t resident_bytes;      /* path 2: scratch + input + perm + 2 output windows     */
} ley_plan_info;
ley_status ley_plan_query(uint64_t n_records, uint64_t device_budget_bytes, ley_plan_info* info);

/* Integer options (process-wide; they change speed, never output):
 *   "warp_tier_max"  K-d: buckets up to this size use the one-warp tier       (1..32, default 32)
 *   "smem_tier_max"  K-d: buckets up to this size are sorted in shared memory; larger ones recurse
 *                    on the next key byte (Alg. 1 bigBucketThreshold) (0..16384, default 16384)
 *   "kd_digit_bits"  K-d: max width of the in-CTA counting digit; 0 = pure comparison sort of each
 *                    bucket (Alg. 1 ComparisonSort); 13-14 apply to the 8192/10240 tiers, the
 *                    others use at most 12                                          (0..14, default 14)
 *   "kd_insert_max"  K-d: sub-buckets up to this size use per-thread insertion sort, larger ones a
 *                    warp bitonic network (tinyBucketThreshold)       (1..64, default 16)
 *   "kd_ws"          1 = warp-specialised K-d+K-e for 513..2048-record buckets (sort warps feed gather
 *                    warps through a ring; TMA bulk record copies), 0 = alternating sort/gather CTAs
 *   "ka_stream"      K-a form: 1 (default) = one persistent CTA per SM streaming only the key rows of the
 *                    records through a ring of TMA tensor copies (64-B L2 fetches: 72 instead of 100
 *                    DRAM bytes per record); 2 = the same ring carrying whole records (TMA bulk
 *                    copies); 0 = one CTA per tile with direct key loads
 *   "dist_fused"     ley_sort_dist / loopback: 1 = fused partition + exchange — K-p stores every record
 *                    straight into its owner's receive window (NCCL symmetric memory over NVLink;
 *                    SURVEY §8f NEXT 1), 0 = K-p into a local send buffer, then an NCCL all-to-all-v
 *   "dist_exchange_g1" 1 = run the splitter, partition and exchange phases even with one rank (tests the
 *                    exchange path on a single GPU), 0 = one rank sorts locally
 *   "key_hybrid"     keys > 10 bytes: 1 = one 10-byte sort + comparison sort of the tie groups (P:164's
 *                    hybrid), 0 = LSD passes over every 10-byte window
 *   "profile"        1 = record CUDA events around every stage (ley_stage_times)
 *   "ext_run_records" external path: force the run size (records; 0 = from the budget)
 *   "resident_path"  1 = host pointers may take path 2 (resident input, streamed output) when in + out
 *                    do not both fit the budget but the input does; 0 = such sorts go external
 *   "resident_chunk_records" path 2 output window (records; 0 = 2^21; never above ceil(n / 4))
 *   "pipe_split"     ley_sort_submit: each H2D / D2H copy in this many pieces on their own streams
 *                    (1..4, default 2: more of the host link busy in each direction)
 *   "l2_fetch_bytes" cudaLimitMaxL2FetchGranularity set before each call (0 = leave the device default;
 *                    32/64/128 accepted; kept for experiments, see profiles/r02_fetch_granularity.txt)
 *   "nccl_timeout_ms" multi-GPU fault handling ("any stage failure aborts the pipeline, reports
 *                    the stage"): every wait on a collective polls ncclCommGetAsyncError; an NCCL error,
 *                    or a collective still incomplete after this many ms (a peer that failed or never
 *                    arrived), aborts the communicator (ncclCommAbort) and returns LEY_ERR_NCCL with the
 *                    stage in ley_last_error(). An aborted communicator refuses further sorts
 *                    (LEY_ERR_NCCL); ley_comm_destroy still releases it. Default 120000, 50..3600000.
 *   "dist_fault_stall" test hook: after the k-th collective of a ley_sort_dist call the stream is held as
 *                    if a peer never completed it (0 = off), exercising the timeout + abort path on one GPU.
 *   "ka_ring"        K-a key-row form: pieces in flight (4, 6 (default), 8 or 11; deeper measured slower)
 *   "tma_l2_promo"   L2 promotion of the record tensor maps: 64 (default), 128, 256 or 0 ("none", which
 *                    behaves like 128 on B200); profiles/r02_fetch_granularity.txt
 *   "ws_gather_tma"  warp-specialised K-d+K-e tier: 0 (default) = record windows by plain bulk copies,
 *                    1 = by tensor copies with 64-B L2 fetches (fewer DRAM bytes, measured slower)
 *   "gather_l2_64"   alternating K-d+K-e tiers: 1 (default) = cp.async with .L2::64B, 0 = without the hint
 *   "ext_keyptr"     external path form: 0 (default) = runs of whole records; 1 = the paper's key-pointer
 *                    pattern: runs of 16-byte (key, ordinal) tuples (host
 *                    scratch 16 instead of 100 B/record), every output record gathered from the pinned
 *                    input by its ordinal over the host link (the input must be mapped pinned memory:
 *                    cudaHostAlloc, or cudaHostRegister with cudaHostRegisterMapped; else
 *                    LEY_ERR_UNSUPPORTED). Same bytes; slower on PCIe (random reads over the link)
 *   "graphs"         1 (default) = level 1 of the internal sort (init .. K-e, 12 launches) is captured once
 *                    per (buffers, n, options) into a CUDA graph and replayed in the caller's stream (C1 1e6
 *                    records: 0.225 -> 0.187 ms when introduced); not while "profile" is on
 *   "pdl"            programmatic dependent launch of the K-d+K-e tier kernels: 0 = plain stream order,
 *                    1 = each tier waits for its predecessor, then lets the next launch, 2 = the first tier
 *                    waits, the later (independent) tiers launch at once and wait only before exiting,
 *                    3 (default) = 2 below 1e7 records, else 0 (measured: pays at C1, costs at C2/C4)
 *   "async"          0 (default) = ley_sort / ley_sort_perm return when the output is complete; 1 = device
 *                    sorts that need no recursion return once enqueued (the host waits only for the
 *                    level-1 classification's big-bucket count; see ley_sort "stream")
 *   "kd_claim"       K-d+K-e tier CTAs take buckets from their list by atomic ticket, one bucket ahead
 *                    (1, default), or by a static stride (0)
 *   "kc_fuse"        level-1 K-c split inside the K-d+K-e kernel of one tier: 0 (default) = its own kernel,
 *                    1 = the tier of the average 16-bit bucket, 2..5 = the 2048 / 8192 / 10240 / 16384
 *                    tier (tests); same bytes, measured slower
 *   "kc_corun"       level-1 K-c kernel narrowed to this many CTAs per SM (1..3) with the warp-specialised
 *                    2048 tier launched beside it (PDL), each bucket sorted once its byte-0 bucket is split;
 *                    applies when the average 16-bit bucket falls in that tier (C2) and kc_fuse is 0, or
 *                    whenever kc_fuse is 2 (tests); 0 = off
 * Returns LEY_ERR_INVALID_ARGUMENT for an unknown name or out-of-range value. */
ley_status ley_set_option(const char* name, int64_t value);
ley_status ley_get_option(const char* name, int64_t* value);

/* Per-stage device times (ms) of the last ley_sort on this thread when "profile" was 1. names[i] points
 * to static strings. Returns the number of stages written (<= max). Kernel launch count of the last call
 * is written to *launches. */
int ley_stage_times(const char** names, float* ms, int max, int* launches);

/* Device memory held by the library (all devices; the cached arena, staging slots, dist buffers) and its
 * high-water mark since the last reset (reset_peak != 0 resets it to the current value). Lets callers and
 * tests check that a call stayed within device_budget_bytes. */
ley_status ley_device_bytes(uint64_t* current_bytes, uint64_t* peak_bytes, int reset_peak);

/* Free the cached arena of `device` (-1 = all devices). */
ley_status ley_release_cache(int device);

uint32_t ley_version(void); /* (major << 16) | minor */

/* ---------------------------------------------------------------- kernel verification hooks
 * Single kernels of the path on caller-provided DEVICE buffers, checked by the tests
 * against CPU models. Synchronous. Not performance paths.
 * ley_test_scan_excl — K-b, the decoupled-look-back exclusive scan ("where each key should be
 *   placed"): out[i] = sum of in[0..i), out[m] = total. in: u32[m]; out: u32[m + 1].
 * ley_test_tile_sort — K-a on n records (P:59 ParallelRadixSort radix 0, P:102 extraction), 4096-record
 *   tiles t = 0..T-1, T = ceil(n / 4096): k1/w = u64[n] / u32[n] (each tile's pairs in byte-0 order:
 *   k1 = key bytes 1..8 big-endian, w = key byte 9 << 24 | index inside the tile), cnt = u32[256 * T]
 *   (cnt[b * T + t] = records of tile t with byte 0 = b), lo = u32[T * 256] (tile-local exclusive offsets),
 *   hist16 = u32[65536] (zeroed, then the count of every 2-byte prefix). stream_form: the K-a form of the
 *   "ka_stream" option (1 = key rows by TMA tensor copies, 2 = whole records by TMA bulk copies, 0 = one
 *   CTA per tile). */
ley_status ley_test_scan_excl(const uint32_t* in, uint32_t* out, uint64_t m, void* stream);
ley_status ley_test_tile_sort(const void* in, uint64_t n, uint64_t* k1, uint32_t* w, uint32_t* cnt, uint32_t* lo,
                              uint32_t* hist16, int stream_form, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LEYENDA_H_ */
