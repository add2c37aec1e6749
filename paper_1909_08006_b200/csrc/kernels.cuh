// kernels.cuh — launch wrappers of the sm_100a kernels (K-a .. K-e) used by the host drivers.
#pragma once
#include <cuda.h>
#include <utility>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "common.cuh"

namespace ley {

// kern<<<grid, block, smem, s>>>(args...), with the programmatic-serialization attribute when pdl (the
// kernel must call pdl_wait() before reading its predecessor's output; common.cuh).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// The 10-byte key window one sort pass orders by: record bytes [off, off + len), off a multiple of 10,
// 1 <= len <= 10 (len < 10: bytes [len, 10) of the window carry the ordinal; k_tile.cu)
struct KeySpec {
  uint32_t off = 0;
  uint32_t len = 10;
};

// TMA tensor map over records [0, 4 floor(n/4)) of `in` viewed as [groups][25 rows][16 B] (400-B group
// pitch), boxes of box_rows x box_groups, L2 promotion 64 B (tmap.cu)
cudaError_t record_group_map(CUtensorMap* map, const uint8_t* in, uint64_t n, uint32_t box_rows, uint32_t box_groups);

// K-a (k_tile.cu). form: 0 = one CTA per tile, direct key loads; 1 = persistent, key rows by TMA tensor
// copies (64-B L2 fetches; keys at record offset 0 only); 2 = persistent, whole records by TMA bulk copies
size_t ka_smem_bytes();
cudaError_t launch_ka_tile_sort(const uint8_t* in, uint64_t n, uint32_t tiles, uint64_t* k1_out, uint32_t* w_out,
                                uint32_t* cnt, uint32_t* lo, uint32_t* hist16, uint32_t copies, int form,
                                KeySpec key, cudaStream_t s);

// K-b (k_scan.cu)
// (two independent exclusive scans in one launch; one ticket word)
// (job b's input may be `copies_b` histogram copies `stride_b` words apart: it scans their sum and writes
// the sum back over copy 0; out2_b: a second copy of its prefix)
cudaError_t launch_scan_excl2(const uint32_t* in_a, uint32_t* out_a, uint64_t m_a, uint64_t* status_a,
                              uint32_t* total_a, uint32_t* in_b, uint32_t* out_b, uint64_t m_b,
                              uint64_t* status_b, uint32_t* total_b, uint32_t copies_b, uint64_t stride_b,
                              uint32_t* ticket, cudaStream_t s, uint32_t* out2_b = nullptr);
cudaError_t launch_scan_excl(const uint32_t* in, uint32_t* out, uint64_t m, uint64_t* status, uint32_t* ticket,
                             uint32_t* total_out, cudaStream_t s);
uint64_t scan_status_words(uint64_t m);
cudaError_t launch_zero3(void* a, uint64_t a_bytes, void* b, uint64_t b_bytes, void* c, uint64_t c_bytes, int sms,
                         cudaStream_t s);
cudaError_t launch_publish_u32(const uint32_t* src, uint32_t* host_mapped_dev, cudaStream_t s);

// K-c / K-c' (k_split.cu). The level-1 plan launch also classifies the level-1 buckets (classify.cuh).
struct ClassifyJob;
size_t split_smem_bytes();
cudaError_t launch_kc_split_level1(const uint64_t* k1_in, const uint32_t* w_in, uint32_t tiles, const uint32_t* off,
                                   const uint32_t* lo, const uint32_t* B16, uint64_t n, uint32_t* cstart,
                                   uint4* plan_a, uint2* plan_b, uint32_t* order, uint32_t* cursor, uint32_t* ticket,
                                   uint64_t* tail_out, uint32_t* idx_out, uint32_t grid_ub, cudaStream_t s,
                                   const ClassifyJob& cls, bool run_split = true,
                                   const uint32_t** order_used = nullptr, uint32_t* done = nullptr,
                                   int corun_per_sm = 0);
cudaError_t launch_kr_nchunks(const Seg* segs, uint32_t nseg, uint32_t* nch, cudaStream_t s);
cudaError_t launch_kr_chunk_map(const uint32_t* cstart, uint32_t nseg, uint32_t ub, uint2* map, cudaStream_t s);
cudaError_t launch_kr_hist(const Seg* segs, uint32_t nseg, const uint32_t* cstart, uint32_t grid,
                           const uint64_t* tails0, const uint32_t* idx0, const uint64_t* tails1, const uint32_t* idx1,
                           uint32_t* seg_hist, const uint2* map, cudaStream_t s);
cudaError_t launch_kr_plan(const Seg* segs, uint32_t nseg, const uint32_t* seg_hist, uint32_t* seg_excl,
                           uint8_t* noscatter, const Tunables& tu, const ListSet& kd, Seg* big_out,
                           uint32_t* big_count, cudaStream_t s);
cudaError_t launch_kr_split(const Seg* segs, uint32_t nseg, const uint32_t* cstart, uint32_t* cursor,
                            const uint8_t* noscatter, uint64_t* tails0, uint32_t* idx0, uint64_t* tails1,
                            uint32_t* idx1, uint32_t* ticket, const uint2* map, uint32_t grid_ub, cudaStream_t s);

// K-d (k_bucket.cu)
// K-d + K-e fused: sorts every listed bucket and gathers its records into out (perm written if non-null;
// out == nullptr: perm-only, no gather; dg non-null: dg[j] = digest of output record j's 10-byte prefix).
// in holds n_in records; no gather reads outside them. Level 1 only: with kc and a fused_tier in
// [kListMed2, kNumKdLists) that tier's kernel runs first and also performs the level-1 split K-c
// (kc_chunk.cuh), claiming its own buckets from kc->kd_ticket (its list is ignored).
struct KcArgs;
cudaError_t launch_kd_all(const ListSet& kd, const uint64_t* t0, const uint32_t* i0, const uint64_t* t1,
                          const uint32_t* i1, uint32_t* perm, const Tunables& tu, int sms, const uint8_t* in,
                          uint64_t n_in, uint8_t* out, uint64_t* dg, cudaStream_t s, int* launches,
                          const KcArgs* kc = nullptr, int fused_tier = -1);

// K-e over one window of the sorted order (k_gather.cu): out[j] = in[perm[j]], j < cnt
cudaError_t launch_ke_gather(const uint8_t* in, const uint32_t* perm, uint64_t cnt, uint8_t* out, int sms,
                             cudaStream_t s);
// keys > 10 bytes, hybrid form (k_ties.cu): runs of equal 10-byte prefixes in sorted records -> unordered
// (first, last) lists (counts[0], counts[1]; entries past cap dropped; dg: the K-e prefix digests of the
// records, or null to compare every adjacent pair on the records); then, driven by those device lists:
// in-place comparison sort of every group of <= 1024 records by key bytes [10, key_bytes) then position,
// and the firsts / lasts of the longer groups appended to large_f / large_l (counts[2], counts[3]; entries
// past large_cap dropped; "large" = more than 1024 records, smaller groups sorted on the device; the
// firsts and lasts arrays are overwritten, counts[4..6] used as scratch counters: the caller's 32-byte
// memset of counts covers them)
cudaError_t launch_tie_groups(const uint8_t* recs, const uint64_t* dg, uint64_t n, uint32_t* firsts, uint32_t* lasts, uint32_t cap,
                              uint32_t* counts, int sms, cudaStream_t s);
// (dg required here)
cudaError_t launch_fix_small_groups(uint8_t* recs, const uint64_t* dg, uint64_t n, uint32_t* firsts,
                                    uint32_t* lasts, uint32_t* counts, uint32_t key_bytes, uint32_t* large_f,
                                    uint32_t* large_l, uint32_t large_cap, int sms, cudaStream_t s);
// multi-pass keys: cur[j] = prev[cur[j]] (the permutation of the passes so far, k_gather.cu)
cudaError_t launch_compose_perm(const uint32_t* prev, uint32_t* cur, uint64_t n, int sms, cudaStream_t s);

// multi-GPU (k_dist.cu)
cudaError_t launch_ks_hist16(const uint8_t* in, uint64_t n, uint32_t* hist, uint16_t* pref, DistKeyMask km, int sms,
                             cudaStream_t s);
uint64_t ks_candidate_tiles(uint64_t n);
cudaError_t launch_ks_candidates(const uint8_t* in, const uint16_t* pref, uint64_t n, uint32_t gbase,
                                 const uint32_t* bins, int nbins,
                                 uint64_t* status, uint32_t* ticket, uint8_t* cand, uint32_t* cand_gidx,
                                 uint32_t* cand_count, cudaStream_t s);
cudaError_t launch_ks_dest_counts(const uint8_t* cand, const uint32_t* cand_gidx, uint32_t ncand,
                                  const DistSplitter* spl, int nspl, unsigned long long* counts, DistKeyMask km,
                                  int sms, cudaStream_t s);
uint64_t kp_tiles(uint64_t n);
// dst_base[d] / dst_off[d] (device arrays, kMaxRanks): where destination d's run starts (records);
// remote = the bases are peers' windows (adds a system-scope fence before the grid completes)
cudaError_t launch_kp_partition(const uint8_t* in, uint64_t n, uint32_t gbase, const DistSplitter* spl, int nspl,
                                uint8_t* const* dst_base, const uint64_t* dst_off, uint64_t* status, uint32_t* ticket,
                                bool remote, DistKeyMask km, cudaStream_t s);

}  // namespace ley
