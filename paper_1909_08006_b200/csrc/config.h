// config.h — compile-time geometry shared by the kernels and the host planner (plain C++).
#pragma once
#include <stdint.h>

namespace ley {

constexpr uint32_t kRecordBytes = 100;   // P:126 "100-byte records"
constexpr uint32_t kKeyBytes = 10;       // P:126 "10-byte key"
constexpr uint32_t kRecordWords = 25;    // 100 / 4

// K-a tile: THREADS x ITEMS records (tile-local stable sort by key byte 0, P:59 ParallelRadixSort).
constexpr int kTileThreads = 512;
constexpr int kTileItems = 8;
constexpr uint32_t kTileRecords = kTileThreads * kTileItems;  // 4096, power of two (< 2^24)
constexpr uint32_t kTileLog2 = 12;
static_assert((1u << kTileLog2) == kTileRecords, "tile must be a power of two");

// K-c / K-c' chunk: THREADS x ITEMS (key-tail, index) pairs. 2048-pair chunks with four 256-thread CTAs
// per SM measured faster than 4096 with two 512-thread CTAs (more independent barrier domains per SM):
// K-c C2 0.89 -> 0.83 ms, C4 5.98 -> 5.72 ms; THREADS must be >= 256 (one thread per digit).
#ifndef LEY_SPLIT_THREADS
#define LEY_SPLIT_THREADS 256
#define LEY_SPLIT_ITEMS 8
#define LEY_SPLIT_MINB 4
#endif
constexpr int kSplitThreads = LEY_SPLIT_THREADS;
constexpr int kSplitItems = LEY_SPLIT_ITEMS;
constexpr int kSplitMinBlocks = LEY_SPLIT_MINB;
constexpr uint32_t kChunk = kSplitThreads * kSplitItems;  // 2048
static_assert(kSplitThreads >= 256, "K-c ranks 256 digits with one thread each");

constexpr int kRadix = 256;

// K-a accumulates hist16 into kHistCopies copies (CTA t -> copy t % kHistCopies) so skewed keys do not
// serialise on a few L2 atomic addresses; K-b sums the copies. 32 (8 MB of L2): C3's K-a 3.90 -> 3.47 ms
// against 16 copies (64 no better; C2 unchanged).
#ifndef LEY_HIST_COPIES
#define LEY_HIST_COPIES 32
#endif
constexpr int kHistCopies = LEY_HIST_COPIES;

// K-b block tile
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr uint32_t kScanTile = kScanThreads * kScanItems;

// K-d tiers (Algorithm 1: bigBucketThreshold / tinyBucketThreshold).
constexpr uint32_t kWarpTierMax = 32;
constexpr uint32_t kSmemTierMax = 16384;
constexpr int kKdMaxBits = 14;
constexpr int kNumKdListsHost = 6;  // = kNumKdLists (common.cuh): K-d work-list tiers, for host planning

// multi-GPU: at most 8 ranks (one 8 x B200 box; BASELINE.json configs)
constexpr int kMaxRanks = 8;

// Exact range splitter (key bytes 0..3, 4..7, 8..9 big-endian; global ordinal) — SURVEY §8e.
struct DistSplitter {
  uint32_t hi, mid, lo16, gidx;
};

// Keys shorter than 10 bytes: the bits of key bytes [key_bytes, 10) in (hi, mid, lo16) are masked
// off wherever the multi-GPU path compares keys, so equal prefixes fall to the global ordinal.
struct DistKeyMask {
  uint32_t hi = ~0u, mid = ~0u, lo16 = 0xFFFFu;
};
inline DistKeyMask dist_key_mask(uint32_t kb) {
  DistKeyMask m;
  m.hi = kb >= 4 ? ~0u : ~(~0u >> (8 * kb));
  m.mid = kb >= 8 ? ~0u : (kb <= 4 ? 0u : ~(~0u >> (8 * (kb - 4))));
  m.lo16 = kb >= 10 ? 0xFFFFu : (kb == 9 ? 0xFF00u : 0u);
  return m;
}

}  // namespace ley
