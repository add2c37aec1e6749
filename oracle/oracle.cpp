/* oracle.cpp — the CPU ORACLE for the Leyenda record sort. TEST INFRASTRUCTURE ONLY.
 *
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 *   or call this library. The product path (paper_1909_08006_b200/, libleyenda.so) never does, and
 *   shares no code with it: no headers, helpers, tables or constants.
 *
 * What it computes — the plain DEFINITION, not a replay of Algorithm 1:
 *   The method (MSD radix sort over (key, pointer) tuples, then a scatter of records; §3.1
 *   lines 50-96 and §3.2) reaches exactly one result: the stable ascending sort of the
 *   100-byte records by their 10-byte key ("a 10-byte key and 90-byte value"), keys compared as
 *   unsigned bytes, most significant first (the radix-digit order of §2.2 line 33), ties
 *   broken by original record index (BASELINE.json north_star: "a comparison sort on the full key
 *   with ties broken by original record index"). Because (key, index) is a strict total
 *   order, exactly one output is correct.
 *
 *   oracle_sort:  E[i] = (key bytes of record i, i)          -- the (key, pointer) tuples of P:102
 *                 sort E by (memcmp(key) , then index)       -- library comparison sort
 *                 perm[j] = E[j].idx;  out[j] = in[perm[j]]  -- the record scatter of P:104-106
 *
 * oracle_sort_kb / oracle_certify_kb: the same definition with key = bytes [0, key_bytes) (§5
 * P:164 flexible key sizes), pinned by brute force for 1..100-byte keys, Python's stable sort on the
 * prefix, and agreement with oracle_sort at key_bytes = 10.
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): brute force over all n! orders for n <= 7, an insertion
 * sort written in Python, Python's stable sorted() on the key alone, closed forms (all-equal ->
 * identity, sorted -> identity, strictly decreasing -> reversal, single-byte-position keys), the §2.2
 * worked example (tests/golden/paper_s2_2_example.json) and the multiset-hash invariants; the
 * __gnu_parallel branch (n >= 2e5) and the stage-timed form against numpy's lexsort at 2e5..5e6 records
 * (uniform, tiny-alphabet, three-key inputs); oracle_is_sorted by accept/reject cases at every key byte.
 * Parity unpinned: none of the functions in this file.
 *
 * Helpers: a permutation-invariant multiset hash (SPEC-style: per-record 128-bit hash summed mod
 * 2^128), an order-dependent digest (for configs whose sorted output is too big to keep on the host),
 * a sortedness check and the certificate check (perm is a permutation, out[j] == in[perm[j]],
 * (key, perm) strictly increasing), which together pin the output to the oracle's.
 */
#include <omp.h>
#include <parallel/algorithm>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

namespace {

struct Tuple {          /* the (key, pointer) tuple of P:102, pointer = ordinal */
  uint8_t key[10];
  uint32_t idx;
};

inline bool tuple_less(const Tuple& a, const Tuple& b) {
  int c = memcmp(a.key, b.key, 10); /* unsigned lexicographic */
  if (c != 0) return c < 0;
  return a.idx < b.idx;             /* stable: original index breaks ties */
}

/* murmur3 fmix64 — the oracle's own mixer (independent of the generator's). */
inline uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

/* 128-bit hash of one 100-byte record: two independent 64-bit chains over its 25 little-endian words. */
inline void record_hash(const uint8_t* r, uint64_t* h0, uint64_t* h1) {
  uint64_t a = 0x243F6A8885A308D3ULL, b = 0x13198A2E03707344ULL;
  for (int q = 0; q < 25; ++q) {
    uint32_t w;
    memcpy(&w, r + 4 * q, 4);
    a = fmix64(a ^ ((uint64_t)w + 0x9E37ULL * (uint64_t)(q + 1)));
    b = fmix64(b + ((uint64_t)w << 17) + (uint64_t)(q + 1) * 0xA4093822299F31D0ULL);
  }
  *h0 = a;
  *h1 = b;
}

inline void add128(uint64_t* lo, uint64_t* hi, uint64_t a_lo, uint64_t a_hi) {
  uint64_t s = *lo + a_lo;
  *hi += a_hi + (s < *lo ? 1 : 0);
  *lo = s;
}

}  // namespace

/* The one sort body behind oracle_sort and oracle_sort_timed: extraction of the (key, pointer) tuples
 * (P:102), the library comparison sort on (key, index), and the record scatter. When
 * secs != NULL the three stages are timed (Table 3's stage breakdown). The comparison sort is
 * std::sort below 2e5 tuples or with one thread, else __gnu_parallel::sort (OpenMP, `threads`); both
 * are pinned by tests/test_oracle.py (the parallel branch against numpy's lexsort at n >= 2e5). */
static int sort_body(const uint8_t* in, uint8_t* out, uint32_t* perm, uint64_t n, int threads, double* secs) {
  if (n > 0xFFFFFFFEULL) return 1;
  if (secs) secs[0] = secs[1] = secs[2] = 0.0;
  if (n == 0) return 0;
  if (threads <= 0) threads = omp_get_max_threads();
  const double t0 = omp_get_wtime();
  std::vector<Tuple> e(n);
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    memcpy(e[i].key, in + 100 * (uint64_t)i, 10);
    e[i].idx = (uint32_t)i;
  }
  const double t1 = omp_get_wtime();
  if (n < 200000 || threads == 1) {
    std::sort(e.begin(), e.end(), tuple_less);
  } else {
    omp_set_num_threads(threads);
    __gnu_parallel::sort(e.begin(), e.end(), tuple_less);
  }
  const double t2 = omp_get_wtime();
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t j = 0; j < (int64_t)n; ++j) {
    uint32_t p = e[j].idx;
    if (perm) perm[j] = p;
    if (out) memcpy(out + 100 * (uint64_t)j, in + 100 * (uint64_t)p, 100);
  }
  const double t3 = omp_get_wtime();
  if (secs) {
    secs[0] = t1 - t0;
    secs[1] = t2 - t1;
    secs[2] = t3 - t2;
  }
  return 0;
}

extern "C" {

/* Returns 0 on success, 1 if n is out of the ordinal range (n > 2^32 - 2). perm may be NULL. */
int oracle_sort(const uint8_t* in, uint8_t* out, uint32_t* perm, uint64_t n, int threads) {
  return sort_body(in, out, perm, n, threads, nullptr);
}

/* Stage-timed form for the CPU baseline (the same sort body; mirrors Table 3's stage breakdown,
 * P:141-144): secs[0] = tuple extraction, secs[1] = sort, secs[2] = record gather. */
int oracle_sort_timed(const uint8_t* in, uint8_t* out, uint64_t n, int threads, double secs[3]) {
  return sort_body(in, out, nullptr, n, threads, secs);
}

/* Permutation-invariant digest: sum over records of a 128-bit record hash, mod 2^128. */
void oracle_multiset_hash(const uint8_t* recs, uint64_t n, uint64_t out[2], int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  uint64_t lo = 0, hi = 0;
#pragma omp parallel num_threads(threads)
  {
    uint64_t l = 0, h = 0;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
      uint64_t a, b;
      record_hash(recs + 100 * (uint64_t)i, &a, &b);
      add128(&l, &h, a, b);
    }
#pragma omp critical
    add128(&lo, &hi, l, h);
  }
  out[0] = lo;
  out[1] = hi;
}

/* Order-dependent digest of a record sequence whose first record has global position j0:
 * sum_j fmix(record_hash(rec_j) ^ position j), mod 2^128. Two sequences agree on it iff (w.h.p.) they
 * are equal; chunk digests add up, so huge outputs can be checked slice by slice. */
void oracle_sequence_digest(const uint8_t* recs, uint64_t n, uint64_t j0, uint64_t out[2], int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  uint64_t lo = 0, hi = 0;
#pragma omp parallel num_threads(threads)
  {
    uint64_t l = 0, h = 0;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
      uint64_t a, b, j = j0 + (uint64_t)i;
      record_hash(recs + 100 * (uint64_t)i, &a, &b);
      add128(&l, &h, fmix64(a ^ (j * 0x9E3779B97F4A7C15ULL)), fmix64(b + j));
    }
#pragma omp critical
    add128(&lo, &hi, l, h);
  }
  out[0] = lo;
  out[1] = hi;
}

/* Digest of the oracle's sorted output without materialising it: tuples are sorted, then records
 * are hashed in sorted order straight from `in` (digest mode for the 60 GB configs). */
int oracle_sorted_digest(const uint8_t* in, uint64_t n, uint64_t out[2], int threads) {
  if (n > 0xFFFFFFFEULL) return 1;
  out[0] = out[1] = 0;
  if (n == 0) return 0;
  if (threads <= 0) threads = omp_get_max_threads();
  std::vector<uint32_t> perm(n);
  int rc = oracle_sort(in, nullptr, perm.data(), n, threads);
  if (rc) return rc;
  uint64_t lo = 0, hi = 0;
#pragma omp parallel num_threads(threads)
  {
    uint64_t l = 0, h = 0;
#pragma omp for schedule(static)
    for (int64_t j = 0; j < (int64_t)n; ++j) {
      uint64_t a, b;
      record_hash(in + 100 * (uint64_t)perm[j], &a, &b);
      add128(&l, &h, fmix64(a ^ ((uint64_t)j * 0x9E3779B97F4A7C15ULL)), fmix64(b + (uint64_t)j));
    }
#pragma omp critical
    add128(&lo, &hi, l, h);
  }
  out[0] = lo;
  out[1] = hi;
  return 0;
}

/* Flexible key size (§5, "flexible key sizes"): the same definition
 * with the key = record bytes [0, key_bytes), 1 <= key_bytes <= 100, compared as unsigned bytes, ties by
 * original index. Written separately from oracle_sort (a comparison of the records themselves, no
 * tuple extraction), so the key_bytes = 10 case also cross-checks the tuple path. Returns 0 on success,
 * 1 if n is out of range, 2 if key_bytes is. */
int oracle_sort_kb(const uint8_t* in, uint8_t* out, uint32_t* perm, uint64_t n, int key_bytes, int threads) {
  if (n > 0xFFFFFFFEULL) return 1;
  if (key_bytes < 1 || key_bytes > 100) return 2;
  if (n == 0) return 0;
  if (threads <= 0) threads = omp_get_max_threads();
  std::vector<uint32_t> idx(n);
  for (uint64_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
  const size_t k = (size_t)key_bytes;
  auto less = [in, k](uint32_t a, uint32_t b) {
    int c = memcmp(in + 100 * (uint64_t)a, in + 100 * (uint64_t)b, k);
    return c != 0 ? c < 0 : a < b;
  };
  if (n < 200000 || threads == 1) {
    std::sort(idx.begin(), idx.end(), less);
  } else {
    omp_set_num_threads(threads);
    __gnu_parallel::sort(idx.begin(), idx.end(), less);
  }
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t j = 0; j < (int64_t)n; ++j) {
    if (perm) perm[j] = idx[j];
    if (out) memcpy(out + 100 * (uint64_t)j, in + 100 * (uint64_t)idx[j], 100);
  }
  return 0;
}

/* 1 if the keys of recs are non-decreasing (unsigned lexicographic), else 0. */
int oracle_is_sorted(const uint8_t* recs, uint64_t n) {
  for (uint64_t j = 1; j < n; ++j)
    if (memcmp(recs + 100 * (j - 1), recs + 100 * j, 10) > 0) return 0;
  return 1;
}

/* Certificate: returns 0 if (a) perm is a permutation of [0,n), (b) out[j] == in[perm[j]] for all j,
 * (c) (key(out[j]), perm[j]) is strictly increasing in j. Together these force out == oracle output.
 * Otherwise returns 1 + the first failing j (or n+1 for a non-permutation). */
uint64_t oracle_certify_kb(const uint8_t* in, const uint8_t* out, const uint32_t* perm, uint64_t n, int key_bytes);
uint64_t oracle_certify(const uint8_t* in, const uint8_t* out, const uint32_t* perm, uint64_t n) {
  return oracle_certify_kb(in, out, perm, n, 10);
}

/* The certificate with key = bytes [0, key_bytes). */
uint64_t oracle_certify_kb(const uint8_t* in, const uint8_t* out, const uint32_t* perm, uint64_t n, int key_bytes) {
  std::vector<uint8_t> seen(n, 0);
  for (uint64_t j = 0; j < n; ++j) {
    if (perm[j] >= n || seen[perm[j]]) return n + 1;
    seen[perm[j]] = 1;
  }
  for (uint64_t j = 0; j < n; ++j) {
    if (memcmp(out + 100 * j, in + 100 * (uint64_t)perm[j], 100) != 0) return j + 1;
    if (j > 0) {
      int c = memcmp(out + 100 * (j - 1), out + 100 * j, (size_t)key_bytes);
      if (c > 0 || (c == 0 && perm[j - 1] >= perm[j])) return j + 1;
    }
  }
  return 0;
}

}  // extern "C"
