/* gen.cpp — host (OpenMP) side of the seeded record generator. See gen_core.h for the spec.
 * Input generation only: no sort arithmetic lives here. Built into gen/libleygen_host.so. */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <omp.h>

#include "gen_core.h"

extern "C" {

/* ZT[v] = floor(2^64 * sum_{u<=v} (u+1)^-1.2 / H), H = sum_{k=1..256} k^-1.2, ZT[255] = 2^64-1.
 * Built once in long double. */
void gen_build_zipf(uint64_t zt[256]) {
  long double h = 0.0L;
  for (int k = 1; k <= 256; ++k) h += powl((long double)k, -1.2L);
  long double acc = 0.0L;
  const long double two64 = 18446744073709551616.0L;
  for (int v = 0; v < 256; ++v) {
    acc += powl((long double)(v + 1), -1.2L);
    long double x = floorl(two64 * (acc / h));
    zt[v] = (x >= two64) ? UINT64_MAX : (uint64_t)x;
  }
  zt[255] = UINT64_MAX;
}

/* Records [i0, i0+count) of distribution `dist` into out (count*100 bytes). */
void gen_records(uint8_t* out, uint64_t i0, uint64_t count, uint64_t seed, int dist, int threads) {
  uint64_t zt[256];
  gen_build_zipf(zt);
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t k = 0; k < (int64_t)count; ++k)
    gen_record(out + 100 * (uint64_t)k, seed, i0 + (uint64_t)k, dist, zt);
}

/* Only the keys (10 bytes each) — used by the generator's statistical tests. */
void gen_keys(uint8_t* out, uint64_t i0, uint64_t count, uint64_t seed, int dist, int threads) {
  uint64_t zt[256];
  gen_build_zipf(zt);
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t k = 0; k < (int64_t)count; ++k)
    gen_key(out + 10 * (uint64_t)k, seed, i0 + (uint64_t)k, dist, zt);
}

/* Duplicate source of record i under GEN_SKEWED, or UINT64_MAX if the record keeps its own key.
 * (One step of the chain; used by tests to check "source index < duplicate index".) */
uint64_t gen_dup_source(uint64_t seed, uint64_t i) {
  if (i > 0 && gen_W(seed, i, 15) < GEN_DUP_THRESHOLD) return gen_mulhi64(gen_W(seed, i, 16), i);
  return UINT64_MAX;
}

}  // extern "C"
