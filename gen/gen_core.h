/* gen_core.h — seeded, counter-based synthetic 100-byte records.
 *
 * This module is INPUT GENERATION ONLY. It holds none of the sort's arithmetic and is shared, as the
 * task allows, by the oracle tests (gen.cpp, host/OpenMP) and by the GPU tests / bench (gen_cuda.cu,
 * the CUDA twin that writes records straight into HBM). Both sides compile this one header, so the
 * twin is byte-identical by construction; tests still check it on samples.
 *
 * Record layout (§4.1: "Each record is made up of a 10-byte key and 90-byte value"):
 *   bytes 0..9 = key, bytes 10..99 = payload.  gensort's byte stream is NOT reproduced.
 *
 * W(seed, i, w) = sm64(seed * 2^40 + i * 32 + w)       i < 2^35, w < 32
 * uniform record i : bytes 0..99 = little-endian bytes of W(seed, i, 0..12) (first 100 of 104)
 * skewed  record i : BASELINE.json configs[2] — byte0 ~ Zipf(s=1.2) over 256 values (rank k -> byte k-1,
 *                    SURVEY Q4), byte1 uniform over {0..7} (Q5), bytes 2..9 uniform, and with
 *                    probability 0.02 the whole key is copied from src = mulhi(W(seed,i,16), i) < i,
 *                    recursively (Q6). The payload always stays the record's own.
 * The other distributions are edge cases for the parity tests.
 */
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define GEN_HD __host__ __device__ __forceinline__
#else
#define GEN_HD static inline
#endif

enum gen_dist {
  GEN_UNIFORM = 0,      /* C1, C2, C4, C5                                                        */
  GEN_SKEWED = 1,       /* C3: Zipf(1.2) byte 0, byte 1 in {0..7}, 2% earlier-key copies          */
  GEN_ALL_EQUAL = 2,    /* every key identical -> output == input (stability is everything)     */
  GEN_THREE_KEYS = 3,   /* keys drawn from 3 fixed values                                        */
  GEN_SORTED = 4,       /* key = 0x0000 ++ BE64(i): strictly increasing                          */
  GEN_REVERSE = 5,      /* key = 0xFFFF ++ BE64(2^64-1-i): strictly decreasing                   */
  GEN_PREFIX2 = 6,      /* constant 2-byte prefix 0xAB 0xCD, bytes 2..9 uniform (forces recursion) */
  GEN_BYTE9 = 7,        /* bytes 0..8 constant, byte 9 uniform (recursion to the last byte)      */
  GEN_ASCII = 8,        /* printable key bytes 0x20..0x7E (the paper's 20 GB ASCII set)   */
  GEN_TINY_ALPHABET = 9,/* each key byte in {0x00, 0x01, 0xFF}: many ties, deep buckets          */
  GEN_NUM_DISTS = 10
};

/* floor(0.02 * 2^64): duplicate-key probability threshold */
#define GEN_DUP_THRESHOLD 368934881474191032ULL

GEN_HD uint64_t gen_sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

GEN_HD uint64_t gen_W(uint64_t seed, uint64_t i, uint32_t w) {
  return gen_sm64((seed << 40) + (i << 5) + (uint64_t)w);
}

GEN_HD uint64_t gen_mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
#endif
}

GEN_HD void gen_put_le64(uint8_t* p, uint64_t v, int nbytes) {
  for (int b = 0; b < nbytes; ++b) p[b] = (uint8_t)(v >> (8 * b));
}
GEN_HD void gen_put_be64(uint8_t* p, uint64_t v) {
  for (int b = 0; b < 8; ++b) p[b] = (uint8_t)(v >> (56 - 8 * b));
}

/* Zipf byte: min v with u < zt[v] (zt[255] = 2^64-1 is the sentinel). Linear search is fine: the
 * distribution is heavily front-loaded and this runs once per record at generation time. */
GEN_HD uint32_t gen_zipf_byte(uint64_t u, const uint64_t* zt) {
  uint32_t v = 0;
  while (v < 255 && !(u < zt[v])) ++v;
  return v;
}

/* The 10-byte key of record i. */
GEN_HD void gen_key(uint8_t key[10], uint64_t seed, uint64_t i, int dist, const uint64_t* zt) {
  switch (dist) {
    case GEN_SKEWED: {
      uint64_t j = i;
      while (j > 0 && gen_W(seed, j, 15) < GEN_DUP_THRESHOLD) j = gen_mulhi64(gen_W(seed, j, 16), j);
      gen_put_le64(key, gen_W(seed, j, 0), 8);
      gen_put_le64(key + 8, gen_W(seed, j, 1), 2);
      key[0] = (uint8_t)gen_zipf_byte(gen_W(seed, j, 13), zt);
      key[1] = (uint8_t)(gen_W(seed, j, 14) & 7);
      return;
    }
    case GEN_ALL_EQUAL: {
      uint64_t a = gen_W(seed, 0, 20), b = gen_W(seed, 0, 21);
      gen_put_le64(key, a, 8);
      gen_put_le64(key + 8, b, 2);
      return;
    }
    case GEN_THREE_KEYS: {
      uint64_t which = gen_W(seed, i, 13) % 3;
      gen_put_le64(key, gen_W(seed, which, 20), 8);
      gen_put_le64(key + 8, gen_W(seed, which, 21), 2);
      return;
    }
    case GEN_SORTED:
      key[0] = 0;
      key[1] = 0;
      gen_put_be64(key + 2, i);
      return;
    case GEN_REVERSE:
      key[0] = 0xFF;
      key[1] = 0xFF;
      gen_put_be64(key + 2, ~i);
      return;
    case GEN_PREFIX2:
      gen_put_le64(key, gen_W(seed, i, 0), 8);
      gen_put_le64(key + 8, gen_W(seed, i, 1), 2);
      key[0] = 0xAB;
      key[1] = 0xCD;
      return;
    case GEN_BYTE9: {
      gen_put_le64(key, gen_W(seed, 0, 20), 8);
      key[8] = (uint8_t)gen_W(seed, 0, 21);
      key[9] = (uint8_t)gen_W(seed, i, 1);
      return;
    }
    case GEN_ASCII: {
      uint64_t a = gen_W(seed, i, 0), b = gen_W(seed, i, 1);
      for (int k = 0; k < 10; ++k) {
        uint64_t src = (k < 5) ? (a >> (12 * k)) : (b >> (12 * (k - 5)));
        key[k] = (uint8_t)(0x20 + (uint32_t)((src & 0xFFF) % 95));
      }
      return;
    }
    case GEN_TINY_ALPHABET: {
      uint64_t a = gen_W(seed, i, 0);
      for (int k = 0; k < 10; ++k) {
        uint32_t s = (uint32_t)((a >> (6 * k)) & 63) % 3;
        key[k] = (uint8_t)(s == 0 ? 0x00 : (s == 1 ? 0x01 : 0xFF));
      }
      return;
    }
    default: /* GEN_UNIFORM */
      gen_put_le64(key, gen_W(seed, i, 0), 8);
      gen_put_le64(key + 8, gen_W(seed, i, 1), 2);
      return;
  }
}

/* Full 100-byte record i. Payload bytes 10..99 = bytes 10..99 of the uniform stream of record i;
 * ASCII records (the paper's 20 GB set is ASCII) map every payload byte into 0x20..0x7E too and
 * end in CR LF, so the whole record is printable text. */
GEN_HD void gen_record(uint8_t rec[100], uint64_t seed, uint64_t i, int dist, const uint64_t* zt) {
  uint8_t tmp[104];
  for (int w = 0; w < 13; ++w) gen_put_le64(tmp + 8 * w, gen_W(seed, i, (uint32_t)w), 8);
  gen_key(tmp, seed, i, dist, zt);
  if (dist == GEN_ASCII) {
    for (int b = 10; b < 98; ++b) tmp[b] = (uint8_t)(0x20 + (((uint32_t)tmp[b] * 95u) >> 8));
    tmp[98] = '\r';
    tmp[99] = '\n';
  }
  for (int b = 0; b < 100; ++b) rec[b] = tmp[b];
}
