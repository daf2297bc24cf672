/*
 * cafs_oracle.c -- CPU restatement of the reference CAFS sort (int64/uint64 path).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels in paper_2605_25040_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path never calls it (there is no CPU fallback).
 *
 * Every function restates the algorithm of the reference Python/numba package
 * (paths relative to /root/reference/pkg/src/cafs):
 *   fast_hash            buckets.py:70-85   (multiplicative hash, top m bits)
 *   table_size_for       buckets.py:88-105
 *   is_monotone          sorter.py:115-129
 *   freqset / spectrum   cardinality.py:31-73, _kernels.py:131-153
 *   chao1                cardinality.py:85-96
 *   sample               cardinality.py:99-110
 *   dispatch             sorter.py:141-162
 *   tiny_counts          _kernels.py:156-169
 *   count_sequence       _kernels.py:25-81 (+ BucketTable, buckets.py:172-292)
 *   reconstruct          sorter.py:254-293 (guard, spill sort + fold, pair sort)
 *   radix_sort_pairs     _kernels.py:185-214
 *   emit_fill            _kernels.py:172-182
 *   cafs_sort            sorter.py:335-386
 *
 * Parity is pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py, run in the build container where the
 * reference is importable) -- see tests/test_oracle_golden.py.
 *
 * Keys are handled in the reference's unsigned domain: int64 inputs are
 * order-mapped by flipping bit 63 (sorter.py:84-94).  The fallback sort is the
 * reference's host comparison sort (sorter.py:132-138); the sorted output is a
 * unique function of the input multiset, so an LSD radix sort restates it.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "cafs_oracle.h"

#define SIGN64 0x8000000000000000ull

/* buckets.py:70-85 */
uint64_t orc_fast_hash(uint64_t x, int m_log2, uint64_t mult) {
  return (x * mult) >> (64 - m_log2);
}

static uint64_t bit_ceil_u64(uint64_t v) { /* buckets.py:88-89 */
  if (v <= 1) return 1;
  return 1ull << (64 - __builtin_clzll(v - 1));
}

/* buckets.py:92-105.  Returns 0 on invalid arguments (the reference raises). */
uint64_t orc_table_size_for(double k_hat, uint64_t n, int cap) {
  if (!(k_hat >= 1.0) || n < 1) return 0;
  if (cap != 4 && cap != 8) return 0;
  uint64_t m = bit_ceil_u64((uint64_t)ceil(8.0 * k_hat / (double)cap));
  uint64_t m2 = bit_ceil_u64((uint64_t)ceil((double)n / (double)cap));
  if (m2 < m) m = m2;
  if (m < 8) m = 8;
  return m;
}

/* cardinality.py:85-96.  u < 1 is rejected by the caller. */
double orc_chao1(int64_t u, int64_t f1, int64_t f2, uint64_t n, int saturated) {
  if (saturated) return (double)n;
  double k_hat = (double)u + (double)(f1 * f1) / (2.0 * (double)(f2 + 1));
  double dn = (double)n;
  return k_hat < dn ? k_hat : dn;
}

static inline uint64_t to_u(int64_t v, int is_signed) {
  return (uint64_t)v ^ (is_signed ? SIGN64 : 0ull);
}

/* sorter.py:115-129: non-decreasing check (chunking only changes speed). */
int orc_is_monotone(const int64_t* x, uint64_t n, int is_signed) {
  for (uint64_t i = 1; i < n; ++i)
    if (to_u(x[i], is_signed) < to_u(x[i - 1], is_signed)) return 0;
  return 1;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

/* cardinality.py:99-110 + _kernels.py:131-153 + cardinality.py:63-73 */
void orc_sample_estimate(const int64_t* x, uint64_t n, int is_signed, uint64_t mult,
                         orc_estimate_t* est) {
  enum { SLOTS = 4096, TARGET = 1024 };
  static __thread uint64_t keys[SLOTS];
  static __thread uint32_t ctr[SLOTS];
  memset(keys, 0, sizeof(keys));
  memset(ctr, 0, sizeof(ctr));
  uint64_t stride = n / TARGET;
  if (stride < 1) stride = 1;
  uint64_t limit = TARGET * stride;
  if (limit > n) limit = n;
  for (uint64_t i = 0; i < limit; i += stride) {
    uint64_t v = to_u(x[i], is_signed);
    uint64_t j = (v * mult) >> 52;
    for (;;) {
      if (ctr[j] == 0) { keys[j] = v; ctr[j] = 1; break; }
      if (keys[j] == v) { ctr[j]++; break; }
      j = (j + 1) & (SLOTS - 1);
    }
  }
  int64_t u = 0, f1 = 0, f2 = 0;
  int nk = 0;
  for (int j = 0; j < SLOTS; ++j) {
    if (ctr[j] > 0) {
      u++;
      if (nk < ORC_TINY_MAX) est->keys[nk] = keys[j];
      nk++;
    }
    if (ctr[j] == 1) f1++;
    if (ctr[j] == 2) f2++;
  }
  est->u = u;
  est->f1 = f1;
  est->f2 = f2;
  est->saturated = (u == TARGET);
  est->k_hat = u >= 1 ? orc_chao1(u, f1, f2, n, est->saturated) : 0.0;
  est->nkeys = nk <= ORC_TINY_MAX ? nk : 0;
  if (est->nkeys) qsort(est->keys, (size_t)est->nkeys, sizeof(uint64_t), cmp_u64);
}

/* sorter.py:141-162 (the caller handles n <= 1 as cafs_sort does, :353-355) */
void orc_dispatch(const int64_t* x, uint64_t n, int is_signed, uint64_t mult,
                  orc_decision_t* d) {
  memset(d, 0, sizeof(*d));
  if (orc_is_monotone(x, n, is_signed)) { d->route = ORC_ALREADY_SORTED; return; }
  if (n < ORC_SMALL_N_CUTOFF) { d->route = ORC_FALLBACK_SMALL_N; return; }
  orc_sample_estimate(x, n, is_signed, mult, &d->est);
  d->has_estimate = 1;
  if (d->est.k_hat <= 8.0 && d->est.u <= 8) { d->route = ORC_TINY_COUNT; return; }
  if (d->est.k_hat * 2.0 > (double)n) { d->route = ORC_FALLBACK_HIGH_ENTROPY; return; }
  d->route = ORC_MAIN;
}

/* _kernels.py:156-169 (keys in the unsigned domain, ascending) */
void orc_tiny_counts(const int64_t* x, uint64_t n, int is_signed, const uint64_t* keys,
                     int nk, int64_t* counts) {
  for (int j = 0; j < nk; ++j) counts[j] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t v = to_u(x[i], is_signed);
    for (int j = 0; j < nk; ++j) counts[j] += (v == keys[j]);
  }
}

/* LSD radix sort of u64 keys with an optional int64 payload; 8-bit digits,
 * stable, skipping digits that are constant over the array.  Restates
 * _kernels.py:185-214 (radix_sort_pairs) and stands in for np.sort. */
static void radix_u64(uint64_t* k, int64_t* v, uint64_t n) {
  if (n < 2) return;
  uint64_t* tk = (uint64_t*)malloc(n * sizeof(uint64_t));
  int64_t* tv = v ? (int64_t*)malloc(n * sizeof(int64_t)) : NULL;
  uint64_t* hist = (uint64_t*)calloc(8 * 256, sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i)
    for (int p = 0; p < 8; ++p) hist[p * 256 + ((k[i] >> (8 * p)) & 0xFF)]++;
  uint64_t *sk = k, *dk = tk;
  int64_t *sv = v, *dv = tv;
  for (int p = 0; p < 8; ++p) {
    uint64_t* h = hist + p * 256;
    int trivial = 0;
    for (int b = 0; b < 256; ++b) if (h[b] == n) trivial = 1;
    if (trivial) continue;
    uint64_t tot = 0;
    for (int b = 0; b < 256; ++b) { uint64_t c = h[b]; h[b] = tot; tot += c; }
    for (uint64_t i = 0; i < n; ++i) {
      uint64_t pos = h[(sk[i] >> (8 * p)) & 0xFF]++;
      dk[pos] = sk[i];
      if (v) dv[pos] = sv[i];
    }
    uint64_t* t = sk; sk = dk; dk = t;
    int64_t* t2 = sv; sv = dv; dv = t2;
  }
  if (sk != k) {
    memcpy(k, sk, n * sizeof(uint64_t));
    if (v) memcpy(v, sv, n * sizeof(int64_t));
  }
  free(tk); free(tv); free(hist);
}

/* sorter.py:132-138: the fallback engine, in place on the original array. */
void orc_fallback_sort(int64_t* x, uint64_t n, int is_signed) {
  uint64_t* u = (uint64_t*)x;
  if (is_signed) for (uint64_t i = 0; i < n; ++i) u[i] ^= SIGN64;
  radix_u64(u, NULL, n);
  if (is_signed) for (uint64_t i = 0; i < n; ++i) u[i] ^= SIGN64;
}

/* _kernels.py:25-81 with the table of buckets.py:172-192.  The spill buffer is
 * allocated at its final size n up front; the reference grows it on demand
 * (buckets.py:227-248), which changes nothing observable. */
typedef struct {
  int m_log2;
  uint64_t* keys;   /* [M][4] */
  uint32_t* counts; /* [M][4] */
  uint64_t* spill;
  uint64_t spill_len, updates, hits, claims, pushes;
} bucket_table_t;

static void count_sequence(bucket_table_t* t, const int64_t* x, uint64_t n, int is_signed,
                           uint64_t mult) {
  const int cap = 4;
  const int shift = 64 - t->m_log2;
  uint64_t i = 0;
  while (i < n) {
    uint64_t v = to_u(x[i], is_signed);
    uint64_t j = i + 1;
    while (j < n && to_u(x[j], is_signed) == v) j++;
    uint64_t inc = j - i;
    uint64_t h = (v * mult) >> shift;
    uint64_t* bk = t->keys + h * cap;
    uint32_t* bc = t->counts + h * cap;
    int placed = 0;
    for (int s = 0; s < cap; ++s) {
      if (bc[s] == 0) { bk[s] = v; bc[s] = (uint32_t)inc; t->claims++; placed = 1; break; }
      if (bk[s] == v) { bc[s] += (uint32_t)inc; t->hits++; placed = 1; break; }
    }
    if (!placed) {
      for (uint64_t q = 0; q < inc; ++q) t->spill[t->spill_len + q] = v;
      t->spill_len += inc;
      t->pushes++;
    }
    t->updates++;
    i = j;
  }
}

/* sorter.py:244-251 + _kernels.py:172-182 */
static void emit_fill(int64_t* out, const uint64_t* keys_u, const int64_t* counts, uint64_t k,
                      int is_signed) {
  uint64_t p = 0;
  for (uint64_t i = 0; i < k; ++i) {
    int64_t key = (int64_t)(keys_u[i] ^ (is_signed ? SIGN64 : 0ull));
    for (int64_t c = 0; c < counts[i]; ++c) out[p++] = key;
  }
}

/* sorter.py:183-196, 254-293, 317-332: count, guard, reconstruct, emit. */
static int run_main(int64_t* x, uint64_t n, int is_signed, double k_hat, uint64_t mult,
                    orc_telemetry_t* tel) {
  uint64_t m = orc_table_size_for(k_hat > 1.0 ? k_hat : 1.0, n, 4);
  bucket_table_t t;
  memset(&t, 0, sizeof(t));
  t.m_log2 = 63 - __builtin_clzll(m);
  t.keys = (uint64_t*)calloc(m * 4, sizeof(uint64_t));
  t.counts = (uint32_t*)calloc(m * 4, sizeof(uint32_t));
  t.spill = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!t.keys || !t.counts || !t.spill) return -1;
  count_sequence(&t, x, n, is_signed, mult);
  uint64_t counted = 0, occupied = 0;
  for (uint64_t i = 0; i < m * 4; ++i) { counted += t.counts[i]; occupied += t.counts[i] > 0; }
  tel->table_buckets = m;
  tel->counted_total = counted;
  tel->updates = t.updates;
  tel->hits = t.hits;
  tel->claims = t.claims;
  tel->spill_pushes = t.pushes;
  tel->spill_len = t.spill_len;
  if (t.spill_len * 2 > n) { /* guard, sorter.py:264-273 */
    tel->guard_fired = 1;
    orc_fallback_sort(x, n, is_signed);
  } else {
    /* spill: sort, fold (sorter.py:219-225), merge with occupied slots */
    radix_u64(t.spill, NULL, t.spill_len);
    uint64_t ns = 0;
    for (uint64_t i = 0; i < t.spill_len; ++i) ns += (i == 0 || t.spill[i] != t.spill[i - 1]);
    uint64_t kp = occupied + ns;
    uint64_t* pk = (uint64_t*)malloc((kp ? kp : 1) * sizeof(uint64_t));
    int64_t* pc = (int64_t*)malloc((kp ? kp : 1) * sizeof(int64_t));
    uint64_t q = 0;
    for (uint64_t i = 0; i < m * 4; ++i)
      if (t.counts[i] > 0) { pk[q] = t.keys[i]; pc[q] = t.counts[i]; q++; }
    for (uint64_t i = 0; i < t.spill_len; ++i) {
      if (i == 0 || t.spill[i] != t.spill[i - 1]) { pk[q] = t.spill[i]; pc[q] = 0; q++; }
      pc[q - 1]++;
    }
    radix_u64(pk, pc, kp); /* pair_sort, sorter.py:228-241 (distinct keys) */
    tel->pairs = kp;
    uint64_t total = 0;
    for (uint64_t i = 0; i < kp; ++i) total += (uint64_t)pc[i];
    if (total != n) { free(pk); free(pc); return -2; } /* emit's ValueError */
    emit_fill(x, pk, pc, kp, is_signed);
    free(pk); free(pc);
  }
  free(t.keys); free(t.counts); free(t.spill);
  return 0;
}

/* sorter.py:335-386 */
int orc_cafs_sort(int64_t* x, uint64_t n, int is_signed, uint64_t mult, orc_telemetry_t* tel) {
  memset(tel, 0, sizeof(*tel));
  tel->n = n;
  if (n <= 1) { tel->decision.route = ORC_ALREADY_SORTED; return 0; }
  orc_dispatch(x, n, is_signed, mult, &tel->decision);
  switch (tel->decision.route) {
    case ORC_ALREADY_SORTED:
      return 0;
    case ORC_FALLBACK_SMALL_N:
    case ORC_FALLBACK_HIGH_ENTROPY:
      orc_fallback_sort(x, n, is_signed);
      return 0;
    case ORC_TINY_COUNT: {
      int64_t counts[ORC_TINY_MAX];
      const orc_estimate_t* e = &tel->decision.est;
      orc_tiny_counts(x, n, is_signed, e->keys, e->nkeys, counts);
      int64_t sum = 0;
      for (int j = 0; j < e->nkeys; ++j) sum += counts[j];
      if ((uint64_t)sum == n) {
        tel->counted_total = n;
        tel->pairs = (uint64_t)e->nkeys;
        emit_fill(x, e->keys, counts, (uint64_t)e->nkeys, is_signed);
        return 0;
      }
      tel->tiny_count_failed = 1; /* sorter.py:378-385: MAIN with the same k_hat */
      tel->decision.route = ORC_MAIN;
      return run_main(x, n, is_signed, e->k_hat, mult, tel);
    }
    default:
      return run_main(x, n, is_signed, tel->decision.est.k_hat, mult, tel);
  }
}

/* ---- synthetic inputs (shared bit-for-bit with the device generator) ---- */

uint64_t orc_fmix64(uint64_t z) { /* datagen.py:32-35 finalizer */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* out[i] = fmix64(seed + (i + 1 + skip) * gamma)  (datagen.py:45-53) */
void orc_mix_outputs(uint64_t seed, uint64_t count, uint64_t skip, uint64_t* out) {
  for (uint64_t i = 0; i < count; ++i)
    out[i] = orc_fmix64(seed + (skip + i + 1) * 0x9E3779B97F4A7C15ull);
}

/* The config generator of oracle/gen.py (Config.generate) in C, for the CPU
 * baseline at full size (numpy takes ~2 min for 2^30 rows).  Rows
 * [start, start + n): uniform draws by multiply-high (cdf == NULL) or Zipf draws
 * by searchsorted(cdf, u, 'right') over k entries; palette == NULL means the
 * dictionary codes 0..k-1.  Bit-identical to gen.py (tests/test_oracle_golden.py). */
void orc_gen_draw(uint64_t seed, uint64_t n, uint64_t start, const int64_t* palette, uint64_t k,
                  const double* cdf, int64_t* out) {
  const uint64_t s = seed ^ 0xD1B54A32D192ED03ull;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t r = orc_fmix64(s + (start + i + 1) * 0x9E3779B97F4A7C15ull);
    uint64_t idx;
    if (!cdf) {
      const uint64_t hi = r >> 32, lo = r & 0xFFFFFFFFull;
      idx = (hi * k + ((lo * k) >> 32)) >> 32;
    } else {
      const double u = (double)(r >> 11) * (1.0 / 9007199254740992.0);
      uint64_t lo = 0, len = k; /* first j with cdf[j] > u */
      while (len > 0) {
        const uint64_t half = len >> 1;
        if (cdf[lo + half] <= u) { lo += half + 1; len -= half + 1; }
        else len = half;
      }
      idx = lo;
    }
    out[i] = palette ? palette[idx] : (int64_t)idx;
  }
}
