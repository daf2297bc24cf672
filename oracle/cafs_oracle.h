/* cafs_oracle.h -- TEST INFRASTRUCTURE ONLY: the CPU restatement of the
 * reference CAFS sort used as the parity checker (see cafs_oracle.c). */
#ifndef CAFS_ORACLE_H
#define CAFS_ORACLE_H
#include <stdint.h>

#define ORC_TINY_MAX 8
#define ORC_SMALL_N_CUTOFF 2048

/* Route values match include/cafs_b200.h and the order of cafs.sorter.Route. */
enum {
  ORC_ALREADY_SORTED = 0,
  ORC_FALLBACK_SMALL_N = 1,
  ORC_TINY_COUNT = 2,
  ORC_FALLBACK_HIGH_ENTROPY = 3,
  ORC_MAIN = 4
};

typedef struct {
  double k_hat;
  int64_t u, f1, f2;
  int32_t saturated;
  int32_t nkeys;               /* sampled distinct keys when u <= 8, else 0 */
  uint64_t keys[ORC_TINY_MAX]; /* ascending, unsigned domain */
} orc_estimate_t;

typedef struct {
  int32_t route;
  int32_t has_estimate;
  orc_estimate_t est;
} orc_decision_t;

typedef struct {
  uint64_t n;
  orc_decision_t decision;
  uint64_t spill_len;
  int32_t guard_fired;
  int32_t tiny_count_failed;
  uint64_t counted_total;
  uint64_t updates, hits, claims, spill_pushes;
  uint64_t table_buckets;
  uint64_t pairs;
} orc_telemetry_t;

uint64_t orc_fast_hash(uint64_t x, int m_log2, uint64_t mult);
uint64_t orc_table_size_for(double k_hat, uint64_t n, int cap);
double orc_chao1(int64_t u, int64_t f1, int64_t f2, uint64_t n, int saturated);
int orc_is_monotone(const int64_t* x, uint64_t n, int is_signed);
void orc_sample_estimate(const int64_t* x, uint64_t n, int is_signed, uint64_t mult,
                         orc_estimate_t* est);
void orc_dispatch(const int64_t* x, uint64_t n, int is_signed, uint64_t mult, orc_decision_t* d);
void orc_tiny_counts(const int64_t* x, uint64_t n, int is_signed, const uint64_t* keys, int nk,
                     int64_t* counts);
void orc_fallback_sort(int64_t* x, uint64_t n, int is_signed);
int orc_cafs_sort(int64_t* x, uint64_t n, int is_signed, uint64_t mult, orc_telemetry_t* tel);
uint64_t orc_fmix64(uint64_t z);
void orc_mix_outputs(uint64_t seed, uint64_t count, uint64_t skip, uint64_t* out);
void orc_gen_draw(uint64_t seed, uint64_t n, uint64_t start, const int64_t* palette, uint64_t k,
                  const double* cdf, int64_t* out);

#endif
