/*
 * bsort_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU implementation of bsort (arxiv 2603.08929) written from
 * the paper's text.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (include/bsort.h,
 * paper_2603_08929_b200/) shares no code with it and never calls it.
 *
 * Representation: every key is a raw word of `width` bits, zero-extended
 * into a uint64_t.  Schemes: Unsigned(w), Signed(w) two's complement, Float(w, e, t) with
 * w = e + t + 1 and layout sign|exponent|mantissa, MSB = sign.
 *
 * R1  = the paper's Algorithms 1-5 with two readings
 *       recorded in DESIGN.md: Q1 (negative float half sorted with the inverted direction,
 *       P:431-432, Fig. 4) and Q2 (prune ranges of size <= 1; output unchanged).
 * R2  = the plain definition: sort by the order-preserving total-order key,
 *       reversed for descending.  R1 == R2 is itself a test.
 */
#ifndef BSORT_ORACLE_H
#define BSORT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { BO_UNSIGNED = 0, BO_SIGNED = 1, BO_FLOAT = 2 };

typedef struct {
  int kind;      /* BO_UNSIGNED / BO_SIGNED / BO_FLOAT                       */
  int width;     /* w, 1..64                                                 */
  int exp_bits;  /* e (Float only)                                           */
  int mant_bits; /* t (Float only), w = e + t + 1                    */
} bo_scheme;

/* SortStats: instrumentation for Theorem 4 / Theorem 5. */
typedef struct {
  uint64_t inspections_per_level[64]; /* level = recursion depth = bit index from the MSB */
  uint64_t inspections;               /* total element examinations                       */
  uint64_t swaps;
  uint64_t partition_calls;
  int max_depth;                      /* deepest level reached (1-based)                  */
} bo_stats;

/* Returns 0 on success, -1 on an invalid scheme / kind mismatch. `st` may be NULL. */
int bo_validate_scheme(const bo_scheme* s);

/* Algorithm 1, singlePassBSort, verbatim single forward scan with swaps. */
uint64_t bo_single_pass(uint64_t* a, uint64_t m, uint64_t ps, uint64_t pe, int asc,
                        bo_stats* st, int level);
/* Algorithm 2, binaryQuickSort + the Q2 size<=1 pruning. */
void bo_binary_quicksort(uint64_t* a, uint64_t m, uint64_t ps, uint64_t pe, int asc,
                         bo_stats* st, int level);
/* Typed entry points: unsigned, Algorithm 3, Algorithm 4 (Q1). */
int bo_bsort_unsigned(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st);
int bo_bsort_signed(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st);
int bo_bsort_float(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st);
/* Algorithm 4 exactly as printed (asc passed to both halves).  Exists only so a
 * test can show the literal reading fails the paper's own Fig. 4 (reading Q1). */
int bo_bsort_float_literal(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st);
/* Algorithm 5, bsortF. */
void bo_bsort_f(uint64_t* a, uint64_t m, uint64_t ps, uint64_t pe, int asc, const bo_scheme* s,
                bo_stats* st, int level);
/* Dispatch on s->kind: R1. */
int bo_bsort(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st);

/* R2: total-order key and a comparison sort on it. */
uint64_t bo_total_order_key(uint64_t word, const bo_scheme* s);
int bo_sort_by_key(uint64_t* a, uint64_t n, const bo_scheme* s, int asc);
/* Batch form of bo_total_order_key (out[i] = key(in[i])). */
void bo_total_order_keys(const uint64_t* in, uint64_t* out, uint64_t n, const bo_scheme* s);

/* Brute force: every array of length 0..max_len over all 2^w patterns, both directions,
 * R1 vs R2.  Returns the number of mismatching (array, direction) cases; *cases gets the
 * number checked.  Only for tiny w (<= 4). */
int64_t bo_bruteforce(const bo_scheme* s, int max_len, uint64_t* cases);

#ifdef __cplusplus
}
#endif
#endif
