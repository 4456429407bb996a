/*
 * bsort_oracle.c — TEST INFRASTRUCTURE ONLY (see bsort_oracle.h).
 *
 * A plain, slow, obviously-correct single-threaded CPU bsort written from arxiv 2603.08929
 * (PAPER.md).  Each function cites the passage it follows.  No blocking, no fusion, no
 * reordering beyond the algorithms as printed, apart from the two readings listed in
 * DESIGN.md ("Readings of the paper"):
 *   Q1  the negative half of a float array is sorted with the inverted direction
 *       (prose P:431-432 "the sort direction for the exponents of negative numbers must be
 *       the inverse", and the Fig. 4 trace P:652-706; Algorithm 4 as printed passes
 *       `asc` to both halves, P:523-525 — kept as bo_bsort_float_literal for a test);
 *   Q2  recursion stops on ranges of size <= 1 (Algorithm 2 as printed recurses on every
 *       sub-range until the mask is 0, i.e. 2^w - 1 calls; pruning cannot change the output).
 * Ranges are half-open [ps, pe) with pe <= n (Q3, the paper's own calls pass |a|).
 */
#include "bsort_oracle.h"

#include <stdlib.h>
#include <string.h>

static uint64_t width_mask(int w) { return (w >= 64) ? ~(uint64_t)0 : (((uint64_t)1 << w) - 1); }

int bo_validate_scheme(const bo_scheme* s) {
  if (!s || s->width < 1 || s->width > 64) return -1;
  if (s->kind == BO_FLOAT) {
    /* sizeof = sizeof_mantissa + sizeof_exponent + 1 */
    if (s->exp_bits < 1 || s->mant_bits < 1) return -1;
    if (s->exp_bits + s->mant_bits + 1 != s->width) return -1;
  } else if (s->kind != BO_UNSIGNED && s->kind != BO_SIGNED) {
    return -1;
  }
  return 0;
}

static void note_level(bo_stats* st, int level, uint64_t count) {
  if (!st) return;
  if (level >= 1 && level <= 64) st->inspections_per_level[level - 1] += count;
  st->inspections += count;
  st->partition_calls += 1;
  if (level > st->max_depth) st->max_depth = level;
}

/* Algorithm 1 — singlePassBSort(a, m, ps, pe, asc).
 *   k := ps
 *   for i <- ps to pe:  if (asc and not(a_i AND m)) or (not asc and (a_i AND m)):
 *                           swap(a_i, a_k); k <- k + 1
 *   return k
 * `level` is only used for the SortStats counters (Theorem 4). */
uint64_t bo_single_pass(uint64_t* a, uint64_t m, uint64_t ps, uint64_t pe, int asc, bo_stats* st,
                        int level) {
  uint64_t k = ps;
  note_level(st, level, pe - ps);
  for (uint64_t i = ps; i < pe; ++i) {
    int bit_set = (a[i] & m) != 0;
    if ((asc && !bit_set) || (!asc && bit_set)) {
      uint64_t tmp = a[i];
      a[i] = a[k];
      a[k] = tmp;
      k = k + 1;
      if (st) st->swaps++;
    }
  }
  return k;
}

/* Algorithm 2 — binaryQuickSort(a, m, ps, pe, asc).
 *   k := singlePassBSort(a, m, ps, pe, asc); m' := m >> 1
 *   if m' = 0: return
 *   binaryQuickSort(a, m', ps, k, asc); binaryQuickSort(a, m', k, pe, asc)
 * plus reading Q2: a range of size <= 1 is already sorted. */
void bo_binary_quicksort(uint64_t* a, uint64_t m, uint64_t ps, uint64_t pe, int asc, bo_stats* st,
                         int level) {
  if (pe - ps <= 1 || m == 0) return; /* Q2 */
  uint64_t k = bo_single_pass(a, m, ps, pe, asc, st, level);
  uint64_t m1 = m >> 1; /* logical shift: masks live in unsigned words (Q5) */
  if (m1 == 0) return;
  bo_binary_quicksort(a, m1, ps, k, asc, st, level + 1);
  bo_binary_quicksort(a, m1, k, pe, asc, st, level + 1);
}

/* Unsigned keys: Algorithm 2 called directly with the MSB mask (m = 1 << (s-1)). */
int bo_bsort_unsigned(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st) {
  if (bo_validate_scheme(s) || s->kind != BO_UNSIGNED) return -1;
  uint64_t m = (uint64_t)1 << (s->width - 1);
  bo_binary_quicksort(a, m, 0, n, asc, st, 1);
  return 0;
}

/* Algorithm 3 — bsortSigned(a, asc).
 *   m := 1 << (sizeof(a_0) - 1); k := singlePassBSort(a, m, 0, |a|, not asc)
 *   m' := m >>> 1; binaryQuickSort(a, m', 0, k, asc); binaryQuickSort(a, m', k, |a|, asc) */
int bo_bsort_signed(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st) {
  if (bo_validate_scheme(s) || s->kind != BO_SIGNED) return -1;
  if (n <= 1) return 0; /* Q2 */
  uint64_t m = (uint64_t)1 << (s->width - 1);
  uint64_t k = bo_single_pass(a, m, 0, n, !asc, st, 1);
  uint64_t m1 = m >> 1;
  if (m1 == 0) return 0; /* 1-bit signed: the sign pass is the whole sort */
  bo_binary_quicksort(a, m1, 0, k, asc, st, 2);
  bo_binary_quicksort(a, m1, k, n, asc, st, 2);
  return 0;
}

/* Algorithm 5 — bsortF(a, m, ps, pe, asc).
 *   k := singlePassBSort(a, m, ps, pe, asc)
 *   if m = (1 << sizeof_mantissa(a_0)):          -- last exponent bit
 *       m' := m >>> 1; binaryQuickSort(a, m', ps, k, asc); binaryQuickSort(a, m', k, pe, asc)
 *       return
 *   m' := m >>> 1; bsortF(a, m', ps, k, asc); bsortF(a, m', k, pe, asc)
 * plus reading Q2. */
void bo_bsort_f(uint64_t* a, uint64_t m, uint64_t ps, uint64_t pe, int asc, const bo_scheme* s,
                bo_stats* st, int level) {
  if (pe - ps <= 1) return; /* Q2 */
  uint64_t k = bo_single_pass(a, m, ps, pe, asc, st, level);
  uint64_t m1 = m >> 1;
  if (m == ((uint64_t)1 << s->mant_bits)) {
    bo_binary_quicksort(a, m1, ps, k, asc, st, level + 1);
    bo_binary_quicksort(a, m1, k, pe, asc, st, level + 1);
    return;
  }
  bo_bsort_f(a, m1, ps, k, asc, s, st, level + 1);
  bo_bsort_f(a, m1, k, pe, asc, s, st, level + 1);
}

/* Algorithm 4 — bsortFloat(a, asc) with reading Q1.
 *   m := 1 << (sizeof(a_0) - 1); k := singlePassBSort(a, m, 0, |a|, not asc)    -- sign pass
 *   m' := m >>> 1; bsortF on both halves.
 * The sign pass with (not asc) puts the negative half first when asc, last when desc.  The
 * negative half gets the inverted direction ("the sort direction for the exponents of
 * negative numbers must be the inverse of the direction for positive numbers", "The
 * sort direction also depends on the sign"); the non-negative half keeps asc. */
int bo_bsort_float(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st) {
  if (bo_validate_scheme(s) || s->kind != BO_FLOAT) return -1;
  if (n <= 1) return 0; /* Q2 */
  uint64_t m = (uint64_t)1 << (s->width - 1);
  uint64_t k = bo_single_pass(a, m, 0, n, !asc, st, 1);
  uint64_t m1 = m >> 1;
  if (asc) {
    bo_bsort_f(a, m1, 0, k, !asc, s, st, 2); /* [0,k): sign bit set = negatives */
    bo_bsort_f(a, m1, k, n, asc, s, st, 2);  /* [k,n): non-negatives            */
  } else {
    bo_bsort_f(a, m1, 0, k, asc, s, st, 2);  /* [0,k): non-negatives            */
    bo_bsort_f(a, m1, k, n, !asc, s, st, 2); /* [k,n): negatives                */
  }
  return 0;
}

/* Algorithm 4 exactly as printed (bsortF(a, m', 0, k, asc); bsortF(a, m', k, |a|,
 * asc)).  Not part of R1; kept so tests can pin reading Q1 against Fig. 4. */
int bo_bsort_float_literal(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st) {
  if (bo_validate_scheme(s) || s->kind != BO_FLOAT) return -1;
  if (n <= 1) return 0;
  uint64_t m = (uint64_t)1 << (s->width - 1);
  uint64_t k = bo_single_pass(a, m, 0, n, !asc, st, 1);
  uint64_t m1 = m >> 1;
  bo_bsort_f(a, m1, 0, k, asc, s, st, 2);
  bo_bsort_f(a, m1, k, n, asc, s, st, 2);
  return 0;
}

int bo_bsort(uint64_t* a, uint64_t n, const bo_scheme* s, int asc, bo_stats* st) {
  if (bo_validate_scheme(s)) return -1;
  for (uint64_t i = 0; i < n; ++i)
    if (a[i] & ~width_mask(s->width)) return -1; /* words are zero-extended */
  switch (s->kind) {
    case BO_UNSIGNED: return bo_bsort_unsigned(a, n, s, asc, st);
    case BO_SIGNED: return bo_bsort_signed(a, n, s, asc, st);
    default: return bo_bsort_float(a, n, s, asc, st);
  }
}

/* ---------------------------------------------------------------- R2: plain definition */

/* total_order_key: Unsigned: identity.  Signed: flip the sign bit.
 * Float: if the sign bit is set complement all w bits, else set the sign bit. */
uint64_t bo_total_order_key(uint64_t word, const bo_scheme* s) {
  uint64_t wm = width_mask(s->width);
  uint64_t sign = (uint64_t)1 << (s->width - 1);
  word &= wm;
  switch (s->kind) {
    case BO_UNSIGNED: return word;
    case BO_SIGNED: return word ^ sign;
    default: return (word & sign) ? (~word & wm) : (word | sign);
  }
}

void bo_total_order_keys(const uint64_t* in, uint64_t* out, uint64_t n, const bo_scheme* s) {
  for (uint64_t i = 0; i < n; ++i) out[i] = bo_total_order_key(in[i], s);
}

typedef struct {
  uint64_t key;
  uint64_t word;
} bo_pair;

static int cmp_pair(const void* x, const void* y) {
  uint64_t a = ((const bo_pair*)x)->key, b = ((const bo_pair*)y)->key;
  return (a > b) - (a < b);
}

/* A comparison sort by total_order_key, reversed for descending.  The key is
 * injective on w-bit words, so the result does not depend on stability (Q12). */
int bo_sort_by_key(uint64_t* a, uint64_t n, const bo_scheme* s, int asc) {
  if (bo_validate_scheme(s)) return -1;
  if (n == 0) return 0;
  bo_pair* p = (bo_pair*)malloc(n * sizeof(bo_pair));
  if (!p) return -1;
  for (uint64_t i = 0; i < n; ++i) {
    p[i].word = a[i];
    p[i].key = bo_total_order_key(a[i], s);
  }
  qsort(p, n, sizeof(bo_pair), cmp_pair);
  for (uint64_t i = 0; i < n; ++i) a[i] = asc ? p[i].word : p[n - 1 - i].word;
  free(p);
  return 0;
}

/* ------------------------------------------------------------------------ brute force */

int64_t bo_bruteforce(const bo_scheme* s, int max_len, uint64_t* cases) {
  if (bo_validate_scheme(s) || s->width > 4 || max_len > 8) return -1;
  uint64_t base = (uint64_t)1 << s->width;
  int64_t bad = 0;
  uint64_t count = 0;
  uint64_t in[8], r1[8], r2[8];
  for (int len = 0; len <= max_len; ++len) {
    uint64_t total = 1;
    for (int i = 0; i < len; ++i) total *= base;
    for (uint64_t code = 0; code < total; ++code) {
      uint64_t c = code;
      for (int i = 0; i < len; ++i) {
        in[i] = c % base;
        c /= base;
      }
      for (int asc = 0; asc <= 1; ++asc) {
        memcpy(r1, in, sizeof(uint64_t) * (size_t)len);
        memcpy(r2, in, sizeof(uint64_t) * (size_t)len);
        bo_bsort(r1, (uint64_t)len, s, asc, NULL);
        bo_sort_by_key(r2, (uint64_t)len, s, asc);
        if (len && memcmp(r1, r2, sizeof(uint64_t) * (size_t)len) != 0) bad++;
        count++;
      }
    }
  }
  if (cases) *cases = count;
  return bad;
}
