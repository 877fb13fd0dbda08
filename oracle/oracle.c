/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle of the hybrid
 * sort's hot path (arXiv 2003.01216, "High Performance Parallel Sort for
 * Shared and Distributed Memory MIMD").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2003_01216_b200/), and neither side includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * "reading #k" = DESIGN.md §3 interpretation table.
 *
 * All keys are handled as int64_t (int32 callers widen first); the method is
 * integer-only, so there is no rounding anywhere.  Every function follows the
 * paper's order of steps; nothing is blocked, fused or reordered.
 *
 * Parity status: every function is pinned by tests/test_oracle.py (worked
 * examples, closed forms, brute force, library special cases).  No function
 * is "parity unpinned".
 *
 * Built twice from this one file: liboracle.so (plain, single thread; the
 * oracle proper) and liboracle_omp.so (-fopenmp; the OpenMP pragmas below run
 * chunks / merge pairs concurrently, the paper's own shared-memory scheme
 * P:58-62, for the timing baseline only -- the output is identical).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_ERR_KEY_OUT_OF_RANGE 1
#define ORACLE_ERR_BAD_DIGITS 2
#define ORACLE_ERR_NOT_POW2 3
#define ORACLE_ERR_NOMEM 4

/* 10^e for 0 <= e <= 18, by repeated multiplication. */
static int64_t pow10_i64(int e) {
    int64_t r = 1;
    for (int i = 0; i < e; i++) r *= 10;
    return r;
}

static int is_pow2(int64_t p) { return p >= 1 && (p & (p - 1)) == 0; }

/* ------------------------------------------------------------------ a1 ---
 * Leading decimal digit of a D-digit key ("divides the data into ten
 * parts based on the most significant digit"; S:290-298 msd_bucket_index):
 *   d(k) = floor(k / 10^(D-1)).
 * Keys with fewer than D digits are zero-padded -> bucket 0 (reading #1).
 * Keys outside [0, 10^D) are clamped to bucket 0 / 9 (reading #3); in strict
 * mode they are an error (S:294 KeyOutOfRange).
 * D is in [1, 19] (int64) -- the caller checks the per-dtype limit.        */
int oracle_digit(int64_t key, int num_digits, int strict, int *digit) {
    if (num_digits < 1 || num_digits > 19) return ORACLE_ERR_BAD_DIGITS;
    int64_t div = pow10_i64(num_digits - 1);
    if (key < 0) {
        if (strict) return ORACLE_ERR_KEY_OUT_OF_RANGE;
        *digit = 0;
        return ORACLE_OK;
    }
    int64_t q = key / div; /* C integer division: floor for key >= 0 */
    if (q > 9) {
        if (strict) return ORACLE_ERR_KEY_OUT_OF_RANGE;
        q = 9;
    }
    *digit = (int)q;
    return ORACLE_OK;
}

/* ---------------------------------------------------------- a1, a2, a3 ---
 * One-step MSD radix partition into ten buckets:
 *   1. d_i for every key; cnt[d]++                       (histogram)
 *   2. off[0] = 0, off[b+1] = off[b] + cnt[b]            (exclusive prefix)
 *   3. pos = off; for i in input order: out[pos[d_i]++] = k_i
 *      (single stable counting pass; reading #4)
 * Buckets are in ascending digit order (reading #5).  out must not alias keys.
 * On a strict-mode error *bad_index receives the first offending index and
 * nothing is written.                                                      */
int oracle_msd_partition(const int64_t *keys, int64_t n, int num_digits, int strict,
                         int64_t *offsets11, int64_t *out, int64_t *bad_index) {
    int64_t cnt[10] = {0};
    int d;
    if (num_digits < 1 || num_digits > 19) return ORACLE_ERR_BAD_DIGITS;
    for (int64_t i = 0; i < n; i++) {
        int rc = oracle_digit(keys[i], num_digits, strict, &d);
        if (rc != ORACLE_OK) {
            if (bad_index) *bad_index = i;
            return rc;
        }
        cnt[d]++;
    }
    offsets11[0] = 0;
    for (int b = 0; b < 10; b++) offsets11[b + 1] = offsets11[b] + cnt[b];
    int64_t pos[10];
    for (int b = 0; b < 10; b++) pos[b] = offsets11[b];
    for (int64_t i = 0; i < n; i++) {
        oracle_digit(keys[i], num_digits, 0, &d);
        out[pos[d]++] = keys[i];
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------ a4 ---
 * Even split of m items among p (power of two) threads ("The data is
 * divided among parallel threads"; "the number of threads should be a
 * power of two"; rule S:135-143): the first (m mod p) parts get ceil(m/p),
 * the rest floor(m/p).                                                     */
int oracle_partition_even(int64_t m, int64_t p, int64_t *lens) {
    if (!is_pow2(p)) return ORACLE_ERR_NOT_POW2;
    int64_t q = m / p, r = m % p;
    for (int64_t i = 0; i < p; i++) lens[i] = q + (i < r ? 1 : 0);
    return ORACLE_OK;
}

/* ------------------------------------------------------------------ a6 ---
 * Binary-tree merge schedule ("threads sort and merge two children
 * sorted lists (its list and its neighbor's list) in a binary tree fashion
 * ... repeated using half of available threads in each round"):
 * round r = 1..log2 p: active i with i mod 2^r == 0 absorbs i + 2^(r-1).
 * Writes (round, active, partner) triples; returns the number of pairs.    */
int64_t oracle_merge_schedule(int64_t p, int64_t *triples) {
    if (!is_pow2(p)) return -1;
    int64_t k = 0;
    for (int64_t r = 1; ((int64_t)1 << r) <= p; r++) {
        int64_t step = (int64_t)1 << r, half = step >> 1;
        for (int64_t i = 0; i < p; i++) {
            if (i % step == 0) {
                if (triples) {
                    triples[3 * k + 0] = r;
                    triples[3 * k + 1] = i;
                    triples[3 * k + 2] = i + half;
                }
                k++;
            }
        }
    }
    return k;
}

/* ------------------------------------------------------------------ a5 ---
 * Sequential recursive quicksort, ascending (Fig 1c; "choose an
 * element as a pivot ..."; reading #8: smaller keys to the LEFT, return on
 * ranges of <= 1 element).  Pivot = median of (first, middle, last)
 * (S:90); Hoare partition that stops on keys equal to the pivot; recurse on
 * the smaller side and loop on the larger, so depth is O(log n).
 * Sorts a[lo..hi] inclusive.                                               */
static void swap64(int64_t *a, int64_t *b) {
    int64_t t = *a;
    *a = *b;
    *b = t;
}

static void quicksort_range(int64_t *a, int64_t lo, int64_t hi) {
    while (hi - lo >= 1) { /* at least two elements */
        int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < a[lo]) swap64(&a[mid], &a[lo]);
        if (a[hi] < a[lo]) swap64(&a[hi], &a[lo]);
        if (a[hi] < a[mid]) swap64(&a[hi], &a[mid]);
        int64_t v = a[mid]; /* median of three */
        int64_t i = lo - 1, j = hi + 1;
        for (;;) {
            do i++; while (a[i] < v);
            do j--; while (a[j] > v);
            if (i >= j) break;
            swap64(&a[i], &a[j]);
        }
        /* S_1 = a[lo..j] <= v <= S_2 = a[j+1..hi] */
        if (j - lo < hi - j) {
            quicksort_range(a, lo, j);
            lo = j + 1;
        } else {
            quicksort_range(a, j + 1, hi);
            hi = j;
        }
    }
}

void oracle_quicksort(int64_t *a, int64_t n) {
    if (n > 1) quicksort_range(a, 0, n - 1);
}

/* Merge of two sorted lists (Fig 1a step d, "merge(S, low, high,
 * mid)"): stable-left -- on equal keys the left element goes first.
 * out must hold nl + nr keys and must not alias the inputs.               */
void oracle_merge_runs(const int64_t *left, int64_t nl, const int64_t *right, int64_t nr, int64_t *out) {
    int64_t i = 0, j = 0, k = 0;
    while (i < nl && j < nr) {
        if (right[j] < left[i]) out[k++] = right[j++];
        else out[k++] = left[i++];
    }
    while (i < nl) out[k++] = left[i++];
    while (j < nr) out[k++] = right[j++];
}

/* Chunk starts of bucket [base, base+m) split into c chunks: starts[0..c]. */
static void chunk_starts(int64_t base, int64_t m, int64_t c, int64_t *lens, int64_t *starts) {
    oracle_partition_even(m, c, lens);
    starts[0] = base;
    for (int64_t i = 0; i < c; i++) starts[i + 1] = starts[i] + lens[i];
}

/* ------------------------------------------------------------------ a5 ---
 * Sort every chunk of every bucket (§3.2 Shared-Parallel Hybrid, phase 1,
 * "sequential recursive Quicksort is used to sort the data assigned to
 * each parallel thread").  Chunks = partition_even(m_b, c) of each
 * bucket (a4).  out may equal in.                                          */
int oracle_sort_chunks(const int64_t *in, int64_t *out, int64_t n, const int64_t *offsets11, int64_t c) {
    if (!is_pow2(c)) return ORACLE_ERR_NOT_POW2;
    if (out != in) memmove(out, in, (size_t)n * sizeof(int64_t));
    int64_t *lens = (int64_t *)malloc((size_t)c * sizeof(int64_t));
    int64_t *starts = (int64_t *)malloc((size_t)(c + 1) * sizeof(int64_t));
    if (!lens || !starts) {
        free(lens);
        free(starts);
        return ORACLE_ERR_NOMEM;
    }
    for (int b = 0; b < 10; b++) {
        chunk_starts(offsets11[b], offsets11[b + 1] - offsets11[b], c, lens, starts);
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t t = 0; t < c; t++) oracle_quicksort(out + starts[t], starts[t + 1] - starts[t]);
    }
    free(lens);
    free(starts);
    return ORACLE_OK;
}

/* ------------------------------------------------------------------ a6 ---
 * Tree merge of the c sorted chunks of every bucket (§3.2 phase 2, P:58-60;
 * S:144-152 schedule, S:46-54 merge).  Round r: worker i (i mod 2^r == 0)
 * merges its run [chunk i, chunk i+2^(r-1)) with its neighbour's run
 * [chunk i+2^(r-1), chunk i+2^r) through a full auxiliary buffer and
 * owns the result.  Buckets never merge with each other: they are
 * range-disjoint.  out may equal in.                          */
int oracle_merge(const int64_t *in, int64_t *out, int64_t n, const int64_t *offsets11, int64_t c) {
    if (!is_pow2(c)) return ORACLE_ERR_NOT_POW2;
    if (out != in) memmove(out, in, (size_t)n * sizeof(int64_t));
    int64_t npairs = oracle_merge_schedule(c, NULL);
    int64_t *sched = (int64_t *)malloc((size_t)(3 * npairs + 1) * sizeof(int64_t));
    int64_t *lens = (int64_t *)malloc((size_t)c * sizeof(int64_t));
    int64_t *starts = (int64_t *)malloc((size_t)(c + 1) * sizeof(int64_t));
    int64_t *aux = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!sched || !lens || !starts || !aux) {
        free(sched);
        free(lens);
        free(starts);
        free(aux);
        return ORACLE_ERR_NOMEM;
    }
    oracle_merge_schedule(c, sched);
    for (int b = 0; b < 10; b++) {
        chunk_starts(offsets11[b], offsets11[b + 1] - offsets11[b], c, lens, starts);
        int64_t k = 0;
        while (k < npairs) {
            int64_t r = sched[3 * k];
            int64_t k_end = k;
            while (k_end < npairs && sched[3 * k_end] == r) k_end++;
            int64_t half = (int64_t)1 << (r - 1);
            /* all pairs of one round run concurrently; a barrier separates rounds */
#pragma omp parallel for schedule(dynamic, 1)
            for (int64_t q = k; q < k_end; q++) {
                int64_t i = sched[3 * q + 1], partner = sched[3 * q + 2];
                int64_t lo = starts[i], mid = starts[partner], hi = starts[partner + half];
                oracle_merge_runs(out + lo, mid - lo, out + mid, hi - mid, aux + lo);
                memcpy(out + lo, aux + lo, (size_t)(hi - lo) * sizeof(int64_t));
            }
            k = k_end;
        }
    }
    free(sched);
    free(lens);
    free(starts);
    free(aux);
    return ORACLE_OK;
}

/* ----------------------------------------------------------- a1 .. a7 ---
 * Whole path, in place (§3.4, Fig 4, with one node: S:326-334):
 * MSD partition into ten buckets -> quicksort each chunk of each bucket ->
 * tree-merge each bucket's chunks; buckets sit at their offsets, so the
 * result is already "in its place in the original array".          */
int oracle_sort(int64_t *keys, int64_t n, int num_digits, int64_t c, int strict, int64_t *bad_index) {
    if (!is_pow2(c)) return ORACLE_ERR_NOT_POW2;
    int64_t off[11];
    int64_t *tmp = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!tmp) return ORACLE_ERR_NOMEM;
    int rc = oracle_msd_partition(keys, n, num_digits, strict, off, tmp, bad_index);
    if (rc == ORACLE_OK) rc = oracle_sort_chunks(tmp, tmp, n, off, c);
    if (rc == ORACLE_OK) rc = oracle_merge(tmp, keys, n, off, c);
    free(tmp);
    return rc;
}

/* ----------------------------------------------------------- f1 -------
 * No-MSD ablation: the Shared-Parallel Hybrid Quicksort +
 * Merge Sort of §3.2 on the whole array: the data is
 * divided among c threads (partition_even, P:58 / S:138), each part is
 * quicksorted (Fig 1c), then the parts are merged in a binary tree.
 * Written as the one-segment case of the bucket routines above: a single
 * "bucket" [0, n) (offsets 0, n, n, ..., n).                              */
int oracle_sort_shared(int64_t *keys, int64_t n, int64_t c) {
    if (!is_pow2(c)) return ORACLE_ERR_NOT_POW2;
    int64_t off[11];
    off[0] = 0;
    for (int b = 1; b < 11; ++b) off[b] = n;
    int rc = oracle_sort_chunks(keys, keys, n, off, c);
    if (rc == ORACLE_OK) rc = oracle_merge(keys, keys, n, off, c);
    return rc;
}

/* ----------------------------------------------------------- f3 -------
 * Key + tag items (SPEC SortItem S:31-37: the tag never
 * influences order), sorted STABLY: equal keys keep their input order.  The
 * steps are the paper's, each in its stable form:
 *   a1-a3  the MSD counting scatter (already stable), moving tags too;
 *   a5     each chunk is sorted by the NON-recursive merge sort of Fig 1b
 *          ("sort pairs, then repeatedly merge adjacent sorted
 *          lists") -- the paper's stable sequential sort, used here
 *          instead of quicksort (Fig 1c), which is not stable;
 *   a6     the binary-tree merge of the chunks, stable-left.
 * Keys are int64 (int32 callers widen), tags uint64.                      */
static void merge_items(const int64_t *kl, const uint64_t *tl, int64_t nl, const int64_t *kr, const uint64_t *tr,
                        int64_t nr, int64_t *ko, uint64_t *to) {
    int64_t i = 0, j = 0, k = 0;
    while (i < nl && j < nr) {
        if (kr[j] < kl[i]) { ko[k] = kr[j]; to[k++] = tr[j++]; }
        else { ko[k] = kl[i]; to[k++] = tl[i++]; }
    }
    while (i < nl) { ko[k] = kl[i]; to[k++] = tl[i++]; }
    while (j < nr) { ko[k] = kr[j]; to[k++] = tr[j++]; }
}

/* Fig 1b: bottom-up merge sort of a[0..n) with tags, widths 1, 2, 4, ... */
static void mergesort_items(int64_t *k, uint64_t *t, int64_t n, int64_t *kb, uint64_t *tb) {
    for (int64_t w = 1; w < n; w *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * w) {
            int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            merge_items(k + lo, t + lo, mid - lo, k + mid, t + mid, hi - mid, kb + lo, tb + lo);
        }
        memcpy(k, kb, (size_t)n * sizeof(int64_t));
        memcpy(t, tb, (size_t)n * sizeof(uint64_t));
    }
}

int oracle_msd_partition_pairs(const int64_t *keys, const uint64_t *tags, int64_t n, int num_digits,
                               int64_t *offsets11, int64_t *out_keys, uint64_t *out_tags) {
    int64_t cnt[10] = {0};
    int d;
    if (num_digits < 1 || num_digits > 19) return ORACLE_ERR_BAD_DIGITS;
    for (int64_t i = 0; i < n; i++) {
        oracle_digit(keys[i], num_digits, 0, &d);
        cnt[d]++;
    }
    offsets11[0] = 0;
    for (int b = 0; b < 10; b++) offsets11[b + 1] = offsets11[b] + cnt[b];
    int64_t pos[10];
    for (int b = 0; b < 10; b++) pos[b] = offsets11[b];
    for (int64_t i = 0; i < n; i++) {
        oracle_digit(keys[i], num_digits, 0, &d);
        out_keys[pos[d]] = keys[i];
        out_tags[pos[d]++] = tags[i];
    }
    return ORACLE_OK;
}

int oracle_sort_pairs(int64_t *keys, uint64_t *tags, int64_t n, int num_digits, int64_t c) {
    if (!is_pow2(c)) return ORACLE_ERR_NOT_POW2;
    size_t nn = (size_t)(n > 0 ? n : 1);
    int64_t *k1 = (int64_t *)malloc(nn * sizeof(int64_t)), *k2 = (int64_t *)malloc(nn * sizeof(int64_t));
    uint64_t *t1 = (uint64_t *)malloc(nn * sizeof(uint64_t)), *t2 = (uint64_t *)malloc(nn * sizeof(uint64_t));
    int64_t *lens = (int64_t *)malloc((size_t)c * sizeof(int64_t)), *starts = (int64_t *)malloc((size_t)(c + 1) * sizeof(int64_t));
    int64_t *sched = (int64_t *)malloc((size_t)(3 * c + 3) * sizeof(int64_t));
    int rc = ORACLE_OK;
    if (!k1 || !k2 || !t1 || !t2 || !lens || !starts || !sched) rc = ORACLE_ERR_NOMEM;
    int64_t off[11];
    if (rc == ORACLE_OK) rc = oracle_msd_partition_pairs(keys, tags, n, num_digits, off, k1, t1);
    for (int b = 0; rc == ORACLE_OK && b < 10; b++) {
        chunk_starts(off[b], off[b + 1] - off[b], c, lens, starts);
        for (int64_t i = 0; i < c; i++)   /* a5: stable sort of every chunk */
            mergesort_items(k1 + starts[i], t1 + starts[i], lens[i], k2 + starts[i], t2 + starts[i]);
        /* a6: round r merges chunk runs [i, i+2^(r-1)) and [i+2^(r-1), i+2^r) */
        for (int64_t w = 1; w < c; w *= 2) {
            for (int64_t i = 0; i < c; i += 2 * w) {
                int64_t lo = starts[i], mid = starts[i + w], hi = starts[i + 2 * w];
                merge_items(k1 + lo, t1 + lo, mid - lo, k1 + mid, t1 + mid, hi - mid, k2 + lo, t2 + lo);
                memcpy(k1 + lo, k2 + lo, (size_t)(hi - lo) * sizeof(int64_t));
                memcpy(t1 + lo, t2 + lo, (size_t)(hi - lo) * sizeof(uint64_t));
            }
        }
    }
    if (rc == ORACLE_OK) {
        memcpy(keys, k1, (size_t)n * sizeof(int64_t));
        memcpy(tags, t1, (size_t)n * sizeof(uint64_t));
    }
    free(k1); free(k2); free(t1); free(t2); free(lens); free(starts); free(sched);
    return rc;
}

/* f3 phases as separate calls (the item forms of oracle_sort_chunks /
 * oracle_merge): a5 -- every chunk (partition_even of each bucket of the
 * given offsets) sorted by Fig 1b's non-recursive merge sort (stable);
 * a6 -- the binary-tree merge of each bucket's chunk runs, round r merging
 * runs [i, i+2^(r-1)) and [i+2^(r-1), i+2^r), stable-left.
 * In place on keys / tags.                                                */
int oracle_sort_chunks_pairs(int64_t *keys, uint64_t *tags, int64_t n, const int64_t *offsets11, int64_t c) {
    if (!is_pow2(c)) return ORACLE_ERR_NOT_POW2;
    size_t nn = (size_t)(n > 0 ? n : 1);
    int64_t *kb = (int64_t *)malloc(nn * sizeof(int64_t));
    uint64_t *tb = (uint64_t *)malloc(nn * sizeof(uint64_t));
    int64_t *lens = (int64_t *)malloc((size_t)c * sizeof(int64_t)), *starts = (int64_t *)malloc((size_t)(c + 1) * sizeof(int64_t));
    int rc = (kb && tb && lens && starts) ? ORACLE_OK : ORACLE_ERR_NOMEM;
    for (int b = 0; rc == ORACLE_OK && b < 10; b++) {
        chunk_starts(offsets11[b], offsets11[b + 1] - offsets11[b], c, lens, starts);
        for (int64_t i = 0; i < c; i++)
            mergesort_items(keys + starts[i], tags + starts[i], lens[i], kb + starts[i], tb + starts[i]);
    }
    free(kb); free(tb); free(lens); free(starts);
    return rc;
}

int oracle_merge_pairs(int64_t *keys, uint64_t *tags, int64_t n, const int64_t *offsets11, int64_t c) {
    if (!is_pow2(c)) return ORACLE_ERR_NOT_POW2;
    size_t nn = (size_t)(n > 0 ? n : 1);
    int64_t *kb = (int64_t *)malloc(nn * sizeof(int64_t));
    uint64_t *tb = (uint64_t *)malloc(nn * sizeof(uint64_t));
    int64_t *lens = (int64_t *)malloc((size_t)c * sizeof(int64_t)), *starts = (int64_t *)malloc((size_t)(c + 1) * sizeof(int64_t));
    int rc = (kb && tb && lens && starts) ? ORACLE_OK : ORACLE_ERR_NOMEM;
    for (int b = 0; rc == ORACLE_OK && b < 10; b++) {
        chunk_starts(offsets11[b], offsets11[b + 1] - offsets11[b], c, lens, starts);
        for (int64_t w = 1; w < c; w *= 2) {
            for (int64_t i = 0; i < c; i += 2 * w) {
                int64_t lo = starts[i], mid = starts[i + w], hi = starts[i + 2 * w];
                merge_items(keys + lo, tags + lo, mid - lo, keys + mid, tags + mid, hi - mid, kb + lo, tb + lo);
                memcpy(keys + lo, kb + lo, (size_t)(hi - lo) * sizeof(int64_t));
                memcpy(tags + lo, tb + lo, (size_t)(hi - lo) * sizeof(uint64_t));
            }
        }
    }
    free(kb); free(tb); free(lens); free(starts);
    return rc;
}

/* Reports whether this build runs the OpenMP pragmas (timing build). */
int oracle_openmp_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
