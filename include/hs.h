/*
 * hs.h -- C ABI of libhybridsort.so: the data-parallel hot path of the hybrid
 * MSD-radix / quicksort / merge sort of Alghamdi & Alaghband, "High
 * Performance Parallel Sort for Shared and Distributed Memory MIMD"
 * (arXiv 2003.01216), re-designed for one NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = the paper's text (PAPER.md line n); S:n = SPEC.md line n;
 * "reading #k" = DESIGN.md §3, the interpretation table for passages the paper
 * leaves open.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Keys are signed integers, HS_INT32 (4 B) or HS_INT64 (8 B), sorted in
 *    ascending order.  Key arrays are contiguous, naturally aligned and may
 *    start at any element offset.
 *  - Every pointer argument is DEVICE memory owned by the caller.  The
 *    library never frees, retains or reallocates it.  It may READ (never
 *    write) up to 15 bytes before the start or past the end of a key array,
 *    inside the same 16-byte-aligned granule (bulk-copy alignment); such
 *    bytes never affect a result.
 *  - Calls are asynchronous: they validate their arguments on the host,
 *    enqueue kernels on `stream` (NULL = the legacy default stream) of the
 *    current device, and return.  No call synchronises the host, so a whole
 *    call can be captured in a CUDA graph.  Scratch (one n-key ping-pong
 *    buffer, lookback status words, plan and co-rank tables, and for
 *    hs_sort / hs_sort_buckets / hs_sort_pairs on chunks larger than one
 *    tile the K5a split table plus the padded-layout buffer of about
 *    1.11 n + 10 c T keys) is taken with stream-ordered
 *    cudaMallocAsync/cudaFreeAsync from the device's default memory pool,
 *    whose release threshold the library raises so repeated calls do not
 *    remap memory.  Under CUDA-graph capture, hs_sort puts the merge levels
 *    past the log2 c tree rounds behind a conditional graph node that the
 *    device plan opens (their body is captured on a per-thread side stream
 *    the first uncaptured call on that thread creates; without one they
 *    are captured as plain launches).
 *  - Calls are reentrant and may run concurrently on distinct streams over
 *    distinct buffers.
 *  - Validation happens before any launch; on an error nothing is enqueued and
 *    no output is touched.  Asynchronous device faults surface at the
 *    caller's next synchronisation, as with any CUDA call.
 *  - n must satisfy 0 <= n < 2^31 (ABI v1 limit).
 *
 * Bucket layout (CSR)
 * -------------------
 *  bucket_offsets is a device int64[11]: bucket b (leading decimal digit b)
 *  occupies [bucket_offsets[b], bucket_offsets[b+1]); [0] = 0, [10] = n.
 *  The leading digit of a key k with D = num_digits decimal digits is
 *      d(k) = clamp(floor(k / 10^(D-1)), 0, 9)
 *  ("divides the data into ten parts based on the most significant
 *  digit"; keys with fewer than D digits are zero-padded, reading #1; keys
 *  < 0 or >= 10^D are clamped to bucket 0 / 9, which preserves order, so
 *  hs_sort sorts ANY int32/int64 input correctly, reading #3).
 *  num_digits is in [1, 10] for HS_INT32 and [1, 19] for HS_INT64.
 *
 * Chunks
 * ------
 *  Bucket b of m_b keys is split into c = chunks_per_bucket contiguous chunks
 *  by partition_even: the first (m_b mod c) chunks hold ceil(m_b/c) keys, the
 *  rest floor(m_b/c) ("The data is divided among parallel threads";
 *  rule S:135-143; reading #7).  c must be a power of two in [1, 65536]
 *  ("the number of threads should be a power of two").
 */
#ifndef HS_H_
#define HS_H_

#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_ABI_VERSION 1

typedef enum { HS_INT32 = 0, HS_INT64 = 1 } hs_dtype_t;

typedef enum {
    HS_OK = 0,
    HS_ERR_INVALID_VALUE = 1,     /* bad size, NULL pointer, D, c, overlap, misalignment */
    HS_ERR_UNSUPPORTED_DTYPE = 2, /* dtype outside hs_dtype_t */
    HS_ERR_OUT_OF_MEMORY = 3,     /* cudaMallocAsync of the scratch failed */
    HS_ERR_CUDA = 4               /* a CUDA runtime call or launch failed */
} hs_status_t;

/*
 * a1-a3: stable one-step MSD radix partition into ten buckets
 * (§3.4: "implemented one step of MSD-Radix algorithm at the
 * beginning of the algorithm.  The master node divides the data into ten
 * parts based on the most significant digit"; stable counting pass S:302,
 * reading #4; buckets in ascending digit order, reading #5).
 *
 *   keys[n]            in : device, not modified.
 *   out[n]             out: device; keys regrouped by leading digit, keeping
 *                           input order inside each bucket.  Must not overlap
 *                           keys (HS_ERR_INVALID_VALUE).
 *   bucket_offsets[11] out: device int64, CSR offsets (above).  Always
 *                           required, also for n = 0 (then all zero).
 *
 * Result is unique, hence bit-exact against any correct implementation.
 */
hs_status_t hs_msd_partition(const void *keys, int64_t n, hs_dtype_t dtype, int num_digits,
                             int64_t *bucket_offsets, void *out, cudaStream_t stream);

/*
 * a4-a5: sort every chunk of every bucket ascending (§3.2 Shared-Parallel
 * Hybrid Quicksort and Merge Sort, phase 1: "sequential recursive
 * Quicksort is used to sort the data assigned to each parallel thread").
 * On the GPU the per-chunk sort is a shared-memory tile sort plus merge-path
 * merge levels inside the chunk; the result is the same unique array.
 *
 *   in[n], out[n]      device; in may equal out (in place); any other overlap
 *                      is HS_ERR_INVALID_VALUE.  in is read-only unless
 *                      in == out.
 *   bucket_offsets[11] in : device int64 CSR offsets (as hs_msd_partition
 *                      writes them).  Must be non-decreasing with [0] = 0 and
 *                      [10] = n; this is NOT checked (it lives on the device).
 *   chunks_per_bucket  c, power of two in [1, 65536].
 */
hs_status_t hs_sort_chunks(const void *in, void *out, int64_t n, hs_dtype_t dtype,
                           const int64_t *bucket_offsets, int chunks_per_bucket, cudaStream_t stream);

/*
 * a6: binary-tree merge of each bucket's c sorted chunks (§3.2 phase 2,
 * "threads sort and merge two children sorted lists (its list and
 * its neighbor's list) in a binary tree fashion.  This step is repeated using
 * half of available threads in each round"; schedule S:144-152: round r
 * merges chunk runs [i, i+2^(r-1)) and [i+2^(r-1), i+2^r) for i mod 2^r = 0).
 * Buckets are range-disjoint, so no bucket merges with another.
 * On the GPU every pair of a round is merged at once by merge-path (co-rank)
 * partitioned CTAs; ties take the left run first (stable-left).
 *
 *   in[n], out[n]      device; in may equal out.  Each chunk of in (chunk
 *                      bounds as above) must be sorted; NOT checked.
 *   bucket_offsets[11], chunks_per_bucket: as hs_sort_chunks.
 * With c = 1 there are no rounds: out = in.
 */
hs_status_t hs_merge(const void *in, void *out, int64_t n, hs_dtype_t dtype,
                     const int64_t *bucket_offsets, int chunks_per_bucket, cudaStream_t stream);

/*
 * a1-a7: the whole path, in place (§3.4 Fig 4, P:76-84 with one node,
 * S:326-334): MSD partition -> sort each chunk -> tree-merge each bucket's
 * chunks.  Buckets land "to its place in the original array" because
 * each bucket's last merge level writes straight into keys.
 * Sorting a chunk larger than one tile starts with one quicksort-style
 * partition step with many pivots (K5a): the chunk is split by key value into
 * equal-width sub-ranges of its bucket's digit range (or, for a bucket whose
 * sampled key distribution is skewed, equal-count groups of 2048 fine bins),
 * each of which is then sorted in one shared-memory tile (a sub-range piece of
 * up to 4 tiles -- duplicates, skew -- is sorted by its CTA as tiles + CTA
 * merges; a piece of any length whose keys are all equal is filled, not
 * sorted); a bucket with a longer, non-constant piece falls back to tile sort
 * + in-chunk merge levels.  Either way the result is the unique ascending
 * array.  (A build with -DHS_SPLIT=0 omits the
 * split, for A/B measurements only; nothing at run time changes the path.)
 *
 *   keys[n]            in/out: device; ascending on return.
 *   num_digits, chunks_per_bucket: as above.
 */
hs_status_t hs_sort(void *keys, int64_t n, hs_dtype_t dtype, int num_digits, int chunks_per_bucket,
                    cudaStream_t stream);

/*
 * SURVEY §8(f) row f1, the no-MSD ablation: the paper's Shared-Parallel
 * Hybrid Quicksort + Merge Sort on the whole array (§3.2, "a hybrid
 * algorithm ... Quicksort is used to sort the data assigned to each parallel
 * thread ... then merged"; phases S:162-170), i.e. hs_sort without the MSD
 * step: one segment of n keys is split by partition_even into
 * `chunks` chunks, every chunk is sorted (tile sort + merge levels inside
 * the chunk), then log2(chunks) tree-merge rounds merge them.
 *
 *   keys[n]            in/out: device; ascending on return.  In place.
 *   chunks             power of two in [1, 65536] ("should be a power of
 *                      two"), else HS_ERR_INVALID_VALUE.
 * Errors as hs_sort.  The result equals hs_sort's (both are the unique
 * ascending order of the keys).
 */
hs_status_t hs_sort_shared(void *keys, int64_t n, hs_dtype_t dtype, int chunks, cudaStream_t stream);

/*
 * SURVEY §8(f) row f3, the key + tag (stable) variant: SPEC's SortItem
 * (a key plus a 64-bit tag that "never influences order"), sorted
 * stably -- equal keys keep their input order, which the paper's merge sort
 * guarantees ("Merge sort is a stable sort algorithm") and which the
 * stable MSD scatter and the stable-left merge preserve.
 * Keys are int32; the items travel through the int64 path as
 * (key << 32) | input index, and the tags follow their index at the end.
 *
 * hs_msd_partition_pairs: a1-a3 on items.  keys[n] / tags[n] in (device);
 *   out_keys[n] / out_tags[n] out (device, no overlap with the inputs);
 *   bucket_offsets[11] as hs_msd_partition.  Within a bucket items keep their
 *   input order.
 * hs_sort_pairs: the whole path on items, in place: keys ascending, ties in
 *   input order, tags permuted with their keys.
 * n < 2^31; num_digits in [1, 10]; errors as hs_msd_partition / hs_sort.
 * Scratch: 16 n bytes (items + one tag copy) on top of hs_sort's 8 n.
 */
hs_status_t hs_msd_partition_pairs(const int32_t *keys, const uint64_t *tags, int64_t n, int num_digits,
                                   int64_t *bucket_offsets, int32_t *out_keys, uint64_t *out_tags,
                                   cudaStream_t stream);
hs_status_t hs_sort_pairs(int32_t *keys, uint64_t *tags, int64_t n, int num_digits, int chunks_per_bucket,
                          cudaStream_t stream);

/*
 * SURVEY §8(f) row f3 on the stable item path (k_kv.cu): SPEC's SortItem
 * (S:31-37), a key plus a 64-bit tag that "never influences order", carried
 * WITH its key through every pass as a 16-byte item (no gather by index).
 * Every kernel the items pass through is stable -- the counting scatter of
 * the MSD step, an odd-even transposition sort of adjacent items plus
 * stable-left merge rounds inside a tile, and the stable-left merge levels of
 * the paper's tree merge -- so equal keys keep their input
 * order ("Merge sort is a stable sort").  No K5a value split on this
 * path (its atomic ranking is not stable): chunks are sorted as tiles + merge
 * levels.  Keys of either dtype (int32 widen to the item's int64 key: same
 * order, same leading digit).  tags / out_tags: device uint64_t[n].
 *
 * hs_sort_pairs64: the whole path (a1-a7) on int64 keys, in place.
 * hs_msd_partition_pairs64: a1-a3 on int64 keys (out of place; outputs must
 *   not overlap the inputs); bucket_offsets[11] as hs_msd_partition.
 * hs_sort_chunks_pairs: a5 only -- every chunk (partition_even of each bucket
 *   of bucket_offsets) sorted stably; in == out allowed.
 * hs_merge_pairs: a6 only -- the log2 c tree-merge rounds of each bucket's
 *   chunk-sorted runs on SortItems with a key-only comparator, ties taking the
 *   left run; in == out allowed.
 * n < 2^31; num_digits in [1, 19]; chunks_per_bucket a power of two in
 * [1, 65536]; errors as hs_sort (HS_ERR_INVALID_VALUE also for keys / tags
 * overlapping).  Scratch: 32 n bytes from the stream-ordered pool.
 */
hs_status_t hs_sort_pairs64(int64_t *keys, uint64_t *tags, int64_t n, int num_digits, int chunks_per_bucket,
                            cudaStream_t stream);
hs_status_t hs_msd_partition_pairs64(const int64_t *keys, const uint64_t *tags, int64_t n, int num_digits,
                                     int64_t *bucket_offsets, int64_t *out_keys, uint64_t *out_tags,
                                     cudaStream_t stream);
hs_status_t hs_sort_chunks_pairs(const void *keys, const uint64_t *tags, void *out_keys, uint64_t *out_tags,
                                 int64_t n, hs_dtype_t dtype, const int64_t *bucket_offsets, int chunks_per_bucket,
                                 cudaStream_t stream);
hs_status_t hs_merge_pairs(const void *keys, const uint64_t *tags, void *out_keys, uint64_t *out_tags, int64_t n,
                           hs_dtype_t dtype, const int64_t *bucket_offsets, int chunks_per_bucket,
                           cudaStream_t stream);

/*
 * SURVEY §8(f) row f2, the sender side of the paper's cluster model with the
 * bucket exchange fused into the scatter (§3.4, "divides the data
 * into ten parts ... Then sends each bucket or buckets to proper node").
 * hs_partition_plan_create runs a1-a2 (tile histograms + lookback prefix) of
 * keys and writes the local bucket_offsets[11] (device); the caller learns
 * the sizes, agrees on an exchange layout with its peers, and then
 * hs_partition_scatter runs a3 writing the key at local bucket position p of
 * digit d straight to dst[d] + (p - bucket_offsets[d]).  dst[d] (host array of
 * 10 device pointers; NULL for an empty bucket) may point into a PEER GPU's
 * memory (CUDA IPC / symmetric memory over NVLink), so the exchange costs no
 * staging copy and no collective call.  Stability as hs_msd_partition.
 *   keys[n] must stay unchanged between create and scatter; the plan owns
 *   stream-ordered scratch released by hs_partition_plan_destroy (same stream).
 *   Errors as hs_msd_partition; dst entries must be dtype-aligned.
 */
typedef struct hs_partition_plan_s *hs_partition_plan_t;
hs_status_t hs_partition_plan_create(const void *keys, int64_t n, hs_dtype_t dtype, int num_digits,
                                     int64_t *bucket_offsets, hs_partition_plan_t *plan, cudaStream_t stream);
hs_status_t hs_partition_scatter(hs_partition_plan_t plan, void *const *dst, cudaStream_t stream);
hs_status_t hs_partition_plan_destroy(hs_partition_plan_t plan, cudaStream_t stream);

/*
 * SURVEY §8(f) row f2, host side of the paper's cluster model (§3.4 Fig 4,
 * P:80 "sends each bucket or buckets to proper node"
 * assign_buckets): split the ten digits into `nodes` contiguous groups of at
 * least one digit each, minimising the largest group total (exhaustive over
 * all C(9, nodes-1) compositions); ties go to the lexicographically earliest
 * sequence of split points.  Group g owns digits [group_start[g],
 * group_start[g+1]).  Plain host code (no device, no stream).
 *
 *   bucket_sizes[10]   host int64 bucket totals (e.g. summed over ranks).
 *   nodes              1 <= nodes <= 10, else HS_ERR_INVALID_VALUE.
 *   group_start[nodes+1] host output: [0] = 0, [nodes] = 10.
 *   max_load           host output (may be NULL): the minimised maximum.
 */
hs_status_t hs_assign_buckets(const int64_t *bucket_sizes, int nodes, int *group_start, int64_t *max_load);

/* Static, human-readable name of a status code. */
const char *hs_status_string(hs_status_t s);

/* Detail of the last error returned on the calling host thread ("" if none). */
const char *hs_last_error_message(void);

/* HS_ABI_VERSION of the loaded library. */
int hs_abi_version(void);

/*
 * Observability (tests / bench only; not part of the method):
 * number of kernel launches the most recent successful call on this host
 * thread enqueued, and the geometry constants compiled into the library:
 * keys per scatter tile, per tile-sort tile and per merge CTA for dtype.
 */
int hs_last_launch_count(void);
int hs_tile_keys(hs_dtype_t dtype, int which /* 0 scatter, 1 tile sort, 2 merge, 3 f3 item tile sort */);

/*
 * Per-kernel timing (bench only): while enabled on the calling host thread,
 * every kernel the library launches is bracketed by two CUDA events recorded
 * on the launching stream.  hs_profile_read synchronises on them, writes
 * per-kind total milliseconds and launch counts for kinds [0, nkinds) and
 * forgets them; returns 0, or -1 if an event query failed.  Kind names:
 * hs_profile_kind_name(k), k = 0 .. 9 (tile_hist, tile_scan, scatter, plan,
 * tile_sort, merge_partition, merge_level, copy, split_count, split_scatter).
 */
int hs_profile_enable(int on);
int hs_profile_read(double *ms, int *count, int nkinds);
const char *hs_profile_kind_name(int kind);

/*
 * Host-side replica of the device plan (bench / tests): from HOST
 * bucket_offsets[11], the merge levels L[b] each bucket runs and its leaf
 * exponent k[b] (chunk = 2^k[b] tile-sort leaves) for mode 0 = hs_sort,
 * 1 = hs_sort_chunks, 2 = hs_merge.  Returns max L, or -1 on a bad argument.
 */
int hs_plan_levels(const int64_t *bucket_offsets_host, hs_dtype_t dtype, int chunks_per_bucket, int mode,
                   int *levels_out, int *tile_levels_out);

/*
 * a4-a7 on keys already partitioned by leading digit (hs_msd_partition's
 * output, or the buckets a rank receives in the f2 exchange): sort every
 * bucket in place -- the same chunk sort (with the K5a value split) and chunk
 * tree merge as hs_sort, without the partition.  The result equals
 * hs_merge(hs_sort_chunks(keys)) for the same offsets (each bucket ascending,
 * buckets left where they are).
 *
 *   keys[n]            in/out: device.
 *   num_digits         D of the keys (the split uses bucket b's digit range
 *                      [b 10^(D-1), (b+1) 10^(D-1)); keys outside it are still
 *                      sorted correctly, only the split may fall back).
 *   bucket_offsets[11] in: device int64 CSR offsets, [0] = 0, [10] = n,
 *                      non-decreasing; NOT checked (it lives on the device).
 *   chunks_per_bucket  c, power of two in [1, 65536].
 * Errors: HS_ERR_INVALID_VALUE (NULL or misaligned pointer, bad D or c),
 * HS_ERR_UNSUPPORTED_DTYPE, HS_ERR_OUT_OF_MEMORY (scratch), HS_ERR_CUDA (a
 * launch failed); detail in hs_last_error_message().  Enqueued on stream; no
 * host synchronisation; scratch from the stream-ordered pool.
 */
hs_status_t hs_sort_buckets(void *keys, int64_t n, hs_dtype_t dtype, int num_digits, const int64_t *bucket_offsets,
                            int chunks_per_bucket, cudaStream_t stream);

/*
 * The device plan hs_sort would run on keys (bench / tests: which buckets the
 * K5a value split takes, hence how many merge levels run).  Runs the
 * partition and the split into scratch memory (keys is not modified),
 * synchronises the stream and writes, per bucket b (host arrays of 10):
 * levels_out[b] = merge levels L[b], split_out[b] = 0 if bucket b's chunks
 * were not value-split, 1 if they were (sub-ranges counted by the K5a count
 * pass), 2 if they were in the padded layout (no count pass: one tile-sized
 * region per chunk sub-range), leaves_out[b] = tile-sort leaves per chunk.
 * Arguments and errors as hs_sort.
 */
hs_status_t hs_sort_plan(const void *keys, int64_t n, hs_dtype_t dtype, int num_digits, int chunks_per_bucket,
                         int32_t *levels_out, int32_t *split_out, int32_t *leaves_out, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* HS_H_ */
