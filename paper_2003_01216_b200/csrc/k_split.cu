// k_split.cu -- K5a: value split of each chunk before its tile sort
// (hs_sort, hs_sort_buckets, hs_sort_pairs).
//
// a5 sorts every chunk of every bucket ("sort the partitions",
// the paper's per-thread quicksort).  A chunk of C3 holds 3.4M keys, far more
// than one shared-memory tile (T = 27,136), so without this step K5 sorts
// T-key leaves and log2(chunk / T) in-chunk merge levels (K6) rebuild the
// chunk -- 7 full read+write passes over the array on C3.  K5a instead does
// what one quicksort partition step does, with nsb - 1 pivots at once: the
// chunk's keys are split by value into nsb equal-width sub-ranges of the
// bucket's range [b 10^(D-1), (b+1) 10^(D-1)) (nsb = ceil(chunk / 0.9 T)),
// so every sub-range is a leaf that K5 sorts in one tile and the sorted
// sub-ranges, laid end to end, ARE the sorted chunk.  What remains of K6 is
// the paper's binary tree merge of the c sorted chunks (a6).
//
//   k_split_setup       1 CTA: per-bucket sub-range counts, slices, table
//                       offsets (ten lanes in parallel); zeroes the table
//   k_split_sample_map  one CTA per chunk of a candidate bucket (per bucket
//                       beyond kMapChunksMax chunks): a 4k-key sample over
//                       8192 fine equal-width bins; a chunk that looks skewed
//                       takes 32k samples and writes its equal-count map, and
//                       puts its bucket in map mode
//   k_split_count       persistent CTAs over slices (<= NT*VT keys of one
//                       chunk) of the partitioned keys: shared-memory histogram
//                       of the sub-ranges, non-zero counts added to the chunk's
//                       table row (next slice's loads in flight during the flush)
//   k_split_plan        one CTA per chunk: exclusive scan of the row -> sub-range
//                       starts (+ cursor copy); a sub-range over T keys marks
//                       the bucket "bad"; the last CTA finalises the Plan: split
//                       buckets get k = 0, L = log2 c, leaves = sub-ranges; bad
//                       buckets keep the tile + in-chunk merge plan (a value
//                       with more than a tile of copies in a chunk: correct
//                       either way, only slower)
//   k_split_scatter     persistent CTAs over the same slices: ranks by shared
//                       atomics, one global atomic per non-empty sub-range
//                       claims the slice's output span, (destination, key)
//                       staged in shared memory and written run by run
//                       (coalesced within a sub-range)
//
// The order of keys inside a sub-range depends on atomic arrival order; the
// tile sort that follows makes the result the unique sorted chunk (keys only;
// hs_sort_pairs sorts unique (key << 32 | index) items, so stays stable).
// Sub-range of a key: min(mulhi(max(x - lo_b, 0), mul), nsb - 1) with mul =
// floor((2^w - 1) / 10^(D-1)) nsb -- non-decreasing in the key, so sub-range
// order is key order; keys clamped into bucket 0 / 9 (P:78 reading #3) land in
// the first / last sub-range.  In map mode the sub-range is map[fine bin], and
// every map is non-decreasing in the fine bin, so the order argument holds.
// Roofline: HBM, 4 B read (count) + 8 B read+write (scatter) per int32 key.
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

namespace hs {

template <typename K>
struct SplGeo;
#ifndef HS_SPL_VT
#define HS_SPL_VT 24  // 12,288-key slices (16: 8,192 -- C3 split count + scatter 0.98 -> 0.90 ms)
#endif
#ifndef HS_SPL_MINB_SCAT
#define HS_SPL_MINB_SCAT 2
#endif
#ifndef HS_SPL_MINB_COUNT
#define HS_SPL_MINB_COUNT 2  // 64 registers: 24 keys per thread without spills
#endif
template <>
struct SplGeo<int32_t> {
    static constexpr int NT = 512, VT = HS_SPL_VT, MINB_COUNT = HS_SPL_MINB_COUNT, MINB_SCAT = HS_SPL_MINB_SCAT;
};
#ifndef HS_SPL_VT64
#define HS_SPL_VT64 12  // 6,144-key slices (8: C5 split count + scatter 4.63 -> 4.00 ms)
#endif
#ifndef HS_SPL_MINB_COUNT64
#define HS_SPL_MINB_COUNT64 2
#endif
template <>
struct SplGeo<int64_t> {
    static constexpr int NT = 512, VT = HS_SPL_VT64, MINB_COUNT = HS_SPL_MINB_COUNT64, MINB_SCAT = 2;
};
constexpr int kSplitMaxSub = 4096;  // sub-ranges per chunk (shared-memory counters)
constexpr int kSplitPlanNT = 512;

#ifndef HS_SPLIT_MAP_PCT
#define HS_SPLIT_MAP_PCT 70  // sampled-map sub-ranges: this share of a tile (slack for the sampling error)
#endif
#ifndef HS_SPLIT_TARGET_PCT
#define HS_SPLIT_TARGET_PCT 90
#endif
// equal-width sub-ranges aim at this share of a tile (uniform keys: the largest of ~10^4
// sub-ranges stays a few standard deviations, ~1%, above the mean)
__host__ __device__ __forceinline__ long long split_target(int tile_keys) {
    return (long long)tile_keys * HS_SPLIT_TARGET_PCT / 100;
}

// ------------------------------------------------------------------ setup
// Row capacity per chunk for a sampled (skewed) bucket: sub-ranges of ~0.7 T
// keys (slack for the sampling error of the map).
__host__ __device__ __forceinline__ long long split_target_map(int tile_keys) { return (long long)tile_keys * HS_SPLIT_MAP_PCT / 100; }

// Constant over-full sub-ranges (a value with more copies in a chunk than the
// big-piece path takes, e.g. all keys equal): for buckets whose sample shows a
// fine bin of more than a tile of keys per chunk (C.cc), the count pass also
// records, per (chunk, sub-range), the min and max key (order-preserving
// unsigned images; min kept as its complement so that both are atomicMax into
// zeroed words).  A piece with min == max is already sorted: k_split_plan
// flags it (cflag), the scatter writes it straight to where the tile sort's
// output goes, and the tile sort only writes its key samples.
struct SplitConst {
    unsigned long long *gminc;  // ~u(min) per split-table word
    unsigned long long *gmax;   // u(max)
    uint32_t *cflag;            // 1: constant piece
    unsigned long long *clist;  // constant pieces (split-table word, absolute chunk start, bucket), C.nconst of them
};
__device__ __forceinline__ unsigned long long ukey(int32_t k) { return (unsigned long long)((uint32_t)k ^ 0x80000000u); }
__device__ __forceinline__ unsigned long long ukey(int64_t k) { return (unsigned long long)k ^ 0x8000000000000000ull; }

__global__ void k_split_setup(Ctl *ctl, unsigned long long div, int key_bits, int key_shift, int tile_keys,
                              int slice_keys, long long tab_cap, int nsb_cap, uint32_t *tab, SplitConst sc,
                              long long pad_cap) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    __shared__ long long s_words;
    if (threadIdx.x < 32) {  // lane b < 10: bucket b's geometry (64-bit divisions in parallel)
        Plan &P = ctl->plan;
        SplitCfg &C = ctl->split;
        const int b = threadIdx.x;
        const long long c = 1LL << P.log2c, target = split_target(tile_keys);
        const long long target_m = split_target_map(tile_keys);
        const unsigned long long wmax = key_bits == 32 ? 0xFFFFFFFFull : ~0ull;
        long long ns = 0, nsa = 0, spc = 0;
        bool cand = false;
        if (b < 10) {
            const long long m = P.off[b + 1] - P.off[b], cm = (m + c - 1) / c;
            ns = (cm + target - 1) / target;
            nsa = (cm + target_m - 1) / target_m;
            if (nsa > nsb_cap) nsa = nsb_cap;
            if (nsa < ns) nsa = ns;
            spc = (cm + slice_keys - 1) / slice_keys;
            // ns <= div: the multiplier below fits the key width (and narrower sub-ranges would be empty)
            cand = P.k[b] > 0 && ns >= 2 && ns <= nsb_cap && (unsigned long long)ns <= div;
        }
        // table capacity check and prefixes, in bucket order (lane 0, ten steps)
        long long words = cand ? c * (nsa + 1) : 0;
        long long ac_t = 0, ac_s = 0, acc_t = 0, acc_s = 0, ac_p = 0, acc_p = 0;
        bool ok = cand, pok = false;
        for (int q = 0; q < 10; ++q) {
            const long long wq = __shfl_sync(0xffffffffu, words, q);
            const long long sq = __shfl_sync(0xffffffffu, cand ? c * spc : 0LL, q);
            const long long pq = __shfl_sync(0xffffffffu, cand ? c * ns * (long long)tile_keys : 0LL, q);
            const bool cq = __shfl_sync(0xffffffffu, cand ? 1 : 0, q) && acc_t + wq <= tab_cap;
            const bool pqok = cq && acc_p + pq <= pad_cap;  // padded regions of the equal-width sub-ranges
            if (q == b) {
                ok = cq;
                pok = pqok;
                ac_t = acc_t;
                ac_s = acc_s;
                ac_p = acc_p;
            }
            if (cq) {
                acc_t += wq;
                acc_s += sq;
            }
            if (pqok) acc_p += pq;
        }
        if (b < 10) {
            C.cand[b] = ok;
            C.mode[b] = 0;
            C.slice_prefix[b] = ac_s;
            C.cc[b] = 0;
            C.pad[b] = pok;
            C.pboff[b] = ac_p;
            C.k0[b] = P.k[b];
            if (ok) {
                C.spc[b] = (int)spc;
                P.nsb[b] = (int)ns;
                C.ns0[b] = (int)ns;
                C.nsa[b] = (int)nsa;
                P.sboff[b] = ac_t;
                C.lo[b] = (long long)b * (long long)div;
                C.mul[b] = wmax / div * (unsigned long long)ns;  // <= wmax since ns <= div
                // fine bins for the sampled map (needs >= 1 value per fine bin; nsa <= kSplitFine)
                C.fmul[b] = (div >= (unsigned long long)kSplitFine && nsa <= kSplitFine)
                                ? wmax / div * (unsigned long long)kSplitFine : 0ull;
            } else {
                C.spc[b] = 1;
                C.lo[b] = 0;
                C.mul[b] = 0;
                C.fmul[b] = 0;
                C.nsa[b] = 0;
            }
        }
        if (b == 0) {
            C.cap = tile_keys;
            C.ticket2 = 0;
            C.slice_prefix[10] = acc_s;
            C.shift = key_shift;
            C.map_chunks = c <= kMapChunksMax ? (int)c : 1;
            s_words = acc_t;
        }
    }
    __syncthreads();
    for (long long q = threadIdx.x; q < s_words; q += blockDim.x) {
        tab[q] = 0;
        sc.gminc[q] = 0;
        sc.gmax[q] = 0;
        sc.cflag[q] = 0;
    }
}

// ------------------------------------------------------------------ sampled map
// Equal-width sub-ranges fit keys spread over the digit range (C2, C3, C5, P3).
// For a skewed bucket (C4: a normal peak) k_split_sample_map histograms a sample
// of the bucket over kSplitFine fine bins and either keeps the equal-
// width sub-ranges (their largest sample count is within mean + 5 sqrt(mean))
// or replaces them by equal-count groups of consecutive fine bins:
// map[i] = floor(excl_prefix(i) * ns' / total), non-decreasing in i, so the
// sub-range order is still key order.  The exact count pass decides as before
// (an over-full sub-range -- e.g. one value with > T copies in a chunk -- makes
// the bucket fall back).
constexpr int kSplitSamplesLog2 = 15, kSplitSamples = 1 << kSplitSamplesLog2;  // per candidate bucket

template <typename K>
__device__ __forceinline__ int fine_bin(K k, int shift, long long lo, unsigned long long fmul);
template <>
__device__ __forceinline__ int fine_bin<int32_t>(int32_t k, int, long long lo, unsigned long long fmul) {
    const int32_t d = max(k - (int32_t)lo, 0);
    return min((int)__umulhi((uint32_t)d, (uint32_t)fmul), kSplitFine - 1);
}
template <>
__device__ __forceinline__ int fine_bin<int64_t>(int64_t k, int shift, long long lo, unsigned long long fmul) {
    const long long d = max((k >> shift) - lo, 0LL);
    return (int)min((long long)__umul64hi((unsigned long long)d, fmul), (long long)(kSplitFine - 1));
}

// One CTA per chunk of a candidate bucket (or per bucket when c > kMapChunksMax):
// a 4k-key sample decides whether the range is skewed; a skewed one takes 32k
// samples for its map.  Shared-memory fine-bin histogram, the chunk's map, and
// the skew flag -- one skewed chunk puts its bucket in map mode (every chunk
// then uses its own map: sorted or locally clustered inputs give each chunk a
// different value range).
template <typename K>
__global__ void __launch_bounds__(1024) k_split_sample_map(Ctl *ctl, const K *__restrict__ S, uint16_t *map,
                                                           int tile_keys) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    constexpr int NT = 1024, PER = kSplitFine / NT, SPT = kSplitSamples / NT;
    static_assert(kSplitFine % NT == 0 && kSplitSamples % NT == 0, "per-thread shares");
    __shared__ uint32_t h[kSplitFine + 1];  // fine-bin histogram, then its exclusive prefix (+ total)
    __shared__ uint32_t wsum[NT / 32];
    __shared__ unsigned s_max;
    static_assert(SPT % 8 == 0, "phase-1 share");
    Plan &P = ctl->plan;
    SplitCfg &C = ctl->split;
    const int mc = C.map_chunks;
    const int b = blockIdx.x / mc, jj = blockIdx.x % mc, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (!C.cand[b] || C.fmul[b] == 0) return;
    const long long mb = P.off[b + 1] - P.off[b];
    long long base = P.off[b], m = mb;  // the sampled range: chunk jj, or the whole bucket
    if (mc > 1) {
        const long long c0 = part_start(mb, P.log2c, jj), c1 = part_start(mb, P.log2c, jj + 1);
        base += c0;
        m = c1 - c0;
    }
    if (m == 0) return;
    const long long lo = C.lo[b];
    const unsigned long long fmul = C.fmul[b];
    const int shift = C.shift;
    const int ns = C.ns0[b];
    // sample rank r in [0, kSplitSamples) -> position (r m) >> log2 (evenly spaced over the range).
    // Phase 1 takes every 8th rank (4k samples): enough to tell a uniform range (the common case,
    // stops here) from a skewed one; a skewed range takes the other 28k ranks for its map.
    auto sample = [&](bool phase2) {
        if (!phase2) {
            constexpr int R1 = SPT / 8;
            K kk[R1];
#pragma unroll
            for (int j = 0; j < R1; ++j) {
                const unsigned long long r = 8ull * (unsigned long long)(j * NT + tid);  // < kSplitSamples
                kk[j] = __ldg(S + base + (long long)((r * (unsigned long long)m) >> kSplitSamplesLog2));
            }
#pragma unroll
            for (int j = 0; j < R1; ++j) atomicAdd(&h[fine_bin<K>(kk[j], shift, lo, fmul)], 1u);
        } else {
            constexpr int R = 8;  // loads per round and thread (in flight together)
#pragma unroll 1
            for (int j0 = 0; j0 < SPT; j0 += R) {
                K kk[R];
                bool ok[R];
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const unsigned long long r = (unsigned long long)((j0 + j) * NT + tid);  // < kSplitSamples
                    ok[j] = (r & 7ull) != 0;  // the phase-1 ranks are already counted
                    kk[j] = ok[j] ? __ldg(S + base + (long long)((r * (unsigned long long)m) >> kSplitSamplesLog2))
                                  : K(0);
                }
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if (ok[j]) atomicAdd(&h[fine_bin<K>(kk[j], shift, lo, fmul)], 1u);
            }
        }
    };
    uint32_t hv[PER], excl0 = 0, total = 0;
    // h holds a fine-bin histogram: hv <- my bins, total, excl0 <- my first bin's exclusive prefix,
    // s_max <- the largest equal-width sub-range count; h ends as the exclusive prefix
    auto analyze = [&]() {
        uint32_t sum = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            hv[j] = h[tid * PER + j];
            sum += hv[j];
        }
        if (tid == 0) s_max = 0;
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        const uint32_t wl = lane < NT / 32 && lane < warp ? wsum[lane] : 0u;
        excl0 = incl - sum + __reduce_add_sync(0xffffffffu, wl);
        const uint32_t wt = lane < NT / 32 ? wsum[lane] : 0u;
        total = __reduce_add_sync(0xffffffffu, wt);
        uint32_t run0 = excl0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            h[tid * PER + j] = run0;
            run0 += hv[j];
        }
        if (tid == 0) h[kSplitFine] = total;
        __syncthreads();
        // equal-width sub-range t holds (about) the fine bins i with floor(i ns / kSplitFine) = t,
        // i.e. [ceil(t F / ns), ceil((t+1) F / ns)): its sample count is a prefix difference
        uint32_t mx = 0;
        for (int t = tid; t < ns; t += NT) {
            const int lo_i = (t * kSplitFine + ns - 1) / ns, hi_i = ((t + 1) * kSplitFine + ns - 1) / ns;
            const uint32_t e = h[hi_i] - h[lo_i];
            mx = e > mx ? e : mx;
        }
        mx = __reduce_max_sync(0xffffffffu, mx);
        if (lane == 0) atomicMax(&s_max, mx);
        __syncthreads();
    };
    // skewed: the largest sample count is beyond the sampling noise of a uniform range,
    // > mean + 5 sqrt(mean) + 1 (mean = total / ns; the max of ns Poisson counts stays
    // within ~3.5 sqrt(mean) of it)
    // A smooth density change (a ramp) is too gentle for the per-sub-range test at 4k samples,
    // but 8 coarse groups of the range average the noise away: a group beyond mean + 5 sqrt(mean)
    // (~1.22x at 4k samples) means equal-width sub-ranges of ~0.9 T would overflow somewhere.
    auto is_skewed = [&]() {
        const float mean_s = (float)total / (float)ns;
        uint32_t cmax = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const uint32_t e = h[(g + 1) * (kSplitFine / 8)] - h[g * (kSplitFine / 8)];  // h: the prefix
            cmax = e > cmax ? e : cmax;
        }
        const float mean_c = (float)total / 8.0f;
        return total > 0 && ((float)s_max > mean_s + 5.0f * sqrtf(mean_s) + 1.0f ||
                             (float)cmax > mean_c + 5.0f * sqrtf(mean_c) + 1.0f);
    };
    __shared__ unsigned s_binmax;
    for (int q = tid; q < kSplitFine; q += NT) h[q] = 0;
    if (tid == 0) s_binmax = 0;
    __syncthreads();
    sample(false);
    __syncthreads();
    analyze();
    {   // a fine bin holding more than a tile of keys per chunk: track constant sub-ranges in the count pass
        uint32_t bm = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) bm = hv[j] > bm ? hv[j] : bm;
        bm = __reduce_max_sync(0xffffffffu, bm);
        if (lane == 0) atomicMax(&s_binmax, bm);
        __syncthreads();
        // a piece over the big-piece limit (2^kBigLog2 tiles) needs a bin of many copies; ask for
        // two tiles' worth of a chunk and >= 32 samples (far above the noise of a smooth density)
        const long long cmk = (mb + (1LL << P.log2c) - 1) >> P.log2c;  // keys per chunk
        if (tid == 0 && s_binmax >= 32 &&
            (unsigned long long)s_binmax * (unsigned long long)cmk >
                2ull * (unsigned long long)tile_keys * (unsigned long long)total)
            C.cc[b] = 1;
    }
    bool skewed = is_skewed();
    if (skewed) {  // uniform per CTA: the full sample for the map
        uint32_t h1[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) h1[j] = hv[j];
        for (int q = tid; q < kSplitFine; q += NT) h[q] = 0;
        __syncthreads();
        sample(true);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) h[tid * PER + j] += h1[j];  // my own bins: no race
        __syncthreads();
        analyze();
        skewed = is_skewed();
    }
    if (!skewed && mc == 1) return;  // a bucket-wide map is only needed when skewed
    const long long c = 1LL << P.log2c, cm = (mb + c - 1) / c;
    const long long tm = split_target_map(tile_keys);
    long long ns2 = (cm + tm - 1) / tm;
    if (ns2 > C.nsa[b]) ns2 = C.nsa[b];
    if (ns2 < 2) ns2 = 2;
    // every chunk writes its map (another chunk of the bucket may be the skewed one): equal-count
    // groups of its sample -- unless the chunk looked uniform and its 4k sample is too thin for
    // ns2 groups (< 64 samples each), then equal-width groups of fine bins
    uint16_t *const cmap = map + ((size_t)b * mc + jj) * kSplitFine;
    const bool by_count = skewed || total >= 64u * (unsigned)ns2;
    uint32_t run = excl0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const long long g = by_count ? (long long)run * ns2 / total : (long long)(tid * PER + j) * ns2 / kSplitFine;
        cmap[tid * PER + j] = (uint16_t)(g < ns2 - 1 ? g : ns2 - 1);
        run += hv[j];
    }
    if (skewed && tid == 0) {  // idempotent: every skewed chunk of the bucket writes the same values
        P.nsb[b] = (int)ns2;
        C.mode[b] = 1;
    }
}

// ------------------------------------------------------------------ helpers
// Sub-range of key k in its bucket: d = x - lo (x = k >> shift) and
// t = min(mulhi(d, mul), ns - 1), t = 0 for d < 0 -- non-decreasing in k, and
// t < ns for 0 <= d < 10^(D-1) (mul <= (2^w - 1) ns / 10^(D-1)).  int32: a key
// of bucket b >= 1 has x >= b 10^(D-1) = lo and bucket 0 has lo = 0, so
// x - lo never overflows.
__device__ __forceinline__ int sub_range_of(int32_t k, int, long long lo, unsigned long long mul, int ns) {
    const int32_t d = max(k - (int32_t)lo, 0);
    return min((int)__umulhi((uint32_t)d, (uint32_t)mul), ns - 1);
}
__device__ __forceinline__ int sub_range_of(int64_t k, int shift, long long lo, unsigned long long mul, int ns) {
    const long long d = max((k >> shift) - lo, 0LL);  // arithmetic shift: the sign of the key survives
    return (int)min((long long)__umul64hi((unsigned long long)d, mul), (long long)(ns - 1));
}

// Ranks in duplicate-heavy slices (buckets with constant tracking: one value may fill a
// whole slice, and 32 lanes taking ranks from one shared counter serialise): a warp whose
// 32 keys all fall in one sub-range takes 32 ranks at once.  All 32 lanes call it (slots
// past a slice's end carry the dummy sub-range).  (The count pass measured slower with
// the same test: its plain atomics return nothing.)
__device__ __forceinline__ uint32_t warp_rank(uint32_t *hist, int t) {
    const int lane = threadIdx.x & 31;
    const int t0 = __shfl_sync(0xffffffffu, t, 0);
    if (__all_sync(0xffffffffu, t == t0)) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&hist[t0], 32u);
        return __shfl_sync(0xffffffffu, base, 0) + (uint32_t)lane;
    }
    return atomicAdd(&hist[t], 1u);
}

// In-place exclusive scan of a[0, n) by the whole CTA (NT threads, contiguous
// segments per thread).  Ends with a barrier.
template <int NT>
__device__ __forceinline__ void cta_excl_scan(uint32_t *a, int n, uint32_t *wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int E = (n + NT - 1) / NT;
    const int b0 = tid * E < n ? tid * E : n, b1 = b0 + E < n ? b0 + E : n;
    uint32_t sum = 0;
    for (int q = b0; q < b1; ++q) sum += a[q];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    const uint32_t wl = lane < NT / 32 && lane < warp ? wsum[lane] : 0u;
    uint32_t base = incl - sum + __reduce_add_sync(0xffffffffu, wl);  // + totals of the warps before mine
    for (int q = b0; q < b1; ++q) {
        const uint32_t t = a[q];
        a[q] = base;
        base += t;
    }
    __syncthreads();
}

// ------------------------------------------------------------- count / scatter
// A slice = <= TS consecutive keys of one chunk (its slices are numbered
// bucket by bucket, chunk by chunk).  Its geometry needs 64-bit divisions, so
// one thread computes it and the CTA reads it from shared memory.
struct SliceDesc {
    long long cs, row, lo;  // chunk start (absolute), split-table row, bucket value base
    long long ocs;          // where the chunk's sub-ranges go: cs, or (padded layout) its first region in the pad buffer
    unsigned long long mul, fmul;
    const uint16_t *bmap;    // sampled sub-range map of the bucket (null: equal width)
    int cnt, ns, shift, a0;  // keys in the slice (0: nothing to do), sub-ranges, item shift, offset in chunk
    int cc;                  // track constant sub-ranges (SplitConst)
    int pad;                 // padded layout (split_pmode): regions of cap keys, no count pass
};

// Called by one thread (the fields share a few cache lines, so after the
// first miss the chain of loads hits L1).
__device__ __forceinline__ void slice_desc(SliceDesc &sd, const Ctl *ctl, long long g, bool need_split, int TS,
                                           const uint16_t *map) {
    const Plan &P = ctl->plan;
    const SplitCfg &C = ctl->split;
    sd.cnt = 0;
    sd.ns = 0;
    if (g >= C.slice_prefix[10]) return;
    int b = 0;
    while (b < 9 && g >= C.slice_prefix[b + 1]) ++b;
    if (need_split && !P.split[b]) return;  // a bucket that fell back keeps its keys in S
    const bool pad = split_pmode(C, b);
    if (!need_split && pad) return;         // the count pass skips padded buckets
    const unsigned r = (unsigned)(g - C.slice_prefix[b]), spc = (unsigned)C.spc[b];  // < 2^31
    const long long j = r / spc, s = r - (unsigned)j * spc;
    const long long m = P.off[b + 1] - P.off[b];
    const long long c0 = part_start(m, P.log2c, j), c1 = part_start(m, P.log2c, j + 1);
    const long long a0 = s * TS;
    if (a0 >= c1 - c0) return;
    sd.cnt = (int)((c1 - c0 - a0) < TS ? (c1 - c0 - a0) : TS);
    sd.pad = pad;
    sd.cs = P.off[b] + c0;
    sd.ocs = pad ? C.pboff[b] + j * (long long)P.nsb[b] * C.cap : sd.cs;
    sd.a0 = (int)a0;
    sd.ns = P.nsb[b];
    sd.row = P.sboff[b] + j * (P.nsb[b] + 1);
    sd.lo = C.lo[b];
    sd.mul = C.mul[b];
    sd.fmul = C.fmul[b];
    sd.bmap = C.mode[b] ? map + ((size_t)b * C.map_chunks + (C.map_chunks > 1 ? j : 0)) * kSplitFine : nullptr;
    sd.shift = C.shift;
    sd.cc = C.cc[b];
}

// Count: persistent CTAs walk the slices with stride gridDim.x.  While the
// shared histogram of slice g is flushed to its chunk's row (and re-zeroed by
// the same threads), the keys of the CTA's next slice are already loading.
// hist[ns] is a dummy sub-range for slots past a slice's end (branch-free).
// CC = false: slices of buckets without constant tracking (the usual case, no extra work);
// CC = true: only slices of C.cc buckets, with the tracking (exits at once when there are none).
template <typename K, int NT, int VT, int MINB, bool CC>
__global__ void __launch_bounds__(NT, MINB) k_split_count(const Ctl *__restrict__ ctl, const K *__restrict__ S,
                                                          uint32_t *tab, int nsb_cap, const uint16_t *map,
                                                          SplitConst sc) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    {   // exit at once when no bucket needs this pass (CC: constant tracking; else: a counted,
        // not padded, candidate bucket)
        bool any = false;
        for (int b = 0; b < 10; ++b)
            any |= CC ? ctl->split.cc[b] != 0 : (ctl->split.cand[b] && !split_pmode(ctl->split, b));
        if (!any) return;
    }
    constexpr int TS = NT * VT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t *const hist = reinterpret_cast<uint32_t *>(smem_raw);  // [nsb_cap + 1]
    // SplitConst tracking (slices of C.cc buckets): a key of each sub-range of the slice, and
    // whether another key of the slice differs from it
    K *const rep = reinterpret_cast<K *>(smem_raw + (((size_t)(nsb_cap + 1) * 4 + 15) & ~(size_t)15));
    unsigned char *const mixed = reinterpret_cast<unsigned char *>(rep + nsb_cap + 1);
    __shared__ SliceDesc sd[2];
    const int tid = threadIdx.x;
    for (int q = tid; q <= nsb_cap; q += NT) {
        hist[q] = 0;
        mixed[q] = 0;
    }
    long long g = blockIdx.x;
    if (tid == 0) slice_desc(sd[0], ctl, g, false, TS, map);
    __syncthreads();
    int cur = 0;
    K v[VT];
    {
        const K *in = S + sd[0].cs + sd[0].a0;
        const int cnt = (sd[0].cc != 0) == CC ? sd[0].cnt : 0;
#pragma unroll
        for (int k = 0; k < VT; ++k) v[k] = k * NT + tid < cnt ? in[k * NT + tid] : K(0);
    }
    const long long nslices = ctl->split.slice_prefix[10];
    for (; g < nslices; g += gridDim.x) {
        const SliceDesc &d = sd[cur];
        if (tid == 0) slice_desc(sd[cur ^ 1], ctl, g + gridDim.x, false, TS, map);
        const int cnt = (d.cc != 0) == CC ? d.cnt : 0, ns = d.ns;  // this instantiation's slices only
        constexpr bool cc = CC;
        // sub-range of slot k (slots past the slice's end: the dummy sub-range ns)
        auto sub = [&](int k) -> int {
            if (k * NT + tid >= cnt) return ns;
            return d.bmap == nullptr ? sub_range_of(v[k], d.shift, d.lo, d.mul, ns)
                                     : (int)__ldg(d.bmap + fine_bin<K>(v[k], d.shift, d.lo, d.fmul));
        };
        if (cnt > 0) {
            HS_DASSERT(ns >= 2 && ns <= nsb_cap);
            if (d.bmap == nullptr) {  // equal width (uniform per slice: the branch is outside the key loop)
                const long long lo = d.lo;
                const unsigned long long mul = d.mul;
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    const int t = k * NT + tid < cnt ? sub_range_of(v[k], d.shift, lo, mul, ns) : ns;
                    atomicAdd(&hist[t], 1u);
                }
            } else {
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    const int t = k * NT + tid < cnt ? (int)__ldg(d.bmap + fine_bin<K>(v[k], d.shift, d.lo, d.fmul)) : ns;
                    atomicAdd(&hist[t], 1u);
                }
            }
            if (cc) {
#pragma unroll 4
                for (int k = 0; k < VT; ++k) rep[sub(k)] = v[k];  // any one key of the sub-range wins
            }
        }
        __syncthreads();  // histogram complete; next descriptor visible
        if (cc && cnt > 0) {  // (a skipped slice's descriptor has no sub-ranges)
#pragma unroll 4
            for (int k = 0; k < VT; ++k) {
                const int t = sub(k);
                if (!(rep[t] <= v[k] && v[k] <= rep[t])) mixed[t] = 1;
            }
            __syncthreads();
        }
        const SliceDesc &dn = sd[cur ^ 1];
        {
            const K *in = S + dn.cs + dn.a0;
            const int cn = (dn.cc != 0) == CC ? dn.cnt : 0;
#pragma unroll
            for (int k = 0; k < VT; ++k) v[k] = k * NT + tid < cn ? in[k * NT + tid] : K(0);
        }
        if (cnt > 0) {
            for (int q = tid; q <= ns; q += NT) {
                const uint32_t h = hist[q];
                if (h && q < ns) {
                    atomicAdd(&tab[d.row + q], h);
                    if (cc) {
                        const unsigned long long u = mixed[q] ? ~0ull : ukey(rep[q]);
                        atomicMax(&sc.gmax[d.row + q], u);
                        atomicMax(&sc.gminc[d.row + q], mixed[q] ? ~0ull : ~u);  // mixed: min 0, max ~0
                    }
                }
                hist[q] = 0;
                mixed[q] = 0;
            }
        }
        __syncthreads();  // histogram zero again; sd[cur] may be overwritten
        cur ^= 1;
    }
}

// Scatter: persistent CTAs walk the slices with stride gridDim.x (the next
// slice's descriptor is computed during this one, its keys load during this
// one's write-out).  Ranks by shared atomics (the dummy sub-range ns takes the
// slots past the slice's end), one global atomic per non-empty sub-range
// claims the slice's span (in flight during the local scan), keys are staged
// at their slice-local sorted position, then written in staged order with
// their sub-range recomputed: consecutive threads write consecutive addresses
// inside a sub-range.
// CC = false: the slices of buckets without constant tracking (the usual case); CC = true: only
// those of C.cc buckets, ranked with warp_rank (exits at once when there are none).
template <typename K, int NT, int VT, int MINB, bool CC>
__global__ void __launch_bounds__(NT, MINB) k_split_scatter(const Ctl *__restrict__ ctl, const K *__restrict__ S,
                                                            K *__restrict__ F, uint32_t *cur, int nsb_cap,
                                                            const uint16_t *map, K *__restrict__ padbuf,
                                                            int cap_keys) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    if (CC) {
        bool any = false;
        for (int b = 0; b < 10; ++b) any |= ctl->split.cc[b] != 0 && ctl->plan.split[b] != 0;
        if (!any) return;
    }
    constexpr int TS = NT * VT;
    static_assert(TS <= 65536, "ranks are packed in 16 bits");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint32_t wsum[NT / 32];
    __shared__ SliceDesc sd[2];
    uint32_t *const hist = reinterpret_cast<uint32_t *>(smem_raw);  // [nsb_cap + 1]
    uint32_t *const sstart = reinterpret_cast<uint32_t *>(
        smem_raw + (((size_t)(nsb_cap + 1) * 4 + 15) & ~(size_t)15));  // [nsb_cap + 1]: slice-local starts
    uint32_t *const sdelta = sstart + (nsb_cap + 1);                   // [nsb_cap + 1]: span - start
    K *const skeys = reinterpret_cast<K *>(sdelta + (nsb_cap + 1));    // [TS] staged keys

    const int tid = threadIdx.x;
    for (int q = tid; q <= nsb_cap; q += NT) hist[q] = 0;
    long long g = blockIdx.x;
    if (tid == 0) slice_desc(sd[0], ctl, g, true, TS, map);
    __syncthreads();
    // this instantiation's slices only (a skipped slice's descriptor has cnt = 0 or another cc)
    auto mine = [](const SliceDesc &x) -> int { return (x.cnt > 0 && (x.cc != 0) == CC) ? x.cnt : 0; };
    K v[VT];
    {
        const K *in = S + sd[0].cs + sd[0].a0;
        const int cnt = mine(sd[0]);
#pragma unroll
        for (int k = 0; k < VT; ++k) v[k] = k * NT + tid < cnt ? in[k * NT + tid] : K(0);
    }
    const long long nslices = ctl->split.slice_prefix[10];
    int cb = 0;
    for (; g < nslices; g += gridDim.x, cb ^= 1) {
        const SliceDesc &d = sd[cb];
        if (tid == 0) slice_desc(sd[cb ^ 1], ctl, g + gridDim.x, true, TS, map);
        const int cnt = mine(d), ns = d.ns;
        if (cnt == 0) {  // nothing here (fallback bucket / past the chunk's end / other instantiation)
            __syncthreads();
            const SliceDesc &dn = sd[cb ^ 1];
            const K *in = S + dn.cs + dn.a0;
            const int cn = mine(dn);
#pragma unroll
            for (int k = 0; k < VT; ++k) v[k] = k * NT + tid < cn ? in[k * NT + tid] : K(0);
            __syncthreads();
            continue;
        }
        HS_DASSERT(ns >= 2 && ns <= nsb_cap);
        uint32_t tr[VT];  // sub-range << 16 | rank within the slice's keys of that sub-range
        {
            const long long lo = d.lo;
            const unsigned long long mul = d.mul, fmul = d.fmul;
            const uint16_t *const bmap = d.bmap;
            const int shift = d.shift;
            if (bmap == nullptr) {
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    const int t = k * NT + tid < cnt ? sub_range_of(v[k], shift, lo, mul, ns) : ns;
                    tr[k] = ((uint32_t)t << 16) | (CC ? warp_rank(hist, t) : atomicAdd(&hist[t], 1u));
                }
            } else {
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    const int t = k * NT + tid < cnt ? (int)__ldg(bmap + fine_bin<K>(v[k], shift, lo, fmul)) : ns;
                    tr[k] = ((uint32_t)t << 16) | (CC ? warp_rank(hist, t) : atomicAdd(&hist[t], 1u));
                }
            }
        }
        __syncthreads();
        // chunk-relative start of this slice's span of sub-range q; the first NT stay in a
        // register while the scan runs (ns > NT is rare: chunks of > 0.9 T NT keys)
        const long long row = d.row;
        uint32_t span0 = 0;
        if (tid < ns) {
            const uint32_t h = hist[tid];
            span0 = h ? atomicAdd(&cur[row + tid], h) : 0u;
        }
        for (int q = tid + NT; q < ns; q += NT) {
            const uint32_t h = hist[q];
            sdelta[q] = h ? atomicAdd(&cur[row + q], h) : 0u;
        }
        cta_excl_scan<NT>(hist, ns + 1, wsum);  // hist -> slice-local starts (overlaps the atomics)
        for (int q = tid; q <= ns; q += NT) {
            const uint32_t sp = q == tid ? span0 : (q < ns ? sdelta[q] : 0u);
            sstart[q] = hist[q];
            sdelta[q] = sp - hist[q];  // destination - staging position inside sub-range q (mod 2^32)
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VT; ++k)  // dummy slots land in [cnt, TS) and are not written out
            skeys[sstart[tr[k] >> 16] + (tr[k] & 0xFFFFu)] = v[k];
        __syncthreads();  // staged; hist is free; the next descriptor is visible
        const SliceDesc &dn = sd[cb ^ 1];
        {
            const K *in = S + dn.cs + dn.a0;
            const int cn = mine(dn);
#pragma unroll
            for (int k = 0; k < VT; ++k) v[k] = k * NT + tid < cn ? in[k * NT + tid] : K(0);
            const int nz = (cn > 0 && dn.ns > ns) ? dn.ns : ns;
            for (int q = tid; q <= nz; q += NT) hist[q] = 0;
        }
        // written in staged order; each key's sub-range is recomputed (the same map as the
        // ranking) to find its destination: only keys are staged, 4 (int64: 8) bytes per key
        {
            const long long lo = d.lo;
            const unsigned long long mul = d.mul, fmul = d.fmul;
            const uint16_t *const bmap = d.bmap;
            const int shift = d.shift;
            if (d.pad) {
                // padded layout: sub-range t owns [t cap, (t + 1) cap) of the chunk's regions; keys
                // past a full region are dropped (k_split_pad_plan sees the cursor beyond it and
                // sends the bucket back to the leaf plan, which reads S)
                K *const oc = padbuf + d.ocs;
                const uint32_t cap = (uint32_t)cap_keys;
                for (int p = tid; p < cnt; p += NT) {
                    const K key = skeys[p];
                    const int t = sub_range_of(key, shift, lo, mul, ns);
                    const uint32_t r = (uint32_t)p + sdelta[t];
                    if (r < (uint32_t)(t + 1) * cap) oc[r] = key;
                }
            } else if (bmap == nullptr) {
                K *const oc = F + d.ocs;
                for (int p = tid; p < cnt; p += NT) {
                    const K key = skeys[p];
                    oc[(uint32_t)p + sdelta[sub_range_of(key, shift, lo, mul, ns)]] = key;
                }
            } else {
                K *const oc = F + d.ocs;
                for (int p = tid; p < cnt; p += NT) {
                    const K key = skeys[p];
                    oc[(uint32_t)p + sdelta[__ldg(bmap + fine_bin<K>(key, shift, lo, fmul))]] = key;
                }
            }
        }
        __syncthreads();  // staging buffer and sd[cb] free
    }
}

// ------------------------------------------------------------- constant pieces
// Every CTA walks the split tables of the buckets tracked for constant pieces
// and writes, grid-strided inside each constant piece, its key over the piece's
// range of tile_out (where the tile sort of split buckets writes); the tile
// sort then only writes the piece's samples.  A fill, not a copy: the key is
// the piece's min == max from the count pass.
template <typename K>
__global__ void __launch_bounds__(256) k_split_fill(const Ctl *__restrict__ ctl, const uint32_t *__restrict__ tab,
                                                    SplitConst sc, K *tile_out) {
    griddep_wait();  // PDL: the scatter has read its input (tile_out may be that buffer)
    const unsigned nc = ctl->split.nconst;
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x, gstride = (long long)gridDim.x * blockDim.x;
    for (unsigned i = 0; i < nc; ++i) {
        // a bucket that still fell back (another piece over the limit and not constant) keeps its
        // partitioned keys where tile_out may point: its constant pieces are not filled
        if (!ctl->plan.split[sc.clist[3 * i + 2]]) continue;
        const long long w = (long long)sc.clist[3 * i], cs = (long long)sc.clist[3 * i + 1];
        const unsigned long long u = sc.gmax[w];
        K val;
        if constexpr (sizeof(K) == 4) val = (K)(int32_t)((uint32_t)u ^ 0x80000000u);
        else val = (K)(long long)(u ^ 0x8000000000000000ull);
        K *const o = tile_out + cs + tab[w];
        const long long len = (long long)tab[w + 1] - tab[w];
        HS_DASSERT(len >= 0 && sc.cflag[w] == 1 && sc.gmax[w] == ~sc.gminc[w]);
        for (long long p = gtid; p < len; p += gstride) o[p] = val;
    }
}

// ------------------------------------------------------------- per-chunk scan
__global__ void __launch_bounds__(kSplitPlanNT) k_split_plan(Ctl *ctl, uint32_t *tab, uint32_t *cur, int tile_keys,
                                                            SplitConst sc) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    __shared__ uint32_t wsum[kSplitPlanNT / 32];
    __shared__ bool s_last;
    Plan &P = ctl->plan;
    SplitCfg &C = ctl->split;
    const int tid = threadIdx.x;
    const int lg = P.log2c;
    const int b = blockIdx.x >> lg;
    const long long j = blockIdx.x & ((1 << lg) - 1);
    if (b < 10 && C.cand[b] && split_pmode(C, b)) {
        // padded layout: nothing was counted; the scatter's cursors start at the regions
        const int ns = P.nsb[b];
        uint32_t *crow = cur + P.sboff[b] + j * (ns + 1);
        for (int q = tid; q < ns; q += kSplitPlanNT) crow[q] = (uint32_t)q * (uint32_t)C.cap;
    } else if (b < 10 && C.cand[b]) {
        const int ns = P.nsb[b];
        uint32_t *row = tab + P.sboff[b] + j * (ns + 1);
        uint32_t *crow = cur + P.sboff[b] + j * (ns + 1);
        bool over = false;
        const long long rb = P.sboff[b] + j * (ns + 1);
        for (int q = tid; q < ns; q += kSplitPlanNT) {
            if (row[q] <= ((uint32_t)tile_keys << kBigLog2)) continue;  // the tile sort takes up to 2^kBigLog2 tiles
            // longer: legal only if every key of the piece is the same (already sorted)
            if (C.cc[b] && sc.gmax[rb + q] == ~sc.gminc[rb + q]) {
                sc.cflag[rb + q] = 1;
                const unsigned slot = atomicAdd(&C.nconst, 1u);  // k_split_fill's work list
                sc.clist[3 * slot] = (unsigned long long)(rb + q);
                sc.clist[3 * slot + 1] = (unsigned long long)(P.off[b] + part_start(P.off[b + 1] - P.off[b], P.log2c, j));
                sc.clist[3 * slot + 2] = (unsigned long long)b;
            } else {
                over = true;
            }
        }
        if (__syncthreads_or(over) && tid == 0) atomicOr(&C.bad, 1u << b);
        cta_excl_scan<kSplitPlanNT>(row, ns, wsum);
        for (int q = tid; q < ns; q += kSplitPlanNT) crow[q] = row[q];
        if (tid == 0) {
            const long long m = P.off[b + 1] - P.off[b];
            const long long len = part_start(m, lg, j + 1) - part_start(m, lg, j);
            row[ns] = (uint32_t)len;
            HS_DASSERT(ns < 1 || row[ns - 1] <= (uint32_t)len);
        }
    }
    // the last CTA to finish turns the candidates without an over-full
    // sub-range into split buckets and re-derives the leaf prefix
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&C.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last || tid != 0) return;
    __threadfence();
    const unsigned bad = *(volatile unsigned *)&C.bad;
    const long long c = 1LL << lg;
    long long acc = 0;
    int lmax = 0;
    for (int bb = 0; bb < 10; ++bb) {
        const int sp = C.cand[bb] && !((bad >> bb) & 1u);
        P.split[bb] = sp;
        if (sp) {
            P.k[bb] = 0;
            P.L[bb] = lg;  // only the chunk tree (a6) remains
        }
        P.tile_prefix[bb] = acc;
        acc += sp ? c * P.nsb[bb] : (c << P.k[bb]);
        lmax = P.L[bb] > lmax ? P.L[bb] : lmax;
    }
    P.tile_prefix[10] = acc;
    P.Lmax = lmax;
}

// ------------------------------------------------------- padded layout plan
// After the scatter, one CTA per chunk of a padded bucket: the final cursor of
// region t is t cap + (keys of sub-range t), so the counts come for free; their
// exclusive scan is the split table row the tile sort reads (where each sorted
// sub-range goes inside the chunk).  A region whose cursor passed its end
// (more than a tile of keys: the sample missed a skew) sends the bucket back to
// the tile + in-chunk merge-level plan -- its keys are still intact in S, and
// the tile sort then reads them there.  The last CTA re-derives the leaf prefix
// and Lmax.
__global__ void __launch_bounds__(kSplitPlanNT) k_split_pad_plan(Ctl *ctl, uint32_t *tab, const uint32_t *cur) {
    griddep_wait();  // PDL: the scatter's cursor atomics are complete
    __shared__ uint32_t wsum[kSplitPlanNT / 32];
    __shared__ bool s_last;
    Plan &P = ctl->plan;
    SplitCfg &C = ctl->split;
    const int tid = threadIdx.x;
    const int lg = P.log2c;
    const int b = blockIdx.x >> lg;
    const long long j = blockIdx.x & ((1 << lg) - 1);
    if (b < 10 && C.cand[b] && P.split[b] && split_pmode(C, b)) {
        const int ns = P.nsb[b];
        uint32_t *row = tab + P.sboff[b] + j * (ns + 1);
        const uint32_t *crow = cur + P.sboff[b] + j * (ns + 1);
        const uint32_t cap = (uint32_t)C.cap;
        bool over = false;
        for (int q = tid; q < ns; q += kSplitPlanNT) {
            const uint32_t k = crow[q] - (uint32_t)q * cap;
            over |= k > cap;
            row[q] = k;
        }
        if (__syncthreads_or(over) && tid == 0) atomicOr(&C.bad, 1u << b);
        cta_excl_scan<kSplitPlanNT>(row, ns, wsum);
        if (tid == 0) {
            const long long m = P.off[b + 1] - P.off[b];
            row[ns] = (uint32_t)(part_start(m, lg, j + 1) - part_start(m, lg, j));
            HS_DASSERT(over || row[ns - 1] <= row[ns]);
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&C.ticket2, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last || tid != 0) return;
    __threadfence();
    const unsigned bad = *(volatile unsigned *)&C.bad;
    const long long c = 1LL << lg;
    long long acc = 0;
    int lmax = 0;
    for (int bb = 0; bb < 10; ++bb) {
        if (P.split[bb] && ((bad >> bb) & 1u)) {  // a padded bucket that overflowed: the leaf plan
            P.split[bb] = 0;
            P.k[bb] = C.k0[bb];
            P.L[bb] = C.k0[bb] + lg;
        }
        P.tile_prefix[bb] = acc;
        acc += P.split[bb] ? c * P.nsb[bb] : (c << P.k[bb]);
        lmax = P.L[bb] > lmax ? P.L[bb] : lmax;
    }
    P.tile_prefix[10] = acc;
    P.Lmax = lmax;
}

// ------------------------------------------------------------------ host
// words after the split table: fine histograms (u32) and sampled maps (u16) of the 10 buckets
static long long split_extra_words(int log2c) {  // the sampled maps (u16) after the split table
    const long long mc = (1LL << log2c) <= kMapChunksMax ? (1LL << log2c) : 1;
    return 10LL * mc * kSplitFine / 2;
}

// The cursor region (split_cur_words) holds the cursors, then the SplitConst arrays.
SplitConst split_const(uint32_t *cur, long long tab_words) {
    const long long tw = (tab_words + 1) & ~1LL;  // 8-byte alignment of the 64-bit arrays
    SplitConst sc;
    sc.gminc = reinterpret_cast<unsigned long long *>(cur + tw);
    sc.gmax = sc.gminc + tw;
    sc.cflag = reinterpret_cast<uint32_t *>(sc.gmax + tw);
    sc.clist = reinterpret_cast<unsigned long long *>(sc.cflag + tw);
    return sc;
}

long long split_cur_words(long long tab_words) { return 12 * ((tab_words + 1) & ~1LL); }

long long split_table_words(long long n, int log2c, int tile_keys) {
    return n / split_target_map(tile_keys) + 40 * (1LL << log2c) + 64 + split_extra_words(log2c);
}

static int nsb_bound(long long n, int log2c, int tile_keys) {
    const long long c = 1LL << log2c, cm = (n + c - 1) / c, t = split_target_map(tile_keys);
    const long long ns = (cm + t - 1) / t;
    return (int)(ns < kSplitMaxSub ? (ns < 2 ? 2 : ns) : kSplitMaxSub);
}

int g_split_sms[kMaxDevices];

// dynamic shared memory of the count / scatter passes at the largest sub-range count (kSplitMaxSub)
template <typename K>
cudaError_t setup_split_t() {
    using G = SplGeo<K>;
    constexpr int TS = G::NT * G::VT;
    const size_t sm_count = (((size_t)(kSplitMaxSub + 1) * 4 + 15) & ~(size_t)15) + (size_t)(kSplitMaxSub + 1) * (sizeof(K) + 1);
    const size_t sm_scat =
        (((size_t)(kSplitMaxSub + 1) * 4 + 15) & ~(size_t)15) + (size_t)(kSplitMaxSub + 1) * 8 + (size_t)TS * sizeof(K);
    cudaError_t e = cudaFuncSetAttribute(k_split_count<K, G::NT, G::VT, G::MINB_COUNT, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_count);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_split_count<K, G::NT, G::VT, G::MINB_COUNT, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_count);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_split_scatter<K, G::NT, G::VT, G::MINB_SCAT, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_scat);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_split_scatter<K, G::NT, G::VT, G::MINB_SCAT, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_scat);
}

cudaError_t setup_split_kernels(int dev) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    g_split_sms[dev] = sms > 0 ? sms : 148;
    if ((e = setup_split_t<int32_t>()) != cudaSuccess) return e;
    return setup_split_t<int64_t>();
}

// Keys of the pad buffer: c nsb0[b] regions of one tile per bucket, nsb0[b] = ceil(ceil(m_b / c) / 0.9 T)
// <= (m_b + c) / (0.9 T) + 1, summed over the ten buckets.
long long split_pad_keys(long long n, int log2c, int tile_keys) {
    const long long c = 1LL << log2c, t = split_target(tile_keys);
    return ((n + 10 * c) + t - 1) / t * tile_keys + 10 * c * (long long)tile_keys + 64;
}

#ifdef HS_DEBUG
#define HS_SPLIT_STEP(i)                                                             \
    do {                                                                             \
        cudaError_t _s = cudaStreamSynchronize(st);                                  \
        if (_s != cudaSuccess) {                                                     \
            fprintf(stderr, "HS_DEBUG: K5a step %d: %s\n", i, cudaGetErrorString(_s)); \
            return _s;                                                               \
        }                                                                            \
    } while (0)
#else
#define HS_SPLIT_STEP(i) \
    do {                 \
    } while (0)
#endif

template <typename K>
static cudaError_t launch_split_t(Ctl *ctl, const K *S, K *F, uint32_t *tab, uint32_t *cur, long long tab_words,
                                  long long n, int log2c, int tile_keys, unsigned long long div, int key_shift,
                                  K *tile_out, K *padbuf, long long pad_keys, cudaStream_t st) {
    using G = SplGeo<K>;
    constexpr int TS = G::NT * G::VT;
    const int nsb_cap = nsb_bound(n, log2c, tile_keys);
    const size_t sm_count = (((size_t)(nsb_cap + 1) * 4 + 15) & ~(size_t)15) + (size_t)(nsb_cap + 1) * (sizeof(K) + 1);
    const SplitConst sc = split_const(cur, tab_words);
    const size_t sm_scat =
        (((size_t)(nsb_cap + 1) * 4 + 15) & ~(size_t)15) + (size_t)(nsb_cap + 1) * 8 + (size_t)TS * sizeof(K);
    auto kc = k_split_count<K, G::NT, G::VT, G::MINB_COUNT, false>;
    auto kcc = k_split_count<K, G::NT, G::VT, G::MINB_COUNT, true>;
    auto ks = k_split_scatter<K, G::NT, G::VT, G::MINB_SCAT, false>;
    auto ksc = k_split_scatter<K, G::NT, G::VT, G::MINB_SCAT, true>;
    cudaError_t e;
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    const int sms = g_split_sms[dev];
    const long long c = 1LL << log2c;
    const long long grid = n / TS + 20 * c + 16;  // >= sum over buckets of c * ceil(chunk / TS)
    const long long tab_cap = tab_words - split_extra_words(log2c);
    uint16_t *const map = reinterpret_cast<uint16_t *>(tab + tab_cap);
    prof_begin(kProfPlan, st);
    if ((e = launch_pdl(k_split_setup, dim3(1), dim3(1024), 0, st, ctl, div, 8 * (int)sizeof(K), key_shift,
                        tile_keys, TS, tab_cap, nsb_cap, tab, sc, padbuf ? pad_keys : 0LL)) != cudaSuccess)
        return e;
    HS_SPLIT_STEP(0);
    const int mc = (1LL << log2c) <= kMapChunksMax ? (int)(1LL << log2c) : 1;
    if ((e = launch_pdl(k_split_sample_map<K>, dim3(10 * mc), dim3(1024), 0, st, ctl, S, map, tile_keys)) !=
        cudaSuccess)
        return e;
    HS_SPLIT_STEP(1);
    prof_end(kProfPlan, st);
    prof_begin(kProfSplitCount, st);
    const long long pgrid = grid < (long long)sms * G::MINB_COUNT ? grid : (long long)sms * G::MINB_COUNT;
    if ((e = launch_pdl(kc, dim3((unsigned)pgrid), dim3(G::NT), sm_count, st, ctl, S, tab, nsb_cap, map, sc)) !=
        cudaSuccess)
        return e;
    HS_SPLIT_STEP(2);
    if ((e = launch_pdl(kcc, dim3((unsigned)pgrid), dim3(G::NT), sm_count, st, ctl, S, tab, nsb_cap, map, sc)) !=
        cudaSuccess)
        return e;
    HS_SPLIT_STEP(3);
    prof_end(kProfSplitCount, st);
    prof_begin(kProfPlan, st);
    if ((e = launch_pdl(k_split_plan, dim3((unsigned)(10 * c)), dim3(kSplitPlanNT), 0, st, ctl, tab, cur,
                        tile_keys, sc)) != cudaSuccess)
        return e;
    HS_SPLIT_STEP(4);
    prof_end(kProfPlan, st);
    prof_begin(kProfSplitScatter, st);
    const long long sgrid = grid < (long long)sms * G::MINB_SCAT ? grid : (long long)sms * G::MINB_SCAT;
    if ((e = launch_pdl(ks, dim3((unsigned)sgrid), dim3(G::NT), sm_scat, st, ctl, S, F, cur, nsb_cap, map, padbuf,
                        tile_keys)) != cudaSuccess)
        return e;
    if ((e = launch_pdl(ksc, dim3((unsigned)sgrid), dim3(G::NT), sm_scat, st, ctl, S, F, cur, nsb_cap, map, padbuf,
                        tile_keys)) != cudaSuccess)
        return e;
    HS_SPLIT_STEP(5);
    prof_end(kProfSplitScatter, st);
    prof_begin(kProfPlan, st);
    if ((e = launch_pdl(k_split_pad_plan, dim3((unsigned)(10 * c)), dim3(kSplitPlanNT), 0, st, ctl, tab,
                        (const uint32_t *)cur)) != cudaSuccess)
        return e;
    HS_SPLIT_STEP(6);
    if ((e = launch_pdl(k_split_fill<K>, dim3((unsigned)(2 * sms)), dim3(256), 0, st, (const Ctl *)ctl,
                        (const uint32_t *)tab, sc, tile_out)) != cudaSuccess)
        return e;
    HS_SPLIT_STEP(7);
    prof_end(kProfPlan, st);
    return cudaGetLastError();
}

cudaError_t launch_split(int dt, Ctl *ctl, const void *S, void *F, uint32_t *tab, uint32_t *cur, long long tab_words,
                         long long n, int log2c, int tile_keys, unsigned long long div, int key_shift, void *tile_out,
                         void *padbuf, long long pad_keys, cudaStream_t st) {
    return dt == 0 ? launch_split_t<int32_t>(ctl, (const int32_t *)S, (int32_t *)F, tab, cur, tab_words, n, log2c,
                                             tile_keys, div, key_shift, (int32_t *)tile_out, (int32_t *)padbuf,
                                             pad_keys, st)
                   : launch_split_t<int64_t>(ctl, (const int64_t *)S, (int64_t *)F, tab, cur, tab_words, n, log2c,
                                             tile_keys, div, key_shift, (int64_t *)tile_out, (int64_t *)padbuf,
                                             pad_keys, st);
}

const uint32_t *split_cflag(uint32_t *cur, long long tab_words) { return split_const(cur, tab_words).cflag; }

}  // namespace hs
