// hs_device.cuh -- device-side building blocks shared by the sm_100a kernels
// of libhybridsort.so: key traits, the leading-decimal-digit function, the
// per-call plan (bucket / chunk / leaf-tile geometry) and thin PTX wrappers
// (bulk async copy, mbarrier, relaxed gpu-scope loads/stores).
//
// Nothing here is shared with oracle/ (the CPU checker).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "hs_launch.h"

// Device-side invariant checks of the debug build (libhybridsort_debug.so,
// -DHS_DEBUG; tests/test_debug_build.py): shared-memory indices, piece
// geometry, scatter positions.  compute-sanitizer is closed on this pool, so
// these asserts stand in for it.  Compiled out of the product library.
#ifdef HS_DEBUG
#include <cstdio>
#define HS_DASSERT(c)                                                                          \
    do {                                                                                       \
        if (!(c)) {                                                                            \
            printf("HS_DASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                         \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define HS_DASSERT(c) \
    do {              \
    } while (0)
#endif

namespace hs {

// --------------------------------------------------------------- key traits
template <typename K>
struct KeyTraits;
template <>
struct KeyTraits<int32_t> {
    using U = uint32_t;
    static constexpr int32_t kMax = 0x7fffffff;
};
template <>
struct KeyTraits<int64_t> {
    using U = unsigned long long;
    static constexpr int64_t kMax = 0x7fffffffffffffffLL;
};

// SURVEY f3 key + tag item of the stable path (hs_sort_pairs on int64 keys,
// hs_merge_pairs, ...): SPEC's SortItem -- the tag travels with
// its key through every pass and "never influences order": items compare by
// key only, so equal keys keep whatever order the kernels give them, and the
// kernels that see items are all stable (the K3 counting scatter, a stable
// in-tile sort, stable-left merges).  16 bytes: one bulk-copy granule.
struct __align__(16) KV64 {
    long long k;
    unsigned long long v;
};
__host__ __device__ __forceinline__ bool operator<(const KV64 &a, const KV64 &b) { return a.k < b.k; }
__host__ __device__ __forceinline__ bool operator<=(const KV64 &a, const KV64 &b) { return a.k <= b.k; }
__host__ __device__ __forceinline__ bool operator>(const KV64 &a, const KV64 &b) { return a.k > b.k; }
template <>
struct KeyTraits<KV64> {
    using U = unsigned long long;
    static constexpr KV64 kMax = {0x7fffffffffffffffLL, 0ull};
};

// Does a merge of K need explicit run ends?  Keys-only merges let an
// exhausted run read as kMax (equal keys are interchangeable); items are not.
template <typename K>
struct ExactEnds {
    static constexpr bool value = false;
};
template <>
struct ExactEnds<KV64> {
    static constexpr bool value = true;
};

// Leading decimal digit of a D-digit key, d(k) = clamp(floor(k / 10^(D-1)), 0, 9)
// (reading #1 zero-padding, #3 clamping).  Division by the runtime
// constant div = 10^(D-1) is exact by one multiply-high and a shift: magic =
// ceil(2^(N+l) / div), l = ceil(log2 div), N = w - 1, valid for every key in
// [0, 2^(w-1)) (Granlund-Montgomery, K1); post = l - 1, or -1
// for div = 1 (the digit is the key itself).
template <typename K>
struct DigitParams {
    typename KeyTraits<K>::U div;
    typename KeyTraits<K>::U magic;
    int shift;  // int64 only: the key is k >> shift (32 for the (key << 32 | index) items of hs_sort_pairs)
    int post;   // post-shift of the multiply-high
};

__device__ __forceinline__ int msd_digit(int32_t k, const DigitParams<int32_t> &p) {
    const uint32_t u = (uint32_t)(k > 0 ? k : 0);  // negative keys clamp to digit 0
    const uint32_t q = p.post >= 0 ? __umulhi(u, p.magic) >> p.post : u;
    return (int)(q < 9u ? q : 9u);
}

__device__ __forceinline__ int msd_digit(int64_t k, const DigitParams<int64_t> &p) {
    k >>= p.shift;  // arithmetic: keeps the sign of the key
    const unsigned long long u = (unsigned long long)(k > 0 ? k : 0);
    const unsigned long long q = p.post >= 0 ? __umul64hi(u, p.magic) >> p.post : u;
    return (int)(q < 9ull ? q : 9ull);
}

__device__ __forceinline__ int msd_digit(const KV64 &it, const DigitParams<KV64> &p) {
    const unsigned long long u = (unsigned long long)(it.k > 0 ? it.k : 0);
    const unsigned long long q = p.post >= 0 ? __umul64hi(u, p.magic) >> p.post : u;
    return (int)(q < 9ull ? q : 9ull);
}

// Programmatic dependent launch (PDL): the kernels of hs_sort after K1 are
// launched with programmatic stream serialization, so each may be scheduled
// while its predecessor drains; every such kernel calls griddep_wait() first
// (full completion + memory flush of the predecessor) before touching memory.
// A no-op for a kernel launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    if (e == cudaSuccess) note_launch();
    return e;
}

// ------------------------------------------------------------------- plan
// Geometry of one call, computed on the device (no host sync).
//  * bucket b = [off[b], off[b+1]).
//  * chunks: partition_even(m_b, c).
//  * leaf tiles: each chunk is split by partition_even into 2^k[b] leaves of
//    at most T keys (T = tile-sort capacity); k[b] is chosen from the largest
//    chunk, so every chunk of a bucket has the same power-of-two leaf count
//    and the bucket's merge tree over its c * 2^k[b] leaves is perfect (no
//    pass-through runs, hence no copies).
//  * merge level lam of bucket b merges leaf runs [2p 2^lam, (2p+1) 2^lam) and
//    [(2p+1) 2^lam, (2p+2) 2^lam).  Levels lam < k[b] are the in-chunk
//    merges of a5; levels k[b] .. k[b]+log2 c - 1 are the paper's tree merge
//    of the chunks (a6).
//  * L[b] = number of merge levels this call runs for bucket b.
//  * split[b] = 1 (hs_sort, K5a): every chunk of bucket b was split by key
//    value into nsb[b] sub-ranges, each at most T keys; the tile-sort leaves
//    are those sub-ranges (bounds in the split table at sboff[b]), k[b] = 0
//    and the merge levels are only the paper's chunk tree (L[b] = log2 c).
struct Plan {
    long long off[11];
    long long tile_prefix[11];  // exclusive prefix of tile-sort leaf counts (c << k[b], or c * nsb[b])
    long long sboff[10];        // split table: chunk j of bucket b owns [sboff + j (nsb+1), ... + nsb]
    int k[10];
    int L[10];
    int split[10];
    int nsb[10];
    int log2c;
    int Lmax;
};

// K5a bookkeeping (value split of the chunks), written by k_split_setup and
// k_split_map.  Fine bins: kSplitFine equal-width bins of a bucket's digit
// range, the unit of the sampled sub-range map of skewed buckets (fine enough
// that one bin near a C4-like peak holds ~0.06 T keys of a chunk).
constexpr int kSplitFine = 8192;
constexpr int kMapChunksMax = 64;  // per-chunk sampled maps up to this many chunks per bucket
struct SplitCfg {
    long long slice_prefix[11];  // CTAs of the count / scatter passes per bucket (c * spc[b])
    long long lo[10];            // bucket b's value range starts at b * 10^(D-1)
    unsigned long long mul[10];  // sub-range of x = mulhi(x - lo, mul), mul = floor((2^w - 1) / 10^(D-1)) nsb[b]
    unsigned long long fmul[10]; // fine bin of x = min(mulhi(x - lo, fmul), kSplitFine - 1) (0: no fine bins)
    int spc[10];                 // slices per chunk
    int cand[10];                // bucket b is split if no sub-range of its chunks exceeds T
    int mode[10];                // 0: equal-width sub-ranges (mul); 1: sub-range = map[b][fine bin] (skewed bucket)
    int nsa[10];                 // split-table row capacity per chunk - 1 (nsb[b] <= nsa[b])
    int ns0[10];                 // equal-width sub-ranges per chunk (nsb[b] before any map)
    int cc[10];                  // track constant sub-ranges (the sample saw a fine bin of > T keys per chunk)
    int map_chunks;              // sampled maps per bucket: c (one per chunk) or 1 (c > kMapChunksMax)
    unsigned bad;                // buckets with an over-full sub-range (fall back to merge levels)
    unsigned ticket;
    unsigned nconst;             // constant pieces listed for k_split_fill
    int shift;                   // sort key of an item = item >> shift (hs_sort_pairs)
    // padded layout (no count pass): an equal-width bucket without constant tracking gives every
    // (chunk, sub-range) a fixed region of cap keys in the pad buffer; the scatter's cursors count
    // the keys, k_split_pad_plan turns the final cursors into the split table (or, if a region
    // overflowed, sends the bucket back to the tile + merge-level plan)
    int pad[10];                 // setup: the pad buffer has room for bucket b (see split_pmode)
    int k0[10];                  // the leaf plan's k[b] (restored by a padded bucket that overflows)
    long long pboff[10];         // bucket b's regions start here in the pad buffer (keys)
    int cap;                     // keys per region (one tile)
    unsigned ticket2;            // k_split_pad_plan's last-CTA ticket
};

// Padded layout for bucket b: room in the pad buffer, equal-width sub-ranges (the
// sample found no skew) and no constant tracking.
__host__ __device__ __forceinline__ bool split_pmode(const SplitCfg &C, int b) {
    return C.pad[b] && !C.mode[b] && !C.cc[b];
}

enum PlanMode { kPlanSort = 0, kPlanChunks = 1, kPlanMerge = 2 };

// A K5a sub-range piece may hold up to 2^kBigLog2 tiles (duplicate-heavy or
// skewed sub-ranges): its CTA sorts it as tiles + CTA-level merges (K5).
constexpr int kBigLog2 = 2;

__device__ __forceinline__ int ceil_log2_ll(long long x) {  // x >= 1
    int r = 0;
    while ((1LL << r) < x) ++r;
    return r;
}

// One thread fills *P from off[11].
__device__ inline void compute_plan(Plan *P, const long long *off, int log2c, int mode, int tile_keys) {
    long long c = 1LL << log2c;
    long long acc = 0;
    int lmax = 0;
    for (int b = 0; b < 10; ++b) {
        long long m = off[b + 1] - off[b];
        int k = 0;
        if (mode != kPlanMerge) {
            long long cm = (m + c - 1) / c;                        // largest chunk
            long long tiles = (cm + tile_keys - 1) / tile_keys;    // leaves it needs
            k = tiles > 1 ? ceil_log2_ll(tiles) : 0;
        }
        int L = (mode == kPlanSort) ? k + log2c : (mode == kPlanChunks ? k : log2c);
        P->off[b] = off[b];
        P->split[b] = 0;
        P->nsb[b] = 0;
        P->sboff[b] = 0;
        P->k[b] = k;
        P->L[b] = L;
        P->tile_prefix[b] = acc;
        acc += (c << k);
        lmax = L > lmax ? L : lmax;
    }
    P->off[10] = off[10];
    P->tile_prefix[10] = acc;
    P->log2c = log2c;
    P->Lmax = lmax;
}

// Start of part i of partition_even(m, p = 2^lg): i*floor(m/p) + min(i, m mod p).
__device__ __forceinline__ long long part_start(long long m, int lg, long long i) {
    long long q = m >> lg, r = m & ((1LL << lg) - 1);
    return i * q + (i < r ? i : r);
}

// Index of the part of partition_even(m, 2^lg) containing y (0 <= y < m).
__device__ __forceinline__ long long part_index(long long m, int lg, long long y) {
    long long q = m >> lg, r = m & ((1LL << lg) - 1);
    long long B = r * (q + 1);
    // positions < 2^31 (ABI limit): 32-bit unsigned division is exact here
    if (y < B) return (long long)((unsigned)y / (unsigned)(q + 1));
    return r + (long long)((unsigned)(y - B) / (unsigned)q);
}

// Absolute start of leaf i of bucket b (0 <= i <= c << k[b]).
__device__ __forceinline__ long long leaf_start(const Plan &P, int b, long long i) {
    long long m = P.off[b + 1] - P.off[b];
    int k = P.k[b];
    long long j = i >> k, t = i & ((1LL << k) - 1);
    long long cs = part_start(m, P.log2c, j);
    if (t == 0) return P.off[b] + cs;
    long long q = m >> P.log2c, r = m & ((1LL << P.log2c) - 1);
    long long len = q + (j < r ? 1 : 0);
    return P.off[b] + cs + part_start(len, k, t);
}

// Leaf of bucket b containing absolute position x (off[b] <= x < off[b+1]).
__device__ __forceinline__ long long leaf_of(const Plan &P, int b, long long x) {
    long long m = P.off[b + 1] - P.off[b];
    int k = P.k[b];
    long long y = x - P.off[b];
    long long j = part_index(m, P.log2c, y);
    if (k == 0) return j;
    long long q = m >> P.log2c, r = m & ((1LL << P.log2c) - 1);
    long long len = q + (j < r ? 1 : 0);
    long long z = y - part_start(m, P.log2c, j);
    return (j << k) + part_index(len, k, z);
}

__device__ __forceinline__ int bucket_of(const Plan &P, long long x) {
    int b = 0;
    while (b < 9 && x >= P.off[b + 1]) ++b;
    return b;
}

// Pair geometry at merge level lam for the pair containing leaf lf.
struct PairGeom {
    long long a_lo, b_lo, b_hi;
};
__device__ __forceinline__ PairGeom pair_of(const Plan &P, int b, long long lf, int lam) {
    long long p = lf >> (lam + 1);
    PairGeom g;
    g.a_lo = leaf_start(P, b, p << (lam + 1));
    g.b_lo = leaf_start(P, b, ((2 * p + 1) << lam));
    g.b_hi = leaf_start(P, b, (p + 1) << (lam + 1));
    return g;
}

// Which buffer holds bucket b's runs before level lam: the last level
// (L-1) must write the final buffer F, so the data before level lam sits in
// F iff (L - lam) is even.
template <typename K>
__device__ __forceinline__ K *level_src(const Plan &P, int b, int lam, K *F, K *S) {
    return ((P.L[b] - lam) & 1) == 0 ? F : S;
}
template <typename K>
__device__ __forceinline__ K *level_dst(const Plan &P, int b, int lam, K *F, K *S) {
    return ((P.L[b] - 1 - lam) & 1) == 0 ? F : S;
}

// Per-call control block (zeroed by one memset before the first kernel).
struct Ctl {
    unsigned long long hist[10];
    unsigned int done;
    unsigned int ticket;
    long long off[11];
    Plan plan;
    SplitCfg split;
};

// --------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk async copy (TMA engine) global -> shared, completion counted in
// bytes on the mbarrier.  dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int4 ld_stream_v4(const void *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Padded shared-memory index: one spare word per 32 keys so that a thread
// reading VT consecutive keys (blocked layout) and a warp reading 32
// consecutive keys (striped layout) are both bank-conflict free.
__device__ __forceinline__ int pad_idx(int i) { return i + (i >> 5); }

template <typename K>
__device__ __forceinline__ void cas(K &a, K &b) {
    K lo = a < b ? a : b;
    K hi = a < b ? b : a;
    a = lo;
    b = hi;
}

// Two 16-bit keys per register (the tile sort's packed bucket sort): one
// comparator orders both halves at once (vmin2/vmax2 = one SIMD op each).
struct H2 {
    uint32_t v;
};
__device__ __forceinline__ void cas(H2 &a, H2 &b) {
    const uint32_t lo = __vminu2(a.v, b.v), hi = __vmaxu2(a.v, b.v);
    a.v = lo;
    b.v = hi;
}

// Batcher odd-even merge sort network on N registers.  The comparator list
// is generated at compile time (comparators touching an index >= N are
// dropped, i.e. the input is padded with +inf, valid for any N), so the
// unrolled loop below has constant register indices and v stays in registers.
template <int N>
struct OddEvenNet {
    int a[N * N], b[N * N];
    int n;
    constexpr OddEvenNet() : a(), b(), n(0) {
        for (int p = 1; p < N; p <<= 1)
            for (int k = p; k >= 1; k >>= 1)
                for (int j = k % p; j + k < N; j += 2 * k)
                    for (int i = 0; i < k; ++i)
                        if (i + j + k < N && (i + j) / (2 * p) == (i + j + k) / (2 * p)) {
                            a[n] = i + j;
                            b[n] = i + j + k;
                            ++n;
                        }
    }
};

template <int N>
struct OddEvenNetHolder {
    static constexpr OddEvenNet<N> net{};
};

// Comparators applied by template recursion, so every register index is a
// compile-time constant however long the network is.
template <int N, int C>
struct OECmp {
    static constexpr int n = OddEvenNetHolder<N>::net.n;
    static constexpr int a = C < n ? OddEvenNetHolder<N>::net.a[C] : 0;
    static constexpr int b = C < n ? OddEvenNetHolder<N>::net.b[C] : 0;
};

template <int N, int C, typename K>
__device__ __forceinline__ void oddeven_cmp(K (&v)[N]) {
    if constexpr (C < OECmp<N, C>::n) cas(v[OECmp<N, C>::a], v[OECmp<N, C>::b]);
}

// 16 comparators per recursion level (keeps the instantiation depth low for
// long networks)
template <int N, int C, typename K>
__device__ __forceinline__ void oddeven_apply(K (&v)[N]) {
    if constexpr (C < OECmp<N, C>::n) {
        oddeven_cmp<N, C + 0>(v);
        oddeven_cmp<N, C + 1>(v);
        oddeven_cmp<N, C + 2>(v);
        oddeven_cmp<N, C + 3>(v);
        oddeven_cmp<N, C + 4>(v);
        oddeven_cmp<N, C + 5>(v);
        oddeven_cmp<N, C + 6>(v);
        oddeven_cmp<N, C + 7>(v);
        oddeven_cmp<N, C + 8>(v);
        oddeven_cmp<N, C + 9>(v);
        oddeven_cmp<N, C + 10>(v);
        oddeven_cmp<N, C + 11>(v);
        oddeven_cmp<N, C + 12>(v);
        oddeven_cmp<N, C + 13>(v);
        oddeven_cmp<N, C + 14>(v);
        oddeven_cmp<N, C + 15>(v);
        oddeven_apply<N, C + 16>(v);
    }
}

template <int N, typename K>
__device__ __forceinline__ void oddeven_sort(K (&v)[N]) {
    oddeven_apply<N, 0>(v);
}


// ------------------------------------------------------------ key samples
// Every kernel that writes a generation of the sorted runs (the tile sort,
// each merge level) also writes samp[p / kSampleQ] = key at position p for
// every p = kSampleQ - 1 (mod kSampleQ).  The next merge level's co-rank
// search runs its coarse phase on these samples (1/kSampleQ of the data,
// stored with an L2 evict_last policy so they stay on chip while the level's
// 2 n s bytes stream past) and touches HBM only for the last ~kSampleQ keys.
constexpr int kSampleQ = 64;

__device__ __forceinline__ void st_keep(int32_t *p, int32_t v) {
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
        "st.global.L2::cache_hint.b32 [%0], %1, pol;\n}" ::"l"(p),
        "r"(v)
        : "memory");
}
__device__ __forceinline__ void st_keep(int64_t *p, int64_t v) {
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
        "st.global.L2::cache_hint.b64 [%0], %1, pol;\n}" ::"l"(p),
        "l"(v)
        : "memory");
}

__device__ __forceinline__ void st_keep(KV64 *p, KV64 v) {
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
        "st.global.L2::cache_hint.v2.b64 [%0], {%1, %2}, pol;\n}" ::"l"(p),
        "l"(v.k), "l"(v.v)
        : "memory");
}

// Read-only cached load of a key (structs have no __ldg overload).
template <typename K>
__device__ __forceinline__ K ldg_key(const K *p) {
    return __ldg(p);
}
template <>
__device__ __forceinline__ KV64 ldg_key<KV64>(const KV64 *p) {
    const longlong2 w = __ldg(reinterpret_cast<const longlong2 *>(p));
    return KV64{w.x, (unsigned long long)w.y};
}

// Write the samples of output positions [x, x + len) whose keys sit at
// stage[p - x] (shared memory), threads tid = 0 .. nthreads-1 cooperating.
template <typename K>
__device__ __forceinline__ void write_samples(K *samp, long long x, int len, const K *stage, int tid, int nthreads) {
    if (!samp) return;
    const long long f = x + (kSampleQ - 1 - x % kSampleQ);  // first sample position >= x
    for (long long p = f + (long long)tid * kSampleQ; p < x + len; p += (long long)nthreads * kSampleQ)
        st_keep(samp + p / kSampleQ, stage[p - x]);
}

}  // namespace hs
