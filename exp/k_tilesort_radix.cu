// k_tilesort.cu -- a4 (chunk plan from given offsets) and a5's first stage:
// the in-shared-memory sort of every leaf tile of every chunk.
//
//   K4 k_plan       chunk / leaf-tile geometry from caller-given offsets
//   K5 k_tile_sort  per-CTA sort of one leaf tile (<= T keys)
//
// The rest of a5 (in-chunk merge levels) and a6 are in k_merge.cu; a1-a3 in
// k_partition.cu.  Design notes and rooflines: DESIGN.md §5.
//
// K5 replaces the paper's per-thread sequential quicksort (Fig 1c, P:50,
// P:62) -- a data-dependent, branchy, serial algorithm that maps badly onto
// SIMT lanes -- by the GPU shape of the same "sort the partitions, then merge
// sorted lists pairwise" idea its parallel sorts are built from:
//   1. each thread sorts VT keys in registers (Batcher odd-even network,
//      compile-time register indices, no branches);
//   2. log2(NT) merge-path merge rounds in shared memory turn the NT sorted
//      runs into one (the binary-tree merge of P:58-60 at CTA scope).
// Keys-only data makes the sorted tile unique, so the (unstable) network
// order is unobservable.
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

#ifndef HS_SORT_NT
#define HS_SORT_NT 512
#endif
#ifndef HS_SORT_VT
#define HS_SORT_VT 27
#endif
#ifndef HS_SORT_MINB
#define HS_SORT_MINB 2
#endif
#ifndef HS_SORT_NT64
#define HS_SORT_NT64 512
#endif
#ifndef HS_SORT_VT64
#define HS_SORT_VT64 15
#endif
#ifndef HS_SORT_MINB64
#define HS_SORT_MINB64 2
#endif
#ifndef HS_TILE_MERGE
#define HS_TILE_MERGE 0  // 0: radix tile sort (default), 1: merge-path tile sort
#endif
#ifndef HS_RSORT_NT
#define HS_RSORT_NT 512
#endif
#ifndef HS_RSORT_VT
#define HS_RSORT_VT 26  // 13,312 int32 keys per leaf
#endif
#ifndef HS_RSORT_VT64
#define HS_RSORT_VT64 13  // 6,656 int64 keys per leaf
#endif

namespace hs {

__device__ __forceinline__ void load_plan(Plan &dst, const Plan *src) {
    static_assert(sizeof(Plan) % 4 == 0, "plan size");
    constexpr int W = sizeof(Plan) / 4;
    const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
    uint32_t *d = reinterpret_cast<uint32_t *>(&dst);
    for (int i = threadIdx.x; i < W; i += blockDim.x) d[i] = __ldg(s + i);
}

// =================================================================== K4
__global__ void k_plan(const long long *__restrict__ user_off, Ctl *ctl, int log2c, int mode, int tile_keys) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        long long off[11];
        for (int b = 0; b < 11; ++b) off[b] = user_off[b];
        compute_plan(&ctl->plan, off, log2c, mode, tile_keys);
    }
}

// K4 for hs_sort_shared (no MSD step): the whole array is bucket 0.
__global__ void k_plan_whole(Ctl *ctl, long long n, int log2c, int tile_keys) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        long long off[11];
        off[0] = 0;
        for (int b = 1; b < 11; ++b) off[b] = n;
        compute_plan(&ctl->plan, off, log2c, kPlanSort, tile_keys);
    }
}

// =================================================================== K5
// Block merge sort of one leaf tile in shared memory.
//   1. one 1-D bulk async copy (TMA engine) brings the leaf (a 16-byte aligned
//      superset of it) into shared memory; positions past the leaf are filled
//      with the dtype maximum (pads sort to the end, are never stored, and
//      equal any real maximum key, so the stored prefix is the same multiset);
//   2. thread t takes the VT consecutive keys t*VT .. t*VT+VT-1 (VT odd, so
//      the blocked reads and writes of a warp hit 32 distinct banks) and sorts
//      them in registers with Batcher's odd-even network (compile-time
//      register indices, no branches);
//   3. log2(NT) merge rounds: runs of R*VT keys are merged pairwise; every
//      thread finds the start of its VT outputs by a merge-path binary search
//      over the two runs in shared memory (ties take A) and merges VT
//      keys serially into registers.  Real keys always occupy positions
//      [0, len) (induction over the rounds), so a thread whose VT outputs all
//      lie at or past len skips the round (ragged leaves cost what they hold);
//   4. the sorted tile goes back to shared memory at the destination's 16-byte
//      phase and leaves with one 1-D bulk async store (+ scalar head/tail).
// This is the GPU shape of the paper's "sort partitions, then merge sorted
// lists pairwise in a binary tree" at CTA scope.
template <typename K>
__device__ __forceinline__ K kmin(K a, K b) { return a < b ? a : b; }
template <typename K>
__device__ __forceinline__ K kmax(K a, K b) { return a < b ? b : a; }

__device__ __forceinline__ void bulk_s2g_ts(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}

// Merge-path split of output diag between A = sm[a0, a0+na) and B = sm[b0, b0+nb) (stable-left).
template <typename K>
__device__ __forceinline__ int smem_merge_path(const K *sm, int a0, int na, int b0, int nb, int diag) {
    int l = diag - nb > 0 ? diag - nb : 0;
    int r = diag < na ? diag : na;
    while (l < r) {
        const int mid = (l + r) >> 1;
        if (sm[a0 + mid] <= sm[b0 + diag - 1 - mid]) l = mid + 1;
        else r = mid;
    }
    return l;
}

template <typename K, int NT, int VT>
struct TSGeo {
    static constexpr int T = NT * VT;
    static constexpr int E = 16 / sizeof(K);
    static constexpr size_t bytes() { return (size_t)(T + 2 * E) * sizeof(K); }
};

template <typename K, int NT, int VT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_tile_sort(const Plan *__restrict__ plan_g, const K *src, K *F, K *S,
                                                        K *samp) {
    static_assert(VT & 1, "odd VT keeps blocked shared-memory accesses conflict-free");
    using G = TSGeo<K, NT, VT>;
    constexpr int T = G::T, E = G::E;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const sbuf = reinterpret_cast<K *>(smem_raw);
    __shared__ Plan P;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    load_plan(P, plan_g);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const long long g = blockIdx.x;
    if (g >= P.tile_prefix[10]) return;
    int b = 0;
    while (b < 9 && g >= P.tile_prefix[b + 1]) ++b;
    const long long i = g - P.tile_prefix[b];
    const long long lo = leaf_start(P, b, i);
    const int len = (int)(leaf_start(P, b, i + 1) - lo);
    if (len == 0) return;
    K *const out = ((P.L[b] & 1) ? S : F) + lo;  // where this bucket's merge level 0 reads
    const K kMax = KeyTraits<K>::kMax;

    // 1. bulk load of the 16-byte aligned superset of the leaf
    const K *in = src + lo;
    const uintptr_t ga0 = (uintptr_t)in & ~(uintptr_t)15;
    const uintptr_t ga1 = ((uintptr_t)(in + len) + 15) & ~(uintptr_t)15;
    const int h = (int)(((uintptr_t)in - ga0) / sizeof(K));
    if (tid == 0) {
        mbar_arrive_expect_tx(&bar, (uint32_t)(ga1 - ga0));
        bulk_g2s(sbuf, (const void *)ga0, (uint32_t)(ga1 - ga0), &bar);
    }
    K *const sm = sbuf + h;  // sm[0 .. len) = the leaf
    mbar_wait(&bar, 0);
    for (int j = len + tid; j < T; j += NT) sm[j] = kMax;
    __syncthreads();

    // 2. register sort of VT consecutive keys
    K v[VT];
    const bool live0 = tid * VT < len;
#pragma unroll
    for (int k = 0; k < VT; ++k) v[k] = sm[tid * VT + k];
    if (live0) oddeven_sort<VT>(v);

    // 3. merge rounds (R = threads per run)
#pragma unroll 1
    for (int R = 1; R < NT; R <<= 1) {
        const bool live = tid * VT < len;
        __syncthreads();  // everyone has read the previous round's runs
        if (live) {
#pragma unroll
            for (int k = 0; k < VT; ++k) sm[tid * VT + k] = v[k];
        }
        __syncthreads();
        if (live) {
            const int j = tid & (2 * R - 1);
            const int a0 = (tid - j) * VT, run = R * VT, b0 = a0 + run;
            const int diag = j * VT;
            const int s = smem_merge_path(sm, a0, run, b0, run, diag);
            const int a_end = b0, b_end = b0 + run;
            int ai = a0 + s, bi = b0 + diag - s;
            K x = ai < a_end ? sm[ai] : kMax;
            K y = bi < b_end ? sm[bi] : kMax;
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                const bool p = x <= y;
                v[k] = p ? x : y;
                if (k + 1 < VT) {
                    const int nx = (p ? ai : bi) + 1;
                    const int lim = p ? a_end : b_end;
                    const K t = sm[nx];  // nx <= T: inside the buffer (T + 2E slots)
                    const K tv = nx < lim ? t : kMax;
                    ai = p ? nx : ai;
                    bi = p ? bi : nx;
                    x = p ? tv : x;
                    y = p ? y : tv;
                }
            }
        }
    }

    // 4. stage at the destination's 16-byte phase, bulk store the aligned middle
    const int sh = (int)(((uintptr_t)out & 15) / sizeof(K));
    K *const so = sbuf + sh;  // so[p] <-> out[p]
    __syncthreads();
    if (tid * VT < len) {
#pragma unroll
        for (int k = 0; k < VT; ++k) so[tid * VT + k] = v[k];
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int m0 = sh == 0 ? 0 : E - sh;            // first output at a 16-byte aligned address
    const int m1 = (sh + len) / E * E - sh;         // end of the aligned middle
    if (m1 > m0) {
        if (tid == 0) {
            bulk_s2g_ts(out + m0, so + m0, (uint32_t)((m1 - m0) * sizeof(K)));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (tid < m0) out[tid] = so[tid];
        else if (tid >= E && tid < 2 * E && m1 + tid - E < len) out[m1 + tid - E] = so[m1 + tid - E];
        if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else {
        for (int p = tid; p < len; p += NT) out[p] = so[p];
    }
    write_samples(samp, lo, len, so, tid, NT);  // coarse index for merge level 0's co-rank search
}

// =================================================================== K5 (radix)
// LSD radix sort of one leaf tile in shared memory (the default K5; the
// merge-path variant above is kept for comparison, -DHS_TILE_MERGE=1).
//   1. one 1-D bulk async copy brings the leaf into shared memory;
//   2. block min/max (warp shuffles): the tile only spans [min, max], so it
//      is sorted on the offsets k - min, which need bits(max - min) bits
//      (27 for a C3 leaf inside one decimal bucket, not 32);
//   3. P = ceil(bits / 7) stable counting passes of b = ceil(bits / P) <= 7
//      bits.  Warp w ranks the keys of its contiguous segment in input order
//      (iteration i, lane l = key w*S + 32 i + l): __match_any_sync groups
//      the lanes holding the same digit, the lowest of them bumps the warp's
//      16-bit counter for that digit, every lane keeps base + #lower peers.
//      A digit-major exclusive scan over the [warp][digit] counters turns
//      them into output offsets and each key is scattered into the other
//      buffer: stable, so after the last pass the tile is sorted;
//   4. the last pass scatters at the destination's 16-byte phase and the
//      tile leaves with one 1-D bulk async store (+ scalar head/tail).
// Keys-only data: the result equals any other ascending sort of the leaf.
template <typename K, int NT, int VT>
struct RSGeo {
    static constexpr int T = NT * VT;
    static constexpr int E = 16 / sizeof(K);
    static constexpr int NW = NT / 32;
    static constexpr int SEG = VT * 32;  // keys per warp segment
    static constexpr int RB = 7;         // max bits per pass
    static constexpr int BINS = 1 << RB;
    static constexpr int BUF = T + 2 * E;  // one key buffer (+ bulk-copy / store phase slack)
    static_assert((BUF * sizeof(K)) % 16 == 0, "buffers stay 16-byte aligned");
    static_assert(SEG < 65536 && T < 65536, "16-bit counters");
    static constexpr size_t bytes() { return 2 * (size_t)BUF * sizeof(K) + (size_t)NW * BINS * sizeof(uint16_t); }
};

template <typename K>
__device__ __forceinline__ K shfl_xor_any(K v, int m) {
    return __shfl_xor_sync(0xffffffffu, v, m);
}

template <typename K, int NT, int VT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_tile_rsort(const Plan *__restrict__ plan_g, const K *src, K *F, K *S,
                                                         K *samp) {
    using G = RSGeo<K, NT, VT>;
    using U = typename KeyTraits<K>::U;
    constexpr int E = G::E, NW = G::NW, SEG = G::SEG, BUF = G::BUF;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const bufA = reinterpret_cast<K *>(smem_raw);
    K *const bufB = bufA + BUF;
    uint16_t *const hist = reinterpret_cast<uint16_t *>(bufB + BUF);  // [warp][digit]
    __shared__ Plan P;
    __shared__ __align__(8) uint64_t bar;
    __shared__ K red[2][NW];
    __shared__ uint32_t wsum[NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    load_plan(P, plan_g);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const long long g = blockIdx.x;
    if (g >= P.tile_prefix[10]) return;
    int b = 0;
    while (b < 9 && g >= P.tile_prefix[b + 1]) ++b;
    const long long i0 = g - P.tile_prefix[b];
    const long long lo = leaf_start(P, b, i0);
    const int len = (int)(leaf_start(P, b, i0 + 1) - lo);
    if (len == 0) return;
    K *const out = ((P.L[b] & 1) ? S : F) + lo;  // where this bucket's merge level 0 reads
    const K kMax = KeyTraits<K>::kMax;

    // 1. bulk load of the 16-byte aligned superset of the leaf
    const K *in = src + lo;
    const uintptr_t ga0 = (uintptr_t)in & ~(uintptr_t)15;
    const uintptr_t ga1 = ((uintptr_t)(in + len) + 15) & ~(uintptr_t)15;
    const int h = (int)(((uintptr_t)in - ga0) / sizeof(K));
    if (tid == 0) {
        mbar_arrive_expect_tx(&bar, (uint32_t)(ga1 - ga0));
        bulk_g2s(bufA, (const void *)ga0, (uint32_t)(ga1 - ga0), &bar);
    }
    mbar_wait(&bar, 0);

    // 2. key range of the tile
    K mn = kMax, mx = kMax;
    {
        const K *cur = bufA + h;
        K lmin = kMax, lmax = -kMax - 1;
        for (int j = tid; j < len; j += NT) {
            const K k = cur[j];
            lmin = k < lmin ? k : lmin;
            lmax = k > lmax ? k : lmax;
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const K a = shfl_xor_any(lmin, o), c = shfl_xor_any(lmax, o);
            lmin = a < lmin ? a : lmin;
            lmax = c > lmax ? c : lmax;
        }
        if (lane == 0) {
            red[0][warp] = lmin;
            red[1][warp] = lmax;
        }
        __syncthreads();
        mn = red[0][0];
        mx = red[1][0];
#pragma unroll
        for (int w = 1; w < NW; ++w) {
            mn = red[0][w] < mn ? red[0][w] : mn;
            mx = red[1][w] > mx ? red[1][w] : mx;
        }
    }
    const U range = (U)mx - (U)mn;
    const int bits = range == 0 ? 0 : (int)(sizeof(U) * 8) - (sizeof(U) == 4 ? __clz((unsigned)range) : __clzll((long long)range));
    const int passes = bits == 0 ? 1 : (bits + G::RB - 1) / G::RB;
    const int rb = bits == 0 ? 1 : (bits + passes - 1) / passes;
    const int bins = 1 << rb;
    const U dmask = (U)(bins - 1);
    const int sh = (int)(((uintptr_t)out & 15) / sizeof(K));
    const unsigned lanemask_lt = (1u << lane) - 1u;

    // 3. stable counting passes
    const K *cur = bufA + h;
    bool curA = true;
    const int seg0 = warp * SEG;
    uint16_t *const wh = hist + warp * bins;
#pragma unroll 1
    for (int p = 0; p < passes; ++p) {
        const int shift = p * rb;
        K *const dst = (curA ? bufB : bufA) + (p == passes - 1 ? sh : 0);
        for (int j = tid; j < NW * bins; j += NT) hist[j] = 0;
        __syncthreads();
        uint32_t rk[(VT + 1) / 2];
#pragma unroll
        for (int i = 0; i < (VT + 1) / 2; ++i) rk[i] = 0;
#pragma unroll
        for (int i = 0; i < VT; ++i) {
            const int idx = seg0 + i * 32 + lane;
            const unsigned m = __ballot_sync(0xffffffffu, idx < len);
            if (idx < len) {
                const unsigned d = (unsigned)((((U)cur[idx] - (U)mn) >> shift) & dmask);
                const unsigned peers = __match_any_sync(m, d);
                const unsigned lower = peers & lanemask_lt;
                const unsigned base = wh[d];
                __syncwarp(m);
                if (lower == 0) wh[d] = (uint16_t)(base + __popc(peers));
                __syncwarp(m);
                rk[i >> 1] |= (base + __popc(lower)) << ((i & 1) * 16);
            }
        }
        __syncthreads();
        // digit-major exclusive offsets: thread d sums its digit over the warps
        unsigned tot = 0;
        if (tid < bins) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const unsigned c = hist[w * bins + tid];
                hist[w * bins + tid] = (uint16_t)tot;
                tot += c;
            }
        }
        // block exclusive scan of tot over the first `bins` threads
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (tid < bins) {
            unsigned before = incl - tot;
            for (int w = 0; w < warp; ++w) before += wsum[w];
#pragma unroll
            for (int w = 0; w < NW; ++w) hist[w * bins + tid] = (uint16_t)(hist[w * bins + tid] + before);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < VT; ++i) {
            const int idx = seg0 + i * 32 + lane;
            if (idx < len) {
                const K key = cur[idx];
                const unsigned d = (unsigned)((((U)key - (U)mn) >> shift) & dmask);
                dst[wh[d] + ((rk[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu)] = key;
            }
        }
        __syncthreads();
        cur = dst;
        curA = !curA;
    }

    // 4. bulk store of the aligned middle (cur = sorted tile at the destination's phase)
    const K *so = cur;  // so[p] <-> out[p]
    fence_proxy_async_smem();
    __syncthreads();
    const int m0 = sh == 0 ? 0 : E - sh;     // first output at a 16-byte aligned address
    const int m1 = (sh + len) / E * E - sh;  // end of the aligned middle
    if (m1 > m0) {
        if (tid == 0) {
            bulk_s2g_ts(out + m0, so + m0, (uint32_t)((m1 - m0) * sizeof(K)));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (tid < m0) out[tid] = so[tid];
        else if (tid >= E && tid < 2 * E && m1 + tid - E < len) out[m1 + tid - E] = so[m1 + tid - E];
    } else {
        for (int q = tid; q < len; q += NT) out[q] = so[q];
    }
    write_samples(samp, lo, len, so, tid, NT);  // coarse index for merge level 0's co-rank search
    if (tid == 0 && m1 > m0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// =============================================================== launchers
template <typename K>
struct SGeo;
#if HS_TILE_MERGE
template <>
struct SGeo<int32_t> {
    static constexpr int kNT = HS_SORT_NT, kVT = HS_SORT_VT, kMinB = HS_SORT_MINB;
};
template <>
struct SGeo<int64_t> {
    static constexpr int kNT = HS_SORT_NT64, kVT = HS_SORT_VT64, kMinB = HS_SORT_MINB64;
};
#else
template <>
struct SGeo<int32_t> {
    static constexpr int kNT = HS_RSORT_NT, kVT = HS_RSORT_VT, kMinB = 2;
};
template <>
struct SGeo<int64_t> {
    static constexpr int kNT = HS_RSORT_NT, kVT = HS_RSORT_VT64, kMinB = 2;
};
#endif

int sort_tile_keys(int dt) {
    return dt == 0 ? SGeo<int32_t>::kNT * SGeo<int32_t>::kVT : SGeo<int64_t>::kNT * SGeo<int64_t>::kVT;
}

cudaError_t launch_plan(const long long *user_off, Ctl *ctl, int log2c, int mode, int tile_keys, cudaStream_t st) {
    prof_begin(kProfPlan, st);
    k_plan<<<1, 32, 0, st>>>(user_off, ctl, log2c, mode, tile_keys);
    prof_end(kProfPlan, st);
    return cudaGetLastError();
}

cudaError_t launch_plan_whole(long long n, Ctl *ctl, int log2c, int tile_keys, cudaStream_t st) {
    prof_begin(kProfPlan, st);
    k_plan_whole<<<1, 32, 0, st>>>(ctl, n, log2c, tile_keys);
    prof_end(kProfPlan, st);
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_tile_sort_t(const Plan *plan, const void *src, void *F, void *S, void *samp, long long max_tiles,
                               cudaStream_t st) {
    using G = SGeo<K>;
#if HS_TILE_MERGE
    constexpr size_t smem = TSGeo<K, G::kNT, G::kVT>::bytes();
    auto kern = k_tile_sort<K, G::kNT, G::kVT, G::kMinB>;
#else
    constexpr size_t smem = RSGeo<K, G::kNT, G::kVT>::bytes();
    auto kern = k_tile_rsort<K, G::kNT, G::kVT, G::kMinB>;
#endif
    static int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured_dev = dev;
    }
    if (max_tiles <= 0) return cudaSuccess;
    prof_begin(kProfTileSort, st);
    kern<<<(unsigned)max_tiles, G::kNT, smem, st>>>(plan, (const K *)src, (K *)F, (K *)S, (K *)samp);
    prof_end(kProfTileSort, st);
    return cudaGetLastError();
}

cudaError_t launch_tile_sort(int dt, const Plan *plan, const void *src, void *F, void *S, void *samp,
                             long long max_tiles, cudaStream_t st) {
    return dt == 0 ? launch_tile_sort_t<int32_t>(plan, src, F, S, samp, max_tiles, st)
                   : launch_tile_sort_t<int64_t>(plan, src, F, S, samp, max_tiles, st);
}

}  // namespace hs
