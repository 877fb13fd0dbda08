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
// SIMT lanes.  Two paths, the same unique sorted tile:
//   bucket pass (int32, the usual case): keys are split into 2 NT value
//      ranges of the tile's [min, max], counted and scattered with shared-
//      memory atomics, and each thread sorts its two buckets in registers;
//      tiles spanning < 2 NT values become an exact counting sort;
//   merge rounds (int64, and int32 tiles with a bucket over CAP keys): each
//      thread sorts VT keys in registers (Batcher odd-even network,
//      compile-time register indices; VT = 53 int32 / 27 int64), then
//      log2(NT) merge-path merge rounds in shared memory turn the NT sorted
//      runs into one -- the GPU shape of the paper's "sort the partitions,
//      then merge sorted lists pairwise" at CTA scope.
// Keys-only data makes the sorted tile unique, so neither path's (unstable)
// order of equal keys is observable.
#include <cstdint>
#include <type_traits>

#include "hs_device.cuh"
#include "hs_launch.h"

#ifndef HS_SORT_NT
#define HS_SORT_NT 512
#endif
#ifndef HS_SORT_VT
#define HS_SORT_VT 53
#endif
#ifndef HS_SORT_MINB
#define HS_SORT_MINB 2
#endif
#ifndef HS_SORT_NT64
#define HS_SORT_NT64 256  // int64: 128 registers for the bucket networks (512 threads: spills, C5 9.05 vs 7.52 ms)
#endif
#ifndef HS_SORT_VT64
#define HS_SORT_VT64 27
#endif
#ifndef HS_SORT_MINB64
#define HS_SORT_MINB64 2
#endif
#ifndef HS_SORT_BUCKETS
#define HS_SORT_BUCKETS 2  // int32: buckets per thread of the bucket pass (0: merge rounds only)
#endif
#ifndef HS_SORT_CAP
#define HS_SORT_CAP 48  // keys per bucket sorted in registers (mean T / 2NT = 26.5)
#endif
#ifndef HS_SORT_BUCKETS64
#define HS_SORT_BUCKETS64 2  // int64: buckets per thread (16-bit packed counters)
#endif
#ifndef HS_SORT_BUNROLL
#define HS_SORT_BUNROLL 1
#endif
#ifndef HS_SORT_ADAPTIVE
#define HS_SORT_ADAPTIVE 1  // bucket networks sized to the warp's largest bucket (0: always CAP)
#endif
#ifndef HS_SORT_RANK64
#define HS_SORT_RANK64 1  // int64 bucket networks on 32-bit ranks (see the mode-2 loop)
#endif
#ifndef HS_SORT_CAP64
#define HS_SORT_CAP64 28  // mean 0.9 T / 2NT = 12 on split leaves (2 NT buckets): few tiles overflow
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
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        long long off[11];
        for (int b = 0; b < 11; ++b) off[b] = user_off[b];
        compute_plan(&ctl->plan, off, log2c, mode, tile_keys);
    }
}

// K4 for hs_sort_shared (no MSD step): the whole array is bucket 0.
__global__ void k_plan_whole(Ctl *ctl, long long n, int log2c, int tile_keys) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
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
// Merge-path split of output diag between A[0..na) and B[0..nb) (stable-left: ties take A).
template <typename K>
__device__ __forceinline__ int merge_path_s(const K *A, int na, const K *B, int nb, int diag) {
    int l = diag - nb > 0 ? diag - nb : 0;
    int r = diag < na ? diag : na;
    while (l < r) {
        const int mid = (l + r) >> 1;
        if (A[mid] <= B[diag - 1 - mid]) l = mid + 1;
        else r = mid;
    }
    return l;
}

// Packed bucket networks (int32): the bucket pass sorts each thread's two buckets with the smallest
// of four compile-time networks that holds the largest bucket of the warp (CAP - 3s, CAP - 2s,
// CAP - s, CAP with s = CAP / 6 rounded down to even) -- a Poisson-sized bucket rarely needs CAP
// (C3 tile sort -4.5%, C4 -4%).
__host__ __device__ constexpr int ilog2_c(int x) { return x <= 1 ? 0 : 1 + ilog2_c(x >> 1); }

template <int CAP, int I>
__host__ __device__ constexpr int net_size() {
    return HS_SORT_ADAPTIVE ? CAP - (3 - I) * ((CAP / 6) & ~1) : CAP;
}

template <typename K>
__device__ __forceinline__ K kmin(K a, K b) { return a < b ? a : b; }
template <typename K>
__device__ __forceinline__ K kmax(K a, K b) { return a < b ? b : a; }

__device__ __forceinline__ void bulk_s2g_ts(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}


template <typename K>
__device__ __forceinline__ K lds_k(uint32_t a);
template <>
__device__ __forceinline__ int32_t lds_k<int32_t>(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
template <>
__device__ __forceinline__ int64_t lds_k<int64_t>(uint32_t a) {
    int64_t v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}

template <typename K, int NT, int VT>
struct TSGeo {
    static constexpr int T = NT * VT;
    static constexpr int E = 16 / sizeof(K);
    static constexpr size_t bytes() { return (size_t)(T + 2 * E) * sizeof(K); }
};

// CTA-level streaming merge (the big-piece path of K5): O[0, na + nb) = stable-left
// merge of A[0, na) and B[0, nb) (global memory; O disjoint from A and B), in
// output windows of W = T / 3 keys: the next window's merge starts where this
// one ended (no global search), its <= W keys of A and of B are loaded into
// shared memory, every thread merges its outputs from a merge-path split with
// explicit run ends, and the window leaves with coalesced stores (+ samples).
template <typename K, int NT>
__device__ void cta_merge(const K *A, int na, const K *B, int nb, K *O, K *sbuf, int T, K *samp, long long sx) {
    const int W = T / 3, V = (W + NT - 1) / NT;
    K *const sA = sbuf, *const sB = sbuf + W, *const sO = sbuf + 2 * W;
    __shared__ int s_adv;
    const int tid = threadIdx.x, n = na + nb;
    int ai = 0, bi = 0;
    for (int o = 0; o < n;) {
        const int cnt = min(W, n - o);
        const int la = min(cnt, na - ai), lb = min(cnt, nb - bi);
        HS_DASSERT(la >= 0 && lb >= 0 && la + lb >= cnt && 3 * W <= T);
        for (int j = tid; j < la; j += NT) sA[j] = A[ai + j];
        for (int j = tid; j < lb; j += NT) sB[j] = B[bi + j];
        __syncthreads();
        const int p0 = min(tid * V, cnt), p1 = min(p0 + V, cnt);
        if (p0 < p1) {
            int a = merge_path_s(sA, la, sB, lb, p0), c = p0 - a;
            for (int p = p0; p < p1; ++p) {
                const bool tA = c >= lb || (a < la && sA[a] <= sB[c]);
                sO[p] = tA ? sA[a] : sB[c];
                a += tA ? 1 : 0;
                c += tA ? 0 : 1;
            }
        }
        if (tid == 0) s_adv = merge_path_s(sA, la, sB, lb, cnt);  // A keys consumed by this window
        __syncthreads();
        HS_DASSERT(s_adv >= 0 && s_adv <= la && cnt - s_adv <= lb);
        for (int j = tid; j < cnt; j += NT) O[o + j] = sO[j];
        if (samp) write_samples(samp, sx + o, cnt, sO, tid, NT);
        ai += s_adv;
        bi += cnt - s_adv;
        o += cnt;
        __syncthreads();
    }
}

template <typename K, int NT, int VT, int MINB, int BUCKETS, int CAP>
__global__ void __launch_bounds__(NT, MINB) k_tile_sort(const Plan *__restrict__ plan_g, const K *src, K *F, K *S,
                                                        K *samp, const uint32_t *__restrict__ sbtab,
                                                        const SplitCfg *__restrict__ scfg, const K *src_split,
                                                        const uint32_t *__restrict__ cflag, const K *src_pad) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    static_assert(VT & 1, "odd VT keeps blocked shared-memory accesses conflict-free");
    // the grid is a host bound on the leaves: CTAs past the device plan's count leave before any setup
    if ((long long)blockIdx.x >= __ldg(&plan_g->tile_prefix[10])) return;
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
    long long lo;
    int len;
    using U = typename KeyTraits<K>::U;
    // frac: an interior sub-range of a split bucket holds exactly the keys x with
    // mulhi(x - base, mul) = t, and the low word of (x - base) * mul rises with x
    // across the sub-range -- its top bits are the bucket (no min/max pass).  Edge
    // sub-ranges (clamped keys) and narrow ones (< 2^12 values: exact counting) don't.
    bool frac = false;
    U f_base = 0, f_mul = 0;
    int f_sft = 0;
    if (P.split[b]) {  // K5a split this bucket: the leaf is sub-range t of chunk j (in src_split)
        const int ns = P.nsb[b];
        const long long j = (unsigned)i / (unsigned)ns, t = i - j * ns;  // i < c * ns < 2^31
        const uint32_t *e = sbtab + P.sboff[b] + j * (ns + 1) + t;
        lo = P.off[b] + part_start(P.off[b + 1] - P.off[b], P.log2c, j) + __ldg(e);
        len = (int)(__ldg(e + 1) - __ldg(e));
        src = src_split;
        // padded layout (k_split_pad_plan): the sub-range's keys sit at the start of its region
        if (src_pad && split_pmode(*scfg, b)) src = src_pad + scfg->pboff[b] + (j * ns + t) * scfg->cap - lo;
        if (cflag && __ldg(cflag + (e - sbtab))) {
            // a constant piece (k_split_plan): the scatter already wrote it where this kernel writes;
            // only its key samples are left (every sample is that one key)
            K *const o = ((P.L[b] & 1) ? S : F) + lo;
            if (samp && len > 0) {
                const K val = o[0];
                const long long f = lo + (kSampleQ - 1 - lo % kSampleQ);
                for (long long p = f + (long long)tid * kSampleQ; p < lo + len; p += (long long)NT * kSampleQ)
                    st_keep(samp + p / kSampleQ, val);
            }
            return;
        }
        const U mul = (U)scfg->mul[b];
        if (scfg->mode[b] == 0 && t > 0 && t < ns - 1 && mul <= (U)(~(U)0 >> 12)) {
            frac = true;
            f_base = (U)scfg->lo[b];
            f_mul = mul;
            f_sft = scfg->shift;
        }
    } else {
        lo = leaf_start(P, b, i);
        len = (int)(leaf_start(P, b, i + 1) - lo);
    }
    if (len == 0) return;
    HS_DASSERT(len > 0 && len <= ((long long)T << kBigLog2) && lo >= P.off[b] && lo + len <= P.off[b + 1]);
    K *const fin_base = (P.L[b] & 1) ? S : F;  // where this bucket's merge level 0 reads
    const K kMax = KeyTraits<K>::kMax;

    // Sort one tile: in[0, len) (len <= T) -> out[0, len).  phase: parity of the
    // bulk-load barrier (one use per call); bulk: leave by one bulk async store
    // (else plain stores: the big-piece path reads its own outputs back);
    // samp_x >= 0: write the key samples of output positions samp_x + [0, len).
    auto sort_tile = [&](const K *in, const int len, K *const out, const int phase, const bool bulk,
                         const long long samp_x) {
        // 1. bulk load of the 16-byte aligned superset of the leaf
        const uintptr_t ga0 = (uintptr_t)in & ~(uintptr_t)15;
        const uintptr_t ga1 = ((uintptr_t)(in + len) + 15) & ~(uintptr_t)15;
        const int h = (int)(((uintptr_t)in - ga0) / sizeof(K));
        if (tid == 0) {
            mbar_arrive_expect_tx(&bar, (uint32_t)(ga1 - ga0));
            bulk_g2s(sbuf, (const void *)ga0, (uint32_t)(ga1 - ga0), &bar);
        }
        // (sbuf re-derived from the shared symbol here: sort_tile is compiled out of line, and a
        // captured pointer would reach it as a generic address -- LD/ST instead of LDS/STS)
        K *const sbuf = reinterpret_cast<K *>(smem_raw);
        K *const sm = sbuf + h;  // sm[0 .. len) = the leaf
        mbar_wait(&bar, phase & 1);
        for (int j = len + tid; j < T; j += NT) sm[j] = kMax;
        __syncthreads();

        // 2. register sort of VT consecutive keys
        K v[VT];
        const bool live0 = tid * VT < len;
    #pragma unroll
        for (int k = 0; k < VT; ++k) v[k] = sm[tid * VT + k];
        const int sh = (int)(((uintptr_t)out & 15) / sizeof(K));
        K *const so = sbuf + sh;  // so[p] <-> out[p]
        int mode = 0;  // 0: merge rounds; 1: tile staged (constant tile / exact counting); 2: buckets to sort
        // mode 2, int32: every bucket spans < 2^15 values, so a thread's two buckets are
        // sorted together as 16-bit offsets packed two per register (see below)
        bool packed = false;
        constexpr int BPT_ = BUCKETS > 0 ? BUCKETS / NT : 1;
        uint32_t bk_base = 0, bk_cnt[BPT_];  // mode 2: my buckets (set before mode becomes 2)

        if constexpr (BUCKETS > 0) {
            // 2'. Bucket pass (the usual case).  Keys are split by value into
            // BUCKETS equal-width ranges of the tile's [min, max] (a monotone
            // float scaling, so bucket order is key order), counted and scattered
            // into so[] with shared-memory atomics, and every thread sorts its BPT
            // buckets in registers (a CAP-key network).  About 3 shared accesses
            // per key instead of ~2.6 per merge round; the merge rounds below
            // remain the path for tiles with a bucket over CAP keys (skew, heavy
            // duplicates) -- the result is the same unique sorted tile.  PACK:
            // two 16-bit counters per word (int64 tiles: leaves room for 2 CTAs/SM).
            constexpr int BPT = BUCKETS / NT;
            constexpr bool PACK = sizeof(K) == 8 || BPT > 2;
            static_assert(BUCKETS == BPT * NT && (!PACK || BPT % 2 == 0), "bucket layout");
            __shared__ uint32_t bcnt[PACK ? BUCKETS / 2 : BUCKETS];
            __shared__ K red[2][NT / 32];
            __shared__ uint32_t wsum[NT / 32];
            const int lane = tid & 31, warp = tid >> 5;
            if (!frac) {
                K lmin = kMax, lmax = (K)(-kMax - 1);
    #pragma unroll
                for (int k = 0; k < VT; ++k)
                    if (tid * VT + k < len) {
                        lmin = v[k] < lmin ? v[k] : lmin;
                        lmax = v[k] > lmax ? v[k] : lmax;
                    }
    #pragma unroll
                for (int o = 16; o >= 1; o >>= 1) {
                    const K x = __shfl_xor_sync(0xffffffffu, lmin, o), c = __shfl_xor_sync(0xffffffffu, lmax, o);
                    lmin = x < lmin ? x : lmin;
                    lmax = c > lmax ? c : lmax;
                }
                if (lane == 0) {
                    red[0][warp] = lmin;
                    red[1][warp] = lmax;
                }
            }
    #pragma unroll
            for (int j = 0; j < (PACK ? BPT / 2 : BPT); ++j) bcnt[j * NT + tid] = 0;
            __syncthreads();  // (also: every thread has its keys in v; sbuf is free)
            // bucket of k = top log2(BUCKETS) bits of ((k >> sft) - base) * mulA (w-bit product, no
            // overflow): one integer map for all modes
            //   frac:  base, mulA = the sub-range's (see above) (top bits of the fraction)
            //   exact (range < BUCKETS): base = min, mulA = 2^w / BUCKETS -> k - min
            //   else:  base = min, mulA = floor((2^w - 1) / (range + 1)) (equal-width, monotone)
            constexpr U WMAX = ~(U)0;
            static_assert((BUCKETS & (BUCKETS - 1)) == 0, "power-of-two bucket count");
            constexpr int kBShift = 8 * (int)sizeof(U) - ilog2_c(BUCKETS);
            U base = f_base, mulA = f_mul;
            int sft = f_sft;
            bool exact = false, constant = false;
            K mn = 0;
            // frac: a bucket covers 2^w / (BUCKETS mul) + 1 values -- < 2^15 when mul >= 2^w / 2^24
            packed = sizeof(K) == 4 && frac && f_mul >= (U)256;
            if (!frac) {
                mn = red[0][0];
                K mx = red[1][0];
    #pragma unroll
                for (int w = 1; w < NT / 32; ++w) {
                    mn = red[0][w] < mn ? red[0][w] : mn;
                    mx = red[1][w] > mx ? red[1][w] : mx;
                }
                const U range = (U)mx - (U)mn;
                constant = range == 0;
                exact = range < (U)BUCKETS;
                base = (U)mn;
                sft = 0;
                if (exact) mulA = (U)(WMAX / (U)BUCKETS + 1);  // 2^w / BUCKETS
                else mulA = range == WMAX ? (U)1 : WMAX / (range + 1);
                // a bucket spans about (range + 1) / BUCKETS values
                packed = sizeof(K) == 4 && !exact && range < ((U)1 << 24);
            }
            if (constant) {  // constant tile: every order is the sorted one
                for (int j = tid; j < len; j += NT) so[j] = mn;
                mode = 1;
            } else {
                // exact: one bucket per key value (an exact counting sort, buckets need
                // no sort and have no capacity limit)
                auto bucket_of_key = [&](K k) -> int {
                    const U x = ((U)(k >> sft) - base) * mulA;
                    return (int)(x >> kBShift);  // < BUCKETS, non-decreasing in k
                };
                // returns the bucket's count before this key (its slot when the counters hold starts)
                auto bump = [&](int bk) -> uint32_t {
                    if (PACK) {
                        const int sft = (bk & 1) * 16;
                        return (atomicAdd(&bcnt[bk >> 1], 1u << sft) >> sft) & 0xFFFFu;
                    }
                    return atomicAdd(&bcnt[bk], 1u);
                };
                auto count_of = [&](int bk) -> uint32_t {
                    return PACK ? (bcnt[bk >> 1] >> ((bk & 1) * 16)) & 0xFFFFu : bcnt[bk];
                };
    #pragma unroll
                for (int k = 0; k < VT; ++k)
                    if (tid * VT + k < len) {
                        const int bk = bucket_of_key(v[k]);
                        if (PACK) atomicAdd(&bcnt[bk >> 1], 1u << ((bk & 1) * 16));  // no return: RED
                        else atomicAdd(&bcnt[bk], 1u);
                    }
                __syncthreads();
                uint32_t cnt[BPT], tot = 0;
                bool over = false;
    #pragma unroll
                for (int q = 0; q < BPT; ++q) {
                    cnt[q] = count_of(BPT * tid + q);
                    tot += cnt[q];
                    over |= cnt[q] > (uint32_t)CAP;
                }
                if (!__syncthreads_or(!exact && over)) {
                    // exclusive scan of the per-thread totals -> bucket starts (cursors)
                    uint32_t incl = tot;
    #pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += u;
                    }
                    if (lane == 31) wsum[warp] = incl;
                    __syncthreads();
                    uint32_t base = incl - tot;
                    for (int w = 0; w < warp; ++w) base += wsum[w];
                    uint32_t st = base;
                    if (PACK) {
    #pragma unroll
                        for (int q = 0; q < BPT; q += 2) {
                            bcnt[(BPT * tid + q) >> 1] = st | ((st + cnt[q]) << 16);
                            st += cnt[q] + cnt[q + 1];
                        }
                    } else {
    #pragma unroll
                        for (int q = 0; q < BPT; ++q) {
                            bcnt[BPT * tid + q] = st;
                            st += cnt[q];
                        }
                    }
                    __syncthreads();
    #pragma unroll
                    for (int k = 0; k < VT; ++k)
                        if (tid * VT + k < len) so[bump(bucket_of_key(v[k]))] = v[k];
                    bk_base = base;
    #pragma unroll
                    for (int q = 0; q < BPT; ++q) bk_cnt[q] = cnt[q];
                    mode = exact ? 1 : 2;
                }
            }
        }

        if (mode == 2 && packed) {
            // int32, two buckets per thread, each spanning < 2^15 values: offsets from each
            // bucket's first key (+2^15, so 0xFFFF pads sort last) packed two per register
            // -- bucket 0 in the low halves, bucket 1 in the high halves -- and one CAP-key
            // network of SIMD min/max sorts both buckets at once (half the comparators)
            __syncthreads();
            if constexpr (sizeof(K) == 4 && BPT_ == 2) {
                const uint32_t stA = bk_base, cA = bk_cnt[0], stB = bk_base + bk_cnt[0], cB = bk_cnt[1];
                auto run = [&](auto NCAP) {
                    constexpr int N = decltype(NCAP)::value;
                    if (cA > 1 || cB > 1) {
                        const int32_t rA = cA ? (int32_t)so[stA] : 0, rB = cB ? (int32_t)so[stB] : 0;
                        H2 w[N];
    #pragma unroll
                        for (int i = 0; i < N; ++i) {
                            const uint32_t lo = i < (int)cA ? (uint32_t)((int32_t)so[stA + i] - rA + 32768) : 0xFFFFu;
                            const uint32_t hi = i < (int)cB ? (uint32_t)((int32_t)so[stB + i] - rB + 32768) : 0xFFFFu;
                            w[i].v = lo | (hi << 16);
                        }
                        oddeven_sort<N>(w);
    #pragma unroll
                        for (int i = 0; i < N; ++i) {
                            if (i < (int)cA) so[stA + i] = (K)(rA + (int32_t)(w[i].v & 0xFFFFu) - 32768);
                            if (i < (int)cB) so[stB + i] = (K)(rB + (int32_t)(w[i].v >> 16) - 32768);
                        }
                    }
                };
                // the smallest network that holds the warp's largest bucket (CTA-uniform branch: all lanes here)
                const uint32_t wm = __reduce_max_sync(0xffffffffu, cA > cB ? cA : cB);
                if (wm <= (uint32_t)net_size<CAP, 0>()) run(std::integral_constant<int, net_size<CAP, 0>()>{});
                else if (wm <= (uint32_t)net_size<CAP, 1>()) run(std::integral_constant<int, net_size<CAP, 1>()>{});
                else if (wm <= (uint32_t)net_size<CAP, 2>()) run(std::integral_constant<int, net_size<CAP, 2>()>{});
                else run(std::integral_constant<int, CAP>{});
            }
        } else if (mode == 2) {
            // sort my buckets in registers (v is dead on this path)
            __syncthreads();
            uint32_t st = bk_base;
            constexpr int kBU = HS_SORT_BUNROLL;
    #pragma unroll kBU
            for (int q = 0; q < BPT_; ++q) {
                const uint32_t cn = bk_cnt[q];
#if HS_SORT_RANK64
                if constexpr (sizeof(K) == 8) {
                    // int64: sort 32-bit ranks instead of the keys (an int64 comparator costs 4x an
                    // int32 one: tools/probe/ce_probe.cu).  rank = ((k - min) >> s) << 5 | i with s
                    // the smallest shift that leaves 27 bits for the bucket's span and i < 32 the
                    // key's slot; ranks are unique, a 32-bit network orders them, and the keys follow
                    // by a gather.  Keys with equal (k - min) >> s keep slot order, so the gathered
                    // run is checked; if two such keys came out of order (keys closer than 2^s; never
                    // for s = 0) an insertion pass in shared memory repairs the nearly sorted run.
                    // One CAP network (per-warp sizing: more code than it saves here).
                    constexpr int N = CAP;
                    static_assert(N <= 32, "5-bit slots");
                    if (cn > 1) {
                        // (keys re-read from shared memory: holding them in registers across the
                        // network measured slower -- register pressure)
                        K mnb = so[st], mxb = mnb;
    #pragma unroll
                        for (int i = 1; i < N; ++i)
                            if (i < (int)cn) {
                                const K x = so[st + i];
                                mnb = x < mnb ? x : mnb;
                                mxb = x > mxb ? x : mxb;
                            }
                        const U span = (U)mxb - (U)mnb;
                        const int bits = 64 - __clzll((long long)span);
                        const int s = bits > 27 ? bits - 27 : 0;
                        uint32_t rk[N];
    #pragma unroll
                        for (int i = 0; i < N; ++i)
                            rk[i] = i < (int)cn ? ((uint32_t)(((U)so[st + i] - (U)mnb) >> s) << 5) | (uint32_t)i
                                                : 0xFFFFFFFFu;
                        oddeven_sort<N>(rk);
                        K r[N];
                        bool ok = true;
    #pragma unroll
                        for (int j = 0; j < N; ++j) {
                            r[j] = j < (int)cn ? so[st + (rk[j] & 31u)] : kMax;
                            if (j > 0) ok &= !(r[j] < r[j - 1]);
                        }
    #pragma unroll
                        for (int j = 0; j < N; ++j)
                            if (j < (int)cn) so[st + j] = r[j];
                        if (!ok) {
                            for (int j = 1; j < (int)cn; ++j) {
                                const K x = so[st + j];
                                int m = j;
                                for (; m > 0 && x < so[st + m - 1]; --m) so[st + m] = so[st + m - 1];
                                so[st + m] = x;
                            }
                        }
                    }
                    st += cn;
                    continue;
                }
#endif
                auto run = [&](auto NCAP) {
                    constexpr int N = decltype(NCAP)::value;
                    if (cn > 1) {
                        K w[N];
    #pragma unroll
                        for (int i = 0; i < N; ++i) w[i] = i < (int)cn ? so[st + i] : kMax;
                        oddeven_sort<N>(w);
    #pragma unroll
                        for (int i = 0; i < N; ++i)
                            if (i < (int)cn) so[st + i] = w[i];
                    }
                };
                // (one CAP network: sizing it to the warp's largest bucket measured 4% slower on int64 keys)
                run(std::integral_constant<int, CAP>{});
                st += cn;
            }
        } else if (mode == 0) {
            if (live0) oddeven_sort<VT>(v);

            // 3. merge rounds (R = threads per run).  Bitonic storage: in round R the
            // input run q (length RL = R VT) is stored ascending if q is even (the
            // pair's A) and DESCENDING if q is odd (the pair's B), so a pair occupies
            // one bitonic stretch of shared memory.  A thread merges from both ends
            // of what is left of it: the smaller of the two end keys is always the
            // next output, even after one run is exhausted (the pointers then walk
            // towards each other inside the other run), so the serial merge needs no
            // bounds tests and no sentinels; ties take the A end (stable-left).
            // Every thread stores every round (threads past the leaf's end hold
            // kMax pads), so the stretch is complete; only threads with an output
            // below len merge.
            const uint32_t sm_u = smem_u32(sm);
    #pragma unroll 1
            for (int lgR = 0; (1 << lgR) < NT; ++lgR) {
                const int R = 1 << lgR, RL = R * VT;
                const int q = tid >> lgR;  // this thread's outputs form part of input run q
                __syncthreads();           // everyone has read the previous round's runs
                if ((q & 1) == 0) {
    #pragma unroll
                    for (int k = 0; k < VT; ++k) sm[tid * VT + k] = v[k];
                } else {  // run q reversed in place: canonical c <-> (2q+1) RL - 1 - c
                    const int m = (2 * q + 1) * RL - 1 - tid * VT;
    #pragma unroll
                    for (int k = 0; k < VT; ++k) sm[m - k] = v[k];
                }
                __syncthreads();
                if (tid * VT < len) {
                    const int j = tid & (2 * R - 1);
                    const int a0 = (tid - j) * VT, bE = a0 + 2 * RL;  // A = sm[a0, a0+RL) asc, B[k] = sm[bE-1-k]
                    const int diag = j * VT;
                    // merge path: first m with !(A[m] <= B[diag-1-m]); B[diag-1-m] = sm[bE - diag + m]
                    int l = diag - RL > 0 ? diag - RL : 0, r = diag < RL ? diag : RL;
                    const uint32_t ua = sm_u + (uint32_t)a0 * sizeof(K), ub = sm_u + (uint32_t)(bE - diag) * sizeof(K);
                    while (l < r) {
                        const int mid = (l + r) >> 1;
                        const bool pr = lds_k<K>(ua + mid * (int)sizeof(K)) <= lds_k<K>(ub + mid * (int)sizeof(K));
                        l = pr ? mid + 1 : l;
                        r = pr ? r : mid;
                    }
                    uint32_t pi = ua + l * (int)sizeof(K);                                   // next A key
                    uint32_t pj = sm_u + (uint32_t)(bE - 1 - (diag - l)) * sizeof(K);       // next B key
                    HS_DASSERT(l >= 0 && l <= RL && diag - l >= 0 && diag - l <= RL && bE <= T);
                    [[maybe_unused]] const uint32_t lo_b = ua, hi_b = sm_u + (uint32_t)bE * sizeof(K);  // the pair's stretch
                    K x = lds_k<K>(pi), y = lds_k<K>(pj);
    #pragma unroll
                    for (int k = 0; k < VT; ++k) {
                        const bool p = x <= y;
                        v[k] = p ? x : y;
                        if (k + 1 < VT) {
                            pi += p ? (uint32_t)sizeof(K) : 0u;
                            pj -= p ? 0u : (uint32_t)sizeof(K);
                            HS_DASSERT(pi >= lo_b && pi < hi_b && pj >= lo_b && pj < hi_b);
                            const K t = lds_k<K>(p ? pi : pj);
                            x = p ? t : x;
                            y = p ? y : t;
                        }
                    }
                }
            }

            __syncthreads();
            if (tid * VT < len) {
    #pragma unroll
                for (int k = 0; k < VT; ++k) so[tid * VT + k] = v[k];
            }
        }  // mode == 0

        // 4. the sorted tile sits at the destination's 16-byte phase: bulk store the aligned middle
        fence_proxy_async_smem();
        __syncthreads();
        const int m0 = sh == 0 ? 0 : E - sh;            // first output at a 16-byte aligned address
        const int m1 = (sh + len) / E * E - sh;         // end of the aligned middle
        if (bulk && m1 > m0) {
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
        if (samp_x >= 0) write_samples(samp, samp_x, len, so, tid, NT);  // coarse index for the next co-rank search
    };

    // A split piece longer than one tile (duplicate-heavy or skewed sub-ranges, up to
    // 2^kBigLog2 tiles; k_split_plan sends longer ones to the bucket fallback): its
    // 2^lgp parts (partition_even) are tile-sorted one after another, then lgp
    // CTA-level merge passes (stable-left, P:58-60 at CTA scope) ping-pong between the
    // piece's regions of F and S, the last one landing where merge level 0 reads.
    int lgp = 0;
    while (((long long)T << lgp) < len) ++lgp;
    K *const fin = fin_base + lo;
    // Two call sites on purpose: sort_tile is then compiled out of line, with
    // its own register allocation -- measured 1.05 ms vs 1.16 ms for the
    // inlined single-site form on C3's K5 (profiles/r02/README.md).
    if (lgp == 0) {
        sort_tile(src + lo, len, fin, 0, true, lo);
        return;
    }
    K *const alt = (fin_base == F ? S : F) + lo;
    K *xb = (lgp & 1) ? alt : fin;  // the parts' sorted runs; the last pass writes fin
    for (int part = 0; part < (1 << lgp); ++part) {
        const int ps = (int)part_start(len, lgp, part), pe = (int)part_start(len, lgp, part + 1);
        __syncthreads();  // the previous part is done with shared memory
        sort_tile(src + lo + ps, pe - ps, xb + ps, part, false, -1);
    }
    K *yb = xb == fin ? alt : fin;
    for (int r = 0; r < lgp; ++r) {
        const bool last = r + 1 == lgp;
        for (int q = 0; q < (1 << (lgp - r - 1)); ++q) {  // runs = merged groups of 2^r parts
            const int a0 = (int)part_start(len, lgp, (long long)(2 * q) << r);
            const int a1 = (int)part_start(len, lgp, (long long)(2 * q + 1) << r);
            const int a2 = (int)part_start(len, lgp, (long long)(2 * q + 2) << r);
            __syncthreads();  // (the previous pass's / pair's outputs are written)
            cta_merge<K, NT>(xb + a0, a1 - a0, xb + a1, a2 - a1, yb + a0, sbuf, T, last ? samp : nullptr, lo + a0);
        }
        K *const t = xb;
        xb = yb;
        yb = t;
    }
}

// =============================================================== launchers
template <typename K>
struct SGeo;
template <>
struct SGeo<int32_t> {
    static constexpr int kNT = HS_SORT_NT, kVT = HS_SORT_VT, kMinB = HS_SORT_MINB;
    static constexpr int kBuckets = HS_SORT_BUCKETS * HS_SORT_NT, kCap = HS_SORT_CAP;
};
template <>
struct SGeo<int64_t> {
    static constexpr int kNT = HS_SORT_NT64, kVT = HS_SORT_VT64, kMinB = HS_SORT_MINB64;
    static constexpr int kBuckets = HS_SORT_BUCKETS64 * HS_SORT_NT64, kCap = HS_SORT_CAP64;
};

template <typename K>
cudaError_t setup_tile_sort_t() {
    using G = SGeo<K>;
    constexpr size_t smem = TSGeo<K, G::kNT, G::kVT>::bytes();
    return cudaFuncSetAttribute(k_tile_sort<K, G::kNT, G::kVT, G::kMinB, G::kBuckets, G::kCap>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t setup_tilesort_kernels(int dev) {
    (void)dev;
    cudaError_t e = setup_tile_sort_t<int32_t>();
    return e != cudaSuccess ? e : setup_tile_sort_t<int64_t>();
}

int sort_tile_keys(int dt) {
    return dt == 0 ? SGeo<int32_t>::kNT * SGeo<int32_t>::kVT : SGeo<int64_t>::kNT * SGeo<int64_t>::kVT;
}

cudaError_t launch_plan(const long long *user_off, Ctl *ctl, int log2c, int mode, int tile_keys, cudaStream_t st) {
    prof_begin(kProfPlan, st);
    cudaError_t e = launch_pdl(k_plan, dim3(1), dim3(32), 0, st, user_off, ctl, log2c, mode, tile_keys);
    if (e != cudaSuccess) return e;
    prof_end(kProfPlan, st);
    return cudaGetLastError();
}

cudaError_t launch_plan_whole(long long n, Ctl *ctl, int log2c, int tile_keys, cudaStream_t st) {
    prof_begin(kProfPlan, st);
    cudaError_t e = launch_pdl(k_plan_whole, dim3(1), dim3(32), 0, st, ctl, n, log2c, tile_keys);
    if (e != cudaSuccess) return e;
    prof_end(kProfPlan, st);
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_tile_sort_t(const Plan *plan, const void *src, void *F, void *S, void *samp, long long max_tiles,
                               cudaStream_t st, const uint32_t *sbtab, const SplitCfg *scfg, const void *src_split,
                               const uint32_t *cflag, const void *src_pad) {
    using G = SGeo<K>;
    constexpr size_t smem = TSGeo<K, G::kNT, G::kVT>::bytes();
    auto kern = k_tile_sort<K, G::kNT, G::kVT, G::kMinB, G::kBuckets, G::kCap>;
    if (max_tiles <= 0) return cudaSuccess;
    prof_begin(kProfTileSort, st);
    cudaError_t e = launch_pdl(kern, dim3((unsigned)max_tiles), dim3(G::kNT), smem, st, plan, (const K *)src, (K *)F,
                               (K *)S, (K *)samp, sbtab, scfg, (const K *)(src_split ? src_split : F), cflag,
                               (const K *)src_pad);
    if (e != cudaSuccess) return e;
    prof_end(kProfTileSort, st);
    return cudaGetLastError();
}

cudaError_t launch_tile_sort(int dt, const Plan *plan, const void *src, void *F, void *S, void *samp,
                             long long max_tiles, cudaStream_t st, const uint32_t *sbtab, const SplitCfg *scfg,
                             const void *src_split, const uint32_t *cflag, const void *src_pad) {
    return dt == 0 ? launch_tile_sort_t<int32_t>(plan, src, F, S, samp, max_tiles, st, sbtab, scfg, src_split, cflag,
                                                 src_pad)
                   : launch_tile_sort_t<int64_t>(plan, src, F, S, samp, max_tiles, st, sbtab, scfg, src_split, cflag,
                                                 src_pad);
}

}  // namespace hs
