// hs_kernels.cu -- the sm_100a kernels of the hybrid-sort hot path
// (arXiv 2003.01216 §3.4), one per method step:
//
//   K1 k_histogram      a1  leading-digit histogram -> bucket_offsets (+ plan)
//   K3 k_scatter        a2+a3 stable scatter into ten buckets, decoupled lookback
//   K4 k_plan           a4  chunk / leaf-tile geometry from given offsets
//   K5 k_tile_sort      a5  in-shared-memory sort of each leaf tile of each chunk
//   K6 k_merge_partition + k_merge_level
//                       a5/a6 merge-path (co-rank) partitioned merge of run pairs,
//                            one launch pair per merge level
//   K7 k_copy           in-place hs_merge with an odd number of rounds only
//
// Design notes, rooflines and algorithmic bytes per kernel: DESIGN.md §5.
#include <cstdint>
#include <cstring>

#include "hs_device.cuh"
#include "hs_launch.h"

namespace hs {

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// Copy the plan into shared memory (one word per thread).
__device__ __forceinline__ void load_plan(Plan &dst, const Plan *src) {
    static_assert(sizeof(Plan) % 4 == 0, "plan size");
    constexpr int W = sizeof(Plan) / 4;
    const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
    uint32_t *d = reinterpret_cast<uint32_t *>(&dst);
    for (int i = threadIdx.x; i < W; i += blockDim.x) d[i] = __ldg(s + i);
}

// =================================================================== K1
// Leading-digit histogram (a1).  Persistent grid-stride over 16-byte vectors
// of a virtual index space aligned to 16 bytes (h = leading misalignment in
// keys), 128-bit streaming loads (ld.global.nc.L1::no_allocate.v4),
// per-thread packed 8-bit counters (3 registers for 10 digits, flushed every
// 63 vectors), warp reduction with redux.sync, shared atomics, then one
// global atomic per digit per CTA.  The last CTA to finish turns the counts
// into bucket_offsets (exclusive prefix) and, if asked, the call's plan.
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_histogram(const K *__restrict__ keys, int n, int h, DigitParams<K> dp,
                                                  Ctl *ctl, long long *user_off, int plan_mode, int log2c,
                                                  int tile_keys) {
    constexpr int E = 16 / sizeof(K);
    __shared__ unsigned s_hist[10];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    if (tid < 10) s_hist[tid] = 0;
    __syncthreads();

    unsigned c[10];
#pragma unroll
    for (int b = 0; b < 10; ++b) c[b] = 0;
    unsigned p0 = 0, p1 = 0, p2 = 0;
    auto count = [&](K key) {
        int d = msd_digit(key, dp);
        unsigned w = (unsigned)d >> 2;
        unsigned inc = 1u << (((unsigned)d & 3u) << 3);
        p0 += (w == 0) ? inc : 0u;
        p1 += (w == 1) ? inc : 0u;
        p2 += (w == 2) ? inc : 0u;
    };
    auto flush = [&]() {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            c[b] += (p0 >> (8 * b)) & 0xFFu;
            c[4 + b] += (p1 >> (8 * b)) & 0xFFu;
        }
        c[8] += p2 & 0xFFu;
        c[9] += (p2 >> 8) & 0xFFu;
        p0 = p1 = p2 = 0;
    };

    const long long nvec = ((long long)n + h + E - 1) / E;
    const long long stride = (long long)gridDim.x * NT;
    int iters = 0;
    for (long long v = (long long)blockIdx.x * NT + tid; v < nvec; v += stride) {
        long long e0 = v * E - h;
        if (e0 >= 0 && e0 + E <= n) {
            int4 q = ld_stream_v4(keys + e0);
            K vals[E];
            memcpy(vals, &q, 16);
#pragma unroll
            for (int j = 0; j < E; ++j) count(vals[j]);
        } else {
#pragma unroll
            for (int j = 0; j < E; ++j) {
                long long e = e0 + j;
                if (e >= 0 && e < n) count(keys[e]);
            }
        }
        if (++iters == 63) {  // 63 * 4 keys <= 255 per 8-bit field
            flush();
            iters = 0;
        }
    }
    flush();

#pragma unroll
    for (int b = 0; b < 10; ++b) {
        unsigned t = __reduce_add_sync(0xffffffffu, c[b]);
        if ((tid & 31) == 0 && t) atomicAdd(&s_hist[b], t);
    }
    __syncthreads();
    if (tid < 10 && s_hist[tid]) atomicAdd(&ctl->hist[tid], (unsigned long long)s_hist[tid]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&ctl->done, 1u) == gridDim.x - 1);
    __syncthreads();
    if (s_last && tid == 0) {
        __threadfence();
        long long off[11];
        off[0] = 0;
        for (int b = 0; b < 10; ++b) off[b + 1] = off[b] + (long long)atomicAdd(&ctl->hist[b], 0ull);
        for (int b = 0; b < 11; ++b) {
            ctl->off[b] = off[b];
            if (user_off) user_off[b] = off[b];
        }
        if (plan_mode >= 0) compute_plan(&ctl->plan, off, log2c, plan_mode, tile_keys);
    }
}

// =================================================================== K3
// Stable scatter into the ten buckets (a2 + a3), onesweep-style:
//  1. tile id from an atomic ticket (forward progress for the lookback);
//  2. 128-bit coalesced loads of T = NT*VT keys into padded shared memory;
//  3. each thread ranks its VT consecutive keys (blocked layout, input
//     order) with 6-bit packed per-digit counters in one 64-bit register;
//  4. block-wide exclusive scan of the per-thread counts (5 words of two
//     16-bit digit fields; warp shuffles + one warp over warp totals);
//  5. decoupled lookback (lanes 0..9 of warp 0, one digit each): publish the
//     tile aggregate, walk back to an inclusive prefix, publish inclusive;
//  6. keys are re-staged in shared memory in digit order, then written out
//     as ten coalesced runs to out[off[d] + prefix_d + rank].
// Output position = bucket base + #same-digit keys before it in input order:
// exactly the stable counting pass of P:78 / S:302.
template <typename K, int NT, int VT>
__global__ void __launch_bounds__(NT) k_scatter(const K *__restrict__ keys, K *__restrict__ out, int n, int h,
                                                DigitParams<K> dp, Ctl *ctl, unsigned long long *status) {
    constexpr int T = NT * VT;
    constexpr int E = 16 / sizeof(K);
    constexpr int NW = NT / 32;
    static_assert(VT <= 16, "ranks are packed in 4 bits");
    static_assert(T <= 16384, "digit counts are packed in 16-bit fields");
    __shared__ K s[T + T / 32];
    __shared__ unsigned s_wtot[NW][5];
    __shared__ int s_dstart[10];
    __shared__ long long s_delta[10];
    __shared__ unsigned s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&ctl->ticket, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const long long v0 = (long long)tile * T - h;  // global index of local slot 0
    const int jlo = v0 < 0 ? (int)(-v0) : 0;
    const int jhi = (int)((long long)n - v0 < T ? (long long)n - v0 : (long long)T);

    // 2. load
#pragma unroll
    for (int r = 0; r < T / E / NT; ++r) {
        const int j0 = (r * NT + tid) * E;
        K vals[E];
        if (j0 >= jlo && j0 + E <= jhi) {
            int4 q = ld_stream_v4(keys + (v0 + j0));
            memcpy(vals, &q, 16);
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) vals[e] = (j0 + e >= jlo && j0 + e < jhi) ? keys[v0 + j0 + e] : K(0);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) s[pad_idx(j0 + e)] = vals[e];
    }
    __syncthreads();

    // 3. per-thread ranks (blocked: thread tid owns local slots tid*VT ..)
    K key[VT];
    unsigned meta[VT / 4 > 0 ? VT / 4 : 1];
#pragma unroll
    for (int i = 0; i < (VT / 4 > 0 ? VT / 4 : 1); ++i) meta[i] = 0;
    unsigned long long cnt = 0;
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const int j = tid * VT + k;
        key[k] = s[pad_idx(j)];
        const bool valid = (j >= jlo) && (j < jhi);
        const int d = valid ? msd_digit(key[k], dp) : 10;  // field 10 = "not a key"
        const unsigned r = (unsigned)(cnt >> (6 * d)) & 63u;
        cnt += 1ull << (6 * d);
        meta[k >> 2] |= ((unsigned)d | (r << 4)) << (8 * (k & 3));
    }

    // 4. block exclusive scan of the 10 per-thread counts (5 words x 2 fields)
    unsigned own[5], w[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        own[i] = (unsigned)((cnt >> (12 * i)) & 63ull) | ((unsigned)((cnt >> (12 * i + 6)) & 63ull) << 16);
        w[i] = own[i];
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            unsigned t = __shfl_up_sync(0xffffffffu, w[i], o);
            if (lane >= o) w[i] += t;
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < 5; ++i) s_wtot[warp][i] = w[i];
    }
    __syncthreads();
    if (warp == 0) {
        unsigned t[5], town[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            town[i] = lane < NW ? s_wtot[lane][i] : 0u;
            t[i] = town[i];
        }
#pragma unroll
        for (int o = 1; o < NW; o <<= 1) {
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                unsigned u = __shfl_up_sync(0xffffffffu, t[i], o);
                if (lane >= o) t[i] += u;
            }
        }
        unsigned tot[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) tot[i] = __shfl_sync(0xffffffffu, t[i], NW - 1);
        __syncwarp();
        if (lane < NW) {
#pragma unroll
            for (int i = 0; i < 5; ++i) s_wtot[lane][i] = t[i] - town[i];
        }
        // 5. decoupled lookback, lane d handles digit d
        if (lane < 10) {
            const int d = lane;
            unsigned agg = 0, dstart = 0;
#pragma unroll
            for (int e = 0; e < 10; ++e) {
                unsigned f = (tot[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
                if (e < d) dstart += f;
                if (e == d) agg = f;
            }
            unsigned long long *my = status + (size_t)tile * 10 + d;
            long long excl = 0;
            if (tile == 0) {
                st_relaxed_u64(my, kFlagIncl | (unsigned long long)agg);
            } else {
                st_relaxed_u64(my, kFlagAgg | (unsigned long long)agg);
                long long p = (long long)tile - 1;
                while (true) {
                    unsigned long long sv;
                    do {
                        sv = ld_relaxed_u64(status + (size_t)p * 10 + d);
                    } while ((sv >> 62) == 0);
                    excl += (long long)(sv & kValMask);
                    if ((sv >> 62) == 2) break;
                    --p;
                }
                st_relaxed_u64(my, kFlagIncl | (unsigned long long)(excl + agg));
            }
            s_dstart[d] = (int)dstart;
            s_delta[d] = ctl->off[d] + excl - (long long)dstart;
        }
    }
    __syncthreads();

    // 6a. re-stage keys in digit order inside the tile
    unsigned base[5];
#pragma unroll
    for (int i = 0; i < 5; ++i)
        base[i] = s_wtot[warp][i] + (w[i] - own[i]) + ((unsigned)s_dstart[2 * i] | ((unsigned)s_dstart[2 * i + 1] << 16));
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const unsigned m = (meta[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        const unsigned d = m & 15u, r = m >> 4;
        if (d < 10) {
            const unsigned wsel = d < 2 ? base[0] : d < 4 ? base[1] : d < 6 ? base[2] : d < 8 ? base[3] : base[4];
            const int pos = (int)((wsel >> ((d & 1u) * 16)) & 0xFFFFu) + (int)r;
            s[pad_idx(pos)] = key[k];
        }
    }
    __syncthreads();

    // 6b. coalesced write-out, ten contiguous runs
    const int nvalid = jhi - jlo;
    for (int j = tid; j < nvalid; j += NT) {
        const K kv = s[pad_idx(j)];
        const int d = msd_digit(kv, dp);
        out[s_delta[d] + j] = kv;
    }
}

// =================================================================== K4
__global__ void k_plan(const long long *__restrict__ user_off, Ctl *ctl, int log2c, int mode, int tile_keys) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        long long off[11];
        for (int b = 0; b < 11; ++b) off[b] = user_off[b];
        compute_plan(&ctl->plan, off, log2c, mode, tile_keys);
    }
}

// =================================================================== K5
// In-shared-memory sort of one leaf tile (a5).  Each thread sorts VT keys
// in registers with a Batcher odd-even network, then log2(T/VT) merge
// passes in shared memory: every thread finds its merge-path split by binary
// search and merges VT outputs serially (stable-left).  Padding with the
// dtype max makes every tile a full power of two; pads sort to the end and
// are never stored (they are indistinguishable from real max keys).
// The tile is written to the buffer where its bucket's level 0 reads.
template <typename K, int NT, int VT>
__global__ void __launch_bounds__(NT) k_tile_sort(const Plan *__restrict__ plan_g, const K *src, K *F, K *S) {
    constexpr int T = NT * VT;
    __shared__ K s[T + T / 32];
    __shared__ Plan P;
    const int tid = threadIdx.x;
    load_plan(P, plan_g);
    __syncthreads();
    const long long g = blockIdx.x;
    if (g >= P.tile_prefix[10]) return;
    int b = 0;
    while (b < 9 && g >= P.tile_prefix[b + 1]) ++b;
    const long long i = g - P.tile_prefix[b];
    const long long lo = leaf_start(P, b, i);
    const int len = (int)(leaf_start(P, b, i + 1) - lo);
    if (len == 0) return;
    K *dst = (P.L[b] & 1) ? S : F;
    const K kMax = KeyTraits<K>::kMax;

    for (int j = tid; j < T; j += NT) s[pad_idx(j)] = j < len ? src[lo + j] : kMax;
    __syncthreads();
    K v[VT];
#pragma unroll
    for (int k = 0; k < VT; ++k) v[k] = s[pad_idx(tid * VT + k)];
    oddeven_sort<VT>(v);

    // only as many passes as the tile needs: runs of width >= span are done
    int span = VT;
    while (span < len) span <<= 1;
    for (int w = VT; w < span; w <<= 1) {
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VT; ++k) s[pad_idx(tid * VT + k)] = v[k];
        __syncthreads();
        const int gd = tid * VT;
        const int ps = gd & ~(2 * w - 1);
        const int diag = gd - ps;
        const int a0 = ps, b0 = ps + w;
        int l = diag - w > 0 ? diag - w : 0;
        int r = diag < w ? diag : w;
        while (l < r) {
            const int mid = (l + r) >> 1;
            if (s[pad_idx(a0 + mid)] <= s[pad_idx(b0 + diag - 1 - mid)]) l = mid + 1;
            else r = mid;
        }
        int ai = a0 + l, bi = b0 + diag - l;
        const int ae = a0 + w, be = b0 + w;
        K av = ai < ae ? s[pad_idx(ai)] : kMax;
        K bv = bi < be ? s[pad_idx(bi)] : kMax;
#pragma unroll
        for (int k = 0; k < VT; ++k) {
            const bool takeA = (bi >= be) || (ai < ae && av <= bv);
            v[k] = takeA ? av : bv;
            if (takeA) {
                ++ai;
                if (ai < ae) av = s[pad_idx(ai)];
            } else {
                ++bi;
                if (bi < be) bv = s[pad_idx(bi)];
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) s[pad_idx(tid * VT + k)] = v[k];
    __syncthreads();
    for (int j = tid; j < len; j += NT) dst[lo + j] = s[pad_idx(j)];
}

// =================================================================== K6
// Co-rank (merge-path) search for every TM-aligned output boundary of one
// merge level: corank[beta] = absolute index into run A of the split of
// output position beta*TM inside its pair (ties: A first, stable-left S:49).
template <typename K>
__global__ void k_merge_partition(const Plan *__restrict__ plan_g, K *F, K *S, const K *src0, int *corank,
                                  int level, int n, int TM, int nbounds) {
    __shared__ Plan P;
    load_plan(P, plan_g);
    __syncthreads();
    const int beta = blockIdx.x * blockDim.x + threadIdx.x;
    if (beta >= nbounds) return;
    const long long x = (long long)beta * TM;
    if (x >= n) return;
    const int b = bucket_of(P, x);
    if (level >= P.L[b]) return;
    const PairGeom g = pair_of(P, b, leaf_of(P, b, x), level);
    const K *src = (level == 0 && src0) ? src0 : level_src(P, b, level, F, S);
    const long long diag = x - g.a_lo;
    const long long na = g.b_lo - g.a_lo, nb = g.b_hi - g.b_lo;
    long long l = diag - nb > 0 ? diag - nb : 0;
    long long r = diag < na ? diag : na;
    const K *A = src + g.a_lo;
    const K *B = src + g.b_lo;
    while (l < r) {
        const long long mid = (l + r) >> 1;
        if (A[mid] <= B[diag - 1 - mid]) l = mid + 1;
        else r = mid;
    }
    corank[beta] = (int)(g.a_lo + l);
}

// One merge level over every active pair of every bucket.  CTA beta owns
// output positions [beta*TM, (beta+1)*TM) and loops over the (bucket, pair)
// pieces of that span (usually one).  Its A and B slices are fetched with two
// 1-D bulk async copies (TMA engine, 16-byte aligned supersets) completing on
// an mbarrier; each thread then merges VT outputs along the merge path in
// shared memory, and the CTA stores the span coalesced through a padded
// staging buffer.  Buckets whose levels are done are skipped (no copies).
template <typename K, int NT, int VT>
__global__ void __launch_bounds__(NT) k_merge_level(const Plan *__restrict__ plan_g, K *F, K *S, const K *src0,
                                                    const int *__restrict__ corank, int level, int n) {
    constexpr int TM = NT * VT;
    constexpr int E = 16 / sizeof(K);
    constexpr int CAP = (TM + TM / 32 > TM + 4 * E) ? TM + TM / 32 : TM + 4 * E;
    __shared__ __align__(128) K s[CAP];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ Plan P;
    const int tid = threadIdx.x;
    const long long P0 = (long long)blockIdx.x * TM;
    if (P0 >= n) return;
    const long long P1 = P0 + TM < n ? P0 + TM : (long long)n;
    load_plan(P, plan_g);
    if (tid == 0) {
        mbar_init(&mbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const K kMax = KeyTraits<K>::kMax;
    uint32_t phase = 0;
    long long x = P0;
    while (x < P1) {
        const int b = bucket_of(P, x);
        if (level >= P.L[b]) {
            x = P.off[b + 1];
            continue;
        }
        const PairGeom g = pair_of(P, b, leaf_of(P, b, x), level);
        const long long e = P1 < g.b_hi ? P1 : g.b_hi;
        const long long ax = (x == g.a_lo) ? g.a_lo : (long long)corank[blockIdx.x];
        const long long ae = (e == g.b_hi) ? g.b_lo : (long long)corank[blockIdx.x + 1];
        const long long bx = g.b_lo + (x - ax);
        const long long be = g.b_lo + (e - ae);
        const K *src = (level == 0 && src0) ? src0 : level_src(P, b, level, F, S);
        K *dst = level_dst(P, b, level, F, S);
        const int na = (int)(ae - ax), nb = (int)(be - bx), len = (int)(e - x);

        const uintptr_t ga0 = (uintptr_t)(src + ax) & ~(uintptr_t)15;
        const uintptr_t ga1 = ((uintptr_t)(src + ae) + 15) & ~(uintptr_t)15;
        const uintptr_t gb0 = (uintptr_t)(src + bx) & ~(uintptr_t)15;
        const uintptr_t gb1 = ((uintptr_t)(src + be) + 15) & ~(uintptr_t)15;
        const uint32_t bytesA = na > 0 ? (uint32_t)(ga1 - ga0) : 0u;
        const uint32_t bytesB = nb > 0 ? (uint32_t)(gb1 - gb0) : 0u;
        const K *sA = s + ((uintptr_t)(src + ax) - ga0) / sizeof(K);
        const K *sB = s + bytesA / sizeof(K) + ((uintptr_t)(src + bx) - gb0) / sizeof(K);
        if (tid == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&mbar, bytesA + bytesB);
            if (bytesA) bulk_g2s(s, (const void *)ga0, bytesA, &mbar);
            if (bytesB) bulk_g2s(s + bytesA / sizeof(K), (const void *)gb0, bytesB, &mbar);
        }
        mbar_wait(&mbar, phase);
        phase ^= 1u;

        K v[VT];
        const int diag = tid * VT;
        if (diag < len) {
            int l = diag - nb > 0 ? diag - nb : 0;
            int r = diag < na ? diag : na;
            while (l < r) {
                const int mid = (l + r) >> 1;
                if (sA[mid] <= sB[diag - 1 - mid]) l = mid + 1;
                else r = mid;
            }
            int ai = l, bi = diag - l;
            K av = ai < na ? sA[ai] : kMax;
            K bv = bi < nb ? sB[bi] : kMax;
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                const bool takeA = (bi >= nb) || (ai < na && av <= bv);
                v[k] = takeA ? av : bv;
                if (takeA) {
                    ++ai;
                    if (ai < na) av = sA[ai];
                } else {
                    ++bi;
                    if (bi < nb) bv = sB[bi];
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VT; ++k)
            if (diag + k < len) s[pad_idx(diag + k)] = v[k];
        __syncthreads();
        for (int j = tid; j < len; j += NT) dst[x + j] = s[pad_idx(j)];
        __syncthreads();
        x = e;
    }
}

// =================================================================== K7
template <typename K>
__global__ void k_copy(const K *__restrict__ src, K *__restrict__ dst, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

// =============================================================== launchers
template <typename K>
struct Geo;
template <>
struct Geo<int32_t> {
    static constexpr int kHistNT = 512;
    static constexpr int kScatNT = 512, kScatVT = 16;
    static constexpr int kSortNT = 512, kSortVT = 16;
    static constexpr int kMergeNT = 256, kMergeVT = 16;
};
template <>
struct Geo<int64_t> {
    static constexpr int kHistNT = 512;
    static constexpr int kScatNT = 512, kScatVT = 8;
    static constexpr int kSortNT = 512, kSortVT = 8;
    static constexpr int kMergeNT = 256, kMergeVT = 8;
};

template <typename K>
int tile_keys_t(int which) {
    using G = Geo<K>;
    if (which == 0) return G::kScatNT * G::kScatVT;
    if (which == 1) return G::kSortNT * G::kSortVT;
    return G::kMergeNT * G::kMergeVT;
}

template <typename K>
cudaError_t launch_histogram_t(const void *keys, int n, int h, unsigned long long div, unsigned long long magic,
                               Ctl *ctl, long long *user_off, int plan_mode, int log2c, int num_sms,
                               cudaStream_t st) {
    using G = Geo<K>;
    constexpr int E = 16 / sizeof(K);
    DigitParams<K> dp;
    dp.div = (typename KeyTraits<K>::U)div;
    dp.magic = (typename KeyTraits<K>::U)magic;
    long long nvec = ((long long)n + h + E - 1) / E;
    long long want = (nvec + G::kHistNT * 8 - 1) / (G::kHistNT * 8);  // >= 8 vectors per thread
    int grid = (int)(want < 1 ? 1 : (want > 4LL * num_sms ? 4LL * num_sms : want));
    k_histogram<K, G::kHistNT><<<grid, G::kHistNT, 0, st>>>((const K *)keys, n, h, dp, ctl, user_off, plan_mode,
                                                              log2c, tile_keys_t<K>(1));
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_scatter_t(const void *keys, void *out, int n, int h, unsigned long long div,
                             unsigned long long magic, Ctl *ctl, unsigned long long *status, cudaStream_t st) {
    using G = Geo<K>;
    constexpr int T = G::kScatNT * G::kScatVT;
    DigitParams<K> dp;
    dp.div = (typename KeyTraits<K>::U)div;
    dp.magic = (typename KeyTraits<K>::U)magic;
    long long tiles = ((long long)n + h + T - 1) / T;
    if (tiles == 0) return cudaSuccess;
    k_scatter<K, G::kScatNT, G::kScatVT><<<(unsigned)tiles, G::kScatNT, 0, st>>>((const K *)keys, (K *)out, n, h, dp,
                                                                                 ctl, status);
    return cudaGetLastError();
}

cudaError_t launch_plan(const long long *user_off, Ctl *ctl, int log2c, int mode, int tile_keys, cudaStream_t st) {
    k_plan<<<1, 32, 0, st>>>(user_off, ctl, log2c, mode, tile_keys);
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_tile_sort_t(const Plan *plan, const void *src, void *F, void *S, long long max_tiles,
                               cudaStream_t st) {
    using G = Geo<K>;
    if (max_tiles <= 0) return cudaSuccess;
    k_tile_sort<K, G::kSortNT, G::kSortVT><<<(unsigned)max_tiles, G::kSortNT, 0, st>>>(plan, (const K *)src, (K *)F,
                                                                                      (K *)S);
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_merge_level_t(const Plan *plan, void *F, void *S, const void *src0, int *corank, int level, int n,
                                 cudaStream_t st) {
    using G = Geo<K>;
    constexpr int TM = G::kMergeNT * G::kMergeVT;
    int nblocks = (int)(((long long)n + TM - 1) / TM);
    if (nblocks == 0) return cudaSuccess;
    int nbounds = nblocks + 1;
    k_merge_partition<K><<<(nbounds + 255) / 256, 256, 0, st>>>(plan, (K *)F, (K *)S, (const K *)src0, corank, level,
                                                                n, TM, nbounds);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_merge_level<K, G::kMergeNT, G::kMergeVT><<<nblocks, G::kMergeNT, 0, st>>>(plan, (K *)F, (K *)S, (const K *)src0,
                                                                              corank, level, n);
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_copy_t(const void *src, void *dst, long long n, int num_sms, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long want = (n + 255) / 256;
    int grid = (int)(want > 8LL * num_sms ? 8LL * num_sms : want);
    k_copy<K><<<grid, 256, 0, st>>>((const K *)src, (K *)dst, n);
    return cudaGetLastError();
}

// ------------------------------------------------------- dtype dispatch
#define HS_DISPATCH(dt, CALL32, CALL64) ((dt) == 0 ? (CALL32) : (CALL64))

int tile_keys(int dt, int which) { return HS_DISPATCH(dt, tile_keys_t<int32_t>(which), tile_keys_t<int64_t>(which)); }

cudaError_t launch_histogram(int dt, const void *keys, int n, int h, unsigned long long div, unsigned long long magic,
                             Ctl *ctl, long long *user_off, int plan_mode, int log2c, int num_sms, cudaStream_t st) {
    return HS_DISPATCH(dt,
                       launch_histogram_t<int32_t>(keys, n, h, div, magic, ctl, user_off, plan_mode, log2c, num_sms, st),
                       launch_histogram_t<int64_t>(keys, n, h, div, magic, ctl, user_off, plan_mode, log2c, num_sms, st));
}

cudaError_t launch_scatter(int dt, const void *keys, void *out, int n, int h, unsigned long long div,
                           unsigned long long magic, Ctl *ctl, unsigned long long *status, cudaStream_t st) {
    return HS_DISPATCH(dt, launch_scatter_t<int32_t>(keys, out, n, h, div, magic, ctl, status, st),
                       launch_scatter_t<int64_t>(keys, out, n, h, div, magic, ctl, status, st));
}

cudaError_t launch_tile_sort(int dt, const Plan *plan, const void *src, void *F, void *S, long long max_tiles,
                             cudaStream_t st) {
    return HS_DISPATCH(dt, launch_tile_sort_t<int32_t>(plan, src, F, S, max_tiles, st),
                       launch_tile_sort_t<int64_t>(plan, src, F, S, max_tiles, st));
}

cudaError_t launch_merge_level(int dt, const Plan *plan, void *F, void *S, const void *src0, int *corank, int level,
                               int n, cudaStream_t st) {
    return HS_DISPATCH(dt, launch_merge_level_t<int32_t>(plan, F, S, src0, corank, level, n, st),
                       launch_merge_level_t<int64_t>(plan, F, S, src0, corank, level, n, st));
}

cudaError_t launch_copy(int dt, const void *src, void *dst, long long n, int num_sms, cudaStream_t st) {
    return HS_DISPATCH(dt, launch_copy_t<int32_t>(src, dst, n, num_sms, st),
                       launch_copy_t<int64_t>(src, dst, n, num_sms, st));
}

}  // namespace hs
