// k_merge.cu -- a5 (in-chunk merge levels) and a6 (the paper's binary-tree
// merge of the chunks) as streaming merge-path merge levels.
//
//   K6 k_merge_level  one merge level over every active run pair of every
//                     bucket (persistent, warp-specialised, sliding windows)
//   K7 k_copy         in-place hs_merge with an odd number of rounds
//
// Work split.  The output positions of the active buckets of a level are cut
// into gridDim.x equal contiguous ranges, one per CTA.  A CTA walks its range
// piece by piece (TM = NC*VT outputs, never crossing a pair), so the merge-path
// split at the end of one piece is the start of the next one: only the first
// piece of a CTA needs a co-rank search in global memory (one warp, a 33-ary
// search), and no co-rank table or search kernel exists.
//
// Sliding windows.  The A runs of the CTA's pairs, concatenated, form its
// "A stream"; likewise the B runs.  Each stream is staged in a shared-memory
// ring of W keys (stream position s lives in slot s mod W).  Every run starts
// at a stream position with the same 16-byte phase as its global address, so
// the producer moves whole 16-byte granules with 1-D bulk async copies (TMA
// engine) and every key is read from HBM exactly once.
//
// Pipeline (per CTA; warps 0..NC/32-1 consume, the last warp produces).
// Barriers: dbar[NB] (bulk-load batches, completion counted in bytes),
// cbar[2] (descriptor k published), done[2] (consumers finished piece k).
//   producer, iteration k >= 1:
//     wait the batch holding piece k-1 -> merge-path split of piece k-1 at its
//     length -> stream positions of piece k -> wait done[k-2] (its descriptor
//     slot and ring slots are free) -> publish descriptor k (cbar) ->
//     bulk-load both streams up to (start of piece k-1) + W as batch k.
//   consumers, piece k: wait cbar[k] and batch k-LOOK -> per-thread merge-path
//     split in the rings + branch-free serial merge of VT outputs
//     (stable-left: ties take A) -> arrive done[k] -> stage outputs at
//     the destination's 16-byte phase -> one 1-D bulk async store (+ scalar
//     head/tail).
// W >= (LOOK+2) TM + padding, so piece k's keys were requested LOOK pieces
// before it is merged: HBM latency hides behind LOOK pieces of merging.
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

#ifndef HS_MERGE_NT
#define HS_MERGE_NT 128
#endif
#ifndef HS_MERGE_VT
#define HS_MERGE_VT 15
#endif
#ifndef HS_MERGE_W
#define HS_MERGE_W 8192
#endif
#ifndef HS_MERGE_VT64
#define HS_MERGE_VT64 9
#endif
#ifndef HS_MERGE_W64
#define HS_MERGE_W64 4096
#endif

namespace hs {

template <typename K>
struct MGeo;
template <>
struct MGeo<int32_t> {
    // odd VT: lanes' merge positions (spaced ~VT/2 words) spread over all banks
    static constexpr int kNT = HS_MERGE_NT, kVT = HS_MERGE_VT, kW = HS_MERGE_W;
};
template <>
struct MGeo<int64_t> {
    static constexpr int kNT = HS_MERGE_NT, kVT = HS_MERGE_VT64, kW = HS_MERGE_W64;
};

template <typename K>
__device__ __forceinline__ void bulk_s2g(K *dst, const K *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void consumer_bar(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ void load_plan_m(Plan &dst, const Plan *src) {
    constexpr int W = sizeof(Plan) / 4;
    const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
    uint32_t *d = reinterpret_cast<uint32_t *>(&dst);
    for (int i = threadIdx.x; i < W; i += blockDim.x) d[i] = __ldg(s + i);
}

// The pair of level lam that contains output position x, searching forward
// from bucket b over positions < X1 (skips buckets this level leaves alone).
// Returns false when no position of an active bucket is left below X1.
__device__ __forceinline__ bool seek_pair(const Plan &P, int lam, long long X1, long long &x, int &b, PairGeom &g) {
    for (;;) {
        if (x >= X1) return false;
        while (b < 9 && x >= P.off[b + 1]) ++b;
        if (lam >= P.L[b]) {
            if (b == 9) return false;
            x = P.off[b + 1];
            continue;
        }
        g = pair_of(P, b, leaf_of(P, b, x), lam);  // x lies in a leaf, so the pair is not empty
        return true;
    }
}

// Output range [X0, X1) of CTA c out of G over the active buckets of level lam.
__device__ __forceinline__ void cta_range(const Plan &P, int lam, int c, int G, long long &X0, long long &X1) {
    long long nact = 0;
    for (int b = 0; b < 10; ++b)
        if (lam < P.L[b]) nact += P.off[b + 1] - P.off[b];
    const long long lo = nact * c / G, hi = nact * (c + 1) / G;
    X0 = X1 = 0;
    if (lo >= hi) return;
    long long acc = 0;
    bool got0 = false;
    for (int b = 0; b < 10; ++b) {
        if (lam >= P.L[b]) continue;
        const long long m = P.off[b + 1] - P.off[b];
        if (!got0 && lo < acc + m) {
            X0 = P.off[b] + (lo - acc);
            got0 = true;
        }
        if (hi <= acc + m) {
            X1 = P.off[b] + (hi - acc);
            return;
        }
        acc += m;
    }
}

template <typename K>
__device__ __forceinline__ const K *pair_src(const Plan &P, int b, int lam, K *F, K *S, const K *src0) {
    return (lam == 0 && src0) ? src0 : level_src(P, b, lam, F, S);
}

template <typename K>
__device__ __forceinline__ int phase_of(const K *p) {
    return (int)(((uintptr_t)p & 15) / sizeof(K));
}

// Merge-path split of output diag between ring windows A = RA[ca, ca+na) and
// B = RB[cb, cb+nb) (slots mod W; stable-left).
template <typename K, int W>
__device__ __forceinline__ int ring_merge_path(const K *RA, int ca, int na, const K *RB, int cb, int nb, int diag) {
    int l = diag - nb > 0 ? diag - nb : 0;
    int r = diag < na ? diag : na;
    while (l < r) {
        const int mid = (l + r) >> 1;
        if (RA[(ca + mid) & (W - 1)] <= RB[(cb + diag - 1 - mid) & (W - 1)]) l = mid + 1;
        else r = mid;
    }
    return l;
}

// One piece as the consumers see it (stream positions are ints: a CTA's
// streams are shorter than n + padding < 2^31).
template <typename K>
struct SPiece {
    long long x;  // first output position
    K *dst;       // destination buffer of the pair
    int len;      // outputs (< 0: no more pieces)
    int ca, cb;   // stream positions of the first unconsumed A / B keys
    int ea, eb;   // stream end of the current A / B run
};

// Producer-side cursor over the runs of one stream (A or B) of a CTA, and the
// bulk loads that stage it.  Runs are taken in pair order; run r occupies
// stream positions [base_r, base_r + len_r) with base_r = align16(end of run
// r-1) + phase(run r's first key), so loads are whole 16-byte granules.
template <typename K, int W>
struct Loader {
    long long px;     // output position where the next pair starts
    int pb;           // bucket cursor
    const K *src;     // buffer of the current run
    long long gcur;   // next global index to load (granule aligned)
    long long gend;   // end of the current run
    int scur;         // stream position of gcur (granule aligned)
    bool has;         // a run is open
    bool first;       // the next run opened is the CTA's first (partial) one
    long long first_lo;

    // Issue bulk loads up to stream position `limit` (granule aligned);
    // returns the bytes issued (completion counted on `bar`).
    __device__ uint32_t fill(const Plan &P, int lam, long long X1, K *F, K *S, const K *src0, bool isA, K *ring,
                             int limit, uint64_t *bar) {
        constexpr int E = 16 / sizeof(K);
        uint32_t bytes = 0;
        for (;;) {
            if (!has) {
                PairGeom g;
                if (!seek_pair(P, lam, X1, px, pb, g)) break;
                src = pair_src(P, pb, lam, F, S, src0);
                const long long lo = first ? first_lo : (isA ? g.a_lo : g.b_lo);
                const long long hi = isA ? g.b_lo : g.b_hi;
                gcur = lo - phase_of(src + lo);
                gend = hi;
                has = true;
                first = false;
                px = g.b_hi;
            }
            if (gcur >= gend) {
                has = false;
                continue;
            }
            const int remr = (int)((gend - gcur + E - 1) / E * E);
            const int room = limit - scur;
            if (room <= 0) break;
            const int take = remr <= room ? remr : room;
            const int slot = scur & (W - 1);
            const int p1 = take < W - slot ? take : W - slot;
            mbar_expect_tx(bar, (uint32_t)(take * sizeof(K)));
            bulk_g2s(ring + slot, src + gcur, (uint32_t)(p1 * sizeof(K)), bar);
            if (take > p1) bulk_g2s(ring, src + gcur + p1, (uint32_t)((take - p1) * sizeof(K)), bar);
            bytes += (uint32_t)(take * sizeof(K));
            gcur += take;
            scur += take;
        }
        return bytes;
    }
};

// Co-rank of output diag of merge(A[0..na), B[0..nb)) by the 32 lanes of one
// warp: each round every lane probes one candidate and a ballot finds the
// crossing, so ~log_33 steps of dependent global loads instead of log_2.
template <typename K>
__device__ __forceinline__ long long warp_corank(const K *A, long long na, const K *B, long long nb, long long diag) {
    const int lane = threadIdx.x & 31;
    long long l = diag - nb > 0 ? diag - nb : 0;  // answer in [l, r]
    long long r = diag < na ? diag : na;
    while (l < r) {
        const long long step = (r - l + 32) / 33;  // >= 1
        const long long c = l + (long long)(lane + 1) * step;
        const bool p = (c <= r) && (A[c - 1] <= B[diag - c]);
        const unsigned m = __ballot_sync(0xffffffffu, p);
        const int cnt = __popc(m);  // probes are monotone: the true ones form a prefix
        const long long fail = l + (long long)(cnt + 1) * step;
        l += (long long)cnt * step;
        if (cnt < 32 && fail - 1 < r) r = fail - 1;
    }
    return l;
}

template <typename K, int NC, int VT, int W>
struct MergeSmem {
    static constexpr int TM = NC * VT;
    static constexpr int E = 16 / sizeof(K);
    static constexpr int OUT = TM + E;
    static_assert((W & (W - 1)) == 0, "ring size must be a power of two");
    // lookahead d: piece k reads keys loaded by the batch issued d pieces
    // earlier; needs W >= (d+2) TM + (d+1) 2E + E (one pair switch per piece)
    static constexpr int LOOK = (W - E + 2 * E) / (TM + 2 * E) - 2;
    static_assert(LOOK >= 1, "ring too small for one piece of lookahead");
    static constexpr int NB = LOOK + 2;  // data-barrier ring depth
    static constexpr size_t bytes() { return (size_t)(2 * W + 2 * OUT) * sizeof(K); }
};

template <typename K, int NC, int VT, int W>
__global__ void __launch_bounds__(NC + 32) k_merge_level(const Plan *__restrict__ plan_g, K *F, K *S, const K *src0,
                                                         int level) {
    using SM = MergeSmem<K, NC, VT, W>;
    constexpr int TM = SM::TM, E = SM::E, OUT = SM::OUT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const RA = reinterpret_cast<K *>(smem_raw);
    K *const RB = RA + W;
    K *const out0 = RB + W;
    constexpr int LOOK = SM::LOOK, NB = SM::NB;
    __shared__ __align__(8) uint64_t dbar[NB];  // bulk-load batches (tx counted)
    __shared__ __align__(8) uint64_t cbar[2];   // descriptor k published
    __shared__ __align__(8) uint64_t done[2];   // consumers finished reading piece k
    __shared__ Plan P;
    __shared__ SPiece<K> desc[2];
    const int tid = threadIdx.x;
    const K kMax = KeyTraits<K>::kMax;

    load_plan_m(P, plan_g);
    if (tid == 0) {
        for (int i = 0; i < NB; ++i) mbar_init(&dbar[i], 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&cbar[i], 1);
            mbar_init(&done[i], NC / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    long long X0, X1;
    cta_range(P, level, blockIdx.x, gridDim.x, X0, X1);
    if (X0 >= X1) return;

    if (tid >= NC) {
        // ---------------------------------------------------------- producer
        const int lane = tid & 31;
        long long dx = X0;
        int db = 0;
        PairGeom g;
        seek_pair(P, level, X1, dx, db, g);  // X0 lies in an active bucket
        const K *src = pair_src(P, db, level, F, S, src0);
        long long ca_abs = g.a_lo;
        if (X0 != g.a_lo)
            ca_abs = g.a_lo + warp_corank(src + g.a_lo, g.b_lo - g.a_lo, src + g.b_lo, g.b_hi - g.b_lo, X0 - g.a_lo);
        if (lane != 0) return;
        const long long cb_abs = g.b_lo + (X0 - ca_abs);

        Loader<K, W> LA, LB;
        LA.px = LB.px = X0;
        LA.pb = LB.pb = 0;
        LA.has = LB.has = false;
        LA.first = LB.first = true;
        LA.first_lo = ca_abs;
        LB.first_lo = cb_abs;
        LA.scur = LB.scur = 0;

        // descriptor cursor: current pair g (bucket db), output position dx,
        // stream positions / run ends of the current A and B runs
        int ca = phase_of(src + ca_abs), cb = phase_of(src + cb_abs);
        int ea = ca + (int)(g.b_lo - ca_abs), eb = cb + (int)(g.b_hi - cb_abs);
        K *dst = level_dst(P, db, level, F, S);
        auto make = [&](SPiece<K> &q) {
            long long e = dx + TM;
            if (e > g.b_hi) e = g.b_hi;
            if (e > X1) e = X1;
            q.x = dx;
            q.dst = dst;
            q.len = (int)(e - dx);
            q.ca = ca;
            q.cb = cb;
            q.ea = ea;
            q.eb = eb;
        };
        SPiece<K> cur;
        make(cur);
        desc[0] = cur;
        mbar_arrive(&cbar[0]);
        int prev_ca = ca, prev_cb = cb;  // consumption pointers at the start of piece k-1
        {
            const int limA = (ca + W) / E * E, limB = (cb + W) / E * E;
            LA.fill(P, level, X1, F, S, src0, true, RA, limA, &dbar[0]);
            LB.fill(P, level, X1, F, S, src0, false, RB, limB, &dbar[0]);
            mbar_arrive(&dbar[0]);
        }
        for (int k = 1;; ++k) {
            // split of piece k-1 (= cur) -> start of piece k (its keys were loaded
            // by batch max(0, k-1-LOOK))
            {
                const int bj = k - 1 - LOOK > 0 ? k - 1 - LOOK : 0;
                mbar_wait(&dbar[bj % NB], (bj / NB) & 1);
            }
            SPiece<K> nxt;
            {
                const int na = cur.ea - cur.ca < cur.len ? cur.ea - cur.ca : cur.len;
                const int nb = cur.eb - cur.cb < cur.len ? cur.eb - cur.cb : cur.len;
                const int da = ring_merge_path<K, W>(RA, cur.ca, na, RB, cur.cb, nb, cur.len);
                ca = cur.ca + da;
                cb = cur.cb + (cur.len - da);
                dx = cur.x + cur.len;
                if (dx >= g.b_hi && dx < X1) {  // next pair: new runs in both streams
                    if (seek_pair(P, level, X1, dx, db, g)) {
                        const K *s2 = pair_src(P, db, level, F, S, src0);
                        dst = level_dst(P, db, level, F, S);
                        ca = (ea + E - 1) / E * E + phase_of(s2 + g.a_lo);
                        cb = (eb + E - 1) / E * E + phase_of(s2 + g.b_lo);
                        ea = ca + (int)(g.b_lo - g.a_lo);
                        eb = cb + (int)(g.b_hi - g.b_lo);
                    } else {
                        dx = X1;
                    }
                }
                if (dx < X1) make(nxt);
                else nxt.len = -1;
            }
            // pieces <= k-2 are merged: their descriptor slot and ring slots are free
            if (k >= 2) mbar_wait(&done[(k - 2) & 1], ((k - 2) >> 1) & 1);
            desc[k & 1] = nxt;
            mbar_arrive(&cbar[k & 1]);
            if (nxt.len < 0) return;  // every batch a consumer waits for is armed
            const int limA = (prev_ca + W) / E * E, limB = (prev_cb + W) / E * E;
            LA.fill(P, level, X1, F, S, src0, true, RA, limA, &dbar[k % NB]);
            LB.fill(P, level, X1, F, S, src0, false, RB, limB, &dbar[k % NB]);
            mbar_arrive(&dbar[k % NB]);
            prev_ca = nxt.ca;
            prev_cb = nxt.cb;
            cur = nxt;
        }
    }

    // -------------------------------------------------------------- consumers
    const int lane = tid & 31;
    for (int it = 0;; ++it) {
        mbar_wait(&cbar[it & 1], (it >> 1) & 1);
        const SPiece<K> q = desc[it & 1];
        if (q.len < 0) {
            // batches 0 .. it-1 are armed; the last LOOK of them may still be
            // landing in the rings: drain them before the CTA's smem is released
            for (int j = it - LOOK > 0 ? it - LOOK : 0; j < it; ++j) mbar_wait(&dbar[j % NB], (j / NB) & 1);
            break;
        }
        {
            const int bj = it - LOOK > 0 ? it - LOOK : 0;
            mbar_wait(&dbar[bj % NB], (bj / NB) & 1);
        }
        const int na = q.ea - q.ca < q.len ? q.ea - q.ca : q.len;
        const int nb = q.eb - q.cb < q.len ? q.eb - q.cb : q.len;
        // staging position p holds output p - sh; sh = destination's 16-byte phase
        const int sh = phase_of(q.dst + q.x);
        const int p_lo = tid * VT > sh ? tid * VT : sh;
        const int diag = p_lo - sh;
        K v[VT];
        if (diag < q.len) {
            const int a0 = ring_merge_path<K, W>(RA, q.ca, na, RB, q.cb, nb, diag);
            // an exhausted run reads as kMax (an exhausted A only "wins" a tie
            // against a real kMax in B, and then emits the same value), so the
            // loop needs no bounds branches
            const int a_end = q.ca + na, b_end = q.cb + nb;
            int ai = q.ca + a0, bi = q.cb + diag - a0;
            K x = ai < a_end ? RA[ai & (W - 1)] : kMax;
            K y = bi < b_end ? RB[bi & (W - 1)] : kMax;
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                const bool p = x <= y;
                v[k] = p ? x : y;
                if (k + 1 < VT) {
                    const int nx = (p ? ai : bi) + 1;
                    const int lim = p ? a_end : b_end;
                    const K t = (p ? RA : RB)[nx & (W - 1)];
                    const K tv = nx < lim ? t : kMax;
                    ai = p ? nx : ai;
                    bi = p ? bi : nx;
                    x = p ? tv : x;
                    y = p ? y : tv;
                }
            }
        }
        // overhang: with sh > 0 a full piece spans up to E-1 positions past NC*VT
        const int over = sh + q.len - NC * VT;
        K vx[E];
        if (over > 0 && tid == NC - 1) {
            const int dxo = NC * VT - sh;
            int ai = ring_merge_path<K, W>(RA, q.ca, na, RB, q.cb, nb, dxo), bi = dxo - ai;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const K x = ai < na ? RA[(q.ca + ai) & (W - 1)] : kMax;
                const K y = bi < nb ? RB[(q.cb + bi) & (W - 1)] : kMax;
                const bool p = (bi >= nb) || (ai < na && x <= y);
                vx[k] = p ? x : y;
                ai += p ? 1 : 0;
                bi += p ? 0 : 1;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[it & 1]);  // this warp is done with the rings

        K *sOut = out0 + (it & 1) * OUT;
        if (tid == 0) bulk_wait_read1();  // the store two pieces ago has read sOut
        consumer_bar(NC);
        const int end = sh + q.len;
        if (diag < q.len) {
            if (tid * VT >= sh && (tid + 1) * VT <= end) {
#pragma unroll
                for (int k = 0; k < VT; ++k) sOut[tid * VT + k] = v[k];  // VT odd: conflict-free
            } else {
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    const int p = p_lo + k;
                    if (p < (tid + 1) * VT && p < end) sOut[p] = v[k];
                }
            }
        }
        if (over > 0 && tid == NC - 1) {
#pragma unroll
            for (int k = 0; k < E; ++k)
                if (k < over) sOut[NC * VT + k] = vx[k];
        }
        fence_proxy_async_smem();  // staged outputs -> visible to the bulk store
        consumer_bar(NC);
        const int m0 = sh == 0 ? 0 : E;  // first 16-byte aligned staging position
        const int m1 = end / E * E;      // last one
        K *const gdst = q.dst + q.x - sh;  // staging position p <-> gdst[p]
        if (m1 > m0) {
            if (tid == 0) bulk_s2g(gdst + m0, sOut + m0, (uint32_t)((m1 - m0) * sizeof(K)));
            if (tid < E) {
                const int p = sh + tid;  // head
                if (p < m0 && p < end) gdst[p] = sOut[p];
            } else if (tid < 2 * E) {
                const int p = m1 + tid - E;  // tail
                if (p < end) gdst[p] = sOut[p];
            }
        } else {
            for (int p = sh + tid; p < end; p += NC) gdst[p] = sOut[p];
        }
        if (tid == 0) bulk_commit();  // one group per piece (possibly empty)
    }
    if (tid == 0) bulk_wait0();
}

// =================================================================== K7
template <typename K>
__global__ void k_copy(const K *__restrict__ src, K *__restrict__ dst, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

// =============================================================== launchers
template <typename K>
int merge_span_t() {
    return MGeo<K>::kNT * MGeo<K>::kVT;
}

template <typename K>
cudaError_t launch_merge_level_t(const Plan *plan, void *F, void *S, const void *src0, int level, int n, int num_sms,
                                 cudaStream_t st) {
    using G = MGeo<K>;
    using SM = MergeSmem<K, G::kNT, G::kVT, G::kW>;
    constexpr int TM = SM::TM;
    auto kern = k_merge_level<K, G::kNT, G::kVT, G::kW>;
    static int configured_dev = -1;
    static int per_sm = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::bytes());
        if (e != cudaSuccess) return e;
        int occ = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::kNT + 32, SM::bytes());
        if (e != cudaSuccess) return e;
        per_sm = occ > 0 ? occ : 1;
        configured_dev = dev;
    }
    const long long pieces = ((long long)n + TM - 1) / TM;
    if (pieces == 0) return cudaSuccess;
    long long grid = (long long)per_sm * num_sms;
    // at least ~8 pieces per CTA so the one co-rank search per CTA stays cheap
    const long long cap = (pieces + 7) / 8;
    if (grid > cap) grid = cap;
    prof_begin(kProfMergeLevel, st);
    kern<<<(unsigned)grid, G::kNT + 32, SM::bytes(), st>>>(plan, (K *)F, (K *)S, (const K *)src0, level);
    prof_end(kProfMergeLevel, st);
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_copy_t(const void *src, void *dst, long long n, int num_sms, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long want = (n + 255) / 256;
    int grid = (int)(want > 8LL * num_sms ? 8LL * num_sms : want);
    prof_begin(kProfCopy, st);
    k_copy<K><<<grid, 256, 0, st>>>((const K *)src, (K *)dst, n);
    prof_end(kProfCopy, st);
    return cudaGetLastError();
}

int merge_span(int dt) { return dt == 0 ? merge_span_t<int32_t>() : merge_span_t<int64_t>(); }

cudaError_t launch_merge_level(int dt, const Plan *plan, void *F, void *S, const void *src0, int *corank, int level,
                               int n, int num_sms, cudaStream_t st) {
    (void)corank;
    return dt == 0 ? launch_merge_level_t<int32_t>(plan, F, S, src0, level, n, num_sms, st)
                   : launch_merge_level_t<int64_t>(plan, F, S, src0, level, n, num_sms, st);
}

cudaError_t launch_copy(int dt, const void *src, void *dst, long long n, int num_sms, cudaStream_t st) {
    return dt == 0 ? launch_copy_t<int32_t>(src, dst, n, num_sms, st) : launch_copy_t<int64_t>(src, dst, n, num_sms, st);
}

}  // namespace hs
