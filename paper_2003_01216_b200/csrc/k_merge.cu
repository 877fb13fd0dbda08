// k_merge.cu -- a5 (in-chunk merge levels) and a6 (the paper's binary-tree
// merge of the chunks) as merge-path partitioned merge levels.
//
//   K6a k_merge_partition  co-rank search for every TM-aligned output boundary
//   K6b k_merge_level      persistent, double-buffered merge of every active
//                          run pair of every bucket at one level
//   K7  k_copy             in-place hs_merge with an odd number of rounds
//
// K6b pipeline (per CTA, one elected producer thread):
//   produce(piece i+1): geometry -> two 1-D bulk async copies (TMA engine) of
//                       the A and B slices into stage[(i+1)&1], mbarrier
//                       completion by byte count
//   consume(piece i):   sentinels after both slices, per-thread merge-path
//                       split in shared memory, branch-free serial merge of VT
//                       outputs (stable-left: ties take A), staging in
//                       shared memory at the destination's 16-byte phase, one
//                       1-D bulk async store of the aligned middle + scalar
//                       head/tail.
// All data movement of the level is bulk copies; threads only merge.
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

namespace hs {

template <typename K>
struct MGeo;
template <>
struct MGeo<int32_t> {
    static constexpr int kNT = 256, kVT = 16;  // 4096 outputs per piece
};
template <>
struct MGeo<int64_t> {
    static constexpr int kNT = 256, kVT = 8;  // 2048 outputs per piece
};

template <typename K>
__device__ __forceinline__ void bulk_s2g(K *dst, const K *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

__device__ __forceinline__ void load_plan_m(Plan &dst, const Plan *src) {
    constexpr int W = sizeof(Plan) / 4;
    const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
    uint32_t *d = reinterpret_cast<uint32_t *>(&dst);
    for (int i = threadIdx.x; i < W; i += blockDim.x) d[i] = __ldg(s + i);
}

// =================================================================== K6a
template <typename K>
__global__ void k_merge_partition(const Plan *__restrict__ plan_g, K *F, K *S, const K *src0, int *corank, int level,
                                  int n, int TM, int nbounds) {
    __shared__ Plan P;
    load_plan_m(P, plan_g);
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

// =================================================================== K6b
template <typename K>
struct Piece {
    long long x;  // first output position
    K *dst;
    int len, na, nb;
    int offA, offB;  // element offsets of the A / B slices inside the stage
};

template <typename K, int NT, int VT>
struct MergeSmem {
    static constexpr int TM = NT * VT;
    static constexpr int E = 16 / sizeof(K);
    // A superset (<= TM_A + 2E) | VT sentinels | pad to 16 B | B superset | VT sentinels
    static constexpr int SLOT = ((TM + 4 * E + 2 * VT + 2 * E) + E - 1) / E * E;
    static constexpr int OUT = TM + E;
    static constexpr size_t bytes() { return (size_t)(2 * SLOT + OUT) * sizeof(K); }
};

template <typename K, int NT, int VT>
__global__ void __launch_bounds__(NT) k_merge_level(const Plan *__restrict__ plan_g, K *F, K *S, const K *src0,
                                                    const int *__restrict__ corank, int level, int n, int nblocks) {
    using SM = MergeSmem<K, NT, VT>;
    constexpr int TM = SM::TM, E = SM::E, SLOT = SM::SLOT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const stage0 = reinterpret_cast<K *>(smem_raw);
    K *const sOut = stage0 + 2 * SLOT;
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ Plan P;
    __shared__ Piece<K> pc[2];
    __shared__ int s_more[2];
    const int tid = threadIdx.x;
    const K kMax = KeyTraits<K>::kMax;

    load_plan_m(P, plan_g);
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    // producer state (meaningful in thread 0 only)
    int blk = blockIdx.x;
    long long px = (long long)blk * TM;

    // Find the next piece after (blk, px), issue its loads into `slot`.
    auto produce = [&](int slot) -> int {
        while (blk < nblocks) {
            const long long P0 = (long long)blk * TM;
            const long long P1 = P0 + TM < n ? P0 + TM : (long long)n;
            if (px >= P1) {
                blk += gridDim.x;
                px = (long long)blk * TM;
                continue;
            }
            const int b = bucket_of(P, px);
            if (level >= P.L[b]) {
                px = P.off[b + 1];
                continue;
            }
            const PairGeom g = pair_of(P, b, leaf_of(P, b, px), level);
            const long long e = P1 < g.b_hi ? P1 : g.b_hi;
            // px is either a pair start or the block start P0 (whose co-rank K6a stored)
            const long long ax = (px == g.a_lo) ? g.a_lo : (long long)corank[blk];
            const long long ae = (e == g.b_hi) ? g.b_lo : (long long)corank[blk + 1];
            const long long bx = g.b_lo + (px - ax);
            const long long be = g.b_lo + (e - ae);
            const K *src = (level == 0 && src0) ? src0 : level_src(P, b, level, F, S);
            Piece<K> q;
            q.x = px;
            q.dst = level_dst(P, b, level, F, S);
            q.na = (int)(ae - ax);
            q.nb = (int)(be - bx);
            q.len = (int)(e - px);
            const uintptr_t ga0 = (uintptr_t)(src + ax) & ~(uintptr_t)15;
            const uintptr_t ga1 = ((uintptr_t)(src + ae) + 15) & ~(uintptr_t)15;
            const uintptr_t gb0 = (uintptr_t)(src + bx) & ~(uintptr_t)15;
            const uintptr_t gb1 = ((uintptr_t)(src + be) + 15) & ~(uintptr_t)15;
            const uint32_t bytesA = q.na > 0 ? (uint32_t)(ga1 - ga0) : 0u;
            const uint32_t bytesB = q.nb > 0 ? (uint32_t)(gb1 - gb0) : 0u;
            q.offA = (int)(((uintptr_t)(src + ax) - ga0) / sizeof(K));
            // B's superset starts at the first 16-byte boundary past A's slice + VT sentinels
            const int bstart = ((q.offA + q.na + VT) + E - 1) / E * E;
            const int bstart2 = bstart * (int)sizeof(K) >= (int)bytesA ? bstart : (int)(bytesA / sizeof(K));
            q.offB = bstart2 + (int)(((uintptr_t)(src + bx) - gb0) / sizeof(K));
            K *st = stage0 + slot * SLOT;
            fence_proxy_async_smem();  // prior generic reads of this slot precede the async writes
            mbar_arrive_expect_tx(&mbar[slot], bytesA + bytesB);
            if (bytesA) bulk_g2s(st, (const void *)ga0, bytesA, &mbar[slot]);
            if (bytesB) bulk_g2s(st + bstart2, (const void *)gb0, bytesB, &mbar[slot]);
            pc[slot] = q;
            px = e;
            return 1;
        }
        return 0;
    };

    if (tid == 0) s_more[0] = produce(0);
    __syncthreads();
    uint32_t phases = 0u;  // bit s = parity of stage s's mbarrier
    int cur = 0;
    while (s_more[cur]) {
        if (tid == 0) s_more[cur ^ 1] = produce(cur ^ 1);
        mbar_wait(&mbar[cur], (phases >> cur) & 1u);
        phases ^= 1u << cur;
        const Piece<K> q = pc[cur];
        K *const sb = stage0 + cur * SLOT;
        // VT sentinels after each slice (overwrites superset spill-over)
        if (tid < VT) sb[q.offA + q.na + tid] = kMax;
        else if (tid < 2 * VT) sb[q.offB + q.nb + tid - VT] = kMax;
        __syncthreads();

        // staging position p holds output p - sh; sh = destination's 16-byte phase
        const int sh = (int)(((uintptr_t)(q.dst + q.x) & 15) / sizeof(K));
        const int p_lo = tid * VT > sh ? tid * VT : sh;
        const int diag = p_lo - sh;
        K v[VT];
        if (diag < q.len) {
            int l = diag - q.nb > 0 ? diag - q.nb : 0;
            int r = diag < q.na ? diag : q.na;
            const K *A = sb + q.offA;
            const K *B = sb + q.offB;
            while (l < r) {
                const int mid = (l + r) >> 1;
                if (A[mid] <= B[diag - 1 - mid]) l = mid + 1;
                else r = mid;
            }
            int ai = q.offA + l, bi = q.offB + diag - l;
            K a = sb[ai], b = sb[bi];
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                const bool p = a <= b;
                v[k] = p ? a : b;
                if (k + 1 < VT) {
                    const int nx = (p ? ai : bi) + 1;
                    const K t = sb[nx];
                    ai = p ? nx : ai;
                    bi = p ? bi : nx;
                    a = p ? t : a;
                    b = p ? b : t;
                }
            }
        }
        // the previous piece's bulk store must have finished reading sOut
        if (tid == 0) bulk_wait_read0();
        __syncthreads();
        const int end = sh + q.len;
        if (diag < q.len) {
            if (tid * VT >= sh && (tid + 1) * VT <= end) {
#pragma unroll
                for (int k = 0; k < VT; k += E) {
                    int4 w;
                    memcpy(&w, &v[k], 16);
                    *reinterpret_cast<int4 *>(sOut + tid * VT + k) = w;
                }
            } else {
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    const int p = p_lo + k;
                    if (p < (tid + 1) * VT && p < end) sOut[p] = v[k];
                }
            }
        }
        fence_proxy_async_smem();  // make the staged outputs visible to the bulk store
        __syncthreads();
        const int m0 = sh == 0 ? 0 : E;       // first 16-byte aligned staging position
        const int m1 = end / E * E;            // last one
        K *const g = q.dst + q.x - sh;        // staging position p <-> g[p]
        if (m1 > m0) {
            if (tid == 0) {
                bulk_s2g(g + m0, sOut + m0, (uint32_t)((m1 - m0) * sizeof(K)));
                bulk_commit();
            }
            if (tid < E) {
                const int p = sh + tid;  // head
                if (p < m0 && p < end) g[p] = sOut[p];
            } else if (tid < 2 * E) {
                const int p = m1 + tid - E;  // tail
                if (p < end && p >= m0) g[p] = sOut[p];
            }
        } else {
            for (int p = sh + tid; p < end; p += NT) g[p] = sOut[p];
        }
        cur ^= 1;
    }
    if (tid == 0) bulk_wait_read0();
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
cudaError_t launch_merge_level_t(const Plan *plan, void *F, void *S, const void *src0, int *corank, int level, int n,
                                 int num_sms, cudaStream_t st) {
    using G = MGeo<K>;
    using SM = MergeSmem<K, G::kNT, G::kVT>;
    constexpr int TM = SM::TM;
    static bool configured = false;  // per process; attribute is per function
    static int per_sm = 1;
    auto kern = k_merge_level<K, G::kNT, G::kVT>;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::bytes());
        if (e != cudaSuccess) return e;
        int occ = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::kNT, SM::bytes());
        if (e != cudaSuccess) return e;
        per_sm = occ > 0 ? occ : 1;
        configured = true;
    }
    const int nblocks = (int)(((long long)n + TM - 1) / TM);
    if (nblocks == 0) return cudaSuccess;
    const int nbounds = nblocks + 1;
    k_merge_partition<K><<<(nbounds + 255) / 256, 256, 0, st>>>(plan, (K *)F, (K *)S, (const K *)src0, corank, level,
                                                                n, TM, nbounds);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    long long grid = (long long)per_sm * num_sms;
    if (grid > nblocks) grid = nblocks;
    kern<<<(unsigned)grid, G::kNT, SM::bytes(), st>>>(plan, (K *)F, (K *)S, (const K *)src0, corank, level, n, nblocks);
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

int merge_span(int dt) { return dt == 0 ? merge_span_t<int32_t>() : merge_span_t<int64_t>(); }

cudaError_t launch_merge_level(int dt, const Plan *plan, void *F, void *S, const void *src0, int *corank, int level,
                               int n, int num_sms, cudaStream_t st) {
    return dt == 0 ? launch_merge_level_t<int32_t>(plan, F, S, src0, corank, level, n, num_sms, st)
                   : launch_merge_level_t<int64_t>(plan, F, S, src0, corank, level, n, num_sms, st);
}

cudaError_t launch_copy(int dt, const void *src, void *dst, long long n, int num_sms, cudaStream_t st) {
    return dt == 0 ? launch_copy_t<int32_t>(src, dst, n, num_sms, st) : launch_copy_t<int64_t>(src, dst, n, num_sms, st);
}

}  // namespace hs
