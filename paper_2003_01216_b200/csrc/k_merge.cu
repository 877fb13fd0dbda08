// k_merge.cu -- a5 (in-chunk merge levels) and a6 (the paper's binary-tree
// merge of the chunks) as merge-path partitioned merge levels.
//
//   K6a k_merge_partition  co-rank search for every TM-aligned output boundary,
//                          coarse phase on the previous generation's key
//                          samples (L2), fine phase over ~64 keys in HBM
//   K6b k_merge_level      persistent, double-buffered merge of every active
//                          run pair of every bucket at one level; writes the
//                          key samples of its output for the next level
//   k_sample               samples of caller-given runs (hs_merge level 0)
//   K7  k_copy             in-place hs_merge with an odd number of rounds
//
// K6b pipeline (per CTA, warp-specialised):
//   producer warp: piece geometry -> two 1-D bulk async copies (TMA engine)
//                  of the A and B slices into a ring of ST stages; full /
//                  empty mbarriers (full completes on the byte count)
//   consumer warps: per-thread merge-path split in shared memory,
//                  branch-free serial merge of VT outputs (stable-left: ties
//                  take A), staging in shared memory at the
//                  destination's 16-byte phase, one 1-D bulk async store of the
//                  aligned middle per piece + scalar head/tail.
// All data movement of the level is bulk copies; threads only merge.
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

#ifndef HS_MERGE_NT
#define HS_MERGE_NT 128
#endif
#ifndef HS_MERGE_VT
#define HS_MERGE_VT 25
#endif
#ifndef HS_MERGE_VT64
#define HS_MERGE_VT64 13
#endif
#ifndef HS_MERGE_ST
#define HS_MERGE_ST 2
#endif

namespace hs {


template <typename K>
struct MGeo;
template <>
struct MGeo<int32_t> {
    // odd VT: lanes' merge positions (spaced ~VT/2 words) spread over all banks
    static constexpr int kNT = HS_MERGE_NT, kVT = HS_MERGE_VT, kST = HS_MERGE_ST;  // default 128 x 25, 2 stages
};
template <>
struct MGeo<int64_t> {
    static constexpr int kNT = HS_MERGE_NT, kVT = HS_MERGE_VT64, kST = HS_MERGE_ST;
};
template <>
struct MGeo<KV64> {  // f3 items (k_kv.cu)
    static constexpr int kNT = HS_MERGE_NT, kVT = 7, kST = HS_MERGE_ST;
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
// Co-rank (merge-path) search for every TM-aligned output boundary of one
// merge level: corank[beta] = absolute index into run A of the split of
// output position beta*TM inside its pair (ties: A first, stable-left S:49).
// Q(m) := A[m] <= B[diag-1-m] is true on a prefix of [l0, r0); the co-rank is
// the first m where it fails.
//   coarse: only at the m whose A[m] is a sample (position = Q-1 mod Q), with
//     B[diag-1-m] bracketed by its two neighbouring B samples, Q(m) is either
//     surely true, surely false or open; two binary searches over these
//     candidates (samples only: L2-resident) leave an interval of ~Q keys;
//   fine: plain binary search of Q(m) over that interval (the only HBM reads).
template <typename K>
__global__ void k_merge_partition(const Plan *__restrict__ plan_g, K *F, K *S, const K *src0,
                                  const K *__restrict__ samp, int *corank, int level, int n, int TM, int nbounds) {
    constexpr long long Q = kSampleQ;
    griddep_wait();
    if (level >= __ldg(&plan_g->Lmax)) return;  // no bucket runs this level (the host only knows a bound)
    __shared__ Plan P;
    load_plan_m(P, plan_g);
    __syncthreads();
    if (level >= P.Lmax) return;  // no bucket runs this level (the host only knows a bound)
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
    long long l = diag - nb > 0 ? diag - nb : 0;  // answer in [l, r]
    long long r = diag < na ? diag : na;
    if (l < r) {
        // candidates m_j = m0 + j Q, j < J, with A[m_j] a sample
        const long long m0 = l + (Q - 1 - (g.a_lo + l) % Q);
        const long long J = m0 < r ? (r - 1 - m0) / Q + 1 : 0;
        // T(j): surely true (A[m_j] <= lower B sample), a prefix of j;
        // F(j): surely false (A[m_j] > upper B sample), a suffix of j.
        // Both binary searches advance together (independent L2 loads).
        long long tlo = 0, thi = J, flo = 0, fhi = J;
        while (tlo < thi || flo < fhi) {
            const long long jt = (tlo + thi) >> 1, jf = (flo + fhi) >> 1;
            const long long mt = m0 + jt * Q, mf = m0 + jf * Q;
            const long long pl = (g.b_lo + diag - 1 - mt) / Q * Q - 1;
            const long long pu = (g.b_lo + diag - 1 - mf) / Q * Q + Q - 1;
            if (tlo < thi) {
                const bool t = pl >= g.b_lo && ldg_key(samp + (g.a_lo + mt) / Q) <= ldg_key(samp + pl / Q);
                if (t) tlo = jt + 1;
                else thi = jt;
            }
            if (flo < fhi) {
                const bool f = pu < g.b_hi && ldg_key(samp + (g.a_lo + mf) / Q) > ldg_key(samp + pu / Q);
                if (f) fhi = jf;
                else flo = jf + 1;
            }
        }
        const long long jT = tlo, jF = flo;
        if (jT > 0) l = m0 + (jT - 1) * Q + 1;
        if (jF < J) r = m0 + jF * Q;
        const K *A = src + g.a_lo;
        const K *B = src + g.b_lo;
        while (l < r) {
            const long long mid = (l + r) >> 1;
            if (A[mid] <= B[diag - 1 - mid]) l = mid + 1;
            else r = mid;
        }
    }
    HS_DASSERT(l >= 0 && l <= na && diag - l >= 0 && diag - l <= nb);
    corank[beta] = (int)(g.a_lo + l);
}

// samp[m] = src[m Q + Q - 1]: the coarse index of caller-given runs (hs_merge).
template <typename K>
__global__ void k_sample(const K *__restrict__ src, K *samp, long long n) {
    const long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long p = m * kSampleQ + kSampleQ - 1;
    if (p < n) st_keep(samp + m, src[p]);
}

// =================================================================== K6b
template <typename K>
struct Piece {
    long long x;  // first output position
    K *dst;
    int len, na, nb;  // len < 0: no more pieces
    int offA, offB;   // element offsets of the A / B slices inside the stage
};

template <typename K, int NC, int VT, int ST>
struct MergeSmem {
    static constexpr int TM = NC * VT;
    static constexpr int E = 16 / sizeof(K);
    // A superset (<= na + 2E) | pad to 16 B | B superset (<= nb + 2E)
    // (+VT: exhausted-run indices may run up to VT past a slice; reads are masked)
    static constexpr int SLOT = (TM + 6 * E + VT + E - 1) / E * E;
    static constexpr int OUT = TM + E;
    static constexpr size_t bytes() { return (size_t)(ST * SLOT + 2 * OUT) * sizeof(K); }
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void consumer_bar(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Merge-path split of output diag between A[0..na) and B[0..nb) (stable-left).
template <typename K>
__device__ __forceinline__ int merge_path(const K *A, int na, const K *B, int nb, int diag) {
    int l = diag - nb > 0 ? diag - nb : 0;
    int r = diag < na ? diag : na;
    while (l < r) {
        const int mid = (l + r) >> 1;
        if (A[mid] <= B[diag - 1 - mid]) l = mid + 1;
        else r = mid;
    }
    return l;
}

// Warp-specialised: warps 0..NC/32-1 merge, the last warp produces.
//   producer: piece geometry -> stage ring (ST slots, full/empty mbarriers),
//             A and B slices fetched by 1-D bulk async copies.
//   consumers: merge-path split + branch-free serial merge of VT outputs per
//             thread, staging (double-buffered) at the destination's 16-byte
//             phase, one bulk async store of the aligned middle per piece.
template <typename K, int NC, int VT, int ST>
__global__ void __launch_bounds__(NC + 32) k_merge_level(const Plan *__restrict__ plan_g, K *F, K *S, const K *src0,
                                                         const int *__restrict__ corank, K *samp_out, int level,
                                                         int n, int nblocks) {
    using SM = MergeSmem<K, NC, VT, ST>;
    constexpr int TM = SM::TM, E = SM::E, SLOT = SM::SLOT, OUT = SM::OUT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const stage0 = reinterpret_cast<K *>(smem_raw);
    K *const out0 = stage0 + ST * SLOT;
    __shared__ __align__(8) uint64_t full[ST];
    __shared__ __align__(8) uint64_t empty[ST];
    __shared__ Plan P;
    __shared__ Piece<K> pc[ST];
    const int tid = threadIdx.x;
    const K kMax = KeyTraits<K>::kMax;

    griddep_wait();
    if (level >= __ldg(&plan_g->Lmax)) return;  // whole CTA: nothing at this level
    load_plan_m(P, plan_g);
    if (tid == 0) {
        for (int i = 0; i < ST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NC / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (level >= P.Lmax) return;  // no bucket runs this level (the host only knows a bound)

    if (tid >= NC) {
        // ------------------------------------------------------ producer
        if (tid != NC) return;
        int blk = blockIdx.x;
        long long px = (long long)blk * TM;
        for (int it = 0;; ++it) {
            const int slot = it % ST;
            mbar_wait(&empty[slot], ((it / ST) & 1) ^ 1);
            Piece<K> q;
            q.len = -1;
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
                // px is either a pair start or the block start P0 (co-rank from K6a)
                const long long ax = (px == g.a_lo) ? g.a_lo : (long long)corank[blk];
                const long long ae = (e == g.b_hi) ? g.b_lo : (long long)corank[blk + 1];
                const long long bx = g.b_lo + (px - ax);
                const long long be = g.b_lo + (e - ae);
                const K *src = (level == 0 && src0) ? src0 : level_src(P, b, level, F, S);
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
                const int bstart = (int)(bytesA / sizeof(K));  // multiple of E
                q.offB = bstart + (int)(((uintptr_t)(src + bx) - gb0) / sizeof(K));
                K *st = stage0 + slot * SLOT;
                pc[slot] = q;
                mbar_arrive_expect_tx(&full[slot], bytesA + bytesB);
                if (bytesA) bulk_g2s(st, (const void *)ga0, bytesA, &full[slot]);
                if (bytesB) bulk_g2s(st + bstart, (const void *)gb0, bytesB, &full[slot]);
                px = e;
                break;
            }
            if (q.len < 0) {
                pc[slot] = q;
                mbar_arrive_expect_tx(&full[slot], 0);
                return;
            }
        }
    }

    // ---------------------------------------------------------- consumers
    const int lane = tid & 31;
    for (int it = 0;; ++it) {
        const int slot = it % ST;
        mbar_wait(&full[slot], (it / ST) & 1);
        const Piece<K> q = pc[slot];
        if (q.len < 0) break;
        HS_DASSERT(q.na >= 0 && q.nb >= 0 && q.na + q.nb == q.len && q.len <= TM);
        // (an empty A slice has no bytes in the stage; its offA is only the phase)
        HS_DASSERT(q.offA >= 0 && q.offA + q.na <= SLOT && (q.na == 0 || q.offB >= q.offA + q.na) &&
                   q.offB >= 0 && q.offB + q.nb <= SLOT);
        const K *sb = stage0 + slot * SLOT;
        const K *A = sb + q.offA;
        const K *B = sb + q.offB;
        const int na = q.na, nb = q.nb;
        // staging position p holds output p - sh; sh = destination's 16-byte phase
        const int sh = (int)(((uintptr_t)(q.dst + q.x) & 15) / sizeof(K));
        const int p_lo = tid * VT > sh ? tid * VT : sh;
        const int diag = p_lo - sh;
        K v[VT];
        if (diag < q.len) {
            const int a0 = merge_path(A, na, B, nb, diag);
            // indices into the stage; an exhausted run reads as kMax (an
            // exhausted A only "wins" a tie against a real kMax in B, and then
            // emits the same value), so the loop needs no bounds branches
            const int a_end = q.offA + na, b_end = q.offB + nb;
            int ai = q.offA + a0, bi = q.offB + diag - a0;
            K x = ai < a_end ? sb[ai] : kMax;
            K y = bi < b_end ? sb[bi] : kMax;
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                // items (ExactEnds): an exhausted run must never win a tie
                const bool p = ExactEnds<K>::value ? (bi >= b_end || (ai < a_end && x <= y)) : x <= y;
                v[k] = p ? x : y;
                if (k + 1 < VT) {
                    const int nx = (p ? ai : bi) + 1;
                    const int lim = p ? a_end : b_end;
                    HS_DASSERT(nx >= 0 && nx < SLOT);
                    const K t = sb[nx];
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
            const int dx = NC * VT - sh;
            int ai = merge_path(A, na, B, nb, dx), bi = dx - ai;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const K x = ai < na ? A[ai] : kMax;
                const K y = bi < nb ? B[bi] : kMax;
                const bool p = (bi >= nb) || (ai < na && x <= y);
                vx[k] = p ? x : y;
                ai += p ? 1 : 0;
                bi += p ? 0 : 1;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the stage

        K *sOut = out0 + (it & 1) * OUT;
        if (tid == 0) bulk_wait_read1();  // the store two pieces ago has read sOut
        consumer_bar(NC);
        const int end = sh + q.len;
        if (diag < q.len) {
            if (VT % E == 0 && tid * VT >= sh && (tid + 1) * VT <= end) {
#pragma unroll
                for (int k = 0; k < (VT % E == 0 ? VT : 0); k += E) {
                    int4 w;
                    memcpy(&w, &v[k], 16);
                    *reinterpret_cast<int4 *>(sOut + tid * VT + k) = w;
                }
            } else if (tid * VT >= sh && (tid + 1) * VT <= end) {
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
        K *const g = q.dst + q.x - sh;   // staging position p <-> g[p]
        if (m1 > m0) {
            if (tid == 0) bulk_s2g(g + m0, sOut + m0, (uint32_t)((m1 - m0) * sizeof(K)));
            if (tid < E) {
                const int p = sh + tid;  // head
                if (p < m0 && p < end) g[p] = sOut[p];
            } else if (tid < 2 * E) {
                const int p = m1 + tid - E;  // tail
                if (p < end) g[p] = sOut[p];
            }
        } else {
            for (int p = sh + tid; p < end; p += NC) g[p] = sOut[p];
        }
        if (tid == 0) bulk_commit();  // one group per piece (possibly empty)
        write_samples(samp_out, q.x, q.len, sOut + sh, tid, NC);  // coarse index for the next level
    }
    if (tid == 0) bulk_wait0();
}

// ============================================================ level gate
// CUDA-graph capture of hs_sort: the merge levels the host launches past the
// log2 c tree levels every plan runs (k[b] + log2 c >= log2 c) sit in the body
// of a conditional (IF) graph node; this one-thread kernel opens it only when
// the device plan has a bucket with more levels (a fallback bucket), so a
// replay of a C3 sort skips all the empty level launches.
__global__ void k_level_gate(cudaGraphConditionalHandle h, const Plan *__restrict__ plan, int lv) {
    griddep_wait();
    if (threadIdx.x == 0) cudaGraphSetConditional(h, plan->Lmax > lv ? 1u : 0u);
}

cudaError_t launch_level_gate(unsigned long long handle, const Plan *plan, int lv, cudaStream_t st) {
    return launch_pdl(k_level_gate, dim3(1), dim3(32), 0, st, (cudaGraphConditionalHandle)handle, plan, lv);
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

int g_merge_per_sm[kMaxDevices][3];  // resident K6b CTAs per SM, per device: [int32, int64, KV64]

template <typename K>
constexpr int kslot() {
    return sizeof(K) == 4 ? 0 : sizeof(K) == 8 ? 1 : 2;
}

template <typename K>
cudaError_t setup_merge_t(int dev) {
    using G = MGeo<K>;
    using SM = MergeSmem<K, G::kNT, G::kVT, G::kST>;
    auto kern = k_merge_level<K, G::kNT, G::kVT, G::kST>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::bytes());
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::kNT + 32, SM::bytes());
    g_merge_per_sm[dev][kslot<K>()] = occ > 0 ? occ : 1;
    return e;
}

cudaError_t setup_merge_kernels(int dev) {
    cudaError_t e = setup_merge_t<int32_t>(dev);
    if (e == cudaSuccess) e = setup_merge_t<int64_t>(dev);
    return e != cudaSuccess ? e : setup_merge_t<KV64>(dev);
}

template <typename K>
cudaError_t launch_merge_level_t(const Plan *plan, void *F, void *S, const void *src0, int *corank,
                                 const void *samp_in, void *samp_out, int level, int n, int num_sms,
                                 cudaStream_t st) {
    using G = MGeo<K>;
    using SM = MergeSmem<K, G::kNT, G::kVT, G::kST>;
    constexpr int TM = SM::TM;
    auto kern = k_merge_level<K, G::kNT, G::kVT, G::kST>;
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    const int per_sm = g_merge_per_sm[dev][kslot<K>()];
    const int nblocks = (int)(((long long)n + TM - 1) / TM);
    if (nblocks == 0) return cudaSuccess;
    const int nbounds = nblocks + 1;
    // both kernels of a level are launched with programmatic stream serialization:
    // each may be scheduled while its predecessor drains (an empty level past the
    // device plan then costs little more than its launch) and waits in griddep_wait
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    prof_begin(kProfMergePartition, st);
    cfg.gridDim = dim3((unsigned)((nbounds + 127) / 128));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_merge_partition<K>, plan, (K *)F, (K *)S, (const K *)src0,
                                       (const K *)samp_in, corank, level, n, TM, nbounds);
    prof_end(kProfMergePartition, st);
    if (e != cudaSuccess) return e;
    note_launch();
    long long grid = (long long)per_sm * num_sms;
    if (grid > nblocks) grid = nblocks;
    prof_begin(kProfMergeLevel, st);
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(G::kNT + 32);
    cfg.dynamicSmemBytes = SM::bytes();
    e = cudaLaunchKernelEx(&cfg, kern, plan, (K *)F, (K *)S, (const K *)src0, (const int *)corank, (K *)samp_out,
                           level, n, nblocks);
    prof_end(kProfMergeLevel, st);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_sample_t(const void *src, void *samp, long long n, cudaStream_t st) {
    const long long m = n / kSampleQ;
    if (m <= 0) return cudaSuccess;
    prof_begin(kProfMergePartition, st);
    k_sample<K><<<(unsigned)((m + 255) / 256), 256, 0, st>>>((const K *)src, (K *)samp, n);
    prof_end(kProfMergePartition, st);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
    return e;
}

template <typename K>
cudaError_t launch_copy_t(const void *src, void *dst, long long n, int num_sms, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long want = (n + 255) / 256;
    int grid = (int)(want > 8LL * num_sms ? 8LL * num_sms : want);
    prof_begin(kProfCopy, st);
    k_copy<K><<<grid, 256, 0, st>>>((const K *)src, (K *)dst, n);
    prof_end(kProfCopy, st);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
    return e;
}

int merge_span(int dt) {
    return dt == 0 ? merge_span_t<int32_t>() : dt == 1 ? merge_span_t<int64_t>() : merge_span_t<KV64>();
}

cudaError_t launch_merge_level(int dt, const Plan *plan, void *F, void *S, const void *src0, int *corank,
                               const void *samp_in, void *samp_out, int level, int n, int num_sms, cudaStream_t st) {
    if (dt == 2)
        return launch_merge_level_t<KV64>(plan, F, S, src0, corank, samp_in, samp_out, level, n, num_sms, st);
    return dt == 0 ? launch_merge_level_t<int32_t>(plan, F, S, src0, corank, samp_in, samp_out, level, n, num_sms, st)
                   : launch_merge_level_t<int64_t>(plan, F, S, src0, corank, samp_in, samp_out, level, n, num_sms, st);
}

cudaError_t launch_sample(int dt, const void *src, void *samp, long long n, int num_sms, cudaStream_t st) {
    (void)num_sms;
    if (dt == 2) return launch_sample_t<KV64>(src, samp, n, st);
    return dt == 0 ? launch_sample_t<int32_t>(src, samp, n, st) : launch_sample_t<int64_t>(src, samp, n, st);
}

cudaError_t launch_copy(int dt, const void *src, void *dst, long long n, int num_sms, cudaStream_t st) {
    if (dt == 2) return launch_copy_t<KV64>(src, dst, n, num_sms, st);
    return dt == 0 ? launch_copy_t<int32_t>(src, dst, n, num_sms, st) : launch_copy_t<int64_t>(src, dst, n, num_sms, st);
}

}  // namespace hs
