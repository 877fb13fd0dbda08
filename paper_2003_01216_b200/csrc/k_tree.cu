// k_tree.cu -- a6, the paper's binary-tree merge of a bucket's c sorted chunks
// (§3.2: "threads sort and merge two children sorted lists ... in a
// binary tree fashion"), run on chip in ONE HBM pass for the buckets whose
// chunks K5a split into equal-width sub-ranges (plan.tree).
//
// Why it is exact: in such a bucket sub-range t of every chunk holds the keys
// of one and the same key interval, and inside it the tile sort of every
// piece (chunk j, sub-range t) recorded e_j[u] = #keys in fine bins <= u of a
// common monotone map of that interval (k_tilesort.cu, tree_bin).  So a cut at
// a fine-bin boundary u is an exact co-rank in all c chunks at once: the keys
// of bins [u0, u1) of the c pieces are exactly the keys the paper's tree
// merge of the whole bucket puts at output positions
//   off[b] + sum_j start_j(t) + sum_j E_j(u0) ... + sum_j E_j(u1),
// E_j(u) = #keys in bins < u, start_j(t) = sub-range t's start in chunk j.
// Merging the c slices of such a segment in log2 c binary rounds (run pairs
// i, i + 2^(r-1), stable-left) is the tree merge restricted to it.
//
//   k_tree_plan   one CTA per sub-range: G[u] = sum_j e_j[u]; cut after bin u
//                 whenever floor(G / TGT) steps (and after the last bin) ->
//                 segments of about TGT keys; a segment over CAP keys (one fine
//                 bin with over CAP - TGT keys: heavy duplicates) marks its bucket
//                 in ctl->treebad, and that bucket runs its merge levels instead
//   k_tree_merge  persistent, warp-specialised: a producer warp computes the c
//                 slices of a segment (lane j <-> chunk j) and fetches them with
//                 1-D bulk async copies into a 2-slot ring; consumer warps run
//                 the log2 c rounds in shared memory (merge path + serial merge,
//                 stable-left) and write the segment with one bulk async store
//
// HBM traffic: read + write of the bucket once (2 n s), instead of 2 n s per
// tree level; the fine-bin tables add 2 KB per piece.
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

namespace hs {

template <typename K>
struct TreeGeo;
template <>
struct TreeGeo<int32_t> {
    static constexpr int NC = 256, VT = 17;  // CAP = 4352 keys per segment (VT odd: see V below)
};
template <>
struct TreeGeo<int64_t> {
    static constexpr int NC = 256, VT = 9;   // CAP = 2304 keys per segment
};
constexpr int kTreeMaxC = 1 << kTreeMaxLog2C;
constexpr int kTreeST = 3;  // stage slots

template <typename K>
struct TreeSmem {
    static constexpr int NC = TreeGeo<K>::NC, VT = TreeGeo<K>::VT;
    static constexpr int CAP = NC * VT;
    static constexpr int TGT = CAP * 3 / 4;  // segment target: room for one fine bin of CAP / 4 keys
    static constexpr int E = 16 / sizeof(K);
    // every run in shared memory is followed by GAP kMax sentinels, so a thread's VT merge steps
    // never need a bounds test (an exhausted run keeps reading kMax)
    static constexpr int GAP = (VT + E - 1) / E * E;
    // a slot holds the c slices' 16-byte aligned supersets (each <= len + 2E - 2 keys, rounded to E)
    // + their gaps, later the even rounds' output; Y the odd rounds' (+ the destination's 16-byte phase)
    static constexpr int SLOT = CAP + (2 * E + GAP) * kTreeMaxC;
    static constexpr int BUF = CAP + GAP * kTreeMaxC / 2 + 2 * E;
    static constexpr size_t bytes() { return (size_t)(kTreeST * SLOT + BUF) * sizeof(K); }
};

struct TreeSeg {
    int s;    // sub-range id: tree buckets in order, sub-ranges in order
    int u01;  // fine bins [u0, u1): u0 | u1 << 16
};

// Sub-range id s -> (bucket, sub-range) over the tree buckets of the plan.
__device__ __forceinline__ bool tree_subrange(const Plan &P, long long s, int &b, int &t) {
    for (b = 0; b < 10; ++b) {
        if (!P.tree[b]) continue;
        if (s < P.nsb[b]) {
            t = (int)s;
            return true;
        }
        s -= P.nsb[b];
    }
    return false;
}

__device__ __forceinline__ long long tree_subranges(const Plan &P) {
    long long s = 0;
    for (int b = 0; b < 10; ++b) s += P.tree[b] ? P.nsb[b] : 0;
    return s;
}

// ================================================================ plan
template <int NT>
__global__ void __launch_bounds__(NT) k_tree_plan(Ctl *ctl, const uint16_t *__restrict__ etab, TreeSeg *seg,
                                                  long long seg_cap, int tgt, int cap) {
    griddep_wait();  // PDL: the tile sort's fine-bin tables are complete
    constexpr int UPT = kTreeFine / NT;
    static_assert(UPT == 4, "one 8-byte load of four u16 bins per thread and chunk");
    __shared__ Plan P;
    __shared__ uint32_t wsum[NT / 32];
    __shared__ int cut_u[kTreeFine];
    __shared__ uint32_t cut_g[kTreeFine];
    __shared__ unsigned s_base;
    {
        constexpr int W = sizeof(Plan) / 4;
        const uint32_t *src = reinterpret_cast<const uint32_t *>(&ctl->plan);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&P);
        for (int i = threadIdx.x; i < W; i += NT) dst[i] = src[i];
    }
    __syncthreads();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long nsub = tree_subranges(P);
    const int c = 1 << P.log2c;
    for (long long s = blockIdx.x; s < nsub; s += gridDim.x) {
        int b, t;
        tree_subrange(P, s, b, t);
        const int ns = P.nsb[b];
        // G[u] = sum over the chunks of e_j[u] (cumulative: so is G)
        uint32_t G[UPT] = {0, 0, 0, 0};
        for (int j = 0; j < c; ++j) {
            const uint16_t *e = etab + (size_t)(P.tile_prefix[b] + (long long)j * ns + t) * kTreeFine;
            const uint2 w = *reinterpret_cast<const uint2 *>(e + tid * UPT);
            G[0] += w.x & 0xFFFFu;
            G[1] += w.x >> 16;
            G[2] += w.y & 0xFFFFu;
            G[3] += w.y >> 16;
        }
        uint32_t gprev = __shfl_up_sync(0xffffffffu, G[UPT - 1], 1);  // G[tid * UPT - 1]
        if (lane == 0) gprev = 0;
        __syncthreads();  // (previous sub-range's cut arrays are consumed)
        if (lane == 31) wsum[warp] = G[UPT - 1];
        __syncthreads();
        if (lane == 0 && warp > 0) gprev = wsum[warp - 1];
        // cut after bin u when floor(G / tgt) steps, and after the last bin
        int ncut = 0;
        bool cut[UPT];
#pragma unroll
        for (int q = 0; q < UPT; ++q) {
            const uint32_t before = q ? G[q - 1] : gprev;
            cut[q] = (G[q] / (uint32_t)tgt != before / (uint32_t)tgt) || (tid * UPT + q == kTreeFine - 1);
            ncut += cut[q];
        }
        // exclusive scan of the cut counts -> each cut's index
        int incl = ncut;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        __syncthreads();
        if (lane == 31) wsum[warp] = (uint32_t)incl;
        __syncthreads();
        int base = incl - ncut;
        for (int w = 0; w < warp; ++w) base += (int)wsum[w];
        int total = 0;
        for (int w = 0; w < NT / 32; ++w) total += (int)wsum[w];
#pragma unroll
        for (int q = 0; q < UPT; ++q)
            if (cut[q]) {
                cut_u[base] = tid * UPT + q;
                cut_g[base] = G[q];
                ++base;
            }
        if (tid == 0) s_base = atomicAdd(&ctl->nseg, (unsigned)total);
        __syncthreads();
        const long long sb = s_base;
        bool over = sb + total > seg_cap;  // (cannot happen with tree_seg_capacity's bound; guarded anyway)
        for (int k = tid; k < total; k += NT) {
            const int u0 = k ? cut_u[k - 1] + 1 : 0, u1 = cut_u[k] + 1;
            const uint32_t size = cut_g[k] - (k ? cut_g[k - 1] : 0u);
            if (size > (uint32_t)cap) over = true;
            TreeSeg q;
            q.s = (int)s;
            q.u01 = u0 | (u1 << 16);
            if (sb + k < seg_cap) seg[sb + k] = q;  // every record below the capacity is written
        }
        if (__syncthreads_or(over) && tid == 0) atomicOr(&ctl->treebad, 1u << b);
    }
}

// ================================================================ merge
template <typename K>
struct TreePiece {
    long long out;  // first output position (absolute)
    int M;          // keys in the segment (< 0: no more segments)
    int off[kTreeMaxC];  // slice j starts at stage + off[j]
    int len[kTreeMaxC];
};

__device__ __forceinline__ void tree_bar(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }
__device__ __forceinline__ void tree_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename K>
__device__ __forceinline__ K tlds(uint32_t a);
template <>
__device__ __forceinline__ int32_t tlds<int32_t>(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
template <>
__device__ __forceinline__ int64_t tlds<int64_t>(uint32_t a) {
    int64_t v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
template <typename K>
__device__ __forceinline__ void tsts(uint32_t a, K v);
template <>
__device__ __forceinline__ void tsts<int32_t>(uint32_t a, int32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
template <>
__device__ __forceinline__ void tsts<int64_t>(uint32_t a, int64_t v) {
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

// Merge-path split of output diag between A[0..na) and B[0..nb) at shared
// addresses ua / ub (stable-left: ties take A).
template <typename K>
__device__ __forceinline__ int tree_path(uint32_t ua, int na, uint32_t ub, int nb, int diag) {
    constexpr int W = sizeof(K);
    int l = diag - nb > 0 ? diag - nb : 0;
    int r = diag < na ? diag : na;
    while (l < r) {
        const int mid = (l + r) >> 1;
        const bool pr = tlds<K>(ua + mid * W) <= tlds<K>(ub + (diag - 1 - mid) * W);
        l = pr ? mid + 1 : l;
        r = pr ? r : mid;
    }
    return l;
}

// Outputs [p, pe) of one round.  Pair q (runs at shared addresses rA[q] /
// rB[q], lengths rl[2q], rl[2q+1], each followed by >= VT kMax sentinels)
// is merged from the merge-path split of p (stable-left); its output run
// starts at shared address uo + (Oq + q gap) s.  Every thread runs VT merge
// steps and stores the first cnt: no bounds tests (an exhausted run reads
// kMax -- an exhausted A then only wins ties against a real kMax in B, with
// the same value -- and at most VT steps past a run end stay in its gap).
template <typename K, int VT>
__device__ __forceinline__ void tree_round_outputs(int p, int pe, const int *rl, int npairs, const uint32_t *rA,
                                                   const uint32_t *rB, uint32_t uo, int gap) {
    constexpr int W = sizeof(K);
    if (p >= pe) return;
    int q = 0, Oq = 0;
    int na = rl[0], nb = rl[1];
    while (Oq + na + nb <= p && q + 1 < npairs) {
        Oq += na + nb;
        ++q;
        na = rl[2 * q];
        nb = rl[2 * q + 1];
    }
    for (;;) {
        const uint32_t ua = rA[q], ub = rB[q];
        const int diag = p - Oq;
        const int a0 = tree_path<K>(ua, na, ub, nb, diag);
        uint32_t pa = ua + a0 * W, pb = ub + (diag - a0) * W;
        K x = tlds<K>(pa), y = tlds<K>(pb);
        const int kend = min(pe, Oq + na + nb), cnt = kend - p;
        const uint32_t o = uo + (p + q * gap) * W;
#pragma unroll
        for (int k = 0; k < VT; ++k) {
            const bool tA = x <= y;
            if (k < cnt) tsts<K>(o + k * W, tA ? x : y);
            if (k + 1 < VT) {
                pa += tA ? W : 0;
                pb += tA ? 0 : W;
                const K t = tlds<K>(tA ? pa : pb);
                x = tA ? t : x;
                y = tA ? y : t;
            }
        }
        p = kend;
        if (p >= pe) return;
        Oq += na + nb;  // my outputs continue in the next pair
        ++q;
        na = rl[2 * q];
        nb = rl[2 * q + 1];
    }
}

// Mbarrier phase wait with a suspend-time hint: a waiting thread sleeps in
// hardware until the phase completes instead of re-issuing the try_wait.
__device__ __forceinline__ void tree_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra TW_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// Persistent, warp-specialised; CTA blk owns the contiguous segment range
// [blk * per, (blk + 1) * per) (consecutive segments of a sub-range share
// their tables' cache lines).
//   producer warp: geometry of the next segment (lane j <-> chunk j: split
//     table, fine-bin prefixes) is loaded BEFORE waiting for a free stage
//     slot, then the c slices are fetched by 1-D bulk async copies (16-byte
//     aligned supersets) into the slot (ST slots, full/empty mbarriers);
//   consumer warps: log2 c rounds -- round r merges run pairs (2q, 2q+1) into
//     run q; odd rounds write Y, even rounds write the stage slot itself
//     (its slices are consumed by round 0), so the last round (odd count)
//     lands in Y at the destination's 16-byte phase; the slot is released
//     after the last round, Y leaves with one bulk async store.
template <typename K>
__global__ void __launch_bounds__(TreeGeo<K>::NC + 32, 2) k_tree_merge(const Ctl *__restrict__ ctl,
                                                                  const uint32_t *__restrict__ sbtab,
                                                                  const uint16_t *__restrict__ etab,
                                                                  const TreeSeg *__restrict__ seg, long long seg_cap,
                                                                  const K *S, K *F) {
    using G = TreeSmem<K>;
    constexpr int NC = G::NC, VT = G::VT, E = G::E, SLOT = G::SLOT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const stage0 = reinterpret_cast<K *>(smem_raw);
    K *const Y = stage0 + kTreeST * SLOT;
    __shared__ __align__(8) uint64_t full[kTreeST];
    __shared__ __align__(8) uint64_t empty[kTreeST];
    __shared__ Plan P;
    __shared__ TreePiece<K> pc[kTreeST];
    __shared__ int rlb[2][kTreeMaxC];       // run lengths of the current / next round
    __shared__ uint32_t rA[kTreeMaxC / 2];  // run pair q of the current round: shared addresses of A and B
    __shared__ uint32_t rB[kTreeMaxC / 2];
    const int tid = threadIdx.x;

    griddep_wait();  // PDL: the tree plan (and the tile sort before it) is complete
    const long long nseg = min((long long)ctl->nseg, seg_cap);
    const long long per = (nseg + gridDim.x - 1) / gridDim.x;
    const long long i0 = (long long)blockIdx.x * per, i1 = min(i0 + per, nseg);
    if (i0 >= i1) return;
    {
        constexpr int W = sizeof(Plan) / 4;
        const uint32_t *src = reinterpret_cast<const uint32_t *>(&ctl->plan);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&P);
        for (int i = tid; i < W; i += blockDim.x) dst[i] = src[i];
    }
    if (tid == 0) {
        for (int i = 0; i < kTreeST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NC / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned tbad = ctl->treebad;
    const int c = 1 << P.log2c;

    if (tid >= NC) {
        // ------------------------------------------------------------ producer warp
        const int lane = tid & 31;
        int it = 0;
        for (long long i = i0;; ++i) {
            int b = 0, t = 0;
            TreeSeg q;
            bool have = false;
            for (; i < i1; ++i) {  // next segment of a bucket that takes the on-chip tree
                q = seg[i];
                tree_subrange(P, q.s, b, t);
                if (!((tbad >> b) & 1u)) {
                    have = true;
                    break;
                }
            }
            int len = 0, outpart = 0;
            const K *src = S;
            if (have && lane < c) {  // lane j: chunk j's slice of the segment
                const int ns = P.nsb[b];
                const int u0 = q.u01 & 0xFFFF, u1 = q.u01 >> 16;
                const long long m = P.off[b + 1] - P.off[b];
                const uint32_t st = __ldg(sbtab + P.sboff[b] + (long long)lane * (ns + 1) + t);
                const uint16_t *e = etab + (size_t)(P.tile_prefix[b] + (long long)lane * ns + t) * kTreeFine;
                const int e0 = u0 ? (int)__ldg(e + u0 - 1) : 0;
                const int e1 = (int)__ldg(e + u1 - 1);
                len = e1 - e0;
                outpart = (int)st + e0;
                src = S + P.off[b] + part_start(m, P.log2c, lane) + st + e0;
            }
            const int slot = it % kTreeST;
            tree_wait(&empty[slot], ((it / kTreeST) & 1) ^ 1);
            if (!have) {
                if (lane == 0) {
                    pc[slot].M = -1;
                    mbar_arrive_expect_tx(&full[slot], 0);
                }
                return;
            }
            const uintptr_t ga0 = (uintptr_t)src & ~(uintptr_t)15;
            const uintptr_t ga1 = ((uintptr_t)(src + len) + 15) & ~(uintptr_t)15;
            const int words = len > 0 ? (int)((ga1 - ga0) / sizeof(K)) : 0;  // multiple of E
            int incl = lane < c ? words + G::GAP : 0;  // each slice region + its sentinel gap
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int region = incl - (lane < c ? words + G::GAP : 0);
            int M = len, outsum = outpart;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                M += __shfl_xor_sync(0xffffffffu, M, o);
                outsum += __shfl_xor_sync(0xffffffffu, outsum, o);
            }
            const int total_words = __shfl_sync(0xffffffffu, incl, 31);  // (incl. gaps: not transferred)
            TreePiece<K> &d = pc[slot];
            if (lane < c) {
                d.off[lane] = region + (int)(((uintptr_t)src - ga0) / sizeof(K));
                d.len[lane] = len;
            }
            if (lane == 0) {
                d.M = M;
                d.out = P.off[b] + outsum;
            }
            int tx = words;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
            HS_DASSERT(M <= G::CAP && total_words <= SLOT);
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(&full[slot], (uint32_t)tx * sizeof(K));
            __syncwarp();
            if (words > 0) bulk_g2s(stage0 + slot * SLOT + region, (const void *)ga0, (uint32_t)words * sizeof(K),
                                    &full[slot]);
            ++it;
        }
    }

    // ---------------------------------------------------------------- consumers
    const K kMax = KeyTraits<K>::kMax;
    constexpr int GAP = G::GAP;
    for (int it = 0;; ++it) {
        const int slot = it % kTreeST;
        tree_wait(&full[slot], (it / kTreeST) & 1);
        const TreePiece<K> &d = pc[slot];
        const int M = d.M;
        if (M < 0) break;
        K *const sb = stage0 + slot * SLOT;
        K *const out = F + d.out;
        const int sh = (int)(((uintptr_t)out & 15) / sizeof(K));
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // Y free again
        int *rl = rlb[0];
        if (tid < c) rl[tid] = d.len[tid];
        const uint32_t usb = smem_u32(sb), uY = smem_u32(Y);
        if (tid < c / 2) {
            rA[tid] = usb + d.off[2 * tid] * (uint32_t)sizeof(K);
            rB[tid] = usb + d.off[2 * tid + 1] * (uint32_t)sizeof(K);
        }
        for (int k = tid; k < c * GAP; k += NC) sb[d.off[k / GAP] + d.len[k / GAP] + k % GAP] = kMax;  // sentinels
        tree_bar(NC);
        // outputs per thread this segment: balanced rounds; odd, so a warp's output runs (stride V) hit
        // 32 distinct banks (V <= VT since M <= NC VT and VT is odd)
        const int V = ((M + NC - 1) / NC) | 1;
        int nruns = c;
        for (int r = 0; (1 << r) < c; ++r) {
            const bool last = (2 << r) >= c;
            K *const ob = (r & 1) ? sb : Y + (last ? sh : 0);
            const uint32_t uo = smem_u32(ob);
            tree_round_outputs<K, VT>(tid * V, min(tid * V + V, M), rl, nruns / 2, rA, rB, uo, GAP);
            tree_bar(NC);  // round complete
            if (!last) {
                // the next round's runs: merged pair q at (its output prefix + q GAP), GAP sentinels after it
                for (int k = tid; k < (nruns / 2) * GAP; k += NC) {
                    const int q = k / GAP;
                    int pre = 0;
                    for (int j = 0; j <= 2 * q + 1; ++j) pre += rl[j];
                    ob[pre + q * GAP + k % GAP] = kMax;
                }
                int *const rn = rlb[(r + 1) & 1];  // (rl is still read by the sentinel writers)
                if (tid == 0) {
                    int pre = 0;
                    for (int k = 0; k < nruns / 4; ++k) {
                        const int la = rl[4 * k] + rl[4 * k + 1], lb = rl[4 * k + 2] + rl[4 * k + 3];
                        rA[k] = uo + (pre + 2 * k * GAP) * (uint32_t)sizeof(K);
                        rB[k] = uo + (pre + la + (2 * k + 1) * GAP) * (uint32_t)sizeof(K);
                        pre += la + lb;
                        rn[2 * k] = la;
                        rn[2 * k + 1] = lb;
                    }
                }
                rl = rn;
            }
            nruns >>= 1;
            tree_bar(NC);
        }
        if ((tid & 31) == 0) tree_arrive(&empty[slot]);  // the slot (inputs and even rounds) is free
        // the sorted segment sits at Y[sh .. sh + M): bulk store the aligned middle
        fence_proxy_async_smem();
        tree_bar(NC);
        const int end = sh + M;
        const int m0 = sh == 0 ? 0 : E;
        const int m1 = end / E * E;
        K *const g = out - sh;
        if (m1 > m0) {
            if (tid == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g + m0),
                             "r"(smem_u32(Y + m0)), "r"((uint32_t)((m1 - m0) * sizeof(K)))
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (tid < E) {
                const int pp = sh + tid;
                if (pp < m0 && pp < end) g[pp] = Y[pp];
            } else if (tid < 2 * E) {
                const int pp = m1 + tid - E;
                if (pp < end) g[pp] = Y[pp];
            }
        } else {
            for (int pp = sh + tid; pp < end; pp += NC) g[pp] = Y[pp];
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ================================================================ launchers
int g_tree_per_sm[kMaxDevices][2];
int g_tree_sms[kMaxDevices];

template <typename K>
cudaError_t setup_tree_t(int dev) {
    using G = TreeSmem<K>;
    auto kern = k_tree_merge<K>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::bytes());
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::NC + 32, G::bytes());
    g_tree_per_sm[dev][sizeof(K) == 8 ? 1 : 0] = occ > 0 ? occ : 1;
    return e;
}

cudaError_t setup_tree_kernels(int dev) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    g_tree_sms[dev] = sms > 0 ? sms : 148;
    if ((e = setup_tree_t<int32_t>(dev)) != cudaSuccess) return e;
    return setup_tree_t<int64_t>(dev);
}

long long tree_seg_capacity(int dt, long long n, long long split_words) {
    const int tgt = dt == 0 ? TreeSmem<int32_t>::TGT : TreeSmem<int64_t>::TGT;
    return n / tgt + split_words + 64;  // <= sum over sub-ranges of (G / TGT + 1)
}

size_t tree_etab_bytes(long long max_tiles) { return (size_t)max_tiles * kTreeFine * sizeof(uint16_t); }

template <typename K>
cudaError_t launch_tree_t(Ctl *ctl, const uint32_t *sbtab, const uint16_t *etab, void *seg, long long seg_cap,
                          const K *S, K *F, cudaStream_t st, bool plan_only) {
    using G = TreeSmem<K>;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const int sms = g_tree_sms[dev];
    prof_begin(kProfTreePlan, st);
    e = launch_pdl(k_tree_plan<256>, dim3((unsigned)(4 * sms)), dim3(256), 0, st, ctl, etab, (TreeSeg *)seg, seg_cap,
                   (int)G::TGT, (int)G::CAP);
    prof_end(kProfTreePlan, st);
    if (e != cudaSuccess || plan_only) return e;
    prof_begin(kProfTreeMerge, st);
    const int grid = g_tree_per_sm[dev][sizeof(K) == 8 ? 1 : 0] * sms;
    e = launch_pdl(k_tree_merge<K>, dim3((unsigned)grid), dim3(G::NC + 32), G::bytes(), st, (const Ctl *)ctl, sbtab,
                   etab, (const TreeSeg *)seg, seg_cap, S, F);
    prof_end(kProfTreeMerge, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_tree(int dt, Ctl *ctl, const uint32_t *sbtab, const uint16_t *etab, void *seg, long long seg_cap,
                        const void *S, void *F, cudaStream_t st, bool plan_only) {
    return dt == 0 ? launch_tree_t<int32_t>(ctl, sbtab, etab, seg, seg_cap, (const int32_t *)S, (int32_t *)F, st,
                                            plan_only)
                   : launch_tree_t<int64_t>(ctl, sbtab, etab, seg, seg_cap, (const int64_t *)S, (int64_t *)F, st,
                                            plan_only);
}

}  // namespace hs
