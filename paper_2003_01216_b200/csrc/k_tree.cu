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
    static constexpr int NC = 256, VT = 17;  // CAP = 4352 keys per segment
};
template <>
struct TreeGeo<int64_t> {
    static constexpr int NC = 256, VT = 9;   // CAP = 2304 keys per segment
};
constexpr int kTreeMaxC = 1 << kTreeMaxLog2C;
constexpr int kTreeST = 2;  // stage slots

template <typename K>
struct TreeSmem {
    static constexpr int NC = TreeGeo<K>::NC, VT = TreeGeo<K>::VT;
    static constexpr int CAP = NC * VT;
    static constexpr int TGT = CAP * 3 / 4;  // segment target: room for one fine bin of CAP / 4 keys
    static constexpr int E = 16 / sizeof(K);
    // a slot holds the c slices' 16-byte aligned supersets (each <= len + 2E - 2 keys, rounded to E)
    static constexpr int SLOT = CAP + 2 * E * kTreeMaxC;
    static constexpr int BUF = CAP + E;  // + the destination's 16-byte phase
    static constexpr size_t bytes() { return (size_t)(kTreeST * SLOT + 2 * BUF) * sizeof(K); }
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
    int c;
    int off[kTreeMaxC];  // slice j starts at stage + off[j]
    int len[kTreeMaxC];
};

__device__ __forceinline__ void tree_bar(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }
__device__ __forceinline__ void tree_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Merge-path split of output diag between A[0..na) and B[0..nb) (stable-left: ties take A).
template <typename K>
__device__ __forceinline__ int tree_path(const K *A, int na, const K *B, int nb, int diag) {
    int l = diag - nb > 0 ? diag - nb : 0;
    int r = diag < na ? diag : na;
    while (l < r) {
        const int mid = (l + r) >> 1;
        if (A[mid] <= B[diag - 1 - mid]) l = mid + 1;
        else r = mid;
    }
    return l;
}

template <typename K>
__global__ void __launch_bounds__(TreeGeo<K>::NC + 32) k_tree_merge(const Ctl *__restrict__ ctl,
                                                                  const uint32_t *__restrict__ sbtab,
                                                                  const uint16_t *__restrict__ etab,
                                                                  const TreeSeg *__restrict__ seg, long long seg_cap,
                                                                  const K *S, K *F) {
    using G = TreeSmem<K>;
    constexpr int NC = G::NC, VT = G::VT, E = G::E, SLOT = G::SLOT, BUF = G::BUF;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const stage0 = reinterpret_cast<K *>(smem_raw);
    K *const X = stage0 + kTreeST * SLOT;
    K *const Y = X + BUF;
    __shared__ __align__(8) uint64_t full[kTreeST];
    __shared__ __align__(8) uint64_t empty[kTreeST];
    __shared__ Plan P;
    __shared__ TreePiece<K> pc[kTreeST];
    __shared__ int rl[kTreeMaxC];  // run lengths of the current round
    const int tid = threadIdx.x;

    griddep_wait();  // PDL: the tree plan (and the tile sort before it) is complete
    const unsigned nseg = (unsigned)min((long long)ctl->nseg, seg_cap);
    if (blockIdx.x >= nseg) return;
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

    if (tid >= NC) {
        // ------------------------------------------------------------ producer warp
        const int lane = tid & 31;
        const int c = 1 << P.log2c;
        int it = 0;
        for (unsigned i = blockIdx.x;; i += gridDim.x) {
            int b = 0, t = 0;
            TreeSeg q;
            bool have = false;
            while (i < nseg) {  // next segment of a bucket that takes the on-chip tree
                q = seg[i];
                tree_subrange(P, q.s, b, t);
                if (!((tbad >> b) & 1u)) {
                    have = true;
                    break;
                }
                i += gridDim.x;
            }
            const int slot = it % kTreeST;
            mbar_wait(&empty[slot], ((it / kTreeST) & 1) ^ 1);
            if (!have) {
                if (lane == 0) {
                    pc[slot].M = -1;
                    mbar_arrive_expect_tx(&full[slot], 0);
                }
                return;
            }
            const int ns = P.nsb[b];
            const int u0 = q.u01 & 0xFFFF, u1 = q.u01 >> 16;
            const long long m = P.off[b + 1] - P.off[b];
            // lane j: chunk j's slice of the segment
            int len = 0, outpart = 0;
            const K *src = S;
            if (lane < c) {
                const uint32_t st = __ldg(sbtab + P.sboff[b] + (long long)lane * (ns + 1) + t);
                const uint16_t *e = etab + (size_t)(P.tile_prefix[b] + (long long)lane * ns + t) * kTreeFine;
                const int e0 = u0 ? (int)__ldg(e + u0 - 1) : 0;
                const int e1 = (int)__ldg(e + u1 - 1);
                len = e1 - e0;
                outpart = (int)st + e0;
                src = S + P.off[b] + part_start(m, P.log2c, lane) + st + e0;
            }
            const uintptr_t ga0 = (uintptr_t)src & ~(uintptr_t)15;
            const uintptr_t ga1 = ((uintptr_t)(src + len) + 15) & ~(uintptr_t)15;
            const int words = len > 0 ? (int)((ga1 - ga0) / sizeof(K)) : 0;  // multiple of E
            int incl = words;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int region = incl - words;
            int M = len, outsum = outpart;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                M += __shfl_xor_sync(0xffffffffu, M, o);
                outsum += __shfl_xor_sync(0xffffffffu, outsum, o);
            }
            const int total_words = __shfl_sync(0xffffffffu, incl, 31);
            TreePiece<K> &d = pc[slot];
            if (lane < c) {
                d.off[lane] = region + (int)(((uintptr_t)src - ga0) / sizeof(K));
                d.len[lane] = len;
            }
            if (lane == 0) {
                d.M = M;
                d.c = c;
                d.out = P.off[b] + outsum;
            }
            HS_DASSERT(M <= G::CAP && total_words <= SLOT);
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(&full[slot], (uint32_t)total_words * sizeof(K));
            __syncwarp();
            if (words > 0) bulk_g2s(stage0 + slot * SLOT + region, (const void *)ga0, (uint32_t)words * sizeof(K),
                                    &full[slot]);
            ++it;
        }
    }

    // ---------------------------------------------------------------- consumers
    const K kMax = KeyTraits<K>::kMax;
    for (int it = 0;; ++it) {
        const int slot = it % kTreeST;
        mbar_wait(&full[slot], (it / kTreeST) & 1);
        const TreePiece<K> &d = pc[slot];
        const int M = d.M;
        if (M < 0) break;
        const int c = d.c;
        const K *sb = stage0 + slot * SLOT;
        K *const out = F + d.out;
        const int sh = (int)(((uintptr_t)out & 15) / sizeof(K));
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // last store done reading
        if (tid < c) rl[tid] = d.len[tid];
        tree_bar(NC);
        // rounds: runs (2q, 2q+1) -> run q; round 1 reads the stage slices, later rounds the
        // previous round's buffer (runs contiguous); the last round writes at the phase sh
        int nruns = c;
        const K *in = nullptr;
        K *dst = Y;
        for (int r = 0; (1 << r) < c; ++r) {
            const bool last = (2 << r) >= c;
            K *const o = dst + (last ? sh : 0);
            // my outputs [p, pe)
            int p = tid * VT;
            const int pe = min(p + VT, M);
            // find the pair holding p: prefix over pairs
            int q = 0, Oq = 0;
            int na = 0, nb = 0;
            auto load_pair = [&](int qq) {
                na = rl[2 * qq];
                nb = rl[2 * qq + 1];
            };
            int runoff = 0;  // start of run 2q in the previous round's buffer
            if (p < pe) {
                load_pair(0);
                while (Oq + na + nb <= p) {
                    Oq += na + nb;
                    ++q;
                    load_pair(q);
                }
                runoff = Oq;
            }
            while (p < pe) {
                const K *A, *B;
                if (r == 0) {
                    A = sb + d.off[2 * q];
                    B = sb + d.off[2 * q + 1];
                } else {
                    A = in + runoff;
                    B = in + runoff + na;
                }
                const int diag = p - Oq;
                const int a0 = tree_path(A, na, B, nb, diag);
                int ai = a0, bi = diag - a0;
                const int kend = min(pe, Oq + na + nb);
                K x = ai < na ? A[ai] : kMax;
                K y = bi < nb ? B[bi] : kMax;
                for (; p < kend; ++p) {
                    const bool tA = bi >= nb || (ai < na && x <= y);
                    o[p] = tA ? x : y;
                    if (tA) {
                        ++ai;
                        x = ai < na ? A[ai] : kMax;
                    } else {
                        ++bi;
                        y = bi < nb ? B[bi] : kMax;
                    }
                }
                if (p < pe) {  // next pair
                    Oq += na + nb;
                    runoff = Oq;
                    ++q;
                    load_pair(q);
                }
            }
            tree_bar(NC);  // round complete: every thread read its inputs
            if (r == 0 && (tid & 31) == 0) tree_arrive(&empty[slot]);  // stage slot free for the next segment
            // next round's runs
            if (tid == 0) {
                for (int k = 0; k < nruns / 2; ++k) rl[k] = rl[2 * k] + rl[2 * k + 1];
            }
            nruns >>= 1;
            in = dst;
            dst = (dst == Y) ? X : Y;
            tree_bar(NC);
        }
        // the sorted segment sits at in[sh .. sh + M): bulk store the aligned middle
        const K *so = in;
        fence_proxy_async_smem();
        tree_bar(NC);
        const int end = sh + M;
        const int m0 = sh == 0 ? 0 : E;
        const int m1 = end / E * E;
        K *const g = out - sh;
        if (m1 > m0) {
            if (tid == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g + m0),
                             "r"(smem_u32(so + m0)), "r"((uint32_t)((m1 - m0) * sizeof(K)))
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (tid < E) {
                const int pp = sh + tid;
                if (pp < m0 && pp < end) g[pp] = so[pp];
            } else if (tid < 2 * E) {
                const int pp = m1 + tid - E;
                if (pp < end) g[pp] = so[pp];
            }
        } else {
            for (int pp = sh + tid; pp < end; pp += NC) g[pp] = so[pp];
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
