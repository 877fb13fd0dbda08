// k_tree.cu -- a6, the paper's binary-tree merge of a bucket's c sorted chunks
// (§3.2: "threads sort and merge two children sorted lists ... in a
// binary tree fashion"), run on chip in ONE HBM pass for the buckets whose
// chunks K5a split into equal-width sub-ranges (plan.tree).
//
// Why it is exact: in such a bucket sub-range t of every chunk holds the keys
// of one and the same key interval, and the tile sort of every piece (chunk
// j, sub-range t) recorded e_j[u] = #keys in fine bins <= u of a common
// monotone map of that interval into kTreeFine bins (k_tilesort.cu,
// tree_bin).  Bins are disjoint key intervals, so every key of bin u is
// smaller than every key of bin u + 1, and a cut at a bin boundary is an exact
// co-rank in all c chunks at once: the keys of bins [u0, u1) of the c pieces
// are exactly the keys the paper's tree merge of the whole bucket puts at
// output positions off[b] + sum_j start_j(t) + sum_j E_j(u0) ... + sum_j
// E_j(u1) (E_j(u) = #keys in bins < u, start_j(t) = sub-range t's start in
// chunk j).  The same holds for every intermediate run of the tree: bin u of
// the merge of pieces J starts at sum_{j in J} E_j(u) inside that run.
//
// Segment = kTreeSegBins consecutive bins of one sub-range (a fixed grid: no
// segment list).  The tree merge runs the log2 c rounds of a segment in shared
// memory; round r merges run pairs (2q, 2q+1) (runs = merged groups of 2^r
// pieces), stable-left, and its work units are (pair q, bin u): their
// A / B parts and output position follow from the bin tables with no search;
// the threads of a unit split it at evenly spaced merge-path diagonals (a
// search over one bin of two runs only).
//
//   k_tree_check  every segment's key count <= CAP, else its bucket is marked
//                 in ctl->treebad and runs its merge levels instead (a bin with
//                 many duplicates, or a locally dense key range)
//   k_tree_merge  persistent, warp-specialised: a producer warp loads a
//                 segment's bin tables and fetches its c slices with 1-D bulk
//                 async copies into a 2-slot ring; consumer warps run the
//                 rounds and write the segment with one bulk async store
//
// HBM traffic: one read + one write of the bucket (2 n s), instead of 2 n s
// per tree level; the bin tables add 2 KB per piece.
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

namespace hs {

constexpr int kTreeSegBins = 32;                           // bins per segment
constexpr int kTreeSegs = kTreeFine / kTreeSegBins;        // segments per sub-range
constexpr int kTreeMaxC = 1 << kTreeMaxLog2C;
constexpr int kTreeLog2TPB = 3;                            // consumer threads per bin: 8
constexpr int kTreeNC = kTreeSegBins << kTreeLog2TPB;      // consumer threads = (pairs x bins x parts) per round
constexpr int kTreeST = 2;                                 // stage slots

template <typename K>
struct TreeSmem {
    // CAP: keys per segment (uniform C3: mean 8 x 32 x ~24 = 6.1k; C5 int64 3.1k)
    static constexpr int CAP = sizeof(K) == 4 ? 8192 : 4096;
    static constexpr int E = 16 / sizeof(K);
    // a slot holds the c slices' 16-byte aligned supersets (each <= len + 2E - 2 keys, rounded to E),
    // later the odd rounds' output; Y the even rounds' (+ the destination's 16-byte phase)
    static constexpr int SLOT = CAP + 3 * E * kTreeMaxC + E;  // (+ E per slice: its sentinel)
    static constexpr int BUF = CAP + kTreeMaxC + 2 * E;
    static constexpr size_t bytes() { return (size_t)(kTreeST * SLOT + BUF) * sizeof(K); }
};

// Segment g -> (bucket, sub-range, first bin) over the tree buckets of the plan.
__device__ __forceinline__ bool tree_segment(const Plan &P, long long g, int &b, int &t, int &u0) {
    long long s = g / kTreeSegs;
    u0 = (int)(g % kTreeSegs) * kTreeSegBins;
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

__device__ __forceinline__ long long tree_segments(const Plan &P) {
    long long s = 0;
    for (int b = 0; b < 10; ++b) s += P.tree[b] ? P.nsb[b] : 0;
    return s * kTreeSegs;
}

__device__ __forceinline__ const uint16_t *tree_etab(const Plan &P, const uint16_t *etab, int b, int j, int t) {
    return etab + (size_t)(P.tile_prefix[b] + (long long)j * P.nsb[b] + t) * kTreeFine;
}

// ================================================================ check
// One thread per segment: its key count sum_j (E_j(u1) - E_j(u0)) must fit CAP.
__global__ void __launch_bounds__(256) k_tree_check(Ctl *ctl, const uint16_t *__restrict__ etab, int cap) {
    griddep_wait();  // PDL: the tile sort's bin tables are complete
    __shared__ Plan P;
    {
        constexpr int W = sizeof(Plan) / 4;
        const uint32_t *src = reinterpret_cast<const uint32_t *>(&ctl->plan);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&P);
        for (int i = threadIdx.x; i < W; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const long long nseg = tree_segments(P);
    const int c = 1 << P.log2c;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < nseg;
         g += (long long)gridDim.x * blockDim.x) {
        int b, t, u0;
        tree_segment(P, g, b, t, u0);
        int M = 0;
        for (int j = 0; j < c; ++j) {
            const uint16_t *e = tree_etab(P, etab, b, j, t);
            M += (int)__ldg(e + u0 + kTreeSegBins - 1) - (u0 ? (int)__ldg(e + u0 - 1) : 0);
        }
        if (M > cap) atomicOr(&ctl->treebad, 1u << b);
    }
}

// ================================================================ merge
template <typename K>
struct TreePiece {
    long long out;                          // first output position (absolute)
    int M;                                  // keys in the segment (< 0: no more segments)
    int off[kTreeMaxC];                     // slice j starts at stage + off[j]
    int T[kTreeMaxC][kTreeSegBins + 1];     // T[j][v]: start of bin u0 + v inside slice j (T[j][NB] = its length)
};

__device__ __forceinline__ void tree_bar() { asm volatile("bar.sync 1, %0;" ::"r"(kTreeNC) : "memory"); }
__device__ __forceinline__ void tree_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Mbarrier phase wait with a suspend-time hint (the thread sleeps in hardware
// until the phase completes instead of re-issuing the try_wait).
__device__ __forceinline__ void tree_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra TW_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
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

// Outputs [d0, d1) of the stable-left merge of A[0, na) and B[0, nb) (shared
// addresses ua, ub) to shared address uo + d0 s: merge-path split of d0, then
// a serial merge.  The element just past each part is >= every key of the
// other part: the next bin's first key (bins are disjoint key intervals), or
// the kMax sentinel after a run.  So B is never taken past its end (taken
// only when strictly smaller), and A's pointer is clamped at its end (a real
// kMax key in B ties the sentinel: A's kMax is emitted, the same value) --
// no bounds tests.
template <typename K>
__device__ __forceinline__ void tree_merge_part(uint32_t ua, int na, uint32_t ub, int nb, int d0, int d1,
                                                uint32_t uo) {
    constexpr uint32_t W = sizeof(K);
    int l = d0 - nb > 0 ? d0 - nb : 0;
    int r = d0 < na ? d0 : na;
    while (l < r) {
        const int mid = (l + r) >> 1;
        const bool pr = tlds<K>(ua + mid * W) <= tlds<K>(ub + (d0 - 1 - mid) * W);
        l = pr ? mid + 1 : l;
        r = pr ? r : mid;
    }
    uint32_t pa = ua + l * W, pb = ub + (d0 - l) * W;
    const uint32_t ea = ua + na * W;
    K x = tlds<K>(pa), y = tlds<K>(pb);
    uint32_t o = uo + d0 * W;
    int cnt = d1 - d0;
    auto step = [&]() {
        const bool tA = x <= y;
        tsts<K>(o, tA ? x : y);
        o += W;
        pa = tA ? min(pa + W, ea) : pa;
        pb += tA ? 0u : W;
        const K t = tlds<K>(tA ? pa : pb);
        x = tA ? t : x;
        y = tA ? y : t;
    };
    for (; cnt >= 4; cnt -= 4) {
        step();
        step();
        step();
        step();
    }
    for (; cnt > 0; --cnt) step();
}

// Persistent, warp-specialised; CTA blk owns the contiguous segment range
// [blk * per, (blk + 1) * per).
//   producer warp: a segment's bin tables (lanes: 32 bins of one chunk at a
//     time) and split-table starts, then the c slices by 1-D bulk async copies
//     (16-byte aligned supersets) into a free stage slot (full/empty mbarriers);
//   consumer warps: round r, thread = (pair q, bin u, part s) with
//     pairs x bins x parts = kTreeNC: parts of unit (q, u) are evenly spaced
//     merge-path cuts of its bin; even rounds write Y, odd rounds the stage slot
//     (its slices are consumed by round 0), the last round (even: log2 c odd)
//     writes Y at the destination's 16-byte phase; Y leaves with one bulk
//     async store.
template <typename K>
__global__ void __launch_bounds__(kTreeNC + 32, 2) k_tree_merge(const Ctl *__restrict__ ctl,
                                                             const uint32_t *__restrict__ sbtab,
                                                             const uint16_t *__restrict__ etab, const K *S, K *F) {
    using G = TreeSmem<K>;
    constexpr int E = G::E, SLOT = G::SLOT, NB = kTreeSegBins, NC = kTreeNC;
    constexpr int W = sizeof(K);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const stage0 = reinterpret_cast<K *>(smem_raw);
    K *const Y = stage0 + kTreeST * SLOT;
    __shared__ __align__(8) uint64_t full[kTreeST];
    __shared__ __align__(8) uint64_t empty[kTreeST];
    __shared__ Plan P;
    __shared__ TreePiece<K> pc[kTreeST];
    const int tid = threadIdx.x;

    griddep_wait();  // PDL: the tree check (and the tile sort before it) is complete
    {
        constexpr int WP = sizeof(Plan) / 4;
        const uint32_t *src = reinterpret_cast<const uint32_t *>(&ctl->plan);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&P);
        for (int i = tid; i < WP; i += blockDim.x) dst[i] = src[i];
    }
    if (tid == 0) {
        for (int i = 0; i < kTreeST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NC / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const long long nseg = tree_segments(P);
    const long long per = (nseg + gridDim.x - 1) / gridDim.x;
    const long long i0 = (long long)blockIdx.x * per, i1 = min(i0 + per, nseg);
    if (i0 >= i1) return;
    const unsigned tbad = ctl->treebad;
    const int lg = P.log2c, c = 1 << lg;

    if (tid >= NC) {
        // ------------------------------------------------------------ producer warp
        const int lane = tid & 31;
        int it = 0;
        for (long long i = i0;; ++i) {
            int b = 0, t = 0, u0 = 0;
            bool have = false;
            for (; i < i1; ++i) {  // next segment of a bucket that takes the on-chip tree
                tree_segment(P, i, b, t, u0);
                if (!((tbad >> b) & 1u)) {
                    have = true;
                    break;
                }
            }
            const int slot = it % kTreeST;
            tree_wait(&empty[slot], ((it / kTreeST) & 1) ^ 1);
            TreePiece<K> &d = pc[slot];
            if (!have) {
                if (lane == 0) {
                    d.M = -1;
                    mbar_arrive_expect_tx(&full[slot], 0);
                }
                return;
            }
            // bin tables: T[j][v] = E_j(u0 + v) - E_j(u0); lane v holds bin u0 + v's end -> T[j][v + 1]
            int len = 0, e0 = 0;
            for (int j = 0; j < c; ++j) {
                const uint16_t *e = tree_etab(P, etab, b, j, t);
                const int eb = u0 ? (int)__ldg(e + u0 - 1) : 0;
                const int ev = (int)__ldg(e + u0 + lane) - eb;
                d.T[j][lane + 1] = ev;
                if (lane == 0) d.T[j][0] = 0;
                const int lj = __shfl_sync(0xffffffffu, ev, NB - 1);
                if (lane == j) {
                    e0 = eb;
                    len = lj;
                }
            }
            const K *src = S;
            int outpart = 0;
            if (lane < c) {  // lane j: chunk j's slice
                const int ns = P.nsb[b];
                const long long m = P.off[b + 1] - P.off[b];
                const uint32_t st = __ldg(sbtab + P.sboff[b] + (long long)lane * (ns + 1) + t);
                outpart = (int)st + e0;
                src = S + P.off[b] + part_start(m, lg, lane) + st + e0;
            }
            const uintptr_t ga0 = (uintptr_t)src & ~(uintptr_t)15;
            const uintptr_t ga1 = ((uintptr_t)(src + len) + 15) & ~(uintptr_t)15;
            const int words = len > 0 ? (int)((ga1 - ga0) / W) : 0;  // multiple of E
            int incl = lane < c ? words + E : 0;  // + a gap for the sentinel after the slice
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int region = incl - (lane < c ? words + E : 0);
            int M = len, outsum = outpart;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                M += __shfl_xor_sync(0xffffffffu, M, o);
                outsum += __shfl_xor_sync(0xffffffffu, outsum, o);
            }
            const int total_words = __shfl_sync(0xffffffffu, incl, 31);  // (incl. gaps)
            int tx = words;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
            if (lane < c) d.off[lane] = len > 0 ? region + (int)(((uintptr_t)src - ga0) / W) : region;
            if (lane == 0) {
                d.M = M;
                d.out = P.off[b] + outsum;
            }
            HS_DASSERT(M <= G::CAP && total_words <= SLOT);
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(&full[slot], (uint32_t)tx * W);
            __syncwarp();
            if (words > 0) bulk_g2s(stage0 + slot * SLOT + region, (const void *)ga0, (uint32_t)words * W, &full[slot]);
            ++it;
        }
    }

    // ---------------------------------------------------------------- consumers
    const uint32_t uY = smem_u32(Y);
    for (int it = 0;; ++it) {
        const int slot = it % kTreeST;
        tree_wait(&full[slot], (it / kTreeST) & 1);
        const TreePiece<K> &d = pc[slot];
        const int M = d.M;
        if (M < 0) break;
        K *const sb = stage0 + slot * SLOT;
        const uint32_t usb = smem_u32(sb);
        K *const out = F + d.out;
        const int sh = (int)(((uintptr_t)out & 15) / W);
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // Y free again
        if (tid < c) sb[d.off[tid] + d.T[tid][NB]] = KeyTraits<K>::kMax;  // sentinel after each slice
        tree_bar();
        for (int r = 0; r < lg; ++r) {
            const bool last = r + 1 == lg;
            const int m = 1 << r;                 // pieces per input run
            // threads per (pair, bin) unit: S_ = NC / (pairs NB) = 2^lS (pairs = c >> (r + 1))
            const int lS = kTreeLog2TPB - lg + r + 1;
            const int unit = tid >> lS, part = tid & ((1 << lS) - 1);
            const int q = unit / NB, u = unit % NB;
            // bin u / u + 1 starts of runs 2q (A: pieces [2qm, 2qm + m)) and 2q + 1 (B); the pieces
            // before 2qm give the pair's base in the round's buffers
            int a_u = 0, a_u1 = 0, b_u = 0, b_u1 = 0, before = 0, la_tot = 0;
            for (int j = 0; j < 2 * q * m; ++j) before += d.T[j][NB];
            for (int j = 2 * q * m; j < 2 * q * m + m; ++j) {
                a_u += d.T[j][u];
                a_u1 += d.T[j][u + 1];
                la_tot += d.T[j][NB];
            }
            for (int j = 2 * q * m + m; j < 2 * q * m + 2 * m; ++j) {
                b_u += d.T[j][u];
                b_u1 += d.T[j][u + 1];
            }
            uint32_t ua, ub;
            if (r == 0) {  // the stage slices
                ua = usb + (d.off[2 * q] + a_u) * W;
                ub = usb + (d.off[2 * q + 1] + b_u) * W;
            } else {       // the previous round's buffer: run k at (pieces before it) + k (one sentinel each)
                const uint32_t in = (r & 1) ? uY : usb;
                ua = in + (before + 2 * q + a_u) * W;
                ub = in + (before + la_tot + 2 * q + 1 + b_u) * W;
            }
            const int na = a_u1 - a_u, nb = b_u1 - b_u, n = na + nb;
            K *const ob = (r & 1) ? sb : Y + (last ? sh : 0);
            const int obase = last ? 0 : before + q;  // pair q's output run, after q sentinels
            tree_merge_part<K>(ua, na, ub, nb, (n * part) >> lS, (n * (part + 1)) >> lS,
                               smem_u32(ob) + (obase + a_u + b_u) * W);
            if (!last && u == NB - 1 && part == 0) {  // the sentinel after pair q's output run
                int lb_tot = 0;
                for (int j = 2 * q * m + m; j < 2 * q * m + 2 * m; ++j) lb_tot += d.T[j][NB];
                ob[obase + la_tot + lb_tot] = KeyTraits<K>::kMax;
            }
            tree_bar();  // round complete
        }
        if ((tid & 31) == 0) tree_arrive(&empty[slot]);  // the slot (inputs and odd rounds) is free
        // the sorted segment sits at Y[sh .. sh + M): bulk store the aligned middle
        fence_proxy_async_smem();
        tree_bar();
        const int end = sh + M;
        const int m0 = sh == 0 ? 0 : E;
        const int m1 = end / E * E;
        K *const g = out - sh;
        if (m1 > m0) {
            if (tid == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g + m0),
                             "r"(uY + m0 * W), "r"((uint32_t)((m1 - m0) * W))
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
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTreeNC + 32, G::bytes());
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

size_t tree_etab_bytes(long long max_tiles) { return (size_t)max_tiles * kTreeFine * sizeof(uint16_t); }

template <typename K>
cudaError_t launch_tree_t(Ctl *ctl, const uint32_t *sbtab, const uint16_t *etab, const K *S, K *F, cudaStream_t st,
                          bool check_only) {
    using G = TreeSmem<K>;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const int sms = g_tree_sms[dev];
    prof_begin(kProfTreePlan, st);
    e = launch_pdl(k_tree_check, dim3((unsigned)(2 * sms)), dim3(256), 0, st, ctl, etab, (int)G::CAP);
    prof_end(kProfTreePlan, st);
    if (e != cudaSuccess || check_only) return e;
    prof_begin(kProfTreeMerge, st);
    const int grid = g_tree_per_sm[dev][sizeof(K) == 8 ? 1 : 0] * sms;
    e = launch_pdl(k_tree_merge<K>, dim3((unsigned)grid), dim3(kTreeNC + 32), G::bytes(), st, (const Ctl *)ctl, sbtab,
                   etab, S, F);
    prof_end(kProfTreeMerge, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_tree(int dt, Ctl *ctl, const uint32_t *sbtab, const uint16_t *etab, const void *S, void *F,
                        cudaStream_t st, bool check_only) {
    return dt == 0 ? launch_tree_t<int32_t>(ctl, sbtab, etab, (const int32_t *)S, (int32_t *)F, st, check_only)
                   : launch_tree_t<int64_t>(ctl, sbtab, etab, (const int64_t *)S, (int64_t *)F, st, check_only);
}

}  // namespace hs
