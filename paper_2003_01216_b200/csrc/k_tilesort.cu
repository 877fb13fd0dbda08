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
//   2. log2(T/VT) bitonic merge passes: strides inside a warp use warp
//      shuffles, strides across warps exchange through shared memory.
// Keys-only data makes the sorted tile unique, so the (unstable) network
// order is unobservable.  The tile is padded to a power of two with the
// dtype maximum; pads sort to the end and are never stored (they equal any
// real maximum key, so the stored prefix is the same multiset).
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

#ifndef HS_SORT_NT
#define HS_SORT_NT 256
#endif
#ifndef HS_SORT_VT
#define HS_SORT_VT 32
#endif
#ifndef HS_SORT_NT64
#define HS_SORT_NT64 256
#endif
#ifndef HS_SORT_VT64
#define HS_SORT_VT64 16
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

// =================================================================== K5
// Bitonic tile sort.  Logical element e = t*VT + k lives in register k of
// thread t.  Sorting runs of width W into runs of 2W ("pass W") is one
// bitonic merge: a mirror stage (e <-> the mirror of e inside its 2W block,
// lower half keeps the min) followed by half-cleaner stages of stride
// W/2 .. 1 (lower index keeps the min).  A stride of S elements is
//   S <  VT        : inside a thread  -> compare-exchange of two registers
//   S >= VT, lanes : inside a warp    -> __shfl_xor_sync + predicated min/max
//   S >= 32*VT     : across warps     -> exchange through shared memory
// No stage depends on the data, so there are no searches and no
// data-dependent shared-memory addresses.
template <typename K>
__device__ __forceinline__ K kmin(K a, K b) { return a < b ? a : b; }
template <typename K>
__device__ __forceinline__ K kmax(K a, K b) { return a < b ? b : a; }

template <typename K>
__device__ __forceinline__ K shfl_xor_k(K v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// Half-cleaner stages with stride < VT (registers only).
template <typename K, int VT>
__device__ __forceinline__ void intra_stages(K (&v)[VT]) {
#pragma unroll
    for (int sd = VT / 2; sd >= 1; sd >>= 1) {
#pragma unroll
        for (int k = 0; k < VT; ++k) {
            if ((k & sd) == 0) {
                const K a = v[k], b = v[k + sd];
                v[k] = kmin(a, b);
                v[k + sd] = kmax(a, b);
            }
        }
    }
}

// Cross-warp exchange through shared memory (register-major layout
// sm[k*NT + t]: conflict-free).  partner thread pt, partner register
// index pk(k) = MIRROR ? VT-1-k : k.
template <typename K, int NT, int VT, bool MIRROR>
__device__ __forceinline__ void smem_stage(K *sm, int tid, int pt, bool keep_min, K (&v)[VT]) {
#pragma unroll
    for (int k = 0; k < VT; ++k) sm[k * NT + tid] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const K o = sm[(MIRROR ? VT - 1 - k : k) * NT + pt];
        v[k] = keep_min ? kmin(v[k], o) : kmax(v[k], o);
    }
    __syncthreads();
}

// Sort a thread's VT registers ascending: bitonic network with constant
// register indices (mirror stage + half-cleaners per block size).
template <typename K, int VT>
__device__ __forceinline__ void reg_sort(K (&v)[VT]) {
#pragma unroll
    for (int size = 2; size <= VT; size <<= 1) {
#pragma unroll
        for (int k = 0; k < VT; ++k) {
            const int base = k & ~(size - 1), off = k - base;
            if (off < size / 2) {
                const int m = base + size - 1 - off;
                const K a = v[k], b = v[m];
                v[k] = kmin(a, b);
                v[m] = kmax(a, b);
            }
        }
#pragma unroll
        for (int sd = size / 4; sd >= 1; sd >>= 1) {
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                if ((k & sd) == 0 && ((k & (size - 1)) + sd) < size) {
                    const K a = v[k], b = v[k + sd];
                    v[k] = kmin(a, b);
                    v[k + sd] = kmax(a, b);
                }
            }
        }
    }
}

// One bitonic merge pass turning runs of width W = VT*R into runs of 2W.
template <typename K, int NT, int VT, int R>
__device__ __forceinline__ void bitonic_pass(K *sm, int tid, K (&v)[VT]) {
    const int lane = tid & 31;
    // mirror stage: thread u (within its 2R-thread block) <-> 2R-1-u, register k <-> VT-1-k
    const bool lower = (tid & R) == 0;
    if constexpr (2 * R <= 32) {
#pragma unroll
        for (int k = 0; k < VT / 2; ++k) {
            const K o1 = __shfl_xor_sync(0xffffffffu, v[VT - 1 - k], 2 * R - 1);
            const K o2 = __shfl_xor_sync(0xffffffffu, v[k], 2 * R - 1);
            v[k] = lower ? kmin(v[k], o1) : kmax(v[k], o1);
            v[VT - 1 - k] = lower ? kmin(v[VT - 1 - k], o2) : kmax(v[VT - 1 - k], o2);
        }
    } else {
        smem_stage<K, NT, VT, true>(sm, tid, tid ^ (2 * R - 1), lower, v);
    }
    // half-cleaners across threads: thread distance R/2 .. 1
#pragma unroll
    for (int d = R / 2; d >= 1; d >>= 1) {
        const bool lo = (tid & d) == 0;
        if (d >= 32) {
            smem_stage<K, NT, VT, false>(sm, tid, tid ^ d, lo, v);
        } else {
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                const K o = __shfl_xor_sync(0xffffffffu, v[k], d);
                v[k] = lo ? kmin(v[k], o) : kmax(v[k], o);
            }
        }
    }
    (void)lane;
    intra_stages<K, VT>(v);
}

template <typename K, int NT, int VT, int R>
__device__ __forceinline__ void bitonic_passes(K *sm, int tid, K (&v)[VT]) {
    if constexpr (R < NT) {
        bitonic_pass<K, NT, VT, R>(sm, tid, v);
        bitonic_passes<K, NT, VT, 2 * R>(sm, tid, v);
    }
}

template <typename K, int NT, int VT>
__global__ void __launch_bounds__(NT) k_tile_sort(const Plan *__restrict__ plan_g, const K *src, K *F, K *S) {
    constexpr int T = NT * VT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K *const sm = reinterpret_cast<K *>(smem_raw);
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
    K *dst = (P.L[b] & 1) ? S : F;  // where this bucket's merge level 0 reads
    const K kMax = KeyTraits<K>::kMax;

    // coalesced loads straight into registers (any placement works before the
    // first network); pads are kMax and sort to the end
    const K *in = src + lo;
    K v[VT];
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const int j = k * NT + tid;
        v[k] = j < len ? in[j] : kMax;
    }
    reg_sort<K, VT>(v);
    bitonic_passes<K, NT, VT, 1>(sm, tid, v);

    // thread t holds sorted elements t*VT .. t*VT+VT-1: transpose through
    // padded shared memory for coalesced stores
#pragma unroll
    for (int k = 0; k < VT; ++k) sm[pad_idx(tid * VT + k)] = v[k];
    __syncthreads();
    K *out = dst + lo;
#pragma unroll 4
    for (int j = tid; j < len; j += NT) out[j] = sm[pad_idx(j)];
    (void)T;
}

// =============================================================== launchers
template <typename K>
struct SGeo;
template <>
struct SGeo<int32_t> {
    static constexpr int kNT = HS_SORT_NT, kVT = HS_SORT_VT;  // default 256 x 32 = 8192 keys
};
template <>
struct SGeo<int64_t> {
    static constexpr int kNT = HS_SORT_NT64, kVT = HS_SORT_VT64;  // default 256 x 16 = 4096 keys
};

int sort_tile_keys(int dt) {
    return dt == 0 ? SGeo<int32_t>::kNT * SGeo<int32_t>::kVT : SGeo<int64_t>::kNT * SGeo<int64_t>::kVT;
}

cudaError_t launch_plan(const long long *user_off, Ctl *ctl, int log2c, int mode, int tile_keys, cudaStream_t st) {
    prof_begin(kProfPlan, st);
    k_plan<<<1, 32, 0, st>>>(user_off, ctl, log2c, mode, tile_keys);
    prof_end(kProfPlan, st);
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_tile_sort_t(const Plan *plan, const void *src, void *F, void *S, long long max_tiles,
                               cudaStream_t st) {
    using G = SGeo<K>;
    constexpr int T = G::kNT * G::kVT;
    constexpr size_t smem = (size_t)(T + T / 32) * sizeof(K);  // padded transpose / cross-warp exchange
    auto kern = k_tile_sort<K, G::kNT, G::kVT>;
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
    kern<<<(unsigned)max_tiles, G::kNT, smem, st>>>(plan, (const K *)src, (K *)F, (K *)S);
    prof_end(kProfTileSort, st);
    return cudaGetLastError();
}

cudaError_t launch_tile_sort(int dt, const Plan *plan, const void *src, void *F, void *S, long long max_tiles,
                             cudaStream_t st) {
    return dt == 0 ? launch_tile_sort_t<int32_t>(plan, src, F, S, max_tiles, st)
                   : launch_tile_sort_t<int64_t>(plan, src, F, S, max_tiles, st);
}

}  // namespace hs
