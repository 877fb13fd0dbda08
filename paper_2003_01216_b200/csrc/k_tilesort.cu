// k_tilesort.cu -- a4 (chunk plan from given offsets) and a5's first stage:
// the in-shared-memory sort of every leaf tile of every chunk.
//
//   K4 k_plan       chunk / leaf-tile geometry from caller-given offsets
//   K5 k_tile_sort  per-CTA sort of one leaf tile (<= T keys)
//
// The rest of a5 (in-chunk merge levels) and a6 are in k_merge.cu; a1-a3 in
// k_partition.cu.  Design notes and rooflines: DESIGN.md §5.
#include <cstdint>
#include <cstring>

#include "hs_device.cuh"
#include "hs_launch.h"

namespace hs {

// Copy the plan into shared memory (one word per thread).
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

// =============================================================== launchers
template <typename K>
struct SGeo;
template <>
struct SGeo<int32_t> {
    static constexpr int kNT = 512, kVT = 16;
};
template <>
struct SGeo<int64_t> {
    static constexpr int kNT = 512, kVT = 8;
};

int sort_tile_keys(int dt) { return dt == 0 ? SGeo<int32_t>::kNT * SGeo<int32_t>::kVT : SGeo<int64_t>::kNT * SGeo<int64_t>::kVT; }

cudaError_t launch_plan(const long long *user_off, Ctl *ctl, int log2c, int mode, int tile_keys, cudaStream_t st) {
    k_plan<<<1, 32, 0, st>>>(user_off, ctl, log2c, mode, tile_keys);
    return cudaGetLastError();
}

template <typename K>
cudaError_t launch_tile_sort_t(const Plan *plan, const void *src, void *F, void *S, long long max_tiles,
                               cudaStream_t st) {
    using G = SGeo<K>;
    if (max_tiles <= 0) return cudaSuccess;
    k_tile_sort<K, G::kNT, G::kVT><<<(unsigned)max_tiles, G::kNT, 0, st>>>(plan, (const K *)src, (K *)F, (K *)S);
    return cudaGetLastError();
}

cudaError_t launch_tile_sort(int dt, const Plan *plan, const void *src, void *F, void *S, long long max_tiles,
                             cudaStream_t st) {
    return dt == 0 ? launch_tile_sort_t<int32_t>(plan, src, F, S, max_tiles, st)
                   : launch_tile_sort_t<int64_t>(plan, src, F, S, max_tiles, st);
}

}  // namespace hs
