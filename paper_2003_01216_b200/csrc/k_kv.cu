// k_kv.cu -- SURVEY §8(f) f3, the key + tag (stable) variant on KV64 items:
// SPEC's SortItem, a key plus a 64-bit tag that travels with it
// through every pass and "never influences order".  Used by hs_sort_pairs64 /
// hs_msd_partition_pairs64 / hs_sort_chunks_pairs / hs_merge_pairs (int32 keys
// widen to the item's int64 key: the same order and the same leading digit).
//
// Every kernel an item passes through is stable, so equal keys keep their
// input order -- the paper's "Merge sort is a stable sort":
//   K1-K3  (k_partition.cu) the counting scatter ranks keys in input order
//   K5kv   k_tile_sort_kv: each thread sorts VT consecutive items with an
//          odd-even transposition network (compare-exchange of ADJACENT
//          items, swapping only on a strictly greater key: stable), then
//          log2(NT) merge-path rounds, stable-left (ties take A), with
//          explicit run ends
//   K6     (k_merge.cu) merge levels, stable-left, explicit run ends
//          (ExactEnds<KV64>) -- the paper's tree merge on items
// No K5a value split here: its atomic ranking is not stable.
//
//   K0kv k_pack_kv    items[i] = {key[i] (widened), tag[i]}
//   K8kv k_unpack_kv  key[i] = items[i].k (narrowed), tag[i] = items[i].v
// Pack and unpack are sequential streams (no gather).
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

namespace hs {

#ifndef HS_KV_NT
#define HS_KV_NT 256
#endif
#ifndef HS_KV_VT
#define HS_KV_VT 15
#endif

// ----------------------------------------------------------------- pack / unpack
__global__ void k_pack_kv(const void *__restrict__ keys, int key64, const unsigned long long *__restrict__ tags,
                          KV64 *__restrict__ items, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const long long k = key64 ? reinterpret_cast<const long long *>(keys)[i]
                                  : (long long)reinterpret_cast<const int32_t *>(keys)[i];
        items[i] = KV64{k, tags[i]};
    }
}

__global__ void k_unpack_kv(const KV64 *__restrict__ items, void *__restrict__ keys, int key64,
                            unsigned long long *__restrict__ tags, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const KV64 it = items[i];
        if (key64) reinterpret_cast<long long *>(keys)[i] = it.k;
        else reinterpret_cast<int32_t *>(keys)[i] = (int32_t)it.k;
        tags[i] = it.v;
    }
}

// ----------------------------------------------------------------- K5kv
__device__ __forceinline__ void cx_stable(KV64 &a, KV64 &b) {
    const bool sw = a.k > b.k;  // strictly greater: equal keys never move past each other
    const KV64 lo = sw ? b : a, hi = sw ? a : b;
    a = lo;
    b = hi;
}

// Odd-even transposition sort of N registers: N rounds of adjacent
// compare-exchanges (compile-time indices, no branches).  Stable.
template <int N>
__device__ __forceinline__ void transposition_sort(KV64 (&v)[N]) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
#pragma unroll
        for (int i = r & 1; i + 1 < N; i += 2) cx_stable(v[i], v[i + 1]);
    }
}

__device__ __forceinline__ void load_plan_kv(Plan &dst, const Plan *src) {
    constexpr int W = sizeof(Plan) / 4;
    const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
    uint32_t *d = reinterpret_cast<uint32_t *>(&dst);
    for (int i = threadIdx.x; i < W; i += blockDim.x) d[i] = __ldg(s + i);
}

// One leaf tile (<= NT VT items) per CTA: bulk load, pads (key INT64_MAX)
// after the leaf -- stable, so they stay behind any real INT64_MAX key and
// are never stored -- register sort, merge rounds, bulk store.  Leaves and
// the output buffer parity as K5 (k_tilesort.cu).
template <int NT, int VT>
__global__ void __launch_bounds__(NT, 3) k_tile_sort_kv(const Plan *__restrict__ plan_g, const KV64 *src, KV64 *F,
                                                        KV64 *S, KV64 *samp) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    constexpr int T = NT * VT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    KV64 *const sm = reinterpret_cast<KV64 *>(smem_raw);
    __shared__ Plan P;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    load_plan_kv(P, plan_g);
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
    const long long lo = leaf_start(P, b, i);
    const int len = (int)(leaf_start(P, b, i + 1) - lo);
    if (len == 0) return;
    HS_DASSERT(len > 0 && len <= T);
    KV64 *const out = ((P.L[b] & 1) ? S : F) + lo;
    if (tid == 0) {  // items are 16 bytes: every leaf is a whole number of bulk-copy granules
        mbar_arrive_expect_tx(&bar, (uint32_t)len * sizeof(KV64));
        bulk_g2s(sm, src + lo, (uint32_t)len * sizeof(KV64), &bar);
    }
    mbar_wait(&bar, 0);
    for (int j = len + tid; j < T; j += NT) sm[j] = KeyTraits<KV64>::kMax;
    __syncthreads();

    KV64 v[VT];
#pragma unroll
    for (int k = 0; k < VT; ++k) v[k] = sm[tid * VT + k];
    transposition_sort<VT>(v);
#pragma unroll 1
    for (int lgR = 0; (1 << lgR) < NT; ++lgR) {
        const int R = 1 << lgR, RL = R * VT;
        __syncthreads();  // everyone has read the previous round's runs
#pragma unroll
        for (int k = 0; k < VT; ++k) sm[tid * VT + k] = v[k];
        __syncthreads();
        const int j = tid & (2 * R - 1);
        const KV64 *A = sm + (tid - j) * VT, *B = A + RL;  // runs of RL items, ascending
        const int diag = j * VT;
        int l = diag - RL > 0 ? diag - RL : 0, r = diag < RL ? diag : RL;
        while (l < r) {
            const int mid = (l + r) >> 1;
            if (A[mid].k <= B[diag - 1 - mid].k) l = mid + 1;
            else r = mid;
        }
        int ai = l, bi = diag - l;
#pragma unroll
        for (int k = 0; k < VT; ++k) {
            const bool takeA = bi >= RL || (ai < RL && A[ai].k <= B[bi].k);  // stable-left
            v[k] = takeA ? A[ai] : B[bi];
            ai += takeA ? 1 : 0;
            bi += takeA ? 0 : 1;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) sm[tid * VT + k] = v[k];
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out), "r"(smem_u32(sm)),
                     "r"((uint32_t)len * (uint32_t)sizeof(KV64))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    write_samples(samp, lo, len, sm, tid, NT);  // coarse index for merge level 0's co-rank search
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ----------------------------------------------------------------- launchers
static int grid_for_kv(long long n, int num_sms) {
    const long long want = (n + 255) / 256;
    return (int)(want > 16LL * num_sms ? 16LL * num_sms : (want > 0 ? want : 1));
}

cudaError_t launch_pack_kv(const void *keys, int key64, const unsigned long long *tags, KV64 *items, long long n,
                           int num_sms, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    prof_begin(kProfCopy, st);
    k_pack_kv<<<grid_for_kv(n, num_sms), 256, 0, st>>>(keys, key64, tags, items, n);
    prof_end(kProfCopy, st);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
    return e;
}

cudaError_t launch_unpack_kv(const KV64 *items, void *keys, int key64, unsigned long long *tags, long long n,
                             int num_sms, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    prof_begin(kProfCopy, st);
    k_unpack_kv<<<grid_for_kv(n, num_sms), 256, 0, st>>>(items, keys, key64, tags, n);
    prof_end(kProfCopy, st);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
    return e;
}

int kv_tile_keys() { return HS_KV_NT * HS_KV_VT; }

cudaError_t setup_kv_kernels(int dev) {
    (void)dev;
    return cudaFuncSetAttribute(k_tile_sort_kv<HS_KV_NT, HS_KV_VT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(HS_KV_NT * HS_KV_VT * sizeof(KV64)));
}

cudaError_t launch_tile_sort_kv(const Plan *plan, const KV64 *src, KV64 *F, KV64 *S, KV64 *samp, long long max_tiles,
                                cudaStream_t st) {
    if (max_tiles <= 0) return cudaSuccess;
    prof_begin(kProfTileSort, st);
    const cudaError_t e = launch_pdl(k_tile_sort_kv<HS_KV_NT, HS_KV_VT>, dim3((unsigned)max_tiles), dim3(HS_KV_NT),
                                     (size_t)HS_KV_NT * HS_KV_VT * sizeof(KV64), st, plan, src, F, S, samp);
    if (e != cudaSuccess) return e;
    prof_end(kProfTileSort, st);
    return cudaGetLastError();
}

}  // namespace hs
