// k_partition.cu -- a1-a3: the one-step MSD radix partition into ten buckets
// (§3.4, "The master node divides the data into ten parts based on
// the most significant digit"), as three sm_100a kernels:
//
//   K1 k_tile_hist  leading-digit histogram of every scatter tile (one warp per
//                   tile, 128-bit streaming loads, packed per-lane counters,
//                   redux.sync warp reduction; no atomics)
//   K2 k_tile_scan  decoupled-lookback exclusive prefix over the tile
//                   histograms -> per-tile per-digit output base; its last CTA
//                   turns the totals into bucket_offsets (and the plan)
//   K3 k_scatter    stable scatter: rank each key among same-digit keys of its
//                   tile (input order), re-stage the tile in digit order in
//                   shared memory, write ten coalesced runs
//
// Output position of key i = off[d_i] + #{j < i : d_j = d_i}: exactly the
// stable counting pass of P:78 / S:302 (reading #4), so the result is unique.
// Tiles live in a virtual index space aligned to 16 bytes (h = leading
// misalignment of keys in elements), so every interior load is one aligned
// 128-bit vector.
#include <cstdint>
#include <cstring>

#include "hs_device.cuh"
#include "hs_launch.h"

#ifndef HS_K3_SBASE
#define HS_K3_SBASE 1
#endif
#ifndef HS_K3_REDIGIT
#define HS_K3_REDIGIT 1  // int32 K3: the write loop recomputes each staged key's digit (no digit bytes in smem)
#endif
#ifndef HS_SCAT_NT
#define HS_SCAT_NT 128
#endif
#ifndef HS_SCAT_VT
#define HS_SCAT_VT 16
#endif

namespace hs {

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

template <typename K>
struct PGeo;
template <>
struct PGeo<int32_t> {
    static constexpr int kScatNT = HS_SCAT_NT, kScatVT = HS_SCAT_VT;  // default 128 x 16 = 2048 keys per tile
};
template <>
struct PGeo<int64_t> {
    static constexpr int kScatNT = HS_SCAT_NT, kScatVT = HS_SCAT_VT / 2;
};
template <>
struct PGeo<KV64> {  // f3 items (k_kv.cu): 16 bytes each
    static constexpr int kScatNT = HS_SCAT_NT, kScatVT = HS_SCAT_VT / 4;
};
constexpr int kHistWarps = 8;
constexpr int kScanNT = 256, kScanIPT = 8;  // 2048 tile histograms per K2 CTA

// 6-bit packed per-digit counters in one 64-bit register (field d at bit 6d).
__device__ __forceinline__ void count6(unsigned long long &cnt, int d) { cnt += 1ull << (6 * d); }
__device__ __forceinline__ void flush6(unsigned long long &cnt, unsigned (&c)[10]) {
#pragma unroll
    for (int d = 0; d < 10; ++d) c[d] += (unsigned)(cnt >> (6 * d)) & 63u;
    cnt = 0;
}

// =================================================================== K1
template <typename K, int TP>
__global__ void __launch_bounds__(kHistWarps * 32) k_tile_hist(const K *__restrict__ keys, int n, int h,
                                                             DigitParams<K> dp, uint32_t *__restrict__ tile_hist,
                                                             int ntiles) {
    constexpr int E = 16 / sizeof(K);
    constexpr int VPL = TP / E / 32;  // vectors per lane per tile
    constexpr int U = 4;              // vectors in flight per lane
    constexpr int FLUSH = 60 / (U * E) > 0 ? 60 / (U * E) : 1;  // groups per flush (<= 63 keys)
    static_assert(VPL % U == 0, "tile shape");
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kHistWarps + (threadIdx.x >> 5);
    const int nw = gridDim.x * kHistWarps;
    for (int t = gw; t < ntiles; t += nw) {
        const long long v0 = (long long)t * TP - h;
        unsigned c[10];
#pragma unroll
        for (int d = 0; d < 10; ++d) c[d] = 0;
        unsigned long long cnt = 0;
        if (v0 >= 0 && v0 + TP <= n) {
            const K *base = keys + v0;
            int g = 0;
#pragma unroll 1
            for (int i = 0; i < VPL; i += U) {
                int4 q[U];
#pragma unroll
                for (int u = 0; u < U; ++u) q[u] = ld_stream_v4(base + ((i + u) * 32 + lane) * E);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    K vals[E];
                    memcpy(vals, &q[u], 16);
#pragma unroll
                    for (int e = 0; e < E; ++e) count6(cnt, msd_digit(vals[e], dp));
                }
                if (++g == FLUSH) {
                    flush6(cnt, c);
                    g = 0;
                }
            }
        } else {
            int g = 0;
            for (int i = 0; i < VPL; ++i) {
                const long long e0 = v0 + (long long)(i * 32 + lane) * E;
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (e0 + e >= 0 && e0 + e < n) count6(cnt, msd_digit(keys[e0 + e], dp));
                if (++g == 60 / E) {
                    flush6(cnt, c);
                    g = 0;
                }
            }
        }
        flush6(cnt, c);
        unsigned tot[10];
#pragma unroll
        for (int d = 0; d < 10; ++d) tot[d] = __reduce_add_sync(0xffffffffu, c[d]);
        if (lane < 5) {
            unsigned w = 0;
#pragma unroll
            for (int i = 0; i < 5; ++i)
                if (lane == i) w = tot[2 * i] | (tot[2 * i + 1] << 16);
            tile_hist[(size_t)t * 5 + lane] = w;
        }
    }
}

// =================================================================== K2
// Exclusive scan over the tile histograms with a decoupled lookback across
// CTAs (tile order = input order).  tile_pref[t][d] = #{keys with digit d in
// tiles < t}.  The CTA holding the last tiles knows the grand totals: it
// writes bucket_offsets (exclusive prefix over digits) and the plan.
__global__ void __launch_bounds__(kScanNT) k_tile_scan(const uint32_t *__restrict__ tile_hist,
                                                       uint32_t *__restrict__ tile_pref, int ntiles,
                                                       unsigned long long *status, Ctl *ctl, long long *user_off,
                                                       int plan_mode, int log2c, int tile_keys) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    constexpr int NW = kScanNT / 32;
    __shared__ unsigned s_wtot[NW][10];
    __shared__ unsigned s_cta_excl[10];
    __shared__ unsigned s_cid;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_cid = atomicAdd(&ctl->ticket, 1u);  // dispatch order = lookback order
    __syncthreads();
    const int cid = (int)s_cid;
    const int t0 = cid * kScanNT * kScanIPT + tid * kScanIPT;

    uint32_t w[kScanIPT][5];
    unsigned agg[10];
#pragma unroll
    for (int d = 0; d < 10; ++d) agg[d] = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) {
#pragma unroll
        for (int k = 0; k < 5; ++k) w[i][k] = (t0 + i < ntiles) ? tile_hist[(size_t)(t0 + i) * 5 + k] : 0u;
#pragma unroll
        for (int d = 0; d < 10; ++d) agg[d] += (w[i][d >> 1] >> ((d & 1) * 16)) & 0xFFFFu;
    }
    // block exclusive scan of agg[10]
    unsigned inc[10];
#pragma unroll
    for (int d = 0; d < 10; ++d) inc[d] = agg[d];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int d = 0; d < 10; ++d) {
            unsigned u = __shfl_up_sync(0xffffffffu, inc[d], o);
            if (lane >= o) inc[d] += u;
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int d = 0; d < 10; ++d) s_wtot[warp][d] = inc[d];
    }
    __syncthreads();
    if (warp == 0) {
        unsigned wt[10], wi[10];
#pragma unroll
        for (int d = 0; d < 10; ++d) {
            wt[d] = lane < NW ? s_wtot[lane][d] : 0u;
            wi[d] = wt[d];
        }
#pragma unroll
        for (int o = 1; o < NW; o <<= 1) {
#pragma unroll
            for (int d = 0; d < 10; ++d) {
                unsigned u = __shfl_up_sync(0xffffffffu, wi[d], o);
                if (lane >= o) wi[d] += u;
            }
        }
        unsigned tot[10];
#pragma unroll
        for (int d = 0; d < 10; ++d) tot[d] = __shfl_sync(0xffffffffu, wi[d], NW - 1);
        __syncwarp();
        if (lane < NW) {
#pragma unroll
            for (int d = 0; d < 10; ++d) s_wtot[lane][d] = wi[d] - wt[d];
        }
        // decoupled lookback across CTAs, lane d <-> digit d
        unsigned my_tot = 0;
#pragma unroll
        for (int d = 0; d < 10; ++d)
            if (lane == d) my_tot = tot[d];
        long long excl = 0;
        if (lane < 10) {
            unsigned long long *my = status + (size_t)cid * 10 + lane;
            if (cid == 0) {
                st_relaxed_u64(my, kFlagIncl | my_tot);
            } else {
                st_relaxed_u64(my, kFlagAgg | my_tot);
                long long p = cid - 1;
                while (true) {
                    unsigned long long sv;
                    do {
                        sv = ld_relaxed_u64(status + (size_t)p * 10 + lane);
                    } while ((sv >> 62) == 0);
                    excl += (long long)(sv & kValMask);
                    if ((sv >> 62) == 2) break;
                    --p;
                }
                st_relaxed_u64(my, kFlagIncl | (unsigned long long)(excl + my_tot));
            }
            s_cta_excl[lane] = (unsigned)excl;
        }
        // the CTA that owns the last tile holds the grand totals
        const int last_tile = cid * kScanNT * kScanIPT + kScanNT * kScanIPT - 1;
        if (last_tile >= ntiles - 1) {
            long long incl = excl + my_tot;
            long long off[11];
            off[0] = 0;
#pragma unroll
            for (int d = 0; d < 10; ++d) off[d + 1] = off[d] + __shfl_sync(0xffffffffu, incl, d);
            if (lane < 11) {
                long long v = 0;
#pragma unroll
                for (int d = 0; d < 11; ++d)
                    if (lane == d) v = off[d];
                ctl->off[lane] = v;
                if (user_off) user_off[lane] = v;
            }
            if (lane == 0 && plan_mode >= 0) compute_plan(&ctl->plan, off, log2c, plan_mode, tile_keys);
        }
    }
    __syncthreads();
    unsigned run[10];
#pragma unroll
    for (int d = 0; d < 10; ++d) run[d] = s_cta_excl[d] + s_wtot[warp][d] + (inc[d] - agg[d]);
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) {
        if (t0 + i < ntiles) {
#pragma unroll
            for (int d = 0; d < 10; ++d) tile_pref[(size_t)(t0 + i) * 10 + d] = run[d];
        }
#pragma unroll
        for (int d = 0; d < 10; ++d) run[d] += (w[i][d >> 1] >> ((d & 1) * 16)) & 0xFFFFu;
    }
}

// =================================================================== K3
// Where digit d's keys go: out (one array, CSR by bucket) unless `use`, in
// which case the key at local bucket position p of digit d is stored to
// dst[d] + (p - off[d]) -- dst[d] may be a peer GPU's buffer (NVLink P2P /
// symmetric memory): the cluster model's bucket exchange fused into the
// scatter (hs_partition_scatter).
template <typename K>
struct DstTable {
    K *dst[10];
    int use;
};

// int32 only: a 64-bit digit (umul64hi) costs more than the staged byte (C5 K3 2.18 vs 2.44 ms)
template <typename K>
__host__ __device__ constexpr bool k3_redigit() {
    return HS_K3_REDIGIT && sizeof(K) == 4;
}

template <typename K, int NT, int VT>
struct ScatSmem {
    static constexpr int T = NT * VT;
    static constexpr size_t bytes() { return (size_t)3 * T * sizeof(K) + (k3_redigit<K>() ? 0 : T); }  // 2 stages + out (+ digits)
};

// Rank + re-stage one tile held in `stage` (blocked: thread tid owns slots
// tid*VT ..).  FULL: every slot is a key (interior tile) -> no validity tests.
template <typename K, int NT, int VT, bool FULL, bool TABLE>
__device__ __forceinline__ void scatter_tile(const K *__restrict__ stage, K *__restrict__ sOut, uint8_t *sDig,
                                             K *__restrict__ out, int jlo, int jhi, int tile, const DigitParams<K> &dp,
                                             const Ctl *__restrict__ ctl, const uint32_t *__restrict__ tile_pref,
                                             unsigned (*s_wtot)[5], int *s_dstart, int *s_delta, K **s_dptr,
                                             const DstTable<K> &dtab) {
    constexpr int E = 16 / sizeof(K);
    constexpr int NW = NT / 32;
    constexpr int NMETA = VT / 4 > 0 ? VT / 4 : 1;
    [[maybe_unused]] constexpr int T_ = NT * VT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    unsigned meta[NMETA];
#pragma unroll
    for (int i = 0; i < NMETA; ++i) meta[i] = 0;
    unsigned long long cnt = 0;
#pragma unroll
    for (int k0 = 0; k0 < VT; k0 += E) {
        K kv[E];
        const int4 q = *reinterpret_cast<const int4 *>(stage + tid * VT + k0);
        memcpy(kv, &q, 16);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int k = k0 + e;
            int d;
            if (FULL) {
                d = msd_digit(kv[e], dp);
            } else {
                const int j = tid * VT + k;
                d = (j >= jlo && j < jhi) ? msd_digit(kv[e], dp) : 10;  // field 10 = "not a key"
            }
            const unsigned r = (unsigned)(cnt >> (6 * d)) & 63u;
            cnt += 1ull << (6 * d);
            meta[k >> 2] |= ((unsigned)d | (r << 4)) << (8 * (k & 3));
        }
    }
    // block exclusive scan of per-thread digit counts (5 words x 2 16-bit fields)
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
            const unsigned t = __shfl_up_sync(0xffffffffu, w[i], o);
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
                const unsigned u = __shfl_up_sync(0xffffffffu, t[i], o);
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
        if (lane < 10) {
            unsigned dstart = 0;
#pragma unroll
            for (int e = 0; e < 10; ++e) {
                const unsigned f = (tot[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
                if (e < lane) dstart += f;
            }
            s_dstart[lane] = (int)dstart;
            // global position of tile-local slot j of digit d = delta[d] + j (< 2^31)
            const long long delta = ctl->off[lane] + (long long)tile_pref[(size_t)tile * 10 + lane] - (long long)dstart;
            if (TABLE) s_dptr[lane] = dtab.dst[lane] - ctl->off[lane] + delta;
            else s_delta[lane] = (int)delta;  // < 2^31
        }
    }
    __syncthreads();

    // re-stage in digit order (stable: rank = input order within the tile)
    unsigned base[5];
#pragma unroll
    for (int i = 0; i < 5; ++i)
        base[i] = s_wtot[warp][i] + (w[i] - own[i]) + ((unsigned)s_dstart[2 * i] | ((unsigned)s_dstart[2 * i + 1] << 16));
#if HS_K3_SBASE
    // this thread's five packed digit bases in its own shared-memory column (read back
    // by the thread itself: no barrier; one LDS per key instead of a 4-deep select chain)
    __shared__ unsigned s_base[5 * NT];
#pragma unroll
    for (int i = 0; i < 5; ++i) s_base[i * NT + tid] = base[i];
#endif
#pragma unroll
    for (int k0 = 0; k0 < VT; k0 += E) {
        K kv[E];
        const int4 q = *reinterpret_cast<const int4 *>(stage + tid * VT + k0);
        memcpy(kv, &q, 16);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int k = k0 + e;
            const unsigned m = (meta[k >> 2] >> (8 * (k & 3))) & 0xFFu;
            const unsigned d = m & 15u, r = m >> 4;
            if (FULL || d < 10) {
#if HS_K3_SBASE
                const unsigned wsel = s_base[(d >> 1) * NT + tid];
#else
                const unsigned wsel = d < 2 ? base[0] : d < 4 ? base[1] : d < 6 ? base[2] : d < 8 ? base[3] : base[4];
#endif
                const int pos = (int)((wsel >> ((d & 1u) * 16)) & 0xFFFFu) + (int)r;
                HS_DASSERT(pos >= 0 && pos < T_ && d < 10);
                sOut[pos] = kv[e];
                if constexpr (!k3_redigit<K>()) sDig[pos] = (uint8_t)d;
            }
        }
    }
    __syncthreads();

    // ten coalesced runs
    const int nvalid = jhi - jlo;
    for (int j = tid; j < nvalid; j += NT) {
        const K key = sOut[j];
        int d;
        if constexpr (k3_redigit<K>()) d = msd_digit(key, dp);  // recomputed: cheaper than a staged digit byte
        else d = sDig[j];
        HS_DASSERT(d >= 0 && d < 10);
        if (TABLE) s_dptr[d][j] = key;
        else out[s_delta[d] + j] = key;
    }
}

// Persistent: each CTA walks tiles blockIdx.x, +gridDim.x, ...; the next
// tile is prefetched by one 1-D bulk async copy into the other stage while
// the current one is ranked and scattered.
template <typename K, int NT, int VT, bool TABLE>
__global__ void __launch_bounds__(NT) k_scatter(const K *__restrict__ keys, K *__restrict__ out, int n, int h,
                                                DigitParams<K> dp, const Ctl *__restrict__ ctl,
                                                const uint32_t *__restrict__ tile_pref, int ntiles, DstTable<K> dtab) {
    griddep_wait();  // PDL: the predecessor kernel's writes are visible from here
    constexpr int T = NT * VT;
    constexpr int NW = NT / 32;
    static_assert(VT <= 16 && T <= 16384, "packing limits");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    K *const stage0 = reinterpret_cast<K *>(smem_raw);
    K *const sOut = stage0 + 2 * T;
    uint8_t *const sDig = reinterpret_cast<uint8_t *>(sOut + T);
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ unsigned s_wtot[NW][5];
    __shared__ int s_dstart[10];
    __shared__ K *s_dptr[TABLE ? 10 : 1];
    __shared__ int s_delta[10];
    const int tid = threadIdx.x;

    // virtual tile t covers [t*T - h, (t+1)*T - h): 16-byte aligned in memory
    auto issue = [&](int t, int slot) {
        const long long v0 = (long long)t * T - h;
        const long long vend = v0 + T < n ? v0 + T : (long long)n;
        const uintptr_t g0 = (uintptr_t)(keys + v0);
        const uintptr_t g1 = ((uintptr_t)(keys + vend) + 15) & ~(uintptr_t)15;
        const uint32_t bytes = (uint32_t)(g1 - g0);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&mbar[slot], bytes);
        bulk_g2s(stage0 + slot * T, (const void *)g0, bytes, &mbar[slot]);
    };
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
        if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    }
    __syncthreads();
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int slot = it & 1;
        mbar_wait(&mbar[slot], (it >> 1) & 1);
        if (tid == 0 && t + (int)gridDim.x < ntiles) issue(t + gridDim.x, slot ^ 1);
        const long long v0 = (long long)t * T - h;
        const int jlo = v0 < 0 ? (int)(-v0) : 0;
        const int jhi = (int)((long long)n - v0 < T ? (long long)n - v0 : (long long)T);
        const K *stage = stage0 + slot * T;
        if (jlo == 0 && jhi == T)
            scatter_tile<K, NT, VT, true, TABLE>(stage, sOut, sDig, out, jlo, jhi, t, dp, ctl, tile_pref, s_wtot,
                                                 s_dstart, s_delta, s_dptr, dtab);
        else
            scatter_tile<K, NT, VT, false, TABLE>(stage, sOut, sDig, out, jlo, jhi, t, dp, ctl, tile_pref, s_wtot,
                                                  s_dstart, s_delta, s_dptr, dtab);
        __syncthreads();  // stage / sOut / tables are reused next iteration
    }
    // TABLE (hs_partition_scatter): the stores may target peer GPUs' memory;
    // order them before whatever signals the peers next (dist.py: grid
    // completion + a symmetric-memory barrier)
    if (TABLE) __threadfence_system();
}

// =============================================================== launchers
// resident K3 CTAs per SM, per device: [int32, int64] x [local CSR, destination table], KV64 items
int g_scatter_per_sm[kMaxDevices][5];

template <typename K, bool TABLE>
cudaError_t setup_scatter_t(int dev, int slot) {
    using G = PGeo<K>;
    using SS = ScatSmem<K, G::kScatNT, G::kScatVT>;
    auto kern = k_scatter<K, G::kScatNT, G::kScatVT, TABLE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS::bytes());
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::kScatNT, SS::bytes());
    g_scatter_per_sm[dev][slot] = occ > 0 ? occ : 1;
    return e;
}

cudaError_t setup_partition_kernels(int dev) {
    cudaError_t e;
    if ((e = setup_scatter_t<int32_t, false>(dev, 0)) != cudaSuccess) return e;
    if ((e = setup_scatter_t<int64_t, false>(dev, 1)) != cudaSuccess) return e;
    if ((e = setup_scatter_t<int32_t, true>(dev, 2)) != cudaSuccess) return e;
    if ((e = setup_scatter_t<int64_t, true>(dev, 3)) != cudaSuccess) return e;
    return setup_scatter_t<KV64, false>(dev, 4);
}

template <typename K>
int scatter_tile_keys_t() {
    return PGeo<K>::kScatNT * PGeo<K>::kScatVT;
}

template <typename K>
cudaError_t launch_partition_t(const void *keys, void *out, int n, int h, unsigned long long div,
                               unsigned long long magic, Ctl *ctl, uint32_t *tile_hist, uint32_t *tile_pref,
                               unsigned long long *status, long long *user_off, int plan_mode, int log2c,
                               int sort_tile_keys, int num_sms, bool do_scatter, int key_shift, cudaStream_t st,
                               bool do_count, void *const *dst10) {
    using G = PGeo<K>;
    constexpr int TP = G::kScatNT * G::kScatVT;
    DigitParams<K> dp;
    dp.div = (typename KeyTraits<K>::U)div;
    dp.magic = (typename KeyTraits<K>::U)magic;
    dp.shift = key_shift;
    {
        int l = 0;
        while ((1ull << l) < div) ++l;
        dp.post = div == 1 ? -1 : l - 1;
    }
    const long long ntiles = ((long long)n + h + TP - 1) / TP;
    if (do_count && ntiles > 0) {
        long long want = (ntiles + kHistWarps - 1) / kHistWarps;
        int grid = (int)(want > 8LL * num_sms ? 8LL * num_sms : want);
        prof_begin(kProfTileHist, st);
        k_tile_hist<K, TP><<<grid, kHistWarps * 32, 0, st>>>((const K *)keys, n, h, dp, tile_hist, (int)ntiles);
        prof_end(kProfTileHist, st);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        note_launch();
    }
    const long long per = (long long)kScanNT * kScanIPT;
    const int sgrid = (int)(ntiles > 0 ? (ntiles + per - 1) / per : 1);
    cudaError_t e = cudaSuccess;
    if (do_count) {
        prof_begin(kProfTileScan, st);
        e = launch_pdl(k_tile_scan, dim3(sgrid), dim3(kScanNT), 0, st, tile_hist, tile_pref, (int)ntiles, status, ctl,
                       user_off, plan_mode, log2c, sort_tile_keys);
        prof_end(kProfTileScan, st);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (e != cudaSuccess || !do_scatter || ntiles == 0) return e;
    using SS = ScatSmem<K, G::kScatNT, G::kScatVT>;
    // local CSR output, or the destination-pointer table of hs_partition_scatter (keys only)
    auto kern = (dst10 && sizeof(K) <= 8) ? k_scatter<K, G::kScatNT, G::kScatVT, sizeof(K) <= 8>
                                          : k_scatter<K, G::kScatNT, G::kScatVT, false>;
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    const int ki = sizeof(K) == 16 ? 4 : (dst10 ? 2 : 0) + (sizeof(K) == 8 ? 1 : 0);
    long long grid = (long long)g_scatter_per_sm[dev][ki] * num_sms;
    if (grid > ntiles) grid = ntiles;
    prof_begin(kProfScatter, st);
    DstTable<K> dtab;
    dtab.use = dst10 != nullptr;
    for (int d = 0; d < 10; ++d) dtab.dst[d] = dst10 ? (K *)dst10[d] : nullptr;
    cudaError_t el = launch_pdl(kern, dim3((unsigned)grid), dim3(G::kScatNT), SS::bytes(), st, (const K *)keys,
                                (K *)out, n, h, dp, ctl, tile_pref, (int)ntiles, dtab);
    if (el != cudaSuccess) return el;
    prof_end(kProfScatter, st);
    return cudaGetLastError();
}

int scatter_tile_keys(int dt) {
    return dt == 0 ? scatter_tile_keys_t<int32_t>() : dt == 1 ? scatter_tile_keys_t<int64_t>() : scatter_tile_keys_t<KV64>();
}

int scan_ctas(long long ntiles) {
    const long long per = (long long)kScanNT * kScanIPT;
    return (int)(ntiles > 0 ? (ntiles + per - 1) / per : 1);
}

cudaError_t launch_partition(int dt, const void *keys, void *out, int n, int h, unsigned long long div,
                             unsigned long long magic, Ctl *ctl, uint32_t *tile_hist, uint32_t *tile_pref,
                             unsigned long long *status, long long *user_off, int plan_mode, int log2c,
                             int sort_tile_keys, int num_sms, bool do_scatter, cudaStream_t st, int key_shift,
                             bool do_count, void *const *dst10) {
    if (dt == 2)  // f3 items (k_kv.cu)
        return launch_partition_t<KV64>(keys, out, n, h, div, magic, ctl, tile_hist, tile_pref, status, user_off,
                                         plan_mode, log2c, sort_tile_keys, num_sms, do_scatter, 0, st, do_count,
                                         nullptr);
    return dt == 0 ? launch_partition_t<int32_t>(keys, out, n, h, div, magic, ctl, tile_hist, tile_pref, status,
                                                 user_off, plan_mode, log2c, sort_tile_keys, num_sms, do_scatter, 0, st,
                                                 do_count, dst10)
                   : launch_partition_t<int64_t>(keys, out, n, h, div, magic, ctl, tile_hist, tile_pref, status,
                                                 user_off, plan_mode, log2c, sort_tile_keys, num_sms, do_scatter,
                                                 key_shift, st, do_count, dst10);
}

}  // namespace hs
