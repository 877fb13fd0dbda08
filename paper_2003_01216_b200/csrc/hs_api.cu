// hs_api.cu -- the C ABI of libhybridsort.so (declared and documented in
// include/hs.h): argument validation, stream-ordered scratch, and the launch
// sequence of each entry point.  Every step of the method runs in the
// kernels of k_partition.cu, k_split.cu, k_tilesort.cu, k_merge.cu and
// k_pairs.cu; this file only sequences them.
//
// HS_SPLIT (compile-time, default 1): the K5a value split of the chunks.
// -DHS_SPLIT=0 builds the A/B variant without it (tools/exp.py); the product
// library has no run-time switch.
#include <cstdarg>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "hs.h"
#include <nvtx3/nvToolsExt.h>
#include "hs_device.cuh"
#include "hs_launch.h"

#ifndef HS_SPLIT
#define HS_SPLIT 1
#endif

namespace {

// NVTX range around every entry point that enqueues work (header-only NVTX3: a
// no-op unless a profiler such as nsys / ncu --nvtx is attached).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define HS_NVTX(name) NvtxRange hs_nvtx_range_(name)

thread_local char g_err[512] = "";
thread_local int g_launches = 0;         // kernels of the last successful call (hs_last_launch_count)
thread_local int g_launch_counter = 0;   // kernels launched so far by the current call

hs_status_t fail(hs_status_t s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
hs_status_t fail(hs_status_t s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

hs_status_t cuda_fail(cudaError_t e, const char *what) {
    return fail(HS_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

using hs::kMaxDevices;
std::once_flag g_dev_once[kMaxDevices];
int g_num_sms[kMaxDevices];

cudaError_t device_setup(int *num_sms) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    cudaError_t err = cudaSuccess;
    std::call_once(g_dev_once[dev], [&]() {
        int sms = 0;
        err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g_num_sms[dev] = sms > 0 ? sms : 148;
        // keep freed scratch in the pool so repeated calls do not remap memory
        cudaMemPool_t pool;
        if (err == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        // kernel attributes and occupancy of the persistent kernels, once per device
        if (err == cudaSuccess) err = hs::setup_partition_kernels(dev);
        if (err == cudaSuccess) err = hs::setup_tilesort_kernels(dev);
        if (err == cudaSuccess) err = hs::setup_merge_kernels(dev);
        if (err == cudaSuccess) err = hs::setup_split_kernels(dev);
        if (err == cudaSuccess) err = hs::setup_kv_kernels(dev);
    });
    if (err != cudaSuccess) return err;
    *num_sms = g_num_sms[dev];
    return cudaSuccess;
}

inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int ksize(hs_dtype_t dt) { return dt == HS_INT32 ? 4 : 8; }

bool overlap(const void *a, const void *b, size_t bytes) {
    uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + bytes && y < x + bytes;
}

// [a, a + na) and [b, b + nb) intersect
bool overlap2(const void *a, size_t na, const void *b, size_t nb) {
    uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

int ceil_log2(long long x) {
    int r = 0;
    while ((1LL << r) < x) ++r;
    return r;
}

hs_status_t check_common(int64_t n, hs_dtype_t dt) {
    if (dt != HS_INT32 && dt != HS_INT64) return fail(HS_ERR_UNSUPPORTED_DTYPE, "dtype %d is not HS_INT32/HS_INT64", (int)dt);
    if (n < 0 || n >= (1LL << 31)) return fail(HS_ERR_INVALID_VALUE, "n = %lld outside [0, 2^31)", (long long)n);
    return HS_OK;
}

hs_status_t check_ptr(const void *p, int64_t n, hs_dtype_t dt, const char *name) {
    if (n > 0 && p == nullptr) return fail(HS_ERR_INVALID_VALUE, "%s is NULL with n > 0", name);
    if (p && ((uintptr_t)p % ksize(dt)) != 0) return fail(HS_ERR_INVALID_VALUE, "%s is not %d-byte aligned", name, ksize(dt));
    return HS_OK;
}

hs_status_t check_digits(int D, hs_dtype_t dt) {
    int hi = dt == HS_INT32 ? 10 : 19;
    if (D < 1 || D > hi) return fail(HS_ERR_INVALID_VALUE, "num_digits = %d outside [1, %d]", D, hi);
    return HS_OK;
}

hs_status_t check_chunks(int c, int *log2c) {
    if (c < 1 || c > 65536 || (c & (c - 1)) != 0)
        return fail(HS_ERR_INVALID_VALUE, "chunks_per_bucket = %d is not a power of two in [1, 65536] (P:80)", c);
    *log2c = ceil_log2(c);
    return HS_OK;
}

hs_status_t check_inout(const void *in, const void *out, int64_t n, hs_dtype_t dt) {
    if (in != out && n > 0 && overlap(in, out, (size_t)n * ksize(dt)))
        return fail(HS_ERR_INVALID_VALUE, "in and out overlap without being equal");
    return HS_OK;
}

// 10^(D-1) and the multiply-high magic floor((2^w - 1) / div) (K1).
// Exact division of a non-negative key u < 2^N (N = w - 1) by div = 10^(D-1):
// with l = ceil(log2 div) and magic = ceil(2^(N+l) / div) (< 2^w, since
// 2^(l-1) < div), floor(u / div) = mulhi_w(u, magic) >> (l - 1) for every such
// u (Granlund & Montgomery 1994, Thm 4.2: 0 <= magic*div - 2^(N+l) < div <= 2^l).
// The post-shift l - 1 is re-derived from div on the device side (div = 1: q = u).
void digit_params(int D, hs_dtype_t dt, unsigned long long *div, unsigned long long *magic) {
    unsigned long long d = 1;
    for (int i = 1; i < D; ++i) d *= 10ull;
    *div = d;
    int l = 0;
    while ((1ull << l) < d) ++l;
    const int N = dt == HS_INT32 ? 31 : 63;
    const unsigned __int128 num = (unsigned __int128)1 << (N + l);
    *magic = d == 1 ? 0ull : (unsigned long long)((num + d - 1) / d);
}

// Scratch for one call, one stream-ordered allocation:
//   [S: n keys][Ctl][K2 lookback status] [K1 tile histograms][K2 tile prefixes][K6 co-ranks]
// Ctl + status are zeroed by one memset.
struct Workspace {
    char *base = nullptr;
    void *S = nullptr;
    hs::Ctl *ctl = nullptr;
    unsigned long long *status = nullptr;
    uint32_t *tile_hist = nullptr;
    uint32_t *tile_pref = nullptr;
    int *corank = nullptr;
    void *samp[2] = {nullptr, nullptr};  // key samples (ping-pong by merge level)
    uint32_t *sbtab = nullptr;           // K5a split table (sub-range starts) and cursors
    uint32_t *sbcur = nullptr;
    void *pad = nullptr;                 // K5a padded layout: one tile-sized region per (chunk, sub-range)
    size_t zero_bytes = 0;
};

hs_status_t ws_alloc(Workspace *w, size_t s_bytes, size_t status_words, size_t ntiles, size_t corank_words,
                     size_t samp_bytes, cudaStream_t st, size_t split_words = 0, size_t pad_bytes = 0) {
    size_t a = round_up(s_bytes, 256) + (s_bytes ? 256 : 0);  // + slack for 16-byte bulk-copy granules
    size_t c = round_up(sizeof(hs::Ctl), 256);
    size_t z = round_up(status_words * 8, 256);
    size_t th = round_up(ntiles * 5 * 4, 256);
    size_t tp = round_up(ntiles * 10 * 4, 256);
    size_t k = round_up(corank_words * 4, 256);
    size_t sp = round_up(samp_bytes, 256);
    size_t sw = round_up(split_words * 4, 256);
    size_t swc = split_words ? round_up((size_t)hs::split_cur_words((long long)split_words) * 4, 256) : 0;
    size_t pb = round_up(pad_bytes, 256);
    size_t total = a + c + z + th + tp + k + 2 * sp + sw + swc + pb;
    void *p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, total, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(HS_ERR_OUT_OF_MEMORY, "cudaMallocAsync(%zu bytes) failed: %s", total, cudaGetErrorString(e));
    }
    char *b = (char *)p;
    w->base = b;
    w->S = s_bytes ? b : nullptr;
    w->ctl = (hs::Ctl *)(b + a);
    w->status = (unsigned long long *)(b + a + c);
    w->tile_hist = (uint32_t *)(b + a + c + z);
    w->tile_pref = (uint32_t *)(b + a + c + z + th);
    w->corank = (int *)(b + a + c + z + th + tp);
    if (samp_bytes) {
        w->samp[0] = b + a + c + z + th + tp + k;
        w->samp[1] = b + a + c + z + th + tp + k + sp;
    }
    if (split_words) {
        w->sbtab = (uint32_t *)(b + a + c + z + th + tp + k + 2 * sp);
        w->sbcur = (uint32_t *)(b + a + c + z + th + tp + k + 2 * sp + sw);
    }
    if (pad_bytes) w->pad = b + a + c + z + th + tp + k + 2 * sp + sw + swc;
    w->zero_bytes = c + z;
    return HS_OK;
}

// One generation of key samples (hs_device.cuh, kSampleQ).
size_t samp_bytes(int64_t n, hs_dtype_t dt) { return (size_t)(n / hs::kSampleQ + 2) * ksize(dt); }

#define HS_TRY_CUDA(expr, what)                                   \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) {                                  \
            if (ws.base) cudaFreeAsync(ws.base, stream);          \
            return cuda_fail(_e, what);                           \
        }                                                         \
    } while (0)

// A successful call: its kernel count becomes hs_last_launch_count().
hs_status_t succeed() {
    g_launches = g_launch_counter;
    g_err[0] = 0;
    return HS_OK;
}

hs_status_t finish(Workspace &ws, cudaStream_t stream) {
    cudaError_t e = cudaFreeAsync(ws.base, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
    return succeed();
}

// Merge levels the host must launch: each bucket runs L[b] <= this many
// (k[b] <= ceil(log2(ceil(ceil(n/c)/T)))); levels with no active bucket
// cost one near-empty launch pair.
int level_bound(long long n, int log2c, int T, int with_tiles, int with_tree) {
    int k = 0;
    if (with_tiles) {
        long long c = 1LL << log2c;
        long long cm = (n + c - 1) / c;
        long long t = (cm + T - 1) / T;
        k = t > 1 ? ceil_log2(t) : 0;
    }
    return k + (with_tree ? log2c : 0);
}

long long tile_bound(long long n, long long c, int T) { return 2 * ((n + T - 1) / T) + 50 * c; }

// ------------------------------------------------------------- profiling
struct ProfRec {
    int kind;
    cudaEvent_t a, b;
};
thread_local bool g_prof_on = false;
thread_local std::vector<ProfRec> g_prof_recs;
thread_local std::vector<cudaEvent_t> g_prof_pool;
thread_local cudaEvent_t g_prof_open = nullptr;

cudaEvent_t prof_event() {
    if (!g_prof_pool.empty()) {
        cudaEvent_t e = g_prof_pool.back();
        g_prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

const char *const kProfNames[hs::kProfKinds] = {"tile_hist", "tile_scan", "scatter", "plan",
                                                 "tile_sort", "merge_partition", "merge_level", "copy",
                                                 "split_count", "split_scatter"};

}  // namespace

namespace hs {
void note_launch() { ++g_launch_counter; }

void prof_begin(int kind, cudaStream_t st) {
    (void)kind;
    if (!g_prof_on) return;
    g_prof_open = prof_event();
    cudaEventRecord(g_prof_open, st);
}
void prof_end(int kind, cudaStream_t st) {
    if (!g_prof_on || !g_prof_open) return;
    cudaEvent_t b = prof_event();
    cudaEventRecord(b, st);
    g_prof_recs.push_back({kind, g_prof_open, b});
    g_prof_open = nullptr;
}
}  // namespace hs

extern "C" {

int hs_profile_enable(int on) {
    g_prof_on = on != 0;
    return 0;
}

int hs_profile_read(double *ms, int *count, int nkinds) {
    for (int k = 0; k < nkinds; ++k) {
        if (ms) ms[k] = 0.0;
        if (count) count[k] = 0;
    }
    int rc = 0;
    for (const ProfRec &r : g_prof_recs) {
        float t = 0.f;
        if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) rc = -1;
        if (r.kind >= 0 && r.kind < nkinds) {
            if (ms) ms[r.kind] += t;
            if (count) count[r.kind] += 1;
        }
        g_prof_pool.push_back(r.a);
        g_prof_pool.push_back(r.b);
    }
    g_prof_recs.clear();
    return rc;
}

const char *hs_profile_kind_name(int kind) { return (kind >= 0 && kind < hs::kProfKinds) ? kProfNames[kind] : ""; }

int hs_plan_levels(const int64_t *bucket_offsets_host, hs_dtype_t dtype, int chunks_per_bucket, int mode,
                   int *levels_out, int *tile_levels_out) {
    if (dtype != HS_INT32 && dtype != HS_INT64) return -1;
    int log2c;
    if (check_chunks(chunks_per_bucket, &log2c) != HS_OK) return -1;
    const long long c = 1LL << log2c;
    const long long T = hs::sort_tile_keys((int)dtype);
    int lmax = 0;
    for (int b = 0; b < 10; ++b) {
        const long long m = bucket_offsets_host[b + 1] - bucket_offsets_host[b];
        int k = 0;
        if (mode != hs::kPlanMerge) {
            const long long cm = (m + c - 1) / c;
            const long long tiles = (cm + T - 1) / T;
            k = tiles > 1 ? ceil_log2(tiles) : 0;
        }
        const int L = mode == hs::kPlanSort ? k + log2c : (mode == hs::kPlanChunks ? k : log2c);
        if (levels_out) levels_out[b] = L;
        if (tile_levels_out) tile_levels_out[b] = k;
        lmax = L > lmax ? L : lmax;
    }
    return lmax;
}

hs_status_t hs_assign_buckets(const int64_t *bucket_sizes, int nodes, int *group_start, int64_t *max_load) {
    if (!bucket_sizes || !group_start) return fail(HS_ERR_INVALID_VALUE, "NULL argument");
    if (nodes < 1 || nodes > 10) return fail(HS_ERR_INVALID_VALUE, "nodes = %d outside [1, 10] (S:310)", nodes);
    for (int d = 0; d < 10; ++d)
        if (bucket_sizes[d] < 0) return fail(HS_ERR_INVALID_VALUE, "bucket_sizes[%d] < 0", d);
    // Split points s_1 < ... < s_{m-1} in [1, 9], enumerated in lexicographic
    // order (first ascending), so the first strict improvement found wins ties.
    int cut[10], best[10];
    long long best_load = -1;
    const int m = nodes;
    for (int i = 0; i < m - 1; ++i) cut[i] = i + 1;
    for (;;) {
        long long load = 0;
        int lo = 0;
        for (int g = 0; g < m; ++g) {
            const int hi = g < m - 1 ? cut[g] : 10;
            long long t = 0;
            for (int d = lo; d < hi; ++d) t += bucket_sizes[d];
            load = t > load ? t : load;
            lo = hi;
        }
        if (best_load < 0 || load < best_load) {
            best_load = load;
            for (int i = 0; i < m - 1; ++i) best[i] = cut[i];
        }
        // next combination of m-1 cut positions out of 1..9
        int i = m - 2;
        while (i >= 0 && cut[i] == 9 - (m - 2 - i)) --i;
        if (i < 0) break;
        ++cut[i];
        for (int j = i + 1; j < m - 1; ++j) cut[j] = cut[j - 1] + 1;
    }
    group_start[0] = 0;
    for (int i = 0; i < m - 1; ++i) group_start[i + 1] = best[i];
    group_start[m] = 10;
    if (max_load) *max_load = best_load;
    g_err[0] = 0;
    return HS_OK;
}

const char *hs_status_string(hs_status_t s) {
    switch (s) {
        case HS_OK: return "HS_OK";
        case HS_ERR_INVALID_VALUE: return "HS_ERR_INVALID_VALUE";
        case HS_ERR_UNSUPPORTED_DTYPE: return "HS_ERR_UNSUPPORTED_DTYPE";
        case HS_ERR_OUT_OF_MEMORY: return "HS_ERR_OUT_OF_MEMORY";
        case HS_ERR_CUDA: return "HS_ERR_CUDA";
    }
    return "HS_ERR_UNKNOWN";
}

const char *hs_last_error_message(void) { return g_err; }
int hs_abi_version(void) { return HS_ABI_VERSION; }
int hs_last_launch_count(void) { return g_launches; }

int hs_tile_keys(hs_dtype_t dtype, int which) {
    if (dtype != HS_INT32 && dtype != HS_INT64) return 0;
    const int dt = (int)dtype;
    if (which == 3) return hs::kv_tile_keys();  // tile-sort capacity of the f3 item path (either key dtype)
    return which == 0 ? hs::scatter_tile_keys(dt) : which == 1 ? hs::sort_tile_keys(dt) : hs::merge_span(dt);
}

}  // extern "C"

namespace {

// a1-a3 on validated arguments.  key_shift: int64 items whose key is k >> 32.
hs_status_t partition_impl(const void *keys, int64_t n, hs_dtype_t dtype, int num_digits, int key_shift,
                           int64_t *bucket_offsets, void *out, cudaStream_t stream) {
    hs_status_t s;
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");

    const int dt = (int)dtype;
    const int Tp = hs::scatter_tile_keys(dt);
    const int h = (int)(((uintptr_t)keys % 16) / ksize(dtype));
    const long long tiles = (n + h + Tp - 1) / Tp;
    unsigned long long div, magic;
    digit_params(num_digits, dtype, &div, &magic);

    Workspace ws;
    if ((s = ws_alloc(&ws, 0, (size_t)hs::scan_ctas(tiles) * 10, (size_t)tiles, 0, 0, stream)) != HS_OK) return s;
    HS_TRY_CUDA(cudaMemsetAsync(ws.ctl, 0, ws.zero_bytes, stream), "memset control block");
    HS_TRY_CUDA(hs::launch_partition(dt, keys, out, (int)n, h, div, magic, ws.ctl, ws.tile_hist, ws.tile_pref, ws.status,
                                     (long long *)bucket_offsets, -1, 0, 0, sms, true, stream, key_shift),
                "K1-K3 partition");
    cudaError_t fe = cudaFreeAsync(ws.base, stream);
    if (fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
    return HS_OK;
}

}  // namespace

extern "C" {

hs_status_t hs_msd_partition(const void *keys, int64_t n, hs_dtype_t dtype, int num_digits, int64_t *bucket_offsets,
                             void *out, cudaStream_t stream) {
    HS_NVTX("hs_msd_partition");
    hs_status_t s;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_digits(num_digits, dtype)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, dtype, "keys")) != HS_OK) return s;
    if ((s = check_ptr(out, n, dtype, "out")) != HS_OK) return s;
    if (!bucket_offsets) return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL");
    if (((uintptr_t)bucket_offsets & 7) != 0) return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is not 8-byte aligned");
    if (n > 0 && overlap(keys, out, (size_t)n * ksize(dtype)))
        return fail(HS_ERR_INVALID_VALUE, "keys and out overlap (the partition is out of place)");
    g_launch_counter = 0;
    if ((s = partition_impl(keys, n, dtype, num_digits, 0, bucket_offsets, out, stream)) != HS_OK) return s;
    return succeed();
}

}  // extern "C"

namespace {

// CUDA-graph capture: the side stream a conditional node's body is captured on
// (one per host thread and device, created by an uncaptured call -- creating a
// stream inside a global-mode capture is not allowed), or null when `stream` is
// not capturing / no side stream exists yet (the caller then launches directly).
cudaStream_t capture_side_stream(cudaStream_t stream) {
    static thread_local cudaStream_t side[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (cs == cudaStreamCaptureStatusNone) {
        if (!side[dev] && cudaStreamCreateWithFlags(&side[dev], cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            side[dev] = nullptr;
        }
        return nullptr;
    }
    return cs == cudaStreamCaptureStatusActive ? side[dev] : nullptr;
}

// In the graph `stream` is capturing: a k_level_gate node (plan Lmax > lv), then an IF node whose
// body -- captured on `side` by body(side) -- runs only when the gate opened it.
template <typename Body>
cudaError_t gated_levels(cudaStream_t stream, cudaStream_t side, const hs::Plan *plan, int lv, Body body) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    cudaError_t e = cudaStreamGetCaptureInfo(stream, &cs, nullptr, &g, &deps, &nd);
    if (e != cudaSuccess) return e;
    cudaGraphConditionalHandle h;
    if ((e = cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault)) != cudaSuccess) return e;
    if ((e = hs::launch_level_gate((unsigned long long)h, plan, lv, stream)) != cudaSuccess) return e;
    if ((e = cudaStreamGetCaptureInfo(stream, &cs, nullptr, &g, &deps, &nd)) != cudaSuccess) return e;
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    if ((e = cudaGraphAddNode(&node, g, deps, nd, &p)) != cudaSuccess) return e;
    if ((e = cudaStreamUpdateCaptureDependencies(stream, &node, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
        return e;
    if ((e = cudaStreamBeginCaptureToGraph(side, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed)) != cudaSuccess)
        return e;
    const cudaError_t eb = body(side);
    cudaGraph_t out = nullptr;
    e = cudaStreamEndCapture(side, &out);
    return eb != cudaSuccess ? eb : e;
}

// a1-a7 on validated arguments (n > 0).  key_shift as partition_impl.
// user_off (device int64[11], hs_sort_buckets): keys are already partitioned by
// digit into those buckets -- a1-a3 are skipped, the plan comes from user_off,
// the split reads keys and writes the scratch, the tile sort reads both.
hs_status_t sort_impl(void *keys, int64_t n, hs_dtype_t dtype, int num_digits, int key_shift, int chunks_per_bucket,
                      int log2c, cudaStream_t stream, hs::Ctl *inspect = nullptr,
                      const int64_t *user_off = nullptr) {
    hs_status_t s;
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");

    const int dt = (int)dtype;
    const int Tp = hs::scatter_tile_keys(dt), T = hs::sort_tile_keys(dt), TM = hs::merge_span(dt);
    const int h = (int)(((uintptr_t)keys % 16) / ksize(dtype));
    const long long ptiles = (n + h + Tp - 1) / Tp;
    const long long nblocks = (n + TM - 1) / TM;
    unsigned long long div, magic;
    digit_params(num_digits, key_shift ? HS_INT64 : dtype, &div, &magic);

    // K5a value split of the chunks (compile-time HS_SPLIT, see the top of this file)
    // No chunk can exceed one tile when ceil(n / c) <= T (a bucket holds at most n keys), so no bucket
    // can take the split: its kernels are not launched at all (small n: launch-bound).
    const bool split_on = HS_SPLIT != 0 && (n + (1LL << log2c) - 1) / (1LL << log2c) > T;
    const long long split_words = split_on ? hs::split_table_words(n, log2c, T) : 0;
    const long long pad_keys = split_on ? hs::split_pad_keys(n, log2c, T) : 0;
    Workspace ws;
    if ((s = ws_alloc(&ws, (size_t)n * ksize(dtype) * (inspect ? 2 : 1), (size_t)hs::scan_ctas(ptiles) * 10,
                      (size_t)ptiles, (size_t)nblocks + 2, samp_bytes(n, dtype), stream, (size_t)split_words,
                      (size_t)pad_keys * ksize(dtype))) != HS_OK)
        return s;
    if (inspect) {  // hs_sort_plan: partition + split into scratch, read the plan back
        void *F = (char *)ws.S + round_up((size_t)n * ksize(dtype), 256);
        cudaError_t e2 = cudaMemsetAsync(ws.ctl, 0, ws.zero_bytes, stream);
        if (e2 == cudaSuccess)
            e2 = hs::launch_partition(dt, keys, ws.S, (int)n, h, div, magic, ws.ctl, ws.tile_hist, ws.tile_pref,
                                      ws.status, nullptr, hs::kPlanSort, log2c, T, sms, true, stream, key_shift);
        if (e2 == cudaSuccess && split_on)
            e2 = hs::launch_split(dt, ws.ctl, ws.S, F, ws.sbtab, ws.sbcur, split_words, n, log2c, T, div, key_shift,
                                  F, ws.pad, pad_keys, stream);
        if (e2 == cudaSuccess) e2 = cudaMemcpyAsync(inspect, ws.ctl, sizeof(hs::Ctl), cudaMemcpyDeviceToHost, stream);
        cudaError_t fe = cudaFreeAsync(ws.base, stream);
        if (e2 == cudaSuccess) e2 = fe;
        if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(stream);
        if (e2 != cudaSuccess) return cuda_fail(e2, "hs_sort_plan");
        return HS_OK;
    }
    const hs::Plan *plan = &ws.ctl->plan;
    HS_TRY_CUDA(cudaMemsetAsync(ws.ctl, 0, ws.zero_bytes, stream), "memset control block");
    // where the partitioned keys are (part) and where the split writes (spl)
    void *part = ws.S, *spl = keys;
    if (user_off) {
        // a4: plan from the caller's bucket offsets (keys already partitioned)
        HS_TRY_CUDA(hs::launch_plan((const long long *)user_off, ws.ctl, log2c, hs::kPlanSort, T, stream), "K4 plan");
        part = keys;
        spl = ws.S;
    } else {
        // a1-a3: tile histograms, lookback prefix (+ offsets + plan), stable scatter keys -> S
        HS_TRY_CUDA(hs::launch_partition(dt, keys, ws.S, (int)n, h, div, magic, ws.ctl, ws.tile_hist, ws.tile_pref,
                                         ws.status, nullptr, hs::kPlanSort, log2c, T, sms, true, stream, key_shift),
                    "K1-K3 partition");
    }
    // a5 (K5a): value split of every chunk that exceeds one tile, part -> spl
    // (constant pieces -- one key throughout, longer than the tile sort takes -- are filled straight
    // into the tile sort's output buffer of split buckets: S for an odd number of chunk rounds)
    void *const tile_out = (log2c & 1) ? ws.S : keys;
    if (split_on)
        HS_TRY_CUDA(hs::launch_split(dt, ws.ctl, part, spl, ws.sbtab, ws.sbcur, split_words, n, log2c, T, div,
                                     key_shift, tile_out, ws.pad, pad_keys, stream),
                    "K5a split");
    // a5: leaf-tile sort (part, or spl for split buckets) -> (keys | S) per bucket parity
    HS_TRY_CUDA(hs::launch_tile_sort(dt, plan, part, keys, ws.S, ws.samp[0], tile_bound(n, chunks_per_bucket, T), stream,
                                     ws.sbtab, &ws.ctl->split, spl,
                                     split_on ? hs::split_cflag(ws.sbcur, split_words) : nullptr, ws.pad),
                "K5 tile sort");
    // a5 (in-chunk levels) + a6 (tree merge of chunks): ping-pong, last level lands in keys.
    // Every plan runs the log2 c tree levels (L[b] = k[b] + log2 c); the host only knows a bound on
    // the rest (fallback buckets' in-chunk levels).  Under CUDA-graph capture those sit behind a
    // conditional node the device plan opens (k_level_gate); otherwise they are launched and exit
    // at once when the plan has no bucket there.
    const int L = level_bound(n, log2c, T, 1, 1);
    const int Lsure = L < log2c ? L : log2c;
    auto level = [&](int lv, cudaStream_t st) {
        return hs::launch_merge_level(dt, plan, keys, ws.S, nullptr, ws.corank, ws.samp[lv & 1],
                                      lv + 1 < L ? ws.samp[(lv + 1) & 1] : nullptr, lv, (int)n, sms, st);
    };
    for (int lv = 0; lv < Lsure; ++lv) HS_TRY_CUDA(level(lv, stream), "K6 merge level");
    if (L > Lsure) {
        cudaStream_t side = capture_side_stream(stream);
        if (side) {
            HS_TRY_CUDA(gated_levels(stream, side, plan, Lsure, [&](cudaStream_t st) -> cudaError_t {
                            for (int lv = Lsure; lv < L; ++lv) {
                                const cudaError_t e = level(lv, st);
                                if (e != cudaSuccess) return e;
                            }
                            return cudaSuccess;
                        }),
                        "K6 gated merge levels");
        } else {
            for (int lv = Lsure; lv < L; ++lv) HS_TRY_CUDA(level(lv, stream), "K6 merge level");
        }
    }
    cudaError_t fe = cudaFreeAsync(ws.base, stream);
    if (fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
    return HS_OK;
}


}  // namespace

extern "C" {

hs_status_t hs_sort(void *keys, int64_t n, hs_dtype_t dtype, int num_digits, int chunks_per_bucket,
                    cudaStream_t stream) {
    HS_NVTX("hs_sort");
    hs_status_t s;
    int log2c;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_digits(num_digits, dtype)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, dtype, "keys")) != HS_OK) return s;
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    g_launch_counter = 0;
    if ((s = sort_impl(keys, n, dtype, num_digits, 0, chunks_per_bucket, log2c, stream)) != HS_OK) return s;
    return succeed();
}

hs_status_t hs_sort_buckets(void *keys, int64_t n, hs_dtype_t dtype, int num_digits, const int64_t *bucket_offsets,
                            int chunks_per_bucket, cudaStream_t stream) {
    HS_NVTX("hs_sort_buckets");
    hs_status_t s;
    int log2c;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_digits(num_digits, dtype)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, dtype, "keys")) != HS_OK) return s;
    if (!bucket_offsets || ((uintptr_t)bucket_offsets & 7) != 0)
        return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL or not 8-byte aligned");
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    g_launch_counter = 0;
    if ((s = sort_impl(keys, n, dtype, num_digits, 0, chunks_per_bucket, log2c, stream, nullptr, bucket_offsets)) !=
        HS_OK)
        return s;
    return succeed();
}

hs_status_t hs_sort_plan(const void *keys, int64_t n, hs_dtype_t dtype, int num_digits, int chunks_per_bucket,
                         int32_t *levels_out, int32_t *split_out, int32_t *leaves_out, cudaStream_t stream) {
    HS_NVTX("hs_sort_plan");
    hs_status_t s;
    int log2c;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_digits(num_digits, dtype)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, dtype, "keys")) != HS_OK) return s;
    if (!levels_out || !split_out || !leaves_out) return fail(HS_ERR_INVALID_VALUE, "output array is NULL");
    hs::Ctl X;
    memset(&X, 0, sizeof(X));
    const hs::Plan &P = X.plan;
    if (n > 0) {
        g_launch_counter = 0;
        if ((s = sort_impl(const_cast<void *>(keys), n, dtype, num_digits, 0, chunks_per_bucket, log2c, stream, &X)) !=
            HS_OK)
            return s;
    }
    for (int b = 0; b < 10; ++b) {
        levels_out[b] = n > 0 ? P.L[b] : 0;
        split_out[b] = P.split[b] ? (hs::split_pmode(X.split, b) ? 2 : 1) : 0;
        leaves_out[b] = P.split[b] ? P.nsb[b] : (1 << P.k[b]);
    }
    g_launches = 0;
    g_err[0] = 0;
    return HS_OK;
}

struct hs_partition_plan_s {
    const void *keys;
    int64_t n;
    hs_dtype_t dtype;
    int h;
    unsigned long long div, magic;
    int sms;
    Workspace ws;
};

hs_status_t hs_partition_plan_create(const void *keys, int64_t n, hs_dtype_t dtype, int num_digits,
                                     int64_t *bucket_offsets, hs_partition_plan_t *plan, cudaStream_t stream) {
    HS_NVTX("hs_partition_plan_create");
    hs_status_t s;
    if (!plan) return fail(HS_ERR_INVALID_VALUE, "plan is NULL");
    *plan = nullptr;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_digits(num_digits, dtype)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, dtype, "keys")) != HS_OK) return s;
    if (!bucket_offsets || ((uintptr_t)bucket_offsets & 7) != 0)
        return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL or not 8-byte aligned");
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    g_launch_counter = 0;
    hs_partition_plan_s *p = new hs_partition_plan_s();
    p->keys = keys;
    p->n = n;
    p->dtype = dtype;
    p->sms = sms;
    const int dt = (int)dtype;
    const int Tp = hs::scatter_tile_keys(dt);
    p->h = (int)(((uintptr_t)keys % 16) / ksize(dtype));
    const long long tiles = (n + p->h + Tp - 1) / Tp;
    digit_params(num_digits, dtype, &p->div, &p->magic);
    if ((s = ws_alloc(&p->ws, 0, (size_t)hs::scan_ctas(tiles) * 10, (size_t)tiles, 0, 0, stream)) != HS_OK) {
        delete p;
        return s;
    }
    Workspace &ws = p->ws;
    if ((e = cudaMemsetAsync(ws.ctl, 0, ws.zero_bytes, stream)) != cudaSuccess ||
        (e = hs::launch_partition(dt, keys, nullptr, (int)n, p->h, p->div, p->magic, ws.ctl, ws.tile_hist, ws.tile_pref,
                                  ws.status, (long long *)bucket_offsets, -1, 0, 0, sms, false, stream)) != cudaSuccess) {
        cudaFreeAsync(ws.base, stream);
        delete p;
        return cuda_fail(e, "K1-K2 count");
    }
    *plan = p;
    return succeed();
}

hs_status_t hs_partition_scatter(hs_partition_plan_t plan, void *const *dst, cudaStream_t stream) {
    HS_NVTX("hs_partition_scatter");
    if (!plan || !dst) return fail(HS_ERR_INVALID_VALUE, "plan or dst is NULL");
    const int ks = ksize(plan->dtype);
    for (int d = 0; d < 10; ++d)
        if (dst[d] && ((uintptr_t)dst[d] % ks) != 0)
            return fail(HS_ERR_INVALID_VALUE, "dst[%d] is not %d-byte aligned", d, ks);
    Workspace &ws = plan->ws;
    g_launch_counter = 0;
    cudaError_t e = hs::launch_partition((int)plan->dtype, plan->keys, nullptr, (int)plan->n, plan->h, plan->div,
                                         plan->magic, ws.ctl, ws.tile_hist, ws.tile_pref, ws.status, nullptr, -1, 0, 0,
                                         plan->sms, true, stream, 0, false, dst);
    if (e != cudaSuccess) return cuda_fail(e, "K3 scatter");
    return succeed();
}

hs_status_t hs_partition_plan_destroy(hs_partition_plan_t plan, cudaStream_t stream) {
    if (!plan) return HS_OK;
    cudaError_t e = cudaFreeAsync(plan->ws.base, stream);
    delete plan;
    if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
    return HS_OK;
}

hs_status_t hs_msd_partition_pairs(const int32_t *keys, const uint64_t *tags, int64_t n, int num_digits,
                                   int64_t *bucket_offsets, int32_t *out_keys, uint64_t *out_tags,
                                   cudaStream_t stream) {
    HS_NVTX("hs_msd_partition_pairs");
    hs_status_t s;
    if ((s = check_common(n, HS_INT32)) != HS_OK) return s;
    if ((s = check_digits(num_digits, HS_INT32)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, HS_INT32, "keys")) != HS_OK) return s;
    if ((s = check_ptr(out_keys, n, HS_INT32, "out_keys")) != HS_OK) return s;
    if ((s = check_ptr(tags, n, HS_INT64, "tags")) != HS_OK) return s;
    if ((s = check_ptr(out_tags, n, HS_INT64, "out_tags")) != HS_OK) return s;
    if (!bucket_offsets || ((uintptr_t)bucket_offsets & 7) != 0)
        return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL or not 8-byte aligned");
    if (n > 0 && (overlap(keys, out_keys, (size_t)n * 4) || overlap(tags, out_tags, (size_t)n * 8)))
        return fail(HS_ERR_INVALID_VALUE, "inputs and outputs overlap (the partition is out of place)");
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    void *buf = nullptr;
    const size_t ib = (size_t)(n > 0 ? n : 1) * 8;
    if ((e = cudaMallocAsync(&buf, 2 * ib + 256, stream)) != cudaSuccess) {
        cudaGetLastError();
        return fail(HS_ERR_OUT_OF_MEMORY, "cudaMallocAsync(%zu bytes) failed", 2 * ib + 256);
    }
    long long *items = (long long *)buf, *parted = (long long *)((char *)buf + round_up(ib, 256));
    g_launch_counter = 0;
    if ((e = hs::launch_pack_items(keys, items, n, sms, stream)) != cudaSuccess) {
        cudaFreeAsync(buf, stream);
        return cuda_fail(e, "K0 pack items");
    }
    if ((s = partition_impl(items, n, HS_INT64, num_digits, 32, bucket_offsets, parted, stream)) != HS_OK) {
        cudaFreeAsync(buf, stream);
        return s;
    }
    if ((e = hs::launch_unpack_items(parted, out_keys, (const unsigned long long *)tags,
                                     (unsigned long long *)out_tags, n, sms, stream)) != cudaSuccess) {
        cudaFreeAsync(buf, stream);
        return cuda_fail(e, "K8 unpack items");
    }
    if ((e = cudaFreeAsync(buf, stream)) != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
    return succeed();
}

hs_status_t hs_sort_pairs(int32_t *keys, uint64_t *tags, int64_t n, int num_digits, int chunks_per_bucket,
                          cudaStream_t stream) {
    HS_NVTX("hs_sort_pairs");
    hs_status_t s;
    int log2c;
    if ((s = check_common(n, HS_INT32)) != HS_OK) return s;
    if ((s = check_digits(num_digits, HS_INT32)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, HS_INT32, "keys")) != HS_OK) return s;
    if ((s = check_ptr(tags, n, HS_INT64, "tags")) != HS_OK) return s;
    if (n > 0 && overlap2(keys, (size_t)n * 4, tags, (size_t)n * 8))
        return fail(HS_ERR_INVALID_VALUE, "keys and tags overlap");
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    void *buf = nullptr;
    const size_t ib = round_up((size_t)n * 8, 256);
    if ((e = cudaMallocAsync(&buf, 2 * ib, stream)) != cudaSuccess) {
        cudaGetLastError();
        return fail(HS_ERR_OUT_OF_MEMORY, "cudaMallocAsync(%zu bytes) failed", 2 * ib);
    }
    long long *items = (long long *)buf;
    unsigned long long *tag_copy = (unsigned long long *)((char *)buf + ib);
    g_launch_counter = 0;
    if ((e = hs::launch_pack_items(keys, items, n, sms, stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(tag_copy, tags, (size_t)n * 8, cudaMemcpyDeviceToDevice, stream)) != cudaSuccess) {
        cudaFreeAsync(buf, stream);
        return cuda_fail(e, "K0 pack items / tag copy");
    }
    if ((s = sort_impl(items, n, HS_INT64, num_digits, 32, chunks_per_bucket, log2c, stream)) != HS_OK) {
        cudaFreeAsync(buf, stream);
        return s;
    }
    if ((e = hs::launch_unpack_items(items, keys, tag_copy, (unsigned long long *)tags, n, sms, stream)) !=
        cudaSuccess) {
        cudaFreeAsync(buf, stream);
        return cuda_fail(e, "K8 unpack items");
    }
    if ((e = cudaFreeAsync(buf, stream)) != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
    return succeed();
}

hs_status_t hs_sort_shared(void *keys, int64_t n, hs_dtype_t dtype, int chunks, cudaStream_t stream) {
    HS_NVTX("hs_sort_shared");
    hs_status_t s;
    int log2c;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_chunks(chunks, &log2c)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, dtype, "keys")) != HS_OK) return s;
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    const int dt = (int)dtype;
    const int T = hs::sort_tile_keys(dt), TM = hs::merge_span(dt);
    const long long nblocks = (n + TM - 1) / TM;
    Workspace ws;
    if ((s = ws_alloc(&ws, (size_t)n * ksize(dtype), 0, 0, (size_t)nblocks + 2, samp_bytes(n, dtype), stream)) != HS_OK)
        return s;
    g_launch_counter = 0;
    const hs::Plan *plan = &ws.ctl->plan;
    HS_TRY_CUDA(hs::launch_plan_whole(n, ws.ctl, log2c, T, stream), "K4 plan");
    // chunk sort: leaf tiles keys -> (keys | S) by parity, in place per leaf
    HS_TRY_CUDA(hs::launch_tile_sort(dt, plan, keys, keys, ws.S, ws.samp[0], tile_bound(n, chunks, T), stream),
                "K5 tile sort");
    const int L = level_bound(n, log2c, T, 1, 1);  // exact: the one segment is the whole array
    for (int lv = 0; lv < L; ++lv) {
        HS_TRY_CUDA(hs::launch_merge_level(dt, plan, keys, ws.S, nullptr, ws.corank, ws.samp[lv & 1],
                                           lv + 1 < L ? ws.samp[(lv + 1) & 1] : nullptr, lv, (int)n, sms, stream),
                    "K6 merge level");
    }
    return finish(ws, stream);
}

hs_status_t hs_sort_chunks(const void *in, void *out, int64_t n, hs_dtype_t dtype, const int64_t *bucket_offsets,
                           int chunks_per_bucket, cudaStream_t stream) {
    HS_NVTX("hs_sort_chunks");
    hs_status_t s;
    int log2c;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if ((s = check_ptr(in, n, dtype, "in")) != HS_OK) return s;
    if ((s = check_ptr(out, n, dtype, "out")) != HS_OK) return s;
    if (!bucket_offsets) return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL");
    if ((s = check_inout(in, out, n, dtype)) != HS_OK) return s;
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    const int dt = (int)dtype;
    const int T = hs::sort_tile_keys(dt), TM = hs::merge_span(dt);
    const long long nblocks = (n + TM - 1) / TM;

    Workspace ws;
    if ((s = ws_alloc(&ws, (size_t)n * ksize(dtype), 0, 0, (size_t)nblocks + 2, samp_bytes(n, dtype), stream)) != HS_OK)
        return s;
    g_launch_counter = 0;
    const hs::Plan *plan = &ws.ctl->plan;
    HS_TRY_CUDA(hs::launch_plan((const long long *)bucket_offsets, ws.ctl, log2c, hs::kPlanChunks, T, stream), "K4 plan");
    HS_TRY_CUDA(hs::launch_tile_sort(dt, plan, in, out, ws.S, ws.samp[0], tile_bound(n, chunks_per_bucket, T), stream),
                "K5 tile sort");
    const int L = level_bound(n, log2c, T, 1, 0);
    for (int lv = 0; lv < L; ++lv) {
        HS_TRY_CUDA(hs::launch_merge_level(dt, plan, out, ws.S, nullptr, ws.corank, ws.samp[lv & 1],
                                           lv + 1 < L ? ws.samp[(lv + 1) & 1] : nullptr, lv, (int)n, sms, stream),
                    "K6 merge level");
    }
    return finish(ws, stream);
}

hs_status_t hs_merge(const void *in, void *out, int64_t n, hs_dtype_t dtype, const int64_t *bucket_offsets,
                     int chunks_per_bucket, cudaStream_t stream) {
    HS_NVTX("hs_merge");
    hs_status_t s;
    int log2c;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if ((s = check_ptr(in, n, dtype, "in")) != HS_OK) return s;
    if ((s = check_ptr(out, n, dtype, "out")) != HS_OK) return s;
    if (!bucket_offsets) return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL");
    if ((s = check_inout(in, out, n, dtype)) != HS_OK) return s;
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    const int dt = (int)dtype;
    const int TM = hs::merge_span(dt);
    const long long nblocks = (n + TM - 1) / TM;
    g_launch_counter = 0;
    Workspace ws;
    if (log2c == 0) {  // c = 1: zero rounds, out = in
        if (in != out) HS_TRY_CUDA(hs::launch_copy(dt, in, out, n, sms, stream), "K7 copy");
        return succeed();
    }
    if ((s = ws_alloc(&ws, (size_t)n * ksize(dtype), 0, 0, (size_t)nblocks + 2, samp_bytes(n, dtype), stream)) !=
        HS_OK)
        return s;
    const hs::Plan *plan = &ws.ctl->plan;
    HS_TRY_CUDA(hs::launch_plan((const long long *)bucket_offsets, ws.ctl, log2c, hs::kPlanMerge, 1, stream), "K4 plan");
    HS_TRY_CUDA(hs::launch_sample(dt, in, ws.samp[0], n, sms, stream), "K6 sample");
    const void *src0 = in;
    if (in == out) {
        src0 = nullptr;
        // level 0 must read the buffer its parity names: S when the round
        // count is odd, so the in-place case starts with one copy (K7).
        if (log2c & 1) HS_TRY_CUDA(hs::launch_copy(dt, in, ws.S, n, sms, stream), "K7 copy");
    }
    for (int lv = 0; lv < log2c; ++lv) {
        HS_TRY_CUDA(hs::launch_merge_level(dt, plan, out, ws.S, src0, ws.corank, ws.samp[lv & 1],
                                           lv + 1 < log2c ? ws.samp[(lv + 1) & 1] : nullptr, lv, (int)n, sms, stream),
                    "K6 merge level");
    }
    return finish(ws, stream);
}

}  // extern "C"

namespace {

// f3 on KV64 items (k_kv.cu), in place on `items` (16-byte aligned scratch):
//   kPlanSort:   a1-a3 (stable K3 on items) + a5 (stable tile sort + in-chunk levels) + a6 (tree levels)
//   kPlanChunks: a5 only, chunks of the caller's bucket_offsets
//   kPlanMerge:  a6 only, the caller's chunk-sorted runs
// Every step is stable (k_kv.cu), so equal keys keep their input order.
hs_status_t kv_impl(hs::KV64 *items, int64_t n, int num_digits, int log2c, int mode, const int64_t *user_off,
                    int64_t *off_out, cudaStream_t stream) {
    hs_status_t s;
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    constexpr int dt = 2;  // KV64
    const int Tp = hs::scatter_tile_keys(dt), T = hs::kv_tile_keys(), TM = hs::merge_span(dt);
    const long long ptiles = mode == hs::kPlanSort ? (n + Tp - 1) / Tp : 0;
    const long long nblocks = (n + TM - 1) / TM;
    unsigned long long div, magic;
    digit_params(num_digits, HS_INT64, &div, &magic);
    const int c = 1 << log2c;
    Workspace ws;
    if ((s = ws_alloc(&ws, (size_t)n * sizeof(hs::KV64), (size_t)hs::scan_ctas(ptiles) * 10, (size_t)ptiles,
                      (size_t)nblocks + 2, (size_t)(n / hs::kSampleQ + 2) * sizeof(hs::KV64), stream)) != HS_OK)
        return s;
    const hs::Plan *plan = &ws.ctl->plan;
    hs::KV64 *S = (hs::KV64 *)ws.S;
    HS_TRY_CUDA(cudaMemsetAsync(ws.ctl, 0, ws.zero_bytes, stream), "memset control block");
    int L = 0;
    if (mode == hs::kPlanSort) {
        // a1-a3: stable counting scatter of the items by the leading digit of their key, items -> S
        HS_TRY_CUDA(hs::launch_partition(dt, items, S, (int)n, 0, div, magic, ws.ctl, ws.tile_hist, ws.tile_pref,
                                         ws.status, (long long *)off_out, hs::kPlanSort, log2c, T, sms, true, stream),
                    "K1-K3 partition (items)");
        HS_TRY_CUDA(hs::launch_tile_sort_kv(plan, S, items, S, (hs::KV64 *)ws.samp[0], tile_bound(n, c, T), stream),
                    "K5kv tile sort");
        L = level_bound(n, log2c, T, 1, 1);
    } else if (mode == hs::kPlanChunks) {
        HS_TRY_CUDA(hs::launch_plan((const long long *)user_off, ws.ctl, log2c, hs::kPlanChunks, T, stream), "K4 plan");
        HS_TRY_CUDA(hs::launch_tile_sort_kv(plan, items, items, S, (hs::KV64 *)ws.samp[0], tile_bound(n, c, T), stream),
                    "K5kv tile sort");
        L = level_bound(n, log2c, T, 1, 0);
    } else {
        HS_TRY_CUDA(hs::launch_plan((const long long *)user_off, ws.ctl, log2c, hs::kPlanMerge, 1, stream), "K4 plan");
        HS_TRY_CUDA(hs::launch_sample(dt, items, ws.samp[0], n, sms, stream), "K6 sample");
        // in place: level 0 reads the buffer its parity names (S when log2 c is odd)
        if (log2c & 1) HS_TRY_CUDA(hs::launch_copy(dt, items, S, n, sms, stream), "K7 copy");
        L = log2c;
    }
    for (int lv = 0; lv < L; ++lv) {
        HS_TRY_CUDA(hs::launch_merge_level(dt, plan, items, S, nullptr, ws.corank, ws.samp[lv & 1],
                                           lv + 1 < L ? ws.samp[(lv + 1) & 1] : nullptr, lv, (int)n, sms, stream),
                    "K6 merge level (items)");
    }
    cudaError_t fe = cudaFreeAsync(ws.base, stream);
    if (fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
    return HS_OK;
}

// Pack (keys, tags) into items, run kv_impl, unpack into (out_keys, out_tags).
hs_status_t kv_call(const void *keys, const uint64_t *tags, void *out_keys, uint64_t *out_tags, int64_t n,
                    hs_dtype_t dtype, int num_digits, int log2c, int mode, const int64_t *user_off, int64_t *off_out,
                    cudaStream_t stream) {
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    g_launch_counter = 0;
    void *buf = nullptr;
    const size_t ib = (size_t)n * sizeof(hs::KV64);
    if ((e = cudaMallocAsync(&buf, ib, stream)) != cudaSuccess) {
        cudaGetLastError();
        return fail(HS_ERR_OUT_OF_MEMORY, "cudaMallocAsync(%zu bytes) failed", ib);
    }
    hs::KV64 *items = (hs::KV64 *)buf;
    const int key64 = dtype == HS_INT64;
    hs_status_t s = HS_OK;
    if ((e = hs::launch_pack_kv(keys, key64, (const unsigned long long *)tags, items, n, sms, stream)) != cudaSuccess)
        s = cuda_fail(e, "K0kv pack");
    if (s == HS_OK) s = kv_impl(items, n, num_digits, log2c, mode, user_off, off_out, stream);
    if (s == HS_OK &&
        (e = hs::launch_unpack_kv(items, out_keys, key64, (unsigned long long *)out_tags, n, sms, stream)) != cudaSuccess)
        s = cuda_fail(e, "K8kv unpack");
    cudaError_t fe = cudaFreeAsync(buf, stream);
    if (s != HS_OK) return s;
    if (fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
    return succeed();
}

hs_status_t check_kv_args(const void *keys, const uint64_t *tags, const void *out_keys, const uint64_t *out_tags,
                          int64_t n, hs_dtype_t dtype, bool in_place_ok) {
    hs_status_t s;
    if ((s = check_common(n, dtype)) != HS_OK) return s;
    if ((s = check_ptr(keys, n, dtype, "keys")) != HS_OK) return s;
    if ((s = check_ptr(out_keys, n, dtype, "out_keys")) != HS_OK) return s;
    if ((s = check_ptr(tags, n, HS_INT64, "tags")) != HS_OK) return s;
    if ((s = check_ptr(out_tags, n, HS_INT64, "out_tags")) != HS_OK) return s;
    const size_t kb = (size_t)n * ksize(dtype), tb = (size_t)n * 8;
    if (n > 0 && (overlap2(keys, kb, tags, tb) || overlap2(out_keys, kb, out_tags, tb) ||
                  overlap2(keys, kb, out_tags, tb) || overlap2(out_keys, kb, tags, tb)))
        return fail(HS_ERR_INVALID_VALUE, "keys and tags overlap");
    if (n > 0 && !in_place_ok && (overlap(keys, out_keys, kb) || overlap(tags, out_tags, tb)))
        return fail(HS_ERR_INVALID_VALUE, "inputs and outputs overlap (out of place)");
    if (n > 0 && in_place_ok && ((keys != out_keys && overlap(keys, out_keys, kb)) ||
                                 (tags != out_tags && overlap(tags, out_tags, tb))))
        return fail(HS_ERR_INVALID_VALUE, "inputs and outputs overlap without being equal");
    return HS_OK;
}

}  // namespace

extern "C" {

hs_status_t hs_sort_pairs64(int64_t *keys, uint64_t *tags, int64_t n, int num_digits, int chunks_per_bucket,
                            cudaStream_t stream) {
    HS_NVTX("hs_sort_pairs64");
    hs_status_t s;
    int log2c;
    if ((s = check_kv_args(keys, tags, keys, tags, n, HS_INT64, true)) != HS_OK) return s;
    if ((s = check_digits(num_digits, HS_INT64)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    return kv_call(keys, tags, keys, tags, n, HS_INT64, num_digits, log2c, hs::kPlanSort, nullptr, nullptr, stream);
}

hs_status_t hs_msd_partition_pairs64(const int64_t *keys, const uint64_t *tags, int64_t n, int num_digits,
                                     int64_t *bucket_offsets, int64_t *out_keys, uint64_t *out_tags,
                                     cudaStream_t stream) {
    HS_NVTX("hs_msd_partition_pairs64");
    hs_status_t s;
    if ((s = check_kv_args(keys, tags, out_keys, out_tags, n, HS_INT64, false)) != HS_OK) return s;
    if ((s = check_digits(num_digits, HS_INT64)) != HS_OK) return s;
    if (!bucket_offsets || ((uintptr_t)bucket_offsets & 7) != 0)
        return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL or not 8-byte aligned");
    if (n == 0) {  // offsets of an empty input: all zero
        cudaError_t e = cudaMemsetAsync(bucket_offsets, 0, 11 * sizeof(int64_t), stream);
        if (e != cudaSuccess) return cuda_fail(e, "memset bucket_offsets");
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    int sms;
    cudaError_t e = device_setup(&sms);
    if (e != cudaSuccess) return cuda_fail(e, "device setup");
    g_launch_counter = 0;
    void *buf = nullptr;
    const size_t ib = (size_t)n * sizeof(hs::KV64);
    if ((e = cudaMallocAsync(&buf, 2 * ib, stream)) != cudaSuccess) {
        cudaGetLastError();
        return fail(HS_ERR_OUT_OF_MEMORY, "cudaMallocAsync(%zu bytes) failed", 2 * ib);
    }
    hs::KV64 *items = (hs::KV64 *)buf, *parted = items + n;
    Workspace ws;
    const int Tp = hs::scatter_tile_keys(2);
    const long long tiles = (n + Tp - 1) / Tp;
    unsigned long long div, magic;
    digit_params(num_digits, HS_INT64, &div, &magic);
    hs_status_t st = HS_OK;
    if ((e = hs::launch_pack_kv(keys, 1, (const unsigned long long *)tags, items, n, sms, stream)) != cudaSuccess)
        st = cuda_fail(e, "K0kv pack");
    if (st == HS_OK) st = ws_alloc(&ws, 0, (size_t)hs::scan_ctas(tiles) * 10, (size_t)tiles, 0, 0, stream);
    if (st == HS_OK) {
        if ((e = cudaMemsetAsync(ws.ctl, 0, ws.zero_bytes, stream)) != cudaSuccess ||
            (e = hs::launch_partition(2, items, parted, (int)n, 0, div, magic, ws.ctl, ws.tile_hist, ws.tile_pref,
                                      ws.status, (long long *)bucket_offsets, -1, 0, 0, sms, true, stream)) !=
                cudaSuccess ||
            (e = hs::launch_unpack_kv(parted, out_keys, 1, (unsigned long long *)out_tags, n, sms, stream)) !=
                cudaSuccess)
            st = cuda_fail(e, "K1-K3 partition (items)");
        cudaFreeAsync(ws.base, stream);
    }
    cudaError_t fe = cudaFreeAsync(buf, stream);
    if (st != HS_OK) return st;
    if (fe != cudaSuccess) return cuda_fail(fe, "cudaFreeAsync");
    return succeed();
}

hs_status_t hs_sort_chunks_pairs(const void *keys, const uint64_t *tags, void *out_keys, uint64_t *out_tags,
                                 int64_t n, hs_dtype_t dtype, const int64_t *bucket_offsets, int chunks_per_bucket,
                                 cudaStream_t stream) {
    HS_NVTX("hs_sort_chunks_pairs");
    hs_status_t s;
    int log2c;
    if ((s = check_kv_args(keys, tags, out_keys, out_tags, n, dtype, true)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if (!bucket_offsets) return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL");
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    return kv_call(keys, tags, out_keys, out_tags, n, dtype, 1, log2c, hs::kPlanChunks, bucket_offsets, nullptr,
                   stream);
}

hs_status_t hs_merge_pairs(const void *keys, const uint64_t *tags, void *out_keys, uint64_t *out_tags, int64_t n,
                           hs_dtype_t dtype, const int64_t *bucket_offsets, int chunks_per_bucket,
                           cudaStream_t stream) {
    HS_NVTX("hs_merge_pairs");
    hs_status_t s;
    int log2c;
    if ((s = check_kv_args(keys, tags, out_keys, out_tags, n, dtype, true)) != HS_OK) return s;
    if ((s = check_chunks(chunks_per_bucket, &log2c)) != HS_OK) return s;
    if (!bucket_offsets) return fail(HS_ERR_INVALID_VALUE, "bucket_offsets is NULL");
    if (n == 0) {
        g_launches = 0;
        g_err[0] = 0;
        return HS_OK;
    }
    return kv_call(keys, tags, out_keys, out_tags, n, dtype, 1, log2c, hs::kPlanMerge, bucket_offsets, nullptr, stream);
}

}  // extern "C"

