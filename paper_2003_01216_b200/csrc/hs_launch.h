// hs_launch.h -- internal host-side launch interface between the C ABI
// (hs_api.cu) and the kernels (k_partition.cu, k_tilesort.cu, k_merge.cu).
// dt: 0 = int32, 1 = int64 (2 = KV64 items, internal: k_kv.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hs {

struct Ctl;
struct Plan;

// Optional per-kernel CUDA-event timing (hs_profile_enable); kinds match
// hs_profile_kind_name().  No-ops unless enabled on the calling thread.
enum ProfKind { kProfTileHist = 0, kProfTileScan, kProfScatter, kProfPlan, kProfTileSort, kProfMergePartition,
                kProfMergeLevel, kProfCopy, kProfSplitCount, kProfSplitScatter, kProfKinds };
void prof_begin(int kind, cudaStream_t st);
void prof_end(int kind, cudaStream_t st);
// Kernel launch accounting (hs_last_launch_count): every successful kernel
// launch of the library calls note_launch() once, on the calling thread.
void note_launch();

// One-time per-device kernel configuration (dynamic shared-memory limits,
// occupancy of the persistent kernels), run under hs_api.cu's per-device
// std::call_once; the launchers only read what it stored.
constexpr int kMaxDevices = 64;
cudaError_t setup_partition_kernels(int dev);
cudaError_t setup_tilesort_kernels(int dev);
cudaError_t setup_merge_kernels(int dev);
cudaError_t setup_split_kernels(int dev);

int scatter_tile_keys(int dt);  // keys per K1/K3 tile
int sort_tile_keys(int dt);     // leaf-tile capacity T of K5
int merge_span(int dt);         // outputs per K6 piece (TM)
int scan_ctas(long long ntiles);

// K1 + K2 (+ K3 if do_scatter): partition keys -> out, offsets -> ctl->off (+ user_off), plan if plan_mode >= 0
cudaError_t launch_partition(int dt, const void *keys, void *out, int n, int h, unsigned long long div,
                             unsigned long long magic, Ctl *ctl, uint32_t *tile_hist, uint32_t *tile_pref,
                             unsigned long long *status, long long *user_off, int plan_mode, int log2c,
                             int sort_tile_keys, int num_sms, bool do_scatter, cudaStream_t st,
                             int key_shift = 0, bool do_count = true, void *const *dst10 = nullptr);
cudaError_t launch_plan(const long long *user_off, Ctl *ctl, int log2c, int mode, int tile_keys, cudaStream_t st);
cudaError_t launch_plan_whole(long long n, Ctl *ctl, int log2c, int tile_keys, cudaStream_t st);  // one segment
// sbtab: K5a split table (leaves of split buckets; null when no bucket can be split)
struct SplitCfg;
cudaError_t launch_tile_sort(int dt, const Plan *plan, const void *src, void *F, void *S, void *samp,
                             long long max_tiles, cudaStream_t st, const uint32_t *sbtab = nullptr,
                             const SplitCfg *scfg = nullptr, const void *src_split = nullptr,  // null: F
                             const uint32_t *cflag = nullptr, const void *src_pad = nullptr);

// K5a (k_split.cu): value split of every chunk of the buckets whose chunks
// exceed one tile: setup (1 thread), count pass over S, per-chunk scan +
// plan finalisation, scatter pass S -> F.  tab / cur hold tab_words words
// (zeroed by k_split_setup before the count pass).
// cur holds split_cur_words(tab_words) words (cursors + constant-piece tracking);
// constant pieces (split_cflag) are written by the scatter straight to tile_out
// (where the tile sort of split buckets writes) and skipped by the tile sort.
long long split_table_words(long long n, int log2c, int tile_keys);
long long split_cur_words(long long tab_words);
const uint32_t *split_cflag(uint32_t *cur, long long tab_words);
// padbuf (pad_keys keys, may be null): the padded layout's regions (SplitCfg::pad); its keys are
// the tile sort's input for padded buckets.
long long split_pad_keys(long long n, int log2c, int tile_keys);
cudaError_t launch_split(int dt, Ctl *ctl, const void *S, void *F, uint32_t *tab, uint32_t *cur, long long tab_words,
                         long long n, int log2c, int tile_keys, unsigned long long div, int key_shift, void *tile_out,
                         void *padbuf, long long pad_keys, cudaStream_t st);
// samp_in: key samples of the level's input runs (kSampleQ stride); samp_out:
// the samples this level writes for the next one (may be null).
cudaError_t launch_merge_level(int dt, const Plan *plan, void *F, void *S, const void *src0, int *corank,
                               const void *samp_in, void *samp_out, int level, int n, int num_sms, cudaStream_t st);
// One-thread kernel: sets the conditional graph node handle to (plan Lmax > lv).
cudaError_t launch_level_gate(unsigned long long handle, const Plan *plan, int lv, cudaStream_t st);
// samp[m] = src[m*kSampleQ + kSampleQ-1] (hs_merge: samples of the caller's runs)
cudaError_t launch_sample(int dt, const void *src, void *samp, long long n, int num_sms, cudaStream_t st);
cudaError_t launch_copy(int dt, const void *src, void *dst, long long n, int num_sms, cudaStream_t st);

// f3 key + tag items on the stable path (k_kv.cu).  dt 2 in the launchers
// above (partition, merge level, sample, copy) = KV64 items.
struct KV64;
int kv_tile_keys();
cudaError_t setup_kv_kernels(int dev);
cudaError_t launch_pack_kv(const void *keys, int key64, const unsigned long long *tags, KV64 *items, long long n,
                           int num_sms, cudaStream_t st);
cudaError_t launch_unpack_kv(const KV64 *items, void *keys, int key64, unsigned long long *tags, long long n,
                             int num_sms, cudaStream_t st);
cudaError_t launch_tile_sort_kv(const Plan *plan, const KV64 *src, KV64 *F, KV64 *S, KV64 *samp, long long max_tiles,
                                cudaStream_t st);

// f3 key + tag items (k_pairs.cu)
cudaError_t launch_pack_items(const int32_t *keys, long long *items, long long n, int num_sms, cudaStream_t st);
cudaError_t launch_unpack_items(const long long *items, int32_t *keys, const unsigned long long *tag_in,
                                unsigned long long *tag_out, long long n, int num_sms, cudaStream_t st);

}  // namespace hs
