// hs_launch.h -- internal host-side launch interface between the C ABI
// (hs_api.cu) and the kernels (hs_kernels.cu).  dt: 0 = int32, 1 = int64.
#pragma once

#include <cuda_runtime.h>

namespace hs {

struct Ctl;
struct Plan;

int tile_keys(int dt, int which);  // 0 scatter tile, 1 tile-sort tile, 2 merge CTA span

cudaError_t launch_histogram(int dt, const void *keys, int n, int h, unsigned long long div, unsigned long long magic,
                             Ctl *ctl, long long *user_off, int plan_mode, int log2c, int num_sms, cudaStream_t st);
cudaError_t launch_scatter(int dt, const void *keys, void *out, int n, int h, unsigned long long div,
                           unsigned long long magic, Ctl *ctl, unsigned long long *status, cudaStream_t st);
cudaError_t launch_plan(const long long *user_off, Ctl *ctl, int log2c, int mode, int tile_keys, cudaStream_t st);
cudaError_t launch_tile_sort(int dt, const Plan *plan, const void *src, void *F, void *S, long long max_tiles,
                             cudaStream_t st);
cudaError_t launch_merge_level(int dt, const Plan *plan, void *F, void *S, const void *src0, int *corank, int level,
                               int n, cudaStream_t st);
cudaError_t launch_copy(int dt, const void *src, void *dst, long long n, int num_sms, cudaStream_t st);

}  // namespace hs
