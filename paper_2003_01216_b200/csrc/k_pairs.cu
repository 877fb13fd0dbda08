// k_pairs.cu -- SURVEY §8(f) f3, the key + tag (stable) variant.
//
// An item (int32 key k, 64-bit tag) at input position i is sorted as the
// int64 value (k << 32) | i: ordering these by value is ordering by key with
// ties in input order, i.e. the stable sort SPEC's SortItem asks for (S:31-37,
// "tag never influences order"; the paper: merge sort "is a stable sort",
// P:29).  The int64 path of the library sorts the items unchanged -- its MSD
// digit reads the key as item >> 32 (DigitParams::shift) -- and the tags
// follow their index afterwards.
//
//   K0 k_pack_items    items[i] = (key[i] << 32) | i
//   K8 k_unpack_items  key[i] = items[i] >> 32, tag_out[i] = tag_in[items[i] & (2^32-1)]
#include <cstdint>

#include "hs_device.cuh"
#include "hs_launch.h"

namespace hs {

__global__ void k_pack_items(const int32_t *__restrict__ keys, long long *__restrict__ items, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        items[i] = (long long)(((unsigned long long)(long long)keys[i] << 32) | (unsigned long long)i);
}

__global__ void k_unpack_items(const long long *__restrict__ items, int32_t *__restrict__ keys,
                               const unsigned long long *__restrict__ tag_in, unsigned long long *__restrict__ tag_out,
                               long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const long long it = items[i];
        keys[i] = (int32_t)(it >> 32);
        tag_out[i] = __ldg(tag_in + (unsigned)(it & 0xFFFFFFFFll));
    }
}

static int grid_for(long long n, int num_sms) {
    const long long want = (n + 255) / 256;
    return (int)(want > 16LL * num_sms ? 16LL * num_sms : (want > 0 ? want : 1));
}

cudaError_t launch_pack_items(const int32_t *keys, long long *items, long long n, int num_sms, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    prof_begin(kProfCopy, st);
    k_pack_items<<<grid_for(n, num_sms), 256, 0, st>>>(keys, items, n);
    prof_end(kProfCopy, st);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
    return e;
}

cudaError_t launch_unpack_items(const long long *items, int32_t *keys, const unsigned long long *tag_in,
                                unsigned long long *tag_out, long long n, int num_sms, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    prof_begin(kProfCopy, st);
    k_unpack_items<<<grid_for(n, num_sms), 256, 0, st>>>(items, keys, tag_in, tag_out, n);
    prof_end(kProfCopy, st);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
    return e;
}

}  // namespace hs
