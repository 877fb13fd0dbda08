// Throughput of one register sorting network (Batcher odd-even, N = 28) per key
// type on sm_100a: int32, int64 (plain a < b ? : selects), int64 with one
// predicate (PTX setp + 2 selp.b64), double (fmin / fmax: exact for integers
// below 2^53), and two int32 halves (hi word compared, 64-bit payload moved).
// Dev aid for the int64 tile sort's bucket networks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2003_01216_b200/csrc
//        -o tools/probe/ce_probe tools/probe/ce_probe.cu
#include <cstdio>
#include <cstdint>

#include "hs_device.cuh"

using namespace hs;

struct P64 {  // int64, one predicate per comparator
    long long v;
};
__device__ __forceinline__ void cas(P64 &a, P64 &b) {
    long long lo, hi;
    asm("{\n\t.reg .pred p;\n\tsetp.lt.s64 p, %2, %3;\n\tselp.b64 %0, %2, %3, p;\n\tselp.b64 %1, %3, %2, p;\n\t}"
        : "=l"(lo), "=l"(hi)
        : "l"(a.v), "l"(b.v));
    a.v = lo;
    b.v = hi;
}
struct D64 {
    double v;
};
__device__ __forceinline__ void cas(D64 &a, D64 &b) {
    const double lo = fmin(a.v, b.v), hi = fmax(a.v, b.v);
    a.v = lo;
    b.v = hi;
}

template <typename T>
__device__ __forceinline__ T mk(unsigned x);
template <>
__device__ __forceinline__ int32_t mk<int32_t>(unsigned x) { return (int32_t)x; }
template <>
__device__ __forceinline__ int64_t mk<int64_t>(unsigned x) { return ((long long)x << 20) ^ x; }
template <>
__device__ __forceinline__ P64 mk<P64>(unsigned x) { return P64{((long long)x << 20) ^ x}; }
template <>
__device__ __forceinline__ D64 mk<D64>(unsigned x) { return D64{(double)(((long long)x << 20) ^ x)}; }
template <typename T>
__device__ __forceinline__ unsigned back(T t);
template <>
__device__ __forceinline__ unsigned back<int32_t>(int32_t t) { return (unsigned)t; }
template <>
__device__ __forceinline__ unsigned back<int64_t>(int64_t t) { return (unsigned)t; }
template <>
__device__ __forceinline__ unsigned back<P64>(P64 t) { return (unsigned)t.v; }
template <>
__device__ __forceinline__ unsigned back<D64>(D64 t) { return (unsigned)(long long)t.v; }

template <typename T, int N>
__global__ void __launch_bounds__(256, 4) k_probe(unsigned *out, int reps, unsigned seed) {
    T v[N];
    unsigned x = seed ^ (threadIdx.x * 2654435761u) ^ blockIdx.x;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        x = x * 1664525u + 1013904223u;
        v[i] = mk<T>(x >> 4);
    }
    for (int r = 0; r < reps; ++r) {
        oddeven_sort<N>(v);
        // reverse-ish perturbation so the next pass has work (and is not elided)
        T t = v[0];
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) v[i] = v[i + 1];
        v[N - 1] = t;
    }
    unsigned acc = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) acc = acc * 31u + back<T>(v[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename T>
float run(const char *name, unsigned *d, int reps) {
    constexpr int N = 28;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 4;
    k_probe<T, N><<<grid, 256>>>(d, 2, 1);
    cudaEventRecord(a);
    k_probe<T, N><<<grid, 256>>>(d, reps, 7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int ncmp = OddEvenNetHolder<N>::net.n;
    double ce = (double)grid * 256 * reps * ncmp;
    printf("%-22s %8.3f ms  %7.1f G comparators/s  (%d comparators per network)\n", name, ms, ce / ms / 1e6, ncmp);
    return ms;
}

int main() {
    unsigned *d;
    cudaMalloc(&d, 148 * 4 * 256 * sizeof(unsigned));
    const int reps = 400;
    run<int32_t>("int32", d, reps);
    run<int64_t>("int64 (a<b selects)", d, reps);
    run<P64>("int64 (one predicate)", d, reps);
    run<D64>("double fmin/fmax", d, reps);
    run<int32_t>("int32", d, reps);
    run<int64_t>("int64 (a<b selects)", d, reps);
    run<P64>("int64 (one predicate)", d, reps);
    run<D64>("double fmin/fmax", d, reps);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
