// Bandwidth probe (dev aid, not product code): what HBM read+write rate does a
// kernel reach on (a) a plain copy and (b) the merge level's stream shape --
// every piece reads two separate input slices and writes one contiguous output
// slice -- with no merge work at all.  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/probe/stream_probe.cu -o /tmp/stream_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_k(const int4 *__restrict__ in, int4 *__restrict__ out, long long n4) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// piece p (TM ints): out[p*TM .. +TM) = in[aoff(p) .. +TM/2) ++ in[boff(p) .. +TM/2), where the
// A slices walk the first half of the input and the B slices the second half (like a merge of
// two runs of a pair)
__global__ void two_in_one_out(const int *__restrict__ in, int *__restrict__ out, long long n, int TM) {
    const long long pieces = n / TM;
    const long long half = n / 2;
    for (long long p = blockIdx.x; p < pieces; p += gridDim.x) {
        const long long a0 = p * (TM / 2), b0 = half + p * (TM / 2);
        const int4 *A = reinterpret_cast<const int4 *>(in + a0);
        const int4 *B = reinterpret_cast<const int4 *>(in + b0);
        int4 *O = reinterpret_cast<int4 *>(out + p * TM);
        const int h4 = TM / 8;  // int4s per half
        for (int i = threadIdx.x; i < h4; i += blockDim.x) {
            O[i] = A[i];
            O[h4 + i] = B[i];
        }
    }
}

int main() {
    const long long n = 1LL << 28;  // 1 GiB of int32
    int *in, *out;
    cudaMalloc(&in, n * 4);
    cudaMalloc(&out, n * 4);
    cudaMemset(in, 1, n * 4);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch, const char *name) {
        for (int w = 0; w < 3; ++w) launch();
        cudaDeviceSynchronize();
        float best = 1e9f;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("%-40s %.3f ms  %.0f GB/s (read + write)\n", name, best, 2.0 * n * 4 / (best * 1e-3) / 1e9);
    };
    timeit([&] { copy_k<<<sms * 8, 256>>>((const int4 *)in, (int4 *)out, n / 4); }, "copy (grid-stride int4)");
    for (int TM : {3200, 6400, 12800, 25600}) {
        for (int per : {4, 8}) {
            char nm[96];
            snprintf(nm, sizeof nm, "2-in/1-out TM=%d, %d CTAs/SM x 256", TM, per);
            timeit([&] { two_in_one_out<<<sms * per, 256>>>(in, out, n, TM); }, nm);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
