// Developer microbenchmark (not product code): random 64-bit atomics and
// loads over an L2-sized array -- the throughput a level-wide dedup set in
// L2 could reach.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_atomics l2_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t rmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int OP, int UNR>
__global__ void __launch_bounds__(256) k(unsigned long long* a, uint64_t n, uint64_t iters, uint64_t seed,
                                         unsigned long long* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = gridDim.x * (uint64_t)blockDim.x;
    unsigned long long acc = 0;
    for (uint64_t it = 0; it < iters; it++) {
        unsigned long long r[UNR];
#pragma unroll
        for (int u = 0; u < UNR; u++) {
            const uint64_t x = rmix(seed + (it * nth + tid) * UNR + u);
            const uint64_t i = __umul64hi(x, n);
            if (OP == 0) r[u] = atomicCAS(a + i, 0ull, x | 1ull);
            else if (OP == 1) r[u] = atomicExch(a + i, x | 1ull);
            else if (OP == 2) r[u] = __ldcg(a + i);
            else { atomicAdd(a + i, 1ull); r[u] = 0; }
        }
#pragma unroll
        for (int u = 0; u < UNR; u++) acc ^= r[u];
    }
    if (acc == 0x12345) atomicAdd(sink, 1ull);
}

template <int OP, int UNR>
double run(unsigned long long* a, uint64_t n, int sms, unsigned long long* sink) {
    const int grid = sms * 8;
    const uint64_t iters = 64;
    cudaMemset(a, 0, n * 8);
    k<OP, UNR><<<grid, 256>>>(a, n, 4, 1, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaMemset(a, 0, n * 8);
    cudaEventRecord(e0);
    k<OP, UNR><<<grid, 256>>>(a, n, iters, 7, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return (double)grid * 256 * iters * UNR / (ms / 1e3);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *a, *sink;
    cudaMalloc(&a, 1ull << 30); cudaMalloc(&sink, 8);
    const char* names[4] = {"CAS64", "EXCH64", "LDCG64", "RED_ADD64"};
    for (uint64_t mb : {4, 16, 32, 64, 96, 1024}) {
        const uint64_t n = (mb << 20) / 8;
        printf("%5llu MB: ", (unsigned long long)mb);
        printf("%s %.3g/s  ", names[0], run<0, 8>(a, n, sms, sink));
        printf("%s %.3g/s  ", names[1], run<1, 8>(a, n, sms, sink));
        printf("%s %.3g/s  ", names[2], run<2, 8>(a, n, sms, sink));
        printf("%s %.3g/s\n", names[3], run<3, 8>(a, n, sms, sink));
        fflush(stdout);
    }
    printf("CAS64 UNR 2/4/16 at 32 MB: %.3g %.3g %.3g\n", run<0, 2>(a, (32 << 20) / 8, sms, sink),
           run<0, 4>(a, (32 << 20) / 8, sms, sink), run<0, 16>(a, (32 << 20) / 8, sms, sink));
    return 0;
}
