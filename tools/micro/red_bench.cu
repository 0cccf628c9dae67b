// Microbenchmark: fp64 red.global.add throughput on B200 for the access
// patterns a push-style backward sweep would use.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// each warp: `iters` times pick a random row (of `rows` rows of 256 doubles),
// and every thread adds into `per` cells of it: mode 0 = slice (thread t owns 8t..8t+7),
// mode 1 = strided (thread t owns t, t+32, ...)
__global__ void red_kernel(double *a, int rows, int iters, int per, int mode, uint64_t seed) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const uint64_t r = mix(seed + wid * 1000003ull + it) % (uint64_t)rows;
        double *row = a + r * 256;
        for (int i = 0; i < per; ++i) {
            const int cell = mode == 0 ? lane * 8 + i : i * 32 + lane;
            atomicAdd(row + cell, 1.0);
        }
    }
}

__global__ void ld_kernel(const double *a, int rows, int iters, int per, int mode, uint64_t seed, double *out) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    double s = 0;
    for (int it = 0; it < iters; ++it) {
        const uint64_t r = mix(seed + wid * 1000003ull + it) % (uint64_t)rows;
        const double *row = a + r * 256;
        for (int i = 0; i < per; ++i) {
            const int cell = mode == 0 ? lane * 8 + i : i * 32 + lane;
            s += row[cell];
        }
    }
    if (s == 12345.0) out[0] = s;
}

int main() {
    const size_t maxrows = (size_t)1 << 20;  // 2 GB of rows
    double *a, *o;
    cudaMalloc(&a, maxrows * 256 * 8);
    cudaMalloc(&o, 8);
    cudaMemset(a, 0, maxrows * 256 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int rowsv[] = {16384, 65536, 1 << 20};
    for (int ri = 0; ri < 3; ++ri)
        for (int mode = 0; mode < 2; ++mode)
            for (int per : {2, 8}) {
                const int rows = rowsv[ri];
                const int blocks = 148 * 8, threads = 256, iters = 200;
                red_kernel<<<blocks, threads>>>(a, rows, 10, per, mode, 1);
                cudaEventRecord(e0);
                red_kernel<<<blocks, threads>>>(a, rows, iters, per, mode, 7);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double nred = (double)blocks * threads * iters * per;
                cudaEventRecord(e0);
                ld_kernel<<<blocks, threads>>>(a, rows, iters, per, mode, 9, o);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms2;
                cudaEventElapsedTime(&ms2, e0, e1);
                printf("rows=%8d (%6.0f MB) mode=%s per=%d: RED %.1f G/s (%.0f GB/s)  LD %.1f G/s\n", rows,
                       rows * 2048.0 / 1e6, mode ? "strided" : "slice  ", per, nred / ms / 1e6, nred * 8 / ms / 1e6,
                       nred / ms2 / 1e6);
            }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
