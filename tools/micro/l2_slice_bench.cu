// Microbenchmark: does one 2 KB accumulator row (8 groups of 32 doubles) sit
// in one L2 slice?  Every warp of a full grid issues coalesced fp64 reds
// (32 lanes x 8 B = one 256 B group per instruction) round-robin over G
// groups placed at base + g * stride.  If the G groups fall into different
// L2 slices the run is ~G times faster than G = 1 (the atomic units of more
// slices share the work); if they share a slice it is no faster.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void red_groups(double *a, int G, long long stride_d, int iters) {
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const int g = (wid + it) % G;
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(a + g * stride_d + lane), "d"(1.0) : "memory");
    }
}

int main() {
    double *a;
    const size_t bytes = 1ull << 30;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 4, threads = 256, iters = 2000;
    const double reds = (double)blocks * threads / 32 * iters;
    const long long strides[] = {32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 65536, 131072, 1 << 20};
    for (int G : {1, 2, 8, 64}) {
        for (long long sb : strides) {
            if ((G - 1) * sb * 8 >= (long long)bytes) continue;
            red_groups<<<blocks, threads>>>(a, G, sb, 10);
            cudaEventRecord(e0);
            red_groups<<<blocks, threads>>>(a, G, sb, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("G=%3d stride=%8lld B  %8.3f ms  %7.2f G red-instr/s\n", G, sb * 8, ms, reds / ms / 1e6);
        }
    }
    return 0;
}
