// util.cuh -- warp/block primitives for the sm_100a BC kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef BC_NT
#define BC_NT 256                 // threads per CTA of the level kernels
#endif
#define BC_NW (BC_NT / 32)        // warps per CTA

// Device-side bounds checks (compute-sanitizer is not available on the GPU
// pool): a -DBC_DEVICE_CHECKS=1 build traps on a violated index invariant,
// which surfaces as a CUDA error in the calling test.  Off in the product build.
#ifndef BC_DEVICE_CHECKS
#define BC_DEVICE_CHECKS 0
#endif
#if BC_DEVICE_CHECKS
#define BC_CHECK(cond)        \
    do {                      \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define BC_CHECK(cond) \
    do {               \
    } while (0)
#endif

namespace bcb {

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

__device__ __forceinline__ int warp_incl_scan(int x) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ long long warp_incl_scan64(long long x) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Block-wide exclusive scan of two ints at once (CTA of BC_NT threads).
// sm: >= 2*BC_NW+2 ints of shared memory.  Ends with a barrier so `sm` can
// be reused immediately.
__device__ __forceinline__ void block_excl_scan2(int a, int b, int &ea, int &eb, int &ta, int &tb,
                                                 int *sm) {
    const int lane = lane_id(), wid = warp_id();
    int ia = warp_incl_scan(a), ib = warp_incl_scan(b);
    if (lane == 31) {
        sm[wid] = ia;
        sm[BC_NW + wid] = ib;
    }
    __syncthreads();
    if (wid == 0) {
        int va = lane < BC_NW ? sm[lane] : 0;
        int vb = lane < BC_NW ? sm[BC_NW + lane] : 0;
        int sa = warp_incl_scan(va), sb = warp_incl_scan(vb);
        if (lane < BC_NW) {
            sm[lane] = sa - va;
            sm[BC_NW + lane] = sb - vb;
        }
        if (lane == BC_NW - 1) {
            sm[2 * BC_NW] = sa;
            sm[2 * BC_NW + 1] = sb;
        }
    }
    __syncthreads();
    ea = sm[wid] + ia - a;
    eb = sm[BC_NW + wid] + ib - b;
    ta = sm[2 * BC_NW];
    tb = sm[2 * BC_NW + 1];
    __syncthreads();
}

// Largest s in [0, nslots) with cd[s] <= e, for strictly increasing cd
// (every slot holds >= 1 item).  The paper's "binary search over the CD
// array"; SPEC.md:125 semantics.
__device__ __forceinline__ int slot_of(const int *cd, int nslots, int e) {
    int lo = 0, hi = nslots - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (cd[mid] <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Streaming 32-bit load of CSR column data: read once per sweep, keep it out
// of L1 and mark it evict-first in L2 so per-vertex state stays resident.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ int ld_stream(const int *p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

}  // namespace bcb
