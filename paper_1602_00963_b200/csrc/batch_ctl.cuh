// batch_ctl.cuh -- control kernels of the device-driven batch (bc_api.cu,
// enqueue_device_batch): one CUDA graph per batch pipeline runs a whole
// batch -- every forward level, the sigma-tier fallbacks and every backward
// level -- with no host round trip.  The paper's per-level termination test
// (the all-reduce of nq, Alg.2 line 22) becomes a device flag
// per level: level L's launch is a no-op unless level L is non-empty, and a
// tier's launches are no-ops unless that tier is in use (gated_off in
// lanes.cuh).  The graph unrolls Lcap forward and backward level slots,
// Lcap = an upper bound on every BFS depth of the graph (bc_graph_create:
// 2 x the eccentricity of a root per component), so no batch runs out of
// slots.
#pragma once
#include "util.cuh"

namespace bcb {

// Batch start: the sources of batch ctl[1] of the pipeline's table (-1 past
// its lane count), the lanes-in-use words, the tier flags cleared, and the
// stat counters saved (a tier that overflows restores them).  One CTA.
__global__ void gb_begin_kernel(const int2 *table, int *ctl, const int *src_all, int K, int *bsrc, uint64_t *active,
                                const unsigned long long *stats, unsigned long long *stats_bak) {
    const int2 e = table[ctl[1]];
    BC_CHECK(e.x >= 0 && e.y >= 1 && e.y <= K);
    for (int l = threadIdx.x; l < K; l += blockDim.x) bsrc[l] = l < e.y ? src_all[e.x + l] : -1;
    if (threadIdx.x < 8) {
        const int lo = 64 * threadIdx.x;
        active[threadIdx.x] = e.y >= lo + 64 ? ~0ull : (e.y > lo ? (1ull << (e.y - lo)) - 1ull : 0ull);
        stats_bak[threadIdx.x] = stats[threadIdx.x];
    }
    if (threadIdx.x == 0) {
        ctl[0] = e.y;
        ctl[2] = 0;
        ctl[3] = 0;
    }
}

// Tier start (no-op unless the tier is in use): the per-batch state every
// forward builds on is cleared -- seen, the level-0/1 masks, the hub scratch
// rows, the level flags -- and the counters restored to their batch-start
// values.  Grid-stride.
__global__ void gb_reset_kernel(uint64_t *seen, uint64_t *m0, uint64_t *m1, size_t nmask, uint64_t *hub,
                                size_t nhub_words, int *flags, int nflags, unsigned long long *stats,
                                const unsigned long long *stats_bak, const int *need, const int *halt) {
    if ((need && *need == 0) || (halt && *halt != 0)) return;
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, step = (size_t)gridDim.x * blockDim.x;
    for (size_t i = i0; i < nmask; i += step) {
        seen[i] = 0;
        m0[i] = 0;
        m1[i] = 0;
    }
    for (size_t i = i0; i < nhub_words; i += step) hub[i] = 0;
    if (i0 < (size_t)nflags) flags[i0] = 0;
    if (i0 < 8) stats[i0] = stats_bak[i0];
}

// Forward slot L (no-op unless the tier is in use): the level-(L+1) mask and
// its "non-empty" flag start at zero.
__global__ void gb_zero_level_kernel(uint64_t *mask, size_t nmask, int *flag, const int *need) {
    if (need && *need == 0) return;
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, step = (size_t)gridDim.x * blockDim.x;
    for (size_t i = i0; i < nmask; i += step) mask[i] = 0;
    if (i0 == 0) *flag = 0;
}

// Batch end (one thread): depth of the batch (deepest non-empty level, read
// from the flags of the tier that completed), tier counters, the batch
// counter, and the depth bound check (level Lcap + 1 must be empty).  With
// 4-byte rows a batch whose 32-bit sigma overflowed is listed for the host's
// fp64 path (`redo`) and its counters are restored (the host run recounts).
// cnt: [0] levels, [1] 16-bit / [2] 32-bit / [3] fp64 batches, [4] redo
// entries, [5] depth-bound violations.
__global__ void gb_end_kernel(int *ctl, const int *flags, int lcap, unsigned long long *cnt, int *redo, int fp64_inline,
                              unsigned long long *stats, const unsigned long long *stats_bak) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const bool done = !ctl[2] || !ctl[3] || fp64_inline;
    if (done) {
        int lm = 0;
        for (int L = 1; L <= lcap + 1 && flags[L]; ++L) lm = L;
        cnt[0] += (unsigned long long)lm;
        if (flags[lcap + 1]) cnt[5] += 1;
    }
    if (!ctl[2]) {
        cnt[1] += 1;
    } else if (!ctl[3]) {
        cnt[2] += 1;
    } else {
        cnt[3] += 1;
        if (!fp64_inline) {
            redo[cnt[4]++] = ctl[1];
            for (int i = 0; i < 8; ++i) stats[i] = stats_bak[i];
        }
    }
    ctl[1] += 1;
}

// the condition of a conditional (IF) graph node: run its body iff *flag != 0
__global__ void gb_set_cond_kernel(cudaGraphConditionalHandle h, const int *flag) {
    cudaGraphSetConditional(h, *flag ? 1u : 0u);
}

}  // namespace bcb
