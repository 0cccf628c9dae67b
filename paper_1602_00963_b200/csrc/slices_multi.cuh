// slices_multi.cuh -- KS sources per CTA in lockstep, for long-diameter
// graphs of bounded degree (the grid / road-network workload).
//
// slices_lowdeg_sm_kernel runs one source per CTA: every BFS level of every
// source pays a chain of dependent loads (queue -> neighbour row -> parents'
// sigma) and a barrier, and the grid has ~1000 levels per source.  Here a
// CTA takes KS sources that are consecutive in the compute order (the
// breadth-first relabelling puts them close together) and sweeps them as
// lanes of ONE level-synchronous traversal: level L's union frontier F_L
// holds every vertex at depth L for at least one lane, so the chain and the
// barrier of a level are paid once for all KS sources, and for nearby
// sources the union frontier is barely larger than one source's.
//
// Per vertex v (CTA-private, global memory):
//   st2[v]       KS 2-bit depth codes: 0 = unvisited, else (d(s_l, v) mod 3) + 1.
//                A neighbour of a level-L vertex lies at L-1, L or L+1 (or is
//                unvisited), so "code == (L-1) mod 3 + 1" finds the parents
//                and "code == (L+1) mod 3 + 1" the children, per lane.
//   sg[v][KS]    sigma_l(v), overwritten in place by coef_l(v) =
//                (1 + omega(v) + delta_l(v)) / sigma_l(v) in the backward step
//                of v's level for lane l (Eq.(5); reading R2).
//   apl[v]       the last level v was appended to the union frontier (dedup).
// Forward level L (Alg.2/Alg.3): a thread takes v in F_L,
// lanes lv = {l : v at depth L}; it pulls sigma_l(v) = sum of sigma_l(u) over
// neighbours u at depth L-1 in lane l (Alg.1 lines 16-19 from the child's
// side), then marks its unvisited neighbours' lanes lv at depth L+1 (atomic
// OR of the codes; a field is only ever set from 0 to code(L+1) during level
// L, so concurrent setters agree) and appends a newly marked neighbour to
// F_{L+1} once (atomicMax on apl).  Backward level L: v in F_L sums the coef
// of its depth-(L+1) neighbours per lane, forms delta and coef, and adds
// sum_l (1 + omega(s_l)) (delta_l(v) + omega(v)) to BC(v) with ONE fp64
// atomic (not one per source, R13).
#pragma once
#include "slices.cuh"

namespace bcb {

struct MultiParams {
    uint32_t *st2;  // [rows][n]
    int *apl;       // [rows][n], -1 between groups
    double *sg;     // [rows][n][KS]
    int *q;         // [rows][qcap] union frontiers of all levels
    long long qcap;
    int *loff;      // [rows][n + 2]
};

#ifndef BC_SMU_NT
#define BC_SMU_NT 512
#endif
#ifndef BC_SMU_MINB
#define BC_SMU_MINB 2
#endif

template <int KS>
__device__ __forceinline__ uint32_t even_bits() {
    return (uint32_t)(0x5555555555555555ull & ((1ull << (2 * KS)) - 1ull));
}
// bit 2l set iff lane l's 2-bit field of s equals c (1..3)
template <int KS>
__device__ __forceinline__ uint32_t fields_eq(uint32_t s, uint32_t c) {
    const uint32_t x = s ^ (c * even_bits<KS>());
    return ~(x | (x >> 1)) & even_bits<KS>();
}
// bit 2l set iff lane l's field is 0 (unvisited)
template <int KS>
__device__ __forceinline__ uint32_t fields_zero(uint32_t s) {
    return ~(s | (s >> 1)) & even_bits<KS>();
}

// the KS values of v's sigma / coef row (16-byte loads)
template <int KS>
__device__ __forceinline__ void load_row(const double *r, double (&x)[KS]) {
#pragma unroll
    for (int l = 0; l < KS; l += 2) {
        const double2 t = *reinterpret_cast<const double2 *>(r + l);
        x[l] = t.x;
        x[l + 1] = t.y;
    }
}

template <int KS, bool ELL, bool CAP = false>
__global__ void __launch_bounds__(BC_SMU_NT, BC_SMU_MINB) slices_multi_kernel(SlicesParams p, MultiParams m) {
    static_assert(KS % 2 == 0 && KS <= 16, "KS lanes: even, at most 16 (2-bit fields in 32 bits)");
    __shared__ int sh_src[KS];
    __shared__ int sh_cs[KS];     // capture slot per lane (CAP)
    __shared__ double sh_w1[KS];  // 1 + omega(s_l)
    __shared__ double sh_ns[KS];  // n_s per lane (pruned graphs, R9)
    __shared__ int sh_cnt[3];     // appends of level L in cnt[(L + 1) % 3] (rotating, as slices_lowdeg_sm_kernel)
    __shared__ int sh_g;
    const size_t n = (size_t)p.n;
    uint32_t *st2 = m.st2 + blockIdx.x * n;
    int *apl = m.apl + blockIdx.x * n;
    double *sg = m.sg + blockIdx.x * n * KS;
    int *Q = m.q + (size_t)blockIdx.x * (size_t)m.qcap;
    int *loff = m.loff + blockIdx.x * (n + 2);
    const int tid = threadIdx.x;
    unsigned long long st_reach = 0, st_adj = 0, st_dag = 0, st_dsum = 0;
    const int ngroups = (p.nsrc + KS - 1) / KS;

    for (;;) {
        if (tid == 0) {
            const int t = atomicAdd(p.next_src, 1);
            if (t == ngroups + (int)gridDim.x - 1) *p.next_src = 0;  // last fetch resets
            sh_g = t;
        }
        __syncthreads();
        const int gi = sh_g;
        if (gi >= ngroups) break;
        const int nl = min(KS, p.nsrc - gi * KS);
        if (tid < KS) {
            const int s = tid < nl ? p.src[gi * KS + tid] : -1;
            sh_src[tid] = s;
            sh_w1[tid] = 1.0 + ((p.omega && s >= 0) ? (double)p.omega[s] : 0.0);
            sh_ns[tid] = 0.0;
            sh_cs[tid] = (CAP && s >= 0) ? p.cap_vslot[s] : -1;
        }
        if (tid < 3) sh_cnt[tid] = 0;
        __syncthreads();
        // level 0: the sources (code 1 in their own lane)
        if (tid < nl) {
            const int s = sh_src[tid];
            atomicOr(&st2[s], 1u << (2 * tid));
            sg[(size_t)s * KS + tid] = 1.0;
            if (atomicMax(&apl[s], 0) < 0) Q[atomicAdd(&sh_cnt[0], 1)] = s;
        }
        __syncthreads();
        int L = 0, qs = 0, qe = sh_cnt[0], r3 = 1;
        if (tid == 0) {
            loff[0] = 0;
            loff[1] = qe;
        }
        // ---------------- forward
        while (qs < qe) {
            const uint32_t cL = (uint32_t)(L % 3) + 1u, cP = (uint32_t)((L + 2) % 3) + 1u,
                           cN = (uint32_t)((L + 1) % 3) + 1u;
            int *cnt = &sh_cnt[r3];
            const int r3n = r3 == 2 ? 0 : r3 + 1;
            if (tid == 0) sh_cnt[r3n] = 0;  // last read right after the barrier that ended level L-2
            for (int i = qs + tid; i < qe; i += BC_SMU_NT) {
                const int v = Q[i];
                const uint32_t lv = fields_eq<KS>(st2[v], cL);
                const int4 row = lowdeg_row<ELL>(p, v);
                if (L >= 1) {
                    double acc[KS];
#pragma unroll
                    for (int l = 0; l < KS; ++l) acc[l] = 0.0;
                    lowdeg_row_nbrs<ELL>(p, row, [&](const int *u) {
#pragma unroll
                        for (int k = 0; k < BC_LD_GRP; ++k) {
                            if (u[k] < 0) continue;
                            const uint32_t par = fields_eq<KS>(st2[u[k]], cP) & lv;
                            if (!par) continue;
                            st_dag += __popc(par);
                            double x[KS];
                            load_row<KS>(sg + (size_t)u[k] * KS, x);
#pragma unroll
                            for (int l = 0; l < KS; ++l)
                                if (par >> (2 * l) & 1u) acc[l] += x[l];
                        }
                    });
#pragma unroll
                    for (int l = 0; l < KS; ++l)
                        if (lv >> (2 * l) & 1u) sg[(size_t)v * KS + l] = acc[l];
                }
                // discovery: v's level-L lanes reach the unvisited lanes of its neighbours
                const uint32_t setc = lv * cN;
                int deg = 0;
                lowdeg_row_nbrs<ELL>(p, row, [&](const int *w) {
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        if (w[k] < 0) continue;
                        ++deg;
                        const uint32_t nb = setc & (fields_zero<KS>(st2[w[k]]) * 3u);
                        if (!nb) continue;
                        atomicOr(&st2[w[k]], nb);
                        if (atomicMax(&apl[w[k]], L + 1) < L + 1) Q[qe + atomicAdd(cnt, 1)] = w[k];
                    }
                });
                const int pc = __popc(lv);
                st_reach += pc;
                st_adj += (unsigned long long)pc * deg;
                st_dsum += (unsigned long long)pc * L;
                if (p.omega) {
                    const double wv = 1.0 + (double)p.omega[v];
#pragma unroll
                    for (int l = 0; l < KS; ++l)
                        if (lv >> (2 * l) & 1u) atomicAdd(&sh_ns[l], wv);
                }
            }
            __syncthreads();
            qs = qe;
            qe += *cnt;
            r3 = r3n;
            ++L;
            if (tid == 0) loff[L + 1] = qe;
        }
        const int Lmax = L - 1;
        const int total = qe;
        // ---------------- backward, L = Lmax .. 1
        for (L = Lmax; L >= 1; --L) {
            const uint32_t cL = (uint32_t)(L % 3) + 1u, cC = (uint32_t)((L + 1) % 3) + 1u;
            const int a = loff[L], b = loff[L + 1];
            for (int i = a + tid; i < b; i += BC_SMU_NT) {
                const int v = Q[i];
                const uint32_t lv = fields_eq<KS>(st2[v], cL);
                const int4 row = lowdeg_row<ELL>(p, v);
                double acc[KS];
#pragma unroll
                for (int l = 0; l < KS; ++l) acc[l] = 0.0;
                lowdeg_row_nbrs<ELL>(p, row, [&](const int *u) {
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        if (u[k] < 0) continue;
                        const uint32_t ch = fields_eq<KS>(st2[u[k]], cC) & lv;
                        if (!ch) continue;
                        double x[KS];
                        load_row<KS>(sg + (size_t)u[k] * KS, x);
#pragma unroll
                        for (int l = 0; l < KS; ++l)
                            if (ch >> (2 * l) & 1u) acc[l] += x[l];
                    }
                });
                const double om = p.omega ? (double)p.omega[v] : 0.0;
                double contrib = 0.0;
#pragma unroll
                for (int l = 0; l < KS; ++l) {
                    if (!(lv >> (2 * l) & 1u)) continue;
                    double *slot = sg + (size_t)v * KS + l;
                    const double sgl = *slot;
                    const double delta = sgl * acc[l];
                    *slot = (1.0 + om + delta) / sgl;
                    contrib += sh_w1[l] * (delta + om);
                    if constexpr (CAP) {
                        if (sh_cs[l] >= 0) {
                            const size_t o = (size_t)sh_cs[l] * n + v;
                            p.cap_depth[o] = L;
                            p.cap_sigma[o] = sgl;
                            p.cap_delta[o] = delta;
                        }
                    }
                }
                if (contrib != 0.0) atomicAdd(p.bc + v, contrib);
            }
            __syncthreads();
        }
        // endpoint terms (R13), then the touched vertices are reset
        if (tid < nl && p.omega) {
            const int s = sh_src[tid];
            const double om = (double)p.omega[s];
            if (om != 0.0) atomicAdd(p.bc + s, om * (sh_ns[tid] - 2.0));
        }
        for (int i = tid; i < total; i += BC_SMU_NT) {
            const int v = Q[i];
            st2[v] = 0u;
            apl[v] = -1;
        }
        __syncthreads();
    }
    const unsigned long long a = warp_sum_u64(st_reach), b = warp_sum_u64(st_adj), c = warp_sum_u64(st_dag),
                             d = warp_sum_u64(st_dsum);
    if (lane_id() == 0) {
        if (a) atomicAdd(p.stats + 0, a);
        if (b) atomicAdd(p.stats + 1, b);
        if (c) atomicAdd(p.stats + 2, c);
        if (d) atomicAdd(p.stats + 3, d);
    }
}

}  // namespace bcb
