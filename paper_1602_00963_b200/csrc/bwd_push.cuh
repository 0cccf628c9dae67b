// bwd_push.cuh -- backward dependency sweep, push form, for the bit-lane
// batches (lanes.cuh).
//
// The pull form (successor checking, Alg.5, reading R2)
// makes every level-L vertex gather the coef rows of its level-(L+1)
// children.  On R-MAT those children are mostly low-degree vertices whose
// rows are read once per parent and miss L2 -- the pull backward moved ~2x
// its algorithmic bytes from DRAM (profiles/ncu_traffic.json).  The same sum
//     delta(x) = sigma(x) * sum_{children v of x} coef(v)
// is formed here from the other side of each DAG edge: once coef(v) of a
// level-L vertex is final, v *pushes* it into an accumulator row A[y] of every
// parent y (level L-1, lanes c = lvl[L][v] & lvl[L-1][y]) with fp64
// red.global.add -- fire-and-forget, so no gather latency is on the critical
// path, each child row is read once, and the parents' accumulators (hubs,
// mostly) stay L2-resident.  Per level L = Lmax .. 1:
//   lanes_bwd_finalize_kernel(L): for x at level L, lanes in lvl[L][x]:
//       acc = A[x] (complete: all children pushed at level L+1); A[x] := 0
//       delta = sigma * acc; coef = (1 + omega(x) + delta) / sigma   (Eq.5)
//       S_L[x] := coef (row stays zero outside level L)
//       BC[x] += sum_lanes (1 + omega(s)) (delta + omega(x))          (R13)
//   lanes_bwd_push_kernel(L), L >= 2: items (x, y) over the adjacency of the
//       level-L vertices, mapped to threads by the tile CD scan + binary
//       search; hubs are cut into segments.  Every cell
//       of A is consumed (and re-zeroed) by exactly one finalize, so A is
//       zero again after every batch.
// Lane-to-thread mapping here is *strided* (lane l -> thread l % 32, group
// l / 32) so one red instruction covers 32 consecutive doubles (256 B); the
// microbenchmark tools/micro/red_bench.cu measured 560 G red/s for that
// pattern on L2-resident rows vs 190 G/s for 8-lane thread slices.
#pragma once
#include "lanes.cuh"

namespace bcb {

#ifndef BC_A_PAD
#define BC_A_PAD 0  // doubles of padding after each accumulator row (row stride K + pad)
#endif
// row stride of the fp64 backward accumulators A[v][K]
template <int W> struct AStride { static constexpr size_t v = 64 * W + BC_A_PAD; };

#ifndef BC_A_PLANES
#define BC_A_PLANES 0  // 1: accumulators group-major, A[j][v][32] (group j of every row in one plane)
#endif
// accumulator row of vertex v (lane 0) and the distance between its 32-lane groups
#define A_ROW(A, vx_) (BC_A_PLANES ? (A) + (size_t)(vx_) * 32 : (A) + (size_t)(vx_) * AStride<W>::v)
#define A_GRP(p) (BC_A_PLANES ? (size_t)(p).n * 32 : (size_t)32)
#ifndef BC_REP_H
#define BC_REP_H 0  // > 0: parents with id < BC_REP_H (degree order: the hubs) get replicated accumulator rows (slower, off)
#endif
#ifndef BC_REP_R
#define BC_REP_R 8   // ... in BC_REP_R copies, so their reds spread over more L2 slices
#endif
// A[y] += sum of the replicas of row y (y < BC_REP_H), replicas re-zeroed.
// Runs before each backward level: every red into A[y][l] comes from the
// push at level d_l(y) + 1 and A[y][l] is read at level d_l(y), so folding
// at every level delivers each lane's sum before it is used.
template <int W>
__global__ void __launch_bounds__(BC_NT) lanes_rep_fold_kernel(LanesParams p, double *__restrict__ A) {
    if ((p.prev_new && *p.prev_new == 0) || gated_off(p)) return;
    constexpr int K = 64 * W;
    const int i = blockIdx.x * BC_NT + threadIdx.x;
    const int y = i / K, l = i % K;
    if (y >= BC_REP_H || y >= p.n) return;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < BC_REP_R; ++r) {
        double *q = p.arep + ((size_t)r * BC_REP_H + y) * K + l;
        const double v = *q;
        if (v != 0.0) {
            s += v;
            *q = 0.0;
        }
    }
    if (s != 0.0) A_ROW(A, y)[(size_t)(l >> 5) * A_GRP(p) + (l & 31)] += s;
}

__device__ __forceinline__ void red_add_f64(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
#ifndef BC_PUSH_RED_HINT
#define BC_PUSH_RED_HINT 2  // L2 policy of the push reds: 0 none, 1 evict_first, 2 evict_last (S20 push 202.3 -> 199.1 ms, profiles/exp_r2_redhint.txt)
#endif
// predicated form: no branch around the red (the per-lane condition is data
// dependent, a branch would diverge)
__device__ __forceinline__ void red_add_f64_if(double *p, double v, uint32_t pred) {
#if BC_PUSH_RED_HINT
    uint64_t pol;
#if BC_PUSH_RED_HINT == 1
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#else
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.global.add.L2::cache_hint.f64 [%0], %1, %3;\n\t}" ::"l"(p),
        "d"(v), "r"(pred), "l"(pol)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.global.add.f64 [%0], %1;\n\t}" ::"l"(p), "d"(v),
        "r"(pred)
        : "memory");
#endif
}

// 1/x for x >= 1 (sigma): hardware approximation + two Newton steps, within
// ~1 ulp, no division subroutine (which costs registers in the push loop)
__device__ __forceinline__ double rcp_f64(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

#ifndef BC_PR4
#define BC_PR4 1  // item steps in flight per warp at W = 4 (keeps 64 registers: occupancy wins)
#endif
#ifndef BC_PUSH_MINB
#define BC_PUSH_MINB 4  // push kernels need fewer registers: 4 CTAs (32 warps) per SM
#endif
#ifndef BC_PUSH_MINB8
#define BC_PUSH_MINB8 3  // ... W = 8: 16 coef values per thread
#endif
#ifndef BC_PUSH_MASK_HINT
#define BC_PUSH_MASK_HINT 0  // L2 policy of the push's parent-mask loads: 0 none, 1 evict_first, 2 evict_last
#endif
#ifndef BC_PUSH_OWN_HINT
#define BC_PUSH_OWN_HINT 1  // the slot's own accumulator row read and re-zeroed with L2 evict_first
                            // (S20 push 198.8 -> 194.1 ms, profiles/exp_r2_push_l2hints.txt); 2: its sigma row too
#endif
__device__ __forceinline__ double ld_ef_f64(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_ef_f64(double *p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
#ifndef BC_PUSH_CFSMEM
#define BC_PUSH_CFSMEM 0  // backward push: the current slot's coef row staged in shared memory, not in registers
#endif
#ifndef BC_PUSH_COMPACT
#define BC_PUSH_COMPACT 0  // 1: backward push over the slot's compacted lanes (measured slower overall, profiles/exp_r2_push.txt)
#endif

template <int W>
struct PushSmem {
    int vert[TV];
    int cd[TV + 1];
    int rs[TV];
    uint64_t u[TV * W];
    alignas(16) uint64_t hc[BC_NW * 32 * W];  // per warp: contributing-lane words of the step's items
    int4 hsv[BC_NW * 32];         // per warp: (slot, y, group mask, -) of the step's items
    static constexpr bool CFS = BC_PUSH_CFSMEM && W <= 4;
    uint16_t lst[BC_PUSH_COMPACT ? BC_NW * 64 * W : 1]; // per warp: the current slot's level-L lanes in lane order (compacted push)
    double cfs[CFS ? BC_NW * 64 * W : 1];  // per warp: the current slot's coef row (BC_PUSH_CFSMEM, W <= 4)
    int scan[2 * BC_NW + 2];
    int unit;
};

// x at level L: finalise coef and BC (warp per vertex, strided lanes; all
// loads of a vertex are issued before its stores)
// COEF = false: only BC and the re-zeroing of A (the fused push computes the
// coef values itself and never reads the coef row)
// RT = storage type of the sigma rows (double, or uint16_t after a narrow forward)
template <int W, bool COEF, typename RT = double>
__device__ __forceinline__ void bwd_finalize_vertex(const LanesParams &p, double *__restrict__ A,
                                                    RT *__restrict__ S, int x, int lane) {
    static_assert(!COEF || std::is_same<RT, double>::value, "coef rows are fp64");
    constexpr int K = 64 * W, NG = 2 * W;
    uint64_t m[W];
    load_mask<W>(p.mask_cur + (size_t)x * W, m);
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < NG; ++j) bits |= (((uint32_t)(m[j >> 1] >> ((j & 1) * 32)) >> lane) & 1u) << j;
    double *arow = A_ROW(A, x) + lane;
    const size_t ag = A_GRP(p);
    RT *row = S + (size_t)x * K;
    double av[NG], sv[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
        av[j] = 0.0;
        sv[j] = 1.0;
        if (bits >> j & 1u) {
            av[j] = arow[j * ag];
            sv[j] = (double)row[row_idx<W, RT>(32 * j + lane)];
        }
    }
    const double om = p.omega ? (double)p.omega[x] : 0.0;
    double contrib = 0.0;
#pragma unroll
    for (int j = 0; j < NG; ++j) {
        if (bits >> j & 1u) {
            const double delta = sv[j] * av[j];
            arow[j * ag] = 0.0;
            if constexpr (COEF) row[32 * j + lane] = (1.0 + om + delta) / sv[j];  // fp64 rows: lane order
            contrib += p.lane_w1[32 * j + lane] * (delta + om);
            cap_delta_put(p, 32 * j + lane, x, delta);
        }
    }
    contrib = warp_sum(contrib);
    if (lane == 0 && contrib != 0.0) bc_add(p.bc + x, contrib);
}

// 32 vertices per warp step: lane i tests vertex base + i, then the warp
// finalises the ones at level L (most vertices are not at any given level)
template <int W, bool COEF, typename RT = double>
__global__ void __launch_bounds__(BC_NT) lanes_bwd_finalize_kernel(LanesParams p, double *__restrict__ A) {
    if ((p.prev_new && *p.prev_new == 0) || gated_off(p)) return;
    const int lane = lane_id();
    const int nwarps = (int)((gridDim.x * (size_t)BC_NT) >> 5);
    RT *__restrict__ S = reinterpret_cast<RT *>(p.S_cur);
    for (int base = (int)(((size_t)blockIdx.x * BC_NT + threadIdx.x) >> 5) * 32; base < p.n; base += nwarps * 32) {
        bool mine = false;
        if (base + lane < p.n) {
            uint64_t mm[W];
            load_mask<W>(p.mask_cur + (size_t)(base + lane) * W, mm);
#pragma unroll
            for (int j = 0; j < W; ++j) mine |= mm[j] != 0;
        }
        unsigned todo = __ballot_sync(0xffffffffu, mine);
        while (todo) {
            const int x = base + __ffs(todo) - 1;
            todo &= todo - 1;
            bwd_finalize_vertex<W, COEF, RT>(p, A, S, x, lane);
        }
    }
}

// Hubs at level L after the fused push: BC and the re-zeroing of A (their
// adjacency segments ran on several CTAs; warp per hub)
template <int W, typename RT = double>
__global__ void __launch_bounds__(BC_NT) lanes_bwd_hub_fin_kernel(LanesParams p, double *__restrict__ A) {
    if ((p.prev_new && *p.prev_new == 0) || gated_off(p)) return;
    const int h = (int)(((size_t)blockIdx.x * BC_NT + threadIdx.x) >> 5);
    if (h >= p.nhub) return;
    const int x = p.hub_ids[h];
    uint64_t m[W];
    load_mask<W>(p.mask_cur + (size_t)x * W, m);
    bool any = false;
#pragma unroll
    for (int j = 0; j < W; ++j) any |= m[j] != 0;
    if (any) bwd_finalize_vertex<W, false, RT>(p, A, reinterpret_cast<RT *>(p.S_cur), x, lane_id());
}

// FWD = true: forward push for a small frontier (level L -> L+1): every
// frontier vertex x pushes sigma_L(x) into A[y] of each neighbour y in the
// lanes c = lvl[L][x] & active & ~seen[y] and ORs c into lvl[L+1][y];
// lanes_fwd_commit_kernel then turns A into the level-(L+1) sigma rows.
// FWD = false: the backward push described above.
template <int W, bool FWD, typename RT = double>
struct PushKernel {
    static_assert(!FWD || std::is_same<RT, double>::value, "forward push uses fp64 rows");
    static constexpr int K = 64 * W, NG = 2 * W;
    static constexpr int R = (W >= 4) ? BC_PR4 : 4;  // item steps in flight per warp
    const LanesParams &p;
    double *A;
    PushSmem<W> &sm;
    const int lane, wid;
#ifndef BC_PUSH_CNT32
#define BC_PUSH_CNT32 1  // 32-bit per-thread counters (fewer live registers in the hit loop)
#endif
#if BC_PUSH_CNT32
    unsigned st_items = 0, st_hits = 0, st_dag = 0;  // per thread per launch: < 2^32 items / hits
#else
    unsigned long long st_items = 0, st_hits = 0, st_dag = 0;
#endif

    __device__ PushKernel(const LanesParams &pp, double *a, PushSmem<W> &s)
        : p(pp), A(a), sm(s), lane(lane_id()), wid(warp_id()) {}

    // one warp: items [ws, we) of the slots in sm; u[slot] = lvl[L][x]
    // backward, fused finalize: coef of slot hs (vertex x at level L) from
    // sigma_L(x) and the accumulator A[x] (complete: all children pushed at
    // L+1), coef = (1 + omega + delta) / sigma, delta = sigma * A   (Eq.5).
    // A slot owned by this warp alone is finalised here (BC, A := 0); split
    // slots after the tile, hubs by lanes_bwd_hub_fin_kernel.
    __device__ __forceinline__ void slot_coef(int hs, bool owned, double (&cf)[NG]) {
        const int x = sm.vert[hs];
        uint32_t bits = 0;
#pragma unroll
        for (int j = 0; j < NG; ++j)
            bits |= (((uint32_t)(sm.u[hs * W + (j >> 1)] >> ((j & 1) * 32)) >> lane) & 1u) << j;
        const RT *row = reinterpret_cast<const RT *>(p.S_cur) + (size_t)x * K;
        double *arow = A_ROW(A, x) + lane;
    const size_t ag = A_GRP(p);
        const double om = p.omega ? (double)p.omega[x] : 0.0;
        double contrib = 0.0;
        // two halves of the groups (bounded live registers: cf stays live in the hit loop)
#pragma unroll
        for (int h = 0; h < NG; h += NG / 2) {
            double sv[NG / 2], av[NG / 2];
#pragma unroll
            for (int q = 0; q < NG / 2; ++q) {
                sv[q] = 1.0;
                av[q] = 0.0;
                if (bits >> (h + q) & 1u) {
#if BC_PUSH_OWN_HINT == 2
                    if constexpr (std::is_same<RT, uint16_t>::value) {
                        unsigned short t;
                        asm volatile("ld.global.L2::cache_hint.u16 %0, [%1], %2;"
                                     : "=h"(t) : "l"(row + row_idx<W, RT>(32 * (h + q) + lane)), "l"(policy_evict_first()));
                        sv[q] = (double)t;
                    } else {
                        sv[q] = (double)row[row_idx<W, RT>(32 * (h + q) + lane)];
                    }
#else
                    sv[q] = (double)row[row_idx<W, RT>(32 * (h + q) + lane)];
#endif
#if BC_PUSH_OWN_HINT
                    av[q] = ld_ef_f64(arow + (h + q) * ag, policy_evict_first());
#else
                    av[q] = arow[(h + q) * ag];
#endif
                }
            }
#pragma unroll
            for (int q = 0; q < NG / 2; ++q) {
                const int j = h + q;
                cf[j] = 0.0;
                if (bits >> j & 1u) {
                    const double delta = sv[q] * av[q];
                    cf[j] = (1.0 + om + delta) * rcp_f64(sv[q]);
                    if (owned) {
#if BC_PUSH_OWN_HINT
                        st_ef_f64(arow + j * ag, 0.0, policy_evict_first());
#else
                        arow[j * ag] = 0.0;
#endif
                        contrib += p.lane_w1[32 * j + lane] * (delta + om);
                        cap_delta_put(p, 32 * j + lane, x, delta);
                    }
                }
            }
        }
        if (owned) {  // warp-uniform
            contrib = warp_sum(contrib);
            if (lane == 0 && contrib != 0.0) bc_add(p.bc + x, contrib);
        }
    }

    // ---- compacted backward push (BC_PUSH_COMPACT).  At a slot change the
    // warp lists the slot's level-L lanes u = lvl[L][x] in lane order (a warp
    // scan over 2W-lane chunks) and thread t takes the u-ranks t, t+32, ...:
    // nr = ceil(|u| / 32) rounds.  coef is formed for those lanes only, and
    // a hit (x, y, c) costs nr rounds of one red each (a lane of u outside
    // c skips its red) instead of 2W lane groups of mostly idle threads.  The
    // lanes of one round are increasing, so a red instruction touches the
    // same L2 sectors of A[y] as the group form.
    // lp[r / 2] holds the lane of round r in its 16-bit half r % 2 (0xffff:
    // no lane of u has rank lane + 32 r).
    __device__ __forceinline__ int compact_slot(int hs, uint32_t (&lp)[NG / 2], int &tot) {
        constexpr int CH = 2 * W;  // lanes per thread chunk (<= 16)
        const int l0 = lane * CH;
        const uint64_t uw = sm.u[hs * W + (l0 >> 6)];
        uint32_t bits = (uint32_t)(uw >> (l0 & 63)) & ((1u << CH) - 1u);
        const int cnt = __popc(bits);
        const int incl = warp_incl_scan(cnt);
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        uint16_t *lst = sm.lst + wid * K;
        int pos = incl - cnt;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            lst[pos++] = (uint16_t)(l0 + b);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NG / 2; ++q) {
            const int k0 = lane + 64 * q, k1 = k0 + 32;
            const uint32_t a = k0 < total ? lst[k0] : 0xffffu, b = k1 < total ? lst[k1] : 0xffffu;
            lp[q] = a | (b << 16);
        }
        __syncwarp();  // the list is rewritten at the next slot change
        tot = total;
        return (total + 31) >> 5;
    }
    __device__ __forceinline__ static int lane_at(const uint32_t (&lp)[NG / 2], int r) {
        return (int)((lp[r >> 1] >> ((r & 1) * 16)) & 0xffffu);
    }

    // coef of the compacted lanes of slot hs (x at level L), Eq.(5) as in
    // slot_coef; an owned slot is also finalised (BC, A[x] := 0)
    __device__ __forceinline__ void slot_coef_c(int hs, bool owned, int nr, const uint32_t (&lp)[NG / 2],
                                                double (&cf)[NG]) {
        const int x = sm.vert[hs];
        const RT *row = reinterpret_cast<const RT *>(p.S_cur) + (size_t)x * K;
        double *arow = A_ROW(A, x);
        const size_t ag = A_GRP(p);
        const double om = p.omega ? (double)p.omega[x] : 0.0;
        double contrib = 0.0;
#pragma unroll
        for (int h = 0; h < NG; h += NG / 2) {
            double sv[NG / 2], av[NG / 2];
#pragma unroll
            for (int q = 0; q < NG / 2; ++q) {
                const int l = lane_at(lp, h + q);
                sv[q] = 1.0;
                av[q] = 0.0;
                if (h + q < nr && l < K) {
                    sv[q] = (double)row[row_idx<W, RT>(l)];
                    av[q] = arow[(size_t)(l >> 5) * ag + (l & 31)];
                }
            }
#pragma unroll
            for (int q = 0; q < NG / 2; ++q) {
                const int r = h + q, l = lane_at(lp, r);
                cf[r] = 0.0;
                if (r < nr && l < K) {
                    const double delta = sv[q] * av[q];
                    cf[r] = (1.0 + om + delta) * rcp_f64(sv[q]);
                    if (owned) {
                        arow[(size_t)(l >> 5) * ag + (l & 31)] = 0.0;
                        contrib += p.lane_w1[l] * (delta + om);
                        cap_delta_put(p, l, x, delta);
                    }
                }
            }
        }
        if (owned) {  // warp-uniform
            contrib = warp_sum(contrib);
            if (lane == 0 && contrib != 0.0) bc_add(p.bc + x, contrib);
        }
    }

    __device__ void warp_push_compact(int nslots, int ws, int we, bool hub_mode) {
        const uint64_t *mpar = p.mask_nxt_ro;  // lvl[L-1] (parents)
        bool has_derived = false;
#pragma unroll
        for (int j = 0; j < W; ++j) has_derived |= p.derived[j] != 0;
        const uint64_t pol = policy_evict_first();
        int cur = -1, nr = 0, tot = 0;
        uint32_t lp[NG / 2];
        double cf[NG];
#pragma unroll
        for (int j = 0; j < NG; ++j) cf[j] = 0.0;
#pragma unroll
        for (int q = 0; q < NG / 2; ++q) lp[q] = 0xffffffffu;
        st_items += (lane == 0) ? (we - ws) : 0;
        for (int e0 = ws; e0 < we; e0 += 32 * R) {
            int sl[R], vv[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int e = e0 + k * 32 + lane;
                sl[k] = -1;
                vv[k] = 0;
                if (e < we) {
                    const int s = slot_of(sm.cd, nslots, e);
                    sl[k] = s;
                    vv[k] = ld_stream(p.col + sm.rs[s] + (e - sm.cd[s]), pol);
                    BC_CHECK(s >= 0 && s < nslots && vv[k] >= 0 && vv[k] < p.n);
                }
            }
            uint64_t cc[R][W];
#pragma unroll
            for (int k = 0; k < R; ++k) {
#pragma unroll
                for (int j = 0; j < W; ++j) cc[k][j] = 0;
                if (sl[k] >= 0) {
                    load_mask<W>(mpar + (size_t)vv[k] * W, cc[k]);
#pragma unroll
                    for (int j = 0; j < W; ++j) cc[k][j] &= sm.u[sl[k] * W + j];
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                bool h = false;
#pragma unroll
                for (int j = 0; j < W; ++j) h |= cc[k][j] != 0;
                unsigned hm = __ballot_sync(0xffffffffu, h);
                st_hits += (lane == 0) ? __popc(hm) : 0;
                if (hm == 0) continue;
                int4 *hsv = sm.hsv + wid * 32;
                hsv[lane] = make_int4(sl[k], vv[k], 0, 0);
#pragma unroll
                for (int j = 0; j < W; ++j) sm.hc[(wid * 32 + lane) * W + j] = cc[k][j];
                __syncwarp();
                while (hm) {
                    const int src = __ffs(hm) - 1;
                    hm &= hm - 1;
                    const int2 rec = *reinterpret_cast<const int2 *>(hsv + src);
                    const int hs = rec.x, y = rec.y;
                    if (hs != cur) {  // warp-uniform: compact the new slot's lanes, form their coef
                        cur = hs;
                        nr = compact_slot(hs, lp, tot);
                        slot_coef_c(hs, !hub_mode && sm.cd[hs] >= ws && sm.cd[hs + 1] <= we, nr, lp, cf);
                    }
                    const uint32_t *c32 = reinterpret_cast<const uint32_t *>(sm.hc + (wid * 32 + src) * W);
                    if (has_derived && lane == 0) {  // only with BC_OPT_TWO_DEGREE: derived lanes' DAG edges
#pragma unroll
                        for (int j = 0; j < W; ++j) st_dag += __popcll(sm.hc[(wid * 32 + src) * W + j] & p.derived[j]);
                    }
                    double *arow = A_ROW(A, y);
                    static_assert(!BC_A_PLANES || !BC_PUSH_COMPACT, "compact push uses row-major accumulators");
#pragma unroll
                    for (int r = 0; r < NG; ++r) {
                        if (r < nr) {  // uniform
                            const int l = lane_at(lp, r);
                            const uint32_t on = l < K ? (c32[l >> 5] >> (l & 31)) & 1u : 0u;
#ifdef BC_EXP_NORED  // experiment build only: traversal cost without the reds (wrong results)
                            red_add_f64_if(arow + (l & (K - 1)), cf[r], on & (cf[r] == -1.0));
#elif defined(BC_PUSH_DENSE)  // experiment: full rounds red 0.0 for the slot's lanes outside c (no branch)
                            if ((r + 1) * 32 <= tot) red_add_f64(arow + l, on ? cf[r] : 0.0);
                            else red_add_f64_if(arow + (l & (K - 1)), cf[r], on);
#else
                            red_add_f64_if(arow + (l & (K - 1)), cf[r], on);
#endif
                        }
                    }
                }
                __syncwarp();
            }
        }
    }

    __device__ void warp_push(int nslots, int ws, int we, bool hub_mode) {
        if constexpr (!FWD && BC_PUSH_COMPACT) {
            warp_push_compact(nslots, ws, we, hub_mode);
            return;
        }
        const uint64_t *mpar = FWD ? p.seen : p.mask_nxt_ro;  // fwd: seen[y]; bwd: lvl[L-1] (parents)
        bool has_derived = false;
#pragma unroll
        for (int j = 0; j < W; ++j) has_derived |= p.derived[j] != 0;
        const double *S = reinterpret_cast<const double *>(p.S_cur);
        const uint64_t pol = policy_evict_first();
        int cur = -1;
        double cf[NG];
#pragma unroll
        for (int j = 0; j < NG; ++j) cf[j] = 0.0;
        st_items += (lane == 0) ? (we - ws) : 0;
        for (int e0 = ws; e0 < we; e0 += 32 * R) {
            int sl[R], vv[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int e = e0 + k * 32 + lane;
                sl[k] = -1;
                vv[k] = 0;
                if (e < we) {
                    const int s = slot_of(sm.cd, nslots, e);
                    sl[k] = s;
                    vv[k] = ld_stream(p.col + sm.rs[s] + (e - sm.cd[s]), pol);
                    BC_CHECK(s >= 0 && s < nslots && vv[k] >= 0 && vv[k] < p.n);
                }
            }
            uint64_t cc[R][W];
#pragma unroll
            for (int k = 0; k < R; ++k) {
#pragma unroll
                for (int j = 0; j < W; ++j) cc[k][j] = 0;
                if (sl[k] >= 0) {
#if BC_PUSH_MASK_HINT
                    {
                        const uint64_t mpol = BC_PUSH_MASK_HINT == 1 ? policy_evict_first() : policy_evict_last();
                        if constexpr (W >= 2) {
#pragma unroll
                            for (int j = 0; j < W; j += 2) {
                                const ulonglong2 t =
                                    ld_pol(reinterpret_cast<const ulonglong2 *>(mpar + (size_t)vv[k] * W + j), mpol);
                                cc[k][j] = t.x;
                                cc[k][j + 1] = t.y;
                            }
                        } else {
                            load_mask<W>(mpar + (size_t)vv[k] * W, cc[k]);
                        }
                    }
#else
                    load_mask<W>(mpar + (size_t)vv[k] * W, cc[k]);
#endif
#pragma unroll
                    for (int j = 0; j < W; ++j) {
                        if (FWD) cc[k][j] = p.active[j] & ~cc[k][j];
                        cc[k][j] &= sm.u[sl[k] * W + j];
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                uint32_t gmk = 0;
#pragma unroll
                for (int j = 0; j < NG; ++j)
                    if ((uint32_t)(cc[k][j >> 1] >> ((j & 1) * 32))) gmk |= 1u << j;
                unsigned hm = __ballot_sync(0xffffffffu, gmk != 0);
                st_hits += (lane == 0) ? __popc(hm) : 0;
                if (hm == 0) continue;
                int4 *hsv = sm.hsv + wid * 32;
                hsv[lane] = make_int4(sl[k], vv[k], (int)gmk, 0);
#pragma unroll
                for (int j = 0; j < W; ++j) sm.hc[(wid * 32 + lane) * W + j] = cc[k][j];
                __syncwarp();
                while (hm) {
                    const int src = __ffs(hm) - 1;
                    hm &= hm - 1;
                    const int4 rec = hsv[src];
                    const int hs = rec.x, y = rec.y;
                    const uint32_t gm = (uint32_t)rec.z;
                    if (hs != cur) {  // warp-uniform: coef of the new slot
                        cur = hs;
                        if constexpr (FWD) {
                            const double *row = S + (size_t)sm.vert[hs] * K + lane;
#pragma unroll
                            for (int j = 0; j < NG; ++j) cf[j] = row[32 * j];
                        } else {
                            slot_coef(hs, !hub_mode && sm.cd[hs] >= ws && sm.cd[hs + 1] <= we, cf);
                            if constexpr (PushSmem<W>::CFS) {
                                __syncwarp();  // the previous slot's row is no longer read
#pragma unroll
                                for (int j = 0; j < NG; ++j) sm.cfs[wid * K + 32 * j + lane] = cf[j];
                                __syncwarp();
                            }
                        }
                    }
                    double *arow = A_ROW(A, y) + lane;
                    size_t ag = A_GRP(p);
                    if (!FWD && BC_REP_H > 0 && y < BC_REP_H && p.arep) {  // uniform: a hub parent's replica
                        arow = p.arep + ((size_t)(blockIdx.x % BC_REP_R) * BC_REP_H + y) * K + lane;
                        ag = 32;
                    }
                    uint64_t myword = 0;  // fwd: thread j < W ORs word j of c into lvl[L+1][y]
                    uint64_t cwords[W];
                    static_assert(W <= 8, "");
#pragma unroll
                    for (int j = 0; j < W; j += (W >= 2 ? 2 : 1)) {
                        if constexpr (W >= 2) {
                            const ulonglong2 t = reinterpret_cast<const ulonglong2 *>(sm.hc + (wid * 32 + src) * W)[j / 2];
                            cwords[j] = t.x;
                            cwords[j + 1] = t.y;
                        } else {
                            cwords[0] = sm.hc[wid * 32 + src];
                        }
                    }
                    if (!FWD && has_derived) {  // uniform; only with BC_OPT_TWO_DEGREE
                        // DAG edges of 2-degree lanes (their forward was derived, not traversed)
                        if (lane == 0) {
#pragma unroll
                            for (int j = 0; j < W; ++j) st_dag += __popcll(cwords[j] & p.derived[j]);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < NG; ++j) {
                        if (gm >> j & 1u) {  // uniform
                            const uint32_t cw = (uint32_t)(cwords[j >> 1] >> ((j & 1) * 32));
#ifdef BC_EXP_NORED  // experiment build only: traversal cost without the reds (wrong results)
                            red_add_f64_if(arow + j * ag, cf[j], (cw >> lane & 1u) & (cf[j] == -1.0));
#elif defined(BC_EXP_REDZERO)  // experiment: unpredicated red of 0.0 outside c (more L2 sectors, no branches)
                            red_add_f64(arow + j * ag, (cw >> lane & 1u) ? cf[j] : 0.0);
#else
                            red_add_f64_if(arow + j * ag, (!FWD && PushSmem<W>::CFS) ? sm.cfs[wid * K + 32 * j + lane] : cf[j],
                                           cw >> lane & 1u);
#endif
                            if (FWD) st_dag += cw >> lane & 1u;
                            if (FWD && lane == (j >> 1)) myword |= (uint64_t)cw << ((j & 1) * 32);
                        }
                    }
                    if (FWD && myword) atomicOr((unsigned long long *)(p.mask_nxt + (size_t)y * W + lane),
                                                (unsigned long long)myword);
                }
                __syncwarp();
            }
        }
    }

    __device__ __forceinline__ static int bnd(int j, int nitems) {
        return (int)(((long long)j * nitems) / BC_NW);
    }

    __device__ void tile(int t) {
        const int v0 = p.tile_vs[t], v1 = p.tile_vs[t + 1];
        const int x = v0 + threadIdx.x;
        int deg = 0, act = 0, rs = 0;
        uint64_t u[W];
#pragma unroll
        for (int j = 0; j < W; ++j) u[j] = 0;
        if (x < v1) {
            rs = p.rp[x];
            deg = p.rp[x + 1] - rs;
            if (deg > 0 && deg <= p.hub_deg) {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    u[j] = p.mask_cur[(size_t)x * W + j];
                    act |= (u[j] != 0);
                }
            }
        }
        int slot, cd, nslots, nitems;
        block_excl_scan2(act, act ? deg : 0, slot, cd, nslots, nitems, sm.scan);
        if (act) {
            sm.vert[slot] = x;
            sm.cd[slot] = cd;
            sm.rs[slot] = rs;
#pragma unroll
            for (int j = 0; j < W; ++j) sm.u[slot * W + j] = u[j];
        }
        if (threadIdx.x == 0) sm.cd[nslots] = nitems;
        __syncthreads();
        if (nslots > 0) {
            const int ws = bnd(wid, nitems), we = bnd(wid + 1, nitems);
            if (ws < we) warp_push(nslots, ws, we, false);
            if (!FWD) {
                __syncthreads();
                // slots split across warps: warp j finalises the slot holding boundary j
                if (wid >= 1) {
                    const int b = bnd(wid, nitems);
                    if (b > 0 && b < nitems) {
                        const int s = slot_of(sm.cd, nslots, b);
                        if (sm.cd[s] < b && (wid == 1 || bnd(wid - 1, nitems) <= sm.cd[s]))
                            bwd_finalize_vertex<W, false, RT>(p, A, reinterpret_cast<RT *>(p.S_cur), sm.vert[s], lane);
                    }
                }
            }
        }
        __syncthreads();
    }

    __device__ void hub_segment(int unit) {
        if (threadIdx.x == 0) {
            int lo = 0, hi = p.nhub - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (p.hub_seg_off[mid] <= unit) lo = mid;
                else hi = mid - 1;
            }
            sm.scan[0] = lo;
        }
        __syncthreads();
        const int h = sm.scan[0];
        __syncthreads();
        const int x = p.hub_ids[h];
        const int seg = unit - p.hub_seg_off[h];
        const int a = p.rp[x] + seg * p.seg_len;
        const int b = min(p.rp[x + 1], a + p.seg_len);
        uint64_t u[W];
        bool any = false;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            u[j] = p.mask_cur[(size_t)x * W + j];
            any |= (u[j] != 0);
        }
        if (any) {
            if (threadIdx.x == 0) {
                sm.vert[0] = x;
                sm.cd[0] = 0;
                sm.cd[1] = b - a;
                sm.rs[0] = a;
#pragma unroll
                for (int j = 0; j < W; ++j) sm.u[j] = u[j];
            }
            __syncthreads();
            const int nitems = b - a;
            const int ws = bnd(wid, nitems), we = bnd(wid + 1, nitems);
            if (ws < we) warp_push(1, ws, we, true);
        }
        __syncthreads();
    }

    __device__ void epilogue() {
        const unsigned long long it = warp_sum_u64((unsigned long long)st_items),
                                 ht = warp_sum_u64((unsigned long long)st_hits),
                                 dg = warp_sum_u64((unsigned long long)st_dag);
        if (lane == 0) {
            if (it) atomicAdd(p.stats + (FWD ? 4 : 6), it);
            if (ht) atomicAdd(p.stats + (FWD ? 5 : 7), ht);
            if (dg) atomicAdd(p.stats + 2, dg);
        }
    }
};

template <int W, bool FWD, typename RT = double>
__global__ void __launch_bounds__(BC_NT, (W == 8 ? BC_PUSH_MINB8 : BC_PUSH_MINB)) lanes_push_kernel(LanesParams p, double *A) {
    // forward: speculative launch past the last level; backward (device-driven
    // batch): level L empty.  Either: tier not in use
    if ((p.prev_new && *p.prev_new == 0) || gated_off(p)) return;
    __shared__ PushSmem<W> sm;
    PushKernel<W, FWD, RT> k(p, A, sm);
    const int total = p.nseg + p.ntiles;
    for (;;) {
        if (threadIdx.x == 0) {
            const int t = atomicAdd(p.work_ctr, 1);
            if (t == total + (int)gridDim.x - 1) *p.work_ctr = 0;  // last fetch resets
            sm.unit = t;
        }
        __syncthreads();
        const int unit = sm.unit;
        __syncthreads();
        if (unit >= total) break;
        if (unit < p.nseg) k.hub_segment(unit);
        else k.tile(unit - p.nseg);
    }
    k.epilogue();
}

// Forward commit after a push level: x with lvl[L+1][x] != 0 gets its
// level-(L+1) sigma row from A (zeros outside the new lanes), A is re-zeroed,
// seen is updated (warp per vertex, strided lanes).
template <int W>
__global__ void __launch_bounds__(BC_NT) lanes_fwd_commit_kernel(LanesParams p, double *__restrict__ A) {
    constexpr int K = 64 * W, NG = 2 * W;
    if (p.prev_new && *p.prev_new == 0) return;
    __shared__ double ns_sm[K];
    const int lane = lane_id();
    if (p.lane_ns) {
        for (int l = threadIdx.x; l < K; l += BC_NT) ns_sm[l] = 0.0;
        __syncthreads();
    }
    const int nwarps = (int)((gridDim.x * (size_t)BC_NT) >> 5);
    double *__restrict__ S = reinterpret_cast<double *>(p.S_nxt);
    unsigned long long st_reach = 0, st_adj = 0, st_dsum = 0;
    int any_new = 0;
    for (int x = (int)(((size_t)blockIdx.x * BC_NT + threadIdx.x) >> 5); x < p.n; x += nwarps) {
        uint64_t m[W];
        bool any = false;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            m[j] = p.mask_nxt[(size_t)x * W + j];
            any |= m[j] != 0;
        }
        if (!any) continue;  // warp-uniform
        double *arow = A_ROW(A, x) + lane;
    const size_t ag = A_GRP(p);
        double *row = S + (size_t)x * K + lane;
        double av[NG];
        uint32_t bits = 0;
#pragma unroll
        for (int j = 0; j < NG; ++j) {
            bits |= (((uint32_t)(m[j >> 1] >> ((j & 1) * 32)) >> lane) & 1u) << j;
            av[j] = (bits >> j & 1u) ? arow[j * ag] : 0.0;
        }
        const double wx = 1.0 + (p.omega ? (double)p.omega[x] : 0.0);
#pragma unroll
        for (int j = 0; j < NG; ++j) {
            row[32 * j] = av[j];
            if (bits >> j & 1u) {
                arow[j * ag] = 0.0;
                if (p.lane_ns) atomicAdd(&ns_sm[32 * j + lane], wx);
            }
        }
        if (lane < W) p.seen[(size_t)x * W + lane] |= m[lane];
        const int pc = __popc(bits);
        const int deg = p.rp[x + 1] - p.rp[x];
        st_reach += pc;
        st_adj += (unsigned long long)pc * deg;
        st_dsum += (unsigned long long)pc * (unsigned)(p.level + 1);
        any_new = 1;
    }
    const unsigned long long a = warp_sum_u64(st_reach), b = warp_sum_u64(st_adj), d = warp_sum_u64(st_dsum);
    if (lane == 0) {
        if (a) atomicAdd(p.stats + 0, a);
        if (b) atomicAdd(p.stats + 1, b);
        if (d) atomicAdd(p.stats + 3, d);
    }
    if (__any_sync(0xffffffffu, any_new) && lane == 0) *p.any_new = 1;
    if (p.lane_ns) {
        __syncthreads();
        for (int l = threadIdx.x; l < K; l += BC_NT)
            if (ns_sm[l] != 0.0) atomicAdd(p.lane_ns + l, ns_sm[l]);
    }
}

}  // namespace bcb
