// lanes.cuh -- multi-source ("bit-lane") Brandes level kernels for sm_100a.
//
// A batch holds K = 64*W sources; source j of the batch is lane j.  Per
// vertex v the batch keeps
//   lvl[L][v]  : W x uint64 -- lanes whose BFS puts v at depth L
//   seen[v]    : W x uint64 -- lanes that have discovered v
//   S_L[v][K]  : per level L, the row of v holds sigma_s(v) in the lanes
//                where v is at depth L and exact zeros elsewhere (written
//                whole by the commit that discovers v at L); the backward
//                sweep overwrites it in place with
//                coef_s(v) = (1 + omega(v) + delta_s(v)) / sigma_s(v)
//                (zeros outside level L).  Zero-filled level rows let a
//                gather add whole lane pairs without per-lane masking.
//
// Forward level L -> L+1 (Alg.2 / Alg.3; Alg.1 lines
// 9-22): every vertex x with undiscovered lanes u = active & ~seen[x] pulls
// from its neighbours v: c = u & lvl[L][v]; for each lane in c,
// sigma(x) += sigma(v).  New lanes = lanes with sigma(x) > 0; they form
// lvl[L+1][x].  Discovery is owner-computes (one CTA owns x), so neither the
// depth nor sigma needs an atomic (reading R4 of DESIGN.md replaces Alg.3's
// racy bmap test-and-set).
//
// Backward level L (Alg.4 / Alg.5, successor checking,
// reading R2): every x with m = lvl[L][x] != 0 sums over successors v
// (lanes in c = m & lvl[L+1][v]) acc += coef(v); then
//   delta(x) = sigma(x) * acc                  (updateDep)
//   coef(x)  = (1 + omega(x) + delta(x)) / sigma(x)        (Eq.5, line 1)
//   BC[x]   += sum_lanes (1 + omega(s)) * (delta(x) + omega(x))    (R13)
//
// Edge-to-thread mapping ("active-edge parallelism"): a
// CTA takes a tile of <= TV consecutive vertex ids, keeps the active ones,
// block-scans their degrees into a shared-memory CD array (the frontier
// offsets of the tile) and splits the tile's items evenly over its warps;
// an item e is mapped to its vertex by binary search in CD.  Items are read
// 32 consecutive per warp instruction (coalesced col reads) and several
// steps are in flight per thread.  Vertices of degree > hub_deg are "hubs":
// their adjacency is cut into segments (separate work units, any CTA) whose
// partial sums meet in a per-hub scratch row via fp64 red.add, finalised by
// lanes_hub_finalize.
#pragma once
#include <type_traits>
#include "util.cuh"

namespace bcb {

constexpr int TV = BC_NT;  // vertices per tile

template <typename T> struct Vec2;
template <> struct Vec2<double> { using t = double2; };
template <> struct Vec2<unsigned long long> { using t = ulonglong2; };
template <> struct Vec2<unsigned> { using t = uint2; };
template <> struct Vec2<long long> { using t = longlong2; };

// Storage type of the level sigma rows for an accumulator type SigT.
// SigT = unsigned is the *narrow* forward: sigma rows hold uint16 (4x fewer
// row bytes gathered and written than fp64); sums are formed in 32-bit
// registers and any sigma > 65535 raises LanesParams::narrow_ovf, after which
// the host re-runs the batch with fp64 rows.  Integer sigma is exact, so
// the narrow and fp64 forwards produce identical sigma wherever both fit
// (R-MAT: max sigma ~1e4 at scale 20, SURVEY.md section 8 constants table).
// SigT = long long is the *mid* tier: uint32 rows, 64-bit sums, limit
// 2^32 - 1 (the fallback of a 16-bit batch before fp64).
template <typename SigT> struct RowOf { using t = SigT; };
template <> struct RowOf<unsigned> { using t = uint16_t; };
template <> struct RowOf<long long> { using t = uint32_t; };

#ifndef BC_NARROW_TMAJOR
#define BC_NARROW_TMAJOR 1  // 16-bit sigma rows thread-major (a thread's W lane pairs are one vector)
#endif
// Position of lane l in a sigma row.  16-bit rows are stored thread-major:
// the pair (2t, 2t+1) of 64-lane word i -- owned by thread t of the level
// kernels -- is 32-bit word t*W + i, so a thread gathers or writes its W
// pairs of a row with one W*4-byte vector access (16 B at W = 4).  Wider
// rows keep lane order.
template <int W, typename RT>
__host__ __device__ __forceinline__ int row_idx(int l) {
    if constexpr (BC_NARROW_TMAJOR && std::is_same<RT, uint16_t>::value)
        return (((l & 63) >> 1) * W + (l >> 6)) * 2 + (l & 1);
    else
        return l;
}
template <typename SigT> struct RowLimit { static constexpr unsigned long long v = 0; };
template <> struct RowLimit<unsigned> { static constexpr unsigned long long v = 65535ull; };
template <> struct RowLimit<long long> { static constexpr unsigned long long v = 4294967295ull; };

// 16-byte read-only load with an L2 cache policy
__device__ __forceinline__ double2 ld_pol(const double2 *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ ulonglong2 ld_pol(const ulonglong2 *p, uint64_t pol) {
    ulonglong2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;" : "=l"(v.x), "=l"(v.y) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---- Blackwell bulk copies (TMA engine, cp.async.bulk) with mbarrier completion
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *mb, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// one arrival that also announces `bytes` of transaction (the bulk copy's completion)
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *mb, uint32_t bytes) {
    uint64_t state;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
                 : "=l"(state) : "r"(smem_u32(mb)), "r"(bytes) : "memory");
    (void)state;
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t *mb, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(mb)), "r"(parity) : "memory");
    } while (!ok);
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16-byte aligned), completing on mb
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)) : "memory");
}
// order earlier generic-proxy accesses of shared memory before later async-proxy (bulk copy) writes
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

#ifndef BC_FWD_MASK_HINT
#define BC_FWD_MASK_HINT 1  // L2 policy of the forward's item mask loads (lvl[L][v]): 0 none, else evict_last (forward 85.0 -> 84.65 ms, profiles/exp_r2_hints3.txt)
#endif
#ifndef BC_FWD_ROW_HINT
#define BC_FWD_ROW_HINT 2  // L2 policy of the 16-bit forward's sigma-row gathers: 0 none, 1 evict_first, 2 evict_last (~1 %, profiles/exp_r2_fwd_rowhint.txt)
#endif
// a 32-bit word of a 16-bit sigma row (read-only path, optional L2 policy)
__device__ __forceinline__ uint32_t ld_row_word(const uint32_t *p, uint64_t pol) {
#if BC_FWD_ROW_HINT
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}
// a thread's W consecutive 32-bit words of a thread-major 16-bit row
template <int W>
__device__ __forceinline__ void ld_row_vec(const uint32_t *p, uint64_t pol, uint32_t (&t)[W]) {
    if constexpr (W >= 4) {
#pragma unroll
        for (int q = 0; q < W; q += 4) {
#if BC_FWD_ROW_HINT
            asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                         : "=r"(t[q]), "=r"(t[q + 1]), "=r"(t[q + 2]), "=r"(t[q + 3]) : "l"(p + q), "l"(pol));
#else
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p + q));
            t[q] = v.x, t[q + 1] = v.y, t[q + 2] = v.z, t[q + 3] = v.w;
#endif
        }
    } else if constexpr (W == 2) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        t[0] = v.x, t[1] = v.y;
        (void)pol;
    } else {
        t[0] = ld_row_word(p, pol);
    }
}
template <int W>
__device__ __forceinline__ void st_row_vec(uint32_t *p, const uint32_t (&t)[W]) {
    if constexpr (W >= 4) {
#pragma unroll
        for (int q = 0; q < W; q += 4) *reinterpret_cast<uint4 *>(p + q) = make_uint4(t[q], t[q + 1], t[q + 2], t[q + 3]);
    } else if constexpr (W == 2) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(t[0], t[1]);
    } else {
        p[0] = t[0];
    }
}

__device__ __forceinline__ uint64_t row_policy() {
#if BC_FWD_ROW_HINT == 1
    return policy_evict_first();
#elif BC_FWD_ROW_HINT == 2
    return policy_evict_last();
#else
    return 0;
#endif
}

#ifndef BC_FWD_HIT2
#define BC_FWD_HIT2 1  // 16-bit forward: two hits per iteration, the second hit's row loads issued before the first is added
#endif
#ifndef BC_FWD_BULK
#define BC_FWD_BULK 0  // 1: 16-bit forward hit rows gathered by bulk copies into a per-warp shared ring (slower: profiles/exp_r2_fwd_bulk.txt)
#endif
// 16-byte async copy with zero fill when !valid, L2 cache policy
__device__ __forceinline__ void cp_async16z(void *smem_dst, const void *gsrc, bool valid, uint64_t pol) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(d), "l"(gsrc),
                 "r"(valid ? 16 : 0), "l"(pol)
                 : "memory");
}

// the W mask words of one vertex with as few L1 wavefronts as possible
// (one 16-byte load per two words; all words share one 32-byte sector)
template <int W>
__device__ __forceinline__ void load_mask(const uint64_t *p, uint64_t (&m)[W]) {
    if constexpr (W >= 2) {
#pragma unroll
        for (int j = 0; j < W; j += 2) {
            const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2 *>(p + j));
            m[j] = t.x;
            m[j + 1] = t.y;
        }
    } else {
        m[0] = __ldg(p);
    }
}

// the W words of one hit record in shared memory (broadcast reads)
template <int W>
__device__ __forceinline__ void load_mask_smem(const uint64_t *p, uint64_t (&m)[W]) {
    if constexpr (W >= 2) {
#pragma unroll
        for (int j = 0; j < W; j += 2) {
            const ulonglong2 t = *reinterpret_cast<const ulonglong2 *>(p + j);
            m[j] = t.x;
            m[j + 1] = t.y;
        }
    } else {
        m[0] = *p;
    }
}

// W 32-bit halves to / from shared memory with vector accesses
template <int W>
__device__ __forceinline__ void store_halves(uint32_t *d, const uint32_t (&h)[W]) {
    if constexpr (W == 8) {
        reinterpret_cast<uint4 *>(d)[0] = make_uint4(h[0], h[1], h[2], h[3]);
        reinterpret_cast<uint4 *>(d)[1] = make_uint4(h[4], h[5], h[6], h[7]);
    } else if constexpr (W == 4) *reinterpret_cast<uint4 *>(d) = make_uint4(h[0], h[1], h[2], h[3]);
    else if constexpr (W == 2) *reinterpret_cast<uint2 *>(d) = make_uint2(h[0], h[1]);
    else d[0] = h[0];
}
template <int W>
__device__ __forceinline__ void load_halves(const uint32_t *d, uint32_t (&h)[W]) {
    if constexpr (W == 8) {
        const uint4 t = reinterpret_cast<const uint4 *>(d)[0], u = reinterpret_cast<const uint4 *>(d)[1];
        h[0] = t.x; h[1] = t.y; h[2] = t.z; h[3] = t.w;
        h[4] = u.x; h[5] = u.y; h[6] = u.z; h[7] = u.w;
    } else if constexpr (W == 4) {
        const uint4 t = *reinterpret_cast<const uint4 *>(d);
        h[0] = t.x; h[1] = t.y; h[2] = t.z; h[3] = t.w;
    } else if constexpr (W == 2) {
        const uint2 t = *reinterpret_cast<const uint2 *>(d);
        h[0] = t.x; h[1] = t.y;
    } else {
        h[0] = d[0];
    }
}

struct LanesParams {
    int n;
    const int *rp;               // residual CSR row_ptr (int32, n+1)
    const int *col;              // residual CSR columns
    const uint32_t *omega;       // omega per vertex, nullable (unpruned)
    const uint64_t *mask_cur;    // lvl[L]
    const uint64_t *mask_nxt_ro; // backward: lvl[L+1]
    uint64_t *mask_nxt;          // forward: lvl[L+1], pre-zeroed
    uint64_t *seen;
    void *S_cur;                 // level-L rows [n][K] SigT (fwd: read sigma; bwd: sigma -> coef in place)
    void *S_nxt;                 // level-(L+1) rows (fwd: written; bwd: read coef)
    uint64_t *ovf;               // verify variant: per-lane sigma overflow bits [n][W]
    double *bc;
    const double *lane_w1;       // [K] 1 + omega(source of lane)
    double *lane_ns;             // [K] n_s accumulators, nullable
    unsigned long long *stats;   // [4] reached, adjacency reached, dag edges, depth sum
    int level;                   // L (forward: lvl[L] -> lvl[L+1]; backward: lvl[L])
    int *any_new;
    int *work_ctr;               // self-resetting dynamic tile counter
    uint64_t active[8];          // lanes in use (K <= 512)
    int hub_deg;
    int nhub;
    const int *hub_ids;
    const int *hub_seg_off;      // [nhub+1] prefix of segment counts
    int nseg;
    int seg_len;
    void *hub_acc;               // [nhub][K] SigT, zero between levels
    uint64_t *hub_ovf;           // verify: [nhub][W]
    int ntiles;
    const int *tile_vs;          // [ntiles+1] tile t = vertices [tile_vs[t], tile_vs[t+1]), <= TV of them
    const int *lane_cap;         // verification capture (bc_set_capture): [K] slot of a captured lane or -1, nullable
    double *cap_delta;           // ... backward: delta_s(x) of captured lanes, [slot][n] (compute ids)
    int *narrow_ovf;             // narrow forward: set when some sigma > 65535 (batch is re-run in fp64)
    uint64_t derived[8];         // 2-degree lanes (NEXT-1): tree derived from lanes l-2, l-1 after the forward
    const int *prev_new;         // forward: flag "level L is non-empty"; 0 -> the launch is a no-op
                                 // (levels are launched one ahead of the host's termination test)
    void *part;                  // [gridDim][BC_NW][2][K] SigT: partial sums of slots split across warps
    // device-driven batches (bc_api.cu graph mode; all nullable): the
    // batch's lanes in use come from device memory, and a launch is a
    // no-op unless *need != 0 and *halt == 0 (sigma-tier fallback)
    const uint64_t *active_dev;  // [8]
    const int *need;
    const int *halt;
    // backward: replicas of the accumulator rows of the BC_REP_H lowest ids
    // (the highest-degree parents), [BC_REP_R][BC_REP_H][K]; a push CTA reds
    // into copy blockIdx % BC_REP_R, lanes_rep_fold_kernel adds the copies
    // into A before each backward level; nullable (no replicas)
    double *arep;
};

__device__ __forceinline__ bool gated_off(const int *need, const int *halt) {
    return (need && *need == 0) || (halt && *halt != 0);
}
__device__ __forceinline__ bool gated_off(const LanesParams &p) { return gated_off(p.need, p.halt); }

// verification capture of delta_s(x) (bc_set_capture): lane l of the batch,
// vertex x; a no-op unless a capture is active (p.lane_cap != nullptr)
__device__ __forceinline__ void cap_delta_put(const LanesParams &p, int l, int x, double delta) {
    if (p.lane_cap) {
        const int c = p.lane_cap[l];
        if (c >= 0) p.cap_delta[(size_t)c * p.n + x] = delta;
    }
}

#ifndef BC_R4
#define BC_R4 1  // item steps in flight per warp at W = 4 (occupancy beats per-warp MLP)
#endif

template <int W, typename SigT>
struct LanesSmem {
    int vert[TV];
    int cd[TV + 1];
    int rs[TV];
    uint64_t u[TV * W];
    // per warp, per item of the step: the contributing-lane words c as 32-bit
    // halves [lo_0..lo_{W-1}, hi_0..hi_{W-1}] (thread t reads the W halves
    // holding its bits 2t, 2t+1 with one vector load)
    alignas(16) uint32_t hc[BC_NW * 32 * 2 * W];
    int2 hsv[BC_NW * 32];                     // per warp: (slot, v) of the step's items
    uint32_t povf[BC_NW * 2 * 32];
    double ns[64 * W];  // per-lane n_s partial sums of this CTA (pruned graphs)
    uint64_t act[8];    // lanes in use (from p.active_dev or p.active)
    unsigned long long st[6];  // CTA statistics (flushed from 32-bit thread counters per work unit)
    int scan[2 * BC_NW + 2];
    int unit;
    // 16-bit forward with BC_FWD_BULK: per warp a ring of RING sigma rows
    // (K x 16 bit) filled by bulk copies, one mbarrier per slot
    static constexpr bool BULK = BC_FWD_BULK && std::is_same<SigT, unsigned>::value;
    static constexpr int RING = BULK ? (W >= 8 ? 2 : (W == 4 ? 4 : 8)) : 1;
    alignas(128) uint32_t ring[BULK ? BC_NW * RING * 32 * W : 4];
    alignas(8) uint64_t mbar[BC_NW * RING];
};

// Lane -> thread mapping of the level kernel ("pair-strided"): thread t of
// a warp owns the LPT = 2W lanes lane_of(i) = 64*(i/2) + 2t + (i%2), i.e.
// bits 2t, 2t+1 of every mask word.  A row gather is then W 16-byte loads
// per thread whose warp footprint is W contiguous 512-byte spans (4 L1
// wavefronts each), and the thread's bits of any mask are pick2(words).
template <int W>
__device__ __forceinline__ uint32_t pick2(const uint64_t (&w)[W], int t2) {
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < W; ++j) r |= (uint32_t)((w[j] >> t2) & 3ull) << (2 * j);
    return r;
}
// bit t of a, b -> bits 2t, 2t+1 of the result
__device__ __forceinline__ uint64_t interleave2(uint32_t a, uint32_t b) {
    uint64_t x = a, y = b;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    y = (y | (y << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    y = (y | (y << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    y = (y | (y << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    y = (y | (y << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    y = (y | (y << 1)) & 0x5555555555555555ull;
    return x | (y << 1);
}
#ifndef BC_BC_RED
#define BC_BC_RED 1  // BC[x] += contribution as a fire-and-forget red.global.add (one adder per x per level: same order)
#endif
__device__ __forceinline__ void bc_add(double *p, double v) {
#if BC_BC_RED
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
#else
    *p += v;
#endif
}
#ifndef BC_FWD_COLPF
#define BC_FWD_COLPF 0  // 1: forward step loop fetches the next step's columns one step ahead
#endif
#ifndef BC_SEEN_RED
#define BC_SEEN_RED 1  // forward commit: seen |= new lanes by a red.global.or instead of a load + store
#endif
#ifndef BC_FWD_PIPE
#define BC_FWD_PIPE 0  // > 0: whole-row forward with a rolling pipeline of BC_FWD_PIPE gathers in flight (else BC_FWD_HIT2)
#endif
#ifndef BC_FWD_UNCOND
#define BC_FWD_UNCOND 1  // 16-bit forward: hit rows loaded whole (no per-pair c test; rows are zero outside their level)
#endif
#ifndef BC_GATHER_REDUX
#define BC_GATHER_REDUX 1  // mask words by two warp OR-reductions per word instead of ballots + bit interleave
#endif
// warp-collective: the W mask words whose thread-t bits are bits of `bits`;
// word j is returned to lane j (other lanes: 0).  Thread t's pair of word j
// sits at bits 2t, 2t+1: threads 0-15 fill the low half, 16-31 the high half,
// so each half is one OR-reduction of the threads' pairs shifted into place.
template <int W>
__device__ __forceinline__ uint64_t gather_words(uint32_t bits, int lane) {
    uint64_t mine = 0;
#pragma unroll
    for (int j = 0; j < W; ++j) {
#if BC_GATHER_REDUX
        const uint32_t v = ((bits >> (2 * j)) & 3u) << ((2 * lane) & 31);
        const uint32_t lo = __reduce_or_sync(0xffffffffu, lane < 16 ? v : 0u);
        const uint32_t hi = __reduce_or_sync(0xffffffffu, lane >= 16 ? v : 0u);
        if (lane == j) mine = (uint64_t)lo | ((uint64_t)hi << 32);
#else
        const uint32_t b0 = __ballot_sync(0xffffffffu, (bits >> (2 * j)) & 1u);
        const uint32_t b1 = __ballot_sync(0xffffffffu, (bits >> (2 * j + 1)) & 1u);
        if (lane == j) mine = interleave2(b0, b1);
#endif
    }
    return mine;
}

// IN16: the level-L rows read by the forward hold 16-bit sigma -- the narrow
// tier (SigT = unsigned), or the level at which a batch widens to 32-bit rows
// (SigT = long long, the "widening" instantiation: 16-bit rows in, 32-bit out)
template <int W, typename SigT, bool BWD = false, bool IN16 = std::is_same<SigT, unsigned>::value>
struct LanesKernel {
    static constexpr int K = 64 * W;
    static constexpr int LPT = 2 * W;           // lanes per thread
    static constexpr int R = (W == 1) ? 4 : (W == 2 ? 2 : BC_R4);  // item steps in flight per warp (W >= 4: BC_R4)
    static constexpr bool VERIFY = std::is_same<SigT, unsigned long long>::value;
    static constexpr bool NARROW = std::is_same<SigT, unsigned>::value;
    static constexpr bool MID = std::is_same<SigT, long long>::value;
    static constexpr bool INTROW = NARROW || MID;  // integer rows with a limit (re-run when exceeded)
    static constexpr unsigned long long LIMIT = RowLimit<SigT>::v;
    using RT = typename RowOf<SigT>::t;  // sigma row storage
    using V = typename Vec2<SigT>::t;
    using Smem = LanesSmem<W, SigT>;

    const LanesParams &p;
    Smem &sm;
    const int lane, wid, t2;
    // per-thread statistics of the current work unit (bounded by its items, so
    // 32 bits suffice except the adjacency sum); flushed by flush_stats()
    unsigned st_reach = 0, st_dag = 0, st_dsum = 0, st_items = 0, st_hits = 0;
    unsigned ring_issued = 0, ring_used = 0;  // BC_FWD_BULK: bulk copies issued / consumed by this warp (uniform)
    unsigned long long st_adj = 0;
    int any_new_loc = 0;

    __device__ LanesKernel(const LanesParams &pp, Smem &s)
        : p(pp), sm(s), lane(lane_id()), wid(warp_id()), t2(2 * lane_id()) {
        if (!BWD && p.lane_ns)
            for (int l = threadIdx.x; l < K; l += BC_NT) sm.ns[l] = 0.0;
        if (threadIdx.x < 6) sm.st[threadIdx.x] = 0;
        if (threadIdx.x < W) sm.act[threadIdx.x] = p.active_dev ? p.active_dev[threadIdx.x] : p.active[threadIdx.x];
        if constexpr (Smem::BULK && !BWD) {
            if (threadIdx.x < BC_NW * Smem::RING) mbar_init(sm.mbar + threadIdx.x, 1);
            mbar_init_fence();
        }
        __syncthreads();
    }

    // warp-reduce the thread counters (bounded by one work unit, so the 32-bit
    // sums cannot wrap), then one shared atomic per counter per warp
    __device__ void flush_stats() {
        const unsigned long long v[6] = {__reduce_add_sync(0xffffffffu, st_reach), warp_sum_u64(st_adj),
                                         __reduce_add_sync(0xffffffffu, st_dag),
                                         __reduce_add_sync(0xffffffffu, st_dsum),
                                         __reduce_add_sync(0xffffffffu, st_items),
                                         __reduce_add_sync(0xffffffffu, st_hits)};
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < 6; ++i)
                if (v[i]) atomicAdd(&sm.st[i], v[i]);
        }
        st_reach = st_dag = st_dsum = st_items = st_hits = 0;
        st_adj = 0;
    }

    // lane index of this thread's i-th accumulator
    __device__ __forceinline__ int lane_of(int i) const { return 64 * (i >> 1) + t2 + (i & 1); }

    __device__ __forceinline__ RT *Scur() const { return reinterpret_cast<RT *>(p.S_cur); }
    __device__ __forceinline__ SigT *part_row(int w, int idx) const {
        return reinterpret_cast<SigT *>(p.part) + ((size_t)(blockIdx.x * BC_NW + w) * 2 + idx) * K;
    }
    __device__ __forceinline__ RT *Snxt() const { return reinterpret_cast<RT *>(p.S_nxt); }

    // this thread's bits of the W words at w (shared or global, generic load)
    __device__ __forceinline__ uint32_t bits_of(const uint64_t *w) const {
        uint64_t m[W];
#pragma unroll
        for (int j = 0; j < W; ++j) m[j] = w[j];
        return pick2<W>(m, t2);
    }

    // write this thread's lanes of a row: v[i] where bit i of keep, else 0
    __device__ __forceinline__ void store_slice(RT *row, uint32_t keep, const SigT (&v)[LPT]) {
        if constexpr (NARROW) {
            // lanes 2t, 2t+1 of a pair are the low / high half of one 32-bit word
            uint32_t wv[W];
#pragma unroll
            for (int pr = 0; pr < W; ++pr) {
                const uint32_t lo = (keep >> (2 * pr) & 1u) ? (v[2 * pr] & 0xffffu) : 0u;
                const uint32_t hi = (keep >> (2 * pr + 1) & 1u) ? (v[2 * pr + 1] & 0xffffu) : 0u;
                wv[pr] = lo | (hi << 16);
            }
            if constexpr (BC_NARROW_TMAJOR) {
                st_row_vec<W>(reinterpret_cast<uint32_t *>(row) + lane * W, wv);
            } else {
#pragma unroll
                for (int pr = 0; pr < W; ++pr) *reinterpret_cast<uint32_t *>(row + 64 * pr + t2) = wv[pr];
            }
            return;
        }
        if constexpr (MID) {
#pragma unroll
            for (int pr = 0; pr < W; ++pr) {
                uint2 t;
                t.x = (keep >> (2 * pr) & 1u) ? (uint32_t)v[2 * pr] : 0u;
                t.y = (keep >> (2 * pr + 1) & 1u) ? (uint32_t)v[2 * pr + 1] : 0u;
                *reinterpret_cast<uint2 *>(row + 64 * pr + t2) = t;
            }
            return;
        }
#pragma unroll
        for (int pr = 0; pr < W; ++pr) {
            V t;
            t.x = (keep >> (2 * pr) & 1u) ? v[2 * pr] : SigT(0);
            t.y = (keep >> (2 * pr + 1) & 1u) ? v[2 * pr + 1] : SigT(0);
            *reinterpret_cast<V *>(row + 64 * pr + t2) = t;
        }
    }

    // ---- forward commit: x discovered in its undiscovered lanes (ub) where
    // acc != 0 (or overflowed); the level-(L+1) row of x is written whole.
    __device__ void commit_fwd(int x, int deg, uint32_t ub, const SigT (&acc)[LPT], uint32_t aovf) {
        BC_CHECK(x >= 0 && x < p.n);
        uint32_t nb = aovf;
#pragma unroll
        for (int i = 0; i < LPT; ++i)
            if (acc[i] != SigT(0)) nb |= 1u << i;
        nb &= ub;
        aovf &= ub;
        const bool any = __any_sync(0xffffffffu, nb != 0);
        if (!any) return;  // warp-uniform
        if constexpr (INTROW) {
            bool big = false;
#pragma unroll
            for (int i = 0; i < LPT; ++i) big |= (nb >> i & 1u) && (unsigned long long)acc[i] > LIMIT;
            if (big) *p.narrow_ovf = 1;
        }
        store_slice(Snxt() + (size_t)x * K, nb, acc);
        if (nb) {
            any_new_loc = 1;
            int pc = __popc(nb);
            st_reach += pc;
            st_adj += (unsigned long long)pc * deg;
            st_dsum += (unsigned)pc * (unsigned)(p.level + 1);
            if (p.lane_ns) {
                double wx = 1.0 + (p.omega ? (double)p.omega[x] : 0.0);
#pragma unroll
                for (int i = 0; i < LPT; ++i)
                    if (nb >> i & 1u) atomicAdd(&sm.ns[lane_of(i)], wx);
            }
        }
        const uint64_t wv = gather_words<W>(nb, lane);
        uint64_t ov = 0;
        if (VERIFY) ov = gather_words<W>(aovf, lane);
        if (lane < W && wv) {
            size_t wi = (size_t)x * W + lane;
            p.mask_nxt[wi] = wv;
#if BC_SEEN_RED
            // fire-and-forget OR: no dependent load of seen in the commit
            asm volatile("red.global.or.b64 [%0], %1;" ::"l"(p.seen + wi), "l"(wv) : "memory");
#else
            p.seen[wi] |= wv;
#endif
            if (VERIFY && ov) p.ovf[wi] |= ov;
        }
    }

    // ---- backward commit (pull form): x is at level L in the lanes of mb and
    // acc = sum of coef(v) over its children v (level L+1); then
    //   delta = sigma * acc, coef = (1 + omega(x) + delta) / sigma      (Eq.5)
    //   BC[x] += sum_lanes (1 + omega(s)) * (delta + omega(x))          (R13)
    // and the level-L row of x becomes its coef row (zeros stay zeros).
    __device__ void commit_bwd(int x, uint32_t mb, const SigT (&acc)[LPT]) {
        if constexpr (BWD && !VERIFY) {
            if (!__any_sync(0xffffffffu, mb != 0)) return;  // warp-uniform
            double *row = Scur() + (size_t)x * K;
            const double om = p.omega ? (double)p.omega[x] : 0.0;
            double contrib = 0.0;
            // pair by pair (few live registers); pairs without level-L lanes
            // stay zero, the other lane of a half-used pair is zero as well
#pragma unroll
            for (int pr = 0; pr < W; ++pr) {
                const uint32_t b2 = (mb >> (2 * pr)) & 3u;
                if (b2) {
                    double2 *cell = reinterpret_cast<double2 *>(row + 64 * pr + t2);
                    const double2 sg = *cell;
                    double2 cf = make_double2(0.0, 0.0);
                    if (b2 & 1u) {
                        const double delta = sg.x * acc[2 * pr];
                        cf.x = (1.0 + om + delta) / sg.x;
                        contrib += p.lane_w1[64 * pr + t2] * (delta + om);
                        cap_delta_put(p, 64 * pr + t2, x, delta);
                    }
                    if (b2 & 2u) {
                        const double delta = sg.y * acc[2 * pr + 1];
                        cf.y = (1.0 + om + delta) / sg.y;
                        contrib += p.lane_w1[64 * pr + t2 + 1] * (delta + om);
                        cap_delta_put(p, 64 * pr + t2 + 1, x, delta);
                    }
                    *cell = cf;
                }
            }
            contrib = warp_sum(contrib);
            if (lane == 0 && contrib != 0.0) bc_add(p.bc + x, contrib);
        }
    }

    __device__ __forceinline__ void commit_slot(int s, const SigT (&acc)[LPT], uint32_t aovf) {
        if constexpr (BWD) {
            commit_bwd(sm.vert[s], bits_of(sm.u + s * W), acc);
        } else {
            const uint32_t ub = bits_of(sm.u + s * W);
            commit_fwd(sm.vert[s], sm.cd[s + 1] - sm.cd[s], ub, acc, aovf);
        }
    }

    // flush the running accumulator of slot s (warp-uniform)
    __device__ void flush(int s, int first, int ws, int we, bool hub_mode, const SigT (&acc)[LPT],
                          uint32_t aovf) {
        bool owned = !hub_mode && sm.cd[s] >= ws && sm.cd[s + 1] <= we;
        if (owned) {
            commit_slot(s, acc, aovf);
        } else {
            int idx = (s == first) ? 0 : 1;
            SigT *dst = part_row(wid, idx);
#pragma unroll
            for (int pr = 0; pr < W; ++pr) {
                V t;
                t.x = acc[2 * pr];
                t.y = acc[2 * pr + 1];
                *reinterpret_cast<V *>(dst + 64 * pr + t2) = t;
            }
            if (VERIFY) sm.povf[(wid * 2 + idx) * 32 + lane] = aovf;
        }
    }

    // One warp walks items [ws, we) of the current tile (slots in sm).
    __device__ void warp_walk(int nslots, int ws, int we, bool hub_mode) {
        const uint64_t *mread = BWD ? p.mask_nxt_ro : p.mask_cur;  // bwd: children at L+1
        int cur = slot_of(sm.cd, nslots, ws);
        const int first = cur;
        const int last = slot_of(sm.cd, nslots, we - 1);
        SigT acc[LPT];
#pragma unroll
        for (int i = 0; i < LPT; ++i) acc[i] = SigT(0);
        uint32_t aovf = 0;
        const uint64_t pol = policy_evict_first();

        st_items += (lane == 0) ? (unsigned)(we - ws) : 0u;
        // BC_FWD_COLPF: the next step's (slot, column) is fetched while this
        // step's masks and hits are processed (the column load latency was
        // the step loop's top stall)
        auto fetch = [&](int e0f, int (&slf)[R], int (&vvf)[R]) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
                int e = e0f + k * 32 + lane;
                slf[k] = -1;
                vvf[k] = 0;
                if (e < we) {
                    int s = slot_of(sm.cd, nslots, e);
                    slf[k] = s;
                    vvf[k] = ld_stream(p.col + sm.rs[s] + (e - sm.cd[s]), pol);
                    BC_CHECK(s >= 0 && s < nslots && vvf[k] >= 0 && vvf[k] < p.n);
                }
            }
        };
        constexpr bool COLPF = BC_FWD_COLPF && !BWD;
        int sln[R], vvn[R];
        if constexpr (COLPF) fetch(ws, sln, vvn);
        for (int e0 = ws; e0 < we; e0 += 32 * R) {
            int sl[R], vv[R];
            if constexpr (COLPF) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    sl[k] = sln[k];
                    vv[k] = vvn[k];
                }
                if (e0 + 32 * R < we) fetch(e0 + 32 * R, sln, vvn);  // uniform
            } else {
                fetch(e0, sl, vv);
            }
            uint64_t cc[R][W];
#pragma unroll
            for (int k = 0; k < R; ++k) {
#pragma unroll
                for (int j = 0; j < W; ++j) cc[k][j] = 0;
                if (sl[k] >= 0) {
#if BC_FWD_MASK_HINT
                    if constexpr (W >= 2) {
                        const uint64_t mpol = policy_evict_last();
#pragma unroll
                        for (int j = 0; j < W; j += 2) {
                            const ulonglong2 t = ld_pol(reinterpret_cast<const ulonglong2 *>(mread + (size_t)vv[k] * W + j), mpol);
                            cc[k][j] = t.x;
                            cc[k][j + 1] = t.y;
                        }
                    } else {
                        load_mask<W>(mread + (size_t)vv[k] * W, cc[k]);
                    }
#else
                    load_mask<W>(mread + (size_t)vv[k] * W, cc[k]);
#endif
#pragma unroll
                    for (int j = 0; j < W; ++j) cc[k][j] &= sm.u[sl[k] * W + j];
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                bool h = false;
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    h |= (cc[k][j] != 0);
                    if (!BWD) st_dag += (unsigned)__popcll(cc[k][j]);
                }
                unsigned hm = __ballot_sync(0xffffffffu, h);
                if (hm == 0) continue;
                st_hits += (lane == 0) ? __popc(hm) : 0;
                // publish (slot, v, c) of every item of this step in shared memory:
                // a hit then costs two shared broadcasts instead of 2 + 2W shuffles
                constexpr bool UNCOND = IN16 && BC_FWD_HIT2 && BC_FWD_UNCOND && !BWD && !Smem::BULK;
                if constexpr (UNCOND) {  // the hit's c words are not read: (slot, v) only
                    sm.hsv[wid * 32 + lane] = make_int2(sl[k], vv[k]);
                    __syncwarp();
                } else {
                    sm.hsv[wid * 32 + lane] = make_int2(sl[k], vv[k]);
                    uint32_t *hc = sm.hc + (wid * 32 + lane) * 2 * W;
                    uint32_t lo[W], hi[W];
#pragma unroll
                    for (int j = 0; j < W; ++j) {
                        lo[j] = (uint32_t)cc[k][j];
                        hi[j] = (uint32_t)(cc[k][j] >> 32);
                    }
                    store_halves<W>(hc, lo);
                    store_halves<W>(hc + W, hi);
                    __syncwarp();
                }
                const uint32_t *hcw = sm.hc + wid * 32 * 2 * W + (lane >> 4) * W;
                const int sh = t2 & 31;
                static_assert(!(Smem::BULK && BC_NARROW_TMAJOR), "the bulk-copy forward reads lane-order rows");
                if constexpr (Smem::BULK && !BWD) {
                    // 16-bit forward, Blackwell bulk copies: lane 0 streams the
                    // hit rows (K x 16 bit, zero outside level L, so whole rows
                    // are added -- lanes outside c only collect what the commit
                    // discards) into the warp's shared ring, up to RING hits
                    // ahead; the warp adds a row once its mbarrier completes
                    constexpr int RG = Smem::RING;
                    constexpr uint32_t RB = (uint32_t)K * 2u;
                    uint32_t *ringw = sm.ring + (size_t)wid * RG * 32 * W;
                    uint64_t *mbw = sm.mbar + wid * RG;
                    unsigned hi = hm;
                    auto issue = [&]() {
                        const int s = __ffs(hi) - 1;
                        hi &= hi - 1;
                        if (lane == 0) {
                            const int slot = (int)(ring_issued & (RG - 1));
                            fence_proxy_async_smem();  // the slot's previous row was read by generic loads
                            mbar_arrive_expect_tx(mbw + slot, RB);
                            bulk_g2s(ringw + slot * 32 * W, Scur() + (size_t)sm.hsv[wid * 32 + s].y * K, RB, mbw + slot);
                        }
                        ++ring_issued;
                    };
#pragma unroll 1
                    for (int q = 0; q < RG && hi; ++q) issue();
                    while (hm) {
                        const int src = __ffs(hm) - 1;
                        hm &= hm - 1;
                        const int hs = sm.hsv[wid * 32 + src].x;
                        if (hs != cur) {
                            while (cur < hs) {
                                flush(cur, first, ws, we, hub_mode, acc, aovf);
                                ++cur;
#pragma unroll
                                for (int i = 0; i < LPT; ++i) acc[i] = SigT(0);
                                aovf = 0;
                            }
                        }
                        const int slot = (int)(ring_used & (RG - 1));
                        mbar_wait_parity(mbw + slot, (ring_used / RG) & 1u);
                        const uint32_t *row = ringw + slot * 32 * W + lane;
#pragma unroll
                        for (int pr = 0; pr < W; ++pr) {
                            const uint32_t t = row[32 * pr];
                            acc[2 * pr] += t & 0xffffu;
                            acc[2 * pr + 1] += t >> 16;
                        }
                        ++ring_used;
                        __syncwarp();
                        if (hi) issue();
                    }
                    __syncwarp();
                    continue;
                }
                if constexpr (UNCOND && BC_NARROW_TMAJOR && BC_FWD_PIPE > 0) {
                    // 16-bit forward, rolling gather pipeline: BC_FWD_PIPE hit rows
                    // in flight at all times within a step -- buffer d is
                    // consumed and at once refilled with the hit BC_FWD_PIPE
                    // places later, so hits are added in order (slot order)
                    constexpr int PD = BC_FWD_PIPE;
                    const uint64_t rpol = row_policy();
                    const uint16_t *S16 = reinterpret_cast<const uint16_t *>(p.S_cur);
                    uint32_t rbuf[PD][W];
                    int rslot[PD];
                    unsigned q = hm;
#pragma unroll
                    for (int d = 0; d < PD; ++d) {
                        rslot[d] = -1;
                        if (q) {  // uniform
                            const int src = __ffs(q) - 1;
                            q &= q - 1;
                            const int2 sv = sm.hsv[wid * 32 + src];
                            rslot[d] = sv.x;
                            ld_row_vec<W>(reinterpret_cast<const uint32_t *>(S16 + (size_t)sv.y * K) + lane * W, rpol,
                                          rbuf[d]);
                        }
                    }
                    bool more = true;
                    while (more) {
#pragma unroll
                        for (int d = 0; d < PD; ++d) {
                            if (more && rslot[d] < 0) more = false;  // uniform: later buffers are empty too
                            if (more) {
                                const int hs = rslot[d];
                                while (cur < hs) {
                                    flush(cur, first, ws, we, hub_mode, acc, aovf);
                                    ++cur;
#pragma unroll
                                    for (int i = 0; i < LPT; ++i) acc[i] = SigT(0);
                                    aovf = 0;
                                }
#pragma unroll
                                for (int pr = 0; pr < W; ++pr) {
                                    acc[2 * pr] += rbuf[d][pr] & 0xffffu;
                                    acc[2 * pr + 1] += rbuf[d][pr] >> 16;
                                }
                                rslot[d] = -1;
                                if (q) {  // uniform: refill with the hit PD places later
                                    const int src = __ffs(q) - 1;
                                    q &= q - 1;
                                    const int2 sv = sm.hsv[wid * 32 + src];
                                    rslot[d] = sv.x;
                                    ld_row_vec<W>(reinterpret_cast<const uint32_t *>(S16 + (size_t)sv.y * K) + lane * W,
                                                  rpol, rbuf[d]);
                                }
                            }
                        }
                    }
                    __syncwarp();
                    continue;
                }
                if constexpr (IN16 && BC_FWD_HIT2 && !BWD) {
                    const uint64_t rpol = row_policy();
                    // 16-bit forward, two hits per iteration: both hits' row
                    // words are loaded before either is added (and before a
                    // slot flush), so a warp has two rows' latency in flight
                    // instead of one (the level kernel stalled on the first
                    // use of each gathered word, profiles/ncu_r2_s20_level.txt)
                    while (hm) {
                        const int src = __ffs(hm) - 1;
                        hm &= hm - 1;
                        const int src2 = hm ? __ffs(hm) - 1 : -1;  // uniform
                        if (src2 >= 0) hm &= hm - 1;
                        const int2 sv = sm.hsv[wid * 32 + src];
                        uint32_t cw[W], t[W], t2[W];
                        const uint32_t *roww = reinterpret_cast<const uint32_t *>(reinterpret_cast<const uint16_t *>(p.S_cur) + (size_t)sv.y * K) + (BC_NARROW_TMAJOR ? lane * W : lane);
                        if constexpr (UNCOND) {
                            // whole rows: lanes outside c read zeros (y not at level L
                            // there) or values the commit discards (x not in u there)
                            if constexpr (BC_NARROW_TMAJOR) {
                                ld_row_vec<W>(roww, rpol, t);
                            } else {
#pragma unroll
                                for (int pr = 0; pr < W; ++pr) t[pr] = ld_row_word(roww + 32 * pr, rpol);
                            }
                        } else {
                            load_halves<W>(hcw + src * 2 * W, cw);
#pragma unroll
                            for (int pr = 0; pr < W; ++pr) t[pr] = (cw[pr] & (3u << sh)) ? ld_row_word(roww + (BC_NARROW_TMAJOR ? pr : 32 * pr), rpol) : 0u;
                        }
                        int2 sv2 = make_int2(-1, 0);
                        if (src2 >= 0) {
                            sv2 = sm.hsv[wid * 32 + src2];
                            const uint32_t *roww2 = reinterpret_cast<const uint32_t *>(reinterpret_cast<const uint16_t *>(p.S_cur) + (size_t)sv2.y * K) + (BC_NARROW_TMAJOR ? lane * W : lane);
                            if constexpr (UNCOND) {
                                if constexpr (BC_NARROW_TMAJOR) {
                                    ld_row_vec<W>(roww2, rpol, t2);
                                } else {
#pragma unroll
                                    for (int pr = 0; pr < W; ++pr) t2[pr] = ld_row_word(roww2 + 32 * pr, rpol);
                                }
                            } else {
                                load_halves<W>(hcw + src2 * 2 * W, cw);
#pragma unroll
                                for (int pr = 0; pr < W; ++pr) t2[pr] = (cw[pr] & (3u << sh)) ? ld_row_word(roww2 + (BC_NARROW_TMAJOR ? pr : 32 * pr), rpol) : 0u;
                            }
                        }
                        if (sv.x != cur) {
                            while (cur < sv.x) {
                                flush(cur, first, ws, we, hub_mode, acc, aovf);
                                ++cur;
#pragma unroll
                                for (int i = 0; i < LPT; ++i) acc[i] = SigT(0);
                                aovf = 0;
                            }
                        }
#pragma unroll
                        for (int pr = 0; pr < W; ++pr) {
                            acc[2 * pr] += t[pr] & 0xffffu;
                            acc[2 * pr + 1] += t[pr] >> 16;
                        }
                        if (src2 >= 0) {
                            if (sv2.x != cur) {
                                while (cur < sv2.x) {
                                    flush(cur, first, ws, we, hub_mode, acc, aovf);
                                    ++cur;
#pragma unroll
                                    for (int i = 0; i < LPT; ++i) acc[i] = SigT(0);
                                    aovf = 0;
                                }
                            }
#pragma unroll
                            for (int pr = 0; pr < W; ++pr) {
                                acc[2 * pr] += t2[pr] & 0xffffu;
                                acc[2 * pr + 1] += t2[pr] >> 16;
                            }
                        }
                    }
                    __syncwarp();
                    continue;
                }
                while (hm) {
                    const int src = __ffs(hm) - 1;
                    hm &= hm - 1;
                    const int2 sv = sm.hsv[wid * 32 + src];
                    uint32_t cw[W];
                    load_halves<W>(hcw + src * 2 * W, cw);
                    if (sv.x != cur) {
                        while (cur < sv.x) {
                            flush(cur, first, ws, we, hub_mode, acc, aovf);
                            ++cur;
#pragma unroll
                            for (int i = 0; i < LPT; ++i) acc[i] = SigT(0);
                            aovf = 0;
                        }
                    }
                    // rows are zero outside their level: add whole pairs
                    // (lanes outside c only collect values the commit discards)
                    if constexpr (IN16) {
                        // 16-bit rows: one 32-bit load per pair (lanes 2t, 2t+1)
                        const uint32_t *roww = reinterpret_cast<const uint32_t *>(reinterpret_cast<const uint16_t *>(p.S_cur) + (size_t)sv.y * K) + (BC_NARROW_TMAJOR ? lane * W : lane);
#pragma unroll
                        for (int pr = 0; pr < W; ++pr) {
                            if (cw[pr] & (3u << sh)) {
                                const uint32_t t = __ldg(roww + (BC_NARROW_TMAJOR ? pr : 32 * pr));
                                acc[2 * pr] += t & 0xffffu;
                                acc[2 * pr + 1] += t >> 16;
                            }
                        }
                        continue;
                    }
                    if constexpr (MID) {
                        // 32-bit rows: one 8-byte load per pair
                        const uint2 *rowp = reinterpret_cast<const uint2 *>(Scur() + (size_t)sv.y * K + t2);
#pragma unroll
                        for (int pr = 0; pr < W; ++pr) {
                            if (cw[pr] & (3u << sh)) {
                                const uint2 t = __ldg(rowp + 32 * pr);
                                acc[2 * pr] += t.x;
                                acc[2 * pr + 1] += t.y;
                            }
                        }
                        continue;
                    }
                    const V *rowv = reinterpret_cast<const V *>((BWD ? Snxt() : Scur()) + (size_t)sv.y * K + t2);
                    if constexpr (!VERIFY) {
#pragma unroll
                        for (int pr = 0; pr < W; ++pr) {
                            if (cw[pr] & (3u << sh)) {
                                const V t = __ldg(rowv + 32 * pr);
                                acc[2 * pr] += t.x;
                                acc[2 * pr + 1] += t.y;
                            }
                        }
                    } else {
                        uint32_t mb = 0;
#pragma unroll
                        for (int pr = 0; pr < W; ++pr) mb |= ((cw[pr] >> sh) & 3u) << (2 * pr);
                        V val[W];
#pragma unroll
                        for (int pr = 0; pr < W; ++pr) {
                            val[pr].x = SigT(0);
                            val[pr].y = SigT(0);
                            if ((mb >> (2 * pr)) & 3u) val[pr] = __ldg(rowv + 32 * pr);
                        }
                        if (mb) {
                            uint64_t ow[W];
                            load_mask<W>(p.ovf + (size_t)sv.y * W, ow);
                            aovf |= mb & pick2<W>(ow, t2);
                        }
#pragma unroll
                        for (int pr = 0; pr < W; ++pr) {
                            SigT o = acc[2 * pr];
                            acc[2 * pr] = o + val[pr].x;
                            if (acc[2 * pr] < o) aovf |= 1u << (2 * pr);
                            o = acc[2 * pr + 1];
                            acc[2 * pr + 1] = o + val[pr].y;
                            if (acc[2 * pr + 1] < o) aovf |= 1u << (2 * pr + 1);
                        }
                    }
                }
                __syncwarp();  // the step's shared hit records are reused by the next step
            }
        }
        while (cur <= last) {
            flush(cur, first, ws, we, hub_mode, acc, aovf);
            ++cur;
#pragma unroll
            for (int i = 0; i < LPT; ++i) acc[i] = SigT(0);
            aovf = 0;
        }
    }

    __device__ __forceinline__ static int bnd(int j, int nitems) {
        return (int)(((long long)j * nitems) / BC_NW);
    }

    // ---- a tile of <= TV consecutive vertices (bounded by items, see build_layout)
    __device__ void tile(int t) {
        const int v0 = p.tile_vs[t], v1 = p.tile_vs[t + 1];
        const int x = v0 + threadIdx.x;
        int deg = 0, act = 0;
        uint64_t u[W];
#pragma unroll
        for (int j = 0; j < W; ++j) u[j] = 0;
        int rs = 0;
        if (x < v1) {
            rs = p.rp[x];
            deg = p.rp[x + 1] - rs;
            if (deg > 0 && deg <= p.hub_deg) {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    u[j] = BWD ? p.mask_cur[(size_t)x * W + j] : sm.act[j] & ~p.seen[(size_t)x * W + j];
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
        if (nslots == 0) return;
        const int ws = bnd(wid, nitems), we = bnd(wid + 1, nitems);
        if (ws < we) warp_walk(nslots, ws, we, false);
        __syncthreads();
        // slots split across warps: warp j finalises the slot holding boundary j
        if (wid >= 1) {
            const int b = bnd(wid, nitems);
            if (b > 0 && b < nitems) {
                const int s = slot_of(sm.cd, nslots, b);
                if (sm.cd[s] < b && (wid == 1 || bnd(wid - 1, nitems) <= sm.cd[s])) {
                    SigT acc[LPT];
#pragma unroll
                    for (int i = 0; i < LPT; ++i) acc[i] = SigT(0);
                    uint32_t aovf = 0;
                    for (int w = 0; w < BC_NW; ++w) {
                        int a0 = bnd(w, nitems), a1 = bnd(w + 1, nitems);
                        if (a0 >= a1 || a1 <= sm.cd[s] || a0 >= sm.cd[s + 1]) continue;
                        int idx = (sm.cd[s] <= a0) ? 0 : 1;
                        const SigT *src = part_row(w, idx);
#pragma unroll
                        for (int i = 0; i < LPT; ++i) {
                            SigT o = acc[i];
                            acc[i] = o + src[lane_of(i)];
                            if (VERIFY && acc[i] < o) aovf |= 1u << i;
                        }
                        if (VERIFY) aovf |= sm.povf[(w * 2 + idx) * 32 + lane];
                    }
                    commit_slot(s, acc, aovf);
                }
            }
        }
        flush_stats();
        __syncthreads();
    }

    // ---- one segment of a hub's adjacency
    __device__ void hub_segment(int unit) {
        if (threadIdx.x == 0) {
            int lo = 0, hi = p.nhub - 1;
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (p.hub_seg_off[mid] <= unit) lo = mid;
                else hi = mid - 1;
            }
            sm.scan[0] = lo;
        }
        __syncthreads();
        const int h = sm.scan[0];
        __syncthreads();
        BC_CHECK(h >= 0 && h < p.nhub);
        const int x = p.hub_ids[h];
        const int seg = unit - p.hub_seg_off[h];
        const int a = p.rp[x] + seg * p.seg_len;
        const int b = min(p.rp[x + 1], a + p.seg_len);
        BC_CHECK(seg >= 0 && a < b);
        uint64_t u[W];
        bool any = false;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            u[j] = BWD ? p.mask_cur[(size_t)x * W + j] : sm.act[j] & ~p.seen[(size_t)x * W + j];
            any |= (u[j] != 0);
        }
        if (!any) return;  // uniform
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
        if (ws < we) warp_walk(1, ws, we, true);
        __syncthreads();
        // lane-wise reduction over warps, then one red.add per lane into the hub row
        for (int l = threadIdx.x; l < K; l += BC_NT) {
            SigT sum = SigT(0);
            bool ovf = false;
            const int tl = (l & 63) >> 1, ti = 2 * (l >> 6) + (l & 1);  // owner thread / acc index of lane l
            for (int w = 0; w < BC_NW; ++w) {
                if (bnd(w, nitems) >= bnd(w + 1, nitems)) continue;
                SigT o = sum;
                sum = o + part_row(w, 0)[l];
                if (VERIFY && sum < o) ovf = true;
                if (VERIFY && (sm.povf[(w * 2) * 32 + tl] >> ti & 1u)) ovf = true;
            }
            // narrow: a segment partial above the limit already means overflow;
            // otherwise each add is <= 65535 and the hub row cannot wrap
            // lanes outside u collect values the commit discards: not checked, not added
            if (!((sm.u[l >> 6] >> (l & 63)) & 1ull)) sum = SigT(0);
            if (INTROW && (unsigned long long)sum > LIMIT) *p.narrow_ovf = 1;
            if (sum != SigT(0)) {
                SigT *dst = reinterpret_cast<SigT *>(p.hub_acc) + (size_t)h * K + l;
                SigT old;
                if constexpr (MID)
                    old = (SigT)atomicAdd(reinterpret_cast<unsigned long long *>(dst), (unsigned long long)sum);
                else
                    old = atomicAdd(dst, sum);
                if (VERIFY && old + sum < old) ovf = true;
            }
            if (VERIFY && ovf) atomicOr((unsigned long long *)(p.hub_ovf + (size_t)h * W + (l >> 6)), 1ull << (l & 63));
        }
        flush_stats();
        __syncthreads();
    }

    __device__ void epilogue() {
        flush_stats();
        __syncthreads();
        if (threadIdx.x < 6 && sm.st[threadIdx.x]) {
            const int slot = BWD ? (threadIdx.x >= 4 ? threadIdx.x + 2 : -1) : (int)threadIdx.x;  // bwd: items, hits
            if (slot >= 0) atomicAdd(p.stats + slot, sm.st[threadIdx.x]);
        }
        int anyw = __any_sync(0xffffffffu, any_new_loc);
        if (lane == 0 && anyw) *p.any_new = 1;
        if (!BWD && p.lane_ns) {
            __syncthreads();
            for (int l = threadIdx.x; l < K; l += BC_NT)
                if (sm.ns[l] != 0.0) atomicAdd(p.lane_ns + l, sm.ns[l]);
        }
    }
};

#ifndef BC_MINB
#define BC_MINB 2  // min resident CTAs per SM for the level kernels at W < 4 (register cap)
#endif
#ifndef BC_MINB4
#define BC_MINB4 5  // ... and at W = 4: 40 resident warps (48 registers, small spills; S20 forward 88.6 -> 85.9 ms, profiles/exp_r2_fwd_minb.txt)
#endif
#ifndef BC_MINB8
#define BC_MINB8 3  // ... and at W = 8 (16 lanes per thread)
#endif

template <int W, typename SigT, bool BWD = false, bool IN16 = std::is_same<SigT, unsigned>::value>
__global__ void __launch_bounds__(BC_NT, (W == 8 ? BC_MINB8 : (W == 4 ? BC_MINB4 : BC_MINB))) lanes_level_kernel(LanesParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    if (p.prev_new && *p.prev_new == 0) return;  // speculative launch past the last level
    if (gated_off(p)) return;                     // device-driven batch: tier not in use
    LanesSmem<W, SigT> &sm = *reinterpret_cast<LanesSmem<W, SigT> *>(smraw);
    LanesKernel<W, SigT, BWD, IN16> k(p, sm);
    const int total = p.nseg + p.ntiles;
    for (;;) {
        if (threadIdx.x == 0) {
            int t = atomicAdd(p.work_ctr, 1);
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

// One warp per hub: commit the hub's summed row.  Resets the scratch row for
// the next level.
template <int W, typename SigT, bool BWD = false>
__global__ void __launch_bounds__(BC_NT) lanes_hub_finalize(LanesParams p) {
    using KK = LanesKernel<W, SigT, BWD>;
    constexpr int K = KK::K, LPT = KK::LPT;
    if (p.prev_new && *p.prev_new == 0) return;
    if (gated_off(p)) return;
    extern __shared__ __align__(16) unsigned char smraw[];
    LanesSmem<W, SigT> &sm = *reinterpret_cast<LanesSmem<W, SigT> *>(smraw);
    KK k(p, sm);
    const int h = (blockIdx.x * BC_NT + threadIdx.x) >> 5;
    if (h < p.nhub) {
        const int x = p.hub_ids[h];
        SigT *row = reinterpret_cast<SigT *>(p.hub_acc) + (size_t)h * K;
        SigT acc[LPT];
#pragma unroll
        for (int i = 0; i < LPT; ++i) {
            acc[i] = row[k.lane_of(i)];
            if (acc[i] != SigT(0)) row[k.lane_of(i)] = SigT(0);
        }
        if constexpr (BWD) {
            k.commit_bwd(x, k.bits_of(p.mask_cur + (size_t)x * W), acc);
        } else {
            uint32_t aovf = 0;
            if (KK::VERIFY) {
                uint64_t *ow = p.hub_ovf + (size_t)h * W;
                aovf = k.bits_of(ow);
                __syncwarp();
                if (k.lane < W) ow[k.lane] = 0;
            }
            uint64_t um[W];
#pragma unroll
            for (int j = 0; j < W; ++j) um[j] = sm.act[j] & ~p.seen[(size_t)x * W + j];
            const uint32_t ub = pick2<W>(um, k.t2);
            k.commit_fwd(x, p.rp[x + 1] - p.rp[x], ub, acc, aovf);
        }
    }
    k.epilogue();
}

// Levels 0 and 1 of every lane (Alg.2 lines 7-12 plus the first expansion):
// one CTA per lane pushes sigma = 1 to the source's neighbours.
template <int W, typename SigT>
__global__ void __launch_bounds__(BC_NT) lanes_init_kernel(LanesParams p, const int *src, uint64_t *mask0,
                                                            uint64_t *mask1) {
    constexpr int K = 64 * W;
    __shared__ double red_d[BC_NW];
    __shared__ unsigned long long red_u[BC_NW];
    if (gated_off(p)) return;
    const int l = blockIdx.x;
    const int s = src[l];
    if (s < 0) return;  // unused lane (2-degree batch layout, or past the end of a device-driven batch)
    const int word = l >> 6;
    const uint64_t bit = 1ull << (l & 63);
    const int rs = p.rp[s], re = p.rp[s + 1];
    if (threadIdx.x == 0) {
        atomicOr((unsigned long long *)(mask0 + (size_t)s * W + word), (unsigned long long)bit);
        atomicOr((unsigned long long *)(p.seen + (size_t)s * W + word), (unsigned long long)bit);
    }
    if (p.derived[word] & bit) {
        // 2-degree source (NEXT-1): only level 0 here; levels >= 1 come from
        // lanes_derive_kernel after the forward.  Counters: the source itself
        // and its two DAG edges to a and b.
        if (threadIdx.x == 0) {
            atomicAdd(p.stats + 0, 1ull);
            atomicAdd(p.stats + 1, (unsigned long long)(re - rs));
            atomicAdd(p.stats + 2, (unsigned long long)(re - rs));
        }
        return;
    }
    double cnt = 0.0;
    unsigned long long adj = 0;
    for (int e = rs + threadIdx.x; e < re; e += BC_NT) {
        const int w = p.col[e];
        atomicOr((unsigned long long *)(mask1 + (size_t)w * W + word), (unsigned long long)bit);
        atomicOr((unsigned long long *)(p.seen + (size_t)w * W + word), (unsigned long long)bit);
        cnt += 1.0 + (p.omega ? (double)p.omega[w] : 0.0);
        adj += (unsigned long long)(p.rp[w + 1] - p.rp[w]);
    }
    cnt = warp_sum(cnt);
    adj = warp_sum_u64(adj);
    if (lane_id() == 0) {
        red_d[warp_id()] = cnt;
        red_u[warp_id()] = adj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double c = 0.0;
        unsigned long long a = 0;
        for (int w = 0; w < BC_NW; ++w) {
            c += red_d[w];
            a += red_u[w];
        }
        const int deg = re - rs;
        if (p.lane_ns) p.lane_ns[l] = 1.0 + (p.omega ? (double)p.omega[s] : 0.0) + c;
        atomicAdd(p.stats + 0, (unsigned long long)(1 + deg));
        atomicAdd(p.stats + 1, (unsigned long long)deg + a);
        atomicAdd(p.stats + 2, (unsigned long long)deg);
        atomicAdd(p.stats + 3, (unsigned long long)deg);
        if (deg > 0) *p.any_new = 1;
    }
}

// NEXT-1, the 2-degree heuristic (Lemma 1, Eq.(6), Alg.7
// with reading R23): a 2-degree source c whose neighbours a, b are lanes of
// the same batch sits in lane 3t+2 of a word whose lanes 3t, 3t+1 hold a, b
// (cmask = bits of such lanes).  After the forward sweep of the other lanes,
// its tree is derived per vertex v without traversing the graph:
//   lvl_c(v) = min(lvl_a(v), lvl_b(v)) + 1,  sigma_c(v) = sum of sigma_x(v)
//   over x in {a, b} at that minimum (Eq.(6), equal levels: both).
// Bit-parallel over the levels L = 0, 1, ...: a lane-c bit becomes set at
// L+1 when the a- or b-bit (shifted onto the c position) is set at L and c
// has no level yet; c's own vertex is at level 0 (set by the init kernel),
// so Lemma 1's exception v = c needs no special case.  The backward sweep
// then treats lane c like any other lane (the Dynamic Merging of Frontiers
// of Alg.8-9 is what a lane-parallel backward does anyway).
struct DeriveParams {
    int n;
    int nlev;                      // levels 0 .. nlev-1 hold the forward's vertices (nlev = Lmax + 1)
    uint64_t *const *lvl;          // [nlev + 1] level masks (level nlev pre-zeroed)
    void *const *rows;             // [nlev + 1] sigma rows (RT)
    const int *rp;
    uint64_t cmask[8];
    unsigned long long *stats;
    int *ovf;                      // integer rows: set when a derived sigma exceeds the row type
};

template <int W, typename RT>
__global__ void __launch_bounds__(256) lanes_derive_kernel(DeriveParams q) {
    constexpr int K = 64 * W;
    constexpr unsigned long long LIMIT = std::is_same<RT, uint16_t>::value ? 65535ull
                                       : (std::is_same<RT, uint32_t>::value ? 4294967295ull : 0ull);
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long st_reach = 0, st_adj = 0, st_dsum = 0;
    if (v < q.n) {
        const int deg = q.rp[v + 1] - q.rp[v];
        uint64_t done[W];
#pragma unroll
        for (int j = 0; j < W; ++j) done[j] = 0;
        bool big = false;
        for (int L = 0; L < q.nlev; ++L) {
            const uint64_t *ml = q.lvl[L] + (size_t)v * W;
            const RT *rl = reinterpret_cast<const RT *>(q.rows[L]) + (size_t)v * K;
            uint64_t *mn = q.lvl[L + 1] + (size_t)v * W;
            RT *rn = reinterpret_cast<RT *>(q.rows[L + 1]) + (size_t)v * K;
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const uint64_t cm = q.cmask[j];
                if (!cm) continue;
                const uint64_t M = ml[j];
                done[j] |= M & cm;                   // c itself (level 0) / set earlier
                const uint64_t ma = (M << 2) & cm, mb = (M << 1) & cm;
                uint64_t nw = (ma | mb) & ~done[j];
                if (!nw) continue;
                done[j] |= nw;
                mn[j] |= nw;
                const int cnt = __popcll(nw);
                st_reach += cnt;
                st_adj += (unsigned long long)cnt * deg;
                st_dsum += (unsigned long long)cnt * (L + 1);
                while (nw) {
                    const int b = __ffsll((long long)nw) - 1;
                    nw &= nw - 1;
                    const int lc = 64 * j + b;
                    double sa = 0.0;
                    unsigned long long ia = 0;
                    if (ma >> b & 1ull) {
                        sa += (double)rl[row_idx<W, RT>(lc - 2)];
                        ia += (unsigned long long)rl[row_idx<W, RT>(lc - 2)];
                    }
                    if (mb >> b & 1ull) {
                        sa += (double)rl[row_idx<W, RT>(lc - 1)];
                        ia += (unsigned long long)rl[row_idx<W, RT>(lc - 1)];
                    }
                    if constexpr (LIMIT != 0) {
                        big |= ia > LIMIT;
                        rn[row_idx<W, RT>(lc)] = (RT)ia;
                    } else {
                        rn[row_idx<W, RT>(lc)] = (RT)sa;
                    }
                }
            }
        }
        if (big) *q.ovf = 1;
    }
    st_reach = warp_sum_u64(st_reach);
    st_adj = warp_sum_u64(st_adj);
    st_dsum = warp_sum_u64(st_dsum);
    if (lane_id() == 0 && st_reach) {
        atomicAdd(q.stats + 0, st_reach);
        atomicAdd(q.stats + 1, st_adj);
        atomicAdd(q.stats + 3, st_dsum);
    }
}

// n_s of a derived lane = n_s of its lane a (same component)
__global__ void derive_ns_kernel(int K, DeriveParams q, double *lane_ns) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < K && (q.cmask[l >> 6] >> (l & 63) & 1ull)) lane_ns[l] = lane_ns[l - 2];
}

// Rows of levels 0 and 1: sigma = 1 in the lanes of the level mask, 0 elsewhere
// (warp per vertex; vertices outside the level skip).
template <int W, typename SigT>
__global__ void lanes_materialize_kernel(int n, const uint64_t *mask, SigT *S, const int *need = nullptr,
                                         const int *halt = nullptr) {
    if (gated_off(need, halt)) return;
    // thread per vertex finds the vertices of the level, then the warp
    // writes each of their rows (most vertices are at neither level)
    constexpr int K = 64 * W, LPT = 2 * W;
    const int base = (int)(((size_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(size_t)31);
    const int lane = lane_id();
    bool mine = false;
    if (base + lane < n) {
#pragma unroll
        for (int j = 0; j < W; ++j) mine |= mask[(size_t)(base + lane) * W + j] != 0;
    }
    unsigned todo = __ballot_sync(0xffffffffu, mine);
    const int word = (lane * LPT) >> 6, off = (lane * LPT) & 63;
    while (todo) {
        const int v = base + __ffs(todo) - 1;
        todo &= todo - 1;
        uint64_t mw = 0;
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (j == word) mw = mask[(size_t)v * W + j];
        SigT *row = S + (size_t)v * K;
#pragma unroll
        for (int i = 0; i < LPT; ++i) row[row_idx<W, SigT>(lane * LPT + i)] = (mw >> (off + i) & 1ull) ? SigT(1) : SigT(0);
    }
}

// verification: sigma of lane 0 for the vertices at level L
template <typename SigT>
__global__ void gather_level_lane0_kernel(int n, const uint64_t *mask, int W, const SigT *S, int K,
                                          const uint64_t *ovf, unsigned long long *sig, uint8_t *ov) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n && (mask[(size_t)v * W] & 1ull)) {
        sig[v] = (unsigned long long)S[(size_t)v * K];
        if (ov) ov[v] = ovf ? (uint8_t)(ovf[(size_t)v * W] & 1ull) : 0;
    }
}

// Endpoint term of the attributed 1-degree form (R13): BC[s] += omega(s)(n_s - 2).
__global__ void lanes_endpoint_kernel(const int *src, int nlanes, const uint32_t *omega, const double *lane_ns,
                                      double *bc, const int *need = nullptr, const int *halt = nullptr) {
    if (gated_off(need, halt)) return;
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < nlanes && src[l] >= 0) {
        const int s = src[l];
        const double om = (double)omega[s];
        if (om != 0.0) bc[s] += om * (lane_ns[l] - 2.0);
    }
}

// Residual-isolated sources with omega > 0 (R10): n_s = 1 + omega(s).
__global__ void trivial_sources_kernel(const int *src, int ns, const uint32_t *omega, double *bc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ns) {
        const int s = src[i];
        const double om = (double)omega[s];
        bc[s] += om * (om - 1.0);
    }
}

// ---- verification capture (bc_set_capture) -----------------------------
// Depth and sigma of the captured lanes at level L, read from the level mask
// and the level sigma rows the production forward wrote (thread per vertex;
// only the captured lanes' bits are visited: capmask = OR of their bits).
template <int W, typename RT>
__global__ void cap_extract_kernel(int n, int L, const uint64_t *mask, const RT *rows, const int *lane_cap,
                                   const uint64_t *capmask, int *cap_depth, double *cap_sigma,
                                   const int *need = nullptr, const int *halt = nullptr, const int *nonempty = nullptr) {
    constexpr int K = 64 * W;
    if (gated_off(need, halt) || (nonempty && *nonempty == 0)) return;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
#pragma unroll
    for (int j = 0; j < W; ++j) {
        uint64_t m = capmask[j];
        if (!m) continue;
        m &= mask[(size_t)v * W + j];
        while (m) {
            const int b = __ffsll((long long)m) - 1;
            m &= m - 1;
            const int l = 64 * j + b, c = lane_cap[l];
            BC_CHECK(c >= 0);
            cap_depth[(size_t)c * n + v] = L;
            cap_sigma[(size_t)c * n + v] = (double)rows[(size_t)v * K + row_idx<W, RT>(l)];
        }
    }
}

// the sigma-row tier (16 / 32 / 64 bits) the captured lanes' batch completed with
__global__ void cap_tier_kernel(int K, const int *lane_cap, int tier, int *cap_tier, const int *need = nullptr,
                                const int *halt = nullptr) {
    if (gated_off(need, halt)) return;
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < K && lane_cap[l] >= 0) cap_tier[lane_cap[l]] = tier;
}

// verification: depth of lane 0 from the level masks
__global__ void depth_from_mask_kernel(const uint64_t *mask, int n, int W, int L, int *depth) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n && (mask[(size_t)v * W] & 1ull)) depth[v] = L;
}

}  // namespace bcb
