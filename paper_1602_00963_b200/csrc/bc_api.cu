// bc_api.cu -- C ABI (include/bc.h) of the B200 BC hot path: graph
// residency, 1-degree pruning, the batched forward/backward level loop and
// the verification entry point.  All arithmetic of the method runs in the
// kernels of lanes.cuh / graph_kernels.cuh; this file only allocates,
// validates arguments, sequences launches and copies results.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#include <thread>
#include <chrono>
#include <cstdlib>

#include "bc.h"
#include "util.cuh"
#include "lanes.cuh"
#include "graph_kernels.cuh"
#include "slices.cuh"
#include "bwd_push.cuh"
#include "batch_ctl.cuh"
#include <cub/device/device_radix_sort.cuh>

using namespace bcb;

namespace {

thread_local std::string g_err;

// BC_TRACE=1 (environment): host-side phase times of bc_compute on stderr
// (diagnosis of launch/sync-bound small graphs; no effect otherwise)
bool trace_on() {
    static const bool on = [] {
        const char *e = std::getenv("BC_TRACE");
        return e && *e && *e != '0';
    }();
    return on;
}
double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bc_status fail(bc_status s, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CU(call)                                                                                      \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) {                                                                      \
            (void)cudaGetLastError();                                                                 \
            return fail(e_ == cudaErrorMemoryAllocation ? BC_ERR_NOMEM : BC_ERR_CUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                           \
        }                                                                                             \
    } while (0)

#define CU_V(call) (void)(call)  // error surfaces through the enclosing cudaGetLastError / capture status

#define CK(expr)                              \
    do {                                      \
        bc_status s_ = (expr);                \
        if (s_ != BC_OK) return s_;           \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

template <typename T>
bc_status dalloc(T **p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    CU(cudaMalloc((void **)p, count * sizeof(T)));
    return BC_OK;
}

template <typename T>
void dfree(T *&p) {
    if (p) cudaFree((void *)p);
    p = nullptr;
}

// A CSR resident on the device plus its hub decomposition.
struct DevCSR {
    int *rp = nullptr;
    int *col = nullptr;
    int64_t nnz = 0;
    int nhub = 0, nseg = 0;
    int *hub_ids = nullptr;
    int *hub_seg_off = nullptr;
    int ntiles = 0;
    int *tile_vs = nullptr;       // [ntiles+1] vertex ranges of the level-kernel tiles
    int *perm = nullptr;          // compute CSR only: new id -> original id
    int *inv = nullptr;           // compute CSR only: original id -> new id
    uint32_t *omega = nullptr;    // compute CSR only: omega in this CSR's labels (pruned)
    std::vector<int> h_deg;
    std::vector<int> h_inv;       // compute CSR only: original id -> new id
    void release() {
        dfree(rp);
        dfree(col);
        dfree(hub_ids);
        dfree(hub_seg_off);
        dfree(tile_vs);
        dfree(perm);
        dfree(inv);
        dfree(omega);
        nhub = nseg = ntiles = 0;
        nnz = 0;
        h_deg.clear();
        h_inv.clear();
    }
};

struct LaneWS {
    int W = 0;
    bool verify = false;
    int row_bytes = 8;  // bytes per lane of the level sigma rows: 4 holds the 16- and 32-bit tiers
    std::vector<void *> slev;  // per-level sigma/coef rows, n*K 8-byte values each
    uint64_t *seen = nullptr;
    uint64_t *ovf = nullptr;
    std::vector<uint64_t *> chunks;  // LCH levels each
    void *hub_acc = nullptr;
    uint64_t *hub_ovf = nullptr;
    int hub_cap = 0;
    double *lane_w1 = nullptr;
    double *lane_ns = nullptr;
    void *part = nullptr;  // split-slot partial sums [max CTAs][BC_NW][2][K]
    double *A = nullptr;   // push-backward accumulators [n][K], zero between batches
    double *Arep = nullptr;  // replicas of the hub parents' rows [BC_REP_R][BC_REP_H][K], zero between levels
    unsigned long long *lvl_snap = nullptr;  // [3][8] counters before each of the last 3 forward levels (widening)
    double *ns_snap = nullptr;               // [3][K] n_s accumulators likewise
    int *lane_cap = nullptr;       // [K] capture slot of each lane or -1 (bc_set_capture)
    uint64_t *capmask = nullptr;   // [8] lanes of the batch that are captured
    uint64_t **d_lv = nullptr;  // device copies of the level mask / row pointers (2-degree derive)
    void **d_rows = nullptr;
    int dptr_cap = 0;
    void release() {
        dfree(d_lv);
        dfree(d_rows);
        dptr_cap = 0;
        dfree(part);
        dfree(A);
        dfree(lane_cap);
        dfree(capmask);
        dfree(lvl_snap);
        dfree(ns_snap);
        for (auto &q : slev) dfree(q);
        slev.clear();
        dfree(seen);
        dfree(ovf);
        for (auto &c : chunks) dfree(c);
        chunks.clear();
        dfree(hub_acc);
        dfree(hub_ovf);
        dfree(lane_w1);
        dfree(lane_ns);
        W = 0;
        hub_cap = 0;
    }
};

constexpr int LCH = 8;           // levels per mask chunk
constexpr int FLAG_RING = 4;     // pinned per-level flag slots (termination test one level behind)
constexpr int TILE_ITEMS = 8192; // non-hub adjacency items per level-kernel tile (soft cap) on large graphs
#ifndef BC_TILE_MIN
#define BC_TILE_MIN 256          // ... and the smallest cap (small graphs, see build_layout)
#endif
#ifndef BC_TILE_PER_SM
#define BC_TILE_PER_SM 1         // tiles are halved until a level's adjacency makes this many per SM
#endif
constexpr int MAX_STREAMS = 8;   // concurrent batch pipelines (BC_OPT_STREAMS)
// level (forward) and push (backward) kernel grids = resident CTAs x NUM / DEN
// when several batch pipelines run concurrently: the gaps let a pipeline's
// forward and another's backward share the SMs (S20, 3 pipelines: 307.5 ->
// 302-304 ms per 8192 sources, profiles/exp_r2_gridfrac.txt).  Since the
// forward runs 5 CTAs per SM its full grid is best (270.7 vs 273.3-276.2 ms,
// profiles/exp_r2_gridfrac.txt); the push keeps 3/4
#ifndef BC_FGRID_NUM
#define BC_FGRID_NUM 1
#endif
#ifndef BC_FGRID_DEN
#define BC_FGRID_DEN 1
#endif
#ifndef BC_PGRID_NUM
#define BC_PGRID_NUM 3
#endif
#ifndef BC_PGRID_DEN
#define BC_PGRID_DEN 4
#endif
#ifndef BC_DEVLOOP_MAX_LEVELS
#define BC_DEVLOOP_MAX_LEVELS 32  // device-driven batches only for graphs whose depth bound is at most this
#endif

// One batch pipeline: a workspace, a stream and the per-stream control state.
// bc_compute runs up to MAX_STREAMS of them concurrently (one host thread
// each), so the level kernels of one batch fill the tails and the host-test
// gaps of another and a forward (L1-bound gathers) overlaps a backward (L2
// reds) on the same SMs.
struct LaneCtx {
    LaneWS ws;
    cudaStream_t st = nullptr;   // stream of the current call (own, or the caller's)
    cudaStream_t own = nullptr;
    unsigned long long *d_stats = nullptr;  // [16]: counters, backup across a narrow re-run
    int *d_work_ctr = nullptr;              // [4]: level work counter, -, narrow overflow flag
    int *d_flags = nullptr;                 // [flag_cap] per-level "non-empty" flags
    int flag_cap = 0;
    int *h_flag = nullptr;                  // pinned [FLAG_RING][2]: level flag, narrow overflow
    cudaEvent_t ev_ring[FLAG_RING] = {};
    cudaEvent_t done = nullptr;
    double *d_bc = nullptr;                 // BC accumulator this pipeline adds into
    double *own_bc = nullptr;               // private partial BC (pipelines > 0)
    bc_stats last{};                        // host counters of the current call
    std::vector<cudaEvent_t> ef, eb, epush; // profile intervals
    double sync_us = 0;                     // BC_TRACE: host time blocked in the per-level test
    int syncs = 0;
    // device-driven batches (graph mode, enqueue_device_batch): per-batch
    // inputs and control live in device memory, so one instantiated CUDA
    // graph runs every batch of the pipeline
    int *gb_src = nullptr;            // [512] sources of the current batch (-1 past its end)
    int *gb_ctl = nullptr;            // [8]: 0 lanes, 1 batch counter, 2 16-bit overflow, 3 32-bit overflow,
                                      //      4 depth-bound violation, 5 scratch
    uint64_t *gb_active = nullptr;    // [8] lanes in use
    int2 *gb_table = nullptr;         // (offset into d_src, lanes) per batch of the pipeline
    int gb_table_cap = 0;
    unsigned long long *gb_cnt = nullptr;       // [8]: levels, 16-bit / 32-bit / fp64 batches, host re-runs
    int *gb_redo = nullptr;           // batch indices left for the host fp64 path (4-byte rows only)
    unsigned long long *gb_stats_bak = nullptr;  // [8] counters at batch start (restored per tier)
    cudaGraphExec_t gexec = nullptr;
    std::vector<uintptr_t> gkey;
    size_t gnodes = 0;                // nodes of the graph (kernels and copies) launched per batch
    cudaStream_t side[2] = {nullptr, nullptr};  // capture of the conditional tiers' bodies
    bool ready = false;
    void release() {
        if (gexec) cudaGraphExecDestroy(gexec), gexec = nullptr;
        gkey.clear();
        for (auto &sd : side)
            if (sd) cudaStreamDestroy(sd), sd = nullptr;
        dfree(gb_src);
        dfree(gb_ctl);
        dfree(gb_active);
        dfree(gb_table);
        gb_table_cap = 0;
        dfree(gb_cnt);
        dfree(gb_redo);
        dfree(gb_stats_bak);
        ws.release();
        dfree(d_stats);
        dfree(d_work_ctr);
        dfree(d_flags);
        dfree(own_bc);
        flag_cap = 0;
        if (h_flag) cudaFreeHost(h_flag);
        h_flag = nullptr;
        for (auto &e : ev_ring)
            if (e) cudaEventDestroy(e), e = nullptr;
        if (done) cudaEventDestroy(done), done = nullptr;
        if (own) cudaStreamDestroy(own), own = nullptr;
        ready = false;
    }
};

}  // namespace

struct SlicesWS {
    int rows = 0;  // CTAs (private rows)
    int *queue = nullptr, *loff = nullptr;
    unsigned *bm = nullptr;
    double *sigma = nullptr, *cf = nullptr, *bcp = nullptr;  // cf / bcp: slices_kernel only
    bool full = false;     // cf and bcp allocated
    int4 *ell = nullptr;   // [n] padded neighbours (max degree <= 4)
    int4 *qrow = nullptr;  // [rows][n] neighbour rows in queue order (BC_SM_QROW)
    int *cdq = nullptr;    // [rows][n] the forward's chunk degree prefixes (prefix-sum reuse variant)
    void release() {
        dfree(cdq);
        dfree(bm);
        dfree(qrow);
        dfree(ell);
        dfree(queue);
        dfree(loff);
        dfree(sigma);
        dfree(cf);
        dfree(bcp);
        rows = 0;
        full = false;
    }
};

struct bc_graph {
    int device = 0;
    int64_t n = 0;
    DevCSR orig, res;  // original labels; res.rp == nullptr while unpruned
    DevCSR run;        // the CSR the level kernels traverse: cur() relabelled by degree
    bool run_valid = false;
    int relabel = 1;
    int bwd_mode = 0;         // 0 = default, 1 = push form (bwd_push.cuh), 2 = pull form (lanes.cuh, BWD)
    int sigma_width = 0;      // BC_OPT_SIGMA_WIDTH: 0 = 16-bit sigma rows first (fp64 re-run on overflow), 64 = fp64 only
    int fwd_push_levels = 0;  // forward levels L <= this use the push form (measured: pull is as fast at L=1)
    int src_order = 2;  // 0 given, 1 degree, 2 anchor clusters
    bool pruned = false;
    uint32_t *omega = nullptr;
    uint8_t *removed = nullptr;
    std::vector<uint32_t> h_omega;
    std::vector<uint8_t> h_removed;
    int hub_deg = 4096;
    int lane_words_opt = 0;
    int profile = 0;
    int mode = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaEvent_t legacy_ev = nullptr;  // orders own_stream after the legacy default stream (NULL-stream calls)
    LaneCtx ctx[MAX_STREAMS];  // batch pipelines of bc_compute
    LaneCtx vctx, sctx;        // bc_sssp: integer verification (W = 1, uint64) and its fp64 delta pass
    int two_degree = 0;        // BC_OPT_TWO_DEGREE (NEXT-1)
    int *td_buf = nullptr;     // 2-degree planning scratch (grow-only)
    int64_t td_cap = 0;
    struct TdBatch {
        int64_t off;
        int nl;
        uint64_t active[8], derived[8];
    };
    std::vector<TdBatch> td_plan;
    std::vector<int> td_lanes;
    int depth_bound = -1;      // every BFS depth of the graph is <= this (bc_graph_create); -1 unknown
    int slices_kernel = 0;     // BC_OPT_SLICES_KERNEL: 0 auto, 1 general, 2 general + prefix reuse, 3/4 degree-bounded
    bool conc = false;         // the current call runs several batch pipelines (kernel grid fraction)
    int device_loop = 1;       // BC_OPT_DEVICE_LOOP: device-driven batches (CUDA graph per pipeline) when eligible
    struct Sizing {            // last call's lane width / row width / pipelines (skips cudaMemGetInfo when unchanged)
        int64_t key[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
        int W = 0, NS = 0, rb = 0;
        bool devloop = false;
    } sizing;
    unsigned long long *h_pin = nullptr;   // pinned: [0, 8) counters, [8 + 8 i, 16 + 8 i) pipeline i device-loop counters
    cudaEvent_t stats_ev = nullptr;        // the call's counters are in h_pin once this completes
    bool stats_pending = false;            // asynchronous call: g->last is completed by bc_get_stats
    bool devloop_used[MAX_STREAMS] = {};
    bool dl_violation = false;             // a device-driven BFS went past depth_bound (impossible by construction)
    int streams_opt = 0;       // 0 = auto: 8 pipelines for n <= 2^18 (launch/sync-bound batches), else 3       // BC_OPT_STREAMS (S20: 1 / 2 / 3 pipelines = 332 / 319 / 316 ms per 8192 sources)
    SlicesWS sws;    // slices-mode workspace
    unsigned long long *d_stats = nullptr;  // [16] slices mode / trivial sources counters
    int *d_work_ctr = nullptr;              // [4]: -, slices source counter
    int *d_src = nullptr;
    int64_t src_cap = 0;
    double *d_bc = nullptr;   // BC in compute (relabelled) ids
    double *d_bc2 = nullptr;  // BC in original ids (host-output staging)
    int *d_tmp = nullptr;  // scan scratch
    int64_t tmp_cap = 0;
    bc_stats last{};
    unsigned long long *cl_kin = nullptr, *cl_kout = nullptr;  // source clustering scratch
    int *cl_vout = nullptr;
    int64_t cl_cap = 0;
    void *cl_tmp = nullptr;
    size_t cl_tmp_bytes = 0;
    // verification capture (bc_set_capture), consumed by the next bc_compute
    struct Capture {
        std::vector<int> src;              // original ids
        std::vector<uint8_t> trivial;      // per slot: residual-isolated source (no traversal)
        int32_t *h_depth = nullptr;        // caller's host arrays [ncap][n]
        double *h_sigma = nullptr, *h_delta = nullptr;
        int32_t *h_tier = nullptr;         // [ncap]
        int *d_vslot = nullptr;            // [n] compute ids -> slot or -1
        int *d_src = nullptr;              // [ncap] original ids
        int *d_depth = nullptr, *d_tier = nullptr;  // compute ids
        double *d_sigma = nullptr, *d_delta = nullptr;
        int *o_depth = nullptr;            // original ids
        double *o_sigma = nullptr, *o_delta = nullptr;
        int64_t cap = 0;                   // allocated slots
        void release() {
            dfree(d_vslot);
            dfree(d_src);
            dfree(d_depth);
            dfree(d_tier);
            dfree(d_sigma);
            dfree(d_delta);
            dfree(o_depth);
            dfree(o_sigma);
            dfree(o_delta);
            cap = 0;
            src.clear();
        }
    } capt;
    DevCSR &cur() { return pruned ? res : orig; }
};

namespace {

// ---------------------------------------------------------------- scans
bc_status ensure_tmp(bc_graph *g, int64_t count) {
    if (g->tmp_cap >= count) return BC_OK;
    dfree(g->d_tmp);
    CK(dalloc(&g->d_tmp, (size_t)count));
    g->tmp_cap = count;
    return BC_OK;
}

// exclusive scan of n ints, total into *d_total (device int)
bc_status dev_scan(bc_graph *g, const int *in, int *out, int64_t n, int *d_total, cudaStream_t st) {
    int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (ntiles == 0) ntiles = 1;
    CK(ensure_tmp(g, ntiles));
    scan_tiles_kernel<<<(unsigned)ntiles, BC_NT, 0, st>>>(in, out, g->d_tmp, n);
    scan_sums_kernel<<<1, BC_NT, 0, st>>>(g->d_tmp, (int)ntiles, d_total);
    scan_add_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, g->d_tmp, n);
    CU(cudaGetLastError());
    return BC_OK;
}

bc_status build_hubs(bc_graph *g, DevCSR &c, cudaStream_t st);

// hubs + item-bounded tiles of <= TV consecutive vertices (host-side cut of
// the degree sequence; it is layout metadata, not part of the method)
bc_status build_layout(bc_graph *g, DevCSR &c, cudaStream_t st) {
    CK(build_hubs(g, c, st));
    std::vector<int> vs;
    vs.push_back(0);
    int cnt = 0;
    int64_t items = 0;
    const int64_t n = g->n;
    // Items per tile: at most TILE_ITEMS, and small enough that a level's
    // adjacency makes BC_TILE_PER_SM tiles per SM -- on a small graph (S12: 97k items) a
    // level's tiles are few, and a warp's serial walk over its share of a
    // large tile is the level's critical path.
    int64_t cap = TILE_ITEMS;
    while (cap > BC_TILE_MIN && c.nnz / cap < (int64_t)BC_TILE_PER_SM * g->num_sms) cap >>= 1;
    for (int64_t v = 0; v < n; ++v) {
        const int d = c.h_deg[v] > g->hub_deg ? 0 : c.h_deg[v];
        if (cnt == TV || (cnt > 0 && items + d > cap)) {
            vs.push_back((int)v);
            cnt = 0;
            items = 0;
        }
        ++cnt;
        items += d;
    }
    vs.push_back((int)n);
    dfree(c.tile_vs);
    c.ntiles = (int)vs.size() - 1;
    CK(dalloc(&c.tile_vs, vs.size()));
    CU(cudaMemcpyAsync(c.tile_vs, vs.data(), vs.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
    return BC_OK;
}

bc_status build_hubs(bc_graph *g, DevCSR &c, cudaStream_t st) {
    dfree(c.hub_ids);
    dfree(c.hub_seg_off);
    c.nhub = c.nseg = 0;
    const int n = (int)g->n;
    int *flag = nullptr, *pos = nullptr, *tot = nullptr;
    CK(dalloc(&flag, n));
    CK(dalloc(&pos, n));
    CK(dalloc(&tot, 2));
    hub_flag_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, c.rp, g->hub_deg, flag);
    CK(dev_scan(g, flag, pos, n, tot, st));
    int nhub = 0;
    CU(cudaMemcpyAsync(&nhub, tot, sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    c.nhub = nhub;
    CK(dalloc(&c.hub_ids, nhub));
    CK(dalloc(&c.hub_seg_off, nhub + 1));
    if (nhub > 0) {
        hub_scatter_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, flag, pos, c.hub_ids);
        int *cnt = nullptr;
        CK(dalloc(&cnt, nhub));
        hub_segcount_kernel<<<(nhub + 255) / 256, 256, 0, st>>>(nhub, c.hub_ids, c.rp, g->hub_deg, cnt);
        CK(dev_scan(g, cnt, c.hub_seg_off, nhub, tot + 1, st));
        CU(cudaMemcpyAsync(c.hub_seg_off + nhub, tot + 1, sizeof(int), cudaMemcpyDeviceToDevice, st));
        int nseg = 0;
        CU(cudaMemcpyAsync(&nseg, tot + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        c.nseg = nseg;
        dfree(cnt);
    }
    CU(cudaGetLastError());
    dfree(flag);
    dfree(pos);
    dfree(tot);
    return BC_OK;
}

// auto mode (BC_OPT_MODE = 0): slices for large sparse (long-diameter-like) graphs
static bool auto_slices(int64_t n, int64_t nnz) { return n > 65536 && (double)nnz / (double)n < 6.0; }

// The compute CSR: cur() relabelled by descending degree (stable, ties by
// id), so hub rows are contiguous at the front of every per-vertex array.
bc_status build_run(bc_graph *g) {
    cudaStream_t st = g->own_stream;
    DevCSR &c = g->cur();
    DevCSR &r = g->run;
    r.release();
    g->run_valid = false;
    const int n = (int)g->n;
    CK(dalloc(&r.perm, n));
    CK(dalloc(&r.inv, n));
    int maxdeg = 0;
    for (int d : c.h_deg) maxdeg = std::max(maxdeg, d);
    unsigned *keys_in = nullptr, *keys_out = nullptr;
    int *vals_in = nullptr;
    CK(dalloc(&keys_in, n));
    CK(dalloc(&keys_out, n));
    CK(dalloc(&vals_in, n));
    relabel_keys_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, c.rp, maxdeg, keys_in, vals_in);
    // relabel 1 (default): degree order, or breadth-first order for degree-bounded
    // graphs that auto mode runs as slices (grid: 33 -> 38 GTEPS; R-MAT S20 is
    // 17 % slower in BFS order, tools/exp43.sh); 2: breadth-first order always
    const bool bfs_order = g->relabel == 2 || (g->relabel == 1 && maxdeg <= BC_LOWDEG && auto_slices(n, c.nnz));
    if (bfs_order && n > 0) {
        // breadth-first (Cuthill-McKee) order from a pseudo-peripheral vertex:
        // a BFS frontier of a long-diameter graph becomes a few contiguous id
        // runs, so the slices kernels' per-vertex sigma/coef slots share sectors
        std::vector<int> hrp(n + 1), hcol((size_t)c.nnz);
        CU(cudaMemcpyAsync(hrp.data(), c.rp, (size_t)(n + 1) * sizeof(int), cudaMemcpyDeviceToHost, st));
        if (c.nnz) CU(cudaMemcpyAsync(hcol.data(), c.col, (size_t)c.nnz * sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        std::vector<int> order, dist(n, -1);
        order.reserve(n);
        auto bfs = [&](int s0) {  // appends s0's component to order; returns its last vertex
            size_t h = order.size();
            dist[s0] = 0;
            order.push_back(s0);
            for (; h < order.size(); ++h) {
                const int v = order[h];
                for (int e = hrp[v]; e < hrp[v + 1]; ++e)
                    if (dist[hcol[e]] < 0) {
                        dist[hcol[e]] = dist[v] + 1;
                        order.push_back(hcol[e]);
                    }
            }
            return order.back();
        };
        for (int v0 = 0; v0 < n; ++v0) {
            if (dist[v0] >= 0) continue;
            const size_t h = order.size();
            const int far = bfs(v0);  // first pass finds a far vertex, the second orders from it
            for (size_t i = h; i < order.size(); ++i) dist[order[i]] = -1;
            order.resize(h);
            bfs(far);
        }
        CU(cudaMemcpyAsync(r.perm, order.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
    } else if (g->relabel && maxdeg > 0) {
        const int end_bit = 32 - __builtin_clz((unsigned)maxdeg);
        size_t tmp_bytes = 0;
        CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in, keys_out, vals_in, r.perm, n, 0, end_bit, st));
        void *tmp = nullptr;
        CU(cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 16)));
        CU(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, vals_in, r.perm, n, 0, end_bit, st));
        CU(cudaStreamSynchronize(st));
        cudaFree(tmp);
    } else {
        CU(cudaMemcpyAsync(r.perm, vals_in, (size_t)n * sizeof(int), cudaMemcpyDeviceToDevice, st));
    }
    invert_perm_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, r.perm, r.inv);
    int *deg_new = nullptr, *tot = nullptr;
    CK(dalloc(&deg_new, n));
    CK(dalloc(&tot, 1));
    permuted_degree_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, r.perm, c.rp, deg_new);
    CK(dalloc(&r.rp, (size_t)n + 1));
    CK(dev_scan(g, deg_new, r.rp, n, tot, st));
    CU(cudaMemcpyAsync(r.rp + n, tot, sizeof(int), cudaMemcpyDeviceToDevice, st));
    r.nnz = c.nnz;
    CK(dalloc(&r.col, (size_t)r.nnz));
    relabel_cols_kernel<<<(unsigned)(((int64_t)n * 32 + 255) / 256), 256, 0, st>>>(n, r.perm, r.inv, c.rp, c.col,
                                                                                   r.rp, r.col);
    if (g->pruned) {
        CK(dalloc(&r.omega, n));
        gather_u32_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, r.perm, g->omega, r.omega);
    }
    std::vector<int> hperm(n);
    CU(cudaMemcpyAsync(hperm.data(), r.perm, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    CU(cudaGetLastError());
    r.h_deg.resize(n);
    r.h_inv.resize(n);
    for (int i = 0; i < n; ++i) {
        r.h_deg[i] = c.h_deg[hperm[i]];
        r.h_inv[hperm[i]] = i;
    }
    dfree(keys_in);
    dfree(keys_out);
    dfree(vals_in);
    dfree(deg_new);
    dfree(tot);
    CK(build_layout(g, r, st));
    g->run_valid = true;
    return BC_OK;
}

// Reorder d_src[0..ns) (compute ids, degree order) by anchor key, stably.
bc_status cluster_sources(bc_graph *g, DevCSR &run, int ns, cudaStream_t st) {
    // grow-only scratch (no per-call cudaMalloc/cudaFree on the timed path)
    if (g->cl_cap < ns) {
        dfree(g->cl_kin);
        dfree(g->cl_kout);
        dfree(g->cl_vout);
        CK(dalloc(&g->cl_kin, ns));
        CK(dalloc(&g->cl_kout, ns));
        CK(dalloc(&g->cl_vout, ns));
        g->cl_cap = ns;
    }
    unsigned long long *kin = g->cl_kin, *kout = g->cl_kout;
    int *vout = g->cl_vout;
    anchor_key_kernel<<<(unsigned)(((int64_t)ns * 32 + 255) / 256), 256, 0, st>>>(g->d_src, ns, run.rp, run.col, kin,
                                                                                 g->src_order == 3 ? 1 : 0);
    const int end_bit = 64;
    size_t tmp_bytes = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin, kout, g->d_src, vout, ns, 0, end_bit, st));
    if (g->cl_tmp_bytes < tmp_bytes) {
        if (g->cl_tmp) cudaFree(g->cl_tmp);
        g->cl_tmp = nullptr;
        CU(cudaMalloc(&g->cl_tmp, std::max<size_t>(tmp_bytes, 16)));
        g->cl_tmp_bytes = tmp_bytes;
    }
    CU(cub::DeviceRadixSort::SortPairs(g->cl_tmp, tmp_bytes, kin, kout, g->d_src, vout, ns, 0, end_bit, st));
    CU(cudaMemcpyAsync(g->d_src, vout, (size_t)ns * 4, cudaMemcpyDeviceToDevice, st));
    return BC_OK;
}

bc_status cluster_sources(bc_graph *g, DevCSR &run, int ns, cudaStream_t st);
__global__ void two_nbr_kernel(const int *cand, int nc, const int *rp, const int *col, int *out);

// NEXT-1 batch plan ("2-degree scheduling"): a source c of
// degree 2 whose neighbours a, b are also sources, none of the three in
// another triple (the paper's restriction: the adjacencies of a 2-degree
// vertex are not adjacencies of another one), becomes a *derived* lane next
// to a and b: lanes 3t, 3t+1, 3t+2 of a word (21 triples per word), so
// lanes_derive_kernel maps a, b onto c with two shifts.  The remaining
// sources fill the other lanes; batches follow the anchor-clustered order of
// the traversed sources, a triple never straddles batches.
bc_status plan_two_degree(bc_graph *g, DevCSR &run, const std::vector<int> &trav, int K, int W, cudaStream_t st,
                          bc_stats &last) {
    const int64_t n = g->n;
    std::vector<int> cand;
    for (int v : trav)
        if (run.h_deg[v] == 2) cand.push_back(v);
    const int64_t need = std::max<int64_t>((int64_t)cand.size() * 3, (int64_t)trav.size());
    if (g->td_cap < need) {
        dfree(g->td_buf);
        CK(dalloc(&g->td_buf, (size_t)need));
        g->td_cap = need;
    }
    std::vector<int> nb(2 * cand.size());
    if (!cand.empty()) {
        CU(cudaMemcpyAsync(g->td_buf, cand.data(), cand.size() * 4, cudaMemcpyHostToDevice, st));
        two_nbr_kernel<<<(unsigned)((cand.size() + 255) / 256), 256, 0, st>>>(g->td_buf, (int)cand.size(), run.rp,
                                                                              run.col, g->td_buf + cand.size());
        CU(cudaMemcpyAsync(nb.data(), g->td_buf + cand.size(), nb.size() * 4, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    std::vector<uint8_t> role((size_t)n, 0);  // 1 = source, 2 = a/b of a triple, 3 = derived c
    for (int v : trav) role[v] = 1;
    std::vector<int> tri_of((size_t)n, -1);
    std::vector<int> tri;  // a, b, c
    for (size_t i = 0; i < cand.size(); ++i) {
        const int c = cand[i], a = nb[2 * i], b = nb[2 * i + 1];
        if (a == b || role[c] != 1 || role[a] != 1 || role[b] != 1) continue;
        role[a] = role[b] = 2;
        role[c] = 3;
        tri_of[a] = tri_of[b] = (int)(tri.size() / 3);
        tri.push_back(a);
        tri.push_back(b);
        tri.push_back(c);
    }
    // traversed sources in anchor-clustered order
    std::vector<int> reals;
    for (int v : trav)
        if (role[v] != 3) reals.push_back(v);
    if (g->src_cap < (int64_t)reals.size()) {
        dfree(g->d_src);
        CK(dalloc(&g->d_src, reals.size()));
        g->src_cap = (int64_t)reals.size();
    }
    CU(cudaMemcpyAsync(g->d_src, reals.data(), reals.size() * 4, cudaMemcpyHostToDevice, st));
    if (g->src_order >= 2 && reals.size() > (size_t)K) {
        CK(cluster_sources(g, run, (int)reals.size(), st));
        CU(cudaMemcpyAsync(reals.data(), g->d_src, reals.size() * 4, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    // pack items (single sources and triples) into batches
    g->td_plan.clear();
    g->td_lanes.clear();
    const int TMAX = 21 * W;
    std::vector<int> bt, bs;  // current batch: triple ids, singles
    std::vector<uint8_t> emitted(tri.size() / 3, 0);
    auto close = [&]() {
        if (bt.empty() && bs.empty()) return;
        bc_graph::TdBatch b{};
        b.off = (int64_t)g->td_lanes.size();
        std::vector<int> lanes(K, -1);
        for (size_t t = 0; t < bt.size(); ++t) {
            const int base = 64 * (int)(t / 21) + 3 * (int)(t % 21);
            for (int r = 0; r < 3; ++r) lanes[base + r] = tri[3 * bt[t] + r];
            b.derived[base / 64] |= 1ull << ((base + 2) & 63);
        }
        size_t si = 0;
        int nl = 0;
        for (int l = 0; l < K; ++l) {
            if (lanes[l] < 0 && si < bs.size()) lanes[l] = bs[si++];
            if (lanes[l] >= 0) nl = l + 1;
        }
        for (int l = 0; l < nl; ++l)
            if (lanes[l] >= 0 && !(b.derived[l >> 6] >> (l & 63) & 1ull)) b.active[l >> 6] |= 1ull << (l & 63);
        b.nl = nl;
        g->td_lanes.insert(g->td_lanes.end(), lanes.begin(), lanes.begin() + nl);
        g->td_plan.push_back(b);
        bt.clear();
        bs.clear();
    };
    for (int v : reals) {
        if (role[v] == 2) {
            const int t = tri_of[v];
            if (emitted[t]) continue;
            if ((int)bt.size() + 1 > TMAX || 3 * ((int)bt.size() + 1) + (int)bs.size() > K) close();
            emitted[t] = 1;
            bt.push_back(t);
        } else {
            if (3 * (int)bt.size() + (int)bs.size() + 1 > K) close();
            bs.push_back(v);
        }
    }
    close();
    last.derived_lanes = (int64_t)(tri.size() / 3);
    const int64_t tot = (int64_t)g->td_lanes.size();
    if (g->src_cap < tot) {
        dfree(g->d_src);
        CK(dalloc(&g->d_src, (size_t)tot));
        g->src_cap = tot;
    }
    CU(cudaMemcpyAsync(g->d_src, g->td_lanes.data(), (size_t)tot * 4, cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));  // td_lanes is pageable host memory
    return BC_OK;
}

bc_status ensure_flags(bc_graph *g, LaneCtx &x, int need) {
    if (x.flag_cap >= need) return BC_OK;
    // sized for the deepest possible BFS (n levels) on first use: the buffer
    // must not move while a level kernel reads its predecessor's flag
    int cap = (int)std::max<int64_t>(need, std::max<int64_t>(g->n + 3, 2 * (int64_t)x.flag_cap));
    dfree(x.d_flags);
    CK(dalloc(&x.d_flags, cap));
    x.flag_cap = cap;
    return BC_OK;
}

bc_status ctx_init(bc_graph *g, LaneCtx &x) {
    if (x.ready) return BC_OK;
    CU(cudaStreamCreateWithFlags(&x.own, cudaStreamNonBlocking));
    CK(dalloc(&x.d_stats, 16));
    CU(cudaMemset(x.d_stats, 0, 16 * sizeof(unsigned long long)));
    CK(dalloc(&x.d_work_ctr, 4));
    CU(cudaMemset(x.d_work_ctr, 0, 4 * sizeof(int)));
    CK(ensure_flags(g, x, 64));
    CU(cudaMallocHost((void **)&x.h_flag, 2 * FLAG_RING * sizeof(int)));
    for (auto &e : x.ev_ring) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming));
    x.ready = true;
    return BC_OK;
}

// fp64 rows on a workspace sized for integer rows: drop the level rows, they
// are re-allocated at 8 bytes per lane by ensure_level (rare: sigma >= 2^32)
bc_status widen_rows(bc_graph *g, LaneWS &ws) {
    if (ws.row_bytes >= 8) return BC_OK;
    CU(cudaDeviceSynchronize());
    for (auto &q : ws.slev) dfree(q);
    ws.slev.clear();
    ws.row_bytes = 8;
    return BC_OK;
}

bc_status ensure_ws(bc_graph *g, LaneWS &ws, int W, bool verify, int nhub, int row_bytes = 8) {
    const size_t n = (size_t)g->n;
    const int K = 64 * W;
    if (ws.W == W && ws.verify == verify && ws.row_bytes != row_bytes) {
        CU(cudaDeviceSynchronize());
        for (auto &q : ws.slev) dfree(q);
        ws.slev.clear();
        ws.row_bytes = row_bytes;
    }
    if (ws.W != W || ws.verify != verify) {
        ws.release();
        ws.row_bytes = row_bytes;
        CK(dalloc(&ws.seen, n * W));
        if (verify) CK(dalloc(&ws.ovf, n * W));
        CK(dalloc(&ws.lane_w1, K));
        CK(dalloc(&ws.lane_ns, K));
        CK(dalloc(&ws.lane_cap, K));
        CK(dalloc(&ws.capmask, 8));
        CK(dalloc(&ws.lvl_snap, 24));
        CK(dalloc(&ws.ns_snap, 3 * (size_t)K));
        CK(dalloc((double **)&ws.part, (size_t)g->num_sms * 8 * BC_NW * 2 * K));
        if (!verify) {
            CK(dalloc(&ws.A, n * (K + BC_A_PAD)));
            CU(cudaMemset(ws.A, 0, n * (K + BC_A_PAD) * sizeof(double)));
            if (BC_REP_H > 0) {
                CK(dalloc(&ws.Arep, (size_t)BC_REP_R * BC_REP_H * K));
                CU(cudaMemset(ws.Arep, 0, (size_t)BC_REP_R * BC_REP_H * K * sizeof(double)));
            }
        }
        ws.W = W;
        ws.verify = verify;
    }
    if (ws.hub_cap < nhub) {
        dfree(ws.hub_acc);
        dfree(ws.hub_ovf);
        CK(dalloc((double **)&ws.hub_acc, (size_t)nhub * K));
        CU(cudaMemset(ws.hub_acc, 0, (size_t)nhub * K * 8));
        if (verify) {
            CK(dalloc(&ws.hub_ovf, (size_t)nhub * W));
            CU(cudaMemset(ws.hub_ovf, 0, (size_t)nhub * W * 8));
        }
        ws.hub_cap = nhub;
    }
    return BC_OK;
}

uint64_t *level_ptr(bc_graph *g, LaneWS &ws, int L) {
    return ws.chunks[L / LCH] + (size_t)(L % LCH) * (size_t)g->n * ws.W;
}

bc_status ensure_level(bc_graph *g, LaneWS &ws, int L) {
    while ((int)ws.chunks.size() * LCH <= L) {
        uint64_t *c = nullptr;
        CK(dalloc(&c, (size_t)g->n * ws.W * LCH));
        ws.chunks.push_back(c);
    }
    const int had = (int)ws.slev.size();
    while ((int)ws.slev.size() <= L) {
        double *q = nullptr;
        bc_status st = dalloc(&q, (size_t)g->n * 8 * ws.W * ws.row_bytes);  // n * K * row_bytes bytes
        if (st != BC_OK)
            return fail(st, "cannot allocate level-%d sigma rows (%.1f GB per level; lower BC_OPT_LANE_WORDS): %s",
                        (int)ws.slev.size(), (double)g->n * 64.0 * ws.W * ws.row_bytes / 1e9, g_err.c_str());
        ws.slev.push_back(q);
    }
    if ((int)ws.slev.size() != had || ws.dptr_cap < (int)ws.slev.size()) {
        // pointer tables for lanes_derive_kernel (grow-only; rare, synchronous)
        const int cap = (int)ws.slev.size();
        if (ws.dptr_cap < cap) {
            dfree(ws.d_lv);
            dfree(ws.d_rows);
            CK(dalloc(&ws.d_lv, (size_t)cap + 8));
            CK(dalloc(&ws.d_rows, (size_t)cap + 8));
            ws.dptr_cap = cap;
        }
        std::vector<uint64_t *> lv(cap);
        for (int l = 0; l < cap; ++l) lv[l] = level_ptr(g, ws, l);
        CU(cudaMemcpy(ws.d_lv, lv.data(), (size_t)cap * sizeof(void *), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ws.d_rows, ws.slev.data(), (size_t)cap * sizeof(void *), cudaMemcpyHostToDevice));
    }
    return BC_OK;
}

// Widening a 16-bit forward at level Lo (bc_api.cu run_batch): the
// discarded expansions wrote levels Lo+1 and Lo+2 -- their lanes leave the
// seen set and their masks are cleared.
__global__ void unsee_levels_kernel(uint64_t *seen, uint64_t *a, uint64_t *b, size_t cnt) {
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, step = (size_t)gridDim.x * blockDim.x;
    for (size_t i = i0; i < cnt; i += step) {
        const uint64_t m = a[i] | b[i];
        if (m) {
            seen[i] &= ~m;
            a[i] = 0;
            b[i] = 0;
        }
    }
}

// per lane: 1 + omega(source) and, with a capture active, the capture slot
// of the lane's source (capmask pre-zeroed)
__global__ void lane_setup_kernel(const int *src, int nl, int K, const uint32_t *omega, double *w1,
                                  const int *cap_vslot, int *lane_cap, unsigned long long *capmask) {
    int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < K) {
        w1[l] = (l < nl && omega && src[l] >= 0) ? 1.0 + (double)omega[src[l]] : 1.0;
        if (cap_vslot) {
            const int c = (l < nl && src[l] >= 0) ? cap_vslot[src[l]] : -1;
            lane_cap[l] = c;
            if (c >= 0) atomicOr(capmask + (l >> 6), 1ull << (l & 63));
        }
    }
}

// occupancy-derived grid for the level kernels
template <typename F>
int level_grid(bc_graph *g, F kern, int units, size_t smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BC_NT, smem);
    if (occ < 1) occ = 1;
    int grid = g->conc ? g->num_sms * occ * BC_FGRID_NUM / BC_FGRID_DEN : g->num_sms * occ;
    return std::max(1, std::min(grid, units));
}

struct BatchCtx {
    const DevCSR *csr;
    const uint32_t *omega;  // nullable
    const int *src;         // device, nl entries
    int nl;
    cudaStream_t st;
    // verification capture (nullable): slot per source (compute ids of this
    // CSR), per-source outputs [slot][n]; cap_depth == nullptr: delta only
    const int *cap_vslot;
    int *cap_depth;
    double *cap_sigma, *cap_delta;
    int *cap_tier;
    bool run_backward;
    bool endpoint;
    std::vector<uint64_t *> *lvl_out;  // verification: level masks used (nullable)
    int *levels_out;
    bool *narrow_failed;    // narrow forward: set when some sigma > 65535 (nothing committed)
    bool *need_fp64;        // ... and set when it had widened to 32-bit rows and sigma >= 2^32 (skip the 32-bit re-run)
    bool *widened;          // set when the forward widened to 32-bit rows at some level (no re-run)
    bool layout;            // 2-degree layout: lanes with src < 0 are unused, derived lanes below
    uint64_t active[8];     // ... lanes traversed by the forward (layout only)
    uint64_t derived[8];    // ... 2-degree lanes (tree derived after the forward)
};

// Run one batch (forward + backward) with K = 64*W lanes.
template <int W, typename SigT>
bc_status run_batch(bc_graph *g, LaneCtx &x, const BatchCtx &c, std::vector<cudaEvent_t> *ev_f,
                    std::vector<cudaEvent_t> *ev_b) {
    constexpr int K = 64 * W;
    const int n = (int)g->n;
    cudaStream_t st = x.st;
    LaneWS &ws = x.ws;
    LanesParams p{};
    p.n = n;
    p.rp = c.csr->rp;
    p.col = c.csr->col;
    p.omega = c.omega;
    p.seen = ws.seen;
    p.ovf = ws.ovf;
    p.bc = x.d_bc;
    p.lane_w1 = ws.lane_w1;
    p.lane_ns = c.omega ? ws.lane_ns : nullptr;
    p.stats = x.d_stats;
    p.work_ctr = x.d_work_ctr;
    for (int j = 0; j < 8; ++j) p.active[j] = 0;
    for (int l = 0; l < c.nl; ++l) p.active[l >> 6] |= 1ull << (l & 63);
    bool any_derived = false;
    for (int j = 0; j < 8; ++j) {
        p.derived[j] = c.layout ? c.derived[j] : 0;
        if (c.layout) p.active[j] = c.active[j];
        any_derived |= p.derived[j] != 0;
    }
    p.hub_deg = g->hub_deg;
    p.nhub = c.csr->nhub;
    p.hub_ids = c.csr->hub_ids;
    p.hub_seg_off = c.csr->hub_seg_off;
    p.nseg = c.csr->nseg;
    p.seg_len = g->hub_deg;
    p.hub_acc = ws.hub_acc;
    p.hub_ovf = ws.hub_ovf;
    p.part = ws.part;
    p.ntiles = c.csr->ntiles;
    p.tile_vs = c.csr->tile_vs;
    p.lane_cap = nullptr;
    p.cap_delta = nullptr;
    p.narrow_ovf = x.d_work_ctr + 2;  // fixed address (d_flags may grow and move with the level count)
    using RT = typename RowOf<SigT>::t;
    // integer rows with a limit (16-bit or 32-bit): re-run the batch wider on overflow
    constexpr bool NARROW = std::is_same<SigT, unsigned>::value || std::is_same<SigT, long long>::value;
    if (NARROW) CU(cudaMemsetAsync(p.narrow_ovf, 0, sizeof(int), st));

    const size_t mbytes = (size_t)n * W * sizeof(uint64_t);
    CK(ensure_level(g, ws, 1));
    if (c.cap_vslot) CU(cudaMemsetAsync(ws.capmask, 0, 8 * sizeof(uint64_t), st));
    lane_setup_kernel<<<(K + 255) / 256, 256, 0, st>>>(c.src, c.nl, K, c.omega, ws.lane_w1, c.cap_vslot, ws.lane_cap,
                                                       (unsigned long long *)ws.capmask);
    CU(cudaMemsetAsync(ws.seen, 0, mbytes, st));
    if (ws.ovf) CU(cudaMemsetAsync(ws.ovf, 0, mbytes, st));
    CU(cudaMemsetAsync(level_ptr(g, ws, 0), 0, mbytes, st));
    CU(cudaMemsetAsync(level_ptr(g, ws, 1), 0, mbytes, st));
    p.any_new = x.d_flags + 1;
    lanes_init_kernel<W, SigT><<<c.nl, BC_NT, 0, st>>>(p, c.src, level_ptr(g, ws, 0), level_ptr(g, ws, 1));
    {
        const unsigned mb = (unsigned)(((int64_t)n + 255) / 256);  // thread per vertex
        lanes_materialize_kernel<W, RT><<<mb, 256, 0, st>>>(n, level_ptr(g, ws, 0), (RT *)ws.slev[0]);
        lanes_materialize_kernel<W, RT><<<mb, 256, 0, st>>>(n, level_ptr(g, ws, 1), (RT *)ws.slev[1]);
    }
    CU(cudaGetLastError());
    x.last.kernel_launches += 4;

    auto kf = lanes_level_kernel<W, SigT>;
    const int units = p.nseg + p.ntiles;
    constexpr size_t SMEM = sizeof(LanesSmem<W, SigT>);
    const int grid = level_grid(g, kf, units, SMEM);
    {
        auto kh = lanes_hub_finalize<W, SigT>;
        cudaFuncSetAttribute(kh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    }
    const int hub_grid = (c.csr->nhub * 32 + BC_NT - 1) / BC_NT;

    // Widening (16-bit tier only): when expansion Lo overflows 16 bits, that
    // one expansion is redone with 32-bit output rows and the batch goes on
    // with 32-bit rows -- levels <= Lo keep their 16-bit rows -- instead of
    // re-running the whole batch.  Counters and n_s are snapshotted before
    // every expansion so the discarded ones can be undone.
    constexpr bool CAN_WIDEN_T = std::is_same<SigT, unsigned>::value;
    const bool can_widen = CAN_WIDEN_T && !any_derived && c.widened != nullptr;
    int wide_from = -1;  // first expansion that writes 32-bit rows
    auto kf_mix = lanes_level_kernel<W, long long, false, true>;  // 16-bit rows in, 32-bit out
    auto kf_32 = lanes_level_kernel<W, long long>;
    constexpr size_t SMEM32 = sizeof(LanesSmem<W, long long>);
    int grid_mix = grid, grid_32 = grid;
    if (can_widen) {
        grid_mix = level_grid(g, kf_mix, units, SMEM32);
        grid_32 = level_grid(g, kf_32, units, SMEM32);
        cudaFuncSetAttribute(lanes_hub_finalize<W, long long>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SMEM32);
    }
    int L = 1, Lmax = 0;
    bool narrow_bad = false;
    for (;;) {
        CK(ensure_level(g, ws, L + 1));
        CK(ensure_flags(g, x, L + 2));
        CU(cudaMemsetAsync(level_ptr(g, ws, L + 1), 0, mbytes, st));
        CU(cudaMemsetAsync(x.d_flags + L + 1, 0, sizeof(int), st));
        if (can_widen && wide_from < 0) {
            CU(cudaMemcpyAsync(ws.lvl_snap + 8 * (L % 3), x.d_stats, 8 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToDevice, st));
            if (p.lane_ns)
                CU(cudaMemcpyAsync(ws.ns_snap + (size_t)K * (L % 3), p.lane_ns, (size_t)K * sizeof(double),
                                   cudaMemcpyDeviceToDevice, st));
        }
        p.level = L;
        p.S_cur = ws.slev[L];
        p.S_nxt = ws.slev[L + 1];
        p.mask_cur = level_ptr(g, ws, L);
        p.mask_nxt = level_ptr(g, ws, L + 1);
        p.mask_nxt_ro = nullptr;
        p.any_new = x.d_flags + L + 1;
        p.prev_new = x.d_flags + L;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (ev_f) {
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, st);
        }
        bool pushed = false;
        if constexpr (std::is_same<SigT, double>::value) {
            if (L <= g->fwd_push_levels) {
                // small frontier: push sigma into the accumulators, then commit
                auto kpf = lanes_push_kernel<W, true>;
                int occp = 1;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occp, kpf, BC_NT, 0);
                const int gridp = std::max(1, std::min(g->conc ? g->num_sms * std::max(1, occp) * BC_PGRID_NUM / BC_PGRID_DEN
                                                          : g->num_sms * std::max(1, occp), units));
                kpf<<<gridp, BC_NT, 0, st>>>(p, ws.A);
                const unsigned cb = (unsigned)std::min<int64_t>(((int64_t)n * 32 + BC_NT - 1) / BC_NT,
                                                                (int64_t)g->num_sms * 8);
                lanes_fwd_commit_kernel<W><<<cb, BC_NT, 0, st>>>(p, ws.A);
                pushed = true;
            }
        }
        if (!pushed) {
            if (wide_from < 0 || L < wide_from) {
                kf<<<grid, BC_NT, SMEM, st>>>(p);
                if (p.nhub > 0) lanes_hub_finalize<W, SigT><<<hub_grid, BC_NT, SMEM, st>>>(p);
            } else {
                if (L == wide_from) kf_mix<<<grid_mix, BC_NT, SMEM32, st>>>(p);
                else kf_32<<<grid_32, BC_NT, SMEM32, st>>>(p);
                if (p.nhub > 0) lanes_hub_finalize<W, long long><<<hub_grid, BC_NT, SMEM32, st>>>(p);
            }
        }
        if (ev_f) {
            cudaEventRecord(e1, st);
            ev_f->push_back(e0);
            ev_f->push_back(e1);
        }
        CU(cudaGetLastError());
        x.last.fwd_launches += 1;
        x.last.kernel_launches += 1 + (p.nhub > 0);
        // termination (the paper's all-reduce of nq) one level
        // behind: the host waits for level L-1's flags while level L runs, so
        // the GPU never idles on the test; the launch past the last level is
        // a no-op (prev_new == 0)
        int *hs = x.h_flag + 2 * (L % FLAG_RING);
        CU(cudaMemcpyAsync(hs, x.d_flags + L + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        if (NARROW) CU(cudaMemcpyAsync(hs + 1, p.narrow_ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaEventRecord(x.ev_ring[L % FLAG_RING], st));
        if (L >= 2) {
            const int *hp = x.h_flag + 2 * ((L - 1) % FLAG_RING);
            const double t0 = trace_on() ? now_us() : 0.0;
            CU(cudaEventSynchronize(x.ev_ring[(L - 1) % FLAG_RING]));
            if (trace_on()) {
                x.sync_us += now_us() - t0;
                x.syncs += 1;
            }
            if (NARROW && hp[1]) {
                if (can_widen && wide_from < 0) {
                    // expansion Lo = L-1 wrote a sigma > 65535: undo it and the
                    // speculative expansion L, then redo Lo with 32-bit rows
                    const int Lo = L - 1;
                    CU(cudaStreamSynchronize(st));
                    const unsigned ub = (unsigned)std::min<size_t>((n * (size_t)W + 255) / 256, (size_t)g->num_sms * 8);
                    unsee_levels_kernel<<<ub, 256, 0, st>>>(ws.seen, level_ptr(g, ws, Lo + 1), level_ptr(g, ws, Lo + 2),
                                                            (size_t)n * W);
                    CU(cudaMemcpyAsync(x.d_stats, ws.lvl_snap + 8 * (Lo % 3), 8 * sizeof(unsigned long long),
                                       cudaMemcpyDeviceToDevice, st));
                    if (p.lane_ns)
                        CU(cudaMemcpyAsync(p.lane_ns, ws.ns_snap + (size_t)K * (Lo % 3), (size_t)K * sizeof(double),
                                           cudaMemcpyDeviceToDevice, st));
                    CU(cudaMemsetAsync(p.narrow_ovf, 0, sizeof(int), st));
                    CU(cudaGetLastError());
                    x.last.kernel_launches += 1;
                    x.last.fwd_launches -= 2;  // the two discarded expansions
                    wide_from = Lo;
                    *c.widened = true;
                    L = Lo;
                    continue;
                }
                narrow_bad = true;  // sigma overflowed: the batch is re-run wider
                if (wide_from >= 0 && c.need_fp64) *c.need_fp64 = true;  // 32-bit rows overflowed too
            }
            if (narrow_bad || hp[0] == 0) {
                Lmax = L - 1;
                x.last.fwd_launches -= 1;  // the no-op launch
                break;
            }
        }
        ++L;
    }
    p.prev_new = nullptr;  // forward-only gate
    x.last.levels_total += Lmax;
    if (c.levels_out) *c.levels_out = Lmax;
    if (c.lvl_out) {
        c.lvl_out->clear();
        for (int l = 0; l <= Lmax; ++l) c.lvl_out->push_back(level_ptr(g, ws, l));
    }
    if constexpr (NARROW) {
        // some sigma exceeded 16 bits: nothing has been committed to BC yet,
        // the caller re-runs this batch with fp64 rows
        if (narrow_bad) {
            if (c.narrow_failed) *c.narrow_failed = true;
            return BC_OK;
        }
    }
    int Lb = Lmax;  // deepest level of the backward sweep
    if (any_derived && !std::is_same<SigT, unsigned long long>::value) {
        // 2-degree lanes (NEXT-1): derive their trees from lanes a, b; they may
        // reach one level deeper than the traversed lanes (levels <= Lmax + 1
        // are allocated and their masks zeroed by the level loop)
        CK(ensure_level(g, ws, Lmax + 1));
        DeriveParams q{};
        q.n = n;
        q.nlev = Lmax + 1;
        q.lvl = ws.d_lv;
        q.rows = ws.d_rows;
        q.rp = c.csr->rp;
        for (int j = 0; j < 8; ++j) q.cmask[j] = p.derived[j];
        q.stats = x.d_stats;
        q.ovf = p.narrow_ovf;
        lanes_derive_kernel<W, RT><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(q);
        if (p.lane_ns) derive_ns_kernel<<<(K + 255) / 256, 256, 0, st>>>(K, q, ws.lane_ns);
        x.last.kernel_launches += 1 + (p.lane_ns != nullptr);
        if constexpr (NARROW) {
            CU(cudaMemcpyAsync(x.h_flag + 1, p.narrow_ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            if (x.h_flag[1]) {
                if (c.narrow_failed) *c.narrow_failed = true;
                return BC_OK;
            }
        }
        Lb = Lmax + 1;
    }
    if (c.cap_vslot && c.cap_depth) {
        // verification capture: depth and sigma of the captured lanes, from
        // the level masks and sigma rows of this (completed) forward
        const unsigned vb = (unsigned)(((int64_t)n + 255) / 256);
        for (int l = 0; l <= Lb; ++l) {
            if (wide_from >= 0 && l > wide_from)  // widened batch: 32-bit rows past the widening level
                cap_extract_kernel<W, uint32_t><<<vb, 256, 0, st>>>(n, l, level_ptr(g, ws, l), (const uint32_t *)ws.slev[l],
                                                                    ws.lane_cap, ws.capmask, c.cap_depth, c.cap_sigma);
            else
                cap_extract_kernel<W, RT><<<vb, 256, 0, st>>>(n, l, level_ptr(g, ws, l), (const RT *)ws.slev[l],
                                                              ws.lane_cap, ws.capmask, c.cap_depth, c.cap_sigma);
        }
        cap_tier_kernel<<<(K + 255) / 256, 256, 0, st>>>(K, ws.lane_cap, wide_from >= 0 ? 32 : 8 * (int)sizeof(RT),
                                                         c.cap_tier);
        CU(cudaGetLastError());
    }
    if constexpr (!std::is_same<SigT, unsigned long long>::value) {
        bool pulled = false;
        if constexpr (std::is_same<SigT, double>::value) {
        if (c.run_backward && g->bwd_mode == 2) {
            pulled = true;
            // pull-form backward (successor checking, Alg.5): level-L vertices
            // gather the coef rows of their level-(L+1) children
            auto kb = lanes_level_kernel<W, SigT, true>;
            const int gridb = level_grid(g, kb, units, SMEM);
            auto khb = lanes_hub_finalize<W, SigT, true>;
            cudaFuncSetAttribute(khb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
            p.lane_cap = c.cap_vslot ? ws.lane_cap : nullptr;
            p.cap_delta = c.cap_delta;
            p.arep = ws.Arep;
            for (int l = Lb; l >= 1; --l) {
                p.level = l;
                p.S_cur = ws.slev[l];
                p.S_nxt = ws.slev[l + 1];
                p.mask_cur = level_ptr(g, ws, l);
                p.mask_nxt_ro = level_ptr(g, ws, l + 1);  // all zero for l == Lmax
                p.mask_nxt = nullptr;
                p.any_new = x.d_flags;  // unused
                cudaEvent_t e0 = nullptr, e1 = nullptr;
                if (ev_b) {
                    cudaEventCreate(&e0);
                    cudaEventCreate(&e1);
                    cudaEventRecord(e0, st);
                }
                kb<<<gridb, BC_NT, SMEM, st>>>(p);
                if (p.nhub > 0) khb<<<hub_grid, BC_NT, SMEM, st>>>(p);
                if (ev_b) {
                    cudaEventRecord(e1, st);
                    ev_b->push_back(e0);
                    ev_b->push_back(e1);
                }
                CU(cudaGetLastError());
                x.last.bwd_launches += 1;
                x.last.kernel_launches += 1 + (p.nhub > 0);
            }
        }
        }
        if (c.run_backward && !pulled) {
            // push-form backward (bwd_push.cuh): for L >= 2 the push kernel forms
            // coef of the level-L vertices from sigma and A (fused finalize) and
            // pushes it into the parents' accumulators; hubs are finalised by a
            // warp-per-hub kernel after it, level 1 by the finalize scan
            auto kpush = lanes_push_kernel<W, false, RT>;
            auto kpush32 = lanes_push_kernel<W, false, uint32_t>;  // levels past a widening (32-bit rows)
            cudaFuncSetAttribute(kpush, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            if (wide_from >= 0) cudaFuncSetAttribute(kpush32, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            int occp = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occp, kpush, BC_NT, 0);
            const int gridp = std::max(1, std::min(g->conc ? g->num_sms * std::max(1, occp) * BC_PGRID_NUM / BC_PGRID_DEN
                                                          : g->num_sms * std::max(1, occp), units));
            const unsigned fin_blocks = (unsigned)std::min<int64_t>(((int64_t)n * 32 + BC_NT - 1) / BC_NT,
                                                                    (int64_t)g->num_sms * 8);
            p.lane_cap = c.cap_vslot ? ws.lane_cap : nullptr;
            p.cap_delta = c.cap_delta;
            for (int l = Lb; l >= 1; --l) {
                p.level = l;
                p.S_cur = ws.slev[l];
                p.S_nxt = nullptr;
                p.mask_cur = level_ptr(g, ws, l);
                p.mask_nxt_ro = level_ptr(g, ws, l - 1);  // parents
                p.mask_nxt = nullptr;
                p.any_new = x.d_flags;  // unused
                cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
                if (ev_b) {
                    cudaEventCreate(&e0);
                    cudaEventCreate(&e1);
                    cudaEventCreate(&e2);
                    cudaEventCreate(&e3);
                    cudaEventRecord(e0, st);
                }
                const bool w32 = wide_from >= 0 && l > wide_from;
                if (p.arep && l < Lb) lanes_rep_fold_kernel<W><<<(BC_REP_H * K + BC_NT - 1) / BC_NT, BC_NT, 0, st>>>(p, ws.A);
                if (l >= 2) {
                    if (w32) kpush32<<<gridp, BC_NT, 0, st>>>(p, ws.A);
                    else kpush<<<gridp, BC_NT, 0, st>>>(p, ws.A);
                }
                if (ev_b) {
                    cudaEventRecord(e1, st);
                    cudaEventRecord(e2, st);
                }
                int nk = (l >= 2);
                if (l == 1) {
                    lanes_bwd_finalize_kernel<W, false, RT><<<fin_blocks, BC_NT, 0, st>>>(p, ws.A);
                    ++nk;
                } else if (p.nhub > 0) {
                    if (w32)
                        lanes_bwd_hub_fin_kernel<W, uint32_t><<<(p.nhub * 32 + BC_NT - 1) / BC_NT, BC_NT, 0, st>>>(p, ws.A);
                    else
                        lanes_bwd_hub_fin_kernel<W, RT><<<(p.nhub * 32 + BC_NT - 1) / BC_NT, BC_NT, 0, st>>>(p, ws.A);
                    ++nk;
                }
                if (ev_b) {
                    cudaEventRecord(e3, st);
                    x.epush.push_back(e0);
                    x.epush.push_back(e1);
                    ev_b->push_back(e2);
                    ev_b->push_back(e3);
                }
                CU(cudaGetLastError());
                x.last.bwd_launches += 1;
                x.last.kernel_launches += nk;
            }
        }
        if (c.run_backward && c.endpoint && c.omega) {
            lanes_endpoint_kernel<<<(c.nl + 255) / 256, 256, 0, st>>>(c.src, c.nl, c.omega, ws.lane_ns, x.d_bc);
            x.last.kernel_launches += 1;
        }
    }
    CU(cudaGetLastError());
    return BC_OK;
}

template <typename SigT>
bc_status run_batch_w(bc_graph *g, LaneCtx &x, int W, const BatchCtx &c, std::vector<cudaEvent_t> *ef,
                      std::vector<cudaEvent_t> *eb) {
    switch (W) {
        case 1: return run_batch<1, SigT>(g, x, c, ef, eb);
        case 2: return run_batch<2, SigT>(g, x, c, ef, eb);
        case 4: return run_batch<4, SigT>(g, x, c, ef, eb);
        case 8: return run_batch<8, SigT>(g, x, c, ef, eb);
        default: return fail(BC_ERR_INTERNAL, "bad lane words %d", W);
    }
}


// ---------------------------------------------------------------------
// Device-driven batch (graph mode).  One batch of K lanes -- the forward
// levels, the sigma-tier fallbacks and the backward levels -- enqueued with
// no host round trip: Lcap forward and backward level slots are unrolled
// (Lcap = the graph's depth bound, so every BFS fits), a slot is a no-op
// when its level is empty, and each sigma tier (16-bit rows, then 32-bit,
// then fp64 when the rows are 8 bytes wide) is a no-op unless the previous
// tier overflowed (batch_ctl.cuh).  The sequence is captured once per
// pipeline into a CUDA graph and launched once per batch; the batch's
// sources come from the pipeline's device table, so the graph does not
// change between batches or calls.
struct DevBatchCfg {
    const DevCSR *csr;
    const uint32_t *omega;  // nullable
    int lcap;               // forward levels 1..lcap are expanded; level lcap+1 must be empty
    bool fp64_inline;       // 8-byte rows: the fp64 tier runs in the graph
    bool capture;           // verification capture (bc_set_capture) rides along
};

template <int W, typename SigT>
void enqueue_tier(bc_graph *g, LaneCtx &x, const DevBatchCfg &cfg, const int *need, int *ovf_self) {
    constexpr int K = 64 * W;
    using RT = typename RowOf<SigT>::t;
    constexpr bool INTROW = !std::is_same<SigT, double>::value;
    const int n = (int)g->n;
    cudaStream_t st = x.st;
    LaneWS &ws = x.ws;
    const DevCSR &csr = *cfg.csr;
    const int *halt = INTROW ? ovf_self : nullptr;
    LanesParams p{};
    p.n = n;
    p.rp = csr.rp;
    p.col = csr.col;
    p.omega = cfg.omega;
    p.seen = ws.seen;
    p.ovf = nullptr;
    p.bc = x.d_bc;
    p.lane_w1 = ws.lane_w1;
    p.lane_ns = cfg.omega ? ws.lane_ns : nullptr;
    p.stats = x.d_stats;
    p.work_ctr = x.d_work_ctr;
    p.active_dev = x.gb_active;
    p.need = need;
    p.halt = halt;
    p.hub_deg = g->hub_deg;
    p.nhub = csr.nhub;
    p.hub_ids = csr.hub_ids;
    p.hub_seg_off = csr.hub_seg_off;
    p.nseg = csr.nseg;
    p.seg_len = g->hub_deg;
    p.hub_acc = ws.hub_acc;
    p.part = ws.part;
    p.ntiles = csr.ntiles;
    p.tile_vs = csr.tile_vs;
    p.narrow_ovf = INTROW ? ovf_self : x.gb_ctl + 5;
    p.lane_cap = cfg.capture ? ws.lane_cap : nullptr;
    p.cap_delta = cfg.capture ? g->capt.d_delta : nullptr;
    const size_t nmask = (size_t)n * W;
    const unsigned zb = (unsigned)std::min<size_t>((nmask + 255) / 256, (size_t)g->num_sms * 8);
    // tier start: state cleared, counters restored
    gb_reset_kernel<<<std::max(zb, (unsigned)((cfg.lcap + 3 + 255) / 256)), 256, 0, st>>>(
        ws.seen, level_ptr(g, ws, 0), level_ptr(g, ws, 1), nmask, (uint64_t *)ws.hub_acc, (size_t)csr.nhub * K,
        x.d_flags, cfg.lcap + 3, x.d_stats, x.gb_stats_bak, need, nullptr);
    if (cfg.capture) CU_V(cudaMemsetAsync(ws.capmask, 0, 8 * sizeof(uint64_t), st));
    lane_setup_kernel<<<(K + 255) / 256, 256, 0, st>>>(x.gb_src, K, K, cfg.omega, ws.lane_w1,
                                                       cfg.capture ? g->capt.d_vslot : nullptr, ws.lane_cap,
                                                       (unsigned long long *)ws.capmask);
    p.any_new = x.d_flags + 1;
    lanes_init_kernel<W, SigT><<<K, BC_NT, 0, st>>>(p, x.gb_src, level_ptr(g, ws, 0), level_ptr(g, ws, 1));
    const unsigned mb = (unsigned)(((int64_t)n + 255) / 256);
    lanes_materialize_kernel<W, RT><<<mb, 256, 0, st>>>(n, level_ptr(g, ws, 0), (RT *)ws.slev[0], need, halt);
    lanes_materialize_kernel<W, RT><<<mb, 256, 0, st>>>(n, level_ptr(g, ws, 1), (RT *)ws.slev[1], need, halt);
    // forward slots
    auto kf = lanes_level_kernel<W, SigT>;
    constexpr size_t SMEM = sizeof(LanesSmem<W, SigT>);
    const int units = p.nseg + p.ntiles;
    const int grid = level_grid(g, kf, units, SMEM);
    cudaFuncSetAttribute(lanes_hub_finalize<W, SigT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    const int hub_grid = (csr.nhub * 32 + BC_NT - 1) / BC_NT;
    for (int L = 1; L <= cfg.lcap; ++L) {
        gb_zero_level_kernel<<<zb, 256, 0, st>>>(level_ptr(g, ws, L + 1), nmask, x.d_flags + L + 1, need);
        p.level = L;
        p.S_cur = ws.slev[L];
        p.S_nxt = ws.slev[L + 1];
        p.mask_cur = level_ptr(g, ws, L);
        p.mask_nxt = level_ptr(g, ws, L + 1);
        p.mask_nxt_ro = nullptr;
        p.any_new = x.d_flags + L + 1;
        p.prev_new = x.d_flags + L;
        kf<<<grid, BC_NT, SMEM, st>>>(p);
        if (p.nhub > 0) lanes_hub_finalize<W, SigT><<<hub_grid, BC_NT, SMEM, st>>>(p);
    }
    if (cfg.capture) {
        const unsigned vb = (unsigned)(((int64_t)n + 255) / 256);
        for (int l = 0; l <= cfg.lcap; ++l)
            cap_extract_kernel<W, RT><<<vb, 256, 0, st>>>(n, l, level_ptr(g, ws, l), (const RT *)ws.slev[l],
                                                          ws.lane_cap, ws.capmask, g->capt.d_depth, g->capt.d_sigma,
                                                          need, halt, l == 0 ? nullptr : x.d_flags + l);
        cap_tier_kernel<<<(K + 255) / 256, 256, 0, st>>>(K, ws.lane_cap, 8 * (int)sizeof(RT), g->capt.d_tier, need,
                                                         halt);
    }
    // backward slots (push form, fused finalize; level 1 by the finalize scan)
    auto kpush = lanes_push_kernel<W, false, RT>;
    cudaFuncSetAttribute(kpush, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occp = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occp, kpush, BC_NT, 0);
    const int gridp = std::max(1, std::min(g->conc ? g->num_sms * std::max(1, occp) * BC_PGRID_NUM / BC_PGRID_DEN
                                                          : g->num_sms * std::max(1, occp), units));
    const unsigned fin_blocks = (unsigned)std::min<int64_t>(((int64_t)n * 32 + BC_NT - 1) / BC_NT, (int64_t)g->num_sms * 8);
    p.arep = ws.Arep;
    for (int l = cfg.lcap; l >= 1; --l) {
        p.level = l;
        p.S_cur = ws.slev[l];
        p.S_nxt = nullptr;
        p.mask_cur = level_ptr(g, ws, l);
        p.mask_nxt_ro = level_ptr(g, ws, l - 1);
        p.mask_nxt = nullptr;
        p.any_new = x.gb_ctl + 5;  // unused
        p.prev_new = x.d_flags + l;  // level l non-empty
        if (p.arep && l < cfg.lcap) lanes_rep_fold_kernel<W><<<(BC_REP_H * K + BC_NT - 1) / BC_NT, BC_NT, 0, st>>>(p, ws.A);
        if (l >= 2) kpush<<<gridp, BC_NT, 0, st>>>(p, ws.A);
        if (l == 1)
            lanes_bwd_finalize_kernel<W, false, RT><<<fin_blocks, BC_NT, 0, st>>>(p, ws.A);
        else if (p.nhub > 0)
            lanes_bwd_hub_fin_kernel<W, RT><<<(p.nhub * 32 + BC_NT - 1) / BC_NT, BC_NT, 0, st>>>(p, ws.A);
    }
    if (cfg.omega)
        lanes_endpoint_kernel<<<(K + 255) / 256, 256, 0, st>>>(x.gb_src, K, cfg.omega, ws.lane_ns, x.d_bc, need, halt);
}

#ifndef BC_DEVLOOP_COND
#define BC_DEVLOOP_COND 1  // on graphs with n > 2^18 the 32-bit / fp64 tiers sit in conditional (IF) graph
#endif                     // nodes instead of gated launches (S20 -0.9 %; on S12 the IF nodes cost more than the
                           // ~70 no-op launches they skip: 1.85 -> 2.55 ms, profiles/exp_r2_devloop_cond.txt)

// At the capture point of x.st: an IF node whose condition (*flag != 0) a
// one-thread kernel sets on the device, with `body` captured into the node's
// body graph on the side stream `side` (x.st points at it meanwhile).
template <typename F>
bc_status capture_if(LaneCtx &x, cudaStream_t side, const int *flag, F &&body) {
    cudaStream_t st = x.st;
    cudaStreamCaptureStatus cs;
    cudaGraph_t graph = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    CU(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &nd));
    cudaGraphConditionalHandle h;
    CU(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault));
    gb_set_cond_kernel<<<1, 1, 0, st>>>(h, flag);
    CU(cudaGetLastError());
    CU(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &nd));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeIf;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CU(cudaGraphAddNode(&node, graph, deps, nd, &np));
    cudaGraph_t body_graph = np.conditional.phGraph_out[0];
    CU(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    CU(cudaStreamBeginCaptureToGraph(side, body_graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    x.st = side;
    const bc_status s = body();
    x.st = st;
    cudaGraph_t tmp = nullptr;
    const cudaError_t e = cudaStreamEndCapture(side, &tmp);
    if (s != BC_OK) return s;
    CU(e);
    return BC_OK;
}

template <int W>
bc_status enqueue_device_batch(bc_graph *g, LaneCtx &x, const DevBatchCfg &cfg, cudaStream_t side1,
                               cudaStream_t side2) {
    constexpr int K = 64 * W;
    gb_begin_kernel<<<1, 512, 0, x.st>>>(x.gb_table, x.gb_ctl, g->d_src, K, x.gb_src, x.gb_active, x.d_stats,
                                         x.gb_stats_bak);
    enqueue_tier<W, unsigned>(g, x, cfg, nullptr, x.gb_ctl + 2);
    if (BC_DEVLOOP_COND && side1 && g->n > (1 << 18)) {
        // 32-bit tier only if the 16-bit one overflowed, fp64 only if the 32-bit one did
        CK(capture_if(x, side1, x.gb_ctl + 2, [&]() -> bc_status {
            enqueue_tier<W, long long>(g, x, cfg, x.gb_ctl + 2, x.gb_ctl + 3);
            if (cfg.fp64_inline)
                CK(capture_if(x, side2, x.gb_ctl + 3, [&]() -> bc_status {
                    enqueue_tier<W, double>(g, x, cfg, x.gb_ctl + 3, nullptr);
                    return BC_OK;
                }));
            return BC_OK;
        }));
    } else {
        enqueue_tier<W, long long>(g, x, cfg, x.gb_ctl + 2, x.gb_ctl + 3);
        if (cfg.fp64_inline) enqueue_tier<W, double>(g, x, cfg, x.gb_ctl + 3, nullptr);
    }
    gb_end_kernel<<<1, 32, 0, x.st>>>(x.gb_ctl, x.d_flags, cfg.lcap, x.gb_cnt, x.gb_redo, cfg.fp64_inline ? 1 : 0,
                                      x.d_stats, x.gb_stats_bak);
    CU(cudaGetLastError());
    return BC_OK;
}

bc_status enqueue_device_batch_w(bc_graph *g, LaneCtx &x, int W, const DevBatchCfg &cfg, cudaStream_t s1,
                                 cudaStream_t s2) {
    switch (W) {
        case 1: return enqueue_device_batch<1>(g, x, cfg, s1, s2);
        case 2: return enqueue_device_batch<2>(g, x, cfg, s1, s2);
        case 4: return enqueue_device_batch<4>(g, x, cfg, s1, s2);
        case 8: return enqueue_device_batch<8>(g, x, cfg, s1, s2);
        default: return fail(BC_ERR_INTERNAL, "bad lane words %d", W);
    }
}

// The pipeline's graph: rebuilt only when something it bakes in changed
// (the buffers, the CSR, the lane width, the depth bound, the tier set).
bc_status device_batch_graph(bc_graph *g, LaneCtx &x, int W, const DevBatchCfg &cfg) {
    std::vector<uintptr_t> key = {(uintptr_t)W,
                                  (uintptr_t)cfg.lcap,
                                  (uintptr_t)cfg.fp64_inline,
                                  (uintptr_t)cfg.capture,
                                  (uintptr_t)cfg.omega,
                                  (uintptr_t)cfg.csr->rp,
                                  (uintptr_t)cfg.csr->col,
                                  (uintptr_t)cfg.csr->tile_vs,
                                  (uintptr_t)cfg.csr->hub_ids,
                                  (uintptr_t)g->hub_deg,
                                  (uintptr_t)g->conc,
                                  (uintptr_t)x.ws.seen,
                                  (uintptr_t)x.ws.A,
                                  (uintptr_t)x.ws.hub_acc,
                                  (uintptr_t)x.ws.part,
                                  (uintptr_t)x.d_flags,
                                  (uintptr_t)x.d_bc,
                                  (uintptr_t)x.gb_table,
                                  (uintptr_t)g->d_src,
                                  (uintptr_t)g->capt.d_vslot,
                                  (uintptr_t)g->capt.d_depth};
    for (int l = 0; l <= cfg.lcap + 1; ++l) {
        key.push_back((uintptr_t)x.ws.slev[l]);
        key.push_back((uintptr_t)level_ptr(g, x.ws, l));
    }
    if (x.gexec && key == x.gkey) return BC_OK;
    if (x.gexec) cudaGraphExecDestroy(x.gexec), x.gexec = nullptr;
    x.gkey.clear();
    if (!x.side[0]) {  // side streams the conditional tiers' bodies are captured on
        CU(cudaStreamCreateWithFlags(&x.side[0], cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&x.side[1], cudaStreamNonBlocking));
    }
    CU(cudaStreamBeginCapture(x.st, cudaStreamCaptureModeThreadLocal));
    bc_status s = enqueue_device_batch_w(g, x, W, cfg, x.side[0], x.side[1]);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(x.st, &graph);
    if (s != BC_OK) {
        if (graph) cudaGraphDestroy(graph);
        return s;
    }
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(BC_ERR_CUDA, "graph capture of the device-driven batch failed: %s", cudaGetErrorString(e));
    }
    cudaGraphGetNodes(graph, nullptr, &x.gnodes);
    const cudaError_t ei = cudaGraphInstantiate(&x.gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        (void)cudaGetLastError();
        x.gexec = nullptr;
        return fail(BC_ERR_CUDA, "graph instantiation failed: %s", cudaGetErrorString(ei));
    }
    x.gkey = key;
    return BC_OK;
}

bc_status ensure_device_batch(bc_graph *g, LaneCtx &x, int nbatches) {
    if (!x.gb_src) {
        CK(dalloc(&x.gb_src, 512));
        CK(dalloc(&x.gb_ctl, 8));
        CK(dalloc(&x.gb_active, 8));
        CK(dalloc(&x.gb_cnt, 8));
        CK(dalloc(&x.gb_stats_bak, 8));
        CU(cudaMemset(x.gb_ctl, 0, 8 * sizeof(int)));
    }
    if (x.gb_table_cap < nbatches) {
        dfree(x.gb_table);
        dfree(x.gb_redo);
        const int cap = std::max(nbatches, 2 * x.gb_table_cap);
        CK(dalloc(&x.gb_table, cap));
        CK(dalloc(&x.gb_redo, cap));
        x.gb_table_cap = cap;
    }
    return BC_OK;
}

bc_status ensure_slices(bc_graph *g, int rows, bool full, bool reuse) {
    if (g->sws.rows >= rows && (g->sws.full || !full) && (g->sws.cdq || !reuse)) return BC_OK;
    g->sws.release();
    const size_t n = (size_t)g->n;
    SlicesWS &w = g->sws;
    const size_t bmw = (n + 31) / 32;
    const size_t cnt = n * rows;
    CK(dalloc(&w.bm, 3 * bmw * rows));
    CK(dalloc(&w.queue, n * rows));
    CK(dalloc(&w.loff, (n + 2) * rows));
    CK(dalloc(&w.sigma, cnt));
    CK(dalloc(&w.ell, n));
#if BC_SM_QROW
    CK(dalloc(&w.qrow, n * rows));
#endif
    if (w.bm) CU(cudaMemset(w.bm, 0, 3 * bmw * rows * sizeof(unsigned)));
    CU(cudaMemset(w.sigma, 0, cnt * 8));
    if (full) {
        CK(dalloc(&w.cf, cnt));
        CK(dalloc(&w.bcp, cnt));
        CU(cudaMemset(w.cf, 0, cnt * 8));
        CU(cudaMemset(w.bcp, 0, cnt * 8));
    }
    if (reuse) CK(dalloc(&w.cdq, cnt));
    CU(cudaDeviceSynchronize());
    w.rows = rows;
    w.full = full;
    return BC_OK;
}

// One CTA per source (persistent grid), for long-diameter graphs.
bc_status run_slices(bc_graph *g, DevCSR &run, const int *d_src, int ns, cudaStream_t st,
                     std::vector<cudaEvent_t> *ev, bool cap) {
#ifndef BC_SLICES_SMEM_BM
#define BC_SLICES_SMEM_BM 0  // shared-memory bitmaps cost occupancy; global (L2-resident) ones measured faster
#endif
#ifndef BC_SLICES_ELL
#define BC_SLICES_ELL 1
#endif
#ifndef BC_SLICES_SM2
#define BC_SLICES_SM2 1  // 2-bit per-vertex state in shared memory when it fits (BC_SLICES_SM2_MAXB)
#endif
#ifndef BC_SLICES_SM2_MAXB
#define BC_SLICES_SM2_MAXB (72 * 1024)
#endif
    int maxdeg = 0;
    for (int d : run.h_deg) maxdeg = std::max(maxdeg, d);
    const size_t sm2_bytes = (size_t)((g->n + 15) / 16) * sizeof(unsigned);
    // kernel: auto = the shared-memory 2-bit state kernel when the graph is
    // degree-bounded and the state fits, else the global-bitmap degree-bounded
    // kernel, else the general one (CD scan + binary search mapping);
    // BC_OPT_SLICES_KERNEL forces one (NEXT-2 ablation)
    const int sk = g->slices_kernel;
    const bool can_low = maxdeg <= BC_LOWDEG;
    const bool can_sm2 = can_low && sm2_bytes <= (size_t)BC_SLICES_SM2_MAXB;
    if ((sk == 3 && !can_low) || (sk == 4 && !can_sm2))
        return fail(BC_ERR_INVALID, "slices kernel %d needs max degree <= %d%s", sk, BC_LOWDEG,
                    sk == 4 ? " and n <= 1179648" : "");
    const bool lowdeg = sk == 0 ? can_low : (sk == 3 || sk == 4);  // vertex-per-thread pull variant, no fp atomics
    const bool reuse = sk == 2;                                    // general kernel with prefix-sum reuse
    const bool ell = BC_SLICES_ELL && maxdeg <= 4;  // neighbours as one int4 load
    const bool sm2 = lowdeg && (sk == 4 || (sk == 0 && BC_SLICES_SM2 && can_sm2));
    const bool smem_bm = !lowdeg && BC_SLICES_SMEM_BM && g->n <= (int64_t)SLICES_SMEM_BM_WORDS * 32;
    const size_t dsm = sm2 ? sm2_bytes : smem_bm ? 2 * SLICES_SMEM_BM_WORDS * sizeof(unsigned) : 0;
    // CAP instantiations (verification capture, bc_set_capture) keep the
    // capture stores out of the timed kernels
    auto kern = sm2      ? (ell ? (cap ? slices_lowdeg_sm_kernel<true, true> : slices_lowdeg_sm_kernel<true>)
                                : (cap ? slices_lowdeg_sm_kernel<false, true> : slices_lowdeg_sm_kernel<false>))
                : lowdeg ? (ell ? (cap ? slices_lowdeg_kernel<true, true> : slices_lowdeg_kernel<true>)
                                : (cap ? slices_lowdeg_kernel<false, true> : slices_lowdeg_kernel<false>))
                : reuse  ? (cap ? slices_kernel<false, true, true> : slices_kernel<false, false, true>)
                         : (smem_bm ? (cap ? slices_kernel<true, true> : slices_kernel<true>)
                                    : (cap ? slices_kernel<false, true> : slices_kernel<false>));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
    int occ = 1;
    const int nt = sm2 ? BC_SM_NT : lowdeg ? BC_SL_NT : BC_NT;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, dsm);
#ifdef BC_SL_OCC
    if (lowdeg) occ = std::min(occ, BC_SL_OCC);  // experiment builds: cap the sources in flight per SM
#endif
    const int rows = std::max(1, std::min(ns, g->num_sms * std::max(1, occ)));
    CK(ensure_slices(g, rows, !lowdeg, reuse));
    if (ell) {
        build_ell4_kernel<<<(unsigned)((g->n + 255) / 256), 256, 0, st>>>((int)g->n, run.rp, run.col, g->sws.ell);
        g->last.kernel_launches += 1;
    }
    SlicesParams p{};
    p.n = (int)g->n;
    p.rp = run.rp;
    p.col = run.col;
    p.omega = g->pruned ? run.omega : nullptr;
    p.src = d_src;
    p.nsrc = ns;
    p.next_src = g->d_work_ctr + 1;
    p.bm = g->sws.bm;
    p.bm_words = (int)((g->n + 31) / 32);
    p.sigma = g->sws.sigma;
    p.cf = g->sws.cf;
    p.queue = g->sws.queue;
    p.loff = g->sws.loff;
    p.bcp = g->sws.bcp;
    p.bc = g->d_bc;
    p.ell4 = ell ? g->sws.ell : nullptr;
    p.qrow = g->sws.qrow;
    p.cdq = g->sws.cdq;
    p.stats = g->d_stats;
    if (cap) {
        p.cap_vslot = g->capt.d_vslot;
        p.cap_depth = g->capt.d_depth;
        p.cap_sigma = g->capt.d_sigma;
        p.cap_delta = g->capt.d_delta;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ev) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
    }
    kern<<<rows, nt, dsm, st>>>(p);
    if (ev) {
        cudaEventRecord(e1, st);
        ev->push_back(e0);
        ev->push_back(e1);
    }
    if (!lowdeg)  // the degree-bounded kernel adds into d_bc directly
        slices_reduce_kernel<<<(unsigned)((g->n + 255) / 256), 256, 0, st>>>((int)g->n, rows, g->sws.bcp, g->d_bc);
    CU(cudaGetLastError());
    g->last.kernel_launches += lowdeg ? 1 : 2;
    g->last.batches += 1;
    g->last.lanes = 1;
    return BC_OK;
}

// Entry points that rebuild or reuse the handle's device state wait for an
// asynchronous bc_compute still in flight.
bc_status wait_idle(bc_graph *g) {
    if (g->stats_ev) CU(cudaEventSynchronize(g->stats_ev));
    return BC_OK;
}

// The call's counters from pinned memory (copied at the end of bc_compute):
// the kernels' A_s / D_s / n_s / item counters and, for device-driven
// pipelines, the level and sigma-tier counters of batch_ctl.cuh.
void finalize_stats(bc_graph *g) {
    const unsigned long long *h = g->h_pin;
    g->last.reached = (int64_t)h[0];
    g->last.adj_reached = (int64_t)h[1];
    g->last.dag_edges = (int64_t)h[2];
    g->last.dist_sum = (int64_t)h[3];
    g->last.fwd_items = (int64_t)h[4];
    g->last.fwd_hits = (int64_t)h[5];
    g->last.bwd_items = (int64_t)h[6];
    g->last.bwd_hits = (int64_t)h[7];
    for (int i = 0; i < MAX_STREAMS; ++i) {
        if (!g->devloop_used[i]) continue;
        const unsigned long long *c = h + 8 + 8 * i;
        g->last.levels_total += (int64_t)c[0];
        g->last.fwd_launches += (int64_t)c[0];
        g->last.bwd_launches += (int64_t)c[0];
        g->last.narrow_batches += (int64_t)c[1];
        g->last.mid_batches += (int64_t)c[2];
        g->last.narrow_fallbacks += (int64_t)(c[2] + c[3]);
        if (c[5]) g->dl_violation = true;
    }
}

// ---- verification capture (bc_set_capture)
// Checks that every captured source is in this call's source set (trav /
// triv, original ids), sizes the buffers and maps the sources to slots in
// the compute CSR's ids.  Runs before the batches are enqueued.
bc_status capture_prepare(bc_graph *g, const int32_t *sources, int64_t num_sources, const std::vector<int> &trav,
                          cudaStream_t st) {
    auto &cp = g->capt;
    const int64_t n = g->n, nc = (int64_t)cp.src.size();
    // 1: in the call's source set, 2: and traversed
    std::vector<uint8_t> in_set((size_t)n, sources ? 0 : 1);
    if (sources)
        for (int64_t i = 0; i < num_sources; ++i) in_set[sources[i]] = 1;
    else if (g->pruned)
        for (int64_t v = 0; v < n; ++v)
            if (g->h_removed[v]) in_set[v] = 0;
    for (int v : trav) in_set[v] = 2;
    for (int s : cp.src)
        if (!in_set[s]) return fail(BC_ERR_INVALID, "captured source %d is not in the source set of this call", s);
    cp.trivial.assign((size_t)nc, 0);
    for (int64_t c = 0; c < nc; ++c) cp.trivial[c] = in_set[cp.src[c]] != 2;
    if (cp.cap < nc || !cp.d_vslot) {
        const int64_t keep_n = nc;
        std::vector<int> keep = cp.src;
        cp.release();
        cp.src = keep;
        CK(dalloc(&cp.d_vslot, (size_t)n));
        CK(dalloc(&cp.d_src, (size_t)keep_n));
        CK(dalloc(&cp.d_tier, (size_t)keep_n));
        CK(dalloc(&cp.d_depth, (size_t)(keep_n * n)));
        CK(dalloc(&cp.d_sigma, (size_t)(keep_n * n)));
        CK(dalloc(&cp.d_delta, (size_t)(keep_n * n)));
        CK(dalloc(&cp.o_depth, (size_t)(keep_n * n)));
        CK(dalloc(&cp.o_sigma, (size_t)(keep_n * n)));
        CK(dalloc(&cp.o_delta, (size_t)(keep_n * n)));
        cp.cap = keep_n;
    }
    std::vector<int> vslot((size_t)n, -1);
    for (int64_t c = 0; c < nc; ++c) vslot[g->run.h_inv[cp.src[c]]] = (int)c;
    CU(cudaMemcpyAsync(cp.d_vslot, vslot.data(), (size_t)n * 4, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(cp.d_src, cp.src.data(), (size_t)nc * 4, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(cp.d_depth, 0xff, (size_t)(nc * n) * 4, st));
    CU(cudaMemsetAsync(cp.d_sigma, 0, (size_t)(nc * n) * 8, st));
    CU(cudaMemsetAsync(cp.d_delta, 0, (size_t)(nc * n) * 8, st));
    CU(cudaMemsetAsync(cp.d_tier, 0, (size_t)nc * 4, st));
    CU(cudaStreamSynchronize(st));  // vslot is pageable host memory
    return BC_OK;
}

// After the batches: compute ids -> original ids, the sources' own entries,
// the removed vertices of a pruned handle, then the copies to the caller's
// host arrays (synchronous at the end of bc_compute).
bc_status capture_finish(bc_graph *g, cudaStream_t st, bool slices) {
    auto &cp = g->capt;
    const int64_t n = g->n, nc = (int64_t)cp.src.size();
    const unsigned blocks = (unsigned)((nc * n + 255) / 256);
    const int *inv = g->run.inv;
    cap_unpermute_kernel<int><<<blocks, 256, 0, st>>>(nc, (int)n, inv, cp.d_depth, cp.o_depth);
    cap_unpermute_kernel<double><<<blocks, 256, 0, st>>>(nc, (int)n, inv, cp.d_sigma, cp.o_sigma);
    cap_unpermute_kernel<double><<<blocks, 256, 0, st>>>(nc, (int)n, inv, cp.d_delta, cp.o_delta);
    cap_sources_kernel<double><<<(unsigned)((nc + 255) / 256), 256, 0, st>>>((int)nc, (int)n, cp.d_src, cp.o_depth,
                                                                          cp.o_sigma);
    if (g->pruned)
        cap_prune_fill_kernel<double><<<blocks, 256, 0, st>>>(nc, (int)n, g->orig.rp, g->orig.col, g->removed, g->omega,
                                                              cp.o_depth, cp.o_sigma, cp.o_delta, nullptr);
    CU(cudaGetLastError());
    if (cp.h_depth) CU(cudaMemcpyAsync(cp.h_depth, cp.o_depth, (size_t)(nc * n) * 4, cudaMemcpyDeviceToHost, st));
    if (cp.h_sigma) CU(cudaMemcpyAsync(cp.h_sigma, cp.o_sigma, (size_t)(nc * n) * 8, cudaMemcpyDeviceToHost, st));
    if (cp.h_delta) CU(cudaMemcpyAsync(cp.h_delta, cp.o_delta, (size_t)(nc * n) * 8, cudaMemcpyDeviceToHost, st));
    if (cp.h_tier) {
        if (slices) {  // one fp64 sigma slot per vertex: the 64-bit tier
            for (int64_t c = 0; c < nc; ++c) cp.h_tier[c] = cp.trivial[c] ? 0 : 64;
        } else {
            CU(cudaMemcpyAsync(cp.h_tier, cp.d_tier, (size_t)nc * 4, cudaMemcpyDeviceToHost, st));
        }
    }
    return BC_OK;
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

__global__ void two_nbr_kernel(const int *cand, int nc, const int *rp, const int *col, int *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nc) {
        const int e = rp[cand[i]];
        out[2 * i] = col[e];
        out[2 * i + 1] = col[e + 1];
    }
}

__global__ void add_kernel(int n, const double *src, double *dst) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) dst[v] += src[v];
}
__global__ void add_stats_kernel(const unsigned long long *src, unsigned long long *dst) {
    if (threadIdx.x < 8) dst[threadIdx.x] += src[threadIdx.x];
}

double sum_events(std::vector<cudaEvent_t> &ev) {
    double tot = 0;
    for (size_t i = 0; i + 1 < ev.size(); i += 2) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, ev[i], ev[i + 1]) == cudaSuccess) tot += ms;
        cudaEventDestroy(ev[i]);
        cudaEventDestroy(ev[i + 1]);
    }
    (void)cudaGetLastError();
    ev.clear();
    return tot;
}

}  // namespace

// =====================================================================
extern "C" {

const char *bc_status_string(bc_status s) {
    switch (s) {
        case BC_OK: return "BC_OK";
        case BC_ERR_INVALID: return "BC_ERR_INVALID";
        case BC_ERR_NOMEM: return "BC_ERR_NOMEM";
        case BC_ERR_CUDA: return "BC_ERR_CUDA";
        case BC_ERR_STATE: return "BC_ERR_STATE";
        case BC_ERR_INTERNAL: return "BC_ERR_INTERNAL";
    }
    return "BC_ERR_UNKNOWN";
}

const char *bc_last_error(void) { return g_err.c_str(); }

bc_status bc_destroy(bc_graph *g) {
    if (!g) return BC_OK;
    {
        DeviceGuard dg(g->device);
        cudaDeviceSynchronize();
        g->orig.release();
        g->res.release();
        dfree(g->omega);
        dfree(g->removed);
        for (auto &x : g->ctx) x.release();
        g->vctx.release();
        g->sctx.release();
        g->sws.release();
        g->capt.release();
        dfree(g->d_stats);
        dfree(g->d_work_ctr);
        dfree(g->d_src);
        dfree(g->td_buf);
        dfree(g->d_bc);
        dfree(g->d_bc2);
        dfree(g->cl_kin);
        dfree(g->cl_kout);
        dfree(g->cl_vout);
        if (g->cl_tmp) cudaFree(g->cl_tmp);
        dfree(g->d_tmp);
        if (g->h_pin) cudaFreeHost(g->h_pin);
        if (g->stats_ev) cudaEventDestroy(g->stats_ev);
        if (g->own_stream) cudaStreamDestroy(g->own_stream);
        if (g->legacy_ev) cudaEventDestroy(g->legacy_ev);
    }
    delete g;
    return BC_OK;
}

// An upper bound on every BFS depth of the graph, for the device-driven
// batches' level slots: in a component with root r, d(s, t) <= d(s, r) +
// d(r, t) <= 2 ecc(r).  Roots are taken in descending degree order (a hub
// is central in a power-law graph, keeping the bound tight).  Host BFS over
// the caller's CSR, O(n + m), once per graph; a pruned graph's residual
// distances between kept vertices are the original ones, so the bound holds
// for it too.
static int depth_bound(int64_t n, const int64_t *rp, const int32_t *col, const std::vector<int> &deg) {
    int maxdeg = 0;
    for (int d : deg) maxdeg = std::max(maxdeg, d);
    std::vector<int64_t> start((size_t)maxdeg + 2, 0);  // counting sort, degree descending
    for (int d : deg) start[(size_t)(maxdeg - d) + 1]++;
    for (size_t i = 1; i < start.size(); ++i) start[i] += start[i - 1];
    std::vector<int> order((size_t)n);
    for (int64_t v = 0; v < n; ++v) order[(size_t)start[(size_t)(maxdeg - deg[v])]++] = (int)v;
    std::vector<int> dist((size_t)n, -1), q((size_t)n);
    int bound = 0;
    for (int r : order) {
        if (dist[r] >= 0) continue;
        size_t h = 0, t = 0;
        q[t++] = r;
        dist[r] = 0;
        int ecc = 0;
        while (h < t) {
            const int v = q[h++];
            ecc = dist[v];
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
                const int w = col[e];
                if (w < 0 || w >= n) return -1;  // malformed CSR (unvalidated): no bound, host-driven loop
                if (dist[w] < 0) {
                    dist[w] = dist[v] + 1;
                    q[t++] = w;
                }
            }
        }
        bound = std::max(bound, 2 * ecc);
    }
    return bound;
}

static bc_status create_impl(bc_graph *g, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                             uint32_t flags) {
    const int64_t nnz = row_ptr[n];
    CU(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
    cudaStream_t st = g->own_stream;
    CU(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device));
    CK(dalloc(&g->d_stats, 16));  // [0, 8) counters, [8, 16) backup across a narrow re-run
    CK(dalloc(&g->d_work_ctr, 4));
    CU(cudaMemset(g->d_work_ctr, 0, 4 * sizeof(int)));
    CK(dalloc(&g->d_bc, (size_t)n));
    // CSR: int64 row_ptr -> int32 on device
    long long *rp64 = nullptr;
    CK(dalloc(&rp64, (size_t)n + 1));
    CU(cudaMemcpy(rp64, row_ptr, ((size_t)n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    CK(dalloc(&g->orig.rp, (size_t)n + 1));
    rp64_to_32_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(rp64, g->orig.rp, n + 1);
    CK(dalloc(&g->orig.col, (size_t)nnz));
    if (nnz > 0)
        CU(cudaMemcpyAsync(g->orig.col, col_idx, (size_t)nnz * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    g->orig.nnz = nnz;
    CU(cudaStreamSynchronize(st));
    dfree(rp64);
    if (flags & BC_CREATE_VALIDATE) {
        int *err = nullptr;
        CK(dalloc(&err, 1));
        CU(cudaMemsetAsync(err, 0, sizeof(int), st));
        validate_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>((int)n, g->orig.rp, g->orig.col, err);
        int herr = 0;
        CU(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        dfree(err);
        if (herr) return fail(BC_ERR_INVALID, "CSR validation failed (flags 0x%x: 2=range 4=self-loop 8=unsorted/dup 16=asymmetric)", herr);
    }
    g->orig.h_deg.resize(n);
    for (int64_t v = 0; v < n; ++v) g->orig.h_deg[v] = (int)(row_ptr[v + 1] - row_ptr[v]);
    g->depth_bound = depth_bound(n, row_ptr, col_idx, g->orig.h_deg);
    CU(cudaMallocHost((void **)&g->h_pin, (8 + 8 * MAX_STREAMS) * sizeof(unsigned long long)));
    CU(cudaEventCreateWithFlags(&g->stats_ev, cudaEventDisableTiming));
    CK(build_layout(g, g->orig, st));
    CK(build_run(g));
    return BC_OK;
}

bc_status bc_graph_create(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, int device, uint32_t flags,
                          bc_graph **out) {
    if (!out) return fail(BC_ERR_INVALID, "out is NULL");
    *out = nullptr;
    if (n <= 0 || n > 2147483647LL) return fail(BC_ERR_INVALID, "n=%lld out of range [1, 2^31-1]", (long long)n);
    if (!row_ptr) return fail(BC_ERR_INVALID, "row_ptr is NULL");
    if (row_ptr[0] != 0) return fail(BC_ERR_INVALID, "row_ptr[0] != 0");
    for (int64_t v = 0; v < n; ++v)
        if (row_ptr[v + 1] < row_ptr[v]) return fail(BC_ERR_INVALID, "row_ptr decreasing at %lld", (long long)v);
    if (row_ptr[n] > 2147483647LL) return fail(BC_ERR_INVALID, "row_ptr[n]=%lld exceeds 2^31-1", (long long)row_ptr[n]);
    if (row_ptr[n] > 0 && !col_idx) return fail(BC_ERR_INVALID, "col_idx is NULL");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        (void)cudaGetLastError();
        return fail(BC_ERR_CUDA, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(BC_ERR_INVALID, "device %d out of range", device);
    bc_graph *g = new (std::nothrow) bc_graph();
    if (!g) return fail(BC_ERR_NOMEM, "host allocation failed");
    g->device = device;
    g->n = n;
    bc_status s;
    {
        DeviceGuard dg(device);
        s = create_impl(g, n, row_ptr, col_idx, flags);
    }
    if (s != BC_OK) {
        std::string keep = g_err;
        bc_destroy(g);
        g_err = keep;
        return s;
    }
    *out = g;
    return BC_OK;
}

// residual CSR from g->omega / g->removed and the residual degrees (device),
// then the compute layout; shared by the single pass and the exchanged shares
static bc_status prune_finish(bc_graph *g, int *rdeg, cudaStream_t st, int64_t *out_removed) {
    const int n = (int)g->n;
    int *tot = nullptr;
    CK(dalloc(&tot, 1));
    const unsigned wblocks = (unsigned)(((int64_t)n * 32 + 255) / 256);
    CK(dalloc(&g->res.rp, (size_t)n + 1));
    CK(dev_scan(g, rdeg, g->res.rp, n, tot, st));
    CU(cudaMemcpyAsync(g->res.rp + n, tot, sizeof(int), cudaMemcpyDeviceToDevice, st));
    int rnnz = 0;
    CU(cudaMemcpyAsync(&rnnz, tot, sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    CK(dalloc(&g->res.col, (size_t)rnnz));
    prune_compact_kernel<<<wblocks, 256, 0, st>>>(n, g->orig.rp, g->orig.col, g->removed, g->res.rp, g->res.col);
    CU(cudaGetLastError());
    g->res.nnz = rnnz;
    g->h_omega.resize(n);
    g->h_removed.resize(n);
    std::vector<int> rd(n);
    CU(cudaMemcpyAsync(g->h_omega.data(), g->omega, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(g->h_removed.data(), g->removed, (size_t)n, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(rd.data(), rdeg, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    g->res.h_deg = rd;
    dfree(tot);
    g->pruned = true;
    CK(build_layout(g, g->res, st));  // bc_sssp traverses the residual graph in caller ids
    CK(build_run(g));
    if (out_removed) {
        int64_t r = 0;
        for (int v = 0; v < n; ++v) r += g->h_removed[v];
        *out_removed = r;
    }
    return BC_OK;
}

bc_status bc_prune_degree1(bc_graph *g, int64_t *out_removed) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    if (g->pruned) return fail(BC_ERR_STATE, "graph already pruned (single pass, PAPER.md:580)");
    DeviceGuard dg(g->device);
    CK(wait_idle(g));
    cudaStream_t st = g->own_stream;
    const int n = (int)g->n;
    CK(dalloc(&g->omega, n));
    CK(dalloc(&g->removed, n));
    int *rdeg = nullptr;
    CK(dalloc(&rdeg, n));
    const unsigned wblocks = (unsigned)(((int64_t)n * 32 + 255) / 256);
    prune_count_kernel<<<wblocks, 256, 0, st>>>(n, g->orig.rp, g->orig.col, g->omega, g->removed, rdeg);
    const bc_status rc = prune_finish(g, rdeg, st, out_removed);
    dfree(rdeg);
    return rc;
}

bc_status bc_prune_degree1_share(const bc_graph *g, int rank, int nranks, uint32_t *omega_part,
                                 uint32_t *removed_part, void *cuda_stream) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    if (g->pruned) return fail(BC_ERR_STATE, "graph already pruned (single pass, PAPER.md:580)");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(BC_ERR_INVALID, "rank %d of %d out of range", rank, nranks);
    if (!omega_part || !removed_part) return fail(BC_ERR_INVALID, "NULL output");
    DeviceGuard dg(g->device);
    if (!is_device_ptr(omega_part) || !is_device_ptr(removed_part))
        return fail(BC_ERR_INVALID, "share outputs must be device memory");
    // reads only the original CSR, which no call modifies; with no caller stream
    // the outputs may still be in use by work on the legacy default stream (the
    // library stream does not synchronise with it): wait for the device first
    if (!cuda_stream) CU(cudaDeviceSynchronize());
    cudaStream_t st = cuda_stream ? (cudaStream_t)cuda_stream : g->own_stream;
    const int n = (int)g->n;
    CU(cudaMemsetAsync(omega_part, 0, (size_t)n * 4, st));
    CU(cudaMemsetAsync(removed_part, 0, (size_t)n * 4, st));
    const long long mine = ((long long)n - rank + nranks - 1) / nranks;  // vertices u = rank, rank + nranks, ...
    if (mine > 0)
        prune_share_kernel<<<(unsigned)((mine + 255) / 256), 256, 0, st>>>(n, g->orig.rp, g->orig.col, rank, nranks,
                                                                            omega_part, removed_part);
    CU(cudaGetLastError());
    if (!cuda_stream) CU(cudaStreamSynchronize(st));
    return BC_OK;
}

bc_status bc_prune_degree1_apply(bc_graph *g, const uint32_t *omega, const uint32_t *removed, void *cuda_stream,
                                 int64_t *out_removed) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    if (g->pruned) return fail(BC_ERR_STATE, "graph already pruned (single pass, PAPER.md:580)");
    if (!omega || !removed) return fail(BC_ERR_INVALID, "NULL input");
    DeviceGuard dg(g->device);
    if (!is_device_ptr(omega) || !is_device_ptr(removed)) return fail(BC_ERR_INVALID, "inputs must be device memory");
    CK(wait_idle(g));
    // the exchange that produced the inputs: its stream, or -- none given --
    // every prior device work (the inputs may come from the legacy default
    // stream, which the library's non-blocking stream does not wait for)
    if (cuda_stream) CU(cudaStreamSynchronize((cudaStream_t)cuda_stream));
    else CU(cudaDeviceSynchronize());
    cudaStream_t st = g->own_stream;
    const int n = (int)g->n;
    uint8_t *rm = nullptr;
    uint32_t *om = nullptr;
    int *rdeg = nullptr, *err = nullptr;
    CK(dalloc(&rm, n));
    CK(dalloc(&om, n));
    CK(dalloc(&rdeg, n));
    CK(dalloc(&err, 1));
    CU(cudaMemsetAsync(err, 0, sizeof(int), st));
    CU(cudaMemcpyAsync(om, omega, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    const unsigned wblocks = (unsigned)(((int64_t)n * 32 + 255) / 256);
    prune_flags_kernel<<<wblocks, 256, 0, st>>>(n, g->orig.rp, g->orig.col, removed, rm, rdeg, err);
    int herr = 0;
    CU(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    dfree(err);
    if (herr) {
        dfree(rm);
        dfree(om);
        dfree(rdeg);
        return fail(BC_ERR_INVALID, "removed flags are not the sum of all shares (a vertex is removed iff its degree is 1)");
    }
    g->omega = om;
    g->removed = rm;
    const bc_status rc = prune_finish(g, rdeg, st, out_removed);
    dfree(rdeg);
    return rc;
}

bc_status bc_set_option(bc_graph *g, int option, int64_t value) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    switch (option) {
        case BC_OPT_LANE_WORDS:
            if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8)
                return fail(BC_ERR_INVALID, "lane words must be 0, 1, 2, 4 or 8");
            g->lane_words_opt = (int)value;
            return BC_OK;
        case BC_OPT_HUB_DEGREE: {
            if (value < 32 || value > (1 << 30)) return fail(BC_ERR_INVALID, "hub degree out of range");
            if (g->hub_deg == (int)value) return BC_OK;
            DeviceGuard dg(g->device);
            CK(wait_idle(g));
            g->hub_deg = (int)value;
            CK(build_layout(g, g->orig, g->own_stream));
            if (g->pruned) CK(build_layout(g, g->res, g->own_stream));
            CK(build_run(g));
            return BC_OK;
        }
        case BC_OPT_FWD_PUSH:
            if (value < 0 || value > 1000) return fail(BC_ERR_INVALID, "fwd push levels out of range");
            g->fwd_push_levels = (int)value;
            return BC_OK;
        case BC_OPT_BWD_MODE:
            if (value < 0 || value > 2) return fail(BC_ERR_INVALID, "backward mode must be 0, 1 or 2");
            g->bwd_mode = (int)value;
            return BC_OK;
        case BC_OPT_SIGMA_WIDTH:
            if (value != 0 && value != 16 && value != 64) return fail(BC_ERR_INVALID, "sigma width must be 0, 16 or 64");
            g->sigma_width = (int)value;
            return BC_OK;
        case BC_OPT_TWO_DEGREE:
            if (value != 0 && value != 1) return fail(BC_ERR_INVALID, "two-degree must be 0 or 1");
            g->two_degree = (int)value;
            return BC_OK;
        case BC_OPT_STREAMS:
            if (value < 0 || value > MAX_STREAMS) return fail(BC_ERR_INVALID, "streams must be 0 (auto) .. %d", MAX_STREAMS);
            g->streams_opt = (int)value;
            return BC_OK;
        case BC_OPT_SOURCE_ORDER:
            if (value < 0 || value > 3) return fail(BC_ERR_INVALID, "source order must be 0..3");
            g->src_order = (int)value;
            return BC_OK;
        case BC_OPT_RELABEL: {
            if (value < 0 || value > 2) return fail(BC_ERR_INVALID, "relabel must be 0, 1 or 2");
            const int v = (int)value;
            if (v == g->relabel) return BC_OK;
            DeviceGuard dg(g->device);
            CK(wait_idle(g));
            g->relabel = v;
            CK(build_run(g));
            return BC_OK;
        }
        case BC_OPT_PROFILE:
            g->profile = value ? 1 : 0;
            return BC_OK;
        case BC_OPT_MODE:
            if (value < 0 || value > 2) return fail(BC_ERR_INVALID, "mode must be 0, 1 or 2");
            g->mode = (int)value;
            return BC_OK;
        case BC_OPT_SLICES_KERNEL:
            if (value < 0 || value > 4) return fail(BC_ERR_INVALID, "slices kernel must be 0..4");
            g->slices_kernel = (int)value;
            return BC_OK;
        case BC_OPT_DEVICE_LOOP:
            if (value < 0 || value > 2) return fail(BC_ERR_INVALID, "device loop must be 0, 1 or 2");
            g->device_loop = (int)value;
            return BC_OK;
    }
    return fail(BC_ERR_INVALID, "unknown option %d", option);
}

bc_status bc_set_capture(bc_graph *g, const int32_t *sources, int64_t n_cap, int32_t *depth, double *sigma,
                         double *delta, int32_t *tier) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    if (n_cap < 0 || n_cap > BC_CAPTURE_MAX) return fail(BC_ERR_INVALID, "n_cap=%lld out of range [0, %d]", (long long)n_cap, BC_CAPTURE_MAX);
    g->capt.src.clear();
    if (n_cap == 0) return BC_OK;
    if (!sources) return fail(BC_ERR_INVALID, "sources is NULL");
    std::vector<int> src((size_t)n_cap);
    for (int64_t i = 0; i < n_cap; ++i) {
        const int s = sources[i];
        if (s < 0 || s >= g->n) return fail(BC_ERR_INVALID, "captured source %d out of range", s);
        for (int64_t j = 0; j < i; ++j)
            if (src[j] == s) return fail(BC_ERR_INVALID, "duplicate captured source %d", s);
        src[i] = s;
    }
    g->capt.src = src;
    g->capt.h_depth = depth;
    g->capt.h_sigma = sigma;
    g->capt.h_delta = delta;
    g->capt.h_tier = tier;
    return BC_OK;
}

bc_status bc_get_stats(const bc_graph *cg, bc_stats *out) {
    if (!cg || !out) return fail(BC_ERR_INVALID, "NULL argument");
    bc_graph *g = const_cast<bc_graph *>(cg);
    if (g->stats_pending) {  // asynchronous bc_compute: its counters land when its stream gets there
        DeviceGuard dg(g->device);
        CU(cudaEventSynchronize(g->stats_ev));
        finalize_stats(g);
        g->stats_pending = false;
    }
    *out = g->last;
    if (g->dl_violation) return fail(BC_ERR_INTERNAL, "a BFS exceeded the graph's depth bound (%d levels)", g->depth_bound);
    return BC_OK;
}

bc_status bc_graph_info(const bc_graph *g, int64_t *n, int64_t *nnz, int64_t *res_nnz, int *device) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    if (n) *n = g->n;
    if (nnz) *nnz = g->orig.nnz;
    if (res_nnz) *res_nnz = g->pruned ? g->res.nnz : g->orig.nnz;
    if (device) *device = g->device;
    return BC_OK;
}

bc_status bc_get_pruning(const bc_graph *g, uint32_t *omega, uint8_t *removed, int64_t *res_row_ptr,
                         int32_t *res_col, int64_t *res_nnz) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    if (!g->pruned) return fail(BC_ERR_STATE, "graph is not pruned");
    DeviceGuard dg(g->device);
    const int64_t n = g->n;
    if (omega) memcpy(omega, g->h_omega.data(), (size_t)n * 4);
    if (removed) memcpy(removed, g->h_removed.data(), (size_t)n);
    if (res_row_ptr) {
        std::vector<int> rp(n + 1);
        CU(cudaMemcpy(rp.data(), g->res.rp, (size_t)(n + 1) * 4, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i <= n; ++i) res_row_ptr[i] = rp[i];
    }
    if (res_col && g->res.nnz > 0)
        CU(cudaMemcpy(res_col, g->res.col, (size_t)g->res.nnz * 4, cudaMemcpyDeviceToHost));
    if (res_nnz) *res_nnz = g->res.nnz;
    return BC_OK;
}

bc_status bc_compute(bc_graph *g, const int32_t *sources, int64_t num_sources, double *out_bc, void *cuda_stream) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    const double tr0 = trace_on() ? now_us() : 0.0;
    double tr_plan = 0, tr_join = 0;
    // a capture (bc_set_capture) applies to this call only, success or not
    const bool capture = !g->capt.src.empty();
    struct CaptureReset {
        bc_graph *g;
        ~CaptureReset() {
            g->capt.src.clear();
            g->capt.h_depth = g->capt.h_tier = nullptr;
            g->capt.h_sigma = g->capt.h_delta = nullptr;
        }
    } capture_reset{g};
    if (!out_bc) return fail(BC_ERR_INVALID, "out_bc is NULL");
    if (num_sources < 0 || (num_sources > 0 && !sources)) return fail(BC_ERR_INVALID, "bad source list");
    DeviceGuard dg(g->device);
    const int64_t n = g->n;
    DevCSR &csr = g->cur();
    // an asynchronous previous call (possibly on another stream) still owns
    // the handle's buffers until its stream reaches stats_ev
    if (g->stats_ev) {
        cudaStream_t st0 = cuda_stream ? (cudaStream_t)cuda_stream : g->own_stream;
        CU(cudaStreamWaitEvent(st0, g->stats_ev, 0));
    }
    // ---- resolve and validate the source set (host-side argument checks)
    std::vector<int> trav, triv;
    if (!sources) {
        for (int64_t v = 0; v < n; ++v) {
            if (g->pruned && g->h_removed[v]) continue;
            if (csr.h_deg[v] > 0) trav.push_back((int)v);
            else if (g->pruned && g->h_omega[v] > 0) triv.push_back((int)v);
        }
    } else {
        std::vector<uint8_t> mark((size_t)n, 0);
        for (int64_t i = 0; i < num_sources; ++i) {
            const int s = sources[i];
            if (s < 0 || s >= n) return fail(BC_ERR_INVALID, "source %d out of range", s);
            if (mark[s]) return fail(BC_ERR_INVALID, "duplicate source %d", s);
            mark[s] = 1;
            if (g->pruned && g->h_removed[s]) return fail(BC_ERR_INVALID, "source %d was removed by 1-degree pruning", s);
            if (csr.h_deg[s] > 0) trav.push_back(s);
            else if (g->pruned && g->h_omega[s] > 0) triv.push_back(s);
        }
    }
    double tr_m[4] = {0, 0, 0, 0};  // BC_TRACE marks: sources resolved, W / pipelines chosen, plan + clustering
    if (trace_on()) tr_m[0] = now_us();
    const bool dev_out = is_device_ptr(out_bc);
    cudaStream_t st = cuda_stream ? (cudaStream_t)cuda_stream : g->own_stream;
    if (!cuda_stream && dev_out) {
        // no caller stream: a device out_bc may still be in use by work on the
        // legacy default stream, which the library's non-blocking stream does
        // not wait for -- order after it
        if (!g->legacy_ev) CU(cudaEventCreateWithFlags(&g->legacy_ev, cudaEventDisableTiming));
        CU(cudaEventRecord(g->legacy_ev, cudaStreamLegacy));
        CU(cudaStreamWaitEvent(st, g->legacy_ev, 0));
    }
    if (!g->run_valid) CK(build_run(g));
    DevCSR &run = g->run;
    if (capture) CK(capture_prepare(g, sources, num_sources, trav, st));
    // batch schedule: compute ids, ascending = degree descending (sources with
    // similar BFS depth profiles share a batch and sit in adjacent lanes)
    for (auto &v : trav) v = run.h_inv[v];
    for (auto &v : triv) v = run.h_inv[v];
    if (g->src_order >= 1) std::stable_sort(trav.begin(), trav.end());
    g->last = bc_stats{};
    g->stats_pending = false;
    g->dl_violation = false;
    g->last.num_sources = (int64_t)trav.size();
    g->last.num_trivial = (int64_t)triv.size();
    // batch mode: bit lanes (low diameter) or one source per CTA (long
    // diameter); auto picks slices for large sparse graphs (mean degree < 6)
    int mode = g->mode;
    if (mode == 0) mode = auto_slices(g->n, run.nnz) ? 2 : 1;
    // ---- lane width W (K = 64 W lanes per batch), level-row width rb, batch
    // pipelines NS and the device-driven batch (graph mode).
    // Rows cost n*64*W*rb bytes per BFS level, the accumulators n*512*W, the
    // level masks n*8*W per level; each pipeline holds its own.  Host-driven
    // batches allocate levels on demand (~11 at R-MAT depths) with 4-byte rows
    // (the 16- and 32-bit sigma tiers; a batch needing fp64 widens them).
    // Device-driven batches preallocate levels 0 .. depth_bound + 1 and use
    // 8-byte rows when they fit (the fp64 tier then runs in the graph too).
    // Measured (prof_batch): S12 1/4/8 pipelines 21.5/6.2/4.0 ms, S16
    // 352/114/110 ms, S20 332/316 (3)/332 (4) ms (host-driven).
    const int lcap = g->depth_bound;
    const bool dl_opts = g->device_loop && mode == 1 && !g->two_degree && g->bwd_mode != 2 &&
                         g->fwd_push_levels == 0 && !g->profile && g->sigma_width != 64 && g->hub_deg <= 65536 &&
                         lcap >= 1 && lcap <= BC_DEVLOOP_MAX_LEVELS;
    const int64_t skey[8] = {(int64_t)trav.size(), mode, dl_opts, g->lane_words_opt, g->streams_opt,
                             g->sigma_width + 1000 * g->bwd_mode + 100000 * g->fwd_push_levels, lcap, g->n};
    int W, NS, rb;
    bool devloop;
    if (std::equal(skey, skey + 8, g->sizing.key)) {
        W = g->sizing.W;
        NS = g->sizing.NS;
        rb = g->sizing.rb;
        devloop = g->sizing.devloop;
    } else {
        rb = g->sigma_width == 64 || g->bwd_mode == 2 || g->fwd_push_levels > 0 ? 8 : 4;
        W = g->lane_words_opt;
        if (W == 0) {
            W = trav.size() > 128 ? 4 : (trav.size() > 64 ? 2 : 1);
            // K = 512 halves the items per source again but doubles the lanes a
            // thread carries: faster only where per-batch overhead dominates
            // (S16: 74 -> 60 ms per 16384 sources; S20: 319 -> 362 ms)
            if (trav.size() > 256 && g->n <= (1 << 18)) W = 8;
        }
        const int ns_auto = g->n <= (1 << 18) ? 8 : 3;
        NS = mode == 1 ? (g->streams_opt > 0 ? g->streams_opt : ns_auto) : 1;
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
            (void)cudaGetLastError();
            free_b = 0;
        }
        for (auto &x : g->ctx)  // reusable
            free_b += (size_t)x.ws.slev.size() * (size_t)g->n * 64 * (size_t)x.ws.W * (size_t)x.ws.row_bytes +
                      (x.ws.A ? (size_t)g->n * 512 * (size_t)x.ws.W : 0);
        const double budget = 0.6 * (double)free_b;
        auto bytes = [&](int w, int r, int levels) {
            return (double)g->n * 64.0 * w * (levels * (double)r + 8.0) + (double)g->n * 8.0 * w * ((levels + 7) / 8 * 8);
        };
        devloop = false;
        if (dl_opts) {
            // device-driven: keep the lane width; 8-byte rows if NS pipelines fit, else 4-byte rows
            const int lv = lcap + 2;
            for (int r : {8, 4}) {
                if (r == 8 && g->device_loop == 2) continue;  // 4-byte rows forced (tests the host fp64 re-run)
                int ns = NS;
                while (ns > 1 && ns * bytes(W, r, lv) > budget) --ns;
                if (bytes(W, r, lv) <= budget) {
                    devloop = true;
                    rb = r;
                    NS = ns;
                    break;
                }
            }
        }
        if (!devloop) {
            if (g->lane_words_opt == 0)  // keep ~9 levels plus the accumulators within budget (S23: W = 4)
                while (W > 1 && bytes(W, rb, 9) > budget) W >>= 1;
            while (NS > 1 && NS * bytes(W, rb, 11) > budget) --NS;
        }
        std::copy(skey, skey + 8, g->sizing.key);
        g->sizing.W = W;
        g->sizing.NS = NS;
        g->sizing.rb = rb;
        g->sizing.devloop = devloop;
    }
    const int K = 64 * W;
    g->last.lanes = K;
    if (trace_on()) tr_m[1] = now_us();
    const int64_t need = (int64_t)(trav.size() + triv.size());
    if (g->src_cap < need) {
        dfree(g->d_src);
        CK(dalloc(&g->d_src, (size_t)need));
        g->src_cap = need;
    }
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (g->profile) {
        cudaEventCreate(&t0);
        cudaEventCreate(&t1);
        cudaEventRecord(t0, st);
    }
    // batch plan: consecutive K-lane slices of the (clustered) source list, or
    // with the 2-degree heuristic an explicit lane layout per batch
    struct Plan {
        int64_t off;
        int nl;
        bool layout;
        uint64_t active[8], derived[8];
    };
    std::vector<Plan> plan;
    int64_t nlanes = (int64_t)trav.size();  // entries of d_src used by the batches
    if (mode == 1 && g->two_degree && !trav.empty()) {
        CK(plan_two_degree(g, run, trav, K, W, st, g->last));
        nlanes = (int64_t)g->td_lanes.size();
        for (auto &b : g->td_plan) {
            Plan q{};
            q.off = b.off;
            q.nl = b.nl;
            q.layout = true;
            for (int j = 0; j < 8; ++j) {
                q.active[j] = b.active[j];
                q.derived[j] = b.derived[j];
            }
            plan.push_back(q);
        }
    } else if (!trav.empty()) {
        CU(cudaMemcpyAsync(g->d_src, trav.data(), trav.size() * 4, cudaMemcpyHostToDevice, st));
        if (mode == 1 && g->src_order >= 2 && trav.size() > (size_t)K) CK(cluster_sources(g, run, (int)trav.size(), st));
        for (size_t off = 0; mode == 1 && off < trav.size(); off += K) {
            Plan q{};
            q.off = (int64_t)off;
            q.nl = (int)std::min<size_t>(K, trav.size() - off);
            plan.push_back(q);
        }
    }
    if (!triv.empty()) {
        if (g->src_cap < nlanes + (int64_t)triv.size()) {
            // grow, keeping the batch lanes (stream-ordered copy through a new buffer)
            int *nbuf = nullptr;
            CK(dalloc(&nbuf, (size_t)(nlanes + (int64_t)triv.size())));
            if (nlanes) CU(cudaMemcpyAsync(nbuf, g->d_src, (size_t)nlanes * 4, cudaMemcpyDeviceToDevice, st));
            CU(cudaStreamSynchronize(st));
            dfree(g->d_src);
            g->d_src = nbuf;
            g->src_cap = nlanes + (int64_t)triv.size();
        }
        CU(cudaMemcpyAsync(g->d_src + nlanes, triv.data(), triv.size() * 4, cudaMemcpyHostToDevice, st));
    }
    if (trace_on()) tr_m[2] = now_us();
    CU(cudaMemsetAsync(g->d_bc, 0, (size_t)n * 8, st));
    CU(cudaMemsetAsync(g->d_stats, 0, 8 * sizeof(unsigned long long), st));
    if (trace_on()) tr_plan = now_us();
    std::vector<cudaEvent_t> ef;
    if (mode == 2 && !trav.empty())
        CK(run_slices(g, run, g->d_src, (int)trav.size(), st, g->profile ? &ef : nullptr, capture));
    for (auto &u : g->devloop_used) u = false;
    if (mode == 1 && !trav.empty() && devloop && !plan.empty() && !plan[0].layout) {
        // ---- device-driven batches: one CUDA graph launch per batch, no host
        // round trip inside a batch (enqueue_device_batch)
        NS = std::max(1, std::min(NS, (int)plan.size()));
        g->conc = NS > 1;
        cudaEvent_t start = nullptr;
        CU(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
        CU(cudaEventRecord(start, st));
        DevBatchCfg cfg{};
        cfg.csr = &run;
        cfg.omega = g->pruned ? run.omega : nullptr;
        cfg.lcap = lcap;
        cfg.fp64_inline = rb >= 8;
        cfg.capture = capture;
        bc_status r = BC_OK;
        for (int i = 0; i < NS && r == BC_OK; ++i) {
            LaneCtx &x = g->ctx[i];
            auto body = [&]() -> bc_status {
                CK(ctx_init(g, x));
                CK(ensure_ws(g, x.ws, W, false, std::max(run.nhub, g->orig.nhub), rb));
                CK(ensure_level(g, x.ws, lcap + 1));
                CK(ensure_flags(g, x, lcap + 3));
                std::vector<int2> tab;
                for (size_t bi = (size_t)i; bi < plan.size(); bi += (size_t)NS)
                    tab.push_back(make_int2((int)plan[bi].off, plan[bi].nl));
                CK(ensure_device_batch(g, x, (int)tab.size()));
                x.last = bc_stats{};
                x.st = x.own;
                cudaStream_t xs = x.st;
                CU(cudaStreamWaitEvent(xs, start, 0));
                CU(cudaMemcpyAsync(x.gb_table, tab.data(), tab.size() * sizeof(int2), cudaMemcpyHostToDevice, xs));
                CU(cudaMemsetAsync(x.gb_ctl, 0, 8 * sizeof(int), xs));
                CU(cudaMemsetAsync(x.gb_cnt, 0, 8 * sizeof(unsigned long long), xs));
                CU(cudaMemsetAsync(x.d_stats, 0, 8 * sizeof(unsigned long long), xs));
                if (i == 0) {
                    x.d_bc = g->d_bc;
                } else {
                    if (!x.own_bc) CK(dalloc(&x.own_bc, (size_t)n));
                    x.d_bc = x.own_bc;
                    CU(cudaMemsetAsync(x.d_bc, 0, (size_t)n * 8, xs));
                }
                CK(device_batch_graph(g, x, W, cfg));
                for (size_t b = 0; b < tab.size(); ++b) CU(cudaGraphLaunch(x.gexec, xs));
                x.last.batches = (int64_t)tab.size();
                g->devloop_used[i] = true;
                return BC_OK;
            };
            r = body();
        }
        cudaEventDestroy(start);
        if (r != BC_OK) {
            if (r == BC_ERR_NOMEM) g->sizing.key[0] = -1;  // re-size on the next call
            return r;
        }
        if (!cfg.fp64_inline) {
            // 4-byte rows: batches whose 32-bit sigma overflowed (sigma >= 2^32,
            // never on R-MAT) re-run on the host-driven fp64 path
            for (int i = 0; i < NS; ++i) CU(cudaMemcpyAsync(g->h_pin + 8 + 8 * i, g->ctx[i].gb_cnt, 64, cudaMemcpyDeviceToHost, g->ctx[i].st));
            for (int i = 0; i < NS; ++i) CU(cudaStreamSynchronize(g->ctx[i].st));
            for (int i = 0; i < NS; ++i) {
                LaneCtx &x = g->ctx[i];
                const int nredo = (int)g->h_pin[8 + 8 * i + 4];
                if (!nredo) continue;
                std::vector<int> redo(nredo);
                CU(cudaMemcpy(redo.data(), x.gb_redo, (size_t)nredo * 4, cudaMemcpyDeviceToHost));
                for (int b : redo) {
                    const Plan &pb = plan[(size_t)i + (size_t)b * NS];
                    BatchCtx c{};
                    c.csr = &run;
                    c.omega = g->pruned ? run.omega : nullptr;
                    c.src = g->d_src + pb.off;
                    c.nl = pb.nl;
                    c.st = x.st;
                    c.run_backward = true;
                    c.endpoint = true;
                    if (capture) {
                        c.cap_vslot = g->capt.d_vslot;
                        c.cap_depth = g->capt.d_depth;
                        c.cap_sigma = g->capt.d_sigma;
                        c.cap_delta = g->capt.d_delta;
                        c.cap_tier = g->capt.d_tier;
                    }
                    CK(widen_rows(g, x.ws));
                    CK(run_batch_w<double>(g, x, W, c, nullptr, nullptr));
                }
            }
        }
        for (int i = 0; i < NS; ++i) {
            LaneCtx &x = g->ctx[i];
            CU(cudaEventRecord(x.done, x.st));
            CU(cudaStreamWaitEvent(st, x.done, 0));
            if (i > 0) {
                add_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((int)n, x.d_bc, g->d_bc);
                g->last.kernel_launches += 1;
            }
            add_stats_kernel<<<1, 32, 0, st>>>(x.d_stats, g->d_stats);
            CU(cudaMemcpyAsync(g->h_pin + 8 + 8 * i, x.gb_cnt, 64, cudaMemcpyDeviceToHost, st));
            g->last.batches += x.last.batches;
            g->last.levels_total += x.last.levels_total;  // host fp64 re-runs
            g->last.kernel_launches += x.last.kernel_launches + (int64_t)x.gnodes * x.last.batches;
        }
    } else if (mode == 1 && !trav.empty()) {
        NS = std::max(1, std::min(NS, (int)plan.size()));
        g->conc = NS > 1;
        for (int i = 0; i < NS; ++i) {
            CK(ctx_init(g, g->ctx[i]));
            CK(ensure_ws(g, g->ctx[i].ws, W, false, std::max(run.nhub, g->orig.nhub), rb));
        }
        // pipeline i runs batches i, i + NS, ...; pipeline 0 adds into d_bc,
        // the others into private partials summed at the end
        cudaEvent_t start = nullptr;
        if (NS > 1) {
            CU(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
            CU(cudaEventRecord(start, st));
        }
        bc_status sts[MAX_STREAMS];
        std::string msgs[MAX_STREAMS];
        auto worker = [&](int i) {
            LaneCtx &x = g->ctx[i];
            DeviceGuard dgw(g->device);
            x.last = bc_stats{};
            x.st = NS > 1 ? x.own : st;
            bc_status r = BC_OK;
            auto body = [&]() -> bc_status {
                cudaStream_t xs = x.st;
                if (NS > 1) CU(cudaStreamWaitEvent(xs, start, 0));
                CU(cudaMemsetAsync(x.d_stats, 0, 8 * sizeof(unsigned long long), xs));
                if (i == 0) {
                    x.d_bc = g->d_bc;
                } else {
                    if (!x.own_bc) CK(dalloc(&x.own_bc, (size_t)n));
                    x.d_bc = x.own_bc;
                    CU(cudaMemsetAsync(x.d_bc, 0, (size_t)n * 8, xs));
                }
                for (size_t bi = (size_t)i; bi < plan.size(); bi += (size_t)NS) {
                    const Plan &pb = plan[bi];
                    BatchCtx c{};
                    c.csr = &run;
                    c.omega = g->pruned ? run.omega : nullptr;
                    c.src = g->d_src + pb.off;
                    c.nl = pb.nl;
                    c.layout = pb.layout;
                    for (int j = 0; j < 8; ++j) {
                        c.active[j] = pb.active[j];
                        c.derived[j] = pb.derived[j];
                    }
                    c.st = xs;
                    c.run_backward = true;
                    c.endpoint = true;
                    if (capture) {
                        c.cap_vslot = g->capt.d_vslot;
                        c.cap_depth = g->capt.d_depth;
                        c.cap_sigma = g->capt.d_sigma;
                        c.cap_delta = g->capt.d_delta;
                        c.cap_tier = g->capt.d_tier;
                    }
                    x.last.batches += 1;
                    // narrow sigma first (16-bit rows, exact integers); a batch whose sigma
                    // overflows is re-run with fp64 rows from scratch (nothing of it was
                    // committed: BC is only touched by the backward sweep)
                    const bool narrow =
                        g->sigma_width != 64 && g->hub_deg <= 65536 && g->bwd_mode != 2 && g->fwd_push_levels == 0;
                    auto *pef = g->profile ? &x.ef : nullptr;
                    auto *peb = g->profile ? &x.eb : nullptr;
                    if (narrow) {
                        // 16-bit rows (widened in place to 32-bit rows at the
                        // level that overflows), else the whole batch again with
                        // 32-bit rows, then fp64
                        bool failed = false, widened = false, need64 = false;
                        c.narrow_failed = &failed;
                        c.widened = &widened;
                        c.need_fp64 = &need64;
                        const int64_t lv = x.last.levels_total;
                        CU(cudaMemcpyAsync(x.d_stats + 8, x.d_stats, 8 * sizeof(unsigned long long),
                                           cudaMemcpyDeviceToDevice, xs));
                        CK(run_batch_w<unsigned>(g, x, W, c, pef, peb));
                        c.widened = nullptr;
                        c.need_fp64 = nullptr;
                        if (!failed) {
                            if (widened) x.last.widened_batches += 1;
                            else x.last.narrow_batches += 1;
                            continue;
                        }
                        CU(cudaMemcpyAsync(x.d_stats, x.d_stats + 8, 8 * sizeof(unsigned long long),
                                           cudaMemcpyDeviceToDevice, xs));
                        x.last.levels_total = lv;
                        x.last.narrow_fallbacks += 1;
                        failed = false;
                        if (!need64) {
                            CK(run_batch_w<long long>(g, x, W, c, pef, peb));
                            if (!failed) {
                                x.last.mid_batches += 1;
                                continue;
                            }
                        }
                        CU(cudaMemcpyAsync(x.d_stats, x.d_stats + 8, 8 * sizeof(unsigned long long),
                                           cudaMemcpyDeviceToDevice, xs));
                        x.last.levels_total = lv;
                        c.narrow_failed = nullptr;
                    }
                    CK(widen_rows(g, x.ws));
                    CK(run_batch_w<double>(g, x, W, c, pef, peb));
                }
                CU(cudaEventRecord(x.done, xs));
                return BC_OK;
            };
            r = body();
            sts[i] = r;
            if (r != BC_OK) msgs[i] = bc_last_error();
        };
        if (NS == 1) {
            worker(0);
        } else {
            std::vector<std::thread> th;
            try {
                for (int i = 0; i < NS; ++i) th.emplace_back(worker, i);
            } catch (...) {  // no exception may cross the C ABI
                for (auto &t : th) t.join();
                if (start) cudaEventDestroy(start);
                return fail(BC_ERR_INTERNAL, "cannot start %d pipeline threads", NS);
            }
            for (auto &t : th) t.join();
        }
        if (start) cudaEventDestroy(start);
        if (trace_on()) tr_join = now_us();
        for (int i = 0; i < NS; ++i)
            if (sts[i] != BC_OK) {
                if (sts[i] == BC_ERR_NOMEM) g->sizing.key[0] = -1;  // re-size on the next call
                return fail(sts[i], "%s", msgs[i].c_str());
            }
        for (int i = 0; i < NS; ++i) {
            LaneCtx &x = g->ctx[i];
            if (NS > 1) CU(cudaStreamWaitEvent(st, x.done, 0));
            if (i > 0) {
                add_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((int)n, x.d_bc, g->d_bc);
                g->last.kernel_launches += 1;
            }
            add_stats_kernel<<<1, 32, 0, st>>>(x.d_stats, g->d_stats);
            g->last.batches += x.last.batches;
            g->last.levels_total += x.last.levels_total;
            g->last.fwd_launches += x.last.fwd_launches;
            g->last.bwd_launches += x.last.bwd_launches;
            g->last.kernel_launches += x.last.kernel_launches;
            g->last.narrow_batches += x.last.narrow_batches;
            g->last.narrow_fallbacks += x.last.narrow_fallbacks;
            g->last.mid_batches += x.last.mid_batches;
            g->last.widened_batches += x.last.widened_batches;
        }
    }
    if (!triv.empty()) {
        trivial_sources_kernel<<<(unsigned)((triv.size() + 255) / 256), 256, 0, st>>>(
            g->d_src + nlanes, (int)triv.size(), run.omega, g->d_bc);
        g->last.kernel_launches += 1;
    }
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(g->h_pin, g->d_stats, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (dev_out) {
        unpermute_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((int)n, run.inv, g->d_bc, out_bc);
    } else {
        if (!g->d_bc2) CK(dalloc(&g->d_bc2, (size_t)n));
        unpermute_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((int)n, run.inv, g->d_bc, g->d_bc2);
        CU(cudaMemcpyAsync(out_bc, g->d_bc2, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    }
    g->last.kernel_launches += 1;
    if (capture) CK(capture_finish(g, st, mode == 2));
    if (g->profile) cudaEventRecord(t1, st);
    bool any_dl = false;
    for (bool u : g->devloop_used) any_dl |= u;
    // Stream-ordered and asynchronous when every batch ran device-driven and
    // the output is on the device: the call returns once the work is
    // enqueued (the counters land in pinned memory; bc_get_stats waits for
    // them).  Otherwise the call has already waited (host-driven level loop,
    // host output, capture, profiling) and completes here.
    const bool device_driven = mode == 2 || any_dl;  // slices mode: one persistent launch, no host round trip
    // (no caller stream to order on: the library's own stream is waited for)
    const bool sync = !dev_out || !cuda_stream || capture || g->profile || trace_on() || !device_driven;
    CU(cudaEventRecord(g->stats_ev, st));
    if (!sync) {
        g->stats_pending = true;
        return BC_OK;
    }
    CU(cudaStreamSynchronize(st));
    if (trace_on()) {
        const double t = now_us();
        double su = 0;
        int sc = 0;
        for (auto &x : g->ctx) {
            su += x.sync_us;
            sc += x.syncs;
            x.sync_us = 0;
            x.syncs = 0;
        }
        fprintf(stderr, "[bc_trace] n=%lld sources=%lld mode=%d device-loop=%d batches=%lld: setup %.0f us (resolve %.0f, "
                        "sizing %.0f, plan %.0f, memset %.0f), pipelines %.0f us "
                        "(per-level waits %d, %.0f us summed over threads), finish %.0f us, total %.0f us\n",
                (long long)n, (long long)trav.size(), mode, (int)any_dl, (long long)g->last.batches, tr_plan - tr0,
                tr_m[0] - tr0, tr_m[1] - tr_m[0], tr_m[2] - tr_m[1], tr_plan - tr_m[2],
                tr_join > 0 ? tr_join - tr_plan : 0.0, sc, su, t - (tr_join > 0 ? tr_join : tr_plan), t - tr0);
    }
    finalize_stats(g);
    if (g->dl_violation)
        return fail(BC_ERR_INTERNAL, "a BFS exceeded the graph's depth bound (%d levels)", g->depth_bound);
    if (g->profile) {
        g->last.fwd_ms = sum_events(ef);
        for (auto &x : g->ctx) {
            g->last.fwd_ms += sum_events(x.ef);
            g->last.bwd_fin_ms += sum_events(x.eb);
            g->last.bwd_push_ms += sum_events(x.epush);
        }
        g->last.bwd_ms = g->last.bwd_fin_ms + g->last.bwd_push_ms;
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        g->last.total_ms = ms;
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
    }
    return BC_OK;
}

bc_status bc_sssp(bc_graph *g, int32_t source, int32_t *depth, uint64_t *sigma, uint8_t *sigma_overflow,
                  double *delta) {
    if (!g) return fail(BC_ERR_INVALID, "NULL handle");
    if (source < 0 || source >= g->n) return fail(BC_ERR_INVALID, "source %d out of range", source);
    if (g->pruned && g->h_removed[source])
        return fail(BC_ERR_INVALID, "source %d was removed by 1-degree pruning", source);
    DeviceGuard dg(g->device);
    CK(wait_idle(g));
    const int n = (int)g->n;
    cudaStream_t st = g->own_stream;
    bc_stats keep = g->last;
    // the caller-id CSR the handle computes on: the original graph, or on a
    // pruned handle the residual graph (the removed vertices are filled in
    // afterwards from their single neighbour, cap_prune_fill_kernel)
    DevCSR &csr = g->cur();
    const uint32_t *omega = g->pruned ? g->omega : nullptr;
    CK(ctx_init(g, g->vctx));
    CK(ensure_ws(g, g->vctx.ws, 1, true, std::max(g->orig.nhub, g->run.nhub)));
    g->vctx.st = st;
    g->vctx.d_bc = g->d_bc;
    if (g->src_cap < 1) {
        dfree(g->d_src);
        CK(dalloc(&g->d_src, 1));
        g->src_cap = 1;
    }
    int *d_depth = nullptr, *d_vs = nullptr;
    unsigned long long *d_sig = nullptr;
    uint8_t *d_ov = nullptr;
    double *d_delta = nullptr;
    CK(dalloc(&d_depth, n));
    CK(dalloc(&d_sig, n));
    CK(dalloc(&d_ov, n));
    CK(dalloc(&d_delta, n));
    CK(dalloc(&d_vs, n));
    CU(cudaMemcpyAsync(g->d_src, &source, 4, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(d_depth, 0xff, (size_t)n * 4, st));
    CU(cudaMemsetAsync(d_delta, 0, (size_t)n * 8, st));
    CU(cudaMemsetAsync(d_sig, 0, (size_t)n * 8, st));
    CU(cudaMemsetAsync(d_ov, 0, (size_t)n, st));
    // delta of lane 0 through the capture path: source -> slot 0
    CU(cudaMemsetAsync(d_vs, 0xff, (size_t)n * 4, st));
    CU(cudaMemsetAsync(d_vs + source, 0, 4, st));
    bc_status s = BC_OK;
    if (csr.h_deg[source] > 0) {
        BatchCtx c{};
        c.csr = &csr;
        c.omega = omega;
        c.src = g->d_src;
        c.nl = 1;
        c.st = st;
        c.run_backward = false;
        std::vector<uint64_t *> lv;
        c.lvl_out = &lv;
        int Lmax = 0;
        c.levels_out = &Lmax;
        s = run_batch<1, unsigned long long>(g, g->vctx, c, nullptr, nullptr);
        if (s == BC_OK) {
            for (int l = 0; l <= Lmax; ++l)
                depth_from_mask_kernel<<<(n + 255) / 256, 256, 0, st>>>(lv[l], n, 1, l, d_depth);
            for (int l = 0; l <= Lmax; ++l)
                gather_level_lane0_kernel<unsigned long long><<<(n + 255) / 256, 256, 0, st>>>(
                    n, lv[l], 1, (const unsigned long long *)g->vctx.ws.slev[l], 64, g->vctx.ws.ovf, d_sig, d_ov);
            // fp64 pass for delta (its own W = 1 pipeline)
            s = ctx_init(g, g->sctx);
            if (s == BC_OK) s = ensure_ws(g, g->sctx.ws, 1, false, std::max(g->orig.nhub, g->run.nhub));
            g->sctx.st = st;
            g->sctx.d_bc = g->d_bc;
            if (s == BC_OK) {
                CU(cudaMemsetAsync(g->d_bc, 0, (size_t)n * 8, st));
                BatchCtx c2 = c;
                c2.run_backward = true;
                c2.endpoint = false;
                c2.cap_vslot = d_vs;
                c2.cap_delta = d_delta;
                c2.lvl_out = nullptr;
                c2.levels_out = nullptr;
                s = run_batch<1, double>(g, g->sctx, c2, nullptr, nullptr);
            }
        }
    } else {
        const int zero = 0;
        CU(cudaMemcpyAsync(d_depth + source, &zero, 4, cudaMemcpyHostToDevice, st));
        const unsigned long long one = 1;
        CU(cudaMemcpyAsync(d_sig + source, &one, 8, cudaMemcpyHostToDevice, st));
    }
    if (s == BC_OK && g->pruned)
        cap_prune_fill_kernel<unsigned long long><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
            1, n, g->orig.rp, g->orig.col, g->removed, g->omega, d_depth, d_sig, d_delta, d_ov);
    if (s == BC_OK) {
        CU(cudaGetLastError());
        if (depth) CU(cudaMemcpyAsync(depth, d_depth, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
        if (sigma) CU(cudaMemcpyAsync(sigma, d_sig, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
        if (sigma_overflow) CU(cudaMemcpyAsync(sigma_overflow, d_ov, (size_t)n, cudaMemcpyDeviceToHost, st));
        if (delta) CU(cudaMemcpyAsync(delta, d_delta, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    dfree(d_depth);
    dfree(d_sig);
    dfree(d_ov);
    dfree(d_delta);
    dfree(d_vs);
    g->last = keep;
    return s;
}

}  // extern "C"
