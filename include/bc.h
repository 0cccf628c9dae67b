/*
 * bc.h -- C ABI of the B200-native exact-Brandes betweenness-centrality hot
 * path (libbcb200.so).  extern "C", plain pointers and sizes, no C++ or torch
 * types, no exceptions cross this boundary.
 *
 * Problem statement (Sec. 2): G = (V, E) undirected and
 * unweighted, n = |V|, m unordered pairs; the betweenness of v is
 *     BC(v) = sum_{s != t != v} sigma_st(v) / sigma_st            (Eq.1)
 *           = sum_{s != v} delta_s(v)                             (Eq.3)
 * with the dependency recursion of Eq.(2).  Scores are
 * UNNORMALISED over ORDERED pairs (Alg.1 adds delta_s(w) once per source; a
 * path P3 has centre score 2).
 *
 * Threading: calls on one handle must be serialised by the caller.  Distinct
 * handles may be used from distinct threads.  Every handle is bound to one
 * CUDA device; the library sets that device for the duration of a call and
 * restores the caller's current device afterwards.
 *
 * Errors: every call returns a bc_status; nothing is thrown.  On error the
 * outputs are unspecified and bc_last_error() (thread-local) carries a
 * one-line detail (for BC_ERR_CUDA it includes cudaGetErrorString()).
 */
#ifndef BC_B200_H
#define BC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bc_graph bc_graph; /* opaque; owns all device memory it allocates */

typedef enum {
    BC_OK = 0,
    BC_ERR_INVALID = 1,  /* bad argument: n<=0 or n>2^31-1, malformed CSR (when
                            validating), source out of range, duplicate source,
                            pruned-away source, unknown option, NULL handle    */
    BC_ERR_NOMEM = 2,    /* cudaMalloc / host allocation failed               */
    BC_ERR_CUDA = 3,     /* any other CUDA runtime failure                    */
    BC_ERR_STATE = 4,    /* call not valid in the handle's state (e.g. second
                            bc_prune_degree1: the paper's single pass,
                            PAPER.md:580 footnote)                            */
    BC_ERR_INTERNAL = 5
} bc_status;

/* bc_graph_create flags */
#define BC_CREATE_VALIDATE 0x1u /* O(m) device check: rows sorted ascending,
                                   symmetric, no self-loops, no duplicates   */

/*
 * bc_graph_create -- copy a simple undirected graph in CSR form to `device`
 * (SPEC.md:22-28 invariants).
 *   n        number of vertices, 1 <= n <= 2^31-1.
 *   row_ptr  HOST int64[n+1], row_ptr[0] = 0, non-decreasing,
 *            row_ptr[n] = 2m <= 2^31-1 (directed entries).
 *   col_idx  HOST int32[row_ptr[n]]: the neighbours of v are
 *            col_idx[row_ptr[v] .. row_ptr[v+1]), strictly ascending.
 *   device   CUDA device ordinal the handle is bound to.
 *   flags    0 or BC_CREATE_VALIDATE.  Without validation a CSR that is not
 *            simple/symmetric gives undefined results (parallel edges would
 *            count as distinct shortest paths).
 *   out      receives the handle.
 * Ownership: the caller keeps its host arrays (they are copied); the handle
 * owns the device copies until bc_destroy.
 */
bc_status bc_graph_create(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, int device,
                          uint32_t flags, bc_graph **out);

/*
 * bc_prune_degree1 -- 1-degree reduction, Alg.6 and
 * Eq.(4), run on the device in one pass (no cascaded
 * tree removal, PAPER.md:580 footnote): every vertex u of degree 1 is
 * removed, omega(v) counts v's removed neighbours, and the residual graph
 * keeps the edges whose two endpoints both survive (a K2 component loses
 * both endpoints).  Subsequent bc_compute calls run Brandes on the residual
 * graph with the Eq.(5) recursion and the endpoint terms (R7-R13)
 * and return the SAME scores as on the unpruned graph.
 *   out_removed  nullable; receives the number of removed vertices.
 * BC_ERR_STATE if the handle was already pruned.
 */
bc_status bc_prune_degree1(bc_graph *g, int64_t *out_removed);

/*
 * bc_prune_degree1_share / bc_prune_degree1_apply -- the distributed form of
 * Alg.6 ("if u mod #P = P_i assign (u,v) to
 * E_i"; 1-D partitioning keeps all edges of u on one processor,
 * PAPER.md:584-586).  Each of `nranks` processes holding the same graph
 * calls _share for its `rank`: the vertices u = rank, rank + nranks, ... are
 * scanned, u with a single edge (u,v) is removed (removed_part[u] = 1) and
 * omega_part[v] is incremented (lines 6-9).  The caller sums the nranks
 * outputs element-wise (one all-reduce of 2 n uint32, e.g. NCCL on the same
 * stream) and passes the sums to _apply, which drops the symmetric edges of
 * the removed ones and leaves the handle in exactly the
 * state bc_prune_degree1 produces (no cascaded tree removal).
 *   omega_part, removed_part  DEVICE uint32[n] on the handle's device,
 *                overwritten (zeroed, then this share's contributions).
 *   cuda_stream  _share: stream-ordered on it and asynchronous (NULL: waits
 *                for all prior device work, runs on the library stream,
 *                synchronous).  _apply: waits for it first (NULL: for all
 *                prior device work -- e.g. an all-reduce on the legacy
 *                default stream).
 *   omega, removed  DEVICE uint32[n]: the sums over all ranks; removed[v]
 *                must be 1 exactly for the degree-1 vertices, else
 *                BC_ERR_INVALID (a share missing or counted twice) and the
 *                handle is unchanged.
 *   out_removed  nullable; number of removed vertices.
 * BC_ERR_STATE if the handle was already pruned; BC_ERR_INVALID on a bad
 * rank, NULL or host pointers.  Ownership: the caller's buffers.
 */
bc_status bc_prune_degree1_share(const bc_graph *g, int rank, int nranks, uint32_t *omega_part,
                                 uint32_t *removed_part, void *cuda_stream);
bc_status bc_prune_degree1_apply(bc_graph *g, const uint32_t *omega, const uint32_t *removed, void *cuda_stream,
                                 int64_t *out_removed);

/*
 * bc_compute -- exact BC restricted to a source set S (Eq.3 with s in S):
 *     out_bc[v] = sum_{s in S, s != v} delta_s(v)
 * computed on the device: per batch of sources, a level-synchronous forward
 * sweep counting sigma and depth (Alg.2/Alg.3), then the
 * backward successor-checking sweep (Alg.4/Alg.5) and the
 * BC update (Alg.1 line 30).  Frontier edges are mapped to threads through a
 * per-tile exclusive scan of frontier degrees plus a binary search
 * (PAPER.md:310-330), many sources run concurrently as bit lanes.
 *   sources      HOST int32[num_sources] distinct vertex ids, or NULL for all
 *                vertices (unpruned) / all eligible vertices (pruned: not
 *                removed and residual degree > 0 or omega > 0).  Isolated
 *                sources contribute 0.
 *   out_bc       double[n], HOST or DEVICE pointer (detected).  Overwritten,
 *                never accumulated.
 *   cuda_stream  cudaStream_t or NULL (library-internal stream).  The call is
 *                stream-ordered on it.  With a DEVICE out_bc and device-driven
 *                batches (BC_OPT_DEVICE_LOOP, the default when eligible; slices
 *                mode always) it is also ASYNCHRONOUS: it returns once the work
 *                is enqueued -- no host wait per level or at the end -- so work
 *                queued behind it on `cuda_stream` (e.g. an NCCL all-reduce of
 *                out_bc) sees the result; bc_get_stats waits for the call's
 *                counters.  It waits before returning when out_bc is a HOST
 *                pointer, when cuda_stream is NULL (nothing to order on), when a
 *                capture is pending (bc_set_capture), under
 *                BC_OPT_PROFILE or BC_TRACE, with the host-driven level loop
 *                (BC_OPT_DEVICE_LOOP 0 or an ineligible configuration: one host
 *                wait per BFS level, the paper's nq test PAPER.md:387), and with
 *                4-byte rows forced or chosen for memory (it must learn whether a
 *                batch needs the fp64 re-run).
 * Pruned handles: S = {s} stands for s plus its removed degree-1 children
 * (R13), i.e. the result equals the unpruned BC over S+; with
 * S = all it is the exact BC.  A removed source is BC_ERR_INVALID.
 */
bc_status bc_compute(bc_graph *g, const int32_t *sources, int64_t num_sources, double *out_bc,
                     void *cuda_stream);

/* bc_destroy -- free every resource of the handle; NULL-safe. */
bc_status bc_destroy(bc_graph *g);

const char *bc_status_string(bc_status s);
const char *bc_last_error(void); /* thread-local detail of the last failure */

/*
 * bc_sssp -- verification only (not timed): one source, exact integer sigma
 * (uint64 rows, W = 1 lane, the caller-id CSR).  On an unpruned handle it
 * traverses the graph; on a PRUNED handle it traverses the residual graph
 * (Eq.(5) recursion) and fills the removed vertices as bc_set_capture
 * describes, so the outputs describe the unpruned graph either way; a
 * removed source is BC_ERR_INVALID.  All outputs are HOST arrays of length n
 * (each nullable):
 *   depth           int32, -1 if unreachable                  (Alg.2 d[])
 *   sigma           uint64 shortest-path counts (exact integer path)
 *   sigma_overflow  uint8, 1 where sigma (or a predecessor's) exceeded 2^64-1
 *   delta           double dependency delta_s(v) (0 for s and unreached)
 * Synchronous.
 */
bc_status bc_sssp(bc_graph *g, int32_t source, int32_t *depth, uint64_t *sigma,
                  uint8_t *sigma_overflow, double *delta);

/*
 * bc_set_capture -- verification only (not timed): the NEXT bc_compute on
 * this handle also records the per-source Brandes state of each captured
 * source, as computed by that call's production kernels -- the same batch,
 * lane width, sigma-row tier (16/32/64 bits), relabelled CSR, hub split and
 * concurrent pipelines (lanes mode), or the same one-source-per-CTA kernel
 * (slices mode, CAP instantiation).  For i < n_cap and every vertex v
 * (caller ids), with s = sources[i]:
 *   depth[i*n + v]  int32   d(s, v), -1 if unreachable       (Alg.2 d[])
 *   sigma[i*n + v]  double  sigma_sv: the integer the tier's rows held,
 *                           converted (exact below 2^53; fp64 rows round
 *                           above it, like the oracle's fp64 sigma)     (Alg.1 line 20)
 *   delta[i*n + v]  double  delta_s(v) (Eq.(2)); 0 at s
 *                           and at unreached vertices
 *   tier[i]         int32   bits of the sigma rows the source's batch
 *                           completed with (16, 32, 64; slices mode: 64);
 *                           0 for a source without a traversal (isolated,
 *                           or residual-isolated on a pruned handle)
 * On a PRUNED handle the outputs describe the UNPRUNED graph (as bc_compute's
 * scores do, R13): a removed vertex u with neighbour p gets
 * d(s,u) = d(s,p) + 1, sigma_su = sigma_sp, delta_s(u) = 0, and a kept
 * vertex v != s gets delta_s(v) = delta'_s(v) + omega(v) (Eq.(5)).
 *   sources   HOST int32[n_cap], distinct; each must be in the source set of
 *             the next bc_compute (else that call fails with BC_ERR_INVALID).
 *   n_cap     0 .. BC_CAPTURE_MAX; 0 cancels a pending capture.
 *   depth, sigma, delta, tier   HOST arrays ([n_cap*n], [n_cap]), each
 *             nullable; owned by the caller and written during the next
 *             bc_compute, which then returns only after they are filled.
 * The capture applies to one bc_compute call, successful or not.  Device
 * memory: 36 bytes per captured source per vertex, allocated on first use.
 */
#define BC_CAPTURE_MAX 4096
bc_status bc_set_capture(bc_graph *g, const int32_t *sources, int64_t n_cap, int32_t *depth, double *sigma,
                         double *delta, int32_t *tier);

/* Tuning options (bc_set_option).  Values are validated. */
typedef enum {
    BC_OPT_LANE_WORDS = 1, /* 0 = auto (8 for n <= 2^18, else 4, fewer for small source sets or short HBM),
                              else 1, 2, 4 or 8: K = 64*value source lanes per batch */
    BC_OPT_HUB_DEGREE = 2, /* vertices with degree > value are processed as split hubs (>= 32) */
    BC_OPT_PROFILE = 3,    /* 1 = record CUDA events around the level kernels (bc_get_stats) */
    BC_OPT_MODE = 4,       /* 0 = auto, 1 = lanes (bit-lane batches), 2 = slices (CTA per source) */
    BC_OPT_RELABEL = 5,    /* traverse a relabelled copy of the graph: 0 = caller's ids, 1 (default) =
                              degree-descending, or breadth-first (Cuthill-McKee, from a far vertex of each
                              component) when max degree <= 64 and auto mode picks slices;
                              2 = breadth-first always.  Results are returned in caller ids either way */
    BC_OPT_SOURCE_ORDER = 6, /* batch schedule: 0 = given order, 1 = degree, 2 (default) = anchor clusters */
    BC_OPT_FWD_PUSH = 7,    /* forward levels L <= value expand in push form (default 0), later ones pull */
    BC_OPT_BWD_MODE = 8,    /* backward sweep: 0 = default, 1 = push form, 2 = pull form (successor checking) */
    BC_OPT_SIGMA_WIDTH = 9  /* lanes forward sigma rows: 0 or 16 (default) = uint16 rows, a batch whose
                               sigma exceeds 65535 is re-run with uint32 rows, then (sigma >= 2^32)
                               with fp64 rows; 64 = fp64 rows only.
                               sigma is an integer (Alg.1 line 20), so both are exact */,
    BC_OPT_STREAMS = 10,    /* lanes mode: concurrent batch pipelines, 0 = auto (8 for n <= 2^18, else 3;
                               fewer if HBM is short), or 1..8.
                               Batches are independent (BC is additive over sources) */
    BC_OPT_TWO_DEGREE = 11, /* lanes mode: 1 = 2-degree heuristic: a degree-2 source
                               whose two neighbours are also sources gets its shortest-path tree derived
                               from theirs (Lemma 1, Eq.(6)) instead of a traversal; default 0 */
    BC_OPT_DEVICE_LOOP = 12, /* lanes mode: 1 (default) = device-driven batches when eligible -- each batch
                               (every level, the sigma-tier fallbacks) is one CUDA graph launch with the
                               termination test on the device; 0 = host-driven level loop
                               (one host wait per level); 2 = device-driven with 4-byte rows forced (the
                               fp64 tier then re-runs on the host-driven path; testing).  Eligible: default
                               sweep options, no profiling, graph depth bound <= 32 levels (bc_graph_create) */
    BC_OPT_SLICES_KERNEL = 13 /* slices mode kernel (NEXT-2 ablation): 0 = auto; 1 = general (frontier
                               degrees block-scanned into CD + binary search; push sigma
                               with fp64 atomics); 2 = general with prefix-sum reuse (the forward's CD
                               prefixes kept and reused by the backward); 3 = degree-
                               bounded, thread per frontier vertex, pull, global bitmaps; 4 = the same with
                               a 2-bit per-vertex state in shared memory (n <= 1179648).  3/4 need max
                               degree <= 64, else bc_compute fails with BC_ERR_INVALID */
} bc_option;

bc_status bc_set_option(bc_graph *g, int option, int64_t value);

/* Statistics of the last bc_compute on this handle. */
typedef struct {
    int64_t num_sources;     /* traversal sources (residual degree > 0)          */
    int64_t num_trivial;     /* endpoint-only sources (pruned, residual-isolated) */
    int64_t batches;         /* source batches                                  */
    int64_t lanes;           /* K, sources per batch                            */
    int64_t levels_total;    /* sum over batches of forward levels               */
    int64_t fwd_launches;    /* forward level-kernel launches                   */
    int64_t bwd_launches;    /* backward level-kernel launches                  */
    int64_t reached;         /* sum over sources of reached vertices (n_s, residual) */
    int64_t adj_reached;     /* sum over sources of reached adjacency (A_s)     */
    int64_t dag_edges;       /* sum over sources of DAG edges (D_s)              */
    double fwd_ms;           /* summed forward level-kernel time (BC_OPT_PROFILE) */
    double bwd_ms;           /* summed backward level-kernel time (BC_OPT_PROFILE) */
    double total_ms;         /* whole bc_compute device time (BC_OPT_PROFILE)    */
    int64_t kernel_launches; /* all library kernel launches of the call          */
    int64_t dist_sum;        /* sum over sources of sum of depths of reached vertices */
    int64_t fwd_items;       /* adjacency items scanned by forward level kernels (per batch, not per lane) */
    int64_t fwd_hits;        /* items with >= 1 contributing lane, forward      */
    int64_t bwd_items;       /* adjacency items scanned by backward level kernels */
    int64_t bwd_hits;        /* items with >= 1 contributing lane, backward     */
    double bwd_fin_ms;       /* backward finalize kernels (BC_OPT_PROFILE)       */
    double bwd_push_ms;      /* backward push kernels (BC_OPT_PROFILE)           */
    int64_t narrow_batches;  /* batches completed with 16-bit sigma rows          */
    int64_t narrow_fallbacks;/* batches re-run whole with wider rows after a sigma > 65535 */
    int64_t mid_batches;     /* ... of which completed with 32-bit rows (the rest: fp64) */
    int64_t derived_lanes;   /* 2-degree sources whose tree was derived (BC_OPT_TWO_DEGREE) */
    int64_t widened_batches; /* host-driven 16-bit batches that switched to 32-bit rows at the level whose
                                sigma exceeded 65535 (only that level re-expanded, no batch re-run) */
} bc_stats;

bc_status bc_get_stats(const bc_graph *g, bc_stats *out);

/* Pruning outputs for bit-exact parity with the Alg.6 oracle (HOST arrays,
 * each nullable): omega uint32[n], removed uint8[n], residual CSR
 * row_ptr int64[n+1] and col int32[capacity >= residual nnz]; *res_nnz gets
 * the residual nnz.  BC_ERR_STATE if the handle is not pruned. */
bc_status bc_get_pruning(const bc_graph *g, uint32_t *omega, uint8_t *removed, int64_t *res_row_ptr,
                         int32_t *res_col, int64_t *res_nnz);

/* Handle facts: n, original nnz, current (residual) nnz, device. */
bc_status bc_graph_info(const bc_graph *g, int64_t *n, int64_t *nnz, int64_t *res_nnz, int *device);

#ifdef __cplusplus
}
#endif
#endif /* BC_B200_H */
