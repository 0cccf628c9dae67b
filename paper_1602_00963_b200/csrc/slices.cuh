// slices.cuh -- "one source per CTA" Brandes for long-diameter graphs
// (batch mode "slices"; the 2-D grid workload).
//
// On a high-diameter graph (grid 512x512: up to 1022 levels, frontiers of a
// few hundred vertices) a level-synchronous sweep over the whole device pays
// a grid-wide barrier per level.  Here every CTA of a persistent kernel owns
// one source at a time and runs the paper's per-source algorithm with a
// __syncthreads() as the level barrier:
//
//   forward (Alg.2 / Alg.3): the frontier Q[qs, qe) is cut
//     into chunks of BC_NT vertices; their degrees are block-scanned into a
//     shared CD array and every thread takes items e -> (vertex, edge) by
//     binary search.  Discovery is an atomic test-and-set
//     on a visited bitmap (reading R4: Alg.3's test-then-set bmap races);
//     sigma[w] += sigma[v] (fp64 atomic) when w is in the next level, which a
//     second bitmap marks.  New vertices are appended to Q with one
//     shared-memory atomic per warp.
//   backward (Alg.4 / Alg.5, successor checking, reading R2): for
//     L = Lmax..1 the level bitmap marks level L+1; items of level-L vertices
//     add coef(v) of successors into cf[w]; then cf[w] := coef(w) =
//     (1 + omega(w) + sigma(w) cf(w)) / sigma(w) and the CTA-private BC row
//     gets (1 + omega(s)) (delta(w) + omega(w)).
//
// The two bitmaps (n bits each) live in shared memory when they fit
// (n <= 2^18: 2 x 32 KB) -- depth is never stored -- and in CTA-private
// global memory otherwise.  sigma / cf / the BC row are CTA-private global
// arrays; only reached vertices are reset after a source.  The private BC
// rows are summed by slices_reduce_kernel at the end.
#pragma once
#include "util.cuh"

namespace bcb {

constexpr int SLICES_SMEM_BM_WORDS = 8192;  // 2 x 32 KB shared bitmaps => n <= 262144

struct SlicesParams {
    int n;
    const int *rp;
    const int *col;
    const uint32_t *omega;  // nullable
    const int *src;         // sources (compute ids)
    int nsrc;
    int *next_src;          // dynamic source counter (self-resetting)
    // CTA-private arrays, each [gridDim.x][n] (loff: [gridDim.x][n + 2])
    double *sigma;          // 0 between sources
    double *cf;             // acc -> coef; 0 between sources
    int *queue;
    int *loff;
    double *bcp;            // private BC rows (slices_kernel)
    double *bc;             // shared BC vector (slices_lowdeg_kernel adds into it)
    const int4 *ell4;       // max degree <= 4: neighbours padded with -1, one 16-byte load per vertex
    int4 *qrow;             // [gridDim.x][n] ELL rows in queue order (BC_SM_QROW), else null
    unsigned *bm;           // global bitmaps [gridDim.x][2][bm_words] (when not in shared memory)
    int *cdq;               // slices_kernel<REUSE>: [gridDim.x][n] inclusive frontier-degree prefix of each
                            // queue position within its chunk (the forward's scan, reused backward)
    int bm_words;
    unsigned long long *stats;  // [4] reached, adjacency, dag edges, depth sum
    // verification capture (bc_set_capture; CAP instantiations only): slot of
    // a source (compute ids) or -1, and the captured per-source state [slot][n]
    const int *cap_vslot;
    int *cap_depth;
    double *cap_sigma, *cap_delta;
};

// capture of w's depth / sigma / delta in source slot cs (backward commit)
template <bool CAP>
__device__ __forceinline__ void slices_cap(const SlicesParams &p, int cs, int w, int L, double sg, double delta) {
    if constexpr (CAP) {
        if (cs >= 0) {
            const size_t o = (size_t)cs * p.n + w;
            p.cap_depth[o] = L;
            p.cap_sigma[o] = sg;
            p.cap_delta[o] = delta;
        }
    }
}

struct SlicesSmem {
    int cd[BC_NT + 1];
    int vs[BC_NT];
    int rs[BC_NT];
    int scan[2 * BC_NW + 2];
    int tail;
    int cnt[3];  // slices_lowdeg_sm_kernel: appends of level L counted in cnt[L % 3] (rotating, see there)
    int src;
    double red[32];
};

// Process the items of frontier chunk Q[c0, c1) (<= BC_NT vertices); calls
// f(v, w) for every item.
// REUSE (prefix-sum reuse): the forward (STORE) writes
// each queue position's inclusive degree prefix within its chunk to cdq; the
// backward (LOAD) walks the same chunks of the same level (both cut Q from
// the level start in steps of BC_NT) and reads the prefixes back instead of
// re-scanning.
template <int CDMODE = 0, typename F>  // 0: scan, 1: scan and store to cdq, 2: load from cdq
__device__ __forceinline__ void slices_chunk_items(const SlicesParams &p, SlicesSmem &sm, const int *Q, int c0,
                                                   int c1, F &&f, int *cdq = nullptr) {
    const int i = threadIdx.x;
    int deg = 0, v = -1, rs = 0;
    int ex, d1, tot, d2;
    const int nv = c1 - c0;
    if constexpr (CDMODE == 2) {
        if (i < nv) {
            v = Q[c0 + i];
            rs = p.rp[v];
            ex = i > 0 ? cdq[c0 + i - 1] : 0;
        }
        tot = cdq[c1 - 1];
    } else {
        if (c0 + i < c1) {
            v = Q[c0 + i];
            rs = p.rp[v];
            deg = p.rp[v + 1] - rs;
        }
        block_excl_scan2(deg, 0, ex, d1, tot, d2, sm.scan);
        if constexpr (CDMODE == 1) {
            if (i < nv) cdq[c0 + i] = ex + deg;
        }
    }
    if (i < nv) {
        sm.cd[i] = ex;
        sm.vs[i] = v;
        sm.rs[i] = rs;
    }
    if (i == 0) sm.cd[nv] = tot;
    __syncthreads();
    for (int e = i; e < tot; e += BC_NT) {
        const int s = slot_of(sm.cd, nv, e);
        f(sm.vs[s], p.col[sm.rs[s] + (e - sm.cd[s])]);
    }
    __syncthreads();
}

template <bool SMEM_BM, bool CAP = false, bool REUSE = false>
__global__ void __launch_bounds__(BC_NT) slices_kernel(SlicesParams p) {
    __shared__ SlicesSmem sm;
    extern __shared__ unsigned smbm[];  // 2 * SLICES_SMEM_BM_WORDS when SMEM_BM
    const size_t n = (size_t)p.n;
    double *sigma = p.sigma + blockIdx.x * n;
    double *cf = p.cf + blockIdx.x * n;
    int *Q = p.queue + blockIdx.x * n;
    int *loff = p.loff + blockIdx.x * (n + 2);
    double *bcp = p.bcp + blockIdx.x * n;
    int *cdq = REUSE ? p.cdq + blockIdx.x * n : nullptr;
    unsigned *vis = SMEM_BM ? smbm : p.bm + (size_t)blockIdx.x * 3 * p.bm_words;
    unsigned *lvb = vis + (SMEM_BM ? SLICES_SMEM_BM_WORDS : p.bm_words);
    const int bmw = p.bm_words;
    const int lane = lane_id();
    unsigned long long st_reach = 0, st_adj = 0, st_dag = 0, st_dsum = 0;

    for (int i = threadIdx.x; i < bmw; i += BC_NT) {
        vis[i] = 0u;
        lvb[i] = 0u;
    }
    __syncthreads();

    for (;;) {
        if (threadIdx.x == 0) {
            const int t = atomicAdd(p.next_src, 1);
            if (t == p.nsrc + (int)gridDim.x - 1) *p.next_src = 0;  // last fetch resets
            sm.src = t;
        }
        __syncthreads();
        const int si = sm.src;
        __syncthreads();
        if (si >= p.nsrc) break;
        const int s = p.src[si];
        const int cs = CAP ? p.cap_vslot[s] : -1;
        if (threadIdx.x == 0) {
            vis[s >> 5] |= 1u << (s & 31);
            sigma[s] = 1.0;
            Q[0] = s;
            loff[0] = 0;
            loff[1] = 1;
            sm.tail = 1;
        }
        __syncthreads();
        // ---------------- forward: level L -> L+1
        int L = 0, qs = 0, qe = 1;
        while (qs < qe) {
            for (int c0 = qs; c0 < qe; c0 += BC_NT) {
                const int c1 = min(qe, c0 + BC_NT);
                slices_chunk_items<REUSE ? 1 : 0>(p, sm, Q, c0, c1, [&](int v, int w) {
                    // visited bit clear => w is discovered now, at level L+1; the
                    // level bit is published before the visited bit, so a thread
                    // that finds w visited also sees whether it is at L+1
                    const unsigned bit = 1u << (w & 31);
                    bool nxt, mine = false;
                    if (!(vis[w >> 5] & bit)) {
                        atomicOr(&lvb[w >> 5], bit);
                        __threadfence_block();
                        mine = !(atomicOr(&vis[w >> 5], bit) & bit);
                        nxt = true;
                    } else {
                        nxt = (lvb[w >> 5] & bit) != 0;
                    }
                    const unsigned bal = __ballot_sync(__activemask(), mine);
                    if (mine) {
                        const int leader = __ffs(bal) - 1;
                        int base = 0;
                        if (lane == leader) base = atomicAdd(&sm.tail, __popc(bal));
                        base = __shfl_sync(bal, base, leader);
                        Q[base + __popc(bal & ((1u << lane) - 1u))] = w;
                    }
                    if (nxt) {
                        atomicAdd(&sigma[w], sigma[v]);
                        ++st_dag;
                    }
                }, cdq);
            }
            __syncthreads();
            qs = qe;
            qe = sm.tail;
            ++L;
            if (threadIdx.x == 0) loff[L + 1] = qe;
            // level L is now complete: clear its level bits
            for (int i = qs + threadIdx.x; i < qe; i += BC_NT) {
                const int w = Q[i];
                atomicAnd(&lvb[w >> 5], ~(1u << (w & 31)));
            }
            __syncthreads();
        }
        const int Lmax = L - 1;  // deepest non-empty level
        const int reached = qe;
        // ---------------- backward: level L = Lmax .. 1
        const double ws1 = 1.0 + (p.omega ? (double)p.omega[s] : 0.0);
        double ns_loc = 0.0;
        for (L = Lmax; L >= 1; --L) {
            const int a = loff[L], b = loff[L + 1];
            if (L < Lmax) {
                const int a1 = loff[L + 1], b1 = loff[L + 2];
                for (int i = a1 + threadIdx.x; i < b1; i += BC_NT) {
                    const int v = Q[i];
                    atomicOr(&lvb[v >> 5], 1u << (v & 31));
                }
                __syncthreads();
                for (int c0 = a; c0 < b; c0 += BC_NT) {
                    const int c1 = min(b, c0 + BC_NT);
                    slices_chunk_items<REUSE ? 2 : 0>(p, sm, Q, c0, c1, [&](int w, int v) {
                        if (lvb[v >> 5] & (1u << (v & 31))) atomicAdd(&cf[w], cf[v]);
                    }, cdq);
                }
                __syncthreads();
                for (int i = a1 + threadIdx.x; i < b1; i += BC_NT) {
                    const int v = Q[i];
                    atomicAnd(&lvb[v >> 5], ~(1u << (v & 31)));
                }
            }
            for (int i = a + threadIdx.x; i < b; i += BC_NT) {
                const int w = Q[i];
                const double om = p.omega ? (double)p.omega[w] : 0.0;
                const double sg = sigma[w];
                const double delta = sg * cf[w];
                cf[w] = (1.0 + om + delta) / sg;
                slices_cap<CAP>(p, cs, w, L, sg, delta);
                const double c = ws1 * (delta + om);
                if (c != 0.0) bcp[w] += c;
                st_dsum += (unsigned long long)L;
            }
            __syncthreads();
        }
        // ---------------- n_s, stats, reset of the reached vertices
        for (int i = threadIdx.x; i < reached; i += BC_NT) {
            const int w = Q[i];
            ns_loc += 1.0 + (p.omega ? (double)p.omega[w] : 0.0);
            st_adj += (unsigned long long)(p.rp[w + 1] - p.rp[w]);
        }
        st_reach += (threadIdx.x == 0) ? (unsigned long long)reached : 0ull;
        ns_loc = warp_sum(ns_loc);
        if (lane == 0) sm.red[warp_id()] = ns_loc;
        __syncthreads();
        if (threadIdx.x == 0 && p.omega) {
            double ns = 0.0;
            for (int w = 0; w < BC_NW; ++w) ns += sm.red[w];
            const double om = (double)p.omega[s];
            if (om != 0.0) bcp[s] += om * (ns - 2.0);
        }
        for (int i = threadIdx.x; i < reached; i += BC_NT) {
            const int w = Q[i];
            vis[w >> 5] = 0u;  // whole word: every vertex of it that was set is in Q too
            sigma[w] = 0.0;
            cf[w] = 0.0;
        }
        __syncthreads();
    }
    const unsigned long long a = warp_sum_u64(st_reach), b = warp_sum_u64(st_adj), c = warp_sum_u64(st_dag),
                             d = warp_sum_u64(st_dsum);
    if (lane == 0) {
        if (a) atomicAdd(p.stats + 0, a);
        if (b) atomicAdd(p.stats + 1, b);
        if (c) atomicAdd(p.stats + 2, c);
        if (d) atomicAdd(p.stats + 3, d);
    }
}


// Degree-bounded graphs (max degree <= BC_LOWDEG, e.g. the 2-D grid): one
// thread per frontier vertex instead of the CD item mapping (no scan, no
// binary search), and no floating-point atomics in the sweeps -- discovery
// pushes only bits (visited bitmap + queue append), sigma is then *pulled* by
// each newly discovered vertex from its level-L neighbours (Alg.1 lines 16-19
// read from the child's side), and the backward step pulls coef from the
// level-(L+1) neighbours.  Level membership is two bitmaps (levels L and L+1).
//
// Graphs with max degree <= 4 (the grid) read a vertex's neighbours as one
// int4 of a padded (ELL) copy of the CSR: one dependent load fewer per
// vertex on every level's critical path.
//
// Per-source state is one fp64 slot per vertex: sigma(w) is *assigned* by the
// pull (never accumulated, so it needs no reset between sources) and
// overwritten in place by coef(w) = (1 + omega(w) + delta(w)) / sigma(w) in
// the backward step of w's level -- after that step sigma(w) is never read
// again and the parents at level L-1 read only coef(w).  BC is added straight
// into the shared BC vector (one fp64 red per reached vertex, L2-resident)
// instead of a CTA-private row: per source and reached vertex the CTA touches
// one 8-byte slot (written forward, read and rewritten backward) and 4 bytes
// of queue, which keeps the concurrently swept frontiers of all CTAs inside
// L2.  Neighbour lists are read BC_LD_GRP edges at a time with all loads of a
// group issued before their use (the grid's 4 neighbours in one round trip).
constexpr int BC_LOWDEG = 64;
#ifndef BC_SL_NT
#define BC_SL_NT 256  // threads per CTA of the degree-bounded slices kernel (more sources in flight)
#endif
#ifndef BC_SL_MINB
#define BC_SL_MINB 4  // resident CTAs per SM the register budget is sized for (measured best on the grid)
#endif
constexpr int BC_LD_GRP = 4;

// The neighbours of v as groups of BC_LD_GRP ids (-1 = none); with ELL the
// whole list is one int4 load (max degree <= 4), else CSR reads.
template <bool ELL, typename F>
__device__ __forceinline__ void lowdeg_nbrs(const SlicesParams &p, int v, F &&f) {
    if (ELL) {
        const int4 q = p.ell4[v];
        int w[BC_LD_GRP] = {q.x, q.y, q.z, q.w};
        f(w);
    } else {
        const int a = p.rp[v], b = p.rp[v + 1];
        for (int e = a; e < b; e += BC_LD_GRP) {
            int w[BC_LD_GRP];
#pragma unroll
            for (int k = 0; k < BC_LD_GRP; ++k) w[k] = e + k < b ? p.col[e + k] : -1;
            f(w);
        }
    }
}

template <bool ELL, bool CAP = false>
__global__ void __launch_bounds__(BC_SL_NT, BC_SL_MINB) slices_lowdeg_kernel(SlicesParams p) {
    __shared__ SlicesSmem sm;
    const size_t n = (size_t)p.n;
    double *sc = p.sigma + blockIdx.x * n;  // sigma, then coef (in place)
    int *Q = p.queue + blockIdx.x * n;
    int *loff = p.loff + blockIdx.x * (n + 2);
    unsigned *vis = p.bm + (size_t)blockIdx.x * 3 * p.bm_words;
    unsigned *lb0 = vis + p.bm_words;  // level bitmaps, alternating
    unsigned *lb1 = lb0 + p.bm_words;
    const int lane = lane_id();
    unsigned long long st_reach = 0, st_adj = 0, st_dag = 0, st_dsum = 0;

    for (;;) {
        if (threadIdx.x == 0) {
            const int t = atomicAdd(p.next_src, 1);
            if (t == p.nsrc + (int)gridDim.x - 1) *p.next_src = 0;  // last fetch resets
            sm.src = t;
        }
        __syncthreads();
        const int si = sm.src;
        __syncthreads();
        if (si >= p.nsrc) break;
        const int s = p.src[si];
        const int cs = CAP ? p.cap_vslot[s] : -1;
        if (threadIdx.x == 0) {
            atomicOr(&vis[s >> 5], 1u << (s & 31));
            atomicOr(&lb0[s >> 5], 1u << (s & 31));
            sc[s] = 1.0;
            Q[0] = s;
            loff[0] = 0;
            loff[1] = 1;
            sm.tail = 1;
        }
        __syncthreads();
        int L = 0, qs = 0, qe = 1;
        unsigned *lcur = lb0, *lnxt = lb1;
        while (qs < qe) {
            // (1) discovery: frontier vertices push visited bits
            for (int i = qs + threadIdx.x; i < qe; i += BC_SL_NT) {
                const int v = Q[i];
                lowdeg_nbrs<ELL>(p, v, [&](const int *w) {
                    unsigned wd[BC_LD_GRP];
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) wd[k] = w[k] >= 0 ? vis[w[k] >> 5] : ~0u;
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        const unsigned bit = 1u << (w[k] & 31);
                        if (!(wd[k] & bit) && !(atomicOr(&vis[w[k] >> 5], bit) & bit)) {
                            atomicOr(&lnxt[w[k] >> 5], bit);
                            Q[atomicAdd(&sm.tail, 1)] = w[k];
                        }
                    }
                });
            }
            __syncthreads();
            const int ne = sm.tail;
            // (2) sigma pull: each new vertex sums sigma of its level-L neighbours
            for (int i = qe + threadIdx.x; i < ne; i += BC_SL_NT) {
                const int w = Q[i];
                double sg = 0.0;
                lowdeg_nbrs<ELL>(p, w, [&](const int *v) {
                    unsigned wd[BC_LD_GRP];
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) wd[k] = v[k] >= 0 ? lcur[v[k] >> 5] : 0u;
                    double x[BC_LD_GRP];
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        const bool par = (wd[k] >> (v[k] & 31)) & 1u;
                        x[k] = par ? sc[v[k]] : 0.0;
                        st_dag += par;
                    }
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) sg += x[k];
                });
                sc[w] = sg;
            }
            __syncthreads();
            // (3) retire level L's bits
            for (int i = qs + threadIdx.x; i < qe; i += BC_SL_NT) {
                const int v = Q[i];
                atomicAnd(&lcur[v >> 5], ~(1u << (v & 31)));
            }
            __syncthreads();
            qs = qe;
            qe = ne;
            ++L;
            if (threadIdx.x == 0) loff[L + 1] = qe;
            unsigned *t = lcur;
            lcur = lnxt;
            lnxt = t;
        }
        // both level bitmaps are empty again here
        const int Lmax = L - 1;
        const int reached = qe;
        const double ws1 = 1.0 + (p.omega ? (double)p.omega[s] : 0.0);
        double ns_loc = 0.0;
        for (L = Lmax; L >= 1; --L) {
            const int a = loff[L], b = loff[L + 1];
            const int a1 = loff[L + 1], b1 = loff[L + 2];
            for (int i = a1 + threadIdx.x; i < b1; i += BC_SL_NT) {
                const int v = Q[i];
                atomicOr(&lb0[v >> 5], 1u << (v & 31));
            }
            __syncthreads();
            for (int i = a + threadIdx.x; i < b; i += BC_SL_NT) {
                const int w = Q[i];
                double acc = 0.0;
                const double sg = sc[w];
                lowdeg_nbrs<ELL>(p, w, [&](const int *v) {
                    unsigned wd[BC_LD_GRP];
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) wd[k] = v[k] >= 0 ? lb0[v[k] >> 5] : 0u;
                    double x[BC_LD_GRP];
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) x[k] = ((wd[k] >> (v[k] & 31)) & 1u) ? sc[v[k]] : 0.0;
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        acc += x[k];
                        st_adj += v[k] >= 0;
                    }
                });
                const double om = p.omega ? (double)p.omega[w] : 0.0;
                const double delta = sg * acc;
                sc[w] = (1.0 + om + delta) / sg;
                slices_cap<CAP>(p, cs, w, L, sg, delta);
                const double c = ws1 * (delta + om);
                if (c != 0.0) atomicAdd(p.bc + w, c);
                st_dsum += (unsigned long long)L;
                ns_loc += 1.0 + om;
            }
            __syncthreads();
            for (int i = a1 + threadIdx.x; i < b1; i += BC_SL_NT) {
                const int v = Q[i];
                atomicAnd(&lb0[v >> 5], ~(1u << (v & 31)));
            }
        }
        __syncthreads();
        st_reach += (threadIdx.x == 0) ? (unsigned long long)reached : 0ull;
        if (threadIdx.x == 0) {
            st_adj += (unsigned long long)(p.rp[s + 1] - p.rp[s]);
            ns_loc += ws1;
        }
        ns_loc = warp_sum(ns_loc);
        if (lane == 0) sm.red[warp_id()] = ns_loc;
        // clear the visited bitmap: whole words when most of it was reached
        if (reached >= p.bm_words) {
            for (int i = threadIdx.x; i < p.bm_words; i += BC_SL_NT) vis[i] = 0u;
        } else {
            for (int i = threadIdx.x; i < reached; i += BC_SL_NT) vis[Q[i] >> 5] = 0u;
        }
        __syncthreads();
        if (threadIdx.x == 0 && p.omega) {
            double ns = 0.0;
            for (int w = 0; w < BC_SL_NT / 32; ++w) ns += sm.red[w];
            const double om = (double)p.omega[s];
            if (om != 0.0) atomicAdd(p.bc + s, om * (ns - 2.0));
        }
        __syncthreads();
    }
    const unsigned long long a = warp_sum_u64(st_reach), b = warp_sum_u64(st_adj), c = warp_sum_u64(st_dag),
                             d = warp_sum_u64(st_dsum);
    if (lane == 0) {
        if (a) atomicAdd(p.stats + 0, a);
        if (b) atomicAdd(p.stats + 1, b);
        if (c) atomicAdd(p.stats + 2, c);
        if (d) atomicAdd(p.stats + 3, d);
    }
}

// Shared-memory state variant of the degree-bounded kernel, for n small
// enough that 2 bits per vertex fit in shared memory (the 512x512 grid: 64 KB
// per CTA).  The 2-bit field of v is 0 while v is unvisited and
// (depth(v) mod 3) + 1 once discovered.  A neighbour of a level-L vertex lies
// at L-1, L or L+1 (or is unvisited), so "field == code(L)" identifies the
// level-L parents in the sigma pull and "field == code(L+1)" the children in
// the backward step: no level bitmaps to set and retire, discovery is a
// shared-memory test-and-set, and a forward level takes two barriers, a
// backward level one.  sigma / coef stay in the one fp64 slot per vertex.
__device__ __forceinline__ unsigned lowdeg_code(int L) { return (unsigned)(L % 3) + 1u; }

#ifndef BC_SM_NT
#define BC_SM_NT 512  // threads per CTA of the shared-memory-state kernel (one pass over most grid levels; 63 registers, no spills)
#endif
#ifndef BC_SM_MINB
#define BC_SM_MINB 2  // two CTAs per SM (64 KB state each)
#endif
#ifndef BC_SM_AGG
#define BC_SM_AGG 1  // one tail atomic per warp per neighbour group (test-and-sets issued together)
#endif
#ifndef BC_SM_PF
#define BC_SM_PF 0  // 1: a thread's next frontier slot loaded while it works on the current one (slower: profiles/exp_r2_grid_pf.txt)
#endif
#ifndef BC_SM_RING
#define BC_SM_RING 0  // > 0: the forward also keeps each level's queue slots (<= BC_SM_RING) in a shared double buffer
#endif
#ifndef BC_SM_BPF2
#define BC_SM_BPF2 0  // backward: the next level's first-slot vertex id is loaded one level earlier (row / sigma at level start)
#endif
#ifndef BC_SM_LOFF
#define BC_SM_LOFF 0  // > 0: level offsets of the first BC_SM_LOFF levels in shared memory (backward: one L2 hop less per level)
#endif
#ifndef BC_SM_QROW
#define BC_SM_QROW 0  // discoverer copies the new vertex's ELL row next to its queue slot
#endif
// A vertex's neighbour "row": the int4 of neighbour ids (ELL) or, for CSR
// reads, the vertex id in .x.
#ifndef BC_SM_L2HINT
#define BC_SM_L2HINT 0  // ELL rows evict-last and queue slots evict-first in L2
#endif
__device__ __forceinline__ int4 ld_row_keep(const int4 *p) {
#if BC_SM_L2HINT
    int4 r;
    asm volatile("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
                 "ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], pol;\n\t}"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
#else
    return *p;
#endif
}
__device__ __forceinline__ void st_slot_stream(int *p, int v) {
#if BC_SM_L2HINT
    asm volatile("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
                 "st.global.L2::cache_hint.b32 [%0], %1, pol;\n\t}" ::"l"(p), "r"(v) : "memory");
#else
    *p = v;
#endif
}
template <bool ELL>
__device__ __forceinline__ int4 lowdeg_row(const SlicesParams &p, int v) {
    if constexpr (ELL) return ld_row_keep(p.ell4 + v);
    else return make_int4(v, 0, 0, 0);
}
template <bool ELL, typename F>
__device__ __forceinline__ void lowdeg_row_nbrs(const SlicesParams &p, int4 row, F &&f) {
    if constexpr (ELL) {
        int w[BC_LD_GRP] = {row.x, row.y, row.z, row.w};
        f(w);
    } else {
        lowdeg_nbrs<false>(p, row.x, f);
    }
}

template <bool ELL, bool CAP = false>
__global__ void __launch_bounds__(BC_SM_NT, BC_SM_MINB) slices_lowdeg_sm_kernel(SlicesParams p) {
    __shared__ SlicesSmem sm;
    extern __shared__ unsigned f2[];  // 2 bits per vertex
#if BC_SM_LOFF
    __shared__ int loff_s[BC_SM_LOFF];  // level offsets of levels < BC_SM_LOFF (the rest: global loff)
#endif
#if BC_SM_RING
    __shared__ int qring[2 * BC_SM_RING];  // level L's slots at qring[(L & 1) * BC_SM_RING + (i - qs)]
#endif
    const size_t n = (size_t)p.n;
    const int nw = (p.n + 15) / 16;
    const int tid = threadIdx.x;
    double *sc = p.sigma + blockIdx.x * n;  // sigma, then coef (in place)
    int *Q = p.queue + blockIdx.x * n;
    int *loff_g = p.loff + blockIdx.x * (n + 2);
#if BC_SM_LOFF
    auto lo_get = [&](int i) -> int { return i < BC_SM_LOFF ? loff_s[i] : loff_g[i]; };
    auto lo_set = [&](int i, int v) {
        if (i < BC_SM_LOFF) loff_s[i] = v;
        else loff_g[i] = v;
    };
#else
    auto lo_get = [&](int i) -> int { return loff_g[i]; };
    auto lo_set = [&](int i, int v) { loff_g[i] = v; };
#endif
    constexpr bool QROW = ELL && BC_SM_QROW;
    int4 *QR = QROW ? p.qrow + blockIdx.x * n : nullptr;
    const int lane = lane_id();
    unsigned long long st_reach = 0, st_adj = 0, st_dag = 0, st_dsum = 0;
    for (int i = tid; i < nw; i += BC_SM_NT) f2[i] = 0u;

    for (;;) {
        if (tid == 0) {
            const int t = atomicAdd(p.next_src, 1);
            if (t == p.nsrc + (int)gridDim.x - 1) *p.next_src = 0;  // last fetch resets
            sm.src = t;
        }
        __syncthreads();
        const int si = sm.src;
        __syncthreads();
        if (si >= p.nsrc) break;
        const int s = p.src[si];
        const int cs = CAP ? p.cap_vslot[s] : -1;
        if (tid == 0) {
            f2[s >> 4] |= lowdeg_code(0) << ((s & 15) * 2);
            sc[s] = 1.0;
            Q[0] = s;
#if BC_SM_RING
            qring[0] = s;
#endif
            lo_set(0, 0);
            lo_set(1, 1);
            sm.cnt[0] = sm.cnt[1] = sm.cnt[2] = 0;
        }
        __syncthreads();
        // forward, one barrier per level: each thread takes a level-L vertex
        // v, loads its row once, first pulls sigma(v) from v's level-(L-1)
        // neighbours (complete before the previous barrier), then discovers
        // v's unvisited neighbours (level L+1) by shared-memory test-and-set,
        // appending them with one shared atomic per warp.  Concurrently set
        // codes are code(L+1) != code(L-1), so the parent test is unaffected.
        // Level L appends to Q[qe + cnt[L % 3]): a fast warp may start level
        // L+1's appends (into cnt[(L+1) % 3]) while a slow one still reads
        // cnt[L % 3] after the barrier, so the counters rotate; cnt[(L+1) % 3]
        // was last read right after the barrier that ended level L-2, and the
        // barrier ending level L-1 separates those reads from its reset here.
        int L = 0, qs = 0, qe = 1, r3 = 0;
        while (qs < qe) {
            const unsigned cn = lowdeg_code(L + 1), cp = lowdeg_code(L + 2);  // (L + 2) mod 3 == (L - 1) mod 3
            int *cnt = &sm.cnt[r3];
            const int r3n = r3 == 2 ? 0 : r3 + 1;
            if (tid == 0) sm.cnt[r3n] = 0;
            int v_pf = -1;  // BC_SM_PF: the next slot's vertex and row, loaded one slot ahead
            int4 row_pf = make_int4(0, 0, 0, 0);
#if BC_SM_RING
            const int *ring_cur = qring + (L & 1) * BC_SM_RING;
            int *ring_nxt = qring + ((L + 1) & 1) * BC_SM_RING;
#endif
            for (int i = qs + tid; i < qe; i += BC_SM_NT) {
#if BC_SM_RING
                const int v = v_pf >= 0 ? v_pf : (i - qs < BC_SM_RING ? ring_cur[i - qs] : Q[i]);
#else
                const int v = v_pf >= 0 ? v_pf : Q[i];
#endif
                const int4 row = v_pf >= 0 ? row_pf : ((QROW && L >= 1) ? QR[i] : lowdeg_row<ELL>(p, v));
                v_pf = -1;
                if (BC_SM_PF && !QROW && i + BC_SM_NT < qe) {
                    v_pf = Q[i + BC_SM_NT];
                    row_pf = lowdeg_row<ELL>(p, v_pf);
                }
                if (L >= 1) {
                    double sg = 0.0;
                    lowdeg_row_nbrs<ELL>(p, row, [&](const int *u) {
                        double x[BC_LD_GRP];
#pragma unroll
                        for (int k = 0; k < BC_LD_GRP; ++k) {
                            const bool par = u[k] >= 0 && ((f2[u[k] >> 4] >> ((u[k] & 15) * 2)) & 3u) == cp;
                            x[k] = par ? sc[u[k]] : 0.0;
                            st_dag += par;
                        }
#pragma unroll
                        for (int k = 0; k < BC_LD_GRP; ++k) sg += x[k];
                    });
                    sc[v] = sg;
                }
                lowdeg_row_nbrs<ELL>(p, row, [&](const int *w) {
#if BC_SM_AGG
                    // all test-and-sets of the group first (independent shared atomics),
                    // then one tail atomic per warp for the group's winners
                    bool won[BC_LD_GRP];
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        won[k] = false;
                        if (w[k] >= 0) {
                            const int sh = (w[k] & 15) * 2;
                            won[k] = ((f2[w[k] >> 4] >> sh) & 3u) == 0u &&
                                     ((atomicOr(&f2[w[k] >> 4], cn << sh) >> sh) & 3u) == 0u;
                        }
                    }
                    const unsigned am = __activemask();
                    unsigned bal[BC_LD_GRP];
                    int tot = 0;
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        bal[k] = __ballot_sync(am, won[k]);
                        tot += __popc(bal[k]);
                    }
                    if (tot) {
                        const int leader = __ffs(am) - 1;
                        int base = 0;
                        if (lane == leader) base = qe + atomicAdd(cnt, tot);
                        base = __shfl_sync(am, base, leader);
                        const unsigned lt = (1u << lane) - 1u;
#pragma unroll
                        for (int k = 0; k < BC_LD_GRP; ++k) {
                            if (won[k]) {
                                const int pos = base + __popc(bal[k] & lt);
                                st_slot_stream(Q + pos, w[k]);
#if BC_SM_RING
                                if (pos - qe < BC_SM_RING) ring_nxt[pos - qe] = w[k];
#endif
                                if constexpr (QROW) QR[pos] = p.ell4[w[k]];
                            }
                            base += __popc(bal[k]);
                        }
                    }
#else
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        bool won = false;
                        if (w[k] >= 0) {
                            const int sh = (w[k] & 15) * 2;
                            won = ((f2[w[k] >> 4] >> sh) & 3u) == 0u &&
                                  ((atomicOr(&f2[w[k] >> 4], cn << sh) >> sh) & 3u) == 0u;
                        }
                        const unsigned am = __activemask();
                        const unsigned bal = __ballot_sync(am, won);
                        if (bal) {
                            const int leader = __ffs(bal) - 1;
                            int base = 0;
                            if (lane == leader) base = qe + atomicAdd(cnt, __popc(bal));
                            base = __shfl_sync(am, base, leader);
                            if (won) {
                                const int pos = base + __popc(bal & ((1u << lane) - 1u));
                                st_slot_stream(Q + pos, w[k]);
#if BC_SM_RING
                                if (pos - qe < BC_SM_RING) ring_nxt[pos - qe] = w[k];
#endif
                                if constexpr (QROW) QR[pos] = p.ell4[w[k]];
                            }
                        }
                    }
#endif
                });
            }
            __syncthreads();
            qs = qe;
            qe += *cnt;
            BC_CHECK(qe <= p.n && L + 2 <= p.n + 1);
            r3 = r3n;
            ++L;
            if (tid == 0) lo_set(L + 1, qe);
        }
        const int Lmax = L - 1;
        const int reached = qe;
        const double ws1 = 1.0 + (p.omega ? (double)p.omega[s] : 0.0);
        double ns_loc = 0.0;
        // backward, one barrier per level; each thread's first slot of the
        // next level (vertex, row, sigma) is loaded before the barrier --
        // level L-1 is not written during level L's step
        int a = 0, b = 0, wq = -1;
        int4 rq = make_int4(0, 0, 0, 0);
        double sq = 0.0;
        int wq1 = -1;  // BC_SM_BPF2: level L-1's first-slot vertex, loaded during level L+1
        if (Lmax >= 1) {
            a = lo_get(Lmax);
            b = lo_get(Lmax + 1);
            if (a + tid < b) {
                wq = Q[a + tid];
                rq = QROW ? QR[a + tid] : lowdeg_row<ELL>(p, wq);
                sq = sc[wq];
            }
            if (BC_SM_BPF2 && Lmax - 1 >= 1 && lo_get(Lmax - 1) + tid < lo_get(Lmax)) wq1 = Q[lo_get(Lmax - 1) + tid];
        }
        for (L = Lmax; L >= 1; --L) {
            const unsigned cch = lowdeg_code(L + 1);
#if BC_SM_BPF2
            // level L-1's first slot (row, sigma: final since the forward) is
            // loaded now, alongside level L's work, and level L-2's vertex id
            int4 rq1 = make_int4(0, 0, 0, 0);
            double sq1 = 0.0;
            if (wq1 >= 0) {
                rq1 = lowdeg_row<ELL>(p, wq1);
                sq1 = sc[wq1];
            }
            int wq2 = -1;
            if (L - 2 >= 1 && lo_get(L - 2) + tid < lo_get(L - 1)) wq2 = Q[lo_get(L - 2) + tid];
#endif
            for (int i = a + tid; i < b; i += BC_SM_NT) {
                // the slot's (vertex, row, sigma): loaded before the level's barrier
                // (first slot) or during the previous slot (BC_SM_PF)
                const bool pre = i == a + tid || (BC_SM_PF && !QROW);
                const int w = pre ? wq : Q[i];
                const int4 row = pre ? rq : (QROW ? QR[i] : lowdeg_row<ELL>(p, w));
                const double sg = pre ? sq : sc[w];
                if (BC_SM_PF && !QROW && i + BC_SM_NT < b) {
                    wq = Q[i + BC_SM_NT];
                    rq = lowdeg_row<ELL>(p, wq);
                    sq = sc[wq];
                }
                double acc = 0.0;
                lowdeg_row_nbrs<ELL>(p, row, [&](const int *v) {
                    double x[BC_LD_GRP];
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        const bool ch = v[k] >= 0 && ((f2[v[k] >> 4] >> ((v[k] & 15) * 2)) & 3u) == cch;
                        x[k] = ch ? sc[v[k]] : 0.0;
                    }
#pragma unroll
                    for (int k = 0; k < BC_LD_GRP; ++k) {
                        acc += x[k];
                        st_adj += v[k] >= 0;
                    }
                });
                const double om = p.omega ? (double)p.omega[w] : 0.0;
                const double delta = sg * acc;
                sc[w] = (1.0 + om + delta) / sg;
                slices_cap<CAP>(p, cs, w, L, sg, delta);
                const double c = ws1 * (delta + om);
                if (c != 0.0) atomicAdd(p.bc + w, c);
                st_dsum += (unsigned long long)L;
                ns_loc += 1.0 + om;
            }
            const int an = lo_get(L - 1), bn = lo_get(L);
#if BC_SM_BPF2
            wq = wq1;
            rq = rq1;
            sq = sq1;
            wq1 = wq2;
#else
            wq = -1;
            if (L - 1 >= 1 && an + tid < bn) {
                wq = Q[an + tid];
                rq = QROW ? QR[an + tid] : lowdeg_row<ELL>(p, wq);
                sq = sc[wq];
            }
#endif
            __syncthreads();
            a = an;
            b = bn;
        }
        st_reach += (tid == 0) ? (unsigned long long)reached : 0ull;
        if (tid == 0) {
            st_adj += (unsigned long long)(p.rp[s + 1] - p.rp[s]);
            ns_loc += ws1;
        }
        ns_loc = warp_sum(ns_loc);
        if (lane == 0) sm.red[warp_id()] = ns_loc;
        if (reached >= nw / 4) {
            for (int i = tid; i < nw; i += BC_SM_NT) f2[i] = 0u;
        } else {
            for (int i = tid; i < reached; i += BC_SM_NT) f2[Q[i] >> 4] = 0u;
        }
        __syncthreads();
        if (tid == 0 && p.omega) {
            double ns = 0.0;
            for (int w = 0; w < BC_SM_NT / 32; ++w) ns += sm.red[w];
            const double om = (double)p.omega[s];
            if (om != 0.0) atomicAdd(p.bc + s, om * (ns - 2.0));
        }
        __syncthreads();
    }
    const unsigned long long a = warp_sum_u64(st_reach), b = warp_sum_u64(st_adj), c = warp_sum_u64(st_dag),
                             d = warp_sum_u64(st_dsum);
    if (lane == 0) {
        if (a) atomicAdd(p.stats + 0, a);
        if (b) atomicAdd(p.stats + 1, b);
        if (c) atomicAdd(p.stats + 2, c);
        if (d) atomicAdd(p.stats + 3, d);
    }
}

// bc[v] += sum over CTAs of the private rows (and clears them)
__global__ void slices_reduce_kernel(int n, int nrows, double *bcp, double *bc) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    double s = 0.0;
    for (int r = 0; r < nrows; ++r) {
        double *q = bcp + (size_t)r * n + v;
        s += *q;
        *q = 0.0;
    }
    bc[v] += s;
}

__global__ void fill_int_kernel(int *p, size_t cnt, int v) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) p[i] = v;
}

}  // namespace bcb

namespace bcb {
// ell[v] = the (<= 4) neighbours of v, padded with -1
__global__ void build_ell4_kernel(int n, const int *rp, const int *col, int4 *ell) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int a = rp[v], d = rp[v + 1] - a;
    int4 q;
    q.x = d > 0 ? col[a] : -1;
    q.y = d > 1 ? col[a + 1] : -1;
    q.z = d > 2 ? col[a + 2] : -1;
    q.w = d > 3 ? col[a + 3] : -1;
    ell[v] = q;
}
}  // namespace bcb
