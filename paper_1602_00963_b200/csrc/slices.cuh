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
    double *bcp;            // private BC rows
    unsigned *bm;           // global bitmaps [gridDim.x][2][bm_words] (when not in shared memory)
    int bm_words;
    unsigned long long *stats;  // [4] reached, adjacency, dag edges, depth sum
};

struct SlicesSmem {
    int cd[BC_NT + 1];
    int vs[BC_NT];
    int rs[BC_NT];
    int scan[2 * BC_NW + 2];
    int tail;
    int src;
    double red[32];
};

// Process the items of frontier chunk Q[c0, c1) (<= BC_NT vertices); calls
// f(v, w) for every item.
template <typename F>
__device__ __forceinline__ void slices_chunk_items(const SlicesParams &p, SlicesSmem &sm, const int *Q, int c0,
                                                   int c1, F &&f) {
    const int i = threadIdx.x;
    int deg = 0, v = -1, rs = 0;
    if (c0 + i < c1) {
        v = Q[c0 + i];
        rs = p.rp[v];
        deg = p.rp[v + 1] - rs;
    }
    int ex, d1, tot, d2;
    block_excl_scan2(deg, 0, ex, d1, tot, d2, sm.scan);
    const int nv = c1 - c0;
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

template <bool SMEM_BM>
__global__ void __launch_bounds__(BC_NT) slices_kernel(SlicesParams p) {
    __shared__ SlicesSmem sm;
    extern __shared__ unsigned smbm[];  // 2 * SLICES_SMEM_BM_WORDS when SMEM_BM
    const size_t n = (size_t)p.n;
    double *sigma = p.sigma + blockIdx.x * n;
    double *cf = p.cf + blockIdx.x * n;
    int *Q = p.queue + blockIdx.x * n;
    int *loff = p.loff + blockIdx.x * (n + 2);
    double *bcp = p.bcp + blockIdx.x * n;
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
                slices_chunk_items(p, sm, Q, c0, c1, [&](int v, int w) {
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
                });
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
                    slices_chunk_items(p, sm, Q, c0, c1, [&](int w, int v) {
                        if (lvb[v >> 5] & (1u << (v & 31))) atomicAdd(&cf[w], cf[v]);
                    });
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
// binary search), and no floating-point atomics at all -- discovery pushes
// only bits (visited bitmap + queue append), sigma is then *pulled* by each
// newly discovered vertex from its level-L neighbours (Alg.1 lines 16-19 read
// from the child's side), and the backward step pulls coef from the level-(L+1)
// neighbours.  Level membership is two bitmaps (levels L and L+1).
constexpr int BC_LOWDEG = 64;
#ifndef BC_SL_NT
#define BC_SL_NT 256  // threads per CTA of the degree-bounded slices kernel (more sources in flight)
#endif

__global__ void __launch_bounds__(BC_SL_NT, 1) slices_lowdeg_kernel(SlicesParams p) {
    __shared__ SlicesSmem sm;
    const size_t n = (size_t)p.n;
    double *sigma = p.sigma + blockIdx.x * n;
    double *cf = p.cf + blockIdx.x * n;
    int *Q = p.queue + blockIdx.x * n;
    int *loff = p.loff + blockIdx.x * (n + 2);
    double *bcp = p.bcp + blockIdx.x * n;
    unsigned *vis = p.bm + (size_t)blockIdx.x * 3 * p.bm_words;
    unsigned *lb0 = vis + p.bm_words;      // level bitmaps, alternating
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
        if (threadIdx.x == 0) {
            atomicOr(&vis[s >> 5], 1u << (s & 31));
            atomicOr(&lb0[s >> 5], 1u << (s & 31));
            sigma[s] = 1.0;
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
                const int a = p.rp[v], b = p.rp[v + 1];
                for (int e = a; e < b; ++e) {
                    const int w = p.col[e];
                    const unsigned bit = 1u << (w & 31);
                    if (!(vis[w >> 5] & bit) && !(atomicOr(&vis[w >> 5], bit) & bit)) {
                        atomicOr(&lnxt[w >> 5], bit);
                        Q[atomicAdd(&sm.tail, 1)] = w;
                    }
                }
            }
            __syncthreads();
            const int ne = sm.tail;
            // (2) sigma pull: each new vertex sums sigma of its level-L neighbours
            for (int i = qe + threadIdx.x; i < ne; i += BC_SL_NT) {
                const int w = Q[i];
                const int a = p.rp[w], b = p.rp[w + 1];
                double sg = 0.0;
                for (int e = a; e < b; ++e) {
                    const int v = p.col[e];
                    if (lcur[v >> 5] & (1u << (v & 31))) {
                        sg += sigma[v];
                        ++st_dag;
                    }
                }
                sigma[w] = sg;
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
        // lcur holds the (empty) last level; clear nothing more
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
                const int ea = p.rp[w], eb = p.rp[w + 1];
                for (int e = ea; e < eb; ++e) {
                    const int v = p.col[e];
                    if (lb0[v >> 5] & (1u << (v & 31))) acc += cf[v];
                }
                const double om = p.omega ? (double)p.omega[w] : 0.0;
                const double sg = sigma[w];
                const double delta = sg * acc;
                cf[w] = (1.0 + om + delta) / sg;
                const double c = ws1 * (delta + om);
                if (c != 0.0) bcp[w] += c;
                st_dsum += (unsigned long long)L;
            }
            __syncthreads();
            for (int i = a1 + threadIdx.x; i < b1; i += BC_SL_NT) {
                const int v = Q[i];
                atomicAnd(&lb0[v >> 5], ~(1u << (v & 31)));
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < reached; i += BC_SL_NT) {
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
            for (int w = 0; w < BC_SL_NT / 32; ++w) ns += sm.red[w];
            const double om = (double)p.omega[s];
            if (om != 0.0) bcp[s] += om * (ns - 2.0);
        }
        for (int i = threadIdx.x; i < reached; i += BC_SL_NT) {
            const int w = Q[i];
            vis[w >> 5] = 0u;
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
