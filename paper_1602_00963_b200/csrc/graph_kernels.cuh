// graph_kernels.cuh -- device-side graph setup: CSR conversion and
// validation, 1-degree pruning (Alg.6) and the hub list.
#pragma once
#include "util.cuh"

namespace bcb {

__global__ void rp64_to_32_kernel(const long long *rp64, int *rp32, long long n1) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n1) rp32[i] = (int)rp64[i];
}

// BC_CREATE_VALIDATE: rows strictly ascending, in range, no self-loops,
// symmetric (binary search of v in adj(u)).  err |= bit on failure.
__global__ void validate_kernel(int n, const int *rp, const int *col, int *err) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    if (gw >= n) return;
    const int v = gw;
    const int a = rp[v], b = rp[v + 1];
    int bad = 0;
    if (b < a) bad |= 1;
    for (int e = a + lane; e < b; e += 32) {
        const int u = col[e];
        if (u < 0 || u >= n) { bad |= 2; continue; }
        if (u == v) bad |= 4;
        if (e > a && col[e - 1] >= u) bad |= 8;
        int lo = rp[u], hi = rp[u + 1] - 1, found = 0;
        while (lo <= hi) {
            int mid = (lo + hi) >> 1;
            int c = col[mid];
            if (c == v) { found = 1; break; }
            if (c < v) lo = mid + 1;
            else hi = mid - 1;
        }
        if (!found) bad |= 16;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicOr(err, bad);
}

// Alg.6 lines 3-9: u with a single edge is removed (R), omega of its
// neighbour incremented.  Warp per vertex v: omega(v) = #neighbours of
// degree 1; residual degree = #neighbours kept (0 if v itself is removed).
__global__ void prune_count_kernel(int n, const int *rp, const int *col, uint32_t *omega, uint8_t *removed,
                                   int *rdeg) {
    const int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    if (v >= n) return;
    const int a = rp[v], b = rp[v + 1];
    const bool self_removed = (b - a) == 1;
    int om = 0, keep = 0;
    for (int e = a + lane; e < b; e += 32) {
        const int u = col[e];
        const bool u_removed = (rp[u + 1] - rp[u]) == 1;
        om += u_removed;
        keep += !u_removed;
    }
    om = __reduce_add_sync(0xffffffffu, om);
    keep = __reduce_add_sync(0xffffffffu, keep);
    if (lane == 0) {
        omega[v] = (uint32_t)om;
        removed[v] = self_removed ? 1 : 0;
        rdeg[v] = self_removed ? 0 : keep;
    }
}

// Alg.6 lines 10-11 + PAPER.md:590-591: residual edge list E' keeps (u,v)
// when neither endpoint was removed (removed[] of the whole graph: this
// device's pass, or the sum of the processors' shares); order within a row
// is preserved.
__global__ void prune_compact_kernel(int n, const int *rp, const int *col, const uint8_t *removed, const int *rrp,
                                     int *rcol) {
    const int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    if (v >= n) return;
    const int a = rp[v], b = rp[v + 1];
    if (removed[v]) return;  // removed vertex: empty residual row
    int out = rrp[v];
    for (int e0 = a; e0 < b; e0 += 32) {
        const int e = e0 + lane;
        int u = 0;
        bool keep = false;
        if (e < b) {
            u = col[e];
            keep = !removed[u];
        }
        unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) rcol[out + __popc(m & ((1u << lane) - 1u))] = u;
        out += __popc(m);
    }
}

// Alg.6 on processor `rank` of `nranks` (the
// 1-D split "u mod #P = P_i"): thread per vertex u of this share; u with a
// single edge (u,v) is removed and omega(v) incremented.  The outputs are
// zero-initialised by the caller; their sums over the ranks are the
// single-pass omega and removed flags.
__global__ void prune_share_kernel(int n, const int *rp, const int *col, int rank, int nranks, uint32_t *omega_part,
                                   uint32_t *removed_part) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long u = i * nranks + rank;
    if (u >= n) return;
    const int a = rp[u], b = rp[u + 1];
    if (b - a == 1) {
        removed_part[u] = 1u;
        atomicAdd(omega_part + col[a], 1u);
    }
}

// From the exchanged (summed) flags: removed as bytes, residual degrees, and
// a consistency check -- a vertex is removed exactly when its degree is 1
// (every share counted once); err |= 1 otherwise.  Warp per vertex.
__global__ void prune_flags_kernel(int n, const int *rp, const int *col, const uint32_t *removed_sum,
                                   uint8_t *removed, int *rdeg, int *err) {
    const int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    if (v >= n) return;
    const int a = rp[v], b = rp[v + 1];
    const uint32_t rv = removed_sum[v];
    int keep = 0;
    for (int e = a + lane; e < b; e += 32) {
        const int u = col[e];
        keep += removed_sum[u] == 0u;
    }
    keep = __reduce_add_sync(0xffffffffu, keep);
    if (lane == 0) {
        if (rv > 1u || (rv == 1u) != (b - a == 1)) atomicOr(err, 1);
        removed[v] = rv ? 1 : 0;
        rdeg[v] = rv ? 0 : keep;
    }
}

// --- exclusive scan of int (values and total < 2^31), three phases
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = BC_NT * SCAN_ITEMS;

__global__ void __launch_bounds__(BC_NT) scan_tiles_kernel(const int *in, int *out, int *tile_sums, long long n) {
    __shared__ int sm[2 * BC_NW + 2];
    const long long base = (long long)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS], s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        s += v[i];
    }
    int ex, dummy, tot, dt;
    block_excl_scan2(s, 0, ex, dummy, tot, dt, sm);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = ex;
        ex += v[i];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(BC_NT) scan_sums_kernel(int *sums, int nt, int *total) {
    __shared__ int sm[2 * BC_NW + 2];
    int carry = 0;
    for (int base = 0; base < nt; base += BC_NT) {
        int i = base + threadIdx.x;
        int v = i < nt ? sums[i] : 0;
        int ex, d, tot, dt;
        block_excl_scan2(v, 0, ex, d, tot, dt, sm);
        if (i < nt) sums[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void scan_add_kernel(int *out, const int *sums, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += sums[i / SCAN_TILE];
}

// hubs: vertices of degree > hub_deg; flags for a scan-based compaction
__global__ void hub_flag_kernel(int n, const int *rp, int hub_deg, int *flag) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) flag[v] = (rp[v + 1] - rp[v]) > hub_deg ? 1 : 0;
}

__global__ void hub_scatter_kernel(int n, const int *flag, const int *pos, int *hub_ids) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n && flag[v]) hub_ids[pos[v]] = v;
}

__global__ void hub_segcount_kernel(int nhub, const int *hub_ids, const int *rp, int seg_len, int *cnt) {
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h < nhub) {
        const int x = hub_ids[h];
        const int d = rp[x + 1] - rp[x];
        cnt[h] = (d + seg_len - 1) / seg_len;
    }
}

}  // namespace bcb

namespace bcb {

// --- degree-descending relabelling of the compute CSR:
// hubs get the lowest ids, so their sigma/coef rows are contiguous at the
// front of S (L2-friendly) and tiles can be cut by item count.
__global__ void relabel_keys_kernel(int n, const int *rp, int maxdeg, unsigned *keys, int *vals) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) {
        keys[v] = (unsigned)(maxdeg - (rp[v + 1] - rp[v]));
        vals[v] = v;
    }
}

__global__ void invert_perm_kernel(int n, const int *perm, int *inv) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) inv[perm[i]] = i;
}

__global__ void permuted_degree_kernel(int n, const int *perm, const int *rp, int *deg_new) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) deg_new[i] = rp[perm[i] + 1] - rp[perm[i]];
}

// warp per new vertex i: row i of the new CSR = inv-mapped row perm[i]
__global__ void relabel_cols_kernel(int n, const int *perm, const int *inv, const int *rp, const int *col,
                                    const int *rp_new, int *col_new) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const int u = perm[i];
    const int a = rp[u], b = rp[u + 1], o = rp_new[i];
    for (int e = a + lane_id(); e < b; e += 32) col_new[o + (e - a)] = inv[col[e]];
}

__global__ void gather_u32_kernel(int n, const int *perm, const uint32_t *src, uint32_t *dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

__global__ void map_ids_kernel(long long cnt, const int *inv, const int *in, int *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) out[i] = inv[in[i]];
}

// Batch scheduling key of a source (compute ids; smaller id = higher degree):
// its highest-degree closed neighbour.  Sources sharing that anchor are at
// distance <= 2, so their BFS depth profiles differ by <= 2 everywhere and a
// batch of them keeps its lanes in step (dense level masks, few levels).
__global__ void anchor_key_kernel(const int *src, int ns, const int *rp, const int *col, unsigned long long *key,
                                  int two_level) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= ns) return;
    const int s = src[i];
    int m = s;
    for (int e = rp[s] + lane_id(); e < rp[s + 1]; e += 32) m = min(m, col[e]);
    m = __reduce_min_sync(0xffffffffu, m);
    // second anchor: the next highest-degree closed neighbour (sub-clusters)
    int m2 = 0x7fffffff;
    if (two_level) {
        if (s != m) m2 = s;
        for (int e = rp[s] + lane_id(); e < rp[s + 1]; e += 32) {
            const int c = col[e];
            if (c != m) m2 = min(m2, c);
        }
        m2 = __reduce_min_sync(0xffffffffu, m2);
    }
    if (lane_id() == 0) key[i] = ((unsigned long long)(unsigned)m << 32) | (unsigned)(two_level ? m2 : 0);
}

// out[v] (original label) = bc_new[inv[v]]
__global__ void unpermute_kernel(int n, const int *inv, const double *bc_new, double *out) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) out[v] = bc_new[inv[v]];
}

// ---- verification capture (bc_set_capture / bc_sssp) --------------------
// [ncap][n] arrays from compute ids to original ids: out[c][v] = in[c][inv[v]]
template <typename T>
__global__ void cap_unpermute_kernel(long long ncap, int n, const int *inv, const T *in, T *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncap * n) return;
    const long long c = i / n;
    const int v = (int)(i - c * n);
    out[i] = in[c * n + inv[v]];
}

// every captured source s (original ids): d(s, s) = 0, sigma_ss = 1 (also
// for residual-isolated sources, which are not traversed, R10)
template <typename ST>
__global__ void cap_sources_kernel(int ncap, int n, const int *src, int *depth, ST *sigma) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncap) return;
    depth[(size_t)c * n + src[c]] = 0;
    sigma[(size_t)c * n + src[c]] = ST(1);
}

// Pruned handle (original ids): turn the residual traversal's per-source
// state into the unpruned graph's (R13).  A removed vertex u hangs off its
// single neighbour p, so d(s, u) = d(s, p) + 1, sigma_su = sigma_sp and
// delta_s(u) = 0 (u lies on no shortest path between other vertices); a
// kept vertex v != s reached by s has delta_s(v) = delta'_s(v) + omega(v)
// (Eq.(5): each of v's removed children adds a pair dependency of 1).  A
// removed u whose neighbour is removed too (a K2) is not reachable from a
// kept source.  Kept vertices' depth / sigma are only read here, removed
// ones only written, so one pass suffices.
template <typename ST>
__global__ void cap_prune_fill_kernel(long long ncap, int n, const int *rp, const int *col, const uint8_t *removed,
                                      const uint32_t *omega, int *depth, ST *sigma, double *delta, uint8_t *ovf) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncap * n) return;
    const long long c = i / n;
    const int u = (int)(i - c * n);
    const size_t base = (size_t)c * n;
    if (removed[u]) {
        const int par = col[rp[u]];
        const int dp = removed[par] ? -1 : depth[base + par];
        depth[i] = dp >= 0 ? dp + 1 : -1;
        sigma[i] = dp >= 0 ? sigma[base + par] : ST(0);
        if (ovf) ovf[i] = dp >= 0 ? ovf[base + par] : 0;
        if (delta) delta[i] = 0.0;
    } else if (delta && depth[i] > 0) {
        delta[i] += (double)omega[u];
    }
}

}  // namespace bcb
