/*
 * graphgen.c — seeded synthetic input generators shared by the CUDA path's
 * tests/bench and by the oracle's tests.  This module holds NONE of the
 * method's arithmetic (no BFS, no sigma, no dependencies): it only produces
 * simple undirected graphs in CSR form.
 *
 *   R-MAT (Sec. 4.1): n = 2^scale vertices, exactly
 *     2^scale * EF sampled pairs by recursive quadrant selection with
 *     probabilities (a,b,c,d) = (0.57, 0.19, 0.19, 0.05).  Every draw is a
 *     counter-based splitmix64 hash of (seed, edge index, level), so the
 *     output is independent of the thread count.  A seeded bijective label
 *     permutation (Graph500 convention) is optional.
 *   grid(R, C): 4-neighbour lattice, id = r*C + c, no wrap (road-network-like
 *     long-diameter workload, SURVEY.md §8 d-i config 2).
 *   normalize: drop self-loops, symmetrize, merge duplicates, sort each
 *     adjacency list ascending.
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC graphgen.c -o libgraphgen.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* splitmix64 evaluated at counter `key` of the stream selected by `seed`. */
static inline uint64_t draw(uint64_t seed, uint64_t key) {
    return mix64(mix64(seed) + (key + 1) * 0x9E3779B97F4A7C15ULL);
}

static inline double u01(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

/* Seeded bijection on [0, 2^scale): three rounds of (odd multiply + add) mod
 * 2^scale followed by an xorshift; each step is invertible. */
static inline uint32_t permute_label(uint32_t x, int scale, uint64_t seed) {
    if (scale <= 0) return x;
    uint64_t mask = (scale >= 64) ? ~0ULL : ((1ULL << scale) - 1ULL);
    uint64_t y = x;
    for (int r = 0; r < 3; ++r) {
        uint64_t k = draw(seed ^ 0x5eedULL, (uint64_t)r);
        uint64_t mul = (k | 1ULL) & mask;
        if (mul == 0) mul = 1;
        uint64_t add = (k >> 32) & mask;
        y = (y * mul + add) & mask;
        int sh = scale / 2 + 1;
        y ^= (y >> sh);
        y &= mask;
    }
    return (uint32_t)y;
}

/* Emit exactly nedges = 2^scale * ef directed pairs (u[e], v[e]). */
int gg_rmat_edges(int scale, int64_t ef, double a, double b, double c, uint64_t seed,
                  int permute, int32_t *u, int32_t *v) {
    if (scale < 1 || scale > 30 || ef < 1) return 1;
    int64_t nedges = ((int64_t)1 << scale) * ef;
    double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < nedges; ++e) {
        uint32_t uu = 0, vv = 0;
        for (int lvl = 0; lvl < scale; ++lvl) {
            double r = u01(draw(seed, ((uint64_t)e << 6) | (uint64_t)lvl));
            uint32_t bit = 1u << (scale - 1 - lvl);
            if (r < a) {
            } else if (r < ab) {
                vv |= bit;
            } else if (r < abc) {
                uu |= bit;
            } else {
                uu |= bit;
                vv |= bit;
            }
        }
        if (permute) {
            uu = permute_label(uu, scale, seed);
            vv = permute_label(vv, scale, seed);
        }
        u[e] = (int32_t)uu;
        v[e] = (int32_t)vv;
    }
    return 0;
}

static int cmp_i32(const void *x, const void *y) {
    int32_t a = *(const int32_t *)x, b = *(const int32_t *)y;
    return (a > b) - (a < b);
}

/* In-place LSD radix sort of a small int32 array of non-negative values
 * (falls back to qsort for short rows). */
static void sort_row(int32_t *p, int64_t len, int32_t *tmp) {
    if (len < 2) return;
    if (len < 256) {
        qsort(p, (size_t)len, sizeof(int32_t), cmp_i32);
        return;
    }
    int32_t *src = p, *dst = tmp;
    for (int pass = 0; pass < 4; ++pass) {
        int64_t cnt[257];
        memset(cnt, 0, sizeof(cnt));
        int sh = pass * 8;
        for (int64_t i = 0; i < len; ++i) cnt[((uint32_t)src[i] >> sh & 0xFF) + 1]++;
        for (int i = 0; i < 256; ++i) cnt[i + 1] += cnt[i];
        for (int64_t i = 0; i < len; ++i) dst[cnt[(uint32_t)src[i] >> sh & 0xFF]++] = src[i];
        int32_t *t = src; src = dst; dst = t;
    }
    /* after 4 passes the data is back in p */
}

/*
 * Normalize an edge list into a simple undirected CSR.
 * Pass 1 (out_row_ptr != NULL, out_col == NULL): computes row_ptr (n+1) and
 *   returns the number of directed entries through *out_nnz; the deduplicated
 *   column data is kept in an internal buffer handed back via *handle.
 * Simpler single-call API: caller provides out_col with capacity 2*nedges.
 */
int gg_normalize(int64_t n, int64_t nedges, const int32_t *u, const int32_t *v,
                 int64_t *row_ptr /* [n+1] out */, int32_t *col /* cap 2*nedges out */,
                 int64_t *out_nnz) {
    if (n <= 0) return 1;
    for (int64_t e = 0; e < nedges; ++e)
        if (u[e] < 0 || u[e] >= n || v[e] < 0 || v[e] >= n) return 2;
    int64_t *deg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!deg) return 3;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < nedges; ++e) {
        if (u[e] == v[e]) continue;
#pragma omp atomic
        deg[u[e]]++;
#pragma omp atomic
        deg[v[e]]++;
    }
    int64_t *pos = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    if (!pos) { free(deg); return 3; }
    pos[0] = 0;
    for (int64_t i = 0; i < n; ++i) pos[i + 1] = pos[i] + deg[i];
    int64_t total = pos[n];
    int32_t *buf = (int32_t *)malloc((size_t)(total > 0 ? total : 1) * sizeof(int32_t));
    int64_t *fill = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    if (!buf || !fill) { free(deg); free(pos); free(buf); free(fill); return 3; }
    memcpy(fill, pos, ((size_t)n + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < nedges; ++e) {
        int32_t a = u[e], b = v[e];
        if (a == b) continue;
        int64_t p, q;
#pragma omp atomic capture
        p = fill[a]++;
#pragma omp atomic capture
        q = fill[b]++;
        buf[p] = b;
        buf[q] = a;
    }
    free(fill);
    /* sort + dedup each row; new degree into deg[] */
#pragma omp parallel
    {
        int64_t cap = 0;
        int32_t *tmp = NULL;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n; ++i) {
            int64_t len = pos[i + 1] - pos[i];
            if (len > cap) {
                free(tmp);
                cap = len * 2;
                tmp = (int32_t *)malloc((size_t)cap * sizeof(int32_t));
            }
            int32_t *p = buf + pos[i];
            sort_row(p, len, tmp);
            int64_t k = 0;
            for (int64_t j = 0; j < len; ++j)
                if (k == 0 || p[j] != p[k - 1]) p[k++] = p[j];
            deg[i] = k;
        }
        free(tmp);
    }
    row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + deg[i];
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i)
        memcpy(col + row_ptr[i], buf + pos[i], (size_t)deg[i] * sizeof(int32_t));
    *out_nnz = row_ptr[n];
    free(buf);
    free(pos);
    free(deg);
    return 0;
}

/* 4-neighbour R x C grid, id = r*C + c; adjacency emitted sorted. */
int gg_grid(int64_t R, int64_t C, int64_t *row_ptr, int32_t *col) {
    if (R <= 0 || C <= 0) return 1;
    int64_t n = R * C;
    row_ptr[0] = 0;
    for (int64_t id = 0; id < n; ++id) {
        int64_t r = id / C, c = id % C;
        int64_t d = (r > 0) + (c > 0) + (c + 1 < C) + (r + 1 < R);
        row_ptr[id + 1] = row_ptr[id] + d;
    }
#pragma omp parallel for schedule(static)
    for (int64_t id = 0; id < n; ++id) {
        int64_t r = id / C, c = id % C, k = row_ptr[id];
        if (r > 0) col[k++] = (int32_t)(id - C);
        if (c > 0) col[k++] = (int32_t)(id - 1);
        if (c + 1 < C) col[k++] = (int32_t)(id + 1);
        if (r + 1 < R) col[k++] = (int32_t)(id + C);
    }
    return 0;
}

/* Uniform sample of `count` distinct vertices with degree > 0, without
 * replacement (PAPER.md:840 footnote: "selected randomly among not isolated
 * vertices").  Partial Fisher-Yates over the eligible list, seeded draws. */
int gg_sample_sources(int64_t n, const int64_t *row_ptr, int64_t count, uint64_t seed,
                      int32_t *out) {
    int32_t *elig = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!elig) return 3;
    int64_t ne = 0;
    for (int64_t i = 0; i < n; ++i)
        if (row_ptr[i + 1] > row_ptr[i]) elig[ne++] = (int32_t)i;
    if (count > ne) { free(elig); return 1; }
    for (int64_t i = 0; i < count; ++i) {
        uint64_t r = draw(seed ^ 0xA5A5A5A5ULL, (uint64_t)i);
        int64_t j = i + (int64_t)(r % (uint64_t)(ne - i));
        int32_t t = elig[i]; elig[i] = elig[j]; elig[j] = t;
        out[i] = elig[i];
    }
    free(elig);
    return 0;
}

int gg_num_threads(void) { return omp_get_max_threads(); }
