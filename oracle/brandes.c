/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the BC hot path.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code, header or
 * constant with the CUDA path (paper_1602_00963_b200/), and the CUDA path
 * never calls it.
 *
 * Every routine follows the paper's text in the paper's order:
 *
 *  brandes_source   Alg.1 "Brandes' algorithm": queue BFS
 *                   from s giving d and sigma, predecessor lists P[w], the
 *                   dequeue order as the stack S, then the backward pops with
 *                   delta[v] += sigma[v]/sigma[w] * (1 + delta[w])   (Eq.2,
 *                   PAPER.md:101-104).  With omega != NULL the recursion is
 *                   Eq.(5) line 1:
 *                   delta[v] += sigma[v]/sigma[w] * (1 + delta[w] + omega[w]).
 *                   Reading §8c-1 (R1): the garbled backward loop is
 *                   read as "pop w; for v in P[w] ...; if w != s BC[w] += delta[w]".
 *                   sigma is kept twice: uint64 with a sticky overflow flag
 *                   (exact integer parity) and fp64 (used for delta).
 *  oracle_bc        Eq.(3): BC(v) = sum_{s in S, s != v}
 *                   delta_s(v), unnormalised ordered pairs (reading R14).
 *  oracle_prune_degree1   Alg.6 "1-Degree Preprocessing",
 *  oracle_prune_degree1_share  Alg.6 on processor i of #P (u mod #P split),
 *                   single processor, one pass, no cascade (PAPER.md:580 fn.).
 *  oracle_bc_pruned Eq.(4)/(5) with the readings R7-R13 of DESIGN.md
 *                   (omega taken before each increment; n_s = sum over reached
 *                   (1+omega); trivial sources; source-attributed form).
 *
 * Parity pins for every routine live in tests/test_oracle_*.py (brute-force
 * exact rationals, closed forms, invariants).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC brandes.c -o liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct {
    int32_t *d;        /* depth, -1 = unreached                          */
    uint64_t *sig;     /* sigma as an integer                           */
    uint8_t *ovf;      /* sticky: sigma overflowed uint64                */
    double *sigf;      /* sigma as fp64                                  */
    double *delta;     /* dependency                                    */
    int32_t *queue;    /* BFS queue; dequeue order is the stack S       */
    int32_t *pcnt;     /* |P[w]|                                         */
    int32_t *pred;     /* P[w] stored at pred[row_ptr[w] .. + pcnt[w])  */
} work_t;

static int work_alloc(work_t *w, int64_t n, int64_t nnz) {
    w->d = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    w->sig = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    w->ovf = (uint8_t *)malloc((size_t)n);
    w->sigf = (double *)malloc(sizeof(double) * (size_t)n);
    w->delta = (double *)malloc(sizeof(double) * (size_t)n);
    w->queue = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    w->pcnt = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    w->pred = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    if (!w->d || !w->sig || !w->ovf || !w->sigf || !w->delta || !w->queue || !w->pcnt || !w->pred)
        return 1;
    for (int64_t v = 0; v < n; ++v) w->d[v] = -1;
    return 0;
}

static void work_free(work_t *w) {
    free(w->d); free(w->sig); free(w->ovf); free(w->sigf);
    free(w->delta); free(w->queue); free(w->pcnt); free(w->pred);
}

/* Alg.1 for one source.  Returns the number of reached vertices (queue
 * length).  On return d/sig/ovf/sigf/delta hold the round's values for the
 * reached vertices; unreached vertices keep d = -1 (their other fields are
 * unspecified).  stats (nullable): [0] n_s reached, [1] A_s = sum of degrees
 * over reached, [2] D_s = number of DAG edges (sum of |P[w]|). */
static int64_t brandes_source(int64_t n, const int64_t *rp, const int32_t *col, int32_t s,
                              const uint32_t *omega, work_t *w, int64_t *stats) {
    (void)n;
    /* Pred[v] <- NULL, sigma[v] <- 0, d[v] <- -1  (d is reset lazily below) */
    int64_t head = 0, tail = 0;
    w->sig[s] = 1; w->ovf[s] = 0; w->sigf[s] = 1.0; w->d[s] = 0; w->pcnt[s] = 0;
    w->queue[tail++] = s;                           /* enqueue s -> Q */
    int64_t A = 0, D = 0;
    while (head < tail) {                           /* while Q not empty */
        int32_t v = w->queue[head++];               /* dequeue v; push v -> S */
        A += rp[v + 1] - rp[v];
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {   /* neighbours w of v */
            int32_t x = col[e];
            if (w->d[x] < 0) {                      /* if d[w] < 0 */
                w->queue[tail++] = x;               /*   enqueue w */
                w->d[x] = w->d[v] + 1;              /*   d[w] <- d[v] + 1 */
                w->sig[x] = 0; w->ovf[x] = 0; w->sigf[x] = 0.0; w->pcnt[x] = 0;
            }
            if (w->d[x] == w->d[v] + 1) {           /* if d[w] = d[v] + 1 */
                uint64_t r;
                if (__builtin_add_overflow(w->sig[x], w->sig[v], &r)) w->ovf[x] = 1;
                w->sig[x] = r;                      /*   sigma[w] += sigma[v] */
                w->ovf[x] |= w->ovf[v];
                w->sigf[x] += w->sigf[v];
                w->pred[rp[x] + w->pcnt[x]++] = v;  /*   append v -> P[w] */
                D++;
            }
        }
    }
    for (int64_t i = 0; i < tail; ++i) w->delta[w->queue[i]] = 0.0;  /* delta[v] <- 0 */
    for (int64_t i = tail - 1; i >= 0; --i) {       /* while S not empty: pop w */
        int32_t x = w->queue[i];
        double coef = 1.0 + w->delta[x] + (omega ? (double)omega[x] : 0.0);
        for (int32_t k = 0; k < w->pcnt[x]; ++k) {  /* for v in P[w] */
            int32_t v = w->pred[rp[x] + k];
            w->delta[v] += w->sigf[v] / w->sigf[x] * coef;
        }
    }
    if (stats) { stats[0] = tail; stats[1] = A; stats[2] = D; }
    return tail;
}

static void reset_reached(work_t *w, int64_t reached) {
    for (int64_t i = 0; i < reached; ++i) w->d[w->queue[i]] = -1;
}

static int pick_threads(int nthreads) {
    int t = nthreads > 0 ? nthreads : omp_get_max_threads();
    return t < 1 ? 1 : t;
}

/* Eq.(3): bc[v] = sum over s in sources, s != v, of delta_s(v).  bc is
 * overwritten.  stats (nullable) is [ns][3] as in brandes_source. */
int oracle_bc(int64_t n, const int64_t *rp, const int32_t *col, const int32_t *sources,
              int64_t ns, int nthreads, double *bc, int64_t *stats) {
    int T = pick_threads(nthreads);
    double *part = (double *)calloc((size_t)T * (size_t)n, sizeof(double));
    if (!part) return 3;
    int err = 0;
#pragma omp parallel num_threads(T)
    {
        int tid = omp_get_thread_num();
        double *mine = part + (size_t)tid * (size_t)n;
        work_t w;
        if (work_alloc(&w, n, rp[n])) {
#pragma omp atomic write
            err = 3;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t i = 0; i < ns; ++i) {
                int32_t s = sources[i];
                int64_t reached = brandes_source(n, rp, col, s, NULL, &w, stats ? stats + 3 * i : NULL);
                for (int64_t k = 0; k < reached; ++k) {
                    int32_t x = w.queue[k];
                    if (x != s) mine[x] += w.delta[x];   /* if w != s: BC[w] += delta[w] */
                }
                reset_reached(&w, reached);
            }
        }
        work_free(&w);
    }
    if (!err) {
        for (int64_t v = 0; v < n; ++v) {
            double acc = 0.0;
            for (int t = 0; t < T; ++t) acc += part[(size_t)t * (size_t)n + v];
            bc[v] = acc;
        }
    }
    free(part);
    return err;
}

/* Per-source vectors for integer parity: depth, sigma (uint64 + overflow),
 * sigma fp64, delta (unpruned Eq.2).  All outputs are [n]. */
int oracle_sssp(int64_t n, const int64_t *rp, const int32_t *col, int32_t s, int32_t *depth,
                uint64_t *sigma, uint8_t *ovf, double *sigf, double *delta) {
    work_t w;
    if (work_alloc(&w, n, rp[n])) { work_free(&w); return 3; }
    brandes_source(n, rp, col, s, NULL, &w, NULL);
    for (int64_t v = 0; v < n; ++v) {
        depth[v] = w.d[v];
        int r = w.d[v] >= 0;
        if (sigma) sigma[v] = r ? w.sig[v] : 0;
        if (ovf) ovf[v] = r ? w.ovf[v] : 0;
        if (sigf) sigf[v] = r ? w.sigf[v] : 0.0;
        if (delta) delta[v] = r ? w.delta[v] : 0.0;
    }
    work_free(&w);
    return 0;
}

/* Alg.7 "Shortest-path tree computation of a 2-degree vertex from its own
 * neighbors", Lemma 1 and Eq.(6)
 * (PAPER.md:673-681): c has exactly the neighbours a and b; from their BFS
 * trees (depth d_a, d_b with -1 = unreached; sigma as uint64 + overflow flag)
 *     lvl_c(v)   = min(lvl_a(v), lvl_b(v)) + 1
 *     sigma_c(v) = sigma_a(v)             if lvl_a(v) < lvl_b(v)
 *                  sigma_b(v)             if lvl_a(v) > lvl_b(v)
 *                  sigma_a(v) + sigma_b(v) if equal
 * Two readings (R23): Alg.7's listing lets the `else` branch of its
 * second test overwrite the equal case with sigma_b alone -- Eq.(6) and the
 * text decide, the three cases are exclusive here; and Lemma 1 does not hold
 * for v = c itself (min + 1 = 2), whose level is 0 and sigma 1 by definition
 * (Alg.1 lines 7-8).  A vertex reached from neither neighbour stays unreached. */
int oracle_two_degree_tree(int64_t n, int32_t c, const int32_t *d_a, const uint64_t *sig_a, const uint8_t *ovf_a,
                           const int32_t *d_b, const uint64_t *sig_b, const uint8_t *ovf_b, int32_t *d_c,
                           uint64_t *sig_c, uint8_t *ovf_c) {
    for (int64_t v = 0; v < n; ++v) {
        int32_t la = d_a[v], lb = d_b[v];
        d_c[v] = -1;
        sig_c[v] = 0;
        ovf_c[v] = 0;
        if (v == c) {
            d_c[v] = 0;
            sig_c[v] = 1;
        } else if (la >= 0 && (lb < 0 || la < lb)) {
            d_c[v] = la + 1;
            sig_c[v] = sig_a[v];
            ovf_c[v] = ovf_a[v];
        } else if (lb >= 0 && (la < 0 || lb < la)) {
            d_c[v] = lb + 1;
            sig_c[v] = sig_b[v];
            ovf_c[v] = ovf_b[v];
        } else if (la >= 0) { /* la == lb */
            d_c[v] = la + 1;
            ovf_c[v] = (uint8_t)(ovf_a[v] | ovf_b[v] | __builtin_add_overflow(sig_a[v], sig_b[v], &sig_c[v]));
        }
    }
    return 0;
}

/* Alg.6, one processor (#P = 1): edges are the CSR entries, already sorted
 * by u.  For each (u,v): if u has no other edge (deg(u) = 1) append (v,u) to
 * R and omega[v]++, else append (u,v) to E'.  Then the symmetric edge (v,u)
 * of every removed (u,v) is dropped too.  Outputs:
 * omega[n], removed[n] (1 if deg(u) = 1), residual CSR in the same vertex-id
 * space (res_rp[n+1], res_col capacity rp[n]), *res_nnz. */
int oracle_prune_degree1(int64_t n, const int64_t *rp, const int32_t *col, uint32_t *omega,
                         uint8_t *removed, int64_t *res_rp, int32_t *res_col, int64_t *res_nnz) {
    for (int64_t v = 0; v < n; ++v) { omega[v] = 0; removed[v] = 0; }
    /* pass over E sorted by u */
    for (int64_t u = 0; u < n; ++u) {
        if (rp[u + 1] - rp[u] == 1) {                /* no other (w,z) with w = u */
            int32_t v = col[rp[u]];
            omega[v] += 1;                           /* omega[v] = omega[v] + 1 */
            removed[u] = 1;                          /* (v,u) -> R */
        }
    }
    /* E' = edges (u,v) with u kept, minus the symmetric copies of removed edges */
    int64_t k = 0;
    res_rp[0] = 0;
    for (int64_t u = 0; u < n; ++u) {
        if (!removed[u]) {
            for (int64_t e = rp[u]; e < rp[u + 1]; ++e)
                if (!removed[col[e]]) res_col[k++] = col[e];
        }
        res_rp[u + 1] = k;
    }
    *res_nnz = k;
    return 0;
}

/* Alg.6 on processor P_i of #P: E_i = the
 * edges (u,v) with u mod #P = i (1-D partitioning: all edges of u on one
 * processor), scanned sorted by u (the CSR order).  For
 * each (u,v) in E_i: if no other edge (w,z) of E_i has w = u, append (v,u)
 * to R -- removed_part[u] = 1 -- and omega_part[v] += 1; otherwise (u,v)
 * belongs to E'_i.  Outputs omega_part[n], removed_part[n] (zero outside
 * this processor's contributions).  Summing the #P outputs gives omega and
 * removed of the single-processor pass; the residual graph is then E' minus
 * the symmetric copies of R, as in oracle_prune_degree1. */
int oracle_prune_degree1_share(int64_t n, const int64_t *rp, const int32_t *col, int P, int i,
                               uint32_t *omega_part, uint32_t *removed_part) {
    if (P < 1 || i < 0 || i >= P) return 1;
    for (int64_t v = 0; v < n; ++v) { omega_part[v] = 0; removed_part[v] = 0; }
    for (int64_t u = 0; u < n; ++u) {
        if (u % P != i) continue;                    /* (u,v) not assigned to E_i */
        for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
            int has_other = (e > rp[u]) || (e + 1 < rp[u + 1]);  /* predecessor / successor with w = u */
            if (!has_other) {
                removed_part[u] = 1;                 /* (v,u) -> R */
                omega_part[col[e]] += 1;             /* omega[v] = omega[v] + 1 */
            }
        }
    }
    return 0;
}

/* BC with 1-degree reduction (Eq.4/Eq.5 with readings R7-R13):
 *   prune (Alg.6); then for every source s of the residual graph:
 *   - residual degree 0 and omega(s) > 0 (R10): n_s = 1 + omega(s);
 *     BC[s] += omega(s) * (n_s - 2);
 *   - otherwise Alg.1 on G' with the Eq.(5) recursion, n_s = sum over reached
 *     x of (1 + omega(x)) (R9), and (R13)
 *       BC[w] += (1 + omega(s)) * (delta_s(w) + omega(w))   for reached w != s,
 *       BC[s] += omega(s) * (n_s - 2).
 * sources == NULL means "all eligible": every non-removed vertex with residual
 * degree > 0 or omega > 0.  A removed source is rejected (return 1). */
int oracle_bc_pruned(int64_t n, const int64_t *rp, const int32_t *col, const int32_t *sources,
                     int64_t ns, int nthreads, double *bc) {
    uint32_t *omega = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
    uint8_t *removed = (uint8_t *)malloc((size_t)n);
    int64_t *rrp = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    int32_t *rcol = (int32_t *)malloc(sizeof(int32_t) * (size_t)(rp[n] > 0 ? rp[n] : 1));
    int32_t *all = NULL;
    int64_t rnnz = 0;
    if (!omega || !removed || !rrp || !rcol) return 3;
    oracle_prune_degree1(n, rp, col, omega, removed, rrp, rcol, &rnnz);
    if (!sources) {
        all = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        ns = 0;
        for (int64_t v = 0; v < n; ++v)
            if (!removed[v] && (rrp[v + 1] > rrp[v] || omega[v] > 0)) all[ns++] = (int32_t)v;
        sources = all;
    }
    for (int64_t i = 0; i < ns; ++i)
        if (sources[i] < 0 || sources[i] >= n || removed[sources[i]]) {
            free(omega); free(removed); free(rrp); free(rcol); free(all);
            return 1;
        }
    int T = pick_threads(nthreads);
    double *part = (double *)calloc((size_t)T * (size_t)n, sizeof(double));
    int err = part ? 0 : 3;
    if (!err) {
#pragma omp parallel num_threads(T)
        {
            int tid = omp_get_thread_num();
            double *mine = part + (size_t)tid * (size_t)n;
            work_t w;
            if (work_alloc(&w, n, rnnz)) {
#pragma omp atomic write
                err = 3;
            } else {
#pragma omp for schedule(dynamic, 1)
                for (int64_t i = 0; i < ns; ++i) {
                    int32_t s = sources[i];
                    double ws = (double)omega[s];
                    if (rrp[s + 1] == rrp[s]) {
                        double n_s = 1.0 + ws;
                        mine[s] += ws * (n_s - 2.0);
                        continue;
                    }
                    int64_t reached = brandes_source(n, rrp, rcol, s, omega, &w, NULL);
                    double n_s = 0.0;
                    for (int64_t k = 0; k < reached; ++k) n_s += 1.0 + (double)omega[w.queue[k]];
                    for (int64_t k = 0; k < reached; ++k) {
                        int32_t x = w.queue[k];
                        if (x != s) mine[x] += (1.0 + ws) * (w.delta[x] + (double)omega[x]);
                    }
                    mine[s] += ws * (n_s - 2.0);
                    reset_reached(&w, reached);
                }
            }
            work_free(&w);
        }
    }
    if (!err) {
        for (int64_t v = 0; v < n; ++v) {
            double acc = 0.0;
            for (int t = 0; t < T; ++t) acc += part[(size_t)t * (size_t)n + v];
            bc[v] = acc;
        }
    }
    free(part); free(omega); free(removed); free(rrp); free(rcol); free(all);
    return err;
}

int oracle_num_threads(void) { return omp_get_max_threads(); }
