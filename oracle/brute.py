"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Exact-rational brute force of the BC *definition* for tiny graphs, sharing
no traversal code with ``brandes.c``:

* all-pairs BFS by repeated frontier expansion over an adjacency-set dict,
  giving d(s,t) and sigma_st ("sigma_st ... number of shortest
  paths");
* Bellman criterion (Lemma 2): v lies on a shortest s-t
  path iff d(s,v) + d(v,t) = d(s,t), and then sigma_st(v) =
  sigma_sv * sigma_vt;
* Eq.(1): BC(v) = sum over ordered pairs s != t != v of
  sigma_st(v) / sigma_st, as Fractions.
"""
from __future__ import annotations

from fractions import Fraction


def adjacency(g):
    adj = {v: set() for v in range(g.n)}
    for v in range(g.n):
        for e in range(int(g.row_ptr[v]), int(g.row_ptr[v + 1])):
            adj[v].add(int(g.col[e]))
    return adj


def all_pairs(g):
    """dist[s][t] (None if unreachable) and sigma[s][t] as Python ints."""
    adj = adjacency(g)
    n = g.n
    dist = [[None] * n for _ in range(n)]
    sigma = [[0] * n for _ in range(n)]
    for s in range(n):
        dist[s][s] = 0
        sigma[s][s] = 1
        frontier = [s]
        level = 0
        while frontier:
            level += 1
            nxt = {}
            for v in frontier:
                for w in adj[v]:
                    if dist[s][w] is None or dist[s][w] == level:
                        if dist[s][w] is None:
                            dist[s][w] = level
                        nxt[w] = nxt.get(w, 0) + sigma[s][v]
            for w, c in nxt.items():
                sigma[s][w] = c
            frontier = sorted(nxt)
    return dist, sigma


def bc_exact(g, sources=None):
    """Eq.(1) restricted to s in ``sources``: list of Fractions."""
    dist, sigma = all_pairs(g)
    n = g.n
    S = range(n) if sources is None else [int(s) for s in sources]
    bc = [Fraction(0)] * n
    for s in S:
        for t in range(n):
            if t == s or dist[s][t] is None:
                continue
            for v in range(n):
                if v == s or v == t or dist[s][v] is None or dist[v][t] is None:
                    continue
                if dist[s][v] + dist[v][t] == dist[s][t]:
                    bc[v] += Fraction(sigma[s][v] * sigma[v][t], sigma[s][t])
    return bc


def delta_exact(g, s):
    """delta_s(v) = sum_t sigma_st(v)/sigma_st (the pair-dependency sum)."""
    dist, sigma = all_pairs(g)
    n = g.n
    out = [Fraction(0)] * n
    for t in range(n):
        if t == s or dist[s][t] is None:
            continue
        for v in range(n):
            if v == s or v == t or dist[s][v] is None or dist[v][t] is None:
                continue
            if dist[s][v] + dist[v][t] == dist[s][t]:
                out[v] += Fraction(sigma[s][v] * sigma[v][t], sigma[s][t])
    return out
