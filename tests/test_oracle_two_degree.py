"""Pins for the 2-degree shortest-path-tree derivation (NEXT-1, PAPER.md
Alg.7 / Lemma 1 / Eq.(6)): the tree of a degree-2 vertex c
derived from the BFS trees of its neighbours a and b must equal the tree of a
direct BFS from c -- checked against the exact all-pairs brute force on tiny
graphs and against the (brute-force-pinned) oracle BFS on larger ones.  Also
shows the two places where the printed algorithm is wrong (reading R23)."""
import numpy as np
import pytest

import graphgen as gg
import oracle
from oracle import brute


def degree2(g):
    deg = np.diff(g.row_ptr)
    return [int(c) for c in np.nonzero(deg == 2)[0]]


def graphs():
    out = [gg.cycle(4), gg.cycle(5), gg.cycle(8), gg.path(5), gg.grid(3, 4), gg.grid(6, 7),
           gg.complete_bipartite(2, 5), gg.petersen(), gg.hypercube(2)]
    for i in range(40):
        out.append(gg.erdos_renyi(6 + i % 14, (0.12, 0.2, 0.3)[i % 3], seed=900 + i))
    for i in range(6):
        out.append(gg.rmat(6 + i % 3, 4, seed=950 + i))
    out.append(gg.disjoint_union(gg.cycle(6), gg.path(4), gg.star(3)))
    return out


def test_derived_tree_equals_brute_force_on_tiny_graphs():
    checked = 0
    for g in graphs():
        if g.n > 40:
            continue
        dist, cnt = brute.all_pairs(g)
        for c in degree2(g):
            d, s, o = oracle.two_degree_tree(g, c)
            want_d = [-1 if x is None else x for x in dist[c]]
            assert [int(x) for x in d] == want_d, (g.n, c)
            want_s = [cnt[c][t] if dist[c][t] is not None else 0 for t in range(g.n)]
            assert [int(x) for x in s] == want_s, (g.n, c)
            assert not o.any()
            checked += 1
    assert checked > 100


def test_derived_tree_equals_direct_bfs():
    checked = 0
    for g in graphs():
        for c in degree2(g):
            d, s, o = oracle.two_degree_tree(g, c)
            dd, ss, oo, _, _ = oracle.sssp(g, c)
            assert np.array_equal(d, dd) and np.array_equal(s, ss) and np.array_equal(o, oo)
            checked += 1
    # 40x40 grid corners (degree 2): sigma to the far corner is C(78, 39) > 2^64,
    # the overflow flags of the derivation agree with the direct BFS
    g = gg.grid(40, 40)
    for c in (0, 39, 1560, 1599):
        d, s, o = oracle.two_degree_tree(g, c)
        dd, ss, oo, _, _ = oracle.sssp(g, c)
        assert np.array_equal(d, dd) and np.array_equal(s, ss) and np.array_equal(o, oo)
        assert oo.any()
    assert checked > 200


def test_closed_forms_cycle():
    # C_n from c: two neighbours, antipode of an even cycle has sigma 2 via both
    for n in (6, 9, 12):
        g = gg.cycle(n)
        d, s, _ = oracle.two_degree_tree(g, 0)
        for v in range(n):
            assert d[v] == min(v, n - v)
            assert s[v] == (2 if n % 2 == 0 and v == n // 2 else 1)


def test_printed_alg7_is_wrong_where_the_readings_say():
    # equal levels: Alg.7's else-branch overwrites sigma_a + sigma_b with sigma_b
    g = gg.cycle(4)  # c = 0, a = 1, b = 3; v = 2 has lvl_a = lvl_b = 1
    lc, sc = oracle.two_degree_tree(g, 0, literal_alg7=True)
    d, s, _ = oracle.two_degree_tree(g, 0)
    assert s[2] == 2 and sc[2] == 1
    # Lemma 1 at v = c: min(lvl_a(c), lvl_b(c)) + 1 = 2, but lvl_c(c) = 0
    assert lc[0] == 2 and d[0] == 0
