"""Pins of the CPU oracle (oracle/brandes.c) against things other than
itself: the exact-rational Eq.(1) brute force (oracle/brute.py), closed forms
of textbook families, printed worked examples (tests/golden/), and
invariants.  A dropped term, a sign or index error or a transposed operand in
Alg.1 / Eq.(2)-(3) fails at least one of these."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import graphgen as gg
import oracle
from oracle import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _close(a, b, rel=1e-12):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= rel * np.maximum(1.0, np.abs(b)))


# ---------------------------------------------------------------- worked examples
@pytest.mark.parametrize("ex", GOLD["bc"], ids=lambda e: e["name"])
def test_golden_bc(ex):
    g = gg.from_pairs(ex["n"], ex["pairs"])
    assert oracle.bc(g).tolist() == [float(x) for x in ex["bc"]]


@pytest.mark.parametrize("ex", GOLD["sssp"], ids=lambda e: e["name"])
def test_golden_sssp(ex):
    g = gg.from_pairs(ex["n"], ex["pairs"])
    d, su, ov, sf, de = oracle.sssp(g, ex["s"])
    assert d.tolist() == ex["depth"]
    assert su.tolist() == ex["sigma"] and not ov.any()
    for v, want in enumerate(ex["delta"]):
        if want is not None:
            assert de[v] == want


# ---------------------------------------------------------------- brute force
def _suite():
    out = []
    for i in range(60):
        n = 2 + (i * 7) % 19
        p = (0.05, 0.1, 0.3)[i % 3]
        out.append(gg.erdos_renyi(n, p if n > 6 else 0.5, seed=100 + i))
    for i in range(40):
        out.append(gg.rmat(2 + i % 4, (2, 8)[i % 2], seed=200 + i))
    for i in range(30):
        out.append(gg.random_tree(3 + i % 15, seed=300 + i))
    for i in range(25):
        a = gg.erdos_renyi(3 + i % 8, 0.4, seed=400 + i)
        b = gg.random_tree(2 + i % 5, seed=500 + i)
        out.append(gg.with_isolated(gg.disjoint_union(a, b, gg.path(2)), i % 3))
    out += [gg.path(n) for n in (1, 2, 3, 6)] + [gg.cycle(n) for n in (3, 5, 8)]
    out += [gg.complete(5), gg.star(5), gg.complete_bipartite(2, 3), gg.hypercube(3), gg.petersen(),
            gg.grid(3, 4), gg.from_pairs(4, [])]
    for i in range(4):
        out.append(gg.erdos_renyi(48 + 4 * i, 0.08, seed=600 + i))
    return out


SUITE = _suite()


def test_suite_size():
    assert len(SUITE) >= 160


@pytest.mark.parametrize("idx", range(len(SUITE)))
def test_oracle_equals_brute_force(idx):
    g = SUITE[idx]
    want = brute.bc_exact(g)
    got = oracle.bc(g)
    assert _close(got, [float(x) for x in want], 1e-12), g.name
    # partial source sets (additivity)
    rng = np.random.default_rng(idx)
    S = rng.permutation(g.n)[: max(1, g.n // 2)]
    want_s = brute.bc_exact(g, S)
    assert _close(oracle.bc(g, S), [float(x) for x in want_s], 1e-12)


@pytest.mark.parametrize("idx", range(0, len(SUITE), 7))
def test_oracle_delta_and_sigma_equal_brute_force(idx):
    g = SUITE[idx]
    dist, sigma = brute.all_pairs(g)
    for s in range(0, g.n, max(1, g.n // 4)):
        d, su, ov, sf, de = oracle.sssp(g, s)
        assert d.tolist() == [-1 if x is None else x for x in dist[s]]
        assert su.tolist() == [sigma[s][t] for t in range(g.n)]
        assert sf.tolist() == [float(sigma[s][t]) for t in range(g.n)]
        want = brute.delta_exact(g, s)
        assert _close([de[v] for v in range(g.n) if v != s], [float(want[v]) for v in range(g.n) if v != s])


# ---------------------------------------------------------------- closed forms
def test_path_cycle_complete_star_bipartite():
    for n in (2, 5, 9, 16):
        assert oracle.bc(gg.path(n)).tolist() == [2.0 * i * (n - 1 - i) for i in range(n)]
    for n in (4, 6, 10):
        assert oracle.bc(gg.cycle(n)).tolist() == [(n - 2) ** 2 / 4.0] * n
    for n in (5, 7, 11):
        assert oracle.bc(gg.cycle(n)).tolist() == [(n - 1) * (n - 3) / 4.0] * n
    for n in (3, 6):
        assert oracle.bc(gg.complete(n)).tolist() == [0.0] * n
    for k in (1, 3, 8):
        assert oracle.bc(gg.star(k)).tolist() == [float(k * (k - 1))] + [0.0] * k
    for a, b in ((2, 3), (3, 5), (4, 4)):
        got = oracle.bc(gg.complete_bipartite(a, b))
        assert _close(got, [b * (b - 1) / a] * a + [a * (a - 1) / b] * b)


def test_trees_closed_form():
    # BC(v) = (n-1)^2 - sum_i |T_i|^2 over the components T_i of T - v
    for seed in range(20):
        n = 5 + seed
        g = gg.random_tree(n, seed)
        adj = brute.adjacency(g)
        want = []
        for v in range(n):
            seen = {v}
            sizes = []
            for r in adj[v]:
                stack, cnt = [r], 0
                seen.add(r)
                while stack:
                    x = stack.pop()
                    cnt += 1
                    for y in adj[x]:
                        if y not in seen:
                            seen.add(y)
                            stack.append(y)
                sizes.append(cnt)
            want.append(float((n - 1) ** 2 - sum(s * s for s in sizes)))
        assert oracle.bc(g).tolist() == want


def test_hypercube_and_petersen():
    for d in (2, 3, 4, 5, 6):
        assert _close(oracle.bc(gg.hypercube(d)), [float((d - 2) * 2 ** (d - 1) + 1)] * (1 << d))
    assert _close(oracle.bc(gg.petersen()), [6.0] * 10)


def test_grid_depth_sigma_binomial():
    R, C = 9, 13
    g = gg.grid(R, C)
    for s in (0, 5 * C + 7, R * C - 1):
        d, su, ov, sf, de = oracle.sssp(g, s)
        r0, c0 = divmod(s, C)
        for v in range(R * C):
            r, c = divmod(v, C)
            dr, dc = abs(r - r0), abs(c - c0)
            assert d[v] == dr + dc
            assert su[v] == math.comb(dr + dc, dr)


def test_hypercube_sigma_factorial_beyond_2p53():
    """Q20: sigma(0, v) = popcount(v)!  -- 20! = 2.43e18 lies in (2^53, 2^64)."""
    g = gg.hypercube(20)
    d, su, ov, sf, de = oracle.sssp(g, 0)
    pc = np.array([bin(v).count("1") for v in range(1 << 20)])
    assert np.array_equal(d, pc)
    fact = np.array([math.factorial(k) for k in range(21)], dtype=np.uint64)
    assert np.array_equal(su, fact[pc]) and not ov.any()
    assert int(su.max()) == math.factorial(20) > 2 ** 53


def test_sigma_overflow_flag_matches_exact():
    """Grid 40x40 from a corner: sigma = C(r+c, r) exceeds 2^64 far away;
    the sticky flag must be set exactly where the exact value >= 2^64."""
    R = C = 40
    g = gg.grid(R, C)
    d, su, ov, sf, de = oracle.sssp(g, 0)
    for v in range(R * C):
        r, c = divmod(v, C)
        exact = math.comb(r + c, r)
        assert bool(ov[v]) == (exact >= 2 ** 64)
        if exact < 2 ** 64:
            assert int(su[v]) == exact


# ---------------------------------------------------------------- invariants
def _sum_d_minus_1(g, S):
    tot = 0
    for s in S:
        d = oracle.sssp(g, s)[0]
        r = d[d > 0]
        tot += int((r - 1).sum())
    return tot


def test_total_bc_equals_sum_of_distances_minus_one():
    for g in (gg.rmat(9, 8, seed=3), gg.grid(12, 10), gg.erdos_renyi(80, 0.05, seed=1)):
        S = np.arange(g.n, dtype=np.int32)
        bc = oracle.bc(g, S)
        assert abs(bc.sum() - _sum_d_minus_1(g, S)) <= 1e-9 * max(1.0, bc.sum())
        assert bc.min() >= 0.0
        deg = g.degrees
        assert np.all(bc[deg <= 1] == 0.0)


def test_additivity_and_thread_independence():
    g = gg.rmat(10, 8, seed=5)
    S = np.arange(g.n, dtype=np.int32)
    full = oracle.bc(g, S, threads=4)
    parts = sum(oracle.bc(g, S[r::3], threads=1) for r in range(3))
    assert _close(parts, full, 1e-12)


def test_stats_per_source():
    g = gg.rmat(8, 8, seed=2)
    S = g.non_isolated()[:10]
    _, st = oracle.bc(g, S, stats=True)
    for i, s in enumerate(S):
        d = oracle.sssp(g, s)[0]
        reached = np.nonzero(d >= 0)[0]
        assert st[i, 0] == len(reached)
        assert st[i, 1] == int(g.degrees[reached].sum())
        src = np.repeat(np.arange(g.n), g.degrees)
        dag = (d[src] >= 0) & (d[g.col] == d[src] + 1)
        assert st[i, 2] == int(dag.sum())
