"""Pins of the 1-degree oracle routines (Alg.6; Eq.4/5
PAPER.md:238-257 with DESIGN.md readings R7-R13) against brute force, the
printed examples and structural invariants."""
import json
import os

import numpy as np
import pytest

import graphgen as gg
import oracle
from oracle import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _close(a, b, rel=1e-11):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= rel * np.maximum(1.0, np.abs(b)))


@pytest.mark.parametrize("ex", GOLD["prune"], ids=lambda e: e["name"])
def test_golden_prune(ex):
    g = gg.from_pairs(ex["n"], ex["pairs"])
    om, rm, rrp, rcol = oracle.prune_degree1(g)
    assert np.nonzero(rm)[0].tolist() == ex["removed"]
    assert om.tolist() == ex["omega"]
    res = gg.CSR(g.n, rrp, rcol)
    assert gg.edges_of(res).tolist() == sorted(sorted(p) for p in ex["residual_pairs"])


@pytest.mark.parametrize("ex", GOLD["n_s"], ids=lambda e: e["name"])
def test_golden_n_s(ex):
    """n_s = size of s's ORIGINAL component (reading R9):
    equals sum over residual-reached x of (1 + omega(x))."""
    g = gg.from_pairs(ex["n"], ex["pairs"])
    om, rm, rrp, rcol = oracle.prune_degree1(g)
    res = gg.CSR(g.n, rrp, rcol)
    d = oracle.sssp(res, ex["s"])[0]
    assert int(sum(1 + int(om[x]) for x in np.nonzero(d >= 0)[0])) == ex["n_s"]


def _rand_graphs():
    out = []
    for i in range(120):
        n = 3 + i % 14
        a = gg.erdos_renyi(n, (0.12, 0.2, 0.35)[i % 3], seed=1000 + i)
        parts = [a]
        if i % 4 == 0:
            parts.append(gg.path(2))          # a K2 component: both ends removed (R11)
        if i % 5 == 0:
            parts.append(gg.star(3))          # centre becomes residual-isolated (R10)
        if i % 3 == 0:
            parts.append(gg.random_tree(4 + i % 6, seed=i))
        g = gg.disjoint_union(*parts) if len(parts) > 1 else a
        out.append(gg.with_isolated(g, i % 2))
    for i in range(20):
        out.append(gg.rmat(5, 2, seed=50 + i))
    return out


RG = _rand_graphs()


@pytest.mark.parametrize("idx", range(len(RG)))
def test_prune_invariants(idx):
    g = RG[idx]
    om, rm, rrp, rcol = oracle.prune_degree1(g)
    deg = g.degrees
    assert np.array_equal(rm.astype(bool), deg == 1)           # every deg-1 vertex, nothing else
    assert int(om.sum()) == int(rm.sum())                        # sum omega = |removed|
    # omega(v) counts v's degree-1 neighbours
    for v in range(g.n):
        nb = g.col[g.row_ptr[v]:g.row_ptr[v + 1]]
        assert om[v] == int((deg[nb] == 1).sum())
    res = gg.CSR(g.n, rrp, rcol)
    assert np.all(res.degrees[rm.astype(bool)] == 0)
    k2 = int(sum(1 for v in range(g.n) if deg[v] == 1 and deg[g.col[g.row_ptr[v]]] == 1)) // 2
    assert res.m == g.m - (int(rm.sum()) - k2)                   # reading R24
    # residual = induced subgraph on kept vertices
    e = gg.edges_of(g)
    keep = e[(deg[e[:, 0]] != 1) & (deg[e[:, 1]] != 1)]
    assert gg.edges_of(res).tolist() == keep.tolist()


@pytest.mark.parametrize("idx", range(len(RG)))
def test_pruned_bc_equals_unpruned_and_brute(idx):
    g = RG[idx]
    want = oracle.bc(g)
    got = oracle.bc_pruned(g)
    assert _close(got, want), g.name
    if g.n <= 24:
        assert _close(got, [float(x) for x in brute.bc_exact(g)])


@pytest.mark.parametrize("idx", range(0, len(RG), 3))
def test_pruned_partial_sources_equal_S_plus(idx):
    """Reading R13: a residual source s stands for {s} + its removed children,
    so the pruned result over S equals the unpruned BC over S+."""
    g = RG[idx]
    om, rm, rrp, rcol = oracle.prune_degree1(g)
    res_deg = np.diff(rrp)
    elig = [v for v in range(g.n) if not rm[v] and (res_deg[v] > 0 or om[v] > 0)]
    if not elig:
        return
    rng = np.random.default_rng(idx)
    S = sorted(rng.choice(elig, size=max(1, len(elig) // 2), replace=False).tolist())
    Splus = set(S)
    for s in S:
        for e in range(g.row_ptr[s], g.row_ptr[s + 1]):
            if rm[g.col[e]]:
                Splus.add(int(g.col[e]))
    want = oracle.bc(g, sorted(Splus))
    assert _close(oracle.bc_pruned(g, S), want)


def test_removed_source_rejected():
    with pytest.raises(ValueError):
        oracle.bc_pruned(gg.path(4), [0])


def test_literal_eq4_increment_order_is_wrong():
    """Reading R7: Eq.(4) literally (omega(v)++ then BC(v) += 2(n - omega(v) - 2))
    gives 0 for the centre of K1,3; brute force says 6.  The oracle's total
    endpoint term with omega taken before each increment,
    2*omega*(n-2) - omega*(omega-1), gives 6."""
    g = gg.star(3)
    n = 4
    literal = 0
    w = 0
    for _ in range(3):
        w += 1
        literal += 2 * (n - w - 2)
    assert literal == 0
    assert float(brute.bc_exact(g)[0]) == 6.0
    assert 2 * 3 * (n - 2) - 3 * 2 == 6
    assert oracle.bc_pruned(g)[0] == 6.0


def test_rmat_pruned_matches_unpruned():
    g = gg.rmat(10, 16, seed=1)
    assert _close(oracle.bc_pruned(g), oracle.bc(g), 1e-10)


# ---- Alg.6 distributed over #P processors (u mod #P = P_i), NEXT-4
@pytest.mark.parametrize("idx", range(0, len(RG), 2))
def test_prune_shares_sum_to_single_pass(idx):
    """The #P processors' shares (Alg.6 lines 3-9 on E_i = edges with
    u mod #P = i) sum to the one-processor omega / removed for every #P: each
    u belongs to exactly one E_i with all its edges."""
    g = RG[idx]
    om, rm, _, _ = oracle.prune_degree1(g)
    deg = g.degrees
    for P in (1, 2, 3, 5):
        oms, rms = zip(*(oracle.prune_degree1_share(g, P, i) for i in range(P)))
        assert np.array_equal(np.sum(oms, axis=0), om.astype(np.int64)), P
        assert np.array_equal(np.sum(rms, axis=0), rm.astype(np.int64)), P
        for i in range(P):  # a share only removes its own vertices, and only degree-1 ones
            own = np.arange(g.n) % P == i
            assert not np.any(rms[i][~own]) and np.array_equal(rms[i][own].astype(bool), deg[own] == 1)


def test_prune_share_star_closed_form():
    """Star K_{1,k} (centre 0): the leaves are removed wherever they sit and
    omega(centre) = k = sum over the shares of the leaves each holds."""
    k = 11
    g = gg.star(k)
    for P in (1, 2, 4):
        tot = np.zeros(g.n, np.int64)
        for i in range(P):
            om, rm = oracle.prune_degree1_share(g, P, i)
            leaves_here = sum(1 for u in range(1, k + 1) if u % P == i)
            assert om[0] == leaves_here and rm[0] == 0
            tot += om
        assert tot[0] == k and tot[1:].sum() == 0


def test_prune_share_rejects_bad_processor():
    with pytest.raises(ValueError):
        oracle.prune_degree1_share(gg.path(4), 2, 2)
