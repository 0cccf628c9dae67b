"""Input generator tests (graphgen/): normalisation rules, R-MAT counts and
determinism, the grid, and the Table-4 1-degree pins."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import graphgen as gg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _check_simple(g):
    rp, col = g.row_ptr, g.col
    assert rp[0] == 0 and rp[-1] == len(col)
    assert np.all(np.diff(rp) >= 0)
    src = np.repeat(np.arange(g.n), np.diff(rp))
    assert not np.any(src == col), "self-loop"
    for v in range(min(g.n, 2000)):
        row = col[rp[v]:rp[v + 1]]
        assert np.all(np.diff(row) > 0), "unsorted / duplicate"
    fwd = set(zip(src.tolist(), col.tolist()))
    assert all((b, a) in fwd for a, b in fwd), "asymmetric"


def test_normalize_examples():
    # SPEC.md:45-47
    g = gg.from_pairs(3, [(0, 1), (1, 2)])
    assert g.degrees.tolist() == [1, 2, 1] and g.m == 2
    g = gg.from_pairs(4, [(0, 1), (1, 2), (2, 3), (3, 0)])
    assert g.degrees.tolist() == [2, 2, 2, 2] and g.m == 4
    g = gg.from_pairs(2, [(0, 1), (1, 0), (0, 0)])
    assert g.degrees.tolist() == [1, 1] and g.m == 1


def test_normalize_random_is_simple_and_idempotent():
    rng = np.random.default_rng(5)
    for n in (1, 7, 50, 300):
        u = rng.integers(0, n, 4 * n)
        v = rng.integers(0, n, 4 * n)
        g = gg.csr_from_edges(n, u, v)
        _check_simple(g)
        e = gg.edges_of(g)
        g2 = gg.csr_from_edges(n, e[:, 0], e[:, 1])
        assert np.array_equal(g.row_ptr, g2.row_ptr) and np.array_equal(g.col, g2.col)


def test_rmat_pair_count_and_params():
    # exactly 2^scale * EF sampled pairs
    u, v = gg.rmat_edges(3, 2, seed=7)
    assert len(u) == 16 and u.max() < 8 and v.max() < 8
    u, v = gg.rmat_edges(10, 16, seed=1, permute=False)
    assert len(u) == 16 * 1024
    # quadrant probabilities: top bit of (u, v) follows (a, b, c, d)
    top_u, top_v = (u >> 9) & 1, (v >> 9) & 1
    q = np.bincount(top_u * 2 + top_v, minlength=4) / len(u)
    assert np.allclose(q, [GOLD["rmat"][k] for k in "abcd"], atol=0.01)


def test_rmat_deterministic_and_permutation_bijective():
    a = gg.rmat_edges(12, 4, seed=3)
    b = gg.rmat_edges(12, 4, seed=3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = gg.rmat_edges(12, 4, seed=4)
    assert not np.array_equal(a[0], c[0])
    # permutation is a bijection: same multiset of degrees with/without it
    gp = gg.rmat(10, 8, seed=2, permute=True)
    gn = gg.rmat(10, 8, seed=2, permute=False)
    assert gp.m == gn.m
    assert sorted(gp.degrees.tolist()) == sorted(gn.degrees.tolist())
    _check_simple(gp)


def test_rmat_thread_count_independent():
    code = ("import graphgen as gg, hashlib;g=gg.rmat(14,8,seed=9);"
            "print(hashlib.sha1(g.row_ptr.tobytes()+g.col.tobytes()).hexdigest())")
    outs = []
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONPATH=os.path.dirname(os.path.dirname(__file__)))
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env).decode().strip())
    assert outs[0] == outs[1]


def test_grid():
    g = gg.grid(3, 4)
    _check_simple(g)
    assert g.m == 3 * 3 + 4 * 2
    assert g.degrees.tolist()[:4] == [2, 3, 3, 2]


def test_sample_sources():
    g = gg.with_isolated(gg.path(10), 5)
    s = gg.sample_sources(g, 10, seed=2)
    assert sorted(s.tolist()) == list(range(10))
    s1 = gg.sample_sources(g, 4, seed=2)
    assert np.array_equal(s1, gg.sample_sources(g, 4, seed=2))
    assert len(set(s1.tolist())) == 4
    with pytest.raises(ValueError):
        gg.sample_sources(g, 11, seed=2)


def test_table4_one_degree_fraction():
    """PAPER.md:1091-1093 (Table 4): 1-degree % of R-MAT S20 EF4/16/32 is
    13.6/13.3/12.1.  Our generator (dedup + symmetrise, a different RNG
    stream from the paper's) must land within 0.5 percentage points."""
    want = GOLD["table4_one_degree_pct"]
    for ef, key in ((4, "rmat20_ef4"), (16, "rmat20_ef16"), (32, "rmat20_ef32")):
        g = gg.rmat(20, ef, seed=1)
        pct = 100.0 * float((g.degrees == 1).sum()) / g.n
        assert abs(pct - want[key]) < 0.5, (ef, pct)
