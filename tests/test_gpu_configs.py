"""Parity at BASELINE.json's configurations, in the launch configuration
bench.py times (auto lane width, sigma tiers, concurrent pipelines, anchor
clustering, relabelled CSR; slices mode on the grid).

Whole-batch BC is compared with the oracle where the oracle finishes the
same source set in seconds; at S23 (where it does not) every batch is checked
through captured per-source state (bc_set_capture: the production kernels'
own depth / sigma / delta for sampled lanes, one by one against oracle.sssp)
plus the total-BC invariant sum_v BC(v) = sum_s sum_t (d(s,t) - 1)
(SURVEY.md §8(c-iii)), computed from the kernels' depth counters."""
import numpy as np
import pytest

import graphgen as gg
import oracle
from test_gpu_capture import assert_capture_matches, oracle_sssp_many
from test_gpu_parity import assert_bc_close

pytestmark = pytest.mark.gpu


def _bcb():
    import paper_1602_00963_b200 as bcb

    return bcb


def _total_invariant(st):
    # sum over sources of sum_t (d(s,t) - 1) = dist_sum - (reached - sources)
    return st["dist_sum"] - (st["reached"] - st["num_sources"])


@pytest.fixture(scope="module")
def rmat20():
    return gg.rmat(20, 16, seed=1)


def test_config4_rmat20_three_pipelines_full_batches(rmat20):
    """768 sampled sources = 3 full 256-lane batches on the 3 auto pipelines,
    anchor-clustered (more sources than lanes), against the oracle's BC for
    the same 768 sources; 12 lanes spread over the batches captured."""
    bcb = _bcb()
    g = rmat20
    S = gg.sample_sources(g, 65536, seed=2)[:768]
    caps = S[::64]
    want = oracle.bc(g, S)
    ws = oracle_sssp_many(g, caps)
    with bcb.Graph.from_csr(g) as G:
        got, depth, sigma, delta, tier = G.compute_captured(S, caps)
        st = G.stats()
    assert st["lanes"] == 256 and st["batches"] == 3
    assert_bc_close(got, want)
    assert abs(got.sum() - _total_invariant(st)) <= 1e-9 * _total_invariant(st)
    assert_capture_matches(g, caps, depth, sigma, delta, want=ws)
    assert set(tier.tolist()) == {16}


def test_config4_rmat20_bench_step_captured(rmat20):
    """One whole bench step (8192 sources, 32 batches on 3 pipelines): 16
    captured lanes against oracle.sssp and the total-BC invariant."""
    bcb = _bcb()
    g = rmat20
    S = gg.sample_sources(g, 65536, seed=2)[:8192]
    caps = S[7::512]
    ws = oracle_sssp_many(g, caps)
    with bcb.Graph.from_csr(g) as G:
        got, depth, sigma, delta, tier = G.compute_captured(S, caps)
        st = G.stats()
    assert st["batches"] == 32
    assert np.all(got >= 0)
    inv = _total_invariant(st)
    assert abs(got.sum() - inv) <= 1e-9 * inv
    assert_capture_matches(g, caps, depth, sigma, delta, want=ws)


def test_config5_rmat23_bench_step_with_32bit_tier():
    """BASELINE config 5 (R-MAT 23 EF16): the bench's first per-GPU step (2048
    of the 16384 sampled sources, auto lane width, 4-byte rows).  Batches
    whose sigma exceeds 16 bits complete in the 32-bit tier; 16 captured
    lanes (two per batch) are checked against oracle.sssp one by one, and
    the whole step against the total-BC invariant.  The overflow test looks
    only at lanes still undiscovered at a vertex, so a tier change here means
    a real sigma above 2^16 (the widening itself: test_gpu_parity's layered
    graphs)."""
    bcb = _bcb()
    g = gg.rmat(23, 16, seed=1)
    S = gg.sample_sources(g, 16384, seed=2)[:2048]
    caps = S[3::128]
    with bcb.Graph.from_csr(g) as G:
        got, depth, sigma, delta, tier = G.compute_captured(S, caps)
        st = G.stats()
    assert st["num_sources"] == 2048
    # host-driven at this size: a batch whose sigma passes 16 bits widens to
    # 32-bit rows at that level (no batch re-run); a 32-bit captured lane
    # implies such a batch, a lane whose exact sigma passes 2^16 implies tier 32
    assert st["narrow_fallbacks"] == 0, st
    if 32 in set(tier.tolist()):
        assert st["widened_batches"] + st["mid_batches"] >= 1, st
    inv = _total_invariant(st)
    assert abs(got.sum() - inv) <= 1e-9 * inv
    assert np.all(got >= 0)
    ws = oracle_sssp_many(g, caps, threads=8)
    for i in range(len(caps)):
        d, su = ws[i][0], ws[i][1]
        if int(su[d >= 0].max()) > 65535:
            assert tier[i] >= 32, (i, tier[i])
    assert_capture_matches(g, caps, depth, sigma, delta, want=ws)


@pytest.fixture(scope="module")
def grid512():
    return gg.grid(512, 512)


def test_config2_grid512_2048_sources(grid512):
    """2048 sampled grid sources (several per resident CTA, so every CTA
    resets its shared state between sources) in the bench's slices kernel,
    against the oracle's BC; 8 sources captured."""
    bcb = _bcb()
    g = grid512
    S = gg.sample_sources(g, 262144, seed=2)[:2048]
    caps = S[::256]
    want = oracle.bc(g, S)
    ws = oracle_sssp_many(g, caps)
    with bcb.Graph.from_csr(g) as G:
        got, depth, sigma, delta, tier = G.compute_captured(S, caps)
        st = G.stats()
    assert st["lanes"] == 1  # slices mode
    assert_bc_close(got, want)
    assert_capture_matches(g, caps, depth, sigma, delta, want=ws)


def test_config2_grid512_all_sources_closed_form(grid512):
    """All 262,144 sources: sum_v BC(v) = sum over ordered pairs of (d - 1)
    with d the Manhattan distance, C^2(R^3-R)/3 + R^2(C^3-C)/3 - n(n-1)
    = 23,387,439,366,144 for R = C = 512, and BC is
    invariant under the grid's D4 symmetries."""
    bcb = _bcb()
    R = C = 512
    n = R * C
    total = C * C * (R ** 3 - R) // 3 + R * R * (C ** 3 - C) // 3 - n * (n - 1)
    assert total == 23_387_439_366_144
    with bcb.Graph.from_csr(grid512) as G:
        got = G.compute()
        st = G.stats()
    assert st["num_sources"] == n
    assert abs(got.sum() - total) <= 1e-9 * total
    assert _total_invariant(st) == total
    B = got.reshape(R, C)
    for T in (B.T, B[::-1, :], B[:, ::-1], B[::-1, ::-1].T):
        assert np.max(np.abs(T - B) / np.maximum(B, 1.0)) <= 1e-9
    assert B[0, 0] > 0 and np.all(B > 0)


def test_config3_rmat16_all_sources_pruning_off_and_on():
    """BASELINE config 3 in full: R-MAT 16 EF16, every source, pruning off
    and on, both against the unpruned oracle's exact all-sources BC."""
    bcb = _bcb()
    g = gg.rmat(16, 16, seed=1)
    want = oracle.bc(g)
    with bcb.Graph.from_csr(g) as G:
        assert_bc_close(G.compute(), want)
        assert G.stats()["num_sources"] == len(g.non_isolated())
        G.prune_degree1()
        assert_bc_close(G.compute(), want)


@pytest.mark.parametrize("levels", [1, 2])
def test_forward_push_variant_against_oracle(levels):
    """BC_OPT_FWD_PUSH (the paper's edge-push forward, Alg.3, for the first
    levels; fp64 rows) on an R-MAT sample with split hubs and a pruned
    small suite, against the oracle."""
    bcb = _bcb()
    g = gg.rmat(16, 16, seed=1)
    S = gg.sample_sources(g, 700, seed=9)
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_FWD_PUSH, levels)
        G.set_option(bcb.OPT_HUB_DEGREE, 512)
        assert_bc_close(G.compute(S), oracle.bc(g, S))
    from test_gpu_parity import SUITE

    for h in SUITE[::2]:
        for prune in (False, True):
            with bcb.Graph.from_csr(h) as G:
                G.set_option(bcb.OPT_MODE, 1)
                G.set_option(bcb.OPT_FWD_PUSH, levels)
                G.set_option(bcb.OPT_HUB_DEGREE, 32)
                if prune:
                    G.prune_degree1()
                assert_bc_close(G.compute(), oracle.bc(h))
