"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

Tolerance: per vertex |gpu - oracle| <= 1e-9 * |oracle|
with exact zeros where the oracle is exactly zero (every BC term is
non-negative, so there is no cancellation; measured fp64 error is ~1e-15).
Integer outputs (depth, sigma < 2^64, overflow flags, omega, removed flags,
residual CSR) are compared bit-exactly."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu

RTOL = 1e-9


def _bcb():
    import paper_1602_00963_b200 as bcb

    return bcb


def assert_bc_close(got, want, rtol=RTOL):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape
    if got.size == 0:
        return
    zero = want == 0.0
    assert np.all(got[zero] == 0.0), f"nonzero where oracle is exactly 0: {np.nonzero(got[zero])[0][:10]}"
    rel = np.abs(got - want) / np.where(zero, 1.0, np.abs(want))
    i = int(np.argmax(rel))
    assert rel.max() <= rtol, f"max rel err {rel.max():.3e} at {i}: gpu {got[i]!r} oracle {want[i]!r}"


def small_suite():
    out = []
    for i in range(24):
        n = 3 + (i * 5) % 40
        out.append(gg.erdos_renyi(n, (0.05, 0.1, 0.3)[i % 3], seed=700 + i))
    for i in range(12):
        out.append(gg.rmat(4 + i % 5, (2, 8, 16)[i % 3], seed=800 + i))
    for i in range(8):
        out.append(gg.with_isolated(gg.disjoint_union(gg.random_tree(5 + i, seed=i), gg.path(2), gg.star(4),
                                                      gg.cycle(5 + i)), i % 3))
    out += [gg.path(2), gg.path(3), gg.path(17), gg.cycle(9), gg.complete(6), gg.star(7),
            gg.complete_bipartite(3, 5), gg.hypercube(5), gg.petersen(), gg.grid(7, 9), gg.from_pairs(5, [])]
    return out


SUITE = small_suite()


@pytest.mark.parametrize("words", [1, 2, 4, 8])
@pytest.mark.parametrize("hub", [32, 4096])
@pytest.mark.parametrize("relabel", [0, 1, 2])
def test_small_suite_all_sources(words, hub, relabel):
    bcb = _bcb()
    for g in SUITE:
        with bcb.Graph.from_csr(g, validate=True) as G:
            G.set_option(bcb.OPT_LANE_WORDS, words)
            G.set_option(bcb.OPT_HUB_DEGREE, hub)
            G.set_option(bcb.OPT_RELABEL, relabel)
            assert_bc_close(G.compute(), oracle.bc(g))


@pytest.mark.parametrize("bwd", [1, 2])
@pytest.mark.parametrize("words", [1, 4, 8])
def test_backward_forms_push_and_pull(bwd, words):
    """Both backward forms (push: bwd_push.cuh; pull / successor checking:
    lanes.cuh BWD) on the small suite with split hubs, unpruned and pruned,
    and on a multi-batch R-MAT sample."""
    bcb = _bcb()
    for g in SUITE:
        for prune in (False, True):
            with bcb.Graph.from_csr(g) as G:
                G.set_option(bcb.OPT_BWD_MODE, bwd)
                G.set_option(bcb.OPT_LANE_WORDS, words)
                G.set_option(bcb.OPT_HUB_DEGREE, 32)
                if prune:
                    G.prune_degree1()
                assert_bc_close(G.compute(), oracle.bc(g))
    g = gg.rmat(13, 16, seed=5)
    S = gg.sample_sources(g, 600, seed=6)
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_BWD_MODE, bwd)
        G.set_option(bcb.OPT_LANE_WORDS, words)
        G.set_option(bcb.OPT_HUB_DEGREE, 64)
        assert_bc_close(G.compute(S), oracle.bc(g, S))


@pytest.mark.parametrize("relabel", [1, 2])
@pytest.mark.parametrize("prune", [False, True])
def test_small_suite_slices_mode(prune, relabel):
    """Batch mode 'slices' (one source per CTA) on the same suite, degree and
    breadth-first relabelling (the latter covers disconnected and isolated
    vertices: every component is ordered from its own far vertex)."""
    bcb = _bcb()
    for g in SUITE:
        with bcb.Graph.from_csr(g) as G:
            G.set_option(bcb.OPT_MODE, 2)
            G.set_option(bcb.OPT_RELABEL, relabel)
            if prune:
                G.prune_degree1()
            assert_bc_close(G.compute(), oracle.bc(g))


def test_grid_slices_and_lanes_agree_with_oracle():
    bcb = _bcb()
    g = gg.grid(64, 80)
    want = oracle.bc(g)
    with bcb.Graph.from_csr(g) as G:
        for mode in (1, 2):
            G.set_option(bcb.OPT_MODE, mode)
            assert_bc_close(G.compute(), want)


def test_config2_grid512_sampled_launch_config():
    """BASELINE config 2 (grid 512x512) in the bench's launch configuration
    (auto mode -> slices), on sampled sources the oracle can finish."""
    bcb = _bcb()
    g = gg.grid(512, 512)
    S = gg.sample_sources(g, 262144, seed=2)[:64]
    want = oracle.bc(g, S)
    with bcb.Graph.from_csr(g) as G:
        got = G.compute(S)
        st = G.stats()
    assert st["lanes"] == 1  # slices mode was chosen
    assert_bc_close(got, want)
    inv = st["dist_sum"] - (st["reached"] - st["num_sources"])
    assert abs(got.sum() - inv) <= 1e-9 * inv


@pytest.mark.parametrize("which", ["ell", "csr", "csr_pruned"])
def test_slices_lowdeg_kernels_large_and_small_n(which):
    """The degree-bounded slices kernels: the global-bitmap kernel (n past
    the shared-memory state, 1.2M vertices) and the shared-memory 2-bit-state
    kernel (small n), each with int4 (ELL, max degree <= 4) or CSR neighbour
    reads, pruning on in one case, on sampled sources of long-diameter graphs.
    The big grid is 40 x 30000 (30038 levels; sigma <= C(30038, 39) < 2^440 --
    a 1100 x 1100 grid would overflow fp64 sigma, C(2198, 1099) > 2^2000)."""
    bcb = _bcb()
    big = gg.grid(40, 30000)
    if which == "csr":
        big = gg.disjoint_union(big, gg.hypercube(6))  # max degree 6
    elif which == "csr_pruned":
        big = gg.disjoint_union(big, gg.random_tree(3000, seed=5), gg.hypercube(5))
    small = gg.grid(300, 301)
    if which != "ell":
        small = gg.disjoint_union(small, gg.random_tree(500, seed=6), gg.hypercube(5))
    for h in (big, small):
        S = gg.sample_sources(h, h.n, seed=4)[:24]
        with bcb.Graph.from_csr(h) as G:
            G.set_option(bcb.OPT_MODE, 2)
            if which == "csr_pruned":
                G.prune_degree1()
                _, rm, _, _ = G.pruning()
                S = S[rm[S] == 0]
                want = oracle.bc_pruned(h, S)
            else:
                want = oracle.bc(h, S)
            got = G.compute(S)
            assert G.stats()["lanes"] == 1
            assert_bc_close(got, want)


@pytest.mark.parametrize("hub", [32, 4096])
def test_small_suite_pruned(hub):
    bcb = _bcb()
    for g in SUITE:
        with bcb.Graph.from_csr(g) as G:
            G.set_option(bcb.OPT_HUB_DEGREE, hub)
            G.prune_degree1()
            assert_bc_close(G.compute(), oracle.bc(g))
            om, rm, rrp, rcol = oracle.prune_degree1(g)
            gom, grm, grp, gcol = G.pruning()
            assert np.array_equal(gom, om) and np.array_equal(grm, rm)
            assert np.array_equal(grp, rrp) and np.array_equal(gcol, rcol)


def test_pruned_partial_sources_equal_S_plus():
    bcb = _bcb()
    rng = np.random.default_rng(3)
    for g in SUITE[:30]:
        om, rm, rrp, rcol = oracle.prune_degree1(g)
        res_deg = np.diff(rrp)
        elig = [v for v in range(g.n) if not rm[v] and (res_deg[v] > 0 or om[v] > 0)]
        if not elig:
            continue
        S = sorted(rng.choice(elig, size=max(1, len(elig) // 2), replace=False).tolist())
        Splus = set(S)
        for s in S:
            Splus.update(int(u) for u in g.col[g.row_ptr[s]:g.row_ptr[s + 1]] if rm[u])
        with bcb.Graph.from_csr(g) as G:
            G.prune_degree1()
            assert_bc_close(G.compute(S), oracle.bc(g, sorted(Splus)))


def test_multibatch_ragged_tail_and_additivity():
    bcb = _bcb()
    g = gg.rmat(11, 16, seed=4)
    S = g.non_isolated()[:600]  # ragged last batch at K = 64, 256 and 512
    want = oracle.bc(g, S)
    with bcb.Graph.from_csr(g) as G:
        for words in (1, 4, 8):
            G.set_option(bcb.OPT_LANE_WORDS, words)
            got = G.compute(S)
            assert_bc_close(got, want)
        parts = sum(G.compute(S[r::3]) for r in range(3))
        assert_bc_close(parts, want)


def test_config1_rmat12_all_sources():
    """BASELINE config 1: R-MAT scale 12 EF16, all 4096 sources."""
    bcb = _bcb()
    g = gg.rmat(12, 16, seed=1)
    want = oracle.bc(g)
    with bcb.Graph.from_csr(g, validate=True) as G:
        got = G.compute()
        assert_bc_close(got, want)
        st = G.stats()
        # sum BC = sum_s sum_t (d(s,t) - 1)  (SURVEY §8c-iii invariant, from the GPU's own depths)
        inv = st["dist_sum"] - (st["reached"] - st["num_sources"])
        assert abs(got.sum() - inv) <= 1e-9 * inv
        G.prune_degree1()
        assert_bc_close(G.compute(), want)


def test_config3_rmat16_sampled_pruning_on_off():
    """BASELINE config 3 shape (R-MAT 16 EF16), pruning off and on, against
    the unpruned oracle on a 1024-source sample (full set: see bench)."""
    bcb = _bcb()
    g = gg.rmat(16, 16, seed=1)
    S = gg.sample_sources(g, 1024, seed=2)
    want = oracle.bc(g, S)
    with bcb.Graph.from_csr(g) as G:
        assert_bc_close(G.compute(S), want)
        G.prune_degree1()
        om, rm, rrp, rcol = oracle.prune_degree1(g)
        gom, grm, grp, gcol = G.pruning()
        assert np.array_equal(gom, om) and np.array_equal(grm, rm) and np.array_equal(grp, rrp)
        assert np.array_equal(gcol, rcol)
        Sr = [int(s) for s in S if not rm[s]]
        Splus = set(Sr)
        for s in Sr:
            Splus.update(int(u) for u in g.col[g.row_ptr[s]:g.row_ptr[s + 1]] if rm[u])
        assert_bc_close(G.compute(Sr), oracle.bc(g, sorted(Splus)))


def test_grid_lanes_small():
    bcb = _bcb()
    g = gg.grid(24, 31)
    with bcb.Graph.from_csr(g) as G:
        assert_bc_close(G.compute(), oracle.bc(g))


def test_sssp_integer_parity():
    bcb = _bcb()
    graphs = [gg.rmat(12, 16, seed=1), gg.grid(40, 40), gg.petersen(), gg.with_isolated(gg.path(9), 3)]
    for g in graphs:
        with bcb.Graph.from_csr(g) as G:
            G.set_option(bcb.OPT_HUB_DEGREE, 64)
            for s in (0, g.n // 3, g.n - 1):
                d, su, ov, sf, de = oracle.sssp(g, s)
                gd, gs, go, gde = G.sssp(s)
                assert np.array_equal(gd, d)
                ok = ov == 0
                assert np.array_equal(go, ov)
                assert np.array_equal(gs[ok & (d >= 0)], su[ok & (d >= 0)])
                m = (d > 0)
                assert_bc_close(gde[m], de[m])


def test_sssp_hypercube_sigma_beyond_2p53():
    bcb = _bcb()
    g = gg.hypercube(20)
    d, su, ov, sf, de = oracle.sssp(g, 0)
    with bcb.Graph.from_csr(g) as G:
        gd, gs, go, gde = G.sssp(0)
    assert np.array_equal(gd, d) and np.array_equal(gs, su) and not go.any()
    assert int(gs.max()) > 2 ** 53


def test_config4_rmat20_sampled_launch_config():
    """BASELINE config 4 (R-MAT 20 EF16) in the bench's launch configuration
    (K = 256 lanes, default hub split), on a sampled source set the oracle
    can finish; by additivity this checks those sources' contributions."""
    bcb = _bcb()
    g = gg.rmat(20, 16, seed=1)
    S = gg.sample_sources(g, 65536, seed=2)[:96]
    want = oracle.bc(g, S)
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_LANE_WORDS, 4)
        got = G.compute(S)
    assert_bc_close(got, want)


def test_edge_cases_and_errors():
    bcb = _bcb()
    g = gg.with_isolated(gg.path(5), 2)
    with bcb.Graph.from_csr(g) as G:
        assert np.all(G.compute([]) == 0.0)
        assert np.all(G.compute([5, 6]) == 0.0)  # isolated sources contribute 0
        for bad in ([0, 0], [7], [-1]):
            with pytest.raises(bcb.BCError) as ei:
                G.compute(bad)
            assert ei.value.name == "BC_ERR_INVALID"
        G.prune_degree1()
        with pytest.raises(bcb.BCError) as ei:
            G.compute([0])  # removed 1-degree vertex
        assert ei.value.name == "BC_ERR_INVALID"
        with pytest.raises(bcb.BCError) as ei:
            G.prune_degree1()
        assert ei.value.name == "BC_ERR_STATE"
    with bcb.Graph.from_csr(gg.from_pairs(1, [])) as G:
        assert G.compute().tolist() == [0.0]
    bad = gg.CSR(3, np.array([0, 1, 2, 2]), np.array([1, 1], np.int32))  # asymmetric
    with pytest.raises(bcb.BCError):
        bcb.Graph.from_csr(bad, validate=True)


def test_device_output_on_torch_stream():
    import torch

    bcb = _bcb()
    g = gg.rmat(10, 8, seed=6)
    want = oracle.bc(g)
    with bcb.Graph.from_csr(g) as G:
        s = torch.cuda.Stream()
        out = torch.empty(g.n, dtype=torch.float64, device="cuda")
        with torch.cuda.stream(s):
            G.compute(None, out=out)
        s.synchronize()
        assert_bc_close(out.cpu().numpy(), want)


@pytest.mark.parametrize("mode", [1, 2])
def test_device_stats_match_oracle_per_source_counts(mode):
    """The kernels' A_s / D_s / n_s counters (used for the roofline's
    algorithmic bytes) equal the oracle's exact per-source statistics."""
    bcb = _bcb()
    g = gg.rmat(12, 16, seed=1)
    S = gg.sample_sources(g, 300, seed=5)
    _, st_o = oracle.bc(g, S, stats=True)
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, mode)
        G.compute(S)
        st = G.stats()
    assert st["reached"] == int(st_o[:, 0].sum())
    assert st["adj_reached"] == int(st_o[:, 1].sum())
    assert st["dag_edges"] == int(st_o[:, 2].sum())


def test_profiling_counters_do_not_disturb_results():
    """BC_OPT_PROFILE records CUDA events around every level kernel (bench's
    roofline timing); the results and the library state must be unaffected."""
    bcb = _bcb()
    g = gg.rmat(11, 16, seed=2)
    S = g.non_isolated()[:700]
    want = oracle.bc(g, S)
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_PROFILE, 1)
        for _ in range(2):
            assert_bc_close(G.compute(S), want)
            st = G.stats()
            assert st["fwd_ms"] > 0 and st["bwd_ms"] > 0
            assert abs(st["bwd_ms"] - st["bwd_fin_ms"] - st["bwd_push_ms"]) < 1e-9


def layered(k: int, layers: int) -> "gg.CSR":
    """Consecutive layers of k vertices joined completely: sigma from an end
    vertex to layer d is k^(d-1), exceeding 16 bits for k = 10, d >= 6."""
    pairs = [(a * k + i, (a + 1) * k + j) for a in range(layers - 1) for i in range(k) for j in range(k)]
    return gg.from_pairs(k * layers, pairs)


@pytest.mark.parametrize("width", [0, 64])
def test_sigma_width_narrow_and_fp64_rows(width):
    """16-bit sigma rows (default) and fp64 rows give the same exact BC."""
    bcb = _bcb()
    for g in SUITE[::3] + [gg.rmat(12, 16, seed=1)]:
        want = oracle.bc(g)
        with bcb.Graph.from_csr(g) as G:
            G.set_option(bcb.OPT_MODE, 1)
            G.set_option(bcb.OPT_SIGMA_WIDTH, width)
            assert_bc_close(G.compute(), want)
            st = G.stats()
            if st["batches"]:
                if width == 64:
                    assert st["narrow_batches"] == 0
                else:
                    assert st["narrow_batches"] == st["batches"] and st["narrow_fallbacks"] == 0


@pytest.mark.parametrize("words", [1, 4, 8])
@pytest.mark.parametrize("layers", [8, 12])
def test_narrow_sigma_overflow_reruns_batch_wider(words, layers):
    """sigma > 65535 in some lanes: those batches are re-run with 32-bit rows
    (layers = 8: sigma <= 10^6) or, past 2^32, with fp64 rows (layers = 12:
    sigma up to 10^10); the others stay 16-bit.  BC and the per-source
    counters match the oracle either way."""
    bcb = _bcb()
    big = layered(10, layers)
    g = gg.disjoint_union(big, gg.rmat(9, 8, seed=3))
    want, stats = oracle.bc(g, stats=True)
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, 1)
        G.set_option(bcb.OPT_LANE_WORDS, words)
        G.set_option(bcb.OPT_SOURCE_ORDER, 0)  # given order: layered sources fill the first batches
        got = G.compute(g.non_isolated())
        st = G.stats()
    assert_bc_close(got, want)
    S = g.non_isolated()
    assert st["reached"] == int(stats[S, 0].sum())  # counters restored across the re-runs
    assert st["adj_reached"] == int(stats[S, 1].sum())
    assert st["dag_edges"] == int(stats[S, 2].sum())
    assert st["narrow_fallbacks"] >= 1
    if layers == 8:
        assert st["mid_batches"] == st["narrow_fallbacks"]
    else:
        assert st["mid_batches"] < st["narrow_fallbacks"]
    if words == 1:
        assert st["narrow_batches"] >= 1
    assert st["narrow_batches"] + st["narrow_fallbacks"] == st["batches"]


def _two_degree_graphs():
    return SUITE[::2] + [gg.cycle(9), gg.cycle(64), gg.grid(12, 12), gg.rmat(12, 16, seed=1),
                         gg.disjoint_union(gg.cycle(10), gg.grid(5, 7), gg.rmat(8, 4, seed=2))]


@pytest.mark.parametrize("words", [1, 4, 8])
def test_two_degree_heuristic_all_sources(words):
    """NEXT-1: degree-2 sources whose neighbours are sources get their tree
    derived (Lemma 1 / Eq.(6)) instead of traversed; BC and the per-source
    counters (n_s, A_s, D_s) equal the oracle's."""
    bcb = _bcb()
    derived = 0
    for g in _two_degree_graphs():
        want, stats = oracle.bc(g, stats=True)
        with bcb.Graph.from_csr(g) as G:
            G.set_option(bcb.OPT_MODE, 1)
            G.set_option(bcb.OPT_LANE_WORDS, words)
            G.set_option(bcb.OPT_TWO_DEGREE, 1)
            got = G.compute()
            st = G.stats()
        assert_bc_close(got, want)
        derived += st["derived_lanes"]
        S = g.non_isolated()  # isolated sources are not traversed (and add 0)
        assert st["reached"] == int(stats[S, 0].sum())
        assert st["adj_reached"] == int(stats[S, 1].sum())
        assert st["dag_edges"] == int(stats[S, 2].sum())
    assert derived > 100


def test_two_degree_heuristic_partial_pruned_and_wide_sigma():
    bcb = _bcb()
    g = gg.rmat(11, 8, seed=6)
    S = gg.sample_sources(g, 700, seed=3)
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_TWO_DEGREE, 1)
        assert_bc_close(G.compute(S), oracle.bc(g, S))
        assert G.stats()["derived_lanes"] > 0
        G.prune_degree1()
        assert_bc_close(G.compute(), oracle.bc(g))
        assert G.stats()["derived_lanes"] > 0
    # 40x40 grid in lanes mode: corners are degree 2, sigma reaches C(78, 39) > 2^64,
    # so the 16- and 32-bit batches overflow and the derivation runs in fp64 too
    g = gg.grid(40, 40)
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, 1)
        G.set_option(bcb.OPT_TWO_DEGREE, 1)
        assert_bc_close(G.compute(), oracle.bc(g))
        st = G.stats()
        assert st["derived_lanes"] > 0 and st["narrow_fallbacks"] > 0


def test_concurrent_pipelines_agree():
    """BC_OPT_STREAMS: 1, 3 and 8 concurrent batch pipelines (host threads,
    private BC partials summed at the end) give the oracle's BC."""
    bcb = _bcb()
    g = gg.rmat(12, 16, seed=2)
    S = g.non_isolated()
    want = oracle.bc(g, S)
    with bcb.Graph.from_csr(g) as G:
        for ns in (1, 3, 8):
            G.set_option(bcb.OPT_STREAMS, ns)
            G.set_option(bcb.OPT_LANE_WORDS, 1)  # many batches
            assert_bc_close(G.compute(S), want)
            assert G.stats()["batches"] == (len(S) + 63) // 64


@pytest.mark.parametrize("loop", [0, 1, 2])
def test_device_loop_and_host_loop_agree(loop):
    """BC_OPT_DEVICE_LOOP: device-driven batches (one CUDA graph launch per
    batch, 8-byte rows with the fp64 tier in the graph, or 4-byte rows with
    the host fp64 re-run) and the host-driven level loop give the oracle's
    BC on the small suite, pruned and unpruned, with split hubs."""
    bcb = _bcb()
    for g in SUITE:
        for prune in (False, True):
            with bcb.Graph.from_csr(g) as G:
                G.set_option(bcb.OPT_MODE, 1)
                G.set_option(bcb.OPT_DEVICE_LOOP, loop)
                G.set_option(bcb.OPT_HUB_DEGREE, 32)
                if prune:
                    G.prune_degree1()
                assert_bc_close(G.compute(), oracle.bc(g))


@pytest.mark.parametrize("loop", [1, 2])
@pytest.mark.parametrize("layers", [8, 12])
def test_device_loop_sigma_tiers(loop, layers):
    """sigma beyond 16 bits (layers = 8) and beyond 32 bits (layers = 12) in
    device-driven batches: the 32-bit tier runs inside the graph, the fp64
    tier too with 8-byte rows (loop 1) or on the host path with 4-byte rows
    (loop 2); BC and the per-source counters match the oracle."""
    bcb = _bcb()
    g = gg.disjoint_union(layered(10, layers), gg.rmat(9, 8, seed=3))
    want, stats = oracle.bc(g, stats=True)
    S = g.non_isolated()
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, 1)
        G.set_option(bcb.OPT_LANE_WORDS, 1)
        G.set_option(bcb.OPT_SOURCE_ORDER, 0)
        G.set_option(bcb.OPT_DEVICE_LOOP, loop)
        got = G.compute(S)
        st = G.stats()
    assert_bc_close(got, want)
    assert st["reached"] == int(stats[S, 0].sum())
    assert st["adj_reached"] == int(stats[S, 1].sum())
    assert st["dag_edges"] == int(stats[S, 2].sum())
    assert st["narrow_fallbacks"] >= 1
    assert st["narrow_batches"] + st["narrow_fallbacks"] == st["batches"]
    if layers == 8:
        assert st["mid_batches"] == st["narrow_fallbacks"]
    else:
        assert st["mid_batches"] < st["narrow_fallbacks"]


def test_device_loop_is_stream_ordered():
    """With a device output on a stream, bc_compute (device-driven) returns
    once enqueued; work queued behind it on the stream sees the result, and
    a second call on the same handle is ordered after the first."""
    import torch

    bcb = _bcb()
    g = gg.rmat(12, 16, seed=1)
    S1, S2 = g.non_isolated()[:1500], g.non_isolated()[1500:]
    w1, w2 = oracle.bc(g, S1), oracle.bc(g, S2)
    with bcb.Graph.from_csr(g) as G:
        s = torch.cuda.Stream()
        a = torch.empty(g.n, dtype=torch.float64, device="cuda")
        b = torch.empty(g.n, dtype=torch.float64, device="cuda")
        with torch.cuda.stream(s):
            G.compute(S1, out=a, stream=s)
            a2 = a * 2.0  # queued behind the call on the same stream
            G.compute(S2, out=b, stream=s)
            tot = a + b
        s.synchronize()
        st = G.stats()
        assert st["batches"] >= 1
        assert_bc_close(a2.cpu().numpy() / 2.0, w1)
        assert_bc_close(b.cpu().numpy(), w2)
        assert_bc_close(tot.cpu().numpy(), w1 + w2)


def test_default_stream_calls_are_ordered_after_pending_work():
    """Calls given no stream run on the library's own non-blocking stream;
    they must still be ordered after work already queued on torch's legacy
    default stream: a device out_bc whose NaN fill sits behind a long GPU
    spin, and distributed-pruning shares whose sum is formed behind one."""
    import torch

    bcb = _bcb()
    g = gg.disjoint_union(gg.rmat(11, 8, seed=5), gg.star(4), gg.random_tree(20, seed=6))
    S = np.nonzero(oracle.prune_degree1(g)[1] == 0)[0].astype(np.int32)
    with bcb.Graph.from_csr(g) as G:
        dev = torch.device("cuda", G.device)
        om = torch.zeros(g.n, dtype=torch.int32, device=dev)
        rm = torch.zeros(g.n, dtype=torch.int32, device=dev)
        parts = []
        for i in range(2):
            a = torch.empty(g.n, dtype=torch.int32, device=dev)
            b = torch.empty(g.n, dtype=torch.int32, device=dev)
            G.prune_degree1_share(i, 2, a, b)
            parts.append((a, b))
        torch.cuda._sleep(200_000_000)  # the sums below run late on the default stream
        for a, b in parts:
            om += a
            rm += b
        G.prune_degree1_apply(om, rm)  # no stream: must wait for the sums
        out = torch.empty(g.n, dtype=torch.float64, device=dev)
        torch.cuda._sleep(200_000_000)
        out.fill_(float("nan"))  # queued late: the call below must run after it
        G.compute(S, out=out)
        got = out.cpu().numpy()
    want = oracle.bc(g)
    assert_bc_close(got, want)


@pytest.mark.parametrize("kernel", [1, 2, 3, 4])
def test_slices_kernel_variants(kernel):
    """BC_OPT_SLICES_KERNEL (NEXT-2 ablation): the general kernel with and
    without the prefix-sum reuse and both degree-bounded kernels agree with
    the oracle; the degree-bounded ones refuse graphs of larger degree."""
    bcb = _bcb()
    for g in SUITE + [gg.grid(40, 300), gg.disjoint_union(gg.grid(30, 31), gg.random_tree(200, seed=8))]:
        for prune in (False, True):
            with bcb.Graph.from_csr(g) as G:
                G.set_option(bcb.OPT_MODE, 2)
                G.set_option(bcb.OPT_SLICES_KERNEL, kernel)
                maxdeg = int(g.degrees.max()) if g.n else 0
                if prune:
                    G.prune_degree1()
                    maxdeg = int(np.diff(G.pruning()[2]).max())
                if kernel >= 3 and maxdeg > 64:
                    with pytest.raises(bcb.BCError):
                        G.compute()
                    continue
                assert_bc_close(G.compute(), oracle.bc(g))


@pytest.mark.parametrize("layers", [8, 12])
def test_host_loop_widens_sigma_rows_in_place(layers):
    """Host-driven level loop: a 16-bit batch whose sigma passes 65535 at
    some level widens to 32-bit rows from that level on (only that level is
    re-expanded; no batch re-run); past 2^32 (layers = 12) it goes to the
    fp64 re-run directly.  BC, counters and the captured sigma of widened
    lanes match the oracle."""
    from test_gpu_capture import assert_capture_matches

    bcb = _bcb()
    g = gg.disjoint_union(layered(10, layers), gg.rmat(9, 8, seed=3))
    want, stats = oracle.bc(g, stats=True)
    S = g.non_isolated()
    caps = [0, 5, int(S[-1])]
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, 1)
        G.set_option(bcb.OPT_LANE_WORDS, 1)
        G.set_option(bcb.OPT_SOURCE_ORDER, 0)
        G.set_option(bcb.OPT_DEVICE_LOOP, 0)
        got, depth, sigma, delta, tier = G.compute_captured(S, caps)
        st = G.stats()
    assert_bc_close(got, want)
    assert st["reached"] == int(stats[S, 0].sum())
    assert st["adj_reached"] == int(stats[S, 1].sum())
    assert st["dag_edges"] == int(stats[S, 2].sum())
    assert_capture_matches(g, caps, depth, sigma, delta)
    assert st["narrow_batches"] + st["widened_batches"] + st["narrow_fallbacks"] == st["batches"]
    if layers == 8:
        assert st["widened_batches"] >= 1 and st["narrow_fallbacks"] == 0, st
        assert 32 in set(tier.tolist())
    else:
        assert st["narrow_fallbacks"] >= 1 and st["mid_batches"] == 0, st
        assert 64 in set(tier.tolist())
