"""Integer and per-source parity of the PRODUCTION kernels (bc_set_capture).

bc_set_capture makes the next bc_compute record, for chosen sources, the
depth, sigma and delta its own kernels produced -- the same batch, lane
width, sigma-row tier, relabelled CSR, hub split and pipelines (lanes mode)
or the same one-source-per-CTA kernel (slices mode).  Each captured source
is compared with the oracle's single-source Brandes (oracle.sssp, Alg.1):

* depth bit-exact everywhere;
* sigma bit-exact where the oracle's exact uint64 sigma is < 2^53 (every
  tier holds an exact integer there; the fp64 tier rounds above 2^53 like
  the oracle's own fp64 sigma, so there: relative 1e-12 against it);
* delta within 1e-9 relative, exact zeros where the oracle's
  delta is exactly zero.

On pruned handles the capture describes the unpruned graph (removed
vertices filled from their neighbour, delta = delta' + omega, R13)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu

TWO53 = float(2 ** 53)


def _bcb():
    import paper_1602_00963_b200 as bcb

    return bcb


def oracle_sssp_many(g, sources, threads=8):
    """oracle.sssp for several sources, in parallel host threads (the C call
    releases the GIL); the oracle's arithmetic is untouched."""
    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        return list(ex.map(lambda s: oracle.sssp(g, int(s)), sources))


def assert_capture_matches(g, caps, depth, sigma, delta, want=None, rtol=1e-9):
    if want is None:
        want = oracle_sssp_many(g, caps)
    for i, s in enumerate(caps):
        d, su, ov, sf, de = want[i]
        assert np.array_equal(depth[i], d), f"depth differs for source {s}: {np.nonzero(depth[i] != d)[0][:8]}"
        reach = d >= 0
        exact = reach & (ov == 0) & (su.astype(np.float64) < TWO53)
        assert np.array_equal(sigma[i][exact], su[exact].astype(np.float64)), f"sigma differs for source {s}"
        big = reach & ~exact
        if big.any():
            rel = np.abs(sigma[i][big] - sf[big]) / sf[big]
            assert rel.max() <= 1e-12, f"large sigma rel err {rel.max():.2e} for source {s}"
        assert np.all(sigma[i][~reach] == 0.0)
        m = reach & (d > 0)
        zero = m & (de == 0.0)
        assert np.all(delta[i][zero] == 0.0), f"nonzero delta where the oracle's is 0 (source {s})"
        nz = m & ~zero
        if nz.any():
            rel = np.abs(delta[i][nz] - de[nz]) / np.abs(de[nz])
            assert rel.max() <= rtol, f"delta rel err {rel.max():.2e} for source {s}"
        assert np.all(delta[i][~m] == 0.0)


def _suite():
    out = []
    for i in range(6):
        out.append(gg.erdos_renyi(12 + 7 * i, (0.08, 0.2)[i % 2], seed=900 + i))
    for i in range(4):
        out.append(gg.rmat(6 + i, 8, seed=910 + i))
    out.append(gg.with_isolated(gg.disjoint_union(gg.random_tree(9, seed=3), gg.path(2), gg.star(5),
                                                  gg.cycle(7)), 2))
    out += [gg.path(17), gg.cycle(10), gg.grid(9, 11), gg.hypercube(6), gg.petersen(), gg.complete_bipartite(3, 6)]
    return out


SUITE = _suite()


@pytest.mark.parametrize("mode,words,hub,relabel", [(1, 1, 32, 1), (1, 4, 32, 0), (1, 8, 4096, 2), (1, 2, 64, 1),
                                                    (2, 0, 4096, 1), (2, 0, 4096, 2), (3, 0, 4096, 2), (4, 0, 4096, 1)])
@pytest.mark.parametrize("prune", [False, True])
def test_capture_small_suite(mode, words, hub, relabel, prune):
    bcb = _bcb()
    for g in SUITE:
        if mode >= 3 and g.n and g.degrees.max() > 64:
            continue
        with bcb.Graph.from_csr(g) as G:
            G.set_option(bcb.OPT_MODE, min(mode, 2))
            if mode >= 3:  # slices mode, degree-bounded kernel 3 / 4 (global bitmaps / shared state)
                G.set_option(bcb.OPT_SLICES_KERNEL, mode)
            if words:
                G.set_option(bcb.OPT_LANE_WORDS, words)
            G.set_option(bcb.OPT_HUB_DEGREE, hub)
            G.set_option(bcb.OPT_RELABEL, relabel)
            if prune:
                G.prune_degree1()
                _, rm, rrp, _ = G.pruning()
                om = G.pruning()[0]
                elig = [v for v in range(g.n) if not rm[v] and (rrp[v + 1] > rrp[v] or om[v] > 0)]
            else:
                elig = list(range(g.n))
            if not elig:
                continue
            caps = elig[:: max(1, len(elig) // 5)][:5]
            bc, depth, sigma, delta, tier = G.compute_captured(None, caps)
            assert_capture_matches(g, caps, depth, sigma, delta)
            # the capture rode along: the BC of the same call is still exact
            want = oracle.bc(g)
            zero = want == 0
            assert np.all(bc[zero] == 0)
            assert np.max(np.abs(bc - want) / np.where(zero, 1, np.abs(want))) <= 1e-9
            if mode >= 2:
                assert set(tier.tolist()) <= {0, 64}  # slices: fp64 sigma (0: residual-isolated source)
            else:
                assert set(tier.tolist()) <= {0, 16, 32, 64}


def layered(k: int, layers: int):
    pairs = [(a * k + i, (a + 1) * k + j) for a in range(layers - 1) for i in range(k) for j in range(k)]
    return gg.from_pairs(k * layers, pairs)


@pytest.mark.parametrize("layers,tiers", [(8, {16, 32}), (12, {16, 64})])
def test_capture_sigma_tiers(layers, tiers):
    """Batches whose sigma overflows 16 bits run in the 32-bit tier (and past
    2^32 in fp64): the captured lanes report the tier that completed and the
    sigma it held is exact (layered: sigma = 10^(d-1) from an end vertex)."""
    bcb = _bcb()
    g = gg.disjoint_union(layered(10, layers), gg.rmat(9, 8, seed=3))
    S = g.non_isolated()
    # layered sources fill the first batches (given order, 64 lanes); the last
    # R-MAT sources share a batch with no layered vertex
    caps = [0, 5, 10 * (layers // 2), int(S[-1]), int(S[-7])]
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, 1)
        G.set_option(bcb.OPT_LANE_WORDS, 1)
        G.set_option(bcb.OPT_SOURCE_ORDER, 0)
        bc, depth, sigma, delta, tier = G.compute_captured(S, caps)
        st = G.stats()
    assert st["narrow_fallbacks"] >= 1
    assert tiers <= set(tier.tolist()), tier
    assert_capture_matches(g, caps, depth, sigma, delta)


def test_capture_consumed_and_validated():
    bcb = _bcb()
    g = gg.with_isolated(gg.path(6), 1)
    with bcb.Graph.from_csr(g) as G:
        with pytest.raises(bcb.BCError) as ei:
            G.compute_captured([0, 1], [3])  # 3 not in the source set
        assert ei.value.name == "BC_ERR_INVALID"
        # consumed by the failed call: the next compute is a plain one
        assert np.allclose(G.compute([0, 1]), oracle.bc(g, [0, 1]))
        with pytest.raises(bcb.BCError):
            G.compute_captured(None, [1, 1])  # duplicate
        with pytest.raises(bcb.BCError):
            G.compute_captured(None, [99])
        bc, depth, sigma, delta, tier = G.compute_captured(None, [6])  # isolated source
        assert depth[0].tolist() == [-1] * 6 + [0]
        assert sigma[0][6] == 1.0 and np.all(delta[0] == 0)


def test_sssp_pruned_handle_fills_removed_vertices():
    """bc_sssp on a pruned handle traverses the residual graph (uint64 rows)
    and fills the removed vertices: the vectors equal the unpruned oracle."""
    bcb = _bcb()
    for g in [gg.rmat(11, 8, seed=5), gg.with_isolated(gg.disjoint_union(gg.random_tree(40, seed=2), gg.star(6),
                                                                          gg.path(2), gg.grid(6, 7)), 3)]:
        with bcb.Graph.from_csr(g) as G:
            G.set_option(bcb.OPT_HUB_DEGREE, 64)
            G.prune_degree1()
            _, rm, _, _ = G.pruning()
            kept = np.nonzero(rm == 0)[0]
            for s in kept[:: max(1, len(kept) // 6)][:6]:
                d, su, ov, sf, de = oracle.sssp(g, int(s))
                gd, gs, go, gde = G.sssp(int(s))
                assert np.array_equal(gd, d)
                assert np.array_equal(go, ov)
                ok = (ov == 0) & (d >= 0)
                assert np.array_equal(gs[ok], su[ok])
                m = d > 0
                zero = m & (de == 0)
                assert np.all(gde[zero] == 0)
                nz = m & ~zero
                if nz.any():
                    assert np.max(np.abs(gde[nz] - de[nz]) / de[nz]) <= 1e-9
            rem = np.nonzero(rm)[0]
            if len(rem):
                with pytest.raises(bcb.BCError):
                    G.sssp(int(rem[0]))
