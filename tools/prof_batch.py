"""Run bc_compute once on a sampled source set (for ncu / sanitizer runs)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_00963_b200 as bcb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--sources", type=int, default=256)
ap.add_argument("--lane-words", type=int, default=4)
ap.add_argument("--hub", type=int, default=0)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--prune", action="store_true")
ap.add_argument("--relabel", type=int, default=1)
ap.add_argument("--order", type=int, default=2)
ap.add_argument("--fwd-push", type=int, default=0)
ap.add_argument("--bwd", type=int, default=0)
ap.add_argument("--sigma", type=int, default=0)
ap.add_argument("--streams", type=int, default=0)
ap.add_argument("--two-degree", type=int, default=0)
ap.add_argument("--sort", default="none", choices=["none", "deg", "degasc"])
ap.add_argument("--no-profile", action="store_true")
ap.add_argument("--slices-kernel", type=int, default=0)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--consecutive", action="store_true", help="the first --sources non-isolated vertices (bench grid steps)")
ap.add_argument("--all", action="store_true", help="all non-isolated sources")
a = ap.parse_args()
g = gg.grid(a.grid, a.grid) if a.grid else gg.rmat(a.scale, a.ef, seed=1)
S = g.non_isolated() if a.all else gg.sample_sources(g, a.sources, seed=2)
if a.consecutive:
    S = g.non_isolated()[:a.sources]
G = bcb.Graph.from_csr(g)
if a.prune:
    G.prune_degree1()
    om, rm, _, _ = G.pruning()
    S = S[rm[S] == 0]
G.set_option(bcb.OPT_LANE_WORDS, a.lane_words)
G.set_option(bcb.OPT_RELABEL, a.relabel)
G.set_option(bcb.OPT_SOURCE_ORDER, a.order)
G.set_option(bcb.OPT_FWD_PUSH, a.fwd_push)
G.set_option(bcb.OPT_BWD_MODE, a.bwd)
G.set_option(bcb.OPT_SIGMA_WIDTH, a.sigma)
G.set_option(bcb.OPT_STREAMS, a.streams)
G.set_option(bcb.OPT_TWO_DEGREE, a.two_degree)
G.set_option(bcb.OPT_SLICES_KERNEL, a.slices_kernel)
G.set_option(bcb.OPT_MODE, a.mode)
if a.sort != "none":
    d = g.degrees[S]
    S = S[np.argsort(-d if a.sort == "deg" else d, kind="stable")]
if a.hub:
    G.set_option(bcb.OPT_HUB_DEGREE, a.hub)
G.set_option(bcb.OPT_PROFILE, 0 if a.no_profile else 1)
for r in range(a.repeat):
    t = time.perf_counter()
    bc = G.compute(S)
    dt = time.perf_counter() - t
    st = G.stats()
    print(f"n={g.n} m={g.m} sources={len(S)} wall={dt*1e3:.1f}ms fwd={st['fwd_ms']:.2f}ms bwd={st['bwd_ms']:.2f}ms "
          f"levels={st['levels_total']} launches={st['kernel_launches']} TEPS={len(S)*g.m/dt/1e9:.1f}G "
          f"A={st['adj_reached']} D={st['dag_edges']} N={st['reached']} fi={st['fwd_items']} fh={st['fwd_hits']} "
          f"bi={st['bwd_items']} bh={st['bwd_hits']} narrow={st['narrow_batches']} fallback={st['narrow_fallbacks']} "
          f"push={st['bwd_push_ms']:.2f}ms derived={st['derived_lanes']}")
