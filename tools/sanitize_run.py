"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): lanes mode (16-bit, 32-bit and fp64
sigma tiers, split hubs, pull and push backward, 2-degree lanes, capture)
and slices mode (shared-memory 2-bit state, global-bitmap and general
kernels), pruned and unpruned, each checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402
import paper_1602_00963_b200 as bcb  # noqa: E402


def close(a, b):
    z = b == 0
    assert np.all(a[z] == 0)
    r = np.abs(a - b) / np.where(z, 1, np.abs(b))
    assert r.max() <= 1e-9, r.max()


which = sys.argv[1] if len(sys.argv) > 1 else "all"
r = gg.rmat(10, 8, seed=3)
grid = gg.grid(24, 28)
layered = gg.from_pairs(60, [(a * 10 + i, (a + 1) * 10 + j) for a in range(5) for i in range(10) for j in range(10)])
cases = []
if which in ("lanes", "all"):
    for words, hub, bwd, prune, td in [(4, 32, 0, False, 0), (1, 4096, 2, True, 0), (8, 64, 0, True, 1), (2, 32, 1, False, 1)]:
        cases.append(("lanes", r, dict(words=words, hub=hub, bwd=bwd, prune=prune, td=td)))
    cases.append(("lanes", layered, dict(words=1, hub=4096, bwd=0, prune=False, td=0)))  # 16 -> 32-bit tier
    cases.append(("lanes", grid, dict(words=2, hub=4096, bwd=0, prune=False, td=0)))     # sigma > 2^32: fp64 tier
if which in ("slices", "all"):
    for g in (grid, gg.disjoint_union(grid, gg.hypercube(5)), r):
        for prune in (False, True):
            cases.append(("slices", g, dict(prune=prune)))
for mode, g, o in cases:
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, 1 if mode == "lanes" else 2)
        if mode == "lanes":
            G.set_option(bcb.OPT_LANE_WORDS, o["words"])
            G.set_option(bcb.OPT_HUB_DEGREE, o["hub"])
            G.set_option(bcb.OPT_BWD_MODE, o["bwd"])
            G.set_option(bcb.OPT_TWO_DEGREE, o["td"])
        if o["prune"]:
            G.prune_degree1()
        caps = [0, g.n // 2]
        if o["prune"]:
            _, rm, _, _ = G.pruning()
            caps = [int(v) for v in np.nonzero(rm == 0)[0][:2]]
        bc, depth, sigma, delta, tier = G.compute_captured(None, caps)
        close(bc, oracle.bc(g))
    print(mode, g.n, o, "ok", flush=True)
print("sanitize run ok")
