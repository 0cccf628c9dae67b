"""NEXT-2 on long-diameter graphs:
the slices-mode kernels switched one at a time (BC_OPT_SLICES_KERNEL) and the
lanes mode, on graphs shaped like the paper's road networks (RoadNet-PA /
RoadNet-CA: EF ~1.4, diameter ~800):

  grid512        the 512 x 512 grid of BASELINE config 2 (EF 2, diameter 1022)
  grid512_holes  the same with 10 % of its edges removed (seed 3): irregular
                 degrees <= 4, longer detours
  ladder8        an 8 x 32768 grid: path-like, diameter 32774

Variants: general kernel (frontier degrees block-scanned into CD + binary
search, push sigma) without and with the paper's
prefix-sum reuse (the forward's CD kept for the backward),
the degree-bounded pull kernel with global bitmaps, the same with a 2-bit
shared-memory state (default), and the lanes mode (256 sources per batch).
One JSON object per (graph, variant); BC is compared with the default
variant's (max relative difference)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_00963_b200 as bcb  # noqa: E402


def holes(g, frac, seed):
    e = gg.edges_of(g)
    keep = np.random.default_rng(seed).random(len(e)) >= frac
    return gg.csr_from_edges(g.n, e[keep, 0], e[keep, 1], name="grid_holes")


VARIANTS = [("sm_state (default)", {}), ("general", {bcb.OPT_SLICES_KERNEL: 1}),
            ("general+prefix_reuse", {bcb.OPT_SLICES_KERNEL: 2}), ("lowdeg_global", {bcb.OPT_SLICES_KERNEL: 3}),
            ("lanes_K256", {bcb.OPT_MODE: 1, bcb.OPT_LANE_WORDS: 4})]

def run_variant(g, S_v, opts):
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, 2)
        for k, v in opts.items():
            G.set_option(k, v)
        out = torch.empty(g.n, dtype=torch.float64, device="cuda:0")
        best = None
        for _ in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            G.compute(S_v, out=out)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            best = dt if best is None else min(best, dt)
        res = out.cpu().numpy()
    return {"n": g.n, "m": g.m, "sources": len(S_v), "ms": best * 1e3, "gteps": len(S_v) * g.m / best / 1e9}, res


graphs = [("grid512", gg.grid(512, 512), 4096), ("grid512_holes", holes(gg.grid(512, 512), 0.10, 3), 4096),
          ("ladder8", gg.grid(8, 32768), 1024)]
for name, g, ns in graphs:
    S = gg.sample_sources(g, ns, seed=2)
    ref = None
    for vname, opts in VARIANTS:
        if vname.startswith("lanes") and name != "grid512":
            continue  # one BFS level per launch pair over 32k levels: minutes per batch
        S_v = S[:256] if vname.startswith("lanes") else S
        try:
            r, res = run_variant(g, S_v, opts)
        except bcb.BCError as e:  # lanes mode keeps one row per BFS level: ~1000 levels may not fit
            print(json.dumps({"graph": name, "variant": vname, "sources": len(S_v), "error": str(e)}), flush=True)
            continue
        if ref is None:
            ref = res
        r.update({"graph": name, "variant": vname})
        if len(S_v) == len(S):
            r["max_rel_diff_vs_default"] = float(np.max(np.abs(res - ref) / np.maximum(np.abs(ref), 1e-300)))
        print(json.dumps(r), flush=True)
