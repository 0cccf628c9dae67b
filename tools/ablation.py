"""NEXT-2 ablation: the design choices of the lanes path
measured one at a time against the default, on R-MAT S16 (all sources) and
R-MAT S20 (8192 sampled sources).  Prints one JSON object per variant.

Variants (bc_set_option): forward push form for the first levels vs pull,
backward pull (successor checking, Alg.5) vs push, fp64 vs 16-bit sigma
rows, batch schedule (given order / degree order / anchor clusters), degree
relabelling off, lane width K = 64 / 128 / 256."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_00963_b200 as bcb  # noqa: E402

VARIANTS = {
    "default": {},
    "fwd_push_L1": {bcb.OPT_FWD_PUSH: 1, bcb.OPT_SIGMA_WIDTH: 64},
    "fwd_push_L2": {bcb.OPT_FWD_PUSH: 2, bcb.OPT_SIGMA_WIDTH: 64},
    "bwd_pull": {bcb.OPT_BWD_MODE: 2},
    "sigma_fp64": {bcb.OPT_SIGMA_WIDTH: 64},
    "order_given": {bcb.OPT_SOURCE_ORDER: 0},
    "order_degree": {bcb.OPT_SOURCE_ORDER: 1},
    "relabel_off": {bcb.OPT_RELABEL: 0},
    "lanes_64": {bcb.OPT_LANE_WORDS: 1},
    "lanes_128": {bcb.OPT_LANE_WORDS: 2},
}


def run(name, g, S, opts, reps=2):
    with bcb.Graph.from_csr(g) as G:
        G.set_option(bcb.OPT_MODE, 1)
        for k, v in opts.items():
            G.set_option(k, v)
        G.set_option(bcb.OPT_PROFILE, 1)
        out = torch.empty(g.n, dtype=torch.float64, device="cuda:0")
        best = None
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            t = time.perf_counter()
            G.compute(S, out=out)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            st = G.stats()
            best = dt if best is None else min(best, dt)
        res = out.cpu().numpy()
    return {"variant": name, "ms": best * 1e3, "gteps": len(S) * g.m / best / 1e9, "fwd_ms": st["fwd_ms"],
            "bwd_ms": st["bwd_ms"], "fwd_items": st["fwd_items"], "fwd_hits": st["fwd_hits"],
            "bwd_items": st["bwd_items"], "bwd_hits": st["bwd_hits"], "lanes": st["lanes"]}, res


for cfg, g, S in (("rmat16_all", gg.rmat(16, 16, seed=1), None),
                  ("rmat20_8192", gg.rmat(20, 16, seed=1), None)):
    S = g.non_isolated() if cfg.startswith("rmat16") else gg.sample_sources(g, 8192, seed=2)
    ref = None
    for name, opts in VARIANTS.items():
        r, res = run(name, g, S, opts)
        if ref is None:
            ref = res
        r["config"] = cfg
        r["max_rel_diff_vs_default"] = float(np.max(np.abs(res - ref) / np.maximum(np.abs(ref), 1e-300)))
        print(json.dumps(r), flush=True)
