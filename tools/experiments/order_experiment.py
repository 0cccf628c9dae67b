"""Experiment: does a within-batch lane order by BFS-profile signature
concentrate each hit's lanes into fewer 32-lane groups?  Sources are ordered
on the host and passed with BC_OPT_SOURCE_ORDER = 0 (given order).

signature(s) = (d(s, h_0), ..., d(s, h_7)) for the 8 highest-degree vertices
h_i (oracle BFS from each hub: depth arrays), anchor(s) = highest-degree
closed neighbour (as the library's clustering)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402
import paper_1602_00963_b200 as bcb  # noqa: E402

g = gg.rmat(20, 16, seed=1)
S = gg.sample_sources(g, 8192, seed=2)
deg = np.diff(g.row_ptr)
hubs = np.argsort(-deg, kind="stable")[:8]
D = np.stack([oracle.sssp(g, int(h))[0] for h in hubs])  # [8][n]
anchor = np.empty(len(S), np.int64)
for i, s in enumerate(S):
    nb = g.col[g.row_ptr[s]:g.row_ptr[s + 1]]
    cand = np.concatenate([[s], nb])
    anchor[i] = cand[np.lexsort((cand, -deg[cand]))[0]]
sig = np.zeros(len(S), np.int64)
for k in range(8):
    sig = sig * 8 + np.clip(D[k][S], 0, 7)
orders = {
    "library_default": None,
    "anchor_deg": np.lexsort((-deg[S], -deg[anchor], anchor)),
    "anchor_sig": np.lexsort((sig, -deg[anchor], anchor)),
    "sig_anchor": np.lexsort((anchor, sig)),
    "sig_only": np.argsort(sig, kind="stable"),
}
out = torch.empty(g.n, dtype=torch.float64, device="cuda:0")
with bcb.Graph.from_csr(g) as G:
    G.set_option(bcb.OPT_STREAMS, 1)
    G.set_option(bcb.OPT_PROFILE, 1)
    ref = None
    for name, o in orders.items():
        G.set_option(bcb.OPT_SOURCE_ORDER, 2 if o is None else 0)
        src = S if o is None else S[o]
        best = None
        for _ in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            G.compute(src, out=out)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            best = dt if best is None else min(best, dt)
        st = G.stats()
        res = out.cpu().numpy()
        if ref is None:
            ref = res
        err = float(np.max(np.abs(res - ref) / np.maximum(np.abs(ref), 1e-300)))
        print(f"{name:16s} {best * 1e3:7.1f} ms fwd {st['fwd_ms']:6.1f} bwd {st['bwd_ms']:6.1f} "
              f"fi {st['fwd_items'] / 1e9:.2f}G fh {st['fwd_hits'] / 1e9:.3f}G bi {st['bwd_items'] / 1e9:.2f}G "
              f"diff {err:.1e}", flush=True)
