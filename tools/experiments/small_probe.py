"""Per-call wall time of bc_compute on the small configs (R-MAT S12 / S16,
all sources) for lane widths and pipeline counts: where small graphs lose
time (per-batch launch and sync overhead)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_00963_b200 as bcb  # noqa: E402

for scale in (12, 16):
    g = gg.rmat(scale, 16, seed=1)
    S = g.non_isolated()
    out = torch.empty(g.n, dtype=torch.float64, device="cuda:0")
    with bcb.Graph.from_csr(g) as G:
        for words, ns, mode in ((4, 1, 1), (4, 4, 1), (8, 4, 1), (4, 8, 1), (8, 8, 1), (0, 1, 2)):
                G.set_option(bcb.OPT_MODE, mode)
                G.set_option(bcb.OPT_LANE_WORDS, words)
                G.set_option(bcb.OPT_STREAMS, ns)
                best = 1e9
                for _ in range(4):
                    torch.cuda.synchronize()
                    t = time.perf_counter()
                    G.compute(S, out=out)
                    torch.cuda.synchronize()
                    best = min(best, time.perf_counter() - t)
                st = G.stats()
                print(f"S{scale} mode={mode} W={words} streams={ns}: {best * 1e3:7.2f} ms  batches={st['batches']} "
                      f"levels={st['levels_total']} launches={st['kernel_launches']} "
                      f"{len(S) * g.m / best / 1e9:6.1f} GTEPS", flush=True)
