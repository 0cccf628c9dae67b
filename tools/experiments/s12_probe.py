"""Why bench's device-timed S12 steps are slower than an isolated call:
time consecutive bc_compute calls (CUDA events on torch's stream) with the
bench's rotating source lists vs a fixed list, with and without stats reads."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_00963_b200 as bcb  # noqa: E402

g = gg.rmat(12, 16, seed=1)
S = g.non_isolated()
out = torch.empty(g.n, dtype=torch.float64, device="cuda:0")
stream = torch.cuda.current_stream()
G = bcb.Graph.from_csr(g)


def src(i, rotate):
    if not rotate:
        return S
    start = (i * len(S)) % len(S) + 7 * i
    return S[(start + np.arange(len(S))) % len(S)]


for rotate in (False, True):
    for stats in (False, True):
        for i in range(3):
            G.compute(src(i, rotate), out=out, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record(stream)
        for i in range(8):
            G.compute(src(3 + i, rotate), out=out, stream=stream)
            if stats:
                G.stats()
        e1.record(stream)
        torch.cuda.synchronize()
        print(f"rotate={rotate} stats={stats}: {e0.elapsed_time(e1) / 8:.2f} ms/step device, "
              f"{(time.perf_counter() - t) / 8 * 1e3:.2f} ms/step wall", flush=True)
for ns in (1, 2, 4, 8):
    G.set_option(bcb.OPT_STREAMS, ns)
    for i in range(3):
        G.compute(S, out=out, stream=stream)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(8):
        G.compute(S, out=out, stream=stream)
    torch.cuda.synchronize()
    print(f"streams={ns}: {(time.perf_counter() - t) / 8 * 1e3:.2f} ms/step wall", flush=True)
