"""Time bc_compute per step with device output (stream-ordered) vs host output
(synchronous, D2H inside) on the bench workload, alternating, to locate the
e2e gap."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_00963_b200 as bcb  # noqa: E402

g = gg.rmat(20, 16, seed=1)
S = gg.sample_sources(g, 65536, seed=2)
G = bcb.Graph.from_csr(g)
out = torch.empty(g.n, dtype=torch.float64, device="cuda:0")
host = np.empty(g.n, np.float64)
pinned = torch.empty(g.n, dtype=torch.float64).pin_memory().numpy()
for i in range(12):
    src = S[(i % 8) * 8192:(i % 8 + 1) * 8192]
    torch.cuda.synchronize()
    t = time.perf_counter()
    kind = ("dev", "host", "pinned")[i % 3]
    if kind == "dev":
        G.compute(src, out=out)
        torch.cuda.synchronize()
    else:
        G.compute(src, out=host if kind == "host" else pinned)
    print(f"{kind:6s} {1e3 * (time.perf_counter() - t):8.1f} ms", flush=True)
