"""NEXT-4 measurement: Alg.6 as one device pass (bc_prune_degree1) vs the
distributed form (bc_prune_degree1_share on every rank + one all-reduce of
the shares + bc_prune_degree1_apply), wall time per phase on each rank.
usage: torchrun --nproc-per-node N tools/prune_dist_bench.py [--scale 23]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import graphgen as gg
from paper_1602_00963_b200 import Graph

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=23)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
dev = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
g = gg.rmat(a.scale, 16, seed=1)
res = {"single_ms": [], "share_ms": [], "allreduce_ms": [], "apply_ms": []}
for _ in range(a.reps):
    with Graph.from_csr(g, device=dev) as G:
        torch.cuda.synchronize(); t0 = time.perf_counter()
        G.prune_degree1()
        res["single_ms"].append((time.perf_counter() - t0) * 1e3)
        single = G.pruning()
    with Graph.from_csr(g, device=dev) as G:
        om = torch.empty(g.n, dtype=torch.int32, device="cuda")
        rm = torch.empty(g.n, dtype=torch.int32, device="cuda")
        dist.barrier(); torch.cuda.synchronize(); t0 = time.perf_counter()
        G.prune_degree1_share(rank, world, om, rm)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        buf = torch.cat([om, rm]); dist.all_reduce(buf); torch.cuda.synchronize(); t2 = time.perf_counter()
        G.prune_degree1_apply(buf[:g.n].contiguous(), buf[g.n:].contiguous())
        t3 = time.perf_counter()
        res["share_ms"].append((t1 - t0) * 1e3); res["allreduce_ms"].append((t2 - t1) * 1e3); res["apply_ms"].append((t3 - t2) * 1e3)
        got = G.pruning()
        assert all(np.array_equal(x, y) for x, y in zip(got, single)), "distributed pruning differs from the single pass"
if rank == 0:
    print(json.dumps({"scale": a.scale, "n": g.n, "nnz": int(g.row_ptr[-1]), "ranks": world,
                      **{k: round(float(np.median(v)), 3) for k, v in res.items()}, "identical": True}))
dist.destroy_process_group()
