"""Debug: distributed pruning + device-output compute vs host-output compute, per rank (torchrun)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import graphgen as gg
from paper_1602_00963_b200 import Graph
from paper_1602_00963_b200.dist import prune_degree1_distributed, shard_sources

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
g = gg.disjoint_union(gg.rmat(13, 16, seed=4), gg.star(6), gg.path(2), gg.random_tree(40, seed=3))
mode = sys.argv[1] if len(sys.argv) > 1 else "dist"
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    with Graph.from_csr(g, device=dev) as G:
        if mode == "dist":
            prune_degree1_distributed(G)
        else:
            G.prune_degree1()
        rm = G.pruning()[1]
        kept = np.nonzero(rm == 0)[0].astype(np.int32)
        shard = shard_sources(kept, rank, world)
        host = G.compute(shard)
        out = torch.empty(g.n, dtype=torch.float64, device="cuda")
        G.compute(shard, out=out)
        torch.cuda.synchronize()
        d = out.cpu().numpy()
        host2 = G.compute(shard)
        bad = np.abs(d - host) > 1e-9 * np.maximum(1, np.abs(host))
        bad2 = np.abs(host2 - host) > 1e-9 * np.maximum(1, np.abs(host))
        print(f"rank {rank} rep {rep} mode {mode}: dev-vs-host bad {bad.sum()}, host-vs-host bad {bad2.sum()}, st={G.stats()['batches']}", flush=True)
dist.destroy_process_group()
