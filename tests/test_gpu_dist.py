"""The multi-GPU reduction on the CUDA path:
dist.graph_bc_distributed -- per-rank bc_compute of a source shard into a
CUDA tensor, then one all_reduce -- against the oracle.  World size 2: NCCL
over two GPUs when the box has them, else gloo with both ranks on cuda:0
(the library and the reduction are the same; only the transport differs)."""
import os
import socket

import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph():
    return gg.rmat(13, 16, seed=4)


def _sources(g):
    return gg.sample_sources(g, 1500, seed=5)


def _worker(rank, world, port, backend, q):
    import torch
    import torch.distributed as dist

    from paper_1602_00963_b200 import Graph
    from paper_1602_00963_b200.dist import graph_bc_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _graph()
    with Graph.from_csr(g, device=dev) as G:
        out = graph_bc_distributed(G, _sources(g), device=torch.device("cuda", dev))
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy()))
    dist.destroy_process_group()


def test_graph_bc_distributed_world2_matches_oracle():
    import torch
    import torch.multiprocessing as mp

    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, backend, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _graph()
    want = oracle.bc(g, _sources(g))
    zero = want == 0
    for r in (0, 1):
        assert np.all(res[r][zero] == 0)
        rel = np.abs(res[r] - want) / np.where(zero, 1, np.abs(want))
        assert rel.max() <= 1e-9, (backend, rel.max())
    assert np.array_equal(res[0], res[1])


def _prune_worker(rank, world, port, backend, q):
    import torch
    import torch.distributed as dist

    from paper_1602_00963_b200 import Graph
    from paper_1602_00963_b200.dist import graph_bc_distributed, prune_degree1_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _prune_graph()
    with Graph.from_csr(g, device=dev) as G:
        removed = prune_degree1_distributed(G)
        om, rm, rrp, rcol = G.pruning()
        kept = np.nonzero(rm == 0)[0].astype(np.int32)  # every residual source: S+ = all vertices (R13)
        out = graph_bc_distributed(G, kept, device=torch.device("cuda", dev))
        torch.cuda.synchronize()
        q.put((rank, removed, om, rm, rrp, rcol, out.cpu().numpy()))
    dist.destroy_process_group()


def _prune_graph():
    return gg.disjoint_union(gg.rmat(13, 16, seed=4), gg.star(6), gg.path(2), gg.random_tree(40, seed=3))


def test_prune_degree1_distributed_world2_matches_oracle():
    """NEXT-4: Alg.6 with the u mod #P split: each rank's
    device share, one all-reduce of the shares, the residual graph built on
    every rank -- bit-identical to the oracle's single pass -- then the
    source-sharded pruned BC over every residual source against the
    oracle's unpruned all-source BC (reading R13: S+ is every vertex)."""
    import torch
    import torch.multiprocessing as mp

    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_prune_worker, args=(r, 2, port, backend, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {t[0]: t[1:] for t in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _prune_graph()
    om, rm, rrp, rcol = oracle.prune_degree1(g)
    want = oracle.bc(g, threads=8)
    zero = want == 0
    for r in (0, 1):
        removed, gom, grm, grp, gcol, bc = res[r]
        assert removed == int(rm.sum())
        assert np.array_equal(gom, om) and np.array_equal(grm, rm), backend
        assert np.array_equal(grp, rrp) and np.array_equal(gcol, rcol), backend
        assert np.all(bc[zero] == 0)
        rel = np.abs(bc - want) / np.where(zero, 1, np.abs(want))
        assert rel.max() <= 1e-9, (backend, rel.max())
