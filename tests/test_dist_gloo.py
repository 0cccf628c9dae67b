"""World-size-2 gloo test of the source-sharded multi-GPU path (host logic):
sharding + one all-reduce of the fp64 BC vector must equal the single-rank
result (additivity).  The per-rank compute here is the CPU
oracle (tests may call it); on GPUs the same helper calls the CUDA path."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen as gg
import oracle
from paper_1602_00963_b200.dist import distributed_bc, prune_shares_reduced, shard_sources


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = gg.rmat(9, 8, seed=3)
    S = gg.sample_sources(g, 200, seed=2)

    def local(shard):
        return torch.from_numpy(oracle.bc(g, shard, threads=1))

    out = distributed_bc(local, S)
    q.put((rank, out.numpy()))
    dist.destroy_process_group()


def test_shards_are_a_partition():
    S = np.arange(103, dtype=np.int32)
    parts = [shard_sources(S, r, 4) for r in range(4)]
    assert sorted(np.concatenate(parts).tolist()) == S.tolist()
    assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_gloo_world2_allreduce_equals_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gg.rmat(9, 8, seed=3)
    S = gg.sample_sources(g, 200, seed=2)
    want = oracle.bc(g, S)
    for r in (0, 1):
        assert np.allclose(res[r], want, rtol=1e-12, atol=0)


def _prune_worker(rank, world, port, q):
    """Alg.6 distributed (NEXT-4) host logic: each rank's share (u mod world
    = rank; the oracle stands in for the device share), one all-reduce of the
    concatenated shares."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = gg.disjoint_union(gg.rmat(8, 4, seed=7), gg.star(5), gg.path(2), gg.random_tree(9, seed=2))

    def share(r, w):
        om, rm = oracle.prune_degree1_share(g, w, r)
        return torch.from_numpy(om.astype(np.int32)), torch.from_numpy(rm.astype(np.int32))

    om, rm = prune_shares_reduced(share, g.n)
    q.put((rank, om.numpy().copy(), rm.numpy().copy()))
    dist.destroy_process_group()


def test_gloo_world3_prune_shares_reduce_to_single_pass():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_prune_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = {r: (om, rm) for r, om, rm in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gg.disjoint_union(gg.rmat(8, 4, seed=7), gg.star(5), gg.path(2), gg.random_tree(9, seed=2))
    om, rm, _, _ = oracle.prune_degree1(g)
    for r in range(3):
        assert np.array_equal(res[r][0], om.astype(np.int32))
        assert np.array_equal(res[r][1], rm.astype(np.int32))
