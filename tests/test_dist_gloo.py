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
from paper_1602_00963_b200.dist import distributed_bc, shard_sources


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
