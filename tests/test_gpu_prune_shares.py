"""NEXT-4: Alg.6 distributed over #P processors with the
u mod #P split, here with the #P shares computed on one
device (the exchange is an element-wise sum; the NCCL form runs in
test_gpu_dist.py).  Each device share must equal the oracle's share of that
processor bit for bit, and the summed shares applied to a fresh handle must
give exactly the single-pass pruning and the same BC."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


def _graph():
    return gg.disjoint_union(gg.rmat(12, 8, seed=21), gg.star(5), gg.path(2), gg.random_tree(30, seed=5))


@pytest.mark.parametrize("P", [1, 2, 3, 7])
def test_shares_then_apply_equal_single_pass(P):
    import torch

    from paper_1602_00963_b200 import Graph

    g = _graph()
    om_o, rm_o, rp_o, col_o = oracle.prune_degree1(g)
    with Graph.from_csr(g) as G1:
        G1.prune_degree1()
        single = G1.pruning()
        bc1 = G1.compute()
    with Graph.from_csr(g) as G2:
        dev = torch.device("cuda", G2.device)
        om = torch.zeros(g.n, dtype=torch.int32, device=dev)
        rm = torch.zeros(g.n, dtype=torch.int32, device=dev)
        for i in range(P):
            a = torch.full((g.n,), 7, dtype=torch.int32, device=dev)  # overwritten, not accumulated
            b = torch.full((g.n,), 7, dtype=torch.int32, device=dev)
            G2.prune_degree1_share(i, P, a, b)
            wa, wb = oracle.prune_degree1_share(g, P, i)
            assert np.array_equal(a.cpu().numpy(), wa.astype(np.int32)), (P, i)
            assert np.array_equal(b.cpu().numpy(), wb.astype(np.int32)), (P, i)
            om += a
            rm += b
        removed = G2.prune_degree1_apply(om, rm)
        got = G2.pruning()
        bc2 = G2.compute()
    assert removed == int(rm_o.sum())
    for x, y, z in zip(got, single, (om_o, rm_o, rp_o, col_o)):
        assert np.array_equal(x, y) and np.array_equal(x, z)
    want = oracle.bc(g, threads=8)
    zero = want == 0
    assert np.all(bc2[zero] == 0)
    assert (np.abs(bc2 - want) / np.where(zero, 1, np.abs(want))).max() <= 1e-9
    assert (np.abs(bc2 - bc1) / np.where(zero, 1, np.abs(want))).max() <= 1e-12


def test_apply_rejects_incomplete_shares_and_keeps_the_handle():
    import torch

    from paper_1602_00963_b200 import BCError, Graph

    g = _graph()
    with Graph.from_csr(g) as G:
        dev = torch.device("cuda", G.device)
        a = torch.empty(g.n, dtype=torch.int32, device=dev)
        b = torch.empty(g.n, dtype=torch.int32, device=dev)
        G.prune_degree1_share(0, 2, a, b)  # rank 1's share missing
        with pytest.raises(BCError):
            G.prune_degree1_apply(a, b)
        with pytest.raises(BCError):
            G.prune_degree1_share(2, 2, a, b)  # rank out of range
        with pytest.raises(ValueError):
            G.prune_degree1_share(0, 1, np.zeros(g.n, np.int32), b)  # host buffer
        assert G.prune_degree1() == int(oracle.prune_degree1(g)[1].sum())  # still unpruned: single pass works
        with pytest.raises(BCError):
            G.prune_degree1_share(0, 1, a, b)  # already pruned
