"""Offline model of the batch schedule: exact hits per batch
(distinct oriented level pairs per edge over the batch's sources) for several
source orders on R-MAT S16 with 2048 sampled sources (8 batches of 256).
Hits are what both sweeps pay per item; lane-edges are fixed by the sources."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, graphgen as gg, scipy.sparse as sp, scipy.sparse.csgraph as cg, time
g = gg.rmat(16, 16, seed=1)
n = g.n
deg = np.diff(g.row_ptr)
A = sp.csr_matrix((np.ones(len(g.col)), g.col, g.row_ptr), shape=(n, n))
S = gg.sample_sources(g, 2048, seed=2)
t = time.time()
D = cg.shortest_path(A, unweighted=True, indices=S)  # [2048, n]
D = np.where(np.isinf(D), -1, D).astype(np.int8)
print("bfs", time.time() - t)
src = np.repeat(np.arange(n), deg); dst = g.col
m = src < dst
eu, ev = src[m], dst[m]
def hits(batches):
    tot_h = 0; tot_l = 0
    for b in batches:
        du = D[b][:, eu].astype(np.int16); dv = D[b][:, ev].astype(np.int16)   # [k, E]
        ok = (du >= 0) & (np.abs(du - dv) == 1)
        # distinct oriented level pairs per edge: key = min level (parent) * 2 + orientation
        key = np.where(du < dv, du * 2, dv * 2 + 1).astype(np.int32)
        key = np.where(ok, key, -1)
        # count distinct keys per edge column
        ks = np.sort(key, axis=0)
        distinct = (ks[1:] != ks[:-1]) & (ks[1:] >= 0)
        nh = distinct.sum(axis=0) + (ks[0] >= 0)
        tot_h += nh.sum(); tot_l += ok.sum()
    return tot_h, tot_l
# anchor key: highest-degree closed neighbour (by degree rank)
rank = np.empty(n, np.int64); rank[np.argsort(-deg, kind='stable')] = np.arange(n)
def anchor(s):
    nb = g.col[g.row_ptr[s]:g.row_ptr[s+1]]
    c = np.concatenate([[s], nb]); return c[np.argmin(rank[c])]
anc = np.array([anchor(s) for s in S])
K = 256
orders = {
  "random": np.arange(len(S)),
  "degree": np.argsort(rank[S], kind='stable'),
  "anchor": np.lexsort((rank[S], rank[anc])),
}
# signature: distances to top-8 hubs
hubs = np.argsort(-deg)[:8]
H = cg.shortest_path(A, unweighted=True, indices=hubs)[:, S].T   # [2048, 8]
orders["anchor+sig"] = np.lexsort(tuple(H[:, i] for i in range(7, -1, -1)) + (rank[anc],))
orders["sig+anchor"] = np.lexsort((rank[anc],) + tuple(H[:, i] for i in range(7, -1, -1)))
# mean distance to hubs then anchor
orders["dist0,anchor"] = np.lexsort((rank[S], rank[anc], H[:, 0]))
for name, o in orders.items():
    batches = [o[i:i+K] for i in range(0, len(o), K)]
    h, l = hits(batches)
    print(f"{name:14s} hits {h:>10} lane-edges {l:>11} lanes/hit {l/h:6.1f}")
rng = np.random.default_rng(0)
samp = rng.choice(n, 2048, replace=False)
P = D[:, samp].astype(np.float64)
P[P < 0] = 20
def rbisect(idx, depth=0):
    if len(idx) <= K:
        return [idx]
    X = P[idx] - P[idx].mean(0)
    u, s_, vt = np.linalg.svd(X, full_matrices=False)
    pc = X @ vt[0]
    o = idx[np.argsort(pc, kind='stable')]
    half = (len(o) // K // 2) * K if len(o) >= 2 * K else len(o) // 2
    half = max(K, half)
    return rbisect(o[:half], depth+1) + rbisect(o[half:], depth+1)
b = rbisect(np.arange(len(S)))
h, l = hits(b); print(f"{'pca-bisect':14s} hits {h:>10} lanes/hit {l/h:6.1f}")
# anchor first, then pca within anchor groups? greedy: sort by anchor rank, then fill
# k-medoids style: assign by nearest of 8 centers with capacity
from scipy.cluster.vq import kmeans2
cent, lab = kmeans2(P, 8, seed=1, minit='++')
# balanced assignment: greedy by distance
dist = ((P[:, None, :] - cent[None]) ** 2).sum(-1)
order = np.argsort(dist.min(1))
cap = np.full(8, K); assign = -np.ones(len(S), int)
for i in np.argsort(dist, axis=None):
    s_, c = divmod(i, 8)
    if assign[s_] < 0 and cap[c] > 0:
        assign[s_] = c; cap[c] -= 1
b = [np.nonzero(assign == c)[0] for c in range(8)]
h, l = hits(b); print(f"{'kmeans-bal':14s} hits {h:>10} lanes/hit {l/h:6.1f}")
# hamming-like: exact level-vector equality on top-32 hub distances, then anchor
H32 = cg.shortest_path(A, unweighted=True, indices=np.argsort(-deg)[:32])[:, S].T
o = np.lexsort((rank[anc],) + tuple(H32[:, i] for i in range(31, -1, -1)))
b = [o[i:i+K] for i in range(0, len(o), K)]
h, l = hits(b); print(f"{'hub32-sig':14s} hits {h:>10} lanes/hit {l/h:6.1f}")
