"""Seeded synthetic graph inputs shared by the CUDA path and the oracle.

This module holds none of the method's arithmetic: it generates simple
undirected graphs (CSR, sorted adjacency, no self-loops, no duplicates --
SPEC.md:22-28) and seeded source samples.  The heavy generators (R-MAT,
grid, normalisation) live in ``graphgen.c`` (built into ``libgraphgen.so``);
the small families used by tests are plain numpy.

R-MAT follows PAPER.md:842-845 (Sec. 4.1): n = 2^scale, 2^scale*EF sampled
pairs, (a, b, c, d) = (0.57, 0.19, 0.19, 0.05).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgraphgen.so")
_lib_handle = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "graphgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", src, "-o", _SO]
        )
    return _SO


def _lib():
    global _lib_handle
    if _lib_handle is None:
        build()
        L = ctypes.CDLL(_SO)
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.gg_rmat_edges.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_uint64, ctypes.c_int, i32p, i32p]
        L.gg_normalize.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, i64p, i32p, i64p]
        L.gg_grid.argtypes = [ctypes.c_int64, ctypes.c_int64, i64p, i32p]
        L.gg_sample_sources.argtypes = [ctypes.c_int64, i64p, ctypes.c_int64, ctypes.c_uint64, i32p]
        _lib_handle = L
    return _lib_handle


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


@dataclass
class CSR:
    """Simple undirected graph: row_ptr int64[n+1], col int32[2m] (sorted rows)."""

    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def m(self) -> int:
        """Unique undirected edges."""
        return self.nnz // 2

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def non_isolated(self) -> np.ndarray:
        return np.nonzero(self.degrees > 0)[0].astype(np.int32)


# ----------------------------------------------------------------- R-MAT, grid
def rmat_edges(scale: int, ef: int, seed: int = 1, a: float = 0.57, b: float = 0.19,
               c: float = 0.19, permute: bool = True):
    ne = (1 << scale) * ef
    u = np.empty(ne, np.int32)
    v = np.empty(ne, np.int32)
    rc = _lib().gg_rmat_edges(scale, ef, a, b, c, seed & (2**64 - 1), int(permute),
                              _p(u, ctypes.c_int32), _p(v, ctypes.c_int32))
    if rc:
        raise ValueError(f"gg_rmat_edges failed ({rc})")
    return u, v


def csr_from_edges(n: int, u, v, name: str = "") -> CSR:
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    assert u.shape == v.shape
    row_ptr = np.empty(n + 1, np.int64)
    col = np.empty(max(1, 2 * len(u)), np.int32)
    nnz = ctypes.c_int64(0)
    rc = _lib().gg_normalize(n, len(u), _p(u, ctypes.c_int32), _p(v, ctypes.c_int32),
                             _p(row_ptr, ctypes.c_int64), _p(col, ctypes.c_int32), ctypes.byref(nnz))
    if rc:
        raise ValueError(f"gg_normalize failed ({rc})")
    return CSR(n, row_ptr, col[: nnz.value].copy(), name)


def rmat(scale: int, ef: int, seed: int = 1, permute: bool = True) -> CSR:
    u, v = rmat_edges(scale, ef, seed, permute=permute)
    g = csr_from_edges(1 << scale, u, v, name=f"rmat{scale}_ef{ef}_s{seed}")
    return g


def grid(R: int, C: int) -> CSR:
    n = R * C
    nnz = 2 * (R * (C - 1) + C * (R - 1))
    row_ptr = np.empty(n + 1, np.int64)
    col = np.empty(max(1, nnz), np.int32)
    rc = _lib().gg_grid(R, C, _p(row_ptr, ctypes.c_int64), _p(col, ctypes.c_int32))
    if rc:
        raise ValueError("gg_grid failed")
    return CSR(n, row_ptr, col[:nnz], name=f"grid{R}x{C}")


def sample_sources(g: CSR, count: int, seed: int = 2) -> np.ndarray:
    """Uniform, without replacement, among non-isolated vertices (PAPER.md:840 fn.)."""
    out = np.empty(count, np.int32)
    rc = _lib().gg_sample_sources(g.n, _p(g.row_ptr, ctypes.c_int64), count, seed, _p(out, ctypes.c_int32))
    if rc:
        raise ValueError("not enough non-isolated vertices to sample")
    return out


# ------------------------------------------------------------ small families
def from_pairs(n: int, pairs, name: str = "") -> CSR:
    pairs = np.asarray(list(pairs), dtype=np.int64).reshape(-1, 2)
    return csr_from_edges(n, pairs[:, 0], pairs[:, 1], name)


def path(n: int) -> CSR:
    return from_pairs(n, [(i, i + 1) for i in range(n - 1)], f"P{n}")


def cycle(n: int) -> CSR:
    return from_pairs(n, [(i, (i + 1) % n) for i in range(n)], f"C{n}")


def complete(n: int) -> CSR:
    return from_pairs(n, [(i, j) for i in range(n) for j in range(i + 1, n)], f"K{n}")


def star(k: int) -> CSR:
    """K_{1,k}; centre is vertex 0."""
    return from_pairs(k + 1, [(0, i) for i in range(1, k + 1)], f"K1,{k}")


def complete_bipartite(a: int, b: int) -> CSR:
    return from_pairs(a + b, [(i, a + j) for i in range(a) for j in range(b)], f"K{a},{b}")


def hypercube(d: int) -> CSR:
    n = 1 << d
    x = np.arange(n, dtype=np.int64)
    us, vs = [], []
    for k in range(d):
        y = x ^ (1 << k)
        keep = x < y
        us.append(x[keep])
        vs.append(y[keep])
    u = np.concatenate(us) if us else np.zeros(0, np.int64)
    v = np.concatenate(vs) if vs else np.zeros(0, np.int64)
    return csr_from_edges(n, u, v, f"Q{d}")


def petersen() -> CSR:
    outer = [(i, (i + 1) % 5) for i in range(5)]
    spokes = [(i, i + 5) for i in range(5)]
    inner = [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
    return from_pairs(10, outer + spokes + inner, "Petersen")


def random_tree(n: int, seed: int) -> CSR:
    rng = np.random.default_rng(seed)
    pairs = [(i, int(rng.integers(0, i))) for i in range(1, n)]
    return from_pairs(n, pairs, f"tree{n}_s{seed}")


def erdos_renyi(n: int, p: float, seed: int) -> CSR:
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < p
    return csr_from_edges(n, iu[keep], ju[keep], f"ER{n}_{p}_s{seed}")


def disjoint_union(*gs: CSR) -> CSR:
    off = 0
    us, vs = [], []
    for g in gs:
        src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
        us.append(src + off)
        vs.append(g.col.astype(np.int64) + off)
        off += g.n
    u = np.concatenate(us) if us else np.zeros(0, np.int64)
    v = np.concatenate(vs) if vs else np.zeros(0, np.int64)
    return csr_from_edges(off, u, v, "+".join(g.name for g in gs))


def with_isolated(g: CSR, k: int) -> CSR:
    row_ptr = np.concatenate([g.row_ptr, np.full(k, g.row_ptr[-1], np.int64)])
    return CSR(g.n + k, row_ptr, g.col.copy(), g.name + f"+{k}iso")


def edges_of(g: CSR):
    """Unique undirected edges (u < v) as an int64 [m, 2] array."""
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
    keep = src < g.col
    return np.stack([src[keep], g.col[keep].astype(np.int64)], axis=1)
