"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain CPU reference for the BC hot path (Alg.1, Eq.2-5, Alg.6).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA path and the CUDA path never imports it.

* ``brandes.c`` (built into ``liboracle.so``): textbook Brandes Alg.1 with
  predecessor lists and a stack, fp64 + uint64/overflow sigma; Alg.6
  pruning; the Eq.(4)/(5) pruned BC with DESIGN.md readings R7-R13.
* ``brute.py``: exact-rational all-pairs definition Eq.(1) for tiny graphs.

Every function is pinned by ``tests/test_oracle_*.py`` against brute force,
closed forms and invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib_handle = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "brandes.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", src, "-o", _SO])
    return _SO


def _lib():
    global _lib_handle
    if _lib_handle is None:
        build()
        L = ctypes.CDLL(_SO)
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        f64p = ctypes.POINTER(ctypes.c_double)
        L.oracle_bc.argtypes = [ctypes.c_int64, i64p, i32p, i32p, ctypes.c_int64, ctypes.c_int, f64p, i64p]
        L.oracle_sssp.argtypes = [ctypes.c_int64, i64p, i32p, ctypes.c_int32, i32p, u64p, u8p, f64p, f64p]
        L.oracle_prune_degree1.argtypes = [ctypes.c_int64, i64p, i32p, u32p, u8p, i64p, i32p, i64p]
        L.oracle_prune_degree1_share.argtypes = [ctypes.c_int64, i64p, i32p, ctypes.c_int, ctypes.c_int, u32p, u32p]
        L.oracle_bc_pruned.argtypes = [ctypes.c_int64, i64p, i32p, i32p, ctypes.c_int64, ctypes.c_int, f64p]
        L.oracle_two_degree_tree.argtypes = [ctypes.c_int64, ctypes.c_int32, i32p, u64p, u8p, i32p, u64p, u8p, i32p,
                                             u64p, u8p]
        L.oracle_num_threads.restype = ctypes.c_int
        _lib_handle = L
    return _lib_handle


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _csr(g):
    return (int(g.n), np.ascontiguousarray(g.row_ptr, np.int64), np.ascontiguousarray(g.col, np.int32))


def num_threads() -> int:
    return int(_lib().oracle_num_threads())


def bc(g, sources=None, threads: int = 0, stats: bool = False):
    """Eq.(3) over ``sources`` (default: every vertex; isolated ones add 0)."""
    n, rp, col = _csr(g)
    src = np.arange(n, dtype=np.int32) if sources is None else np.ascontiguousarray(sources, np.int32)
    out = np.zeros(n, np.float64)
    st = np.zeros((len(src), 3), np.int64) if stats else None
    rc = _lib().oracle_bc(n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), _p(src, ctypes.c_int32),
                          len(src), threads, _p(out, ctypes.c_double),
                          _p(st, ctypes.c_int64) if stats else None)
    if rc:
        raise RuntimeError(f"oracle_bc failed ({rc})")
    return (out, st) if stats else out


def sssp(g, s: int):
    """(depth int32, sigma uint64, overflow uint8, sigma fp64, delta fp64) for source s."""
    n, rp, col = _csr(g)
    d = np.empty(n, np.int32)
    su = np.empty(n, np.uint64)
    ov = np.empty(n, np.uint8)
    sf = np.empty(n, np.float64)
    de = np.empty(n, np.float64)
    rc = _lib().oracle_sssp(n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), int(s),
                            _p(d, ctypes.c_int32), _p(su, ctypes.c_uint64), _p(ov, ctypes.c_uint8),
                            _p(sf, ctypes.c_double), _p(de, ctypes.c_double))
    if rc:
        raise RuntimeError("oracle_sssp failed")
    return d, su, ov, sf, de


def two_degree_tree(g, c: int, literal_alg7: bool = False):
    """Alg.7 / Eq.(6): (depth, sigma uint64, overflow) of the 2-degree vertex
    ``c`` derived from the oracle BFS trees of its two neighbours (Lemma 1).
    ``literal_alg7`` evaluates the listing as printed (its ``else`` overwrites
    the equal-level case, reading R23) -- only for the test that shows it is
    wrong."""
    n, rp, col = _csr(g)
    if rp[c + 1] - rp[c] != 2:
        raise ValueError("c must have degree 2")
    a, b = int(col[rp[c]]), int(col[rp[c] + 1])
    da, sa, oa, _, _ = sssp(g, a)
    db, sb, ob, _, _ = sssp(g, b)
    if literal_alg7:
        # PAPER.md:703-716 line by line, unreached = infinity
        inf = np.iinfo(np.int64).max
        la = np.where(da < 0, inf, da.astype(np.int64))
        lb = np.where(db < 0, inf, db.astype(np.int64))
        sc = np.zeros(n, np.uint64)
        lc = np.full(n, inf, np.int64)
        for v in range(n):
            if la[v] == lb[v]:
                sc[v] = sa[v] + sb[v]
                lc[v] = la[v] + 1
            if la[v] < lb[v]:
                sc[v] = sa[v]
                lc[v] = la[v] + 1
            else:
                sc[v] = sb[v]
                lc[v] = lb[v] + 1
        return lc, sc
    dc = np.empty(n, np.int32)
    sc = np.empty(n, np.uint64)
    oc = np.empty(n, np.uint8)
    _lib().oracle_two_degree_tree(n, int(c), _p(da, ctypes.c_int32), _p(sa, ctypes.c_uint64), _p(oa, ctypes.c_uint8),
                                  _p(db, ctypes.c_int32), _p(sb, ctypes.c_uint64), _p(ob, ctypes.c_uint8),
                                  _p(dc, ctypes.c_int32), _p(sc, ctypes.c_uint64), _p(oc, ctypes.c_uint8))
    return dc, sc, oc


def prune_degree1(g):
    """Alg.6: (omega uint32[n], removed uint8[n], residual row_ptr, residual col)."""
    n, rp, col = _csr(g)
    om = np.empty(n, np.uint32)
    rm = np.empty(n, np.uint8)
    rrp = np.empty(n + 1, np.int64)
    rcol = np.empty(max(1, len(col)), np.int32)
    nnz = ctypes.c_int64(0)
    _lib().oracle_prune_degree1(n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), _p(om, ctypes.c_uint32),
                                _p(rm, ctypes.c_uint8), _p(rrp, ctypes.c_int64), _p(rcol, ctypes.c_int32),
                                ctypes.byref(nnz))
    return om, rm, rrp, rcol[: nnz.value].copy()


def prune_degree1_share(g, nprocs: int, i: int):
    """Alg.6 on processor i of nprocs (edges (u,v) with u mod nprocs = i):
    (omega_part uint32[n], removed_part uint32[n]); the sums over i are
    prune_degree1's omega and removed."""
    n, rp, col = _csr(g)
    om = np.empty(n, np.uint32)
    rm = np.empty(n, np.uint32)
    rc = _lib().oracle_prune_degree1_share(n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), int(nprocs), int(i),
                                           _p(om, ctypes.c_uint32), _p(rm, ctypes.c_uint32))
    if rc != 0:
        raise ValueError("processor index out of range")
    return om, rm


def bc_pruned(g, sources=None, threads: int = 0):
    """Eq.(4)/(5) BC with 1-degree reduction (readings R7-R13)."""
    n, rp, col = _csr(g)
    out = np.zeros(n, np.float64)
    if sources is None:
        sp, ns = None, 0
    else:
        src = np.ascontiguousarray(sources, np.int32)
        sp, ns = _p(src, ctypes.c_int32), len(src)
    rc = _lib().oracle_bc_pruned(n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), sp, ns, threads,
                                 _p(out, ctypes.c_double))
    if rc == 1:
        raise ValueError("source removed by 1-degree pruning")
    if rc:
        raise RuntimeError(f"oracle_bc_pruned failed ({rc})")
    return out
