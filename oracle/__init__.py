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
        L.oracle_bc_pruned.argtypes = [ctypes.c_int64, i64p, i32p, i32p, ctypes.c_int64, ctypes.c_int, f64p]
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
