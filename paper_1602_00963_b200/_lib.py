"""ctypes loader of libbcb200.so (the C ABI of include/bc.h).

Argument marshalling only: every step of the BC path runs in the CUDA
kernels behind this library.  There is no CPU fallback -- if the shared
library is missing or fails to load, the import of the binding raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO = os.environ.get("BC_SO") or os.path.join(PKG, "libbcb200.so")
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def _sources():
    out = [os.path.join(INCLUDE, "bc.h")]
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cuh", ".h")):
            out.append(os.path.join(CSRC, f))
    return out


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libbcb200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    if not force and not needs_build():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-I" + INCLUDE, "-o", SO + ".tmp", os.path.join(CSRC, "bc_api.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    os.replace(SO + ".tmp", SO)
    if verbose:
        print(res.stderr)
    return SO


class bc_stats(ctypes.Structure):
    _fields_ = [
        ("num_sources", ctypes.c_int64), ("num_trivial", ctypes.c_int64), ("batches", ctypes.c_int64),
        ("lanes", ctypes.c_int64), ("levels_total", ctypes.c_int64), ("fwd_launches", ctypes.c_int64),
        ("bwd_launches", ctypes.c_int64), ("reached", ctypes.c_int64), ("adj_reached", ctypes.c_int64),
        ("dag_edges", ctypes.c_int64), ("fwd_ms", ctypes.c_double), ("bwd_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double), ("kernel_launches", ctypes.c_int64), ("dist_sum", ctypes.c_int64),
        ("fwd_items", ctypes.c_int64), ("fwd_hits", ctypes.c_int64), ("bwd_items", ctypes.c_int64),
        ("bwd_hits", ctypes.c_int64), ("bwd_fin_ms", ctypes.c_double), ("bwd_push_ms", ctypes.c_double),
        ("narrow_batches", ctypes.c_int64), ("narrow_fallbacks", ctypes.c_int64), ("mid_batches", ctypes.c_int64),
        ("derived_lanes", ctypes.c_int64), ("widened_batches", ctypes.c_int64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# exported symbols of include/bc.h and their signatures
_i64, _i32, _u32, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p
SIGNATURES = {
    "bc_graph_create": (ctypes.c_int, [_i64, _vp, _vp, ctypes.c_int, _u32, ctypes.POINTER(_vp)]),
    "bc_prune_degree1": (ctypes.c_int, [_vp, ctypes.POINTER(_i64)]),
    "bc_prune_degree1_share": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "bc_prune_degree1_apply": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.POINTER(_i64)]),
    "bc_compute": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "bc_destroy": (ctypes.c_int, [_vp]),
    "bc_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "bc_last_error": (ctypes.c_char_p, []),
    "bc_sssp": (ctypes.c_int, [_vp, _i32, _vp, _vp, _vp, _vp]),
    "bc_set_capture": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "bc_set_option": (ctypes.c_int, [_vp, ctypes.c_int, _i64]),
    "bc_get_stats": (ctypes.c_int, [_vp, ctypes.POINTER(bc_stats)]),
    "bc_get_pruning": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, ctypes.POINTER(_i64)]),
    "bc_graph_info": (ctypes.c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                     ctypes.POINTER(ctypes.c_int)]),
}

_lib = None


def load(auto_build: bool = True):
    """Load (building first if stale) the CUDA library; raises if unavailable."""
    global _lib
    if _lib is None:
        # an explicitly chosen library (BC_SO, e.g. an experiment build with
        # its own -D defines) is never rebuilt with the default flags
        if auto_build and not os.environ.get("BC_SO") and needs_build():
            build()
        if not os.path.exists(SO):
            raise ImportError(f"libbcb200.so not built ({SO}); run __graft_entry__.build()")
        L = ctypes.CDLL(SO)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
