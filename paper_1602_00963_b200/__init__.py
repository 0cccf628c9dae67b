"""paper_1602_00963_b200 -- B200-native exact Brandes betweenness centrality.

Thin Python binding (same names as include/bc.h) over ``libbcb200.so``.
It only marshals arguments: CSR upload, pruning, the forward/backward level
loop and the BC update all run in the library's sm_100a kernels.  PyTorch is
optional here and used only for device tensors / streams (``out=`` a CUDA
tensor) and for ``torch.distributed`` in :mod:`.dist`.

    g = Graph(row_ptr, col, device=0)     # bc_graph_create
    g.prune_degree1()                     # bc_prune_degree1 (Alg.6)
    bc = g.compute(sources)               # bc_compute -> numpy float64[n]
    g.close()                             # bc_destroy
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as _L

__all__ = ["Graph", "BCError", "build", "BC_CREATE_VALIDATE", "OPT_LANE_WORDS", "OPT_HUB_DEGREE",
           "OPT_PROFILE", "OPT_MODE", "OPT_RELABEL", "OPT_SOURCE_ORDER", "OPT_FWD_PUSH",
           "OPT_BWD_MODE", "OPT_SIGMA_WIDTH", "OPT_STREAMS", "OPT_TWO_DEGREE", "OPT_DEVICE_LOOP",
           "OPT_SLICES_KERNEL"]

BC_CREATE_VALIDATE = 0x1
OPT_LANE_WORDS, OPT_HUB_DEGREE, OPT_PROFILE, OPT_MODE, OPT_RELABEL, OPT_SOURCE_ORDER, OPT_FWD_PUSH = 1, 2, 3, 4, 5, 6, 7
OPT_BWD_MODE = 8
OPT_SIGMA_WIDTH = 9
OPT_STREAMS = 10
OPT_TWO_DEGREE = 11
OPT_DEVICE_LOOP = 12
OPT_SLICES_KERNEL = 13
build = _L.build


class BCError(RuntimeError):
    def __init__(self, status: int, detail: str):
        lib = _L.load()
        name = lib.bc_status_string(status).decode()
        super().__init__(f"{name}: {detail}")
        self.status = status
        self.name = name


def _check(status: int):
    if status != 0:
        raise BCError(status, _L.load().bc_last_error().decode())


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


_EMPTY = np.zeros(1, np.int32)


class Graph:
    """A graph resident on one CUDA device (bc_graph handle)."""

    def __init__(self, row_ptr, col, device: int = 0, validate: bool = False):
        lib = _L.load()
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col, dtype=np.int32)
        self.n = int(len(rp) - 1)
        self.device = int(device)
        h = ctypes.c_void_p()
        _check(lib.bc_graph_create(self.n, _ptr(rp), _ptr(ci) if len(ci) else None, self.device,
                                   BC_CREATE_VALIDATE if validate else 0, ctypes.byref(h)))
        self._h = h
        self.pruned = False

    @classmethod
    def from_csr(cls, csr, device: int = 0, validate: bool = False):
        return cls(csr.row_ptr, csr.col, device=device, validate=validate)

    # --------------------------------------------------------------- lifecycle
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _L.load().bc_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --------------------------------------------------------------- the path
    def prune_degree1(self) -> int:
        removed = ctypes.c_int64(0)
        _check(_L.load().bc_prune_degree1(self._h, ctypes.byref(removed)))
        self.pruned = True
        return int(removed.value)

    def prune_degree1_share(self, rank: int, nranks: int, omega_part, removed_part, stream=None):
        """Alg.6 share of processor ``rank`` of ``nranks`` (u mod nranks =
        rank) into two torch uint32/int32 CUDA tensors of n elements,
        stream-ordered on ``stream`` (default: torch's current stream)."""
        import torch

        for t in (omega_part, removed_part):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.numel() == self.n and t.element_size() == 4
                    and t.is_contiguous()):
                raise ValueError("share outputs must be contiguous 4-byte CUDA tensors of n elements")
        st = stream if stream is not None else torch.cuda.current_stream(omega_part.device)
        _check(_L.load().bc_prune_degree1_share(self._h, int(rank), int(nranks), omega_part.data_ptr(),
                                                removed_part.data_ptr(), st.cuda_stream))

    def prune_degree1_apply(self, omega, removed, stream=None) -> int:
        """Residual graph from the summed shares (see bc.h); returns the
        number of removed vertices."""
        import torch

        for t in (omega, removed):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.numel() == self.n and t.element_size() == 4
                    and t.is_contiguous()):
                raise ValueError("inputs must be contiguous 4-byte CUDA tensors of n elements")
        st = stream if stream is not None else torch.cuda.current_stream(omega.device)
        r = ctypes.c_int64(0)
        _check(_L.load().bc_prune_degree1_apply(self._h, omega.data_ptr(), removed.data_ptr(), st.cuda_stream,
                                                ctypes.byref(r)))
        self.pruned = True
        return int(r.value)

    def compute(self, sources=None, out=None, stream=None):
        """BC over ``sources`` (None = all / all eligible).

        ``out``: None (returns a new numpy float64[n]), a numpy float64[n]
        (host, synchronous) or a torch float64 CUDA tensor (device,
        stream-ordered on ``stream`` or torch's current stream)."""
        lib = _L.load()
        if sources is None:
            sp, ns, keep = None, 0, None
        else:
            keep = np.ascontiguousarray(sources, dtype=np.int32)
            ns = len(keep)
            sp = _ptr(keep) if ns else _ptr(_EMPTY)  # non-NULL pointer: explicitly empty set
        if out is None:
            out = np.empty(self.n, np.float64)
        if isinstance(out, np.ndarray):
            if out.dtype != np.float64 or out.shape != (self.n,) or not out.flags.c_contiguous:
                raise ValueError("out must be a contiguous float64[n] array")
            _check(lib.bc_compute(self._h, sp, ns, _ptr(out), None))
            return out
        # torch tensor
        import torch

        if not (out.is_cuda and out.dtype == torch.float64 and out.is_contiguous() and out.numel() == self.n):
            raise ValueError("out must be a contiguous float64 CUDA tensor of n elements")
        st = stream if stream is not None else torch.cuda.current_stream(out.device)
        _check(lib.bc_compute(self._h, sp, ns, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
        return out

    def sssp(self, source: int):
        """(depth int32, sigma uint64, overflow uint8, delta float64) of the
        unpruned graph (a pruned handle traverses the residual graph and
        fills the removed vertices)."""
        d = np.empty(self.n, np.int32)
        s = np.empty(self.n, np.uint64)
        o = np.empty(self.n, np.uint8)
        de = np.empty(self.n, np.float64)
        _check(_L.load().bc_sssp(self._h, int(source), _ptr(d), _ptr(s), _ptr(o), _ptr(de)))
        return d, s, o, de

    def compute_captured(self, sources=None, capture=(), out=None, stream=None):
        """bc_set_capture + bc_compute: the BC over ``sources`` (as
        :meth:`compute`) and, for each vertex of ``capture``, the per-source
        state the production kernels of that call computed:
        ``(bc, depth int32[c, n], sigma float64[c, n], delta float64[c, n],
        tier int32[c])``."""
        cap = np.ascontiguousarray(capture, dtype=np.int32)
        c = len(cap)
        depth = np.empty((c, self.n), np.int32)
        sigma = np.empty((c, self.n), np.float64)
        delta = np.empty((c, self.n), np.float64)
        tier = np.empty(max(c, 1), np.int32)
        _check(_L.load().bc_set_capture(self._h, _ptr(cap) if c else None, c, _ptr(depth), _ptr(sigma),
                                        _ptr(delta), _ptr(tier)))
        bc = self.compute(sources, out=out, stream=stream)
        return bc, depth, sigma, delta, tier[:c]

    def set_option(self, option: int, value: int):
        _check(_L.load().bc_set_option(self._h, int(option), int(value)))

    def stats(self) -> dict:
        st = _L.bc_stats()
        _check(_L.load().bc_get_stats(self._h, ctypes.byref(st)))
        return st.as_dict()

    def pruning(self):
        """(omega uint32[n], removed uint8[n], residual row_ptr int64[n+1], residual col int32)."""
        lib = _L.load()
        nnz = ctypes.c_int64(0)
        n_, nnz0, rnnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        dev = ctypes.c_int()
        _check(lib.bc_graph_info(self._h, ctypes.byref(n_), ctypes.byref(nnz0), ctypes.byref(rnnz), ctypes.byref(dev)))
        om = np.empty(self.n, np.uint32)
        rm = np.empty(self.n, np.uint8)
        rp = np.empty(self.n + 1, np.int64)
        col = np.empty(max(1, rnnz.value), np.int32)
        _check(lib.bc_get_pruning(self._h, _ptr(om), _ptr(rm), _ptr(rp), _ptr(col), ctypes.byref(nnz)))
        return om, rm, rp, col[: nnz.value].copy()

    def info(self) -> dict:
        n_, nnz0, rnnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        dev = ctypes.c_int()
        _check(_L.load().bc_graph_info(self._h, ctypes.byref(n_), ctypes.byref(nnz0), ctypes.byref(rnnz),
                                       ctypes.byref(dev)))
        return {"n": n_.value, "nnz": nnz0.value, "res_nnz": rnnz.value, "device": dev.value}
