"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a,
loads, exports every function include/bc.h declares, and fails loudly (an
error status, not a crash or a CPU fallback) when no GPU is present."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "bc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bc_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_1602_00963_b200 import _lib

    _lib.build()
    return ctypes.CDLL(_lib.SO)


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("bc_graph_create", "bc_prune_degree1", "bc_compute", "bc_destroy", "bc_sssp"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_1602_00963_b200 import _lib

    for name in _declared():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"binding lacks {name}"


def test_library_is_sm100a_code():
    from paper_1602_00963_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_null_safety(lib):
    lib.bc_status_string.restype = ctypes.c_char_p
    assert lib.bc_status_string(0) == b"BC_OK"
    assert lib.bc_status_string(4) == b"BC_ERR_STATE"
    assert lib.bc_destroy(None) == 0


def test_create_rejects_bad_arguments_without_touching_the_gpu(lib):
    import graphgen as gg

    g = gg.path(4)
    h = ctypes.c_void_p()
    rp = np.ascontiguousarray(g.row_ptr, np.int64)
    col = np.ascontiguousarray(g.col, np.int32)
    lib.bc_graph_create.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32,
                                    ctypes.POINTER(ctypes.c_void_p)]
    assert lib.bc_graph_create(0, rp.ctypes.data, col.ctypes.data, 0, 0, ctypes.byref(h)) == 1
    bad = rp.copy()
    bad[2] = 0  # decreasing
    assert lib.bc_graph_create(4, bad.ctypes.data, col.ctypes.data, 0, 0, ctypes.byref(h)) == 1


def test_no_gpu_means_cuda_error_not_fallback(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import graphgen as gg

    g = gg.path(4)
    h = ctypes.c_void_p()
    rp = np.ascontiguousarray(g.row_ptr, np.int64)
    col = np.ascontiguousarray(g.col, np.int32)
    assert lib.bc_graph_create(4, rp.ctypes.data, col.ctypes.data, 0, 0, ctypes.byref(h)) == 3
    import paper_1602_00963_b200 as bcb

    with pytest.raises(bcb.BCError):
        bcb.Graph(g.row_ptr, g.col)


def test_distributed_pruning_entry_points_reject_bad_arguments(lib):
    """bc_prune_degree1_share / _apply (NEXT-4) fail with BC_ERR_INVALID on a
    NULL handle, before touching any device."""
    from paper_1602_00963_b200 import _lib

    fn = lib.bc_prune_degree1_share
    fn.restype, fn.argtypes = _lib.SIGNATURES["bc_prune_degree1_share"]
    assert fn(None, 0, 1, None, None, None) == 1
    fn = lib.bc_prune_degree1_apply
    fn.restype, fn.argtypes = _lib.SIGNATURES["bc_prune_degree1_apply"]
    r = ctypes.c_int64(0)
    assert fn(None, None, None, None, ctypes.byref(r)) == 1
