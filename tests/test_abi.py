"""CPU checks of the C ABI: the library builds / loads and exports every symbol include/*.h declares.
No compute call is made (there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparse_mlp.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sparse_mlp_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2102_01732_b200 import build as B
    path = B.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary_calls():
    names = declared_functions()
    for required in ("sparse_mlp_create", "sparse_mlp_forward", "sparse_mlp_backward", "sparse_mlp_step",
                     "sparse_mlp_evolve_topology", "sparse_mlp_prune_neurons"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    from paper_2102_01732_b200 import sparse_mlp as S
    assert sorted(S.EXPORTED) == declared_functions()


def test_version_and_create_errors_without_gpu(lib):
    """Argument validation happens before any device call, so it is testable on CPU."""
    from paper_2102_01732_b200 import sparse_mlp as S
    L = S.load_library()
    assert b"sm_100a" in L.sparse_mlp_version()
    h = ctypes.c_void_p()
    sizes = (ctypes.c_int64 * 2)(4, 2)
    cfg = S.smlp_config(2, sizes, 1.0, 1, 0.5, 0.0, 2, 0, 0, 8, 0, 0, None, None)
    assert L.sparse_mlp_create(ctypes.byref(cfg), ctypes.byref(h)) == -1          # L < 3
    assert b"n_layers" in L.sparse_mlp_last_error(None)
    sizes3 = (ctypes.c_int64 * 3)(4, 3, 2)
    cfg = S.smlp_config(3, sizes3, 1.0, 1, 0.5, 1.5, 2, 0, 0, 8, 0, 0, None, None)
    assert L.sparse_mlp_create(ctypes.byref(cfg), ctypes.byref(h)) == -1          # dropout >= 1
    cfg = S.smlp_config(3, sizes3, 1.0, 1, 0.5, 0.0, 2, 0, 0, 8, 48, 0, None, None)
    assert L.sparse_mlp_create(ctypes.byref(cfg), ctypes.byref(h)) == -1          # chunk_batch not pow2
    cfg = S.smlp_config(3, sizes3, -1.0, 1, 0.5, 0.0, 2, 0, 0, 8, 0, 0, None, None)
    assert L.sparse_mlp_create(ctypes.byref(cfg), ctypes.byref(h)) == -1          # eps <= 0
    assert L.sparse_mlp_destroy(None) == 0
