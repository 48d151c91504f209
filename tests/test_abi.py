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


def test_chunk_plan_rule_without_gpu(lib):
    """The chunk widths create picks, as a host-only call: L2-resident slabs,
    a narrower forward slab when the backward's exceeds half the L2, and the widest chunk when no
    32-column slab fits at all."""
    from paper_2102_01732_b200.sparse_mlp import plan_chunks
    from synth import get_config
    l2 = 126 * 2**20 + 2**19                                           # B200: 126.5 MiB
    want = {"C1": (128, 128), "C2": (128, 128), "C3": (8, 8), "C4": (128, 128), "C5": (64, 32),
            "T1": (64, 32), "T2": (128, 128), "T3": (128, 128), "T4": (128, 128), "T5": (128, 128)}
    for name, cbs in want.items():
        cfg = get_config(name)
        assert plan_chunks(cfg.sizes, cfg.batch, 0, l2) == cbs, name
    assert plan_chunks((100, 50, 10), 37, 0, l2) == (64, 64)           # next_pow2(37)
    assert plan_chunks((100, 50, 10), 3, 0, l2) == (4, 4)              # never below 4
    assert plan_chunks((500_000, 10), 128, 32, l2) == (32, 32)         # explicit: both widths
    assert plan_chunks((100_000, 10), 128, 0, l2) == (128, 128)        # 51 MB slab
    assert plan_chunks((200_000, 10), 128, 0, l2) == (128, 64)         # 102 MB > L2 / 2 -> 51 MB forward
    assert plan_chunks((300_000, 10), 128, 0, l2) == (64, 32)          # 77 MB backward slab, 38 MB forward
    assert plan_chunks((1_100_000, 10), 128, 0, l2) == (128, 128)      # 141 MB at 32 columns > L2
    with pytest.raises(ValueError):
        plan_chunks((100, 10), 128, 48, l2)                             # not a power of two
    with pytest.raises(ValueError):
        plan_chunks((100, 10), 0, 0, l2)                                # max_batch < 1
