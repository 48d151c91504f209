"""Helpers shared by the GPU parity tests: build the CUDA-side model and the oracle state from the
same seeded configuration, move an ORACLE state into the GPU model (never the other way), and
compare.  Only tests import this module."""
from __future__ import annotations

import numpy as np

from oracle import model as M
from oracle.compare import int_mismatch, rel_err

TOL = 1e-4          # BASELINE.json north_star: max relative error 1e-4 per step (fp32)


def pair(cfg, seed=None, max_batch=None, chunk_batch=0, dropout=None):
    from paper_2102_01732_b200 import SparseMLP
    seed = cfg.model_seed if seed is None else seed
    drop = cfg.dropout if dropout is None else dropout
    g = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, drop, cfg.init, seed, 0,
                  max_batch or cfg.batch, chunk_batch)
    st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, drop, cfg.init, seed)
    return g, st


def load_oracle_state_into_gpu(g, st):
    """Op-by-op parity: the GPU op runs on the oracle's pre-op state (identical inputs); the
    oracle's running error bound restarts at zero (R24)."""
    st.reset_error()
    for Ly in st.layers:
        g.import_layer(Ly.l, Ly.row_ptr.astype(np.int32), Ly.col, Ly.w, Ly.v)
        g.sparse_mlp_import_bias(Ly.l, st.b[Ly.l - 2], st.vb[Ly.l - 2])
    for l in range(1, st.L + 1):
        g.sparse_mlp_import_alive(l, st.alive[l - 1])


def assert_topology_equal(g, st, what=""):
    for Ly in st.layers:
        e = g.export_layer(Ly.l)
        mm = int_mismatch(e["row_ptr"], Ly.row_ptr.astype(np.int32))
        assert mm is None, f"{what} W^({Ly.l}) row_ptr mismatch {mm}"
        mm = int_mismatch(e["col"], Ly.col)
        assert mm is None, f"{what} W^({Ly.l}) col mismatch {mm}"
    for l in range(1, st.L + 1):
        assert np.array_equal(g.sparse_mlp_export_alive(l), st.alive[l - 1]), f"{what} alive[{l}]"


def assert_values_bitexact(g, st, what=""):
    for Ly in st.layers:
        e = g.export_layer(Ly.l)
        mm = int_mismatch(e["w"].view(np.uint32), Ly.w.view(np.uint32))
        assert mm is None, f"{what} W^({Ly.l}) values differ {mm}"
        mm = int_mismatch(e["v"].view(np.uint32), Ly.v.view(np.uint32))
        assert mm is None, f"{what} W^({Ly.l}) momentum differs {mm}"


def assert_values_close(g, st, tol=TOL, what=""):
    """Weights, momenta and biases of every layer within the R24 metric (the oracle's running
    error magnitudes of its state as the fp32 bound)."""
    for Ly in st.layers:
        e = g.export_layer(Ly.l)
        err = rel_err(e["w"], Ly.w, Ly.wmag)
        assert err <= tol, f"{what} W^({Ly.l}) w err {err}"
        if np.any(Ly.v != 0):
            err = rel_err(e["v"], Ly.v, Ly.vmag)
            assert err <= tol, f"{what} W^({Ly.l}) v err {err}"
        b, vb = g.sparse_mlp_export_bias(Ly.l)
        bm = None if st.bmag is None else st.bmag[Ly.l - 2]
        err = rel_err(b, st.b[Ly.l - 2], bm)
        assert err <= tol, f"{what} b_{Ly.l} err {err}"


def to_dev(a, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.cuda() if dtype is None else t.to(dtype).cuda()


def check_and_resync(g, st, what="", tol=TOL):
    """Per-step parity (BASELINE.json north_star: "within 1e-4 ... per step"): compare the GPU
    state with the oracle's after this step, then give the GPU the oracle's state so the next step
    starts from identical inputs (the oracle's R24 bound is a single-step bound; free-running
    accumulation is what the 5-epoch loss-curve tests hold to 1e-3)."""
    assert_values_close(g, st, tol, what)
    load_oracle_state_into_gpu(g, st)
