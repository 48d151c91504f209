"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element, on the same
seeded inputs (SURVEY.md §8(c) comparison metric).  Topology / CSR / integer decisions bit-exact;
fp32 values within max relative error 1e-4 per step."""
import numpy as np
import pytest

from oracle import model as M
from oracle import topology as T
from oracle.compare import int_mismatch, rel_err
from synth import get_config, make_dataset
from tests.gpu_helpers import (TOL, assert_topology_equal, assert_values_bitexact, assert_values_close,
                               check_and_resync, load_oracle_state_into_gpu, pair, to_dev)

pytestmark = pytest.mark.gpu

SMALL = ["C1", "C2", "C4", "C3"]


def _torch():
    import torch
    return torch


def _batch(cfg, st, B=None, step=0, tries=12):
    """A seeded batch whose hidden pre-activations are not within fp32 rounding of the All-ReLU
    kink (R32): the first of `tries` candidate batches the oracle reports kink-free."""
    B = B or cfg.batch
    X, y = make_dataset(cfg, n=B * tries)
    for t in range(tries):
        x, yy = X[t * B:(t + 1) * B], y[t * B:(t + 1) * B]
        tr = M.forward(st, x, True, step)
        if sum(tr.ambiguous) == 0:
            return x, yy, tr
    raise AssertionError("no kink-free batch among the candidates")


def _tiny(**kw):
    base = dict(sizes=(37, 45, 33, 7), epsilon=3.0, alpha=0.6, dropout=0.25, init="he_uniform", batch=13)
    base.update(kw)
    return get_config("C1", **base)


# ----------------------------------------------------------------------------------------- init
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_er_init_bitexact(name):
    cfg = get_config(name)
    g, st = pair(cfg)
    assert_topology_equal(g, st, name)
    if cfg.init == "normal":
        # Box-Muller through libm / CUDA fp64 log and cos: positions are exact, values agree to
        # the last bits of fp64 (reading R3) -> compare within 1e-6
        for Ly in st.layers:
            e = g.export_layer(Ly.l)
            assert rel_err(e["w"], Ly.w) < 1e-6
    else:
        assert_values_bitexact(g, st, name)
    inf = g.info()
    assert inf["nnz"][1:] == [Ly.nnz for Ly in st.layers]
    assert inf["dense_capped"][1:] == [int(Ly.dense_capped) for Ly in st.layers]


# ----------------------------------------------------------------------------------------- forward
@pytest.mark.parametrize("name", SMALL + ["tiny"])
def test_forward_parity(name):
    torch = _torch()
    cfg = _tiny() if name == "tiny" else get_config(name)
    g, st = pair(cfg)
    x, y, tr = _batch(cfg, st, step=3)
    B = len(x)
    probs = torch.empty((B, cfg.sizes[-1]), dtype=torch.float32, device="cuda")
    g.forward(to_dev(x), train=True, step=3, probs=probs)
    torch.cuda.synchronize()
    for l in range(1, cfg.n_layers):
        a = g.sparse_mlp_export_trace(0, l, B)
        assert rel_err(a, tr.a[l - 1], tr.amag[l - 1]) <= TOL, (name, l, rel_err(a, tr.a[l - 1], tr.amag[l - 1]))
        if l >= 2 and cfg.dropout > 0:
            # dropout masks are integer decisions: exactly the same zeros
            assert np.array_equal(a == 0, tr.a[l - 1] == 0)
    zL = g.sparse_mlp_export_trace(0, cfg.n_layers, B)
    assert rel_err(zL, tr.z[-1], tr.zmag[-1]) <= TOL
    assert rel_err(probs.cpu().numpy(), tr.p, tr.pmag) <= TOL


def test_eval_forward_has_no_dropout():
    torch = _torch()
    cfg = get_config("C2")
    g, st = pair(cfg)
    x, _ = make_dataset(cfg, n=cfg.batch)
    probs = torch.empty((len(x), 10), device="cuda")
    g.forward(to_dev(x), train=False, step=0, probs=probs)
    tr = M.forward(st, x, False, 0)
    assert rel_err(probs.cpu().numpy(), tr.p, tr.pmag) <= TOL


# ----------------------------------------------------------------------------------------- backward
@pytest.mark.parametrize("name", SMALL + ["tiny"])
def test_backward_parity_unfused(name):
    torch = _torch()
    cfg = _tiny() if name == "tiny" else get_config(name)
    g, st = pair(cfg)
    x, y, tr = _batch(cfg, st, step=7)
    B = len(x)
    loss = torch.zeros(1, device="cuda")
    g.forward(to_dev(x), train=True, step=7)
    g.backward(to_dev(y), loss=loss, fused=None)
    torch.cuda.synchronize()
    gr = M.backward(st, tr, y)
    assert abs(float(loss.item()) - gr.loss) <= TOL * max(1.0, abs(gr.loss))
    for Ly in st.layers:
        l = Ly.l
        gg = g.sparse_mlp_export_trace(2, l)
        e = rel_err(gg, gr.g[l - 2], gr.gmag[l - 2])
        assert e <= TOL, (name, l, "g", e)
        gb = g.sparse_mlp_export_trace(3, l)
        e = rel_err(gb, gr.gb[l - 2], gr.gbmag[l - 2])
        assert e <= TOL, (name, l, "gb", e)
        if l >= 3 or l == cfg.n_layers:
            d = g.sparse_mlp_export_trace(1, l, B)
            e = rel_err(d, gr.deltas[l - 1], gr.dmag[l - 1])
            assert e <= TOL, (name, l, "delta", e)


@pytest.mark.parametrize("name", SMALL)
def test_fused_steps_parity(name):
    torch = _torch()
    cfg = get_config(name)
    g, st = pair(cfg)
    X, Y = make_dataset(cfg, n=cfg.batch * 3)
    from paper_2102_01732_b200 import SGD
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    for s in range(3):
        x, y = X[s * cfg.batch:(s + 1) * cfg.batch], Y[s * cfg.batch:(s + 1) * cfg.batch]
        g.forward(to_dev(x), train=True, step=s)
        g.backward(to_dev(y), fused=sgd)
        M.train_step(st, x, y, cfg.lr, cfg.momentum, cfg.weight_decay, s)
        torch.cuda.synchronize()
        check_and_resync(g, st, f"{name} step {s}")                  # 1e-4 after every step


def test_unfused_step_equals_fused():
    torch = _torch()
    cfg = get_config("C2")
    from paper_2102_01732_b200 import SGD
    g1, st = pair(cfg)
    g2, _ = pair(cfg)
    x, y = make_dataset(cfg, n=cfg.batch)
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    g1.forward(to_dev(x), step=1)
    g1.backward(to_dev(y), fused=sgd)
    g2.forward(to_dev(x), step=1)
    g2.backward(to_dev(y))
    g2.step(sgd)
    torch.cuda.synchronize()
    for l in range(2, cfg.n_layers + 1):
        a, b = g1.export_layer(l), g2.export_layer(l)
        assert rel_err(a["w"], b["w"]) <= 1e-6
    M.train_step(st, x, y, cfg.lr, cfg.momentum, cfg.weight_decay, 1)
    assert_values_close(g2, st, TOL)


@pytest.mark.parametrize("B,fchunk", [(128, None), (100, None), (33, None), (5, None), (1, None), (1, 32), (65, 32)])
def test_chunked_layout_parity(B, fchunk, monkeypatch):
    """chunk_batch = 32 (64 with a 32-wide forward when fchunk is set): the batch is split in
    ceil(B/CB) chunks (ragged last chunk; B = 1 is one column), gradients accumulate over chunks in
    a fixed order."""
    torch = _torch()
    cfg = get_config("C2", batch=B)
    from paper_2102_01732_b200 import SGD
    if fchunk:
        monkeypatch.setenv("SMLP_FWD_CB", str(fchunk))
    g, st = pair(cfg, max_batch=128, chunk_batch=64 if fchunk else 32)
    x, y, tr = _batch(cfg, st, B=B, step=2)
    g.forward(to_dev(x), train=True, step=2)
    g.backward(to_dev(y))
    torch.cuda.synchronize()
    gr = M.backward(st, tr, y)
    for Ly in st.layers:
        assert rel_err(g.sparse_mlp_export_trace(2, Ly.l), gr.g[Ly.l - 2], gr.gmag[Ly.l - 2]) <= TOL
        assert rel_err(g.sparse_mlp_export_trace(3, Ly.l), gr.gb[Ly.l - 2], gr.gbmag[Ly.l - 2]) <= TOL
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    g.step(sgd)
    M.step(st, gr, cfg.lr, cfg.momentum, cfg.weight_decay)
    torch.cuda.synchronize()
    assert_values_close(g, st, TOL)


def test_index_gather_and_errors():
    torch = _torch()
    from paper_2102_01732_b200 import SparseMLPError
    cfg = _tiny(dropout=0.0)
    g, st = pair(cfg)
    X, Y = make_dataset(cfg, n=64)
    idx = np.array([5, 3, 60, 7, 7, 11, 0, 2, 9, 13, 40, 41, 1], np.int32)
    g.forward(to_dev(X), x_idx=to_dev(idx), train=True, step=0)
    tr = M.forward(st, X[idx], True, 0)
    assert rel_err(g.sparse_mlp_export_trace(0, 2, len(idx)), tr.a[1], tr.amag[1]) <= TOL
    g.backward(to_dev(Y), y_idx=to_dev(idx))
    with pytest.raises(SparseMLPError, match="E_STALE"):
        g.backward(to_dev(Y), y_idx=to_dev(idx))                  # trace consumed
    with pytest.raises(SparseMLPError, match="E_SHAPE"):
        g.forward(to_dev(X), train=True)                          # 64 > max_batch = 13
    g.step(__import__("paper_2102_01732_b200").SGD(0.0))          # consumes the pending gradients
    with pytest.raises(SparseMLPError, match="E_STATE"):
        g.step(__import__("paper_2102_01732_b200").SGD(0.0))      # nothing pending any more
    g.forward(to_dev(X[:13]), train=False)
    with pytest.raises(SparseMLPError, match="E_STALE"):
        g.backward(to_dev(Y[:13]))                                # eval-mode trace
    bad = Y[:13].copy()
    bad[3] = 99
    g.forward(to_dev(X[:13]), train=True)
    g.backward(to_dev(bad))
    with pytest.raises(SparseMLPError, match="E_DATA"):
        g.evolve_topology(0.3, 0)                                 # flagged label reported at next sync call


# ----------------------------------------------------------------------------------------- evolve
@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C3", "tiny"])
def test_evolve_parity_op_by_op(name):
    cfg = _tiny() if name == "tiny" else get_config(name)
    g, st = pair(cfg)
    X, Y = make_dataset(cfg, n=cfg.batch * 2)
    for s in range(2):       # non-trivial weights and momenta, produced by the oracle only
        M.train_step(st, X[s * cfg.batch:(s + 1) * cfg.batch], Y[s * cfg.batch:(s + 1) * cfg.batch],
                     cfg.lr * 10, cfg.momentum, cfg.weight_decay, s)
    load_oracle_state_into_gpu(g, st)
    for e in (0, 1):
        rg = g.evolve_topology(cfg.zeta, e)
        ro = T.evolve(st, cfg.zeta, e)
        assert rg[1:] == ro, (rg, ro)
        assert_topology_equal(g, st, f"{name} evolve {e}")
        if cfg.init == "normal":
            for Ly in st.layers:
                assert rel_err(g.export_layer(Ly.l)["w"], Ly.w) < 1e-6
            load_oracle_state_into_gpu(g, st)    # identical inputs for the next op
        else:
            assert_values_bitexact(g, st, f"{name} evolve {e}")


def test_evolve_with_dead_neurons_and_saturated_layer():
    cfg = _tiny(sizes=(6, 5, 4, 3), epsilon=2.0, dropout=0.0)
    g, st = pair(cfg)
    st.alive[1][2] = 0
    st.layers[0] = T._rebuild(st.layers[0], st.layers[0].col != 2)
    st.layers[1] = T._rebuild(st.layers[1], st.layers[1].rows() != 2)
    load_oracle_state_into_gpu(g, st)
    for e in range(4):
        rg = g.evolve_topology(0.5, e)
        ro = T.evolve(st, 0.5, e)
        assert rg[1:] == ro
        assert_topology_equal(g, st)
        assert_values_bitexact(g, st)


# ----------------------------------------------------------------------------------------- prune
@pytest.mark.parametrize("name,rho", [("C3", 5.0), ("C2", 20.0), ("tiny", 30.0), ("C1", 0.0)])
def test_importance_and_prune_parity(name, rho):
    cfg = _tiny() if name == "tiny" else get_config(name)
    g, st = pair(cfg)
    X, Y = make_dataset(cfg, n=cfg.batch)
    M.train_step(st, X, Y, cfg.lr * 10, cfg.momentum, cfg.weight_decay, 0)
    load_oracle_state_into_gpu(g, st)
    for h in range(2, st.L):
        Ig = g.sparse_mlp_importance(h)
        Io = T.importance(st, h)
        assert np.array_equal(Ig.view(np.uint64), Io.view(np.uint64)), f"importance layer {h}"
    pg, rg = g.prune_neurons(rho)
    po, ro = T.prune(st, rho)
    assert pg == po and rg == ro
    assert_topology_equal(g, st, f"{name} prune")
    assert_values_bitexact(g, st, f"{name} prune")
    # prune then evolve (Alg. 2 order) stays bit-exact
    rg = g.evolve_topology(cfg.zeta, 3)
    ro = T.evolve(st, cfg.zeta, 3)
    assert rg[1:] == ro
    assert_topology_equal(g, st, f"{name} prune+evolve")


def test_prune_rho_zero_removes_nothing():
    # rho = 0 -> t = min I -> no alive neuron has I < t
    cfg = get_config("C2")
    g, _ = pair(cfg)
    before = g.info()["nnz"]
    pg, rg = g.prune_neurons(0.0)
    assert sum(rg) == 0 and g.info()["nnz"] == before


# ----------------------------------------------------------------------------------------- after prune: training still matches
def _kink_free(st, X, Y, B, step):
    """The first batch of X (in B-row slices) with no kink-ambiguous pre-activation (R32), decided
    by the oracle alone."""
    for t in range(len(X) // B):
        x, y = X[t * B:(t + 1) * B], Y[t * B:(t + 1) * B]
        tr = M.forward(st, x, True, step)
        if sum(tr.ambiguous) == 0:
            return x, y, tr
    raise AssertionError("no kink-free batch among the candidates")


@pytest.mark.parametrize("name", ["C2", "big"])
def test_training_after_prune_and_evolve_parity(name):
    """Alg. 2's epoch order: train, Importance Pruning, SET evolution, train on.
    Op by op on identical state: a fused GPU step (which, on the > 4M-parameter model with B > CB,
    fills the split last-chunk gradient buffer), then prune and evolve on both sides (bit-exact,
    the layers shrink), then another fused step compared within R24 -- and the param view holds
    zeros in every layer's pruned tail (the second gradient buffer's stale tail must
    not leak into the Eq. 1 pass)."""
    torch = _torch()
    from paper_2102_01732_b200 import SGD
    if name == "big":
        # > 4M parameters (the split last-chunk gradient buffer exists) with few hidden neurons
        # (kink-free batches stay likely): W^(2) 20000 x 400 at 51% density, dense-capped W^(3), W^(4)
        cfg = get_config("C2", sizes=(20000, 400, 400, 10), epsilon=200.0, dropout=0.2, batch=128)
        g, st = pair(cfg, chunk_batch=32)
        assert sum(L.nnz for L in st.layers) > (1 << 22) and g.info()["chunk_batch"] < cfg.batch
        rng = np.random.default_rng(31)
        X = rng.standard_normal((cfg.batch * 8, 20000)).astype(np.float32)
        Y = rng.integers(0, 10, cfg.batch * 8).astype(np.int32)
    else:
        cfg = get_config("C2")
        g, st = pair(cfg)
        X, Y = make_dataset(cfg, n=cfg.batch * 8)
    sgd = SGD(cfg.lr * 10, cfg.momentum, cfg.weight_decay)
    x, y = X[:cfg.batch], Y[:cfg.batch]
    g.forward(to_dev(x), train=True, step=0)
    g.backward(to_dev(y), fused=sgd)
    M.train_step(st, x, y, sgd.lr, sgd.momentum, sgd.weight_decay, 0)
    torch.cuda.synchronize()
    load_oracle_state_into_gpu(g, st)          # identical state again; grad2 keeps step 0's values
    pg, rg = g.prune_neurons(20.0)
    po, ro = T.prune(st, 20.0)
    assert pg == po and rg == ro and sum(ro) > 0
    eg = g.evolve_topology(0.3, 0)
    eo = T.evolve(st, 0.3, 0)
    assert eg[1:] == eo
    assert_topology_equal(g, st, f"{name} prune+evolve")
    assert_values_bitexact(g, st, f"{name} prune+evolve")
    x, y, tr = _kink_free(st, X[cfg.batch:], Y[cfg.batch:], cfg.batch, 1)
    g.forward(to_dev(x), train=True, step=1)
    g.backward(to_dev(y), fused=sgd)
    M.step(st, M.backward(st, tr, y), sgd.lr, sgd.momentum, sgd.weight_decay)
    torch.cuda.synchronize()
    assert_values_close(g, st, TOL, f"{name} after prune+evolve")
    # the param view holds zeros in the pruned tail of each layer
    pv, _ = g.param_view()
    inf = g.info()
    pvh = pv.cpu().numpy()
    for l in range(2, cfg.n_layers + 1):
        o, n, c = inf["val_offset"][l - 1], inf["nnz"][l - 1], inf["cap"][l - 1]
        assert n < c or l == cfg.n_layers
        assert np.all(pvh[o + n:o + c] == 0), (name, l)
