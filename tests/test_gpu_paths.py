"""GPU parity of the specialised paths of the hot path, against the oracle (element by element on
the same seeded inputs; fp32 within 1e-4, integers bit-exact):

* the exact binary-input path of W^(2) (bit-packed input), taken when every input
  value is 0 or 1, and its fp32 fallback when one is not;
* the generic (gather) output layer, used when n_L > 32 (every BASELINE config has n_L <= 32 and
  takes the narrow streaming path, which the other parity tests cover);
* the full-size C5 model in the launch configuration bench.py times (B = 128, auto chunk_batch),
  on seeded SAMPLES of the gradient / update that the oracle computes by its cone evaluation
  (oracle/sampled.py), plus every forward activation.
"""
import numpy as np
import pytest

from oracle import model as M
from oracle.compare import rel_err
from synth import get_config, make_dataset
from tests.gpu_helpers import (TOL, assert_topology_equal, assert_values_close, check_and_resync,
                               load_oracle_state_into_gpu, pair, to_dev)

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _binary_cfg(**kw):
    base = dict(sizes=(300, 400, 350, 2), epsilon=10.0, alpha=0.5, dropout=0.0, init="he_uniform", batch=128)
    base.update(kw)
    return get_config("C1", **base)


def _binary_data(n, d, seed, density=0.05):
    rng = np.random.default_rng([seed, 4242])
    X = (rng.random((n, d)) < density).astype(np.float32)
    y = rng.integers(0, 2, size=n).astype(np.int32)
    return X, y


def _check_step(g, st, x, y, step, cfg, path_flag):
    torch = _torch()
    B = len(x)
    tr = M.forward(st, x, True, step)
    assert sum(tr.ambiguous) == 0, "kink-ambiguous batch"
    g.forward(to_dev(x), train=True, step=step)
    assert g.sparse_mlp_export_trace(4, 0)[0] == path_flag
    g.backward(to_dev(y), fused=None)
    torch.cuda.synchronize()
    for l in range(2, cfg.n_layers):
        assert rel_err(g.sparse_mlp_export_trace(0, l, B), tr.a[l - 1], tr.amag[l - 1]) <= TOL, ("a", l)
    gr = M.backward(st, tr, y)
    for Ly in st.layers:
        assert rel_err(g.sparse_mlp_export_trace(2, Ly.l), gr.g[Ly.l - 2], gr.gmag[Ly.l - 2]) <= TOL, ("g", Ly.l)
        assert rel_err(g.sparse_mlp_export_trace(3, Ly.l), gr.gb[Ly.l - 2], gr.gbmag[Ly.l - 2]) <= TOL, ("gb", Ly.l)
    return tr, gr


@pytest.mark.parametrize("B,chunk,fchunk,dropout", [(128, 0, None, 0.0), (128, 32, None, 0.3), (100, 32, None, 0.0),
                                                    (37, 8, None, 0.3), (128, 128, 32, 0.3), (100, 64, 32, 0.0)])
def test_binary_input_path_parity(B, chunk, fchunk, dropout, monkeypatch):
    from paper_2102_01732_b200 import SGD
    torch = _torch()
    cfg = _binary_cfg(batch=B, dropout=dropout)
    if fchunk:
        monkeypatch.setenv("SMLP_FWD_CB", str(fchunk))
    g, st = pair(cfg, max_batch=B, chunk_batch=chunk)
    if fchunk:
        assert g.info()["fwd_chunk_batch"] == fchunk
    X, Y = _binary_data(4 * B, cfg.sizes[0], seed=B + chunk + (fchunk or 0))
    sgd = SGD(cfg.lr * 5, cfg.momentum, cfg.weight_decay)
    for s in range(3):
        x, y = X[s * B:(s + 1) * B], Y[s * B:(s + 1) * B]
        _, gr = _check_step(g, st, x, y, s, cfg, 1.0)
        g.step(sgd)
        M.step(st, gr, sgd.lr, sgd.momentum, sgd.weight_decay)
        torch.cuda.synchronize()
        check_and_resync(g, st, f"binary path step {s}")
    # fused path (the 1-GPU bench path) on the last batch
    x, y = X[3 * B:], Y[3 * B:]
    g.forward(to_dev(x), train=True, step=3)
    g.backward(to_dev(y), fused=sgd)
    M.train_step(st, x, y, sgd.lr, sgd.momentum, sgd.weight_decay, 3)
    torch.cuda.synchronize()
    assert_values_close(g, st, TOL, "binary path fused")


def test_binary_path_falls_back_on_non_binary_input():
    cfg = _binary_cfg(batch=64)
    g, st = pair(cfg, max_batch=64, chunk_batch=32)
    X, Y = _binary_data(64, cfg.sizes[0], seed=9)
    X[17, 5] = 0.5                                   # one non-binary value -> fp32 gather path
    _check_step(g, st, X, Y, 0, cfg, 0.0)
    X[17, 5] = 1.0                                   # binary again -> bit path
    g2, st2 = pair(cfg, max_batch=64, chunk_batch=32)
    _check_step(g2, st2, X, Y, 0, cfg, 1.0)


def test_real_input_kind_skips_the_bit_path():
    """input_kind = SMLP_INPUT_REAL: no {0,1} detection and no bit path (trace flag -1), the fp32
    gather kernels serve layer 2 even for a binary batch, same parity; and the small-model update
    (one Eq. 1 launch over the whole view + one mirror launch) matches the oracle's Eq. 1."""
    from paper_2102_01732_b200 import SGD, SparseMLP
    torch = _torch()
    cfg = _binary_cfg(batch=64, dropout=0.3)
    st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed)
    g = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed, 0, 64,
                  32, input_kind=1)
    X, Y = _binary_data(128, cfg.sizes[0], seed=21)
    sgd = SGD(cfg.lr * 5, cfg.momentum, cfg.weight_decay)
    for s_ in range(2):
        x, y = X[s_ * 64:(s_ + 1) * 64], Y[s_ * 64:(s_ + 1) * 64]
        tr = M.forward(st, x, True, s_)
        assert sum(tr.ambiguous) == 0
        g.forward(to_dev(x), train=True, step=s_)
        assert g.sparse_mlp_export_trace(4, 0)[0] == -1.0
        for l in range(2, cfg.n_layers):
            assert rel_err(g.sparse_mlp_export_trace(0, l, 64), tr.a[l - 1], tr.amag[l - 1]) <= TOL, ("a", l)
        g.backward(to_dev(y), fused=sgd)
        M.train_step(st, x, y, sgd.lr, sgd.momentum, sgd.weight_decay, s_)
        torch.cuda.synchronize()
        check_and_resync(g, st, f"real input kind step {s_}")


def test_binary_input_kind_checked_promise():
    """input_kind = SMLP_INPUT_BINARY: binary batches take the bit path (same parity as the oracle);
    a batch that breaks the promise is still trained correctly -- through the fp32 layer-2 kernels,
    weights equal to the oracle's step on that batch, nothing corrupted -- and is
    reported as SMLP_E_DATA at the next synchronising call."""
    from paper_2102_01732_b200 import SGD, SparseMLP, SparseMLPError
    torch = _torch()
    cfg = _binary_cfg(batch=64, dropout=0.3)
    st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed)
    g = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed, 0, 64,
                  32, input_kind=2)
    X, Y = _binary_data(192, cfg.sizes[0], seed=21)
    X[128 + 3, 7] = 0.5                              # the third batch breaks the promise
    sgd = SGD(cfg.lr * 5, cfg.momentum, cfg.weight_decay)
    for s_ in range(3):
        x, y = X[s_ * 64:(s_ + 1) * 64], Y[s_ * 64:(s_ + 1) * 64]
        tr = M.forward(st, x, True, s_)
        assert sum(tr.ambiguous) == 0
        g.forward(to_dev(x), train=True, step=s_)
        assert g.sparse_mlp_export_trace(4, 0)[0] == (1.0 if s_ < 2 else 0.0)
        for l in range(2, cfg.n_layers):
            assert rel_err(g.sparse_mlp_export_trace(0, l, 64), tr.a[l - 1], tr.amag[l - 1]) <= TOL, ("a", s_, l)
        g.backward(to_dev(y), fused=sgd)
        M.step(st, M.backward(st, tr, y), sgd.lr, sgd.momentum, sgd.weight_decay)
        torch.cuda.synchronize()
        check_and_resync(g, st, f"binary input kind, step {s_}")
    with pytest.raises(SparseMLPError, match="E_DATA"):
        g.sync()
    g.sync()                                         # reported once, then cleared
    with pytest.raises(SparseMLPError, match="E_ARG"):
        SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed, 0, 256,
                  0, input_kind=2)                  # the bit path needs max_batch <= 128


def test_binary_and_fp32_paths_agree_on_forward():
    """The bit path and the fp32 gather path compute the same a_2 up to the summation order
    (each is a fixed order, R27): every batch row but the changed one agrees to fp32 rounding."""
    torch = _torch()
    cfg = _binary_cfg(batch=64, dropout=0.3)
    g, _ = pair(cfg, max_batch=64, chunk_batch=32)
    X, _ = _binary_data(64, cfg.sizes[0], seed=3)
    g.forward(to_dev(X), train=True, step=5)
    a_bits = g.sparse_mlp_export_trace(0, 2, 64)
    X2 = X.copy()
    X2[63, 299] = 2.0                                # non-binary: forces the fp32 gather path
    g.forward(to_dev(X2), train=True, step=5)
    assert g.sparse_mlp_export_trace(4, 0)[0] == 0.0
    a_f32 = g.sparse_mlp_export_trace(0, 2, 64)
    torch.cuda.synchronize()
    keep = np.ones(a_bits.shape[0], bool)
    keep[63] = False                                 # only batch row 63's input changed
    a, b = a_bits[keep].astype(np.float64), a_f32[keep].astype(np.float64)
    scale = np.maximum(np.abs(a), 1e-3 * np.abs(a).max())
    assert np.max(np.abs(a - b) / scale) < 1e-5
    assert not np.array_equal(a_bits[63], a_f32[63])


def test_generic_output_layer_parity():
    """n_L = 40 > 32: the output layer goes through the gather kernels (fwd_kernel / bwd_kernel)."""
    from paper_2102_01732_b200 import SGD
    torch = _torch()
    cfg = get_config("C1", sizes=(120, 90, 70, 40), epsilon=6.0, dropout=0.2, batch=50)
    g, st = pair(cfg, max_batch=50, chunk_batch=16)
    rng = np.random.default_rng(12)       # a batch with no kink-ambiguous pre-activation (R32)
    X = rng.standard_normal((100, 120)).astype(np.float32)
    Y = rng.integers(0, 40, size=100).astype(np.int32)
    sgd = SGD(cfg.lr * 5, cfg.momentum, cfg.weight_decay)
    for s in range(2):
        x, y = X[s * 50:(s + 1) * 50], Y[s * 50:(s + 1) * 50]
        tr = M.forward(st, x, True, s)
        assert sum(tr.ambiguous) == 0
        g.forward(to_dev(x), train=True, step=s)
        assert g.sparse_mlp_export_trace(4, 0)[0] == 0.0     # normal inputs: not binary
        assert rel_err(g.sparse_mlp_export_trace(0, 4, 50), tr.z[-1], tr.zmag[-1]) <= TOL
        g.backward(to_dev(y), fused=sgd)
        M.train_step(st, x, y, sgd.lr, sgd.momentum, sgd.weight_decay, s)
        torch.cuda.synchronize()
        check_and_resync(g, st, f"generic output layer step {s}")


# ----------------------------------------------------------------------------------------- C5 full size
def _kept_ok(k, Ly, cfg, B, min_kept):
    """>= min_kept untainted gradient entries, bias gradients and delta elements of the layer, or
    all there are when the layer has fewer (e.g. the 2 output neurons)."""
    n = cfg.sizes[Ly.l - 1]
    return k[0] >= min(min_kept, Ly.nnz) and k[1] >= min(min_kept, n) and k[2] >= min(min_kept, B * n)


def _full_size_sampled_parity(name, B, widths, min_kept=256):
    """Full-size model in the bench launch configuration (max_batch = cfg.batch).  Checked: ER
    topology and values bit-exact, every forward activation and logit of a B-row batch, every
    exported delta_l element of the cone of the sampled neurons whose (b, j) does not depend on a
    kink-ambiguous f' (R32), and for seeded samples of connections / neurons of every layer the
    gradient (unfused) and the Eq. 1 update (fused) against the oracle's cone evaluation
    (oracle/sampled.py).  Samples are drawn until >= min_kept untainted gradient entries, bias
    gradients and delta elements per layer are compared; the per-layer counts are printed."""
    from oracle import sampled as S
    from paper_2102_01732_b200 import SGD
    from synth.data import c5_host_rows
    torch = _torch()
    cfg = get_config(name)
    g, st = pair(cfg)
    assert (g.info()["chunk_batch"], g.info()["fwd_chunk_batch"]) == widths
    assert_topology_equal(g, st, f"{name} init")
    for Ly in st.layers:
        e = g.export_layer(Ly.l)
        assert np.array_equal(e["w"].view(np.uint32), Ly.w.view(np.uint32)), f"{name} W^({Ly.l}) init values"
    x, y = c5_host_rows(cfg, np.arange(B))
    tr = M.forward(st, x, True, 0)
    g.forward(to_dev(x), train=True, step=0)
    assert g.sparse_mlp_export_trace(4, 0)[0] == 1.0
    for l in range(2, cfg.n_layers):
        assert rel_err(g.sparse_mlp_export_trace(0, l, B), tr.a[l - 1], tr.amag[l - 1]) <= TOL, ("a", l)
    assert rel_err(g.sparse_mlp_export_trace(0, cfg.n_layers, B), tr.z[-1], tr.zmag[-1]) <= TOL
    g.backward(to_dev(y), fused=None)
    torch.cuda.synchronize()
    L = cfg.n_layers
    dexp = {l: g.sparse_mlp_export_trace(1, l, B) for l in range(2, L + 1)}
    gexp = {Ly.l: g.sparse_mlp_export_trace(2, Ly.l) for Ly in st.layers}
    gbexp = {l: g.sparse_mlp_export_trace(3, l) for l in range(2, L + 1)}
    # seeded samples, drawn in rounds of 512 connections / 128 neurons per layer until every layer
    # has >= min_kept untainted ones (all of them when a layer is smaller)
    rng = np.random.default_rng(2025)
    ent = {Ly.l: np.zeros(0, np.int64) for Ly in st.layers}
    neu = {l: np.zeros(0, np.int64) for l in range(2, L + 1)}
    for rnd in range(8):
        for Ly in st.layers:
            free = np.setdiff1d(np.arange(Ly.nnz), ent[Ly.l]) if Ly.nnz <= 4096 else None
            new = (rng.choice(free, size=min(512, len(free)), replace=False) if free is not None
                   else rng.choice(Ly.nnz, size=512, replace=False))
            ent[Ly.l] = np.unique(np.concatenate([ent[Ly.l], new]))
        for l in neu:
            n = cfg.sizes[l - 1]
            neu[l] = np.unique(np.concatenate([neu[l], rng.choice(n, size=min(128, n), replace=False)]))
        need = {l: set(neu[l].tolist()) for l in neu}
        for Ly in st.layers:
            need[Ly.l] |= set(Ly.col[ent[Ly.l]].tolist())
        deltas, tainted, dmags = S.delta_columns(st, tr, y, need)
        gsamp, kept = {}, {}
        for Ly in st.layers:
            l = Ly.l
            ok = np.array([not tainted[l][int(j)].any() for j in Ly.col[ent[l]]])
            go, gm = S.grad_entries(st, tr, deltas, dmags, l, ent[l])
            gsamp[l] = (go, gm, ok)
            okn = np.array([not tainted[l][int(j)].any() for j in neu[l]])
            gbo, gbm = S.bias_grad_columns(deltas, dmags, l, neu[l])
            J = np.array(sorted(deltas[l]), np.int64)
            T = np.stack([tainted[l][int(j)] for j in J], axis=1)
            kept[l] = (int(ok.sum()), int(okn.sum()), int((~T).sum()))
        if all(_kept_ok(kept[Ly.l], Ly, cfg, B, min_kept) for Ly in st.layers):
            break
    print(f"{name} kept per layer (gradient entries, bias gradients, delta elements):", kept)
    for Ly in st.layers:
        l = Ly.l
        assert _kept_ok(kept[l], Ly, cfg, B, min_kept), (l, kept[l])
        go, gm, ok = gsamp[l]
        gg = gexp[l][ent[l]]
        assert rel_err(gg[ok], go[ok], gm[ok]) <= TOL, ("g", l, rel_err(gg[ok], go[ok], gm[ok]))
        okn = np.array([not tainted[l][int(j)].any() for j in neu[l]])
        gbo, gbm = S.bias_grad_columns(deltas, dmags, l, neu[l])
        gbg = gbexp[l][neu[l]]
        assert rel_err(gbg[okn], gbo[okn], gbm[okn]) <= TOL, ("gb", l)
    for l in range(2, L + 1):
        J = np.array(sorted(deltas[l]), np.int64)
        D = np.stack([deltas[l][int(j)] for j in J], axis=1)
        Dm = np.stack([dmags[l][int(j)] for j in J], axis=1)
        T = np.stack([tainted[l][int(j)] for j in J], axis=1)
        dg = dexp[l][:, J]
        assert rel_err(dg[~T], D[~T], Dm[~T]) <= TOL, ("delta", l, rel_err(dg[~T], D[~T], Dm[~T]))
    # the fused Eq. 1 update in the bench configuration, on a second handle with the same init
    del g
    g2, _ = pair(cfg)
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    g2.forward(to_dev(x), train=True, step=0)
    g2.backward(to_dev(y), fused=sgd)
    torch.cuda.synchronize()
    # expected update: the oracle's Eq. 1 (model.step) with the sampled gradients (zero elsewhere)
    G = M.Grads([np.zeros(Ly.nnz, np.float32) for Ly in st.layers],
                [np.zeros(n, np.float32) for n in cfg.sizes[1:]], 0.0, [],
                [np.zeros(Ly.nnz) for Ly in st.layers], [np.zeros(n) for n in cfg.sizes[1:]])
    for Ly in st.layers:
        G.g[Ly.l - 2][ent[Ly.l]] = gsamp[Ly.l][0]
        G.gmag[Ly.l - 2][ent[Ly.l]] = gsamp[Ly.l][1]
    M.step(st, G, sgd.lr, sgd.momentum, sgd.weight_decay)
    for Ly in st.layers:
        l = Ly.l
        ok = gsamp[l][2]
        e = g2.export_layer(l)
        k = ent[l][ok]
        assert rel_err(e["w"][k], Ly.w[k], Ly.wmag[k]) <= TOL, ("w", l)
        assert rel_err(e["v"][k], Ly.v[k], Ly.vmag[k]) <= TOL, ("v", l)


def test_c5_full_size_sampled_parity():
    """BASELINE configs[4] at full size (65536-500000-500000-500000-2, 52.3M connections), B = 128:
    chunk_batch auto = 64 -> 2 backward chunks, forward tensors 32 wide -> 4 forward chunks,
    binary-input path, fused update."""
    _full_size_sampled_parity("C5", 128, (64, 32))


def test_width_scaling_t4_full_size_sampled_parity():
    """Table 4 row 4 at full size (65536-5M x 4-2, eps 1: four 5M-neuron hidden layers, 40.1M
    connections, ~2 connections per row, a SPARSE narrow output layer of 5M x 2 -> the row-streaming
    bwd_narrow_kernel), 4-row batch in the 128-column bench layout."""
    _full_size_sampled_parity("T4", 4, (128, 128))


def test_width_scaling_t2_full_size_sampled_parity():
    """Width scaling: Table 4 row 2 at full size (65536-2.5M-2.5M-2,
    eps 5, 42.8M connections, dropout 0.4) in the bench layout (max_batch 128 -> one 128-column
    chunk: no 32-column slab of a 2.5M-neuron layer fits the L2), on an 8-row batch (a ragged
    chunk; the oracle's full forward at 128 rows needs 52 GB and 6 minutes)."""
    _full_size_sampled_parity("T2", 8, (128, 128))


# salt: data seed chosen (by the oracle alone) so that no pre-activation of the checked steps
# sits within rounding of a kink (R32)
@pytest.mark.parametrize("chunk,fchunk,B,dropout,eps,salt",
                         [(8, 8, 29, 0.2, 40.0, 0), (16, 16, 64, 0.0, 40.0, 1), (32, 32, 77, 0.3, 40.0, 0),
                          (64, 64, 128, 0.0, 40.0, 0), (128, 128, 128, 0.2, 40.0, 0),
                          # mixed layout: forward tensors CBf wide, deltas CB wide (ragged both ways)
                          (64, 32, 100, 0.3, 40.0, 0), (128, 32, 128, 0.2, 40.0, 0), (128, 64, 77, 0.0, 40.0, 0),
                          # sparse narrow output layer: row-streaming forward; backward through the row
                          # kernels, or (chunk == fchunk == 64) the narrow bwd_narrow_kernel (SMLP_NARROW_SPARSE_BWD)
                          (64, 64, 90, 0.2, 5.0, 0), (64, 32, 90, 0.2, 5.0, 0), (128, 32, 128, 0.0, 5.0, 0),
                          # 3 forward chunks: the output layer's forward pass covers 96 of its 128 columns
                          (64, 32, 70, 0.2, 5.0, 0), (128, 32, 70, 0.0, 40.0, 0),
                          # eps = 1: ~1-8 entries per row -> the row-streaming short-row kernels
                          (128, 128, 128, 0.2, 1.0, 0), (128, 128, 77, 0.0, 1.0, 0)])
def test_long_rows_and_chunk_widths_parity(chunk, fchunk, B, dropout, eps, salt, monkeypatch):
    """Rows longer than one 64-entry segment in both orientations (partials + fixed-order finish
    kernels), every chunk width of the row kernels (slot / group layouts, ragged last chunk), the
    mixed forward / backward chunk widths (SMLP_FWD_CB), the unfused and the fused (Eq. 1 in the
    backward) update paths."""
    from paper_2102_01732_b200 import SGD
    torch = _torch()
    # W^(2) 30 x 200 is dense-capped (canonical rows of 200 entries: 4 segments); W^(3) 200 x 150
    # at eps 40 has ~70-entry canonical rows and ~93-entry mirror rows
    cfg = get_config("C1", sizes=(30, 200, 150, 10), epsilon=eps, alpha=0.6, dropout=dropout, batch=B)
    monkeypatch.setenv("SMLP_FWD_CB", str(fchunk))
    if eps == 1.0:   # the row-streaming short-row kernels, at this small size too
        monkeypatch.setenv("SMLP_SHORT_MIN_ROWS", "0")
    if eps == 5.0 and chunk == fchunk == 64:
        monkeypatch.setenv("SMLP_NARROW_SPARSE_BWD", "1")
    g, st = pair(cfg, max_batch=B, chunk_batch=chunk)
    assert (g.info()["chunk_batch"], g.info()["fwd_chunk_batch"]) == (chunk, fchunk)
    assert st.layers[-1].dense_capped == (eps == 40.0)
    if eps == 40.0:
        assert max(np.diff(st.layers[1].row_ptr)) > 64
    rng = np.random.default_rng([chunk, B, salt])
    X = rng.standard_normal((16 * B, 30)).astype(np.float32)
    Y = rng.integers(0, 10, size=16 * B).astype(np.int32)
    sgd = SGD(cfg.lr * 5, cfg.momentum, cfg.weight_decay)
    nxt = 0
    for s in range(2):
        while True:           # the next candidate batch the oracle finds kink-free (R32)
            assert nxt < 16, "no kink-free batch among the candidates"
            x, y = X[nxt * B:(nxt + 1) * B], Y[nxt * B:(nxt + 1) * B]
            nxt += 1
            tr = M.forward(st, x, True, s)
            if sum(tr.ambiguous) == 0:
                break
        g.forward(to_dev(x), train=True, step=s)
        g.backward(to_dev(y), fused=None)
        torch.cuda.synchronize()
        for l in range(2, cfg.n_layers):
            assert rel_err(g.sparse_mlp_export_trace(0, l, B), tr.a[l - 1], tr.amag[l - 1]) <= TOL, ("a", l)
        gr = M.backward(st, tr, y)
        for Ly in st.layers:
            assert rel_err(g.sparse_mlp_export_trace(2, Ly.l), gr.g[Ly.l - 2], gr.gmag[Ly.l - 2]) <= TOL, ("g", Ly.l)
            assert rel_err(g.sparse_mlp_export_trace(3, Ly.l), gr.gb[Ly.l - 2], gr.gbmag[Ly.l - 2]) <= TOL, ("gb", Ly.l)
        g.step(sgd)
        M.step(st, gr, sgd.lr, sgd.momentum, sgd.weight_decay)
        torch.cuda.synchronize()
        check_and_resync(g, st, f"long rows step {s}")
    while True:
        assert nxt < 16, "no kink-free batch among the candidates"
        x, y = X[nxt * B:(nxt + 1) * B], Y[nxt * B:(nxt + 1) * B]
        nxt += 1
        tr = M.forward(st, x, True, 2)
        if sum(tr.ambiguous) == 0:
            break
    g.forward(to_dev(x), train=True, step=2)
    g.backward(to_dev(y), fused=sgd)
    M.step(st, M.backward(st, tr, y), sgd.lr, sgd.momentum, sgd.weight_decay)
    torch.cuda.synchronize()
    assert_values_close(g, st, TOL, "long rows fused")
    assert_topology_equal(g, st)


def test_pipelined_host_step_matches_sync():
    """sparse_mlp_train_step_host_async (double-buffered staging on a copy stream) computes the
    same training trajectory as the synchronous host-buffer step and the device-buffer path,
    bit for bit, and delivers every step's loss."""
    from paper_2102_01732_b200 import SGD
    torch = _torch()
    cfg = _binary_cfg(batch=64, dropout=0.2)
    g1, _ = pair(cfg, max_batch=64)
    g2, _ = pair(cfg, max_batch=64)
    X, Y = _binary_data(4 * 64, cfg.sizes[0], seed=21)
    xp, yp = torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory()
    losses = torch.zeros(4, dtype=torch.float32).pin_memory()
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    ref = []
    for s in range(4):
        ref.append(g1.train_step_host(xp[s * 64:(s + 1) * 64], yp[s * 64:(s + 1) * 64], 64, s, sgd))
        g2.train_step_host_async(xp[s * 64:(s + 1) * 64], yp[s * 64:(s + 1) * 64], 64, s, sgd, losses[s:])
    g2.sync()
    torch.cuda.synchronize()
    assert np.array_equal(losses.numpy(), np.array(ref, np.float32))
    for l in range(2, cfg.n_layers + 1):
        a, b = g1.export_layer(l), g2.export_layer(l)
        assert np.array_equal(a["w"].view(np.uint32), b["w"].view(np.uint32))


def test_overlapped_dp_path_matches_fused_on_one_rank():
    """The K > 1 step structure on one GPU: unfused backward, per-layer grad slices (output layer
    first, then the bias block) released by the library's layer events to a side stream (identity
    'allreduce'), Eq. 1 update kernel + mirror refresh -- the same trajectory as the fused 1-GPU
    step (up to the update's rounding)."""
    from paper_2102_01732_b200 import SGD, SparseMLPError
    from paper_2102_01732_b200.dp import OverlappedAllreduce
    torch = _torch()
    cfg = _binary_cfg(batch=64, dropout=0.1)
    g1, _ = pair(cfg, max_batch=64)
    g2, _ = pair(cfg, max_batch=64)
    side = torch.cuda.Stream()
    with pytest.raises(SparseMLPError, match="E_STATE"):
        g2.wait_layer(2, side)                            # no backward recorded yet
    X, Y = _binary_data(3 * 64, cfg.sizes[0], seed=5)
    ov = OverlappedAllreduce(g2, bucket_bytes=1)          # one bucket per layer (then the biases)
    assert len(OverlappedAllreduce(g2).buckets) == 1        # default: a small view is one collective
    layout, bb = g2.view_layout()
    assert layout[0][0] == 0 and all(o2 >= o1 + c1 for (o1, c1), (o2, _) in zip(layout, layout[1:]))
    seen = []
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    for s in range(3):
        x, y = to_dev(X[s * 64:(s + 1) * 64]), to_dev(Y[s * 64:(s + 1) * 64])
        g1.forward(x, train=True, step=s)
        g1.backward(y, fused=sgd)
        g2.forward(x, train=True, step=s)
        g2.backward(y, fused=None)
        ov(reduce=lambda t: seen.append(t.numel()))
        g2.step(sgd)
    torch.cuda.synchronize()
    assert seen[:cfg.n_layers] == [c for _, c in reversed(layout)] + [g2.info()["param_count"] - bb]
    for l in range(2, cfg.n_layers + 1):
        a, b = g1.export_layer(l), g2.export_layer(l)
        assert np.array_equal(a["col"], b["col"])
        assert rel_err(b["w"], a["w"]) <= 1e-6, l


@pytest.mark.parametrize("cfg_name", ["C1", "C2"])
def test_gradient_flow_parity(cfg_name):
    """sparse_mlp_gradient_flow against oracle.model.gradient_flow on the same
    unfused backward; deterministic (two calls give the same bits); E_STATE without pending
    gradients."""
    from paper_2102_01732_b200 import SparseMLPError
    torch = _torch()
    cfg = get_config(cfg_name, dropout=0.0)
    g, st = pair(cfg)
    rng = np.random.default_rng(17)
    X = rng.standard_normal((cfg.batch, cfg.sizes[0])).astype(np.float32)
    Y = rng.integers(0, cfg.sizes[-1], cfg.batch).astype(np.int32)
    with pytest.raises(SparseMLPError, match="E_STATE"):
        g.gradient_flow()
    g.forward(to_dev(X), train=True, step=0)
    g.backward(to_dev(Y), fused=None)
    f1, f2 = g.gradient_flow(), g.gradient_flow()
    torch.cuda.synchronize()
    tr = M.forward(st, X, True, 0)
    gr = M.backward(st, tr, Y)
    ref = M.gradient_flow(gr)
    assert f1 == f2
    # R24: each GPU gradient value is within KAPPA_U * mag of the oracle's, so sum g^2 moves by
    # at most sum 2 |g| KAPPA_U mag (first order); on top of that, 1e-4 relative
    from oracle.compare import KAPPA_U
    bound = sum(float(np.sum(2.0 * np.abs(gv.astype(np.float64)) * KAPPA_U * m)) for gv, m in zip(gr.g + gr.gb, gr.gmag + gr.gbmag))
    assert abs(f1 - ref) <= 1e-4 * ref + bound, (f1, ref, bound)


def test_post_training_prune_sweep_parity():
    """Supp. C: one-shot Importance Pruning of a trained model at rho =
    5..25.  Every sweep point equals the oracle's prune of the same trained state: identical
    remaining connection counts (bit-exact topology decision) and the same test accuracy up to
    arg-max ties; the trained model is restored after each point."""
    from oracle import topology as T
    from paper_2102_01732_b200 import SGD
    from paper_2102_01732_b200.trainer import prune_sweep
    torch = _torch()
    cfg = get_config("C1", dropout=0.0)
    g, st = pair(cfg)
    X, Y = make_dataset(cfg, n=6 * cfg.batch)
    sgd = SGD(cfg.lr * 10, cfg.momentum, cfg.weight_decay)
    for s in range(4):                                   # a short training run, oracle in lockstep
        x, y = X[s * cfg.batch:(s + 1) * cfg.batch], Y[s * cfg.batch:(s + 1) * cfg.batch]
        g.forward(to_dev(x), train=True, step=s)
        g.backward(to_dev(y.astype(np.int32)), fused=sgd)
        M.train_step(st, x, y, sgd.lr, sgd.momentum, sgd.weight_decay, s)
    torch.cuda.synchronize()
    for Ly in st.layers:                                 # identical trained state on both sides
        g.import_layer(Ly.l, Ly.row_ptr.astype(np.int32), Ly.col, Ly.w, Ly.v)
        g.sparse_mlp_import_bias(Ly.l, st.b[Ly.l - 2], st.vb[Ly.l - 2])
    Xt, Yt = to_dev(X[4 * cfg.batch:]), to_dev(Y[4 * cfg.batch:].astype(np.int32))
    sweep = prune_sweep(g, Xt, Yt, cfg.batch)
    assert sweep[0][0] is None and sweep[0][2] == sum(len(L.w) for L in st.layers)
    xt, yt = X[4 * cfg.batch:], Y[4 * cfg.batch:]
    import copy
    for rho, acc, conns in sweep[1:]:
        so = copy.deepcopy(st)
        T.prune(so, rho)
        assert conns == sum(len(L.w) for L in so.layers), rho
        p = M.forward(so, xt, False, 0).p
        acc_o = float(np.mean(np.argmax(p, 1) == yt))
        assert abs(acc - acc_o) <= 2.0 / len(yt), (rho, acc, acc_o)
    e = g.export_layer(3)                                # restored after the sweep
    assert np.array_equal(e["col"], st.layers[1].col) and np.array_equal(e["w"], st.layers[1].w)


def test_union_average_parity():
    """WASAP phase 2 end: K = 3 replicas evolved independently, averaged over
    the union of their supports and re-sparsified to the phase-1 counts.  Every replica runs the
    library merge on the same gathered (position, value) lists and ends bit-identical; topology
    and values are bit-exact to oracle.dp.average_union (the arithmetic that decides the
    selection is shared, DESIGN R31)."""
    from oracle import dp as ODP
    from oracle import topology as T
    torch = _torch()
    cfg = get_config("C1", dropout=0.0)
    K = 3
    gs, sts = [], []
    for k in range(K):
        g, st = pair(cfg)
        g.evolve_topology(cfg.zeta, 50 + k)
        T.evolve(st, cfg.zeta, 50 + k)
        gs.append(g)
        sts.append(st)
    targets = [L.nnz for L in sts[0].layers]
    for l in range(2, cfg.n_layers + 1):
        lists = [g.export_positions(l) for g in gs]
        pos = torch.cat([p for p, _ in lists])
        val = torch.cat([v for _, v in lists])
        for g in gs:
            assert g.union_average_layer(l, K, pos, val, targets[l - 2]) == min(targets[l - 2], len(set(pos.tolist())))
    torch.cuda.synchronize()
    kept = ODP.average_union(sts, targets)
    for g in gs:
        for Ly in sts[0].layers:
            e = g.export_layer(Ly.l)
            assert np.array_equal(e["row_ptr"], Ly.row_ptr.astype(np.int32)), Ly.l
            assert np.array_equal(e["col"], Ly.col), Ly.l
            assert np.array_equal(e["w"].view(np.uint32), Ly.w.view(np.uint32)), Ly.l
            assert not np.any(e["v"])
    assert kept == [g.info()["nnz"][l - 1] for l in range(2, cfg.n_layers + 1) for g in gs[:1]]
    # the averaged model still trains (mirror and work lists rebuilt)
    from paper_2102_01732_b200 import SGD
    X, Y = make_dataset(cfg, n=cfg.batch)
    gs[0].forward(to_dev(X), train=True, step=0)
    gs[0].backward(to_dev(Y.astype(np.int32)), fused=SGD(cfg.lr, cfg.momentum, cfg.weight_decay))
    torch.cuda.synchronize()


def test_retain_valid_updates_parity():
    """Async phase-1 analogue: a gradient taken on topology version t is
    applied after a SET evolution (version t') through RetainValidUpdates -- the retained
    gradient is bit-exact to oracle.dp.retain_valid_updates (intersection of supports), and the
    resulting Eq. 1 update matches the oracle's."""
    from oracle import dp as ODP
    from oracle import topology as T
    from paper_2102_01732_b200 import SGD
    from paper_2102_01732_b200.dp import StaleGradient, apply_stale_gradient
    torch = _torch()
    cfg = get_config("C1", dropout=0.0)
    g, st = pair(cfg)
    X, Y = make_dataset(cfg, n=cfg.batch)
    g.forward(to_dev(X), train=True, step=0)
    g.backward(to_dev(Y.astype(np.int32)), fused=None)
    stale = StaleGradient(g)                                   # gradient at version t
    torch.cuda.synchronize()
    tr = M.forward(st, X, True, 0)
    gr = M.backward(st, tr, Y)
    keys_t = [L.keys() for L in st.layers]
    g.step(SGD(0.0))                                          # consume (no update) before evolving
    g.evolve_topology(cfg.zeta, 7)                             # topology moves on (version t')
    T.evolve(st, cfg.zeta, 7)
    assert_topology_equal(g, st)
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    ref = ODP.retain_valid_updates(keys_t, gr.g, st)
    rmag = [m.astype(np.float64) for m in ODP.retain_valid_updates(keys_t, [x.astype(np.float32) for x in gr.gmag], st)]
    for (pos, gv), Ly, r, rm in zip(stale.layers, st.layers, ref, rmag):
        k = g.retain_valid_updates(Ly.l, pos, gv)
        assert k == len(set(keys_t[Ly.l - 2].tolist()) & set(Ly.keys().tolist()))
        # pure data movement: bit-exact against the same mapping of the GPU's own stale values
        table = dict(zip(pos.cpu().numpy().tolist(), gv.cpu().numpy().tolist()))
        mapped = np.array([table.get(p, 0.0) for p in Ly.keys().tolist()], np.float32)
        got = g.sparse_mlp_export_trace(2, Ly.l)[:len(mapped)]
        assert np.array_equal(got.view(np.uint32), mapped.view(np.uint32)), Ly.l
        assert rel_err(mapped, r, rm) <= TOL                  # and the oracle's retained gradient
    kept = apply_stale_gradient(g, stale, sgd)                 # the full server step
    torch.cuda.synchronize()
    assert kept == [len(set(keys_t[L.l - 2].tolist()) & set(L.keys().tolist())) for L in st.layers]
    M.step(st, M.Grads(ref, gr.gb, gr.loss, gr.deltas, rmag, gr.gbmag), sgd.lr, sgd.momentum, sgd.weight_decay)
    assert_values_close(g, st, TOL)


def test_c5_full_size_evolve_and_prune_bitexact():
    """SET evolution and Importance Pruning at full C5 size (52.3M connections; op-by-op parity on all five
    configs, C5 included): from the identical ER init (bit-exact, checked), one evolution on each
    side gives the identical topology and identical values -- survivors keep theirs, the ~6M
    regrown connections per hidden layer take the same Philox positions and init values."""
    from oracle import topology as T
    torch = _torch()
    cfg = get_config("C5")
    g, st = pair(cfg)
    assert_topology_equal(g, st, "C5 init")
    removed_g = g.evolve_topology(cfg.zeta, 3)
    removed_o = T.evolve(st, cfg.zeta, 3)
    torch.cuda.synchronize()
    assert list(removed_g[1:]) == list(removed_o)
    assert_topology_equal(g, st, "C5 evolve")
    for Ly in st.layers:
        e = g.export_layer(Ly.l)
        assert np.array_equal(e["w"].view(np.uint32), Ly.w.view(np.uint32)), f"C5 W^({Ly.l}) values"
        assert np.array_equal(e["v"].view(np.uint32), Ly.v.view(np.uint32)), f"C5 W^({Ly.l}) momentum"
    # Importance Pruning at full size (rho = 5, the paper's best post-training threshold): the fp64
    # importance sums and percentile decisions are reproduced exactly, so the same neurons die
    pruned_g, removed_g = g.prune_neurons(5.0)
    pruned_o, removed_o = T.prune(st, 5.0)
    torch.cuda.synchronize()
    assert list(pruned_g) == list(pruned_o) and list(removed_g) == list(removed_o)
    assert_topology_equal(g, st, "C5 prune")


@pytest.mark.gpu
@pytest.mark.parametrize("B,chunk,fchunk", [(128, 64, 32), (100, 64, None), (33, 32, None), (128, 32, None), (7, 16, None)])
def test_implicit_delta_matches_gathered_and_oracle(B, chunk, fchunk, monkeypatch):
    """Layer L-1 under a dense-capped 2-output layer (C1, like C4 / C5 / T1-T5): the backward of
    W^(L-1) recomputes delta_{L-1}[j] from 16-B per-neuron records (sign bits, w_j0, w_j1) and
    delta_L instead of gathering its rows.  Bit-identical to the gathering kernels
    (SMLP_IMPLICIT_DELTA=0) over several fused steps and a prune + evolve, and within 1e-4 of the
    oracle (P:596-599 for the step; Eq. 3's derivative P:106-112 is what the records carry)."""
    torch = _torch()
    from paper_2102_01732_b200 import SGD
    from tests.test_gpu_parity import _batch     # a kink-free seeded batch (R32)
    cfg = get_config("C1", batch=B)
    if fchunk:
        monkeypatch.setenv("SMLP_FWD_CB", str(fchunk))
    g1, st = pair(cfg, max_batch=128, chunk_batch=chunk)
    monkeypatch.setenv("SMLP_IMPLICIT_DELTA", "0")
    g0, _ = pair(cfg, max_batch=128, chunk_batch=chunk)
    assert g1.info()["implicit_delta"] == 1 and g0.info()["implicit_delta"] == 0
    assert g1.info()["dense_capped"][-1] == 1
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    L = cfg.n_layers
    for step in range(3):
        x, y, tr = _batch(cfg, st, B=B, step=step)
        for g in (g0, g1):
            g.forward(to_dev(x), train=True, step=step)
            g.backward(to_dev(y))
        torch.cuda.synchronize()
        for l in range(2, L + 1):
            for kind in (2, 3):       # weight and bias gradients: the same bits
                a, b = g0.sparse_mlp_export_trace(kind, l), g1.sparse_mlp_export_trace(kind, l)
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (step, kind, l)
        gr = M.backward(st, tr, y)
        for Ly in st.layers:
            assert rel_err(g1.sparse_mlp_export_trace(2, Ly.l), gr.g[Ly.l - 2], gr.gmag[Ly.l - 2]) <= TOL, ("g", Ly.l)
            assert rel_err(g1.sparse_mlp_export_trace(3, Ly.l), gr.gb[Ly.l - 2], gr.gbmag[Ly.l - 2]) <= TOL, ("gb", Ly.l)
        for g in (g0, g1):
            g.step(sgd)
        M.step(st, gr, cfg.lr, cfg.momentum, cfg.weight_decay)
        torch.cuda.synchronize()
        for l in range(2, L + 1):     # the updated weights and momenta: the same bits
            a, b = g0.export_layer(l), g1.export_layer(l)
            assert np.array_equal(a["w"].view(np.uint32), b["w"].view(np.uint32)), (step, "w", l)
            assert np.array_equal(a["v"].view(np.uint32), b["v"].view(np.uint32)), (step, "v", l)
        check_and_resync(g1, st)      # within 1e-4 of the oracle, then both restart from its state
        load_oracle_state_into_gpu(g0, st)
        if step == 0:     # pruned hidden neurons leave EMPTY rows in the dense-capped output layer
            import oracle.topology as T
            for g in (g0, g1):
                g.prune_neurons(0.3)
                g.evolve_topology(cfg.zeta, 0)
            T.prune(st, 0.3)
            T.evolve(st, cfg.zeta, 0)
            assert_topology_equal(g1, st, "after prune + evolve")
