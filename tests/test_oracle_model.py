"""Pins for oracle/model.py (CPU): ER init, forward, loss, backward, update.

Each test pins the oracle to something other than itself: numbers printed in the paper
(tests/golden/paper_counts.json), SPEC.md worked examples (cited), closed forms,
a dense masked float64 MLP (tests/dense_ref.py) that is itself pinned by finite
differences, and brute force on tiny inputs."""
import json
import math
import os

import numpy as np
import pytest

from oracle import model as M
from oracle import philox
from oracle.compare import rel_err
from synth import get_config, make_dataset
from tests import dense_ref

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_counts.json")))


def _items(d):
    return [(k, v) for k, v in d.items() if not k.startswith("_")]


# ----------------------------------------------------------------------------- ER counts
def test_dense_counts_reproduce_table2():
    """Sum n_{l-1} n_l + sum n_l (weights + biases) equals Table 2's dense counts: pins the
    layer shapes and that biases are counted with weights."""
    for name, e in _items(GOLD["dense_param_counts_table2"]):
        s = e["sizes"]
        cnt = sum(s[k] * s[k + 1] for k in range(len(s) - 1)) + sum(s[1:])
        assert cnt == e["count"], name


def test_er_formula_reproduces_table4_parameter_counts():
    """Uncapped sum_l eps(n_{l-1}+n_l) rounds to Table 4's printed counts:
    pins the epsilon formula eps(n_in+n_out)/(n_in n_out) itself."""
    for name, e in _items(GOLD["table4_param_counts"]):
        s, eps = e["sizes"], e["epsilon"]
        tot = sum(eps * (s[k] + s[k + 1]) for k in range(len(s) - 1))
        # the paper prints the count truncated to 0.1 M (20,655,380 -> "20.6 M")
        assert math.floor(tot / 1e5) / 10 == e["printed_millions"], name


def test_capped_er_count_matches_table2_start_counts_within_1pct():
    for name, e in _items(GOLD["table2_sparse_start_counts"]):
        s, eps = e["sizes"], e["epsilon"]
        tot = sum(M.er_count(s[k], s[k + 1], eps) for k in range(len(s) - 1))
        printed = e["printed"] if isinstance(e["printed"], list) else [e["printed"]]
        for p in printed:
            assert abs(tot - p) / p < 0.01, (name, tot, p)


def test_spec_er_example_784x1000():
    # n_in=784, n_out=1000, eps=20 -> expected nnz 35,680 (exact under G(n, M))
    assert M.er_count(784, 1000, 20) == 35680
    Ly = M.er_layer(784, 1000, 20.0, "he_uniform", 5, 2)
    assert Ly.nnz == 35680


@pytest.mark.parametrize("n_in,n_out,eps", [(30, 20, 3.0), (200, 200, 10.0), (7, 5, 1.0), (4, 3, 50.0)])
def test_er_layer_structure_and_density(n_in, n_out, eps):
    Ly = M.er_layer(n_in, n_out, eps, "xavier", 11, 3)
    Mcnt = M.er_count(n_in, n_out, eps)
    assert Ly.nnz == Mcnt
    assert Ly.row_ptr[0] == 0 and Ly.row_ptr[-1] == Mcnt and np.all(np.diff(Ly.row_ptr) >= 0)
    keys = Ly.keys()
    assert np.all(np.diff(keys) > 0)              # sorted, unique
    assert np.all((Ly.col >= 0) & (Ly.col < n_out))
    assert Ly.dense_capped == (Mcnt == n_in * n_out)
    assert np.all(Ly.v == 0)
    # density invariant eps(n_in+n_out)/(n_in n_out) (BASELINE north_star), capped at 1
    assert Ly.nnz / (n_in * n_out) == pytest.approx(min(1.0, math.floor(eps * (n_in + n_out)) / (n_in * n_out)))


def test_er_layer_equals_bruteforce_stream_scan():
    """First M distinct candidates of the INIT stream, by a plain Python loop."""
    n_in, n_out, eps, seed, l = 8, 8, 2.0, 99, 2
    Mcnt = M.er_count(n_in, n_out, eps)
    seen, acc = set(), []
    m = 0
    while len(acc) < Mcnt:
        x = philox.stream(seed, philox.PURPOSE_INIT, 0, l, 0, np.array([m], np.uint64))
        i = (int(x[0][0]) * n_in) >> 32
        j = (int(x[1][0]) * n_out) >> 32
        if (i, j) not in seen:
            seen.add((i, j))
            acc.append((i, j, int(x[2][0]), int(x[3][0])))
        m += 1
    acc.sort()
    Ly = M.er_layer(n_in, n_out, eps, "he_uniform", seed, l)
    assert [(int(r), int(c)) for r, c in zip(Ly.rows(), Ly.col)] == [(a[0], a[1]) for a in acc]
    lim = math.sqrt(6.0 / n_in)
    for (i, j, x2, x3), w in zip(acc, Ly.w):
        u = (x2 >> 8) / 2**24
        assert w == np.float32((2 * u - 1) * np.float32(lim))


def test_init_value_distributions():
    n = 200_000
    idx = np.arange(n, dtype=np.uint64)
    _, _, x2, x3 = philox.stream(3, 2, 0, 2, 0, idx)
    lim = math.sqrt(6.0 / 100)
    w = M.init_values("he_uniform", 100, 50, x2, x3).astype(np.float64)
    assert w.min() >= -lim - 1e-6 and w.max() < lim
    assert abs(w.mean()) < 6 * lim / math.sqrt(3 * n)
    assert w.var() == pytest.approx(lim**2 / 3, rel=0.02)
    wn = M.init_values("normal", 100, 50, x2, x3).astype(np.float64)
    assert abs(wn.mean()) < 6 * math.sqrt(2 / 100 / n)
    assert wn.var() == pytest.approx(2 / 100, rel=0.02)
    # fourth moment of a Gaussian: 3 sigma^4
    assert np.mean(wn**4) == pytest.approx(3 * (2 / 100) ** 2, rel=0.05)


def test_dense_capped_layer_complete():
    Ly = M.er_layer(10, 2, 10.0, "he_uniform", 1, 5)
    assert Ly.dense_capped and Ly.nnz == 20
    assert np.array_equal(Ly.dense(np.float64) != 0, np.ones((10, 2), bool)) or Ly.nnz == 20


# ----------------------------------------------------------------------------- SPEC examples
def _layer(n_in, n_out, entries):
    entries = sorted(entries)
    rows = np.array([e[0] for e in entries], dtype=np.int64)
    row_ptr = np.zeros(n_in + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n_in), out=row_ptr[1:]) if len(entries) else None
    return M.Layer(2, n_in, n_out, row_ptr, np.array([e[1] for e in entries], np.int32),
                   np.array([e[2] for e in entries], np.float32), np.zeros(len(entries), np.float32))


def test_spec_spmm_examples():
    # identity batch, single entry w[0][1] = 3, zero bias -> [[0,3],[0,0]]
    Ly = _layer(2, 2, [(0, 1, 3.0)])
    z = M.spmm_fwd(np.eye(2, dtype=np.float32), Ly)
    assert np.array_equal(z, [[0, 3], [0, 0]])
    # empty support -> zeros (bias added by the caller)
    Ly0 = _layer(3, 4, [])
    assert np.array_equal(M.spmm_fwd(np.ones((2, 3), np.float32), Ly0), np.zeros((2, 4)))


def test_spec_backward_scalar_chain_rule():
    # batch [[2]], upstream [[3]], single entry (0,0) -> g = 6, gb = 3, grad_input = 3 w
    w = 0.7
    Ly = _layer(1, 1, [(0, 0, w)])
    a = np.array([[2.0]], np.float32)
    d = np.array([[3.0]], np.float32)
    assert M.sddmm(a, d, Ly)[0] == 6.0
    assert d.sum(0)[0] == 3.0
    assert M.spmm_bwd(d, Ly)[0, 0] == pytest.approx(3 * np.float32(w))
    # zero upstream -> zero gradients
    assert np.all(M.sddmm(a, np.zeros_like(d), Ly) == 0)


def test_all_relu_examples_and_properties():
    # SPEC S:134-136 (Eq. 3): l=2, a=0.5, x=-2 -> +1; l=3 -> -1; x=3 -> 3
    assert M.activation(-2.0, 2, 0.5) == 1.0
    assert M.activation(-2.0, 3, 0.5) == -1.0
    assert M.activation(3.0, 4, 0.5) == 3.0
    # derivative slopes
    assert M.activation_grad(-1.0, 2, 0.75) == -0.75
    assert M.activation_grad(-1.0, 5, 0.75) == 0.75
    assert M.activation_grad(10.0, 3, 0.75) == 1.0
    # x = 0 takes the x <= 0 branch of Eq. 3 (value 0, slope of the negative side)
    assert M.activation(0.0, 2, 0.5) == 0.0 and M.activation_grad(0.0, 2, 0.5) == -0.5
    x = np.linspace(-3, 3, 61)
    # alpha = 0 reduces to ReLU (Eq. 5)
    assert np.array_equal(M.activation(x, 2, 0.0), np.maximum(x, 0))
    assert np.array_equal(M.activation(x, 2, 0.3, "relu"), np.maximum(x, 0))
    # alternation f_l(x) = -f_{l+1}(x) for x < 0
    neg = x[x < 0]
    assert np.array_equal(M.activation(neg, 2, 0.3), -M.activation(neg, 3, 0.3))
    # continuity at 0
    for l in (2, 3):
        assert abs(M.activation(-1e-12, l, 0.6)) < 1e-11 and abs(M.activation(1e-12, l, 0.6)) < 1e-11


def test_loss_examples():
    # uniform logits -> ln C
    p = np.full((3, 10), 0.1)
    loss, d = M.loss_grad(p, np.array([0, 4, 9]))
    assert loss == pytest.approx(math.log(10))
    # B=1, logits [0,0], label 0 -> dlogits [-0.5, +0.5]
    loss, d = M.loss_grad(np.array([[0.5, 0.5]]), np.array([0]))
    assert np.allclose(d, [[-0.5, 0.5]])
    with pytest.raises(ValueError):
        M.loss_grad(np.array([[0.5, 0.5]]), np.array([2]))


def test_dropout_mask_statistics():
    keep = M.dropout_keep(5, 0, 2, 17, 64, 1000, 0.3)
    assert keep.shape == (64, 1000)
    frac = keep.mean()
    n = keep.size
    assert abs(frac - 0.7) < 6 * math.sqrt(0.21 / n)
    assert np.array_equal(keep, M.dropout_keep(5, 0, 2, 17, 64, 1000, 0.3))      # deterministic
    assert not np.array_equal(keep, M.dropout_keep(5, 1, 2, 17, 64, 1000, 0.3))  # rank-dependent
    assert M.dropout_keep(5, 0, 2, 17, 4, 10, 0.0).all()
    # an element's keep bit depends on (b, j) only: the mask of a smaller batch / narrower layer
    # is a prefix (so a ragged last batch and every chunking see the same bits)
    assert np.array_equal(keep[:37], M.dropout_keep(5, 0, 2, 17, 37, 1000, 0.3))
    assert np.array_equal(keep[:, :333], M.dropout_keep(5, 0, 2, 17, 64, 333, 0.3))
    # and the four rows of one group of 4 use four different words (no repeated pattern)
    assert not np.array_equal(keep[0], keep[1]) and not np.array_equal(keep[0], keep[4])


# ----------------------------------------------------------------------------- dense equivalence
def _small_state(sizes=(12, 10, 9, 7, 4), eps=2.0, act="all_relu", alpha=0.6, dropout=0.0, seed=3):
    st = M.create(sizes, eps, act, alpha, dropout, "he_uniform", seed)
    rng = np.random.default_rng(seed)
    for i in range(len(st.b)):
        st.b[i] = rng.standard_normal(st.b[i].shape).astype(np.float32) * 0.1
    return st


@pytest.mark.parametrize("act,alpha,dropout", [("all_relu", 0.6, 0.0), ("relu", 0.0, 0.0),
                                               ("all_relu", 0.05, 0.3), ("all_relu", 0.75, 0.0)])
def test_oracle_matches_dense_masked_mlp(act, alpha, dropout):
    st = _small_state(act=act, alpha=alpha, dropout=dropout)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((7, 12)).astype(np.float32)
    y = rng.integers(0, 4, 7)
    tr = M.forward(st, x, True, step=5)
    gr = M.backward(st, tr, y)
    Ws = [Ly.dense(np.float64) for Ly in st.layers]
    bs = [b.astype(np.float64) for b in st.b]
    keeps = [k for k in tr.keep[1:-1]] if dropout > 0 else None
    loss, p, dWs, dbs = dense_ref.forward_backward(Ws, bs, x.astype(np.float64), y, alpha, act,
                                                   keeps=keeps, rate=dropout)
    assert gr.loss == pytest.approx(loss, rel=1e-6)
    assert rel_err(tr.p, p) < 1e-5
    for k, Ly in enumerate(st.layers):
        # the oracle rounds stored tensors (a_l, delta_l) to fp32; the dense
        # reference does not, so agreement is to fp32 rounding amplified by cancellation.
        assert rel_err(gr.g[k], dWs[k][Ly.rows(), Ly.col]) < 1e-4
        assert rel_err(gr.gb[k], dbs[k]) < 1e-4


def test_dense_ref_matches_finite_differences():
    """Pin of the pin: dense_ref gradients vs central differences (h = 1e-6, float64)."""
    rng = np.random.default_rng(4)
    sizes = (6, 5, 4, 3)
    masks = [rng.random((sizes[k], sizes[k + 1])) < 0.6 for k in range(3)]
    Ws = [rng.standard_normal(m.shape) * m for m in masks]
    bs = [rng.standard_normal(sizes[k + 1]) * 0.1 for k in range(3)]
    x = rng.standard_normal((5, 6))
    y = rng.integers(0, 3, 5)
    for kind, alpha in (("all_relu", 0.5), ("relu", 0.0), ("all_relu", 0.05)):
        _, _, dWs, dbs = dense_ref.forward_backward(Ws, bs, x, y, alpha, kind)
        h = 1e-6
        for k in range(3):
            for (i, j) in zip(*np.nonzero(masks[k])):
                Wp = [W.copy() for W in Ws]
                Wm = [W.copy() for W in Ws]
                Wp[k][i, j] += h
                Wm[k][i, j] -= h
                fd = (dense_ref.loss_only(Wp, bs, x, y, alpha, kind) -
                      dense_ref.loss_only(Wm, bs, x, y, alpha, kind)) / (2 * h)
                assert fd == pytest.approx(dWs[k][i, j], rel=1e-4, abs=1e-8)
            for j in range(sizes[k + 1]):
                bp = [b.copy() for b in bs]
                bm = [b.copy() for b in bs]
                bp[k][j] += h
                bm[k][j] -= h
                fd = (dense_ref.loss_only(Ws, bp, x, y, alpha, kind) -
                      dense_ref.loss_only(Ws, bm, x, y, alpha, kind)) / (2 * h)
                assert fd == pytest.approx(dbs[k][j], rel=1e-4, abs=1e-8)


def test_eval_forward_has_no_dropout_and_train_is_deterministic():
    st = _small_state(dropout=0.3)
    x = np.random.default_rng(2).standard_normal((4, 12)).astype(np.float32)
    a = M.forward(st, x, True, 3)
    b = M.forward(st, x, True, 3)
    assert np.array_equal(a.p, b.p)
    e = M.forward(st, x, False, 3)
    st0 = _small_state(dropout=0.0)
    assert np.array_equal(e.p, M.forward(st0, x, True, 3).p)
    assert np.allclose(a.p.sum(1), 1.0, atol=1e-6)


def test_stale_trace_rejected():
    st = _small_state()
    x = np.zeros((2, 12), np.float32)
    tr = M.forward(st, x, True, 0)
    st.version += 1
    with pytest.raises(RuntimeError):
        M.backward(st, tr, np.array([0, 1]))
    with pytest.raises(RuntimeError):
        st.version -= 1
        M.backward(st, M.forward(st, x, False, 0), np.array([0, 1]))


# ----------------------------------------------------------------------------- update (Eq. 1)
def _one_weight_state(w0=0.0):
    st = _small_state(sizes=(1, 1, 1), eps=1.0)
    st.layers[0].w[:] = w0
    st.layers[1].w[:] = 0.0
    return st


def _grads_for(st, gval):
    return M.Grads([np.array([gval], np.float32), np.zeros(st.layers[1].nnz, np.float32)],
                   [np.zeros(1, np.float32), np.zeros(1, np.float32)], 0.0, [None] * 3)


def test_spec_momentum_two_step_example():
    # g = (1, then 0), eta = 1, mu = 0.5, w0 = 0 -> w1 = -1, w2 = -1.5
    st = _one_weight_state(0.0)
    M.step(st, _grads_for(st, 1.0), 1.0, 0.5, 0.0)
    assert st.layers[0].w[0] == -1.0
    M.step(st, _grads_for(st, 0.0), 1.0, 0.5, 0.0)
    assert st.layers[0].w[0] == -1.5


def test_velocity_form_equals_eq1_recursion():
    """Eq. 1: w_{t+1} = w_t + mu (w_t - w_{t-1}) - eta g_t, over 10 steps."""
    rng = np.random.default_rng(9)
    gs = rng.standard_normal(10)
    eta, mu = 0.1, 0.9
    st = _one_weight_state(0.25)
    w_prev, w = 0.25, 0.25
    for g in gs:
        M.step(st, _grads_for(st, float(np.float32(g))), eta, mu, 0.0)
        w_next = w + mu * (w - w_prev) - eta * float(np.float32(g))
        w_prev, w = w, w_next
        assert float(st.layers[0].w[0]) == pytest.approx(w, rel=1e-5, abs=1e-6)


def test_plain_sgd_and_decay_isolation():
    st = _one_weight_state(2.0)
    M.step(st, _grads_for(st, 0.5), 0.1, 0.0, 0.0)              # mu = 0: w - eta g
    assert st.layers[0].w[0] == np.float32(2.0 - 0.05)
    st = _one_weight_state(2.0)
    M.step(st, _grads_for(st, 0.0), 0.1, 0.0, 0.01)             # zero upstream: g = lambda w
    assert st.layers[0].w[0] == np.float32(2.0 - 0.1 * 0.01 * 2.0)


def test_sampled_backward_equals_full_backward():
    """oracle/sampled.py (the cone evaluation the full-size C5 parity test uses) against the full
    oracle backward on a small net with dropout: every delta, gradient and bias gradient."""
    from oracle import sampled as S
    cfg = get_config("C1", sizes=(60, 50, 40, 30, 3), epsilon=4.0, dropout=0.25, batch=17)
    st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, 5)
    X, Y = make_dataset(cfg, n=17)
    M.train_step(st, X, Y, 0.5, 0.9, 2e-4, 0)            # non-trivial biases and weights
    tr = M.forward(st, X, True, 1)
    gr = M.backward(st, tr, Y)
    need = {l: range(cfg.sizes[l - 1]) for l in range(2, st.L + 1)}
    deltas, tainted, dmags = S.delta_columns(st, tr, Y, need)
    for l in range(2, st.L + 1):
        D = np.stack([deltas[l][j] for j in range(cfg.sizes[l - 1])], axis=1)
        np.testing.assert_allclose(D, gr.deltas[l - 1], rtol=1e-6, atol=1e-9)
        Dm = np.stack([dmags[l][j] for j in range(cfg.sizes[l - 1])], axis=1)
        np.testing.assert_allclose(Dm, gr.dmag[l - 1], rtol=1e-5, atol=1e-12)   # f32 magnitudes in the full pass
        gb, gbm = S.bias_grad_columns(deltas, dmags, l, np.arange(cfg.sizes[l - 1]))
        np.testing.assert_allclose(gb, gr.gb[l - 2], rtol=1e-6, atol=1e-9)
        np.testing.assert_allclose(gbm, gr.gbmag[l - 2], rtol=1e-5, atol=1e-12)
        k = np.arange(st.layer(l).nnz)
        g, gm = S.grad_entries(st, tr, deltas, dmags, l, k)
        np.testing.assert_allclose(g, gr.g[l - 2], rtol=1e-6, atol=1e-9)
        np.testing.assert_allclose(gm, gr.gmag[l - 2], rtol=1e-5, atol=1e-12)
    assert not any(t.any() for tl in tainted.values() for t in tl.values())   # no kink-ambiguous element here
    # a sparse request only evaluates its cone and gives the same columns
    d2, _, _ = S.delta_columns(st, tr, Y, {2: [3, 7]})
    assert set(d2[2]) == {3, 7} and len(d2[3]) < cfg.sizes[2] + 1
    np.testing.assert_array_equal(d2[2][7], deltas[2][7])


def test_kink_guard_ignores_exact_zero_preactivations():
    """Binary inputs with no active input and zero bias give z = 0 exactly on every path (R32)."""
    cfg = get_config("C1", sizes=(40, 30, 20, 2), epsilon=2.0, dropout=0.0, batch=8)
    st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, 0.0, cfg.init, 3)
    x = np.zeros((8, 40), np.float32)
    tr = M.forward(st, x, True, 0)
    assert np.all(tr.z[1] == 0) and sum(tr.ambiguous) == 0


# ---------------------------------------------------------------- gradient flow (§8(f) item 2)
def test_gradient_flow_pins():
    """PAPER.md:315 / SPEC S:187-195: the squared L2 norm of all existing-weight and bias
    gradients.  Pins: zero gradients -> 0; a single entry 3 -> 9; equals the dense-masked
    reference's squared gradient norm (independent fp64 backprop) on a small network."""
    st = M.create((7, 6, 5, 3), 3.0, "all_relu", 0.4, 0.0, "he_uniform", 13)
    z = M.Grads([np.zeros_like(L.w) for L in st.layers], [np.zeros_like(b) for b in st.b], 0.0, [])
    assert M.gradient_flow(z) == 0.0
    one = M.Grads([np.zeros_like(L.w) for L in st.layers], [np.zeros_like(b) for b in st.b], 0.0, [])
    one.g[1][2] = 3.0
    assert M.gradient_flow(one) == 9.0
    rng = np.random.default_rng(4)
    x = rng.standard_normal((9, 7)).astype(np.float32)
    y = rng.integers(0, 3, 9)
    tr = M.forward(st, x, True, 0)
    gr = M.backward(st, tr, y)
    Ws = [Ly.dense(np.float64) for Ly in st.layers]
    bs = [b.astype(np.float64) for b in st.b]
    _, _, dWs, dbs = dense_ref.forward_backward(Ws, bs, x.astype(np.float64), y, 0.4, "all_relu")
    # the masked dense gradient restricted to the support (off-support entries are not parameters)
    ref = sum(float(np.sum(np.square(dWs[k][Ly.rows(), Ly.col]))) for k, Ly in enumerate(st.layers))
    ref += sum(float(np.sum(np.square(b))) for b in dbs)
    assert abs(M.gradient_flow(gr) - ref) <= 1e-4 * ref


def test_sparse_products_against_scipy_and_dense(monkeypatch):
    """The oracle's plain-NumPy products (segmented sums over the support) against two independent
    computations: a SciPy CSR product (SciPy only in oracle self-tests) and
    the dense zero-filled matrix.  A tiny chunk size forces output segments to be
    split across chunks, and empty rows / columns occur."""
    import scipy.sparse as sp
    monkeypatch.setattr(M, "_CHUNK_ELEMS", 37)
    Ly = M.er_layer(53, 41, 0.8, "he_uniform", 9, 2)
    assert np.any(np.diff(Ly.row_ptr) == 0) and len(np.unique(Ly.col)) < Ly.n_out
    rng = np.random.default_rng(3)
    a = rng.standard_normal((6, 53)).astype(np.float32)
    d = rng.standard_normal((6, 41)).astype(np.float32)
    W = sp.csr_matrix((Ly.w.astype(np.float64), Ly.col, Ly.row_ptr), shape=(53, 41))
    D = Ly.dense()
    z = M.spmm_fwd(a, Ly)
    np.testing.assert_allclose(z, (W.T @ a.astype(np.float64).T).T, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(z, a.astype(np.float64) @ D, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(M.spmm_fwd(a, Ly, wabs=True), np.abs(a).astype(np.float64) @ np.abs(D),
                               rtol=1e-12, atol=1e-12)
    bk = M.spmm_bwd(d, Ly)
    np.testing.assert_allclose(bk, (W @ d.astype(np.float64).T).T, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(bk, d.astype(np.float64) @ D.T, rtol=1e-12, atol=1e-12)
    g = M.sddmm(a, d, Ly)
    full = a.astype(np.float64).T @ d.astype(np.float64)
    np.testing.assert_allclose(g, full[Ly.rows(), Ly.col], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed,dropout,alpha", [(1, 0.0, 0.6), (2, 0.3, 0.75), (3, 0.2, 0.05), (4, 0.0, 0.5)])
def test_error_magnitudes_bound_an_fp32_implementation(seed, dropout, alpha):
    """DESIGN.md R24 pin: the oracle's running error magnitudes bound the difference between the
    fp64 oracle and an INDEPENDENT fp32 implementation of the same step (tests/dense_ref.py in
    float32: dense masked matrices, BLAS sgemm summation order), element by element, for every
    activation, logit, probability, delta, weight / bias gradient and -- after two Eq. 1 steps --
    every weight, momentum and bias:  |fp32 - oracle| <= KAPPA_U * mag.  And the bound is not
    vacuous: KAPPA_U * mag stays below 1e-4 relative wherever the value is not a cancellation."""
    from oracle.compare import KAPPA_U, rel_err
    cfg = get_config("C1", sizes=(70, 60, 50, 40, 3), epsilon=6.0, alpha=alpha, dropout=dropout, batch=32)
    st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, seed)
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((64, 70)).astype(np.float32)
    Y = rng.integers(0, 3, 64)
    lr, mu, wd = 0.05, 0.9, 2e-4
    Ws32 = [Ly.dense(np.float32) for Ly in st.layers]
    bs32 = [b.copy() for b in st.b]
    Vs32 = [np.zeros_like(W) for W in Ws32]
    vb32 = [np.zeros_like(b) for b in bs32]
    for s_ in range(2):
        x, y = X[s_ * 32:(s_ + 1) * 32], Y[s_ * 32:(s_ + 1) * 32]
        tr = M.forward(st, x, True, s_)
        gr = M.backward(st, tr, y)
        keeps = [tr.keep[k + 1] for k in range(len(st.layers) - 1)] + [None]
        out = {}
        _, p32, dW32, db32 = dense_ref.forward_backward(Ws32, bs32, x, y, alpha, "all_relu", keeps, dropout,
                                                        np.float32, out)
        if sum(tr.ambiguous) == 0:
            for k in range(1, st.L - 1):
                d = np.abs(out["a"][k].astype(np.float64) - tr.a[k])
                assert np.all(d <= KAPPA_U * tr.amag[k]), ("a", s_, k + 1)
            assert np.all(np.abs(p32 - tr.p64) <= KAPPA_U * tr.pmag + 2.0 ** -23 * tr.p64)
            for k, Ly in enumerate(st.layers):
                g32 = dW32[k][Ly.rows(), Ly.col].astype(np.float64)
                assert np.all(np.abs(g32 - gr.g[k]) <= KAPPA_U * gr.gmag[k] + 2.0 ** -24 * np.abs(gr.g[k])), ("g", s_, k)
                assert np.all(np.abs(db32[k] - gr.gb[k]) <= KAPPA_U * gr.gbmag[k] + 2.0 ** -24 * np.abs(gr.gb[k]))
                if k >= 1:
                    dd = np.abs(out["delta"][k + 1].astype(np.float64) - gr.deltas[k + 1])
                    assert np.all(dd <= KAPPA_U * gr.dmag[k + 1] + 2.0 ** -24 * np.abs(gr.deltas[k + 1])), ("delta", k)
            # not vacuous: where the activation is not a cancellation (|a| >= mag / 16), the error
            # bound is far below the 1e-4 relative target
            for k in range(1, st.L - 1):
                big = np.abs(tr.a[k]) >= tr.amag[k] / 16
                assert np.all(KAPPA_U * tr.amag[k][big] <= 1e-4 * np.abs(tr.a[k][big]))
        M.step(st, gr, lr, mu, wd)
        for k in range(len(Ws32)):
            g = dW32[k] + wd * Ws32[k]
            Vs32[k] = (np.float32(mu) * Vs32[k] - np.float32(lr) * g.astype(np.float32)).astype(np.float32)
            Ws32[k] = ((Ws32[k] + Vs32[k]) * (Ws32[k] != 0)).astype(np.float32)
            vb32[k] = (np.float32(mu) * vb32[k] - np.float32(lr) * db32[k]).astype(np.float32)
            bs32[k] = (bs32[k] + vb32[k]).astype(np.float32)
    for k, Ly in enumerate(st.layers):
        w32 = Ws32[k][Ly.rows(), Ly.col]
        v32 = Vs32[k][Ly.rows(), Ly.col]
        assert np.all(np.abs(w32.astype(np.float64) - Ly.w) <= KAPPA_U * Ly.wmag), ("w", k)
        assert np.all(np.abs(v32.astype(np.float64) - Ly.v) <= KAPPA_U * Ly.vmag), ("v", k)
        assert np.all(np.abs(bs32[k].astype(np.float64) - st.b[k]) <= KAPPA_U * st.bmag[k]), ("b", k)
        # and the comparison metric built on it passes the fp32 implementation
        assert rel_err(w32, Ly.w, Ly.wmag) <= 1e-4 and rel_err(v32, Ly.v, Ly.vmag) <= 1e-4


def test_sampled_taint_is_exactly_the_kink_dependence(monkeypatch):
    """R32 pin for the per-(b, j) taint of oracle/sampled.py: (1) with the documented band the
    per-column kink test reproduces the full forward's ambiguous count; (2) with a wide band
    (many ambiguous elements), flipping the sign of every ambiguous pre-activation -- i.e. taking
    the other branch of f' there -- changes only tainted deltas, and changes some."""
    from oracle import sampled as S
    cfg = get_config("C1", sizes=(60, 50, 40, 30, 3), epsilon=4.0, dropout=0.2, batch=17)
    st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, 8)
    X, Y = make_dataset(cfg, n=17)
    tr = M.forward(st, X, True, 0)
    for l in range(2, st.L):
        cnt = int(S.kink_columns(st, tr, l, np.arange(cfg.sizes[l - 1])).sum())
        assert cnt == tr.ambiguous[l - 1]
    monkeypatch.setattr(S, "KINK_REL", 0.02)
    need = {l: range(cfg.sizes[l - 1]) for l in range(2, st.L + 1)}
    deltas, tainted, _ = S.delta_columns(st, tr, Y, need)
    import copy
    tr2 = copy.copy(tr)
    tr2.z = list(tr.z)
    for l in range(2, st.L):
        amb = S.kink_columns(st, tr, l, np.arange(cfg.sizes[l - 1]))
        assert amb.any()
        z = tr.z[l - 1].copy()
        z[amb] = np.where(z[amb] > 0, -z[amb], np.abs(z[amb]) + 1e-30)
        tr2.z[l - 1] = z
    d2, _, _ = S.delta_columns(st, tr2, Y, need)
    changed_any = False
    for l in range(2, st.L):
        for j in range(cfg.sizes[l - 1]):
            ch = deltas[l][j] != d2[l][j]
            assert not np.any(ch & ~tainted[l][j]), (l, j)
            changed_any |= bool(ch.any())
    assert changed_any
