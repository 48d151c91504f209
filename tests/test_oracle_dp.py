"""Pins for oracle/dp.py (CPU): K-rank synchronous DP (WASSP phase 1) and Eq. 2 averaging."""
import numpy as np
import pytest

from oracle import dp
from oracle import model as M
from oracle.compare import rel_err


def _st(dropout=0.0, seed=4):
    return M.create((16, 12, 10, 3), 2.0, "all_relu", 0.5, dropout, "he_uniform", seed)


def _batch(rng, B):
    return rng.standard_normal((B, 16)).astype(np.float32), rng.integers(0, 3, B)


def test_k1_equals_sequential_bit_exactly():
    # K = 1 degenerate sync is sequential training
    a, b = _st(0.3), _st(0.3)
    rng = np.random.default_rng(0)
    for t in range(3):
        x, y = _batch(rng, 8)
        dp.dp_step(a, [(x, y)], 0.05, 0.9, 1e-4, t)
        M.train_step(b, x, y, 0.05, 0.9, 1e-4, t)
    for p, q in zip(a.layers, b.layers):
        assert np.array_equal(p.w.view(np.uint32), q.w.view(np.uint32))
        assert np.array_equal(p.v.view(np.uint32), q.v.view(np.uint32))


def test_k_ranks_equal_one_rank_with_union_batch():
    """Mean of per-rank gradients (1/B_k each) == gradient of the union batch (exact
    arithmetic), so K ranks of B equal 1 rank of K*B up to summation order."""
    K, B = 4, 6
    a, b = _st(), _st()
    rng = np.random.default_rng(1)
    batches = [_batch(rng, B) for _ in range(K)]
    dp.dp_step(a, batches, 0.05, 0.9, 0.0, 0)
    X = np.concatenate([x for x, _ in batches])
    Y = np.concatenate([y for _, y in batches])
    M.train_step(b, X, Y, 0.05, 0.9, 0.0, 0)
    for p, q in zip(a.layers, b.layers):
        assert rel_err(p.w, q.w) < 1e-5
        assert rel_err(p.v, q.v) < 1e-4


def test_known_gradients_average_exactly():
    # scripted per-rank gradients -> applied gradient is their mean
    st = _st()
    gs = []
    for k in range(3):
        g = [np.full(Ly.nnz, float(k + 1), np.float32) for Ly in st.layers]
        gb = [np.full(len(b), float(2 * k), np.float32) for b in st.b]
        gs.append(M.Grads(g, gb, 0.0, [None] * st.L))
    tot = dp.allreduce_sum(gs)
    w0 = [Ly.w.copy() for Ly in st.layers]
    M.step(st, tot, 1.0, 0.0, 0.0, grad_scale=1.0 / 3)
    for Ly, w in zip(st.layers, w0):
        assert np.array_equal(Ly.w, (w.astype(np.float64) - 2.0).astype(np.float32))


def test_scaled_lr_warmup():
    assert dp.scaled_lr(0.01, 1, 5, 10) == 0.01
    assert dp.scaled_lr(0.01, 8, 0, 10) == 0.01
    assert dp.scaled_lr(0.01, 8, 5, 10) == pytest.approx(0.01 * 4.5)
    assert dp.scaled_lr(0.01, 8, 50, 10) == pytest.approx(0.08)


def test_average_identity_and_mean():
    a = _st(seed=4)
    dp.average([a])
    assert np.array_equal(a.layers[0].w, _st(seed=4).layers[0].w)     # K = 1 identity
    sts = [_st(seed=4) for _ in range(3)]
    for k, s in enumerate(sts):
        for Ly in s.layers:
            Ly.w = Ly.w + np.float32(k)
    ref = [np.mean([s.layers[i].w.astype(np.float64) for s in sts], axis=0) for i in range(3)]
    dp.average(sts)
    for s in sts:
        for i, Ly in enumerate(s.layers):
            assert np.max(np.abs(Ly.w - ref[i])) <= 1e-6 * np.max(np.abs(ref[i]))
    with pytest.raises(ValueError):
        dp.average([_st(seed=4), _st(seed=5)])
