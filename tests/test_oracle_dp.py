"""Pins for oracle/dp.py (CPU): K-rank synchronous DP (WASSP phase 1) and Eq. 2 averaging."""
import copy

import numpy as np
import pytest

from oracle import dp
from oracle import model as M
from oracle import topology as T
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


# ---------------------------------------------------------------- union averaging (WASAP phase 2)
def _tiny_pair_disjoint():
    """Two replicas of a 2 x 2 layer with one connection each at different positions."""
    sts = []
    for pos, w in (((0, 1), 4.0), ((1, 0), 2.0)):
        st = M.create((2, 2, 2), 0.5, "all_relu", 0.5, 0.0, "he_uniform", 1)
        Ly = st.layers[0]
        Ly.row_ptr = np.array([0, 1 if pos[0] == 0 else 0, 1], np.int64)
        Ly.col = np.array([pos[1]], np.int32)
        Ly.w = np.array([w], np.float32)
        Ly.v = np.zeros(1, np.float32)
        sts.append(st)
    return sts


def test_union_average_spec_example():
    """Disjoint single entries 4 and 2 -> union values {2, 1} after / K = 2; prune to 1 keeps 2."""
    a, b = _tiny_pair_disjoint()
    kept = dp.average_union([a, b], [1, a.layers[1].nnz])
    assert kept[0] == 1
    for s in (a, b):
        Ly = s.layers[0]
        assert Ly.w.tolist() == [2.0] and Ly.col.tolist() == [1] and Ly.row_ptr.tolist() == [0, 1, 1]
    a, b = _tiny_pair_disjoint()
    dp.average_union([a, b], [2, a.layers[1].nnz])   # no pruning: the union, position order
    assert a.layers[0].w.tolist() == [2.0, 1.0] and a.layers[0].keys().tolist() == [1, 2]


def test_union_average_k1_identity_and_identical_supports():
    st = _st()
    ref = copy.deepcopy(st)
    dp.average_union([st], [L.nnz for L in st.layers])          # K = 1, own counts: identity
    for p, q in zip(st.layers, ref.layers):
        assert np.array_equal(p.col, q.col) and np.array_equal(p.w.view(np.uint32), q.w.view(np.uint32))
        assert not np.any(p.v)
    # identical supports, target = nnz: the plain Eq. 2 mean (average()) up to the float32 sum
    a, b = _st(seed=4), _st(seed=4)
    rng = np.random.default_rng(2)
    for L in b.layers:
        L.w = (L.w + rng.standard_normal(L.w.shape).astype(np.float32) * 0.01).astype(np.float32)
    a2, b2 = copy.deepcopy(a), copy.deepcopy(b)
    dp.average_union([a, b], [L.nnz for L in a.layers])
    dp.average([a2, b2])
    for p, q in zip(a.layers, a2.layers):
        assert np.array_equal(p.col, q.col)
        assert np.max(np.abs(p.w - q.w)) <= 1e-7


def test_union_average_evolved_replicas_invariants_and_brute_force():
    """K = 4 replicas evolved independently: union >= every support, exactly `target` kept, and
    the kept set is the brute-force top-target |mean| (ties by position)."""
    base = _st(seed=11)
    sts = []
    for k in range(4):
        s = copy.deepcopy(base)
        T.evolve(s, 0.3, 100 + k)                              # independent topologies
        sts.append(s)
    targets = [L.nnz for L in base.layers]
    supports = [[set(L.keys().tolist()) for L in s.layers] for s in sts]
    vals = [[dict(zip(L.keys().tolist(), L.w.tolist())) for L in s.layers] for s in sts]
    kept = dp.average_union(sts, targets)
    for idx, target in enumerate(targets):
        union = set().union(*[supports[k][idx] for k in range(4)])
        assert len(union) >= max(len(supports[k][idx]) for k in range(4))
        assert kept[idx] == min(target, len(union)) and sts[0].layers[idx].nnz == kept[idx]
        mean = {}
        for p in sorted(union):
            sv = None
            for k in range(4):
                if p in vals[k][idx]:
                    w = np.float32(vals[k][idx][p])
                    sv = w if sv is None else np.float32(sv + w)
            mean[p] = np.float32(sv) / np.float32(4)
        ranked = sorted(union, key=lambda p: (int(np.float32(mean[p]).view(np.uint32)) & 0x7fffffff, p))
        expect = sorted(ranked[len(union) - kept[idx]:])
        assert sts[0].layers[idx].keys().tolist() == expect
        assert sts[0].layers[idx].w.tolist() == [float(mean[p]) for p in expect]
    for s in sts[1:]:                                          # every replica holds the same model
        for p, q in zip(s.layers, sts[0].layers):
            assert np.array_equal(p.keys(), q.keys()) and np.array_equal(p.w, q.w)


# ---------------------------------------------------------------- RetainValidUpdates (async phase 1)
def test_retain_valid_updates_pins():
    """identity when the topology did not change; worker {(0,0),(0,1)} vs server
    {(0,1),(1,1)} keeps only (0,1); after a random evolution the applied support is a subset of
    the server support and equals the set intersection (brute force)."""
    st = _st(seed=8)
    keys = [L.keys() for L in st.layers]
    gs = [np.arange(1, L.nnz + 1, dtype=np.float32) for L in st.layers]
    same = dp.retain_valid_updates(keys, gs, st)
    assert all(np.array_equal(a, b) for a, b in zip(same, gs))
    # the 2 x 2 example
    srv = M.create((2, 2, 2), 0.5, "all_relu", 0.5, 0.0, "he_uniform", 1)
    Ly = srv.layers[0]
    Ly.row_ptr = np.array([0, 1, 2], np.int64)
    Ly.col = np.array([1, 1], np.int32)                # server: (0,1), (1,1)
    Ly.w = np.ones(2, np.float32)
    Ly.v = np.zeros(2, np.float32)
    worker_keys = [np.array([0, 1], np.int64)] + [L.keys() for L in srv.layers[1:]]   # (0,0), (0,1)
    worker_g = [np.array([5.0, 7.0], np.float32)] + [np.zeros(L.nnz, np.float32) for L in srv.layers[1:]]
    g = dp.retain_valid_updates(worker_keys, worker_g, srv)
    assert g[0].tolist() == [7.0, 0.0]
    # randomized: evolve between push and apply
    rng = np.random.default_rng(0)
    for trial in range(5):
        s = _st(seed=20 + trial)
        k0 = [L.keys() for L in s.layers]
        g0 = [rng.standard_normal(L.nnz).astype(np.float32) for L in s.layers]
        T.evolve(s, 0.3, trial)
        g1 = dp.retain_valid_updates(k0, g0, s)
        for L, kk, gg, out in zip(s.layers, k0, g0, g1):
            inter = set(kk.tolist()) & set(L.keys().tolist())
            nz = {p for p, v in zip(L.keys().tolist(), out.tolist()) if v != 0.0}
            assert nz <= inter
            table = dict(zip(kk.tolist(), gg.tolist()))
            assert out.tolist() == [np.float32(table.get(p, 0.0)) for p in L.keys().tolist()]
