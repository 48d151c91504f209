"""Pins for oracle/topology.py (CPU): SET evolve, importance (Eq. 4), Importance Pruning."""
import math

import numpy as np
import pytest

from oracle import model as M
from oracle import philox
from oracle import topology as T


def _state(sizes=(20, 16, 16, 4), eps=2.0, seed=5, init="he_uniform"):
    return M.create(sizes, eps, "all_relu", 0.5, 0.0, init, seed)


# ----------------------------------------------------------------------------- selection
def test_spec_set_examples():
    # {+4, +0.1, -0.05, -7}, zeta = 0.5 -> removes +0.1 and -0.05
    w = np.array([4.0, 0.1, -0.05, -7.0], np.float32)
    flags, kp, kn = T.select_removals(w, 0.5)
    assert list(np.flatnonzero(flags)) == [1, 2] and (kp, kn) == (1, 1)
    # 1 positive weight, zeta = 0.3 -> floor(0.3) = 0 removals
    flags, kp, kn = T.select_removals(np.array([0.5], np.float32), 0.3)
    assert not flags.any() and kp == kn == 0


def test_selection_equals_bruteforce_sort_with_ties_and_signed_zero():
    rng = np.random.default_rng(0)
    for trial in range(50):
        n = int(rng.integers(1, 60))
        w = rng.choice(np.array([-0.0, 0.0, 0.25, -0.25, 1.0, -1.0, 0.5], np.float32), size=n)
        w = np.where(rng.random(n) < 0.5, w, rng.standard_normal(n).astype(np.float32))
        zeta = float(rng.choice([0.1, 0.3, 0.5, 0.9]))
        flags, kp, kn = T.select_removals(w, zeta)
        # brute force: Python sort of (|w|, index) per sign class (sign via math.copysign)
        pos = [k for k in range(n) if math.copysign(1.0, float(w[k])) > 0]
        neg = [k for k in range(n) if math.copysign(1.0, float(w[k])) < 0]
        exp = set(sorted(pos, key=lambda k: (abs(float(w[k])), k))[:int(zeta * len(pos))])
        exp |= set(sorted(neg, key=lambda k: (abs(float(w[k])), k))[:int(zeta * len(neg))])
        assert set(np.flatnonzero(flags)) == exp


# ----------------------------------------------------------------------------- evolve
def test_evolve_invariants():
    st = _state()
    rng = np.random.default_rng(1)
    for Ly in st.layers:
        Ly.v[:] = rng.standard_normal(Ly.nnz).astype(np.float32)
    pre = st.copy()
    out = T.evolve(st, 0.3, 0)
    assert st.version == pre.version + 1
    for k, (a, b) in enumerate(zip(pre.layers, st.layers)):
        if a.dense_capped:
            assert out[k] == -1 and np.array_equal(a.w, b.w)
            continue
        assert b.nnz == a.nnz                                   # conserved
        pre_keys = a.keys()
        post_keys = b.keys()
        assert np.all(np.diff(post_keys) > 0)
        surv = np.isin(pre_keys, post_keys)
        npos = int((a.w.view(np.uint32) >> 31 == 0).sum())
        nneg = a.nnz - npos
        assert (~surv).sum() == math.floor(0.3 * npos) + math.floor(0.3 * nneg) == out[k]
        # survivors keep w and v bit-exactly
        loc = np.searchsorted(post_keys, pre_keys[surv])
        assert np.array_equal(b.w[loc].view(np.uint32), a.w[surv].view(np.uint32))
        assert np.array_equal(b.v[loc].view(np.uint32), a.v[surv].view(np.uint32))
        # regrown positions are outside the pre-call support and start with v = 0
        new = ~np.isin(post_keys, pre_keys)
        assert new.sum() == out[k]
        assert np.all(b.v[new] == 0)


def test_evolve_equals_bruteforce_stream_scan():
    """Regrowth = first R distinct valid candidates of the REGROW stream (plain Python loop)."""
    st = _state(sizes=(8, 8, 8, 3), eps=2.0, seed=21)
    st.alive[1][3] = 0                                      # a dead neuron excluded from regrowth
    Ly = st.layers[1]
    keep = ~((Ly.rows() == 3))
    st.layers[1] = T._rebuild(Ly, keep)
    Ly = st.layers[0]
    st.layers[0] = T._rebuild(Ly, Ly.col != 3)
    pre = st.copy()
    e = 4
    T.evolve(st, 0.3, e)
    for k in range(2):
        a = pre.layers[k]
        flags, kp, kn = T.select_removals(a.w, 0.3)
        R = kp + kn
        pre_set = set(zip(a.rows().tolist(), a.col.tolist()))
        al_in, al_out = pre.alive[k], pre.alive[k + 1]
        acc, seen, m = [], set(), 0
        while len(acc) < R:
            x = philox.stream(pre.seed, philox.PURPOSE_REGROW, 0, a.l, e, np.array([m], np.uint64))
            i = (int(x[0][0]) * a.n_in) >> 32
            j = (int(x[1][0]) * a.n_out) >> 32
            if (i, j) not in pre_set and al_in[i] and al_out[j] and (i, j) not in seen:
                seen.add((i, j))
                acc.append((i, j))
            m += 1
        survivors = {p for p, f in zip(zip(a.rows().tolist(), a.col.tolist()), flags) if not f}
        b = st.layers[k]
        assert set(zip(b.rows().tolist(), b.col.tolist())) == survivors | set(acc)
        assert all(al_out[j] for j in b.col.tolist())


def test_evolve_skip_rule_on_saturated_layer():
    # 3x3 layer with 8 of 9 positions filled: R = floor(.3*#pos)+floor(.3*#neg) > A = 1
    st = M.create((3, 3, 2), 1.0, "all_relu", 0.5, 0.0, "he_uniform", 1)
    Ly = st.layers[0]
    keys = np.arange(8)
    w = np.array([1, 2, 3, 4, -1, -2, -3, -4], np.float32)
    st.layers[0] = M.Layer(2, 3, 3, np.array([0, 3, 6, 8]), (keys % 3).astype(np.int32), w,
                           np.zeros(8, np.float32), False)
    before = st.layers[0].copy()
    out = T.evolve(st, 0.3, 0)
    assert out[0] == -1
    assert np.array_equal(st.layers[0].w, before.w) and np.array_equal(st.layers[0].col, before.col)


def test_evolve_is_deterministic_and_index_dependent():
    a, b = _state(), _state()
    T.evolve(a, 0.3, 7)
    T.evolve(b, 0.3, 7)
    for x, y in zip(a.layers, b.layers):
        assert np.array_equal(x.keys(), y.keys()) and np.array_equal(x.w, y.w)
    c = _state()
    T.evolve(c, 0.3, 8)
    assert not all(np.array_equal(x.keys(), y.keys()) for x, y in zip(a.layers, c.layers))


def test_evolve_rejects_bad_zeta():
    with pytest.raises(ValueError):
        T.evolve(_state(), 1.0, 0)
    with pytest.raises(ValueError):
        T.evolve(_state(), 0.0, 0)


# ----------------------------------------------------------------------------- importance
def test_spec_importance_examples():
    # incoming {0.5, -0.3, 0.2} -> I = 1.0 ; isolated neuron -> 0
    st = M.create((3, 2, 2), 1.0, "all_relu", 0.5, 0.0, "he_uniform", 1)
    st.layers[0] = M.Layer(2, 3, 2, np.array([0, 1, 2, 3]), np.array([0, 0, 0], np.int32),
                           np.array([0.5, -0.3, 0.2], np.float32), np.zeros(3, np.float32))
    I = T.importance(st, 2)
    assert I[0] == pytest.approx(1.0, abs=1e-7) and I[1] == 0.0


def test_importance_equals_sequential_loop_and_exact_sum():
    st = _state(sizes=(40, 30, 20, 5), eps=4.0)
    for l in (2, 3):
        I = T.importance(st, l)
        Ly = st.layer(l)
        D = Ly.dense(np.float64)
        for j in range(Ly.n_out):
            acc = 0.0
            for i in range(Ly.n_in):                      # sequential, ascending i (brute force)
                if D[i, j] != 0:
                    acc = acc + abs(float(np.float32(D[i, j])))
            assert I[j] == acc
            exact = math.fsum(abs(float(v)) for v in D[:, j] if v != 0)
            assert abs(I[j] - exact) <= 40 * 2**-52 * exact + 1e-300
    # invariant to sign flips
    st2 = st.copy()
    st2.layers[0].w = -st2.layers[0].w
    assert np.array_equal(T.importance(st2, 2), T.importance(st, 2))


# ----------------------------------------------------------------------------- percentile / prune
def test_percentile_examples():
    v = np.array([1.0, 2.0, 3.0, 4.0, 100.0])
    t = T.percentile_threshold(v, 25.0)
    assert 1.0 < t <= 2.0 and t == 2.0            # h = 1.0 -> exactly I[1]
    t2 = T.percentile_threshold(v, 10.0)
    assert 1.0 < t2 < 2.0
    rng = np.random.default_rng(3)
    for _ in range(200):
        x = np.sort(rng.standard_normal(int(rng.integers(1, 50))))
        rho = float(rng.uniform(0, 99.9))
        t = T.percentile_threshold(x, rho)
        ref = float(np.percentile(x, rho, method="linear"))
        # numpy rounds h = (n-1)(rho/100) differently (one ulp of h times |I[hi]-I[lo]|),
        # so agreement is to a few ulps of the operands' scale, not bit for bit
        assert abs(t - ref) <= 64 * np.spacing(max(abs(x[0]), abs(x[-1]), 1e-300))


def test_prune_spec_examples():
    # importances {1,2,3,4,100}, rho = 25 -> exactly the I = 1 neuron removed
    st = M.create((5, 5, 2), 1.0, "all_relu", 0.5, 0.0, "he_uniform", 1)
    vals = [1.0, 2.0, 3.0, 4.0, 100.0]
    st.layers[0] = M.Layer(2, 5, 5, np.arange(6), np.arange(5, dtype=np.int32),
                           np.array(vals, np.float32), np.zeros(5, np.float32))
    st.layers[1] = M.Layer(3, 5, 2, np.arange(0, 11, 2), np.tile(np.arange(2, dtype=np.int32), 5),
                           np.ones(10, np.float32), np.zeros(10, np.float32), True)
    pruned, removed = T.prune(st, 25.0)
    assert pruned[1] == 1 and st.alive[1].tolist() == [0, 1, 1, 1, 1]
    assert removed[1] == 1 and removed[2] == 2          # incoming column + outgoing row
    assert 0 not in st.layers[0].col.tolist() and 0 not in st.layers[1].rows().tolist()
    # rho = 0 -> nothing removed
    st2 = _state()
    n0 = sum(Ly.nnz for Ly in st2.layers)
    pruned, removed = T.prune(st2, 0.0)
    assert sum(removed) == 0 and sum(Ly.nnz for Ly in st2.layers) == n0


def test_prune_invariants_and_skip():
    st = _state(sizes=(30, 25, 25, 4), eps=3.0)
    n0 = sum(Ly.nnz for Ly in st.layers)
    pruned, removed = T.prune(st, 20.0)
    n1 = sum(Ly.nnz for Ly in st.layers)
    assert n1 == n0 - sum(removed) and n1 < n0          # monotone
    for h in (2, 3):
        dead = np.flatnonzero(st.alive[h - 1] == 0)
        assert len(dead) == pruned[h - 1]
        assert not np.isin(st.layer(h).col, dead).any()
        assert not np.isin(st.layer(h + 1).rows(), dead).any()
    # a layer whose neurons all share one importance: I < t never holds -> nothing pruned;
    # a layer where pruning would kill all alive neurons is skipped
    st3 = M.create((2, 2, 2), 1.0, "all_relu", 0.5, 0.0, "he_uniform", 1)
    st3.layers[0] = M.Layer(2, 2, 2, np.array([0, 1, 2]), np.array([0, 1], np.int32),
                            np.array([1.0, 1.0], np.float32), np.zeros(2, np.float32))
    pruned, _ = T.prune(st3, 50.0)
    assert pruned[1] == 0 and st3.alive[1].all()


def test_prune_uses_snapshot_of_all_layers():
    """Decisions of layer h+1 use importances computed before layer h's outgoing cleanup."""
    st = _state(sizes=(30, 25, 25, 4), eps=3.0, seed=9)
    I = {h: T.importance(st, h) for h in (2, 3)}
    pre = st.copy()
    T.prune(st, 20.0)
    for h in (2, 3):
        ids = np.flatnonzero(pre.alive[h - 1])
        t = T.percentile_threshold(np.sort(I[h][ids]), 20.0)
        assert set(np.flatnonzero(st.alive[h - 1] == 0)) == set(ids[I[h][ids] < t])


def test_candidate_stream_bound_fails_like_the_cuda_path(monkeypatch):
    """R33: the candidate stream is searched over at most MAX_CANDIDATES draws (2^31 - 1 on both
    sides, the CUDA path's 32-bit candidate index); with fewer distinct valid positions in that
    prefix than needed, ER init and regrowth raise instead of drawing on (the library returns
    SMLP_E_ARG "could not find enough distinct candidates").  Exercised with a small bound."""
    from oracle import model as M
    from oracle import topology as T
    monkeypatch.setattr(M, "MAX_CANDIDATES", 50)
    with pytest.raises(ValueError, match="distinct candidates"):
        M.er_layer(30, 30, 3.0, "he_uniform", 1, 2)            # M = 180 distinct needed in 50 draws
    monkeypatch.setattr(M, "MAX_CANDIDATES", (1 << 31) - 1)
    st = M.create((40, 40, 3), 4.0, "all_relu", 0.5, 0.0, "he_uniform", 2)
    monkeypatch.setattr(T, "MAX_CANDIDATES", 10)
    with pytest.raises(ValueError, match="distinct candidates"):
        T.evolve(st, 0.3, 0)
