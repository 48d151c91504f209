"""K-rank synchronous data parallelism and model averaging (ORACLE — test infrastructure only).

WASSP-SGD phase 1: every rank computes the gradient of
its own minibatch on the same snapshot (dropout streams include the rank), the K gradients
are summed (the allreduce), and every rank applies Eq. 1 with grad_scale = 1/K and the
learning rate of the "gradual warmup and linear scaling rule" (DESIGN
reading 20).  Eq. 2 model averaging for identical supports is the plain
mean of (w, b).  The paper's CPU parameter server itself is prior art (BASELINE.json
north_star), so it is not modelled here.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .model import F32, F64, Grads, State, backward, forward, step


def scaled_lr(base_lr: float, K: int, step_idx: int, warmup_steps: int) -> float:
    """eta_t = eta * (1 + (K - 1) * min(1, t / warmup)): linear scaling with gradual warmup."""
    if K <= 1:
        return base_lr
    frac = 1.0 if warmup_steps <= 0 else min(1.0, step_idx / float(warmup_steps))
    return base_lr * (1.0 + (K - 1) * frac)


def allreduce_sum(grads: Sequence[Grads]) -> Grads:
    """SUM over ranks of every gradient value (float64 sum, one rounding to float32).  Running
    error magnitude (R24): sum_k (|g_k| + gmag_k) -- an fp32 reduction in any order."""
    g = [np.sum([gr.g[i].astype(F64) for gr in grads], axis=0).astype(F32) for i in range(len(grads[0].g))]
    gb = [np.sum([gr.gb[i].astype(F64) for gr in grads], axis=0).astype(F32) for i in range(len(grads[0].gb))]

    def mag(vals, mags, i):
        return np.sum([np.abs(v[i]).astype(F64) + (0.0 if m is None else m[i]) for v, m in zip(vals, mags)], axis=0)

    gmag = [mag([gr.g for gr in grads], [gr.gmag for gr in grads], i) for i in range(len(g))]
    gbmag = [mag([gr.gb for gr in grads], [gr.gbmag for gr in grads], i) for i in range(len(gb))]
    return Grads(g, gb, float(np.mean([gr.loss for gr in grads])), [None] * len(grads[0].deltas), gmag, gbmag)


def dp_step(st: State, batches: Sequence[Tuple[np.ndarray, np.ndarray]], lr: float,
            momentum: float, weight_decay: float, step_idx: int) -> float:
    """One synchronous step of K = len(batches) replicas sharing ``st`` (identical topology).
    Returns the mean loss over ranks."""
    K = len(batches)
    grads = []
    for k, (x, y) in enumerate(batches):
        tr = forward(st, x, True, step_idx, rank=k)
        grads.append(backward(st, tr, y))
    total = allreduce_sum(grads)
    step(st, total, lr, momentum, weight_decay, grad_scale=1.0 / K)
    return total.loss


def average(states: List[State]) -> None:
    """Eq. 2: theta_f = (1/K) sum_i theta_i over (w, b) of replicas with identical supports
    (the union-and-re-sparsify form is SURVEY §8(f) item 1).  Momentum stays local.
    Modifies every state in place."""
    K = len(states)
    for s in states[1:]:
        for a, b in zip(states[0].layers, s.layers):
            if not (np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col)):
                raise ValueError("averaging requires identical supports")
    for idx in range(len(states[0].layers)):
        w = (np.sum([s.layers[idx].w.astype(F64) for s in states], axis=0) / K).astype(F32)
        b = (np.sum([s.b[idx].astype(F64) for s in states], axis=0) / K).astype(F32)
        # running error magnitudes (R24): the mean of (|value| + its magnitude)
        wm = np.sum([np.abs(s.layers[idx].w).astype(F64) + (0.0 if s.layers[idx].wmag is None else s.layers[idx].wmag)
                     for s in states], axis=0) / K
        bm = np.sum([np.abs(s.b[idx]).astype(F64) + (0.0 if s.bmag is None else s.bmag[idx]) for s in states], axis=0) / K
        for s in states:
            s.layers[idx].w = w.copy()
            s.layers[idx].wmag = wm.copy()
            s.b[idx] = b.copy()
            if s.bmag is None:
                s.bmag = [np.zeros(len(x), F64) for x in s.b]
                s.vbmag = [np.zeros(len(x), F64) for x in s.b]
            s.bmag[idx] = bm.copy()


def average_union(states: List[State], targets: Sequence[int]) -> List[int]:
    """WASAP phase-2 averaging (Alg. 1; Eq. 2; SPEC S:282-290;
    SURVEY.md §8(f) item 1) of K replicas whose topologies evolved independently, written out per
    layer exactly as the paper states it: the averaged support is the union of the K supports,
    each union entry's value is (sum over replicas of its value, absent = 0) / K, and then the
    connections closest to zero are pruned ("unimportant connections ... the largest negative
    weights and the smallest positive weights") down to targets[l-2] (the
    pre-phase-2 count).
    Arithmetic (DESIGN reading R31, shared with the CUDA path because it decides which entries
    survive): the sum is taken in float32 over the PRESENT values in rank order, then divided by
    K in float32; removal order is (|w| bit pattern, position) ascending.  Momentum of the
    averaged model is 0; biases are averaged (sum in rank order in float64, / K, rounded once).
    Every state is replaced by the averaged model.  Returns the kept count per layer."""
    K = len(states)
    L = states[0].L
    kept = []
    new_layers = []
    for idx in range(L - 1):
        lays = [s.layers[idx] for s in states]
        n_in, n_out = lays[0].n_in, lays[0].n_out
        vals = {}
        for Ly in lays:                                   # rank order
            pos = Ly.rows().astype(np.uint64) * np.uint64(n_out) + Ly.col.astype(np.uint64)
            for p, w in zip(pos.tolist(), Ly.w.tolist()):
                w32 = np.float32(w)
                vals[p] = w32 if p not in vals else np.float32(vals[p] + w32)
        upos = np.array(sorted(vals), dtype=np.uint64)
        uval = np.array([np.float32(vals[int(p)]) / np.float32(K) for p in upos], dtype=F32)
        U = len(upos)
        keep_n = min(U, int(targets[idx]))
        keys = (uval.view(np.uint32).astype(np.uint64) & np.uint64(0x7fffffff)) << np.uint64(32)
        keys |= np.arange(U, dtype=np.uint64)
        order = np.argsort(keys, kind="stable")
        keep = np.ones(U, bool)
        keep[order[:U - keep_n]] = False
        kp, kv = upos[keep], uval[keep]
        rows = (kp // np.uint64(n_out)).astype(np.int64)
        cols = (kp % np.uint64(n_out)).astype(np.int32)
        row_ptr = np.zeros(n_in + 1, np.int64)
        np.add.at(row_ptr, rows + 1, 1)
        new_layers.append((np.cumsum(row_ptr), cols, kv.astype(F32)))
        kept.append(keep_n)
    b_avg = [(np.sum([s.b[i].astype(F64) for s in states], axis=0) / K).astype(F32) for i in range(L - 1)]
    for s in states:
        for idx, (rp, cols, w) in enumerate(new_layers):
            Ly = s.layers[idx]
            Ly.row_ptr = rp.copy()
            Ly.col = cols.copy()
            Ly.w = w.copy()
            Ly.v = np.zeros_like(w)
            s.b[idx] = b_avg[idx].copy()
            s.vb[idx] = np.zeros_like(s.vb[idx])
        s.version += 1
    return kept


def retain_valid_updates(stale_keys: Sequence[np.ndarray], stale_g: Sequence[np.ndarray], st_now: State) -> List[np.ndarray]:
    """RetainValidUpdates of Alg. 1 (Fig. 4):
    a worker's gradient computed on the topology at time t (per layer: canonical positions
    i * n_out + j and values) restricted to the server's CURRENT topology: each current connection
    takes the stale gradient at its position if that position existed at t, else 0 -- the
    intersection of the two supports.  Returns per-layer gradients aligned to st_now's canonical
    order."""
    out = []
    for Ly, keys, g in zip(st_now.layers, stale_keys, stale_g):
        table = dict(zip(np.asarray(keys).tolist(), np.asarray(g, dtype=F32).tolist()))
        out.append(np.array([table.get(p, 0.0) for p in Ly.keys().tolist()], dtype=F32))
    return out
