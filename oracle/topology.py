"""SET topology evolution, neuron importance and Importance Pruning (ORACLE — test
infrastructure only; see oracle/__init__.py).

Follows Alg. 2 step by step in the paper's order, with the readings
of DESIGN.md where the paper is silent.
"""
from __future__ import annotations

import math
from typing import List, Tuple

import numpy as np

from . import philox
from .model import F32, F64, Layer, State, candidate_ij, init_values


def _rebuild(Ly: Layer, keep: np.ndarray, add_pos: np.ndarray = None,
             add_w: np.ndarray = None) -> Layer:
    """New support = (old support restricted to ``keep``) U additions, sorted by (i, j).
    Survivors keep w and v bit-exactly; additions get v = 0."""
    keys = Ly.keys()[keep]
    w = Ly.w[keep]
    v = Ly.v[keep]
    if add_pos is not None and len(add_pos):
        keys = np.concatenate([keys, add_pos.astype(np.int64)])
        w = np.concatenate([w, add_w.astype(F32)])
        v = np.concatenate([v, np.zeros(len(add_pos), F32)])
    order = np.argsort(keys, kind="stable")
    keys, w, v = keys[order], w[order], v[order]
    rows = keys // Ly.n_out
    row_ptr = np.zeros(Ly.n_in + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=Ly.n_in), out=row_ptr[1:])
    return Layer(Ly.l, Ly.n_in, Ly.n_out, row_ptr, (keys % Ly.n_out).astype(np.int32),
                 w, v, Ly.dense_capped)


def select_removals(w: np.ndarray, zeta: float) -> Tuple[np.ndarray, int, int]:
    """Alg. 2 lines "Remove a fraction zeta of the smallest positive weights" and "... of the
    largest negative weights" (DESIGN readings 5-7):
      P = entries with sign bit 0, N = entries with sign bit 1;
      k+ = floor(zeta |P|), k- = floor(zeta |N|);
      remove the k+ of P and the k- of N with the smallest key (|w| bits, canonical index),
      i.e. the positives closest to zero and the negatives closest to zero.
    Returns (removal flags, k+, k-)."""
    bits = w.view(np.uint32)
    neg = (bits >> np.uint32(31)).astype(bool)
    absb = bits & np.uint32(0x7FFFFFFF)
    idx = np.arange(len(w), dtype=np.int64)
    flags = np.zeros(len(w), dtype=bool)
    ks = []
    for cls in (~neg, neg):
        members = idx[cls]
        k = int(math.floor(zeta * len(members)))
        order = np.lexsort((members, absb[members]))      # by |w| bits, then canonical index
        flags[members[order[:k]]] = True
        ks.append(k)
    return flags, ks[0], ks[1]


# The candidate streams (ER init, regrowth) are searched over at most 2^31 - 1 draws m (DESIGN.md
# R33, the CUDA path's 32-bit candidate index): fewer than R distinct valid positions in that
# prefix is an error on both sides.
MAX_CANDIDATES = (1 << 31) - 1


def regrow_candidates(st: State, Ly: Layer, e: int, R: int, pre_keys: np.ndarray):
    """Alg. 2 "Add randomly new weights in the equivalent amount" (DESIGN reading 8):
    the first R distinct candidates of the REGROW stream (c3 = e) that are outside the
    pre-call support and connect two alive neurons.  Returns (positions, m indices)."""
    alive_in = st.alive[Ly.l - 2].astype(bool)
    alive_out = st.alive[Ly.l - 1].astype(bool)
    n_pos = Ly.n_in * Ly.n_out
    free = max(1, int(alive_in.sum()) * int(alive_out.sum()) - len(pre_keys))
    frac = free / n_pos
    C = int(R / frac * 1.25) + 1024
    while True:
        C = min(C, MAX_CANDIDATES)
        m = np.arange(C, dtype=np.uint64)
        x0, x1, x2, x3 = philox.stream(st.seed, philox.PURPOSE_REGROW, 0, Ly.l, e, m)
        i, j = candidate_ij(x0, x1, Ly.n_in, Ly.n_out)
        pos = i * Ly.n_out + j
        loc = np.searchsorted(pre_keys, pos)
        in_pre = (loc < len(pre_keys)) & (pre_keys[np.minimum(loc, len(pre_keys) - 1)] == pos) \
            if len(pre_keys) else np.zeros(len(pos), bool)
        valid = alive_in[i] & alive_out[j] & ~in_pre
        mv = np.flatnonzero(valid)
        _, first = np.unique(pos[mv], return_index=True)
        if len(first) >= R:
            acc = mv[np.sort(first)[:R]]
            return pos[acc], acc, x2[acc], x3[acc]
        if C >= MAX_CANDIDATES:
            raise ValueError("could not find enough distinct candidates (layer too saturated)")
        C *= 2


def evolve_layer(st: State, Ly: Layer, zeta: float, e: int):
    """One layer of the weight pruning-regrowing cycle (Alg. 2).
    Returns (new layer, removed count, skipped flag)."""
    if Ly.dense_capped:
        return Ly, 0, True
    flags, kp, kn = select_removals(Ly.w, zeta)
    R = kp + kn
    alive_in = st.alive[Ly.l - 2].astype(bool)
    alive_out = st.alive[Ly.l - 1].astype(bool)
    rows = Ly.rows()
    occupied = int(np.count_nonzero(alive_in[rows] & alive_out[Ly.col]))
    A = int(alive_in.sum()) * int(alive_out.sum()) - occupied
    if R == 0:
        return Ly, 0, False
    if A < R:                                   # skip rule (DESIGN reading 9)
        return Ly, 0, True
    pre_keys = Ly.keys()
    add_pos, acc_m, x2, x3 = regrow_candidates(st, Ly, e, R, pre_keys)
    add_w = init_values(st.init, Ly.n_in, Ly.n_out, x2, x3)
    return _rebuild(Ly, ~flags, add_pos, add_w), R, False


def evolve(st: State, zeta: float, e: int) -> List[int]:
    """sparse_mlp_evolve_topology: SET prune/regrow on every weight layer; version += 1.
    Returns removed-per-weight-layer (index l-2; -1 marks a skipped layer)."""
    if not (0.0 < zeta < 1.0):
        raise ValueError("zeta must be in (0, 1)")
    out = []
    for idx, Ly in enumerate(st.layers):
        new, r, skipped = evolve_layer(st, Ly, zeta, e)
        st.layers[idx] = new
        out.append(-1 if skipped else r)
    st.version += 1
    return out


# --------------------------------------------------------------------------------------
# Importance (Eq. 4) and Importance Pruning (Alg. 2)
# --------------------------------------------------------------------------------------
def importance(st: State, l: int) -> np.ndarray:
    """I_j^(l) = sum_{i in Gamma_j} |w_ij^(l)| over the incoming connections of neuron j of
    layer l (Eq. 4).  Evaluated as a sequential float64 sum in ascending i (DESIGN reading:
    fixed order so the result is reproducible bit for bit); isolated neurons get 0."""
    Ly = st.layer(l)
    rows = Ly.rows()
    order = np.lexsort((rows, Ly.col))           # column j, then ascending i
    cols = Ly.col[order].astype(np.int64)
    absw = np.abs(Ly.w[order].astype(F64))
    counts = np.bincount(cols, minlength=Ly.n_out)
    starts = np.zeros(Ly.n_out, dtype=np.int64)
    np.cumsum(counts[:-1], out=starts[1:])
    acc = np.zeros(Ly.n_out, dtype=F64)
    for t in range(int(counts.max()) if len(counts) else 0):
        has = counts > t
        acc[has] = acc[has] + absw[starts[has] + t]          # one IEEE add per column per step
    return acc


def percentile_threshold(values_sorted: np.ndarray, rho: float) -> float:
    """Linear-interpolation percentile (Hyndman-Fan type 7) written out explicitly:
    h = (n-1) rho / 100, lo = floor(h), hi = min(lo+1, n-1), t = I[lo] + (h - lo)(I[hi] - I[lo]).
    Each operation is one IEEE double op (no fused multiply-add)."""
    n = len(values_sorted)
    h = (float(n - 1) * float(rho)) / 100.0
    lo = int(math.floor(h))
    hi = min(lo + 1, n - 1)
    a = float(values_sorted[lo])
    b = float(values_sorted[hi])
    return a + (h - float(lo)) * (b - a)


def prune(st: State, rho: float, outgoing: bool = True):
    """sparse_mlp_prune_neurons (Alg. 2; DESIGN readings 15-19).
    Over hidden layers h = 2..L-1: snapshot I for all of them; t = rho-th percentile over the
    alive neurons; kill alive j with I_j < t (strict) unless that kills every alive neuron
    (layer skipped); remove the incoming column j of W^(h) and (outgoing cleanup) row j of
    W^(h+1); version += 1.
    Returns (pruned_per_neuron_layer [L] (-1 = skipped), removed_conn_per_weight_layer [L])."""
    if not (0.0 <= rho < 100.0):
        raise ValueError("rho must be in [0, 100)")
    L = st.L
    I = {h: importance(st, h) for h in range(2, L)}
    decisions = {}
    pruned = [0] * L
    for h in range(2, L):
        ids = np.flatnonzero(st.alive[h - 1])
        if len(ids) == 0:
            continue
        Is = np.sort(I[h][ids])
        t = percentile_threshold(Is, rho)
        D = ids[I[h][ids] < t]
        if len(D) == len(ids):
            pruned[h - 1] = -1
            continue
        decisions[h] = D
        pruned[h - 1] = len(D)
    removed = [0] * L
    for h, D in decisions.items():
        dead = np.zeros(st.sizes[h - 1], dtype=bool)
        dead[D] = True
        Lin = st.layer(h)
        keep = ~dead[Lin.col]
        removed[h - 1] += int((~keep).sum())
        st.layers[h - 2] = _rebuild(Lin, keep)
        if outgoing:
            Lout = st.layer(h + 1)
            keep2 = ~dead[Lout.rows()]
            removed[h] += int((~keep2).sum())
            st.layers[h - 1] = _rebuild(Lout, keep2)
        st.alive[h - 1][D] = 0
    st.version += 1
    return pruned, removed
