"""Sampled backward at full size (ORACLE — test infrastructure only; see oracle/__init__.py).

At C5 size (52.3M connections, 1.5M hidden neurons) the oracle's full backward takes minutes, so
the full-size parity test checks a seeded SAMPLE of gradient entries instead.  This module
computes, for chosen neurons, exactly what `model.backward` computes for them (SURVEY.md §8(c)
O5; PAPER.md:47 — gradients "just from the existing parameters"):

    delta_L           = (p - onehot) / B                                   (O4, reading R12)
    delta_l[:, j]     = (sum_{k in out(j)} w_jk delta_{l+1}[:, k]) * f'_l(z_l[:, j]) * keep/(1-r)
    g_ij              = sum_b a_{l-1}[b, i] delta_l[b, j]      for (i, j) in the support of W^(l)
    gb_l[j]           = sum_b delta_l[b, j]

walking the "cone" of neurons each requested delta depends on (its out-neighbours, theirs, ...),
in float64 with one rounding to float32 per stored delta, like `model.backward`.

It also reports which samples depend on a pre-activation within fp32 summation error of the
All-ReLU kink (|z| <= mag 2^-20 with mag = sum |a w| + |b| > 0; reading R32, the kink guard): there
f' (1 or the negative slope) may legitimately differ between an fp32 kernel and the fp64 oracle,
so such samples are excluded by the caller, not compared.
"""
from __future__ import annotations

from typing import Dict, Iterable

import numpy as np

from .model import F32, F64, State, Trace, activation_grad, loss_grad

KINK_REL = 2.0 ** -20


_CHUNK_ELEMS = 1 << 24


def _segment_products(ptr: np.ndarray, order, J: np.ndarray, other: np.ndarray, src: np.ndarray,
                      w: np.ndarray) -> np.ndarray:
    """out[t, :] = sum over the entries e of segment J[t] of other[src[e], :] * w[e]  (float64
    [len(J) x B]).  Segment k holds the entries order[ptr[k]:ptr[k+1]] (order None = identity).
    Chunked over J; np.add.reduceat adds each segment's products."""
    B = other.shape[1]
    out = np.zeros((len(J), B), dtype=F64)
    lens_all = (ptr[J + 1] - ptr[J]).astype(np.int64)
    t0 = 0
    while t0 < len(J):
        acc, t1 = 0, t0
        while t1 < len(J) and (acc == 0 or (acc + lens_all[t1]) * B <= _CHUNK_ELEMS):
            acc += lens_all[t1]
            t1 += 1
        lens = lens_all[t0:t1]
        nz = lens > 0
        if acc > 0:
            starts = ptr[J[t0:t1]].astype(np.int64)
            seg_begin = np.cumsum(lens) - lens
            pos = np.repeat(starts - seg_begin, lens) + np.arange(acc)
            e = pos if order is None else order[pos]
            prod = other[src[e]] * w[e][:, None]
            out[t0:t1][nz] = np.add.reduceat(prod, seg_begin[nz], axis=0)
        t0 = t1
    return out


def _column_index(Ly):
    """Entries of W^(l) grouped by output neuron j (i ascending within a column): (order, cptr)."""
    order = np.argsort(Ly.col, kind="stable")
    cptr = np.searchsorted(Ly.col[order], np.arange(Ly.n_out + 1))
    return order, cptr


def kink_columns(st: State, tr: Trace, l: int, cols: np.ndarray) -> np.ndarray:
    """bool [B x len(cols)]: z_l[b, j] within fp32 summation error of the kink (hidden layer l):
    |z| <= 2^-20 mag, mag[b, j] = sum_i |a_{l-1}[b, i] w_ij| + |b_j| (R32)."""
    Ly = st.layer(l)
    order, cptr = _column_index(Ly)
    aT = np.ascontiguousarray(np.abs(tr.a[l - 2]).astype(F64).T)
    mag = _segment_products(cptr, order, np.asarray(cols, np.int64), aT, Ly.rows(), np.abs(Ly.w).astype(F64)).T
    mag = mag + np.abs(st.b[l - 2][cols].astype(F64))[None, :]
    z = tr.z[l - 1][:, cols]
    return (np.abs(z) <= mag * KINK_REL) & (mag > 0)


def delta_columns(st: State, tr: Trace, y, need: Dict[int, Iterable[int]]):
    """delta_l[:, j] for the requested neurons j of each layer l (2..L).

    Returns (deltas, tainted, dmags): dicts l -> {j: float32 [B]}, l -> {j: bool [B]} (tainted[l][j][b]
    is True when delta_l[b, j] depends, through f', on a kink-ambiguous pre-activation of batch row
    b: its own z_l[b, j] or a tainted delta_{l+1}[b, k] of an out-neighbour k) and l -> {j: float64
    [B]}, the running error magnitudes of `model.backward` (R24) for those columns."""
    L = st.L
    B = tr.B
    sets = {l: set(int(j) for j in need.get(l, ())) for l in range(2, L + 1)}
    for l in range(2, L):                       # the cone: delta_l[:, j] needs delta_{l+1}[:, out(j)]
        Ly = st.layer(l + 1)
        for j in sets[l]:
            sets[l + 1].update(int(k) for k in Ly.col[Ly.row_ptr[j]:Ly.row_ptr[j + 1]])
    _, dz = loss_grad(tr.p64, y)
    deltas: Dict[int, Dict[int, np.ndarray]] = {L: {j: dz[:, j].astype(F32) for j in sets[L]}}
    tainted: Dict[int, Dict[int, np.ndarray]] = {L: {j: np.zeros(B, bool) for j in sets[L]}}
    pm = tr.pmag / B
    dmags: Dict[int, Dict[int, np.ndarray]] = {L: {j: pm[:, j] for j in sets[L]}}
    scale = 1.0 / (1.0 - st.dropout) if st.dropout > 0 else 1.0
    for l in range(L - 1, 1, -1):
        J = np.array(sorted(sets[l]), dtype=np.int64)
        deltas[l], tainted[l], dmags[l] = {}, {}, {}
        if len(J) == 0:
            continue
        Ly = st.layer(l + 1)                     # W^(l+1): rows are the neurons of layer l
        K = np.array(sorted(deltas[l + 1].keys()), dtype=np.int64)
        Dn = np.zeros((B, Ly.n_out), dtype=F64)
        Dn[:, K] = np.stack([deltas[l + 1][k] for k in K], axis=1).astype(F64)
        Tn = np.zeros((B, Ly.n_out), dtype=bool)
        Tn[:, K] = np.stack([tainted[l + 1][k] for k in K], axis=1)
        Mn = np.zeros((B, Ly.n_out), dtype=F64)  # dmag_{l+1} on the cone
        Mn[:, K] = np.stack([dmags[l + 1][k] for k in K], axis=1)
        wa = np.abs(Ly.w).astype(F64)
        wm = wa + (0.0 if Ly.wmag is None else Ly.wmag)
        # [B x |J|] = delta_{l+1} W^(l+1)T on the cone, and its first-order magnitude
        # |delta| . (|W| + wmag)^T + dmag . |W|^T  (model.backward)
        back = _segment_products(Ly.row_ptr, None, J, np.ascontiguousarray(Dn.T), Ly.col, Ly.w.astype(F64)).T
        bmag = (_segment_products(Ly.row_ptr, None, J, np.ascontiguousarray(np.abs(Dn).T), Ly.col, wm).T
                + _segment_products(Ly.row_ptr, None, J, np.ascontiguousarray(Mn.T), Ly.col, wa).T)
        fp = activation_grad(tr.z[l - 1][:, J], l, st.alpha, st.activation)
        d = back * fp
        dm = bmag * np.abs(fp)
        if tr.keep[l - 1] is not None:
            d = d * tr.keep[l - 1][:, J] * scale
            dm = dm * tr.keep[l - 1][:, J] * scale
        d = d.astype(F32)
        amb = kink_columns(st, tr, l, J)        # [B x |J|]
        # taint of delta_l[b, j]: its own kink, or any out-neighbour's tainted delta_{l+1}[b, k]
        tn = _segment_products(Ly.row_ptr, None, J, np.ascontiguousarray(Tn.T.astype(F64)), Ly.col,
                               np.ones(Ly.nnz, F64)).T > 0
        taint = amb | tn
        for t, j in enumerate(J):
            deltas[l][int(j)] = d[:, t]
            dmags[l][int(j)] = dm[:, t]
            tainted[l][int(j)] = taint[:, t]
    return deltas, tainted, dmags


def grad_entries(st: State, tr: Trace, deltas, dmags, l: int, entries: np.ndarray):
    """g of the canonical entries `entries` of W^(l): sum_b a_{l-1}[b, i] delta_l[b, j] (fp64 -> f32),
    and its first-order running error magnitude sum_b (|a| + amag)|delta| + |a| dmag (R24)."""
    Ly = st.layer(l)
    rows = Ly.rows()[entries]
    cols = Ly.col[entries].astype(np.int64)
    a = tr.a[l - 2][:, rows].astype(F64)
    am = np.abs(a) + tr.amag[l - 2][:, rows]
    d = np.stack([deltas[l][int(j)] for j in cols], axis=1).astype(F64)
    dm = np.stack([dmags[l][int(j)] for j in cols], axis=1)
    return (a * d).sum(axis=0).astype(F32), (am * np.abs(d) + np.abs(a) * dm).sum(axis=0)


def bias_grad_columns(deltas, dmags, l: int, cols: np.ndarray):
    """gb_l[j] = sum_b delta_l[b, j] for the requested neurons (fp64 -> f32), and its magnitude."""
    gb = np.array([deltas[l][int(j)].astype(F64).sum() for j in cols], dtype=F64).astype(F32)
    gm = np.array([(np.abs(deltas[l][int(j)].astype(F64)) + dmags[l][int(j)]).sum() for j in cols], dtype=F64)
    return gb, gm
