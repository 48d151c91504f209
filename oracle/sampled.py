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
All-ReLU kink (|z| <= mag 2^-20 with mag = sum |a w| + |b| > 0; DESIGN.md kink guard R30): there
f' (1 or the negative slope) may legitimately differ between an fp32 kernel and the fp64 oracle,
so such samples are excluded by the caller, not compared.
"""
from __future__ import annotations

from typing import Dict, Iterable

import numpy as np
import scipy.sparse as sp

from .model import F32, F64, State, Trace, activation_grad, loss_grad

KINK_REL = 2.0 ** -20


def _rows_csr(Ly, rows: np.ndarray, wabs: bool = False):
    """W^(l)[rows, :] as a float64 CSR matrix [len(rows) x n_out] (library sparse container)."""
    W = sp.csr_matrix((np.abs(Ly.w).astype(F64) if wabs else Ly.w.astype(F64), Ly.col.astype(np.int64),
                       Ly.row_ptr.astype(np.int64)), shape=(Ly.n_in, Ly.n_out))
    return W[rows, :]


def _cols_csc(Ly, cols: np.ndarray, wabs: bool = False):
    """W^(l)[:, cols] as a float64 CSC matrix [n_in x len(cols)]."""
    W = sp.csr_matrix((np.abs(Ly.w).astype(F64) if wabs else Ly.w.astype(F64), Ly.col.astype(np.int64),
                       Ly.row_ptr.astype(np.int64)), shape=(Ly.n_in, Ly.n_out)).tocsc()
    return W[:, cols]


def kink_columns(st: State, tr: Trace, l: int, cols: np.ndarray) -> np.ndarray:
    """bool [B x len(cols)]: z_l[b, j] within fp32 summation error of the kink (hidden layer l)."""
    Ly = st.layer(l)
    Wc = _cols_csc(Ly, cols, wabs=True)
    mag = np.asarray((Wc.T @ np.abs(tr.a[l - 2]).astype(F64).T).T) + np.abs(st.b[l - 2][cols].astype(F64))
    z = tr.z[l - 1][:, cols]
    return (np.abs(z) <= mag * KINK_REL) & (mag > 0)


def delta_columns(st: State, tr: Trace, y, need: Dict[int, Iterable[int]]):
    """delta_l[:, j] for the requested neurons j of each layer l (2..L).

    Returns (deltas, tainted): dicts l -> {j: float32 [B]} and l -> {j: bool} (True when the
    column depends, through f', on a kink-ambiguous pre-activation)."""
    L = st.L
    sets = {l: set(int(j) for j in need.get(l, ())) for l in range(2, L + 1)}
    for l in range(2, L):                       # the cone: delta_l[:, j] needs delta_{l+1}[:, out(j)]
        Ly = st.layer(l + 1)
        for j in sets[l]:
            sets[l + 1].update(int(k) for k in Ly.col[Ly.row_ptr[j]:Ly.row_ptr[j + 1]])
    _, dz = loss_grad(tr.p64, y)
    deltas: Dict[int, Dict[int, np.ndarray]] = {L: {j: dz[:, j].astype(F32) for j in sets[L]}}
    tainted: Dict[int, Dict[int, bool]] = {L: {j: False for j in sets[L]}}
    scale = 1.0 / (1.0 - st.dropout) if st.dropout > 0 else 1.0
    for l in range(L - 1, 1, -1):
        J = np.array(sorted(sets[l]), dtype=np.int64)
        deltas[l], tainted[l] = {}, {}
        if len(J) == 0:
            continue
        Ly = st.layer(l + 1)                     # W^(l+1): rows are the neurons of layer l
        K = np.array(sorted(deltas[l + 1].keys()), dtype=np.int64)
        Dn = np.zeros((tr.B, Ly.n_out), dtype=F64)
        Dn[:, K] = np.stack([deltas[l + 1][k] for k in K], axis=1).astype(F64)
        Tn = np.zeros(Ly.n_out, dtype=bool)
        Tn[K] = [tainted[l + 1][k] for k in K]
        Wr = _rows_csr(Ly, J)
        back = np.asarray((Wr @ Dn.T).T)         # [B x |J|] = delta_{l+1} W^(l+1)T on the cone
        d = back * activation_grad(tr.z[l - 1][:, J], l, st.alpha, st.activation)
        if tr.keep[l - 1] is not None:
            d = d * tr.keep[l - 1][:, J] * scale
        d = d.astype(F32)
        amb = kink_columns(st, tr, l, J).any(axis=0)
        for t, j in enumerate(J):
            row = Ly.col[Ly.row_ptr[j]:Ly.row_ptr[j + 1]]
            deltas[l][int(j)] = d[:, t]
            tainted[l][int(j)] = bool(amb[t] or Tn[row].any())
    return deltas, tainted


def grad_entries(st: State, tr: Trace, deltas, l: int, entries: np.ndarray) -> np.ndarray:
    """g of the canonical entries `entries` of W^(l): sum_b a_{l-1}[b, i] delta_l[b, j] (fp64 -> f32)."""
    Ly = st.layer(l)
    rows = Ly.rows()[entries]
    cols = Ly.col[entries].astype(np.int64)
    a = tr.a[l - 2][:, rows].astype(F64)
    d = np.stack([deltas[l][int(j)] for j in cols], axis=1).astype(F64)
    return (a * d).sum(axis=0).astype(F32)


def bias_grad_columns(deltas, l: int, cols: np.ndarray) -> np.ndarray:
    """gb_l[j] = sum_b delta_l[b, j] for the requested neurons (fp64 -> f32)."""
    return np.array([deltas[l][int(j)].astype(F64).sum() for j in cols], dtype=F64).astype(F32)
