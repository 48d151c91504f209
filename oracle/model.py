"""Sparse MLP state, ER initialisation, forward, loss, backward and update (ORACLE — test
infrastructure only; see oracle/__init__.py).

Notation follows the paper: neuron layers l = 1..L with the input at l = 1;
weight matrix W^(l) connects layer l-1 to layer l and has shape n_{l-1} x n_l, w_ij = 0
meaning "no connection".  W^(l) is stored as CSR by input row i with sorted,
unique columns (the paper orientation), aligned momentum v, dense biases b_l.

Every stored tensor is float32 ("32-bit float precision") computed in float64
and rounded once.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import philox

F32 = np.float32
F64 = np.float64


def _cp(x):
    return None if x is None else x.copy()


def _m(x, like):
    """An error magnitude, or zeros when it is exactly known (None)."""
    return np.zeros(np.shape(like), F64) if x is None else x


# --------------------------------------------------------------------------------------
# state
# --------------------------------------------------------------------------------------
@dataclass
class Layer:
    """Weight layer W^(l), CSR by input neuron i."""
    l: int
    n_in: int
    n_out: int
    row_ptr: np.ndarray      # int64 [n_in + 1]
    col: np.ndarray          # int32 [nnz], sorted unique within each row
    w: np.ndarray            # float32 [nnz]
    v: np.ndarray            # float32 [nnz] momentum (Eq. 1 history)
    dense_capped: bool = False
    # running fp32 error magnitudes of w and v (R24; None = exactly known, e.g. after
    # init or an import into the GPU model): an fp32 implementation that took the same steps may
    # differ by up to KAPPA_U * mag (compare.py)
    wmag: Optional[np.ndarray] = None
    vmag: Optional[np.ndarray] = None

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    def rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_in, dtype=np.int64), np.diff(self.row_ptr))

    def keys(self) -> np.ndarray:
        """Linear positions i * n_out + j (ascending in canonical order)."""
        return self.rows() * self.n_out + self.col.astype(np.int64)

    def dense(self, dtype=F64) -> np.ndarray:
        D = np.zeros((self.n_in, self.n_out), dtype=dtype)
        D[self.rows(), self.col] = self.w
        return D

    def copy(self) -> "Layer":
        return Layer(self.l, self.n_in, self.n_out, self.row_ptr.copy(), self.col.copy(),
                     self.w.copy(), self.v.copy(), self.dense_capped, _cp(self.wmag), _cp(self.vmag))

    def reset_error(self) -> None:
        self.wmag = None
        self.vmag = None


@dataclass
class State:
    sizes: List[int]
    epsilon: float
    activation: str          # "all_relu" | "relu"
    alpha: float
    dropout: float
    init: str                # "normal" | "xavier" | "he_uniform"
    seed: int
    rank: int
    layers: List[Layer]      # layers[l-2] = W^(l), l = 2..L
    b: List[np.ndarray]      # b[l-2] = bias of neuron layer l
    vb: List[np.ndarray]     # bias momentum
    alive: List[np.ndarray]  # alive[l-1] = uint8 liveness of neuron layer l (l = 1..L)
    version: int = 0
    bmag: Optional[List[np.ndarray]] = None    # running error magnitudes of b and vb (R24)
    vbmag: Optional[List[np.ndarray]] = None

    @property
    def L(self) -> int:
        return len(self.sizes)

    def layer(self, l: int) -> Layer:
        return self.layers[l - 2]

    def copy(self) -> "State":
        return State(list(self.sizes), self.epsilon, self.activation, self.alpha, self.dropout,
                     self.init, self.seed, self.rank, [x.copy() for x in self.layers],
                     [x.copy() for x in self.b], [x.copy() for x in self.vb],
                     [x.copy() for x in self.alive], self.version,
                     None if self.bmag is None else [x.copy() for x in self.bmag],
                     None if self.vbmag is None else [x.copy() for x in self.vbmag])

    def reset_error(self) -> None:
        """The state is now known exactly on both sides (e.g. it was just imported into the GPU
        model): the running error bound restarts from zero."""
        for Ly in self.layers:
            Ly.reset_error()
        self.bmag = None
        self.vbmag = None


# --------------------------------------------------------------------------------------
# Erdos-Renyi initialisation (Alg. 2)
# --------------------------------------------------------------------------------------
MAX_CANDIDATES = (1 << 31) - 1      # DESIGN.md R33 (same bound as oracle/topology.py)


def er_count(n_in: int, n_out: int, epsilon: float) -> int:
    """M = min(n_in * n_out, floor(eps * (n_in + n_out))): the ER density
    eps(n_in+n_out)/(n_in n_out) of BASELINE.json north_star, capped at 1 (DESIGN reading 1)."""
    return int(min(n_in * n_out, math.floor(epsilon * (n_in + n_out))))


def candidate_ij(x0: np.ndarray, x1: np.ndarray, n_in: int, n_out: int):
    """Map two uniform 32-bit words to a position: i = floor(x0 * n_in / 2^32), j likewise."""
    i = (x0.astype(np.uint64) * np.uint64(n_in)) >> np.uint64(32)
    j = (x1.astype(np.uint64) * np.uint64(n_out)) >> np.uint64(32)
    return i.astype(np.int64), j.astype(np.int64)


def init_values(init: str, n_in: int, n_out: int, x2: np.ndarray, x3: np.ndarray) -> np.ndarray:
    """Initial / regrown weight values (Table 5 scheme names; DESIGN reading 3).

    he_uniform: U(-lim, lim), lim = sqrt(6 / n_in); xavier: lim = sqrt(6 / (n_in + n_out)).
      u = (x2 >> 8) * 2^-24 in [0, 1); value = fp32((2u - 1) * lim)  (all steps exact but the last).
    normal: N(0, 2 / n_in) by Box-Muller on (x2, x3), in float64, rounded to fp32."""
    if init in ("he_uniform", "xavier"):
        lim64 = math.sqrt(6.0 / n_in) if init == "he_uniform" else math.sqrt(6.0 / (n_in + n_out))
        lim = F32(lim64)
        u = (x2 >> np.uint32(8)).astype(F32) * F32(2.0 ** -24)
        t = u * F32(2.0) - F32(1.0)
        return (t * lim).astype(F32)
    if init == "normal":
        u1 = ((x2 >> np.uint32(8)).astype(F64) + 1.0) * (2.0 ** -24)
        u2 = (x3 >> np.uint32(8)).astype(F64) * (2.0 ** -24)
        r = np.sqrt(-2.0 * np.log(u1))
        c = np.cos((2.0 * math.pi) * u2)
        std = math.sqrt(2.0 / n_in)
        return ((r * c) * std).astype(F32)
    raise ValueError(f"unknown init scheme {init!r}")


def er_layer(n_in: int, n_out: int, epsilon: float, init: str, seed: int, l: int) -> Layer:
    """G(n, M) Erdos-Renyi layer: the first M distinct positions of the INIT candidate
    stream (DESIGN reading 2), values from the accepting candidate's words (x2, x3).
    A dense-capped layer (M = n_in n_out) takes every position; its values come from
    the INIT_DENSE stream at index = linear position."""
    total = n_in * n_out
    M = er_count(n_in, n_out, epsilon)
    if M == total:
        pos = np.arange(total, dtype=np.int64)
        x0, x1, x2, x3 = philox.stream(seed, philox.PURPOSE_INIT_DENSE, 0, l, 0, pos.astype(np.uint64))
        w = init_values(init, n_in, n_out, x2, x3)
        row_ptr = np.arange(n_in + 1, dtype=np.int64) * n_out
        col = np.tile(np.arange(n_out, dtype=np.int32), n_in)
        return Layer(l, n_in, n_out, row_ptr, col, w, np.zeros(total, F32), True)
    C = M + M // 8 + 1024
    while True:
        C = min(C, MAX_CANDIDATES)
        m = np.arange(C, dtype=np.uint64)
        x0, x1, x2, x3 = philox.stream(seed, philox.PURPOSE_INIT, 0, l, 0, m)
        i, j = candidate_ij(x0, x1, n_in, n_out)
        pos = i * n_out + j
        _, first = np.unique(pos, return_index=True)      # first occurrence of every distinct pos
        if len(first) >= M:
            break
        if C >= MAX_CANDIDATES:                           # R33: the stream prefix searched is bounded
            raise ValueError("could not find enough distinct candidates (layer too saturated)")
        C *= 2
    acc = np.sort(first)[:M]                                # the first M distinct, in stream order
    w_acc = init_values(init, n_in, n_out, x2[acc], x3[acc])
    p_acc = pos[acc]
    order = np.argsort(p_acc, kind="stable")
    p_sorted = p_acc[order]
    rows = p_sorted // n_out
    col = (p_sorted % n_out).astype(np.int32)
    row_ptr = np.zeros(n_in + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_in), out=row_ptr[1:])
    return Layer(l, n_in, n_out, row_ptr, col, w_acc[order], np.zeros(M, F32), False)


def create(sizes, epsilon, activation="all_relu", alpha=0.5, dropout=0.0, init="he_uniform",
           seed=0, rank=0) -> State:
    """sparse_mlp_create: ER init of every weight layer, zero momentum and biases, version 0."""
    sizes = [int(s) for s in sizes]
    if len(sizes) < 3 or min(sizes) < 1 or not epsilon > 0 or alpha < 0 or not (0 <= dropout < 1):
        raise ValueError("invalid configuration")
    layers, b, vb = [], [], []
    for l in range(2, len(sizes) + 1):
        layers.append(er_layer(sizes[l - 2], sizes[l - 1], epsilon, init, seed, l))
        b.append(np.zeros(sizes[l - 1], F32))
        vb.append(np.zeros(sizes[l - 1], F32))
    alive = [np.ones(n, np.uint8) for n in sizes]
    return State(sizes, float(epsilon), activation, float(alpha), float(dropout), init,
                 int(seed), int(rank), layers, b, vb, alive, 0)


# --------------------------------------------------------------------------------------
# sparse products, plain NumPy in float64 (W zero-filled off the support, so a
# product over W is a sum over the connections (i, j) in S_l only).  Chunked over connections so
# the C5 layers fit in memory; np.add.reduceat (a library segmented sum) adds each output's
# contiguous run of connection products.  No SciPy.
# --------------------------------------------------------------------------------------
_CHUNK_ELEMS = 1 << 24
# Worker threads for the chunk loops (NumPy releases the GIL in its gathers / ufuncs / reduceat);
# chunks write disjoint output rows, so the result does not depend on the thread count.  The
# bench's cpu_baseline sets 1.
THREADS = os.cpu_count() or 1
_POOL = None


def _pool():
    global _POOL
    if _POOL is None or _POOL._max_workers != THREADS:
        _POOL = ThreadPoolExecutor(max_workers=THREADS)
    return _POOL


def _segment_sums(rows_of_terms: np.ndarray, seg_key: np.ndarray, out: np.ndarray) -> None:
    """out[k, :] = sum of rows_of_terms[e, :] over the entries e with seg_key[e] == k, where
    seg_key is non-decreasing (entries grouped by output).  Outputs with no entry are untouched."""
    if len(seg_key) == 0:
        return
    starts = np.flatnonzero(np.r_[True, seg_key[1:] != seg_key[:-1]])
    out[seg_key[starts]] += np.add.reduceat(rows_of_terms, starts, axis=0)


def _chunks(n: int, B: int, key: Optional[np.ndarray] = None):
    """[s0, s1) entry ranges of about _CHUNK_ELEMS / B entries; with a non-decreasing key, every
    boundary falls between two different keys (no output row is split across chunks)."""
    step = max(1, _CHUNK_ELEMS // max(B, 1))
    s0 = 0
    while s0 < n:
        s1 = min(n, s0 + step)
        if key is not None and s1 < n:
            s1 = int(np.searchsorted(key, key[s1 - 1], side="right"))
        yield s0, s1
        s0 = s1


def _run_chunks(fn, chunks) -> None:
    """fn(s0, s1) over the chunks, on THREADS workers (each chunk owns its output rows)."""
    chunks = list(chunks)
    if THREADS <= 1 or len(chunks) <= 1:
        for c in chunks:
            fn(*c)
        return
    for f in [_pool().submit(fn, *c) for c in chunks]:
        f.result()


def column_order(Ly: Layer) -> np.ndarray:
    """Permutation of the canonical entries sorting them by output neuron j (stable: i ascending
    within a column)."""
    return np.argsort(Ly.col, kind="stable")


def _spmm_fwd_stack(aT: np.ndarray, ws, Ly: Layer, dtype) -> np.ndarray:
    """zT [n_out x sum of column blocks]: aT [n_in x K B] holds K stacked column blocks of width B;
    block k is multiplied by the weights ws[k] (values on the support of W^(l), canonical order)."""
    K = len(ws)
    Bk = aT.shape[1] // K
    order = column_order(Ly)
    rows, cols = Ly.rows()[order], Ly.col[order].astype(np.int64)
    wo = [np.asarray(w, dtype)[order] for w in ws]
    zT = np.zeros((Ly.n_out, aT.shape[1]), dtype=dtype)

    def part(s0, s1):
        t = aT[rows[s0:s1]].astype(dtype, copy=False)
        for k in range(K):
            t[:, k * Bk:(k + 1) * Bk] *= wo[k][s0:s1, None]
        _segment_sums(t, cols[s0:s1], zT)
    _run_chunks(part, _chunks(Ly.nnz, aT.shape[1], cols))
    return zT


def spmm_fwd(a: np.ndarray, Ly: Layer, wabs: bool = False, w: Optional[np.ndarray] = None) -> np.ndarray:
    """z = a . W^(l)  ([B x n_in] x [n_in x n_out]) in float64:
    z[b, j] = sum over the connections (i, j) of W^(l) of a[b, i] w_ij.
    wabs: |a| . |W|;  w: other values on the support of W^(l) (e.g. error magnitudes)."""
    aT = np.ascontiguousarray((np.abs(a) if wabs else a).astype(F64).T)      # [n_in x B]
    if w is None:
        w = (np.abs(Ly.w) if wabs else Ly.w).astype(F64)
    return _spmm_fwd_stack(aT, [w], Ly, F64).T


def spmm_fwd_abs(blocks, Ly: Layer):
    """[a_k . W_k for (a_k, W_k) in blocks] for non-negative magnitude operands (a_k [B x n_in],
    W_k values on the support), in float32 -- magnitudes are error bounds (R24), relative
    accuracy ~1e-6 is ample -- in one pass over the connections."""
    B = blocks[0][0].shape[0]
    aT = np.ascontiguousarray(np.concatenate([x for x, _ in blocks], axis=0).astype(F32).T)   # [n_in x K B]
    zT = _spmm_fwd_stack(aT, [w for _, w in blocks], Ly, F32)
    return [zT[:, k * B:(k + 1) * B].T.astype(F64) for k in range(len(blocks))]


def spmm_bwd(delta: np.ndarray, Ly: Layer, w: Optional[np.ndarray] = None) -> np.ndarray:
    """delta . W^(l)^T  ([B x n_out] x [n_out x n_in]) in float64:
    out[b, i] = sum over the connections (i, j) of W^(l) of delta[b, j] w_ij (w overrides the values)."""
    dT = np.ascontiguousarray(delta.astype(F64).T)                          # [n_out x B]
    w = Ly.w.astype(F64) if w is None else w
    rows, col = Ly.rows(), Ly.col.astype(np.int64)
    oT = np.zeros((Ly.n_in, dT.shape[1]), dtype=F64)

    def part(s0, s1):
        _segment_sums(dT[col[s0:s1]] * w[s0:s1, None], rows[s0:s1], oT)
    _run_chunks(part, _chunks(Ly.nnz, dT.shape[1], rows))
    return oT.T


def spmm_bwd_abs(blocks, Ly: Layer) -> np.ndarray:
    """sum over (d_k, W_k) in blocks of d_k . W_k^T, for non-negative magnitude operands, float32
    (see spmm_fwd_abs), one pass over the connections."""
    B = blocks[0][0].shape[0]
    K = len(blocks)
    dT = np.ascontiguousarray(np.concatenate([d for d, _ in blocks], axis=0).astype(F32).T)   # [n_out x K B]
    ws = [np.asarray(w, F32) for _, w in blocks]
    rows, col = Ly.rows(), Ly.col.astype(np.int64)
    oT = np.zeros((Ly.n_in, K * B), dtype=F32)

    def part(s0, s1):
        t = dT[col[s0:s1]]
        for k in range(K):
            t[:, k * B:(k + 1) * B] *= ws[k][s0:s1, None]
        _segment_sums(t, rows[s0:s1], oT)
    _run_chunks(part, _chunks(Ly.nnz, K * B, rows))
    return sum(oT[:, k * B:(k + 1) * B].T.astype(F64) for k in range(K))


def sddmm(a: np.ndarray, delta: np.ndarray, Ly: Layer) -> np.ndarray:
    """g_ij = sum_b a[b, i] delta[b, j] for (i, j) in the support only (fp64)."""
    aT = np.ascontiguousarray(a.astype(F64).T)
    dT = np.ascontiguousarray(delta.astype(F64).T)
    rows, col = Ly.rows(), Ly.col.astype(np.int64)
    g = np.zeros(Ly.nnz, dtype=F64)

    def part(s0, s1):
        g[s0:s1] = (aT[rows[s0:s1]] * dT[col[s0:s1]]).sum(axis=1)
    _run_chunks(part, _chunks(Ly.nnz, aT.shape[1]))
    return g


# --------------------------------------------------------------------------------------
# activations (Eq. 3 All-ReLU PAPER.md:106-112; Eq. 5 ReLU PAPER.md:533-539)
# --------------------------------------------------------------------------------------
def neg_slope(st_or_act, alpha: float, l: int) -> float:
    """Slope of f_l for x <= 0: -alpha for even l, +alpha for odd l (All-ReLU); 0 for ReLU."""
    act = st_or_act.activation if hasattr(st_or_act, "activation") else st_or_act
    if act == "relu":
        return 0.0
    return -alpha if l % 2 == 0 else alpha


def activation(x, l: int, alpha: float, act: str = "all_relu"):
    s = neg_slope(act, alpha, l)
    x = np.asarray(x, dtype=F64)
    return np.where(x > 0, x, s * x)


def activation_grad(x, l: int, alpha: float, act: str = "all_relu"):
    """f_l'(x): 1 for x > 0, the negative-side slope for x <= 0 (x = 0 takes the x <= 0
    branch of Eq. 3 literally)."""
    s = neg_slope(act, alpha, l)
    x = np.asarray(x, dtype=F64)
    return np.where(x > 0, 1.0, s)


def dropout_keep(seed: int, rank: int, l: int, step: int, B: int, n: int, rate: float) -> np.ndarray:
    """Inverted-dropout keep mask [B x n] of hidden layer l (PAPER.md:957 rate; DESIGN reading 13):
    element (b, j) -> word (b & 3) of Philox(DROPOUT, idx = j * 2^32 + (b >> 2), c3 = step), i.e.
    one Philox block per neuron j and group of 4 consecutive batch rows; kept iff
    word >= floor(rate * 2^32)."""
    if rate <= 0.0:
        return np.ones((B, n), dtype=bool)
    nb4 = (B + 3) // 4
    b4 = np.arange(nb4, dtype=np.uint64)[:, None]
    j = np.arange(n, dtype=np.uint64)[None, :]
    idx = ((j << np.uint64(32)) | b4).ravel()                     # [nb4 * n], row-major in (b4, j)
    W = np.stack(philox.stream(seed, philox.PURPOSE_DROPOUT, rank, l, step & 0xFFFFFFFF, idx), axis=0)
    W = W.reshape(4, nb4, n)                                      # W[w, b4, j]
    b = np.arange(B)
    word = W[b & 3, b >> 2, :]                                    # [B x n]
    thr = np.uint64(math.floor(rate * 4294967296.0))
    return word.astype(np.uint64) >= thr


# --------------------------------------------------------------------------------------
# forward / loss / backward / update
# --------------------------------------------------------------------------------------
@dataclass
class Trace:
    B: int
    train: bool
    step: int
    version: int
    a: List[np.ndarray]                # a[l-1] = float32 activations of layer l (a[0] = x)
    z: List[Optional[np.ndarray]]      # z[l-1] = float64 pre-activations (None for l = 1)
    keep: List[Optional[np.ndarray]]   # dropout keep masks of hidden layers
    p: np.ndarray                      # float32 softmax probabilities [B x n_L]
    p64: np.ndarray
    ambiguous: List[int]               # per layer: #elements with |z| within fp32 rounding of 0
    # running fp32 error magnitudes (R24): an fp32 implementation of the same step
    # may differ from a[l-1] / z[l-1] / p by up to KAPPA_U times these (first-order bound)
    amag: List[Optional[np.ndarray]] = None
    zmag: List[Optional[np.ndarray]] = None
    pmag: Optional[np.ndarray] = None


# Test instrumentation (the R24 error magnitudes and the R32 kink count) is on by default; the
# bench's cpu_baseline times the method's own arithmetic with it off (bench.py).
INSTRUMENT = True


def forward(st: State, x: np.ndarray, train: bool = True, step: int = 0, rank: Optional[int] = None) -> Trace:
    """sparse_mlp_forward: z_l = a_{l-1} W^(l) + b_l, a_l = f_l(z_l) (Eq. 3) then inverted dropout
    in train mode (hidden layers only); p = softmax(z_L) computed stably.

    Alongside, the running error magnitudes of R24 (Higham, Accuracy and Stability of Numerical
    Algorithms, 2nd ed., §3.1-3.3: a sum of products computed in fp32 differs from its exact
    value by at most gamma times the same sum of absolute values; errors of the inputs propagate
    through the absolute values of what multiplies them; first order in u, so products of two
    magnitudes are dropped):
        zmag_l = |a_{l-1}| . |W^(l)| + amag_{l-1} . |W^(l)| + |a_{l-1}| . wmag + |b_l| + bmag_l,
        amag_1 = 0 (x exact)
        amag_l = zmag_l * max(1, |slope_l|) * keep/(1-r)     (f_l is Lipschitz with that constant)
        pmag   = 2 p max_k zmag_L[:, k]                    (|dp_c| <= p_c (|dz_c| + sum_k p_k |dz_k|))"""
    rank = st.rank if rank is None else rank
    x = np.asarray(x, dtype=F32)
    B = x.shape[0]
    a = [x]
    zs: List[Optional[np.ndarray]] = [None]
    keeps: List[Optional[np.ndarray]] = [None]
    amags: List[Optional[np.ndarray]] = [np.zeros(x.shape, F64)]
    zmags: List[Optional[np.ndarray]] = [None]
    amb = [0]
    L = st.L
    scale = 1.0 / (1.0 - st.dropout) if st.dropout > 0 else 1.0
    for l in range(2, L + 1):
        Ly = st.layer(l)
        z = spmm_fwd(a[-1], Ly) + st.b[l - 2].astype(F64)
        if INSTRUMENT:
            aa = np.abs(a[-1]).astype(F64)
            wa = np.abs(Ly.w)
            blocks = [(aa, wa)]
            if np.any(amags[-1]):
                blocks.append((amags[-1], wa))
            if Ly.wmag is not None:
                blocks.append((aa, Ly.wmag))
            res = spmm_fwd_abs(blocks, Ly)
            mag = res[0] + np.abs(st.b[l - 2].astype(F64))
            zmag = sum(res) + np.abs(st.b[l - 2].astype(F64)) + (0.0 if st.bmag is None else st.bmag[l - 2])
        else:
            mag = zmag = np.zeros_like(z)
        # pre-activations within fp32 summation error of the All-ReLU kink (hidden layers):
        # there the branch taken by an fp32 kernel may legitimately differ (R32, kink
        # guard).  mag == 0 means every term is an exact zero (e.g. no active binary input and a
        # zero bias): z is exactly 0 on every path, so that element is not ambiguous.
        amb.append(int(np.count_nonzero((np.abs(z) <= mag * (2.0 ** -20)) & (mag > 0))) if l < L else 0)
        zs.append(z)
        zmags.append(zmag)
        if l < L:
            h = activation(z, l, st.alpha, st.activation)
            hm = zmag * max(1.0, abs(neg_slope(st, st.alpha, l)))
            keep = None
            if train and st.dropout > 0:
                keep = dropout_keep(st.seed, rank, l, step, B, Ly.n_out, st.dropout)
                h = h * keep * scale
                hm = hm * keep * scale
            keeps.append(keep)
            a.append(h.astype(F32))
            amags.append(hm)
        else:
            keeps.append(None)
    zL = zs[-1]
    zmax = zL.max(axis=1, keepdims=True)
    ez = np.exp(zL - zmax)
    p64 = ez / ez.sum(axis=1, keepdims=True)
    pmag = 2.0 * p64 * zmags[-1].max(axis=1, keepdims=True)
    return Trace(B, bool(train), int(step), st.version, a, zs, keeps, p64.astype(F32), p64, amb,
                 amags, zmags, pmag)


def loss_grad(p64: np.ndarray, y: np.ndarray):
    """Softmax cross-entropy (DESIGN reading 12): L = (1/B) sum_b -ln p[b, y_b];
    dL/dz_L = (p - onehot) / B, the 1/B applied exactly once."""
    y = np.asarray(y, dtype=np.int64)
    B, C = p64.shape
    if np.any(y < 0) or np.any(y >= C):
        raise ValueError("label out of range")
    loss = float(-np.log(p64[np.arange(B), y]).mean())
    d = p64.copy()
    d[np.arange(B), y] -= 1.0
    return loss, d / B


@dataclass
class Grads:
    g: List[np.ndarray]      # g[l-2]: float32 [nnz of W^(l)] aligned to canonical CSR order
    gb: List[np.ndarray]     # gb[l-2]: float32 [n_l]
    loss: float
    deltas: List[Optional[np.ndarray]]   # deltas[l-1]: float32 [B x n_l] (None for l = 1)
    # running error magnitudes (R24), aligned with g / gb / deltas; None = exact
    gmag: Optional[List[np.ndarray]] = None
    gbmag: Optional[List[np.ndarray]] = None
    dmag: Optional[List[Optional[np.ndarray]]] = None


def backward(st: State, tr: Trace, y: np.ndarray) -> Grads:
    """sparse_mlp_backward: for l = L..2, g_ij = sum_b a_{l-1}[b,i] delta_l[b,j] on the support
    only (SDDMM), gb_l = sum_b delta_l, delta_{l-1} = (delta_l W^(l)T) * f'_{l-1}(z_{l-1}) * keep/(1-r)
    for l >= 3.  delta_L = (p - onehot)/B.

    Running error magnitudes (R24), first order as in `forward`, with f' exact away from the kink
    (R32):
        dmag_L     = pmag / B
        gmag_ij    = sum_b [(|a_{l-1}| + amag_{l-1})[b, i] |delta_l|[b, j] + |a_{l-1}|[b, i] dmag_l[b, j]]
        gbmag_j    = sum_b (|delta_l| + dmag_l)[b, j]
        dmag_{l-1} = (|delta_l| . (|W^(l)| + wmag)^T + dmag_l . |W^(l)|^T) * |f'_{l-1}| * keep/(1-r)"""
    if tr.version != st.version or not tr.train:
        raise RuntimeError("stale trace")
    L = st.L
    loss, dz = loss_grad(tr.p64, y)
    delta = dz.astype(F32)
    scale = 1.0 / (1.0 - st.dropout) if st.dropout > 0 else 1.0
    g: List[Optional[np.ndarray]] = [None] * (L - 1)
    gb: List[Optional[np.ndarray]] = [None] * (L - 1)
    gmag: List[Optional[np.ndarray]] = [None] * (L - 1)
    gbmag: List[Optional[np.ndarray]] = [None] * (L - 1)
    deltas: List[Optional[np.ndarray]] = [None] * L
    dmags: List[Optional[np.ndarray]] = [None] * L
    deltas[L - 1] = delta
    dmag = (tr.pmag if tr.pmag is not None else np.zeros(dz.shape)) / tr.B
    dmags[L - 1] = dmag
    for l in range(L, 1, -1):
        Ly = st.layer(l)
        g[l - 2] = sddmm(tr.a[l - 2], delta, Ly).astype(F32)
        gb[l - 2] = delta.astype(F64).sum(axis=0).astype(F32)
        dabs = np.abs(delta).astype(F64)
        if INSTRUMENT:
            aabs = np.abs(tr.a[l - 2]).astype(F64)
            am = tr.amag[l - 2] if tr.amag is not None else np.zeros_like(aabs)
            # stacking along the batch axis sums the two products: sum_b A1 D1 + sum_b A2 D2
            gmag[l - 2] = sddmm(np.concatenate([aabs + am, aabs]), np.concatenate([dabs, dmag]), Ly)
        else:
            gmag[l - 2] = np.zeros(Ly.nnz)
        gbmag[l - 2] = (dabs + dmag).sum(axis=0)
        if l >= 3:
            fp = activation_grad(tr.z[l - 2], l - 1, st.alpha, st.activation)
            d = spmm_bwd(delta, Ly) * fp
            if INSTRUMENT:
                wa = np.abs(Ly.w).astype(F64)
                dmag = spmm_bwd_abs([(dabs, wa + _m(Ly.wmag, wa)), (dmag, wa)], Ly) * np.abs(fp)
            else:
                dmag = np.zeros_like(d)
            if tr.keep[l - 2] is not None:
                d = d * tr.keep[l - 2] * scale
                dmag = dmag * tr.keep[l - 2] * scale
            delta = d.astype(F32)
            deltas[l - 2] = delta
            dmags[l - 2] = dmag
    return Grads(g, gb, loss, deltas, gmag, gbmag, dmags)


def step(st: State, grads: Grads, lr: float, momentum: float, weight_decay: float,
         grad_scale: float = 1.0) -> None:
    """sparse_mlp_step: Eq. 1 in velocity form, weight decay folded into the
    gradient (DESIGN reading 14):  v <- mu v - eta (s g + lambda w);  w <- w + v.
    Biases: vb <- mu vb - eta s gb; b <- b + vb (no decay).

    Running error magnitudes (R24): vmag' = mu (|v| + vmag) + eta (s (|g| + gmag) + lambda (|w| + wmag)),
    wmag' = |w| + wmag + |v'| + vmag' (likewise for the biases, without lambda)."""
    if st.bmag is None:
        st.bmag = [np.zeros(len(b), F64) for b in st.b]
        st.vbmag = [np.zeros(len(b), F64) for b in st.b]
    for idx, Ly in enumerate(st.layers):
        g = grads.g[idx].astype(F64) * grad_scale
        gm = (np.abs(grads.g[idx]).astype(F64) + _m(None if grads.gmag is None else grads.gmag[idx], g)) * grad_scale
        w64 = Ly.w.astype(F64)
        wm = np.abs(w64) + _m(Ly.wmag, w64)
        v = momentum * Ly.v.astype(F64) - lr * (g + weight_decay * w64)
        vm = momentum * (np.abs(Ly.v).astype(F64) + _m(Ly.vmag, w64)) + lr * (gm + weight_decay * wm)
        Ly.v = v.astype(F32)
        Ly.w = (w64 + Ly.v.astype(F64)).astype(F32)
        Ly.vmag = vm
        Ly.wmag = wm + np.abs(Ly.v).astype(F64) + vm
        gbv = grads.gb[idx].astype(F64) * grad_scale
        gbm = (np.abs(gbv) + _m(None if grads.gbmag is None else grads.gbmag[idx] * grad_scale, gbv))
        bm = np.abs(st.b[idx]).astype(F64) + st.bmag[idx]
        vb = momentum * st.vb[idx].astype(F64) - lr * gbv
        vbm = momentum * (np.abs(st.vb[idx]).astype(F64) + st.vbmag[idx]) + lr * gbm
        st.vb[idx] = vb.astype(F32)
        st.b[idx] = (st.b[idx].astype(F64) + st.vb[idx].astype(F64)).astype(F32)
        st.vbmag[idx] = vbm
        st.bmag[idx] = bm + np.abs(st.vb[idx]).astype(F64) + vbm


def train_step(st: State, x, y, lr, momentum, weight_decay, step_idx: int = 0):
    """One minibatch: forward (train) -> backward -> update.  Returns (loss, trace, grads)."""
    tr = forward(st, x, True, step_idx)
    gr = backward(st, tr, y)
    step(st, gr, lr, momentum, weight_decay)
    return gr.loss, tr, gr


def gradient_flow(grads: Grads) -> float:
    """Gradient flow ("the first-order approximation of the decrease in the loss
    expected after a gradient step"): the squared L2 norm of the whole
    gradient, sum over layers of sum g_ij^2 over the existing connections plus sum gb^2 over the
    biases.  Each fp32 gradient value is squared and summed in float64 (a plain definition: the
    order of the float64 sum is the only freedom)."""
    tot = 0.0
    for g in grads.g:
        tot += float(np.sum(np.square(g.astype(F64))))
    for gb in grads.gb:
        tot += float(np.sum(np.square(gb.astype(F64))))
    return tot
