"""Dense masked MLP in float64 with hand-written backprop — a PIN for the oracle, not part of it.

An independent formulation of the same network: W^(l) as a dense n_{l-1} x n_l float64
matrix that is zero off the support ("w_ij = 0 when there is no connection"),
plain matrix products, All-ReLU (Eq. 3), softmax cross-entropy.  Used by
tests/test_oracle_model.py (dense-oracle equivalence, SURVEY O3/O5 pins) and itself pinned
by central finite differences there.
"""
from __future__ import annotations

import numpy as np


def act(z, l, alpha, kind="all_relu"):
    s = 0.0 if kind == "relu" else (-alpha if l % 2 == 0 else alpha)
    return np.where(z > 0, z, s * z), np.where(z > 0, 1.0, s)


def forward_backward(Ws, bs, x, y, alpha, kind="all_relu", keeps=None, rate=0.0, dtype=np.float64, out=None):
    """Ws[k] dense [n_{l-1} x n_l] (l = k+2), bs[k] [n_l]; keeps[k] optional dropout masks of
    hidden layer l = k+2.  Returns (loss, probs, dW list, db list).  dtype = np.float32 runs the
    whole computation in fp32 (BLAS sgemm order): another fp32 implementation of the step, for
    the error-bound pin of tests/test_oracle_model.py.  out (dict): receives the activations
    "a" and the deltas "delta" (index k = layer l - 1)."""
    L = len(Ws) + 1
    B = x.shape[0]
    Ws = [np.asarray(W, dtype) for W in Ws]
    bs = [np.asarray(b, dtype) for b in bs]
    a = [np.asarray(x, dtype)]
    d = []
    scale = 1.0 / (1.0 - rate) if rate > 0 else 1.0
    for k, (W, b) in enumerate(zip(Ws, bs)):
        l = k + 2
        z = a[-1] @ W + b
        if l < L:
            h, dh = act(z, l, alpha, kind)
            if keeps is not None and keeps[k] is not None:
                h = h * keeps[k] * scale
                dh = dh * keeps[k] * scale
            a.append(h)
            d.append(dh)
        else:
            a.append(z)
    zL = a[-1]
    e = np.exp(zL - zL.max(1, keepdims=True))
    p = e / e.sum(1, keepdims=True)
    loss = -np.log(p[np.arange(B), y]).mean()
    delta = p.copy()
    delta[np.arange(B), y] -= 1.0
    delta /= dtype(B)
    dWs, dbs = [None] * len(Ws), [None] * len(Ws)
    deltas = [None] * L
    for k in range(len(Ws) - 1, -1, -1):
        deltas[k + 1] = delta
        dWs[k] = a[k].T @ delta
        dbs[k] = delta.sum(0)
        if k > 0:
            delta = (delta @ Ws[k].T) * d[k - 1].astype(dtype)
    if out is not None:
        out["a"] = a
        out["delta"] = deltas
    return loss, p, dWs, dbs


def loss_only(Ws, bs, x, y, alpha, kind="all_relu"):
    return forward_backward(Ws, bs, x, y, alpha, kind)[0]
