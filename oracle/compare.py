"""Comparison metric for the parity tests (ORACLE — test infrastructure only).

Floating point (BASELINE.json north_star "max relative error 1e-4 in fp32 per step"; DESIGN.md
reading R24):

    err = max_i |gpu_i - ora_i| / max(|ora_i|,  FLOOR * max_j |ora_j|,  (KAPPA_U / TOL) * mag_i)

with FLOOR = 1e-3 and TOL = 1e-4, so err <= 1e-4 means: every element within
1e-4 relative, elements below 1e-3 of the tensor's largest held to 1e-7 of it, and -- the third
term -- no element held tighter than the fp32 error bound of its own computation, KAPPA_U * mag_i.
``mag`` is the oracle's running error magnitude of that element (model.forward / backward / step:
the same computation on absolute values, inputs' magnitudes propagated; Higham, Accuracy and
Stability of Numerical Algorithms, §3.1-3.3).  A result that cancels to ~0 (a sum of n products
of either sign) carries an fp32 rounding error ~ sqrt(n) u mag in ANY summation order, which no
relative or floor test can hold: the third term admits exactly that and nothing more.

KAPPA_U = 64 u = 2^-18 (u = 2^-24): the probabilistic summation bound lambda sqrt(n) u (Higham &
Mary, SIAM J. Sci. Comput. 41(5), 2019, Thm 2.4) with lambda = 8 and n = 64 terms per fixed-order
chain (the kernels' work segments hold <= 64 entries; longer sums are short fixed-order trees of
segment partials), exceeded with probability <= 2 exp(-lambda^2 / 2) ~ 1e-14 per element.

Integers: exact equality, with the first mismatching position reported.
"""
from __future__ import annotations

import numpy as np

FLOOR = 1e-3
TOL = 1e-4
KAPPA_U = 2.0 ** -18


def rel_err(gpu, ora, mag=None, floor: float = FLOOR) -> float:
    gpu = np.asarray(gpu, dtype=np.float64)
    ora = np.asarray(ora, dtype=np.float64)
    if gpu.shape != ora.shape:
        raise ValueError(f"shape mismatch {gpu.shape} vs {ora.shape}")
    if ora.size == 0:
        return 0.0
    scale = float(np.max(np.abs(ora)))
    if scale == 0.0 and mag is None:
        return float(np.max(np.abs(gpu)))          # an all-zero reference: the absolute error
    den = np.maximum(np.abs(ora), floor * scale)
    if mag is not None:
        mag = np.asarray(mag, dtype=np.float64)
        if mag.shape != ora.shape:
            raise ValueError(f"mag shape mismatch {mag.shape} vs {ora.shape}")
        den = np.maximum(den, (KAPPA_U / TOL) * mag)
    if not np.all(den > 0):
        zero = den == 0
        if np.any(gpu[zero] != 0):
            return float("inf")
        den = np.where(zero, 1.0, den)
    return float(np.max(np.abs(gpu - ora) / den))


def int_mismatch(gpu, ora):
    """None if equal, else (index, gpu value, oracle value) of the first mismatch."""
    gpu = np.asarray(gpu)
    ora = np.asarray(ora)
    if gpu.shape != ora.shape:
        return ("shape", gpu.shape, ora.shape)
    bad = np.flatnonzero(gpu.ravel() != ora.ravel())
    if len(bad) == 0:
        return None
    k = int(bad[0])
    return (k, gpu.ravel()[k].item(), ora.ravel()[k].item())
