"""Comparison metric for the parity tests (ORACLE — test infrastructure only).

Floating point (BASELINE.json north_star "max relative error 1e-4"; DESIGN reading 24):
    err = max_i |gpu_i - ora_i| / max(|ora_i|, floor * max_j |ora_j|),   floor = 1e-2
so elements near zero are judged against the tensor's scale instead of dividing by ~0: an fp32
sum of n terms carries an absolute error ~ sqrt(n) 2^-24 sum|terms| whatever its order, which is
unbounded relative to a result that cancels to ~0 (e.g. a logit that is a sum of 1000 products).
Elements >= 1% of the tensor's max are held to 1e-4 relative, smaller ones to 1e-6 of the max.
Integers: exact equality, with the first mismatching position reported.
"""
from __future__ import annotations

import numpy as np


def rel_err(gpu, ora, floor: float = 1e-2) -> float:
    gpu = np.asarray(gpu, dtype=np.float64)
    ora = np.asarray(ora, dtype=np.float64)
    if gpu.shape != ora.shape:
        raise ValueError(f"shape mismatch {gpu.shape} vs {ora.shape}")
    if ora.size == 0:
        return 0.0
    scale = float(np.max(np.abs(ora)))
    if scale == 0.0:
        return float(np.max(np.abs(gpu)))
    den = np.maximum(np.abs(ora), floor * scale)
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
