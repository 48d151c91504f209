"""Seeded synthetic stand-ins for the paper's datasets (SURVEY.md §8(d) "Synthetic inputs").

None of the paper's datasets (Table 1) is in the container; only
their shapes, sizes, class counts and value distributions are reproduced here.  No
dataset item is reproduced.

Rows are generated in fixed chunks of ``CHUNK`` rows, chunk ``c`` drawing from
``PCG64([data_seed, c])``, so any prefix / any chunk is reproducible on its own.
C5 rows are generated per row (``PCG64([data_seed, 7, row])``) so tests can draw a
handful of rows of the 100k x 65536 set; bench.py draws the full C5 set on the
device with a seeded torch generator (same distribution, different stream).
"""
from __future__ import annotations

import numpy as np

from .configs import WorkloadConfig

CHUNK = 65536


def _param_rng(cfg: WorkloadConfig) -> np.random.Generator:
    return np.random.default_rng([cfg.data_seed, 999_999])


def _params(cfg: WorkloadConfig):
    """Dataset-level parameters (teacher vectors, class means ...)."""
    rng = _param_rng(cfg)
    d = cfg.sizes[0]
    C = cfg.n_classes
    if cfg.name == "C1":
        r = np.zeros(d)
        pos = rng.choice(d, size=5, replace=False)
        r[pos] = rng.standard_normal(5)
        return {"r": r}
    if cfg.name == "C2":
        return {"mu": rng.uniform(0.0, 1.0, size=(C, d))}
    if cfg.name == "C3":
        sig = np.zeros((C, d))
        k = max(1, d // 100)
        for c in range(C):
            pos = rng.choice(d, size=k, replace=False)
            sig[c, pos] = rng.choice([-1.0, 1.0], size=k)
        p = (np.arange(C) + 1.0) ** -2.0
        return {"sig": sig, "p": p / p.sum()}
    if cfg.name == "C4":
        U = rng.standard_normal((d, 64)) / np.sqrt(d)
        v = rng.standard_normal(64)
        # median of h.v estimated once on a fixed probe set (labels balanced)
        probe = np.random.default_rng([cfg.data_seed, 424242]).standard_normal((200_000, d))
        thr = float(np.median(np.tanh(probe @ U) @ v))
        return {"U": U, "v": v, "thr": thr}
    if cfg.binary_input:
        r = np.zeros(d)
        k = d // 20
        pos = rng.choice(d, size=k, replace=False)
        r[pos] = rng.standard_normal(k)
        return {"r": r, "thr": 0.05 * float(r.sum())}
    # generic: gaussian features, random linear teacher over all classes
    return {"W": rng.standard_normal((d, C))}


def _chunk(cfg: WorkloadConfig, P: dict, c: int, rows: int):
    rng = np.random.default_rng([cfg.data_seed, c])
    d = cfg.sizes[0]
    C = cfg.n_classes
    if cfg.name == "C1":
        X = rng.standard_normal((rows, d))
        y = (X @ P["r"] > 0).astype(np.int32)
    elif cfg.name == "C2":
        y = rng.integers(0, C, size=rows).astype(np.int32)
        X = np.clip(P["mu"][y] + 0.2 * rng.standard_normal((rows, d)), 0.0, 1.0)
    elif cfg.name == "C3":
        y = rng.choice(C, size=rows, p=P["p"]).astype(np.int32)
        X = rng.standard_normal((rows, d)) + 0.5 * P["sig"][y]
    elif cfg.name == "C4":
        X = rng.standard_normal((rows, d))
        y = ((np.tanh(X @ P["U"]) @ P["v"]) > P["thr"]).astype(np.int32)
    else:
        X = rng.standard_normal((rows, d))
        y = np.argmax(X @ P["W"], axis=1).astype(np.int32)
    return X.astype(np.float32), y


def make_dataset(cfg: WorkloadConfig, n: int | None = None):
    """First ``n`` rows (default: all ``cfg.n_samples``) as (X float32 [n x d], y int32 [n])."""
    if cfg.binary_input:
        n = cfg.n_samples if n is None else n
        return c5_host_rows(cfg, np.arange(n))
    n = cfg.n_samples if n is None else min(n, cfg.n_samples)
    P = _params(cfg)
    Xs, ys = [], []
    c = 0
    done = 0
    while done < n:
        rows = min(CHUNK, cfg.n_samples - c * CHUNK)
        X, y = _chunk(cfg, P, c, rows)
        take = min(rows, n - done)
        Xs.append(X[:take])
        ys.append(y[:take])
        done += take
        c += 1
    return np.concatenate(Xs), np.concatenate(ys)


def c5_host_rows(cfg: WorkloadConfig, rows):
    """C5 rows by index: binary features Bernoulli(0.05) stored fp32; y = 1[x.r > 0.05*sum(r)]."""
    P = _params(cfg)
    rows = np.asarray(rows, dtype=np.int64)
    d = cfg.sizes[0]
    X = np.empty((len(rows), d), dtype=np.float32)
    for t, rr in enumerate(rows):
        rng = np.random.default_rng([cfg.data_seed, 7, int(rr)])
        X[t] = (rng.random(d) < 0.05).astype(np.float32)
    y = (X.astype(np.float64) @ P["r"] > P["thr"]).astype(np.int32)
    return X, y


def c5_device_dataset(cfg: WorkloadConfig, n: int, device, seed_offset: int = 0):
    """Full-size C5 shard generated on the device (bench only): same distribution as
    ``c5_host_rows``, drawn from a seeded torch generator.  Returns (X [n x d] fp32, y [n] int32)."""
    import torch
    P = _params(cfg)
    g = torch.Generator(device=device)
    g.manual_seed(cfg.data_seed * 1_000_003 + seed_offset)
    d = cfg.sizes[0]
    X = torch.empty((n, d), dtype=torch.float32, device=device)
    r = torch.from_numpy(P["r"].astype(np.float32)).to(device)
    y = torch.empty((n,), dtype=torch.int32, device=device)
    step = 4096
    for s in range(0, n, step):
        e = min(n, s + step)
        blk = (torch.rand((e - s, d), generator=g, device=device) < 0.05).to(torch.float32)
        X[s:e] = blk
        y[s:e] = (blk @ r > P["thr"]).to(torch.int32)
    return X, y


def make_batch_indices(n: int, batch: int, epoch: int, seed: int, rank: int = 0, world: int = 1):
    """Minibatch index lists for one epoch of one rank (Alg. 1).

    Rank k owns samples [k*n/K, (k+1)*n/K) of a fixed seeded permutation and reshuffles its
    shard every epoch with PCG64([seed, epoch, rank]).  The last partial batch is kept."""
    base = np.random.default_rng([seed, 31337]).permutation(n)
    lo = (rank * n) // world
    hi = ((rank + 1) * n) // world
    shard = base[lo:hi]
    perm = np.random.default_rng([seed, epoch, rank]).permutation(len(shard))
    order = shard[perm]
    return [order[s:s + batch] for s in range(0, len(order), batch)]
