"""Synchronous data parallelism for the sparse MLP (WASSP-SGD phase 1).

One process per GPU; every rank holds the full, identical replica (same seed -> same ER topology,
same values).  Per step every rank runs forward + unfused backward on its own minibatch, the
contiguous grad view is SUM-allreduced over the process group (NCCL over NVLink / NVSwitch on
B200 boxes; gloo in the CPU tests), and every rank applies the same Eq. 1 update with
grad_scale = 1/K, so replicas stay bit-identical.  SET evolution and importance pruning are
deterministic functions of (seed, evolve index, weights) and run replicated with no collective.
Averaging points (Eq. 2) allreduce the param view and divide by K.

The learning rate follows the "gradual warmup and linear scaling rule" of PAPER.md:323
(DESIGN reading R20): eta_t = eta (1 + (K - 1) min(1, t / warmup_steps)).
"""
from __future__ import annotations

import os
from typing import Optional, Tuple

import numpy as np


def init_process_group(backend: Optional[str] = None) -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment; world 1 without one."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            import torch
            backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(local)
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world, local


def scaled_lr(base_lr: float, world: int, step: int, warmup_steps: int) -> float:
    if world <= 1:
        return base_lr
    frac = 1.0 if warmup_steps <= 0 else min(1.0, step / float(warmup_steps))
    return base_lr * (1.0 + (world - 1) * frac)


def shard_bounds(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Rank k owns samples [k n / K, (k+1) n / K) of the (globally permuted) training set."""
    return (rank * n) // world, ((rank + 1) * n) // world


def allreduce_sum_(t, group=None):
    """In-place SUM allreduce of a flat tensor (the grad view, X1)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def average_model_(model, group=None, biases_only: bool = False):
    """Eq. 2 over the process group (X2): SUM-allreduce the model's param view
    (or only its bias block), then the library divides by K and refreshes the mirror copy
    (sparse_mlp_params_averaged) -- no method arithmetic outside the library."""
    import torch.distributed as dist
    K = dist.get_world_size(group) if dist.is_initialized() else 1
    if K > 1:
        p, _ = model.param_view()
        if biases_only:
            _, bias_base = model.view_layout()
            p = p[bias_base:]
        dist.all_reduce(p, op=dist.ReduceOp.SUM, group=group)
        model.params_averaged(K, biases_only)
    return K


def tensor_hash(t) -> int:
    """64-bit hash of a float32 tensor's bit pattern (X3 replica-identity check)."""
    import torch
    bits = t.detach().contiguous().view(torch.int32).to(torch.int64).cpu().numpy().astype(np.uint64)
    idx = np.arange(1, len(bits) + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = np.bitwise_xor.reduce(bits * np.uint64(0x9E3779B97F4A7C15) + idx * np.uint64(0xC2B2AE3D27D4EB4F))
        h = int(h) ^ int(np.sum(bits * idx, dtype=np.uint64))
    return h & ((1 << 63) - 1)


def replicas_identical(t, group=None) -> bool:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return True
    h = torch.tensor([tensor_hash(t)], dtype=torch.int64, device=t.device)
    hs = [torch.zeros_like(h) for _ in range(dist.get_world_size(group))]
    dist.all_gather(hs, h, group=group)
    return all(int(x.item()) == int(h.item()) for x in hs)


def dp_train_step(model, X, Y, idx, step: int, lr: float, momentum: float, weight_decay: float,
                  world: int, loss=None, group=None):
    """One synchronous step on this rank: forward / unfused backward on the local batch, X1
    allreduce of the grad view, Eq. 1 update with grad_scale = 1/K (identical on every rank)."""
    from .sparse_mlp import SGD
    if world == 1:
        model.forward(X, x_idx=idx, train=True, step=step)
        model.backward(Y, y_idx=idx, loss=loss, fused=SGD(lr, momentum, weight_decay))
        return
    model.forward(X, x_idx=idx, train=True, step=step)
    model.backward(Y, y_idx=idx, loss=loss, fused=None)
    g, _ = model.grad_view()
    allreduce_sum_(g, group)
    model.step(SGD(lr, momentum, weight_decay, 1.0 / world))


class OverlappedAllreduce:
    """X1 with the communication overlapped on the backward: after an UNFUSED
    backward is enqueued, the grad view is SUM-allreduced bucket by bucket on a side stream, each
    bucket as soon as the library's per-layer event says its last layer's gradient is final -- the
    output layer first, while the backward of the layers below is still running.  A bucket is a
    run of consecutive weight layers W^(L), W^(L-1), ... (contiguous in the view) of at least
    `bucket_bytes`; the bucket holding W^(2) also takes the bias block b_2..b_L, which is final once
    W^(2)'s backward ran (and is contiguous with it when that bucket spans every layer).  Small
    models (C4's 0.22 MB view) thus make ONE collective per step -- latency, not bandwidth, is
    their cost -- and C5 one per layer (215 MB: the overlap pays).  The caller's stream waits for
    all of them before the Eq. 1 update.  Every rank issues the same collectives in the same order
    (same topology and layout), so the reduction is the plain value allreduce.  Everything is
    stream-ordered (events, no host sync), so the step can be captured in a CUDA graph, NCCL
    collectives included."""

    def __init__(self, model, group=None, bucket_bytes: int = 4 << 20):
        import torch
        self.m = model
        self.group = group
        self.stream = torch.cuda.Stream(device=model.device) if torch.cuda.is_available() else None
        self.layout, self.bias_base = model.view_layout()
        self.buckets = self.plan(self.layout, self.bias_base, model.L, bucket_bytes)

    @staticmethod
    def plan(layout, bias_base: int, L: int, bucket_bytes: int):
        """[(wait_layer, lo, hi)]: slices [lo, hi) of the grad view in issue order; a slice is
        final once layer wait_layer's backward has run (host-only arithmetic on the layout)."""
        out, l = [], L
        while l >= 2:
            top = l
            off, cap = layout[l - 2]
            hi = off + cap
            lo, nbytes = off, 4 * cap
            while nbytes < bucket_bytes and l > 2:     # extend downwards (contiguous in the view)
                l -= 1
                off, cap = layout[l - 2]
                lo, nbytes = off, nbytes + 4 * cap
            if l == 2 and top == L:                       # every layer: one slice through the biases
                out.append((2, lo, None))
                return out
            out.append((l, lo, hi))
            l -= 1
        out.append((2, bias_base, None))                  # b_2..b_L
        return out

    def __call__(self, reduce=None):
        """reduce(tensor_slice) -> work handle (default: torch.distributed.all_reduce SUM, async)."""
        import torch
        import torch.distributed as dist
        if reduce is None:
            def reduce(t):
                return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        g, _ = self.m.grad_view()
        works = []
        main = torch.cuda.current_stream()
        # no blanket wait on the main stream: each bucket waits only for its own layer's event, so
        # the collectives overlap the rest of the backward
        with torch.cuda.stream(self.stream):
            for l, lo, hi in self.buckets:
                self.m.wait_layer(l, self.stream)
                works.append(reduce(g[lo:hi]))
        for w in works:
            if w is not None:
                w.wait()                                     # the current stream waits for the collective
        main.wait_stream(self.stream)


def dp_train_step_overlapped(model, X, Y, idx, step: int, lr: float, momentum: float, weight_decay: float,
                             world: int, overlap: "OverlappedAllreduce", loss=None):
    """dp_train_step with the per-layer allreduce overlapped on the backward."""
    from .sparse_mlp import SGD
    model.forward(X, x_idx=idx, train=True, step=step)
    model.backward(Y, y_idx=idx, loss=loss, fused=None)
    overlap()
    model.step(SGD(lr, momentum, weight_decay, 1.0 / world))


def union_average_(model, targets, group=None) -> list:
    """WASAP phase 2 end (Alg. 1): average K replicas
    whose topologies evolved independently over the UNION of their supports and re-sparsify each
    layer to targets[l-2] connections (the phase-1 count), then average the biases (Eq. 2).
    Collectives: per layer an all-gather of the nnz counts and of the (position, value) lists
    (padded to the largest), concatenated in rank order; the merge / selection / rebuild runs in
    the library identically on every rank, so the replicas end bit-identical.  Returns the kept
    count per weight layer."""
    import torch
    import torch.distributed as dist
    K = dist.get_world_size(group) if dist.is_initialized() else 1
    kept = []
    for l in range(2, model.L + 1):
        pos, val = model.export_positions(l)
        if K > 1:
            n = torch.tensor([pos.numel()], dtype=torch.int64, device=pos.device)
            ns = [torch.zeros_like(n) for _ in range(K)]
            dist.all_gather(ns, n, group=group)
            counts = [int(x.item()) for x in ns]
            m = max(counts)
            pp = torch.zeros(m, dtype=torch.int64, device=pos.device)
            vp = torch.zeros(m, dtype=torch.float32, device=pos.device)
            pp[:pos.numel()] = pos
            vp[:val.numel()] = val
            P = [torch.empty_like(pp) for _ in range(K)]
            V = [torch.empty_like(vp) for _ in range(K)]
            dist.all_gather(P, pp, group=group)
            dist.all_gather(V, vp, group=group)
            pos = torch.cat([P[k][:counts[k]] for k in range(K)])
            val = torch.cat([V[k][:counts[k]] for k in range(K)])
        kept.append(model.union_average_layer(l, K, pos, val, int(targets[l - 2])))
    average_model_(model, group, biases_only=True)
    return kept


class StaleGradient:
    """A gradient together with the topology it was computed on (version-tagged), for the
    asynchronous phase-1 analogue (Alg. 1): taken after an
    unfused backward, applied later -- possibly after the model's topology evolved -- through
    RetainValidUpdates."""

    def __init__(self, model):
        g, version = model.grad_view()
        layout, bias_base = model.view_layout()
        nnz = model.info()["nnz"]
        self.version = version
        self.layers = []
        for l in range(2, model.L + 1):
            pos, _ = model.export_positions(l)
            off = layout[l - 2][0]
            self.layers.append((pos.clone(), g[off:off + nnz[l - 1]].clone()))
        self.bias = g[bias_base:].clone()


def apply_stale_gradient(model, stale: "StaleGradient", sgd) -> list:
    """Server side of Alg. 1 phase 1: g = RetainValidUpdates(stale gradient, current model) per
    layer (intersection of supports), the biases unchanged (dense), then the Eq. 1 update.
    Returns the retained connection count per layer."""
    kept = [model.retain_valid_updates(l, pos, gv) for l, (pos, gv) in zip(range(2, model.L + 1), stale.layers)]
    g, _ = model.grad_view()
    _, bias_base = model.view_layout()
    g[bias_base:].copy_(stale.bias)
    model.step(sgd)
    return kept
