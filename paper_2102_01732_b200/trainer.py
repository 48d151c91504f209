"""Epoch driver for the sparse MLP (Alg. 2; SURVEY.md §3 call stacks 3-4).

Per epoch: the rank's shard is reshuffled (Alg. 1), every full minibatch runs the hot path
(forward, backward, Eq. 1 update; for K > 1 the grad-view allreduce and the update kernel), the
last partial batch is kept and normalised by its own size; at the epoch end, when
scheduled, Importance Pruning runs first and SET evolution second (Alg. 2 order, reading R18),
replicated on every rank with no communication.  Evolution is skipped after the final epoch
(reading R10).

Full batches replay one CUDA graph of ``graph_steps`` captured steps (forward + backward + the
dropout-counter increment), reading their sample indices from a static device window that is
refilled before each replay; the graph stays valid across evolve / prune because the library
keeps every device pointer stable and reads its work-list sizes from device memory.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .dp import allreduce_sum_, average_model_, scaled_lr, shard_bounds, union_average_
from .sparse_mlp import SGD, SparseMLP


@dataclass
class EpochRecord:
    epoch: int
    loss: float
    samples: int
    train_s: float
    evolve_s: float
    prune_s: float
    nnz: List[int]
    alive: List[int]
    removed: List[int] = field(default_factory=list)
    pruned: List[int] = field(default_factory=list)


class Trainer:
    def __init__(self, model: SparseMLP, cfg, X, Y, rank: int = 0, world: int = 1, use_graph: bool = True,
                 graph_steps: int = 8, group=None, average_every_epoch: bool = False):
        import torch
        self.torch = torch
        self.m = model
        self.cfg = cfg
        self.X, self.Y = X, Y                 # resident device tensors of this rank's shard
        self.rank, self.world, self.group = rank, world, group
        self.B = cfg.batch
        self.use_graph = use_graph and world == 1
        self.graph_steps = graph_steps
        self.average_every_epoch = average_every_epoch
        self.n = X.shape[0]
        self.global_step = 0
        self.dev = X.device
        self.counter = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.loss_buf = torch.zeros(max(1, graph_steps), dtype=torch.float32, device=self.dev)
        self.idx_win = torch.zeros(self.B * max(1, graph_steps), dtype=torch.int32, device=self.dev)
        self.graph = None
        self._graph_lr = None
        self.warmup_steps = max(1, cfg.n_samples // (self.B * max(1, world)))

    # ---------------------------------------------------------------------------------- batches
    def epoch_order(self, epoch: int) -> np.ndarray:
        return np.random.default_rng([self.cfg.data_seed, epoch, self.rank]).permutation(self.n).astype(np.int32)

    def _sgd(self, step: int, grad_scale: float = 1.0) -> SGD:
        lr = scaled_lr(self.cfg.lr, self.world, step, self.warmup_steps)
        return SGD(lr, self.cfg.momentum, self.cfg.weight_decay, grad_scale)

    def _eager_step(self, idx, loss_slot, step: int):
        B = int(idx.shape[0])
        self.m.forward(self.X, x_idx=idx, train=True, step=step)
        if self.world == 1:
            self.m.backward(self.Y, y_idx=idx, loss=loss_slot, fused=self._sgd(step))
        else:
            self.m.backward(self.Y, y_idx=idx, loss=loss_slot, fused=None)
            g, _ = self.m.grad_view()
            allreduce_sum_(g, self.group)
            self.m.step(self._sgd(step, 1.0 / self.world))
        return B

    def _capture(self, lr: SGD):
        torch = self.torch
        self.m.sparse_mlp_set_step_counter(self.counter)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for k in range(self.graph_steps):
                    idx = self.idx_win[k * self.B:(k + 1) * self.B]
                    self.m.forward(self.X, x_idx=idx, train=True, step=0)
                    self.m.backward(self.Y, y_idx=idx, loss=self.loss_buf[k:k + 1], fused=lr)
                    self.counter.add_(1)
                self.m.join()                        # the library's side-stream work rejoins the capture
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g
        self._graph_lr = lr

    # ---------------------------------------------------------------------------------- epoch
    def train_epoch(self, epoch: int, last: bool = False) -> EpochRecord:
        torch = self.torch
        cfg = self.cfg
        order = torch.from_numpy(self.epoch_order(epoch)).to(self.dev)
        nfull = self.n // self.B
        loss_sum = torch.zeros(1, dtype=torch.float64, device=self.dev)
        one = torch.zeros(1, dtype=torch.float32, device=self.dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = 0
        if self.use_graph and self.world == 1:
            lr = self._sgd(self.global_step)
            while s + self.graph_steps <= nfull:
                if self.graph is None or self._graph_lr != lr:
                    self.counter.fill_(self.global_step)
                    self._capture(lr)
                    # the capture does not execute: the counter is restored for the replay
                self.counter.fill_(self.global_step)
                self.idx_win.copy_(order[s * self.B:(s + self.graph_steps) * self.B])
                self.graph.replay()
                loss_sum += self.loss_buf.double().sum() * self.B
                s += self.graph_steps
                self.global_step += self.graph_steps
            self.m.sparse_mlp_set_step_counter(None)
        while s < nfull:
            self._eager_step(order[s * self.B:(s + 1) * self.B], one, self.global_step)
            loss_sum += one.double() * self.B
            s += 1
            self.global_step += 1
        tail = self.n - nfull * self.B
        if tail > 0:
            self._eager_step(order[nfull * self.B:], one, self.global_step)
            loss_sum += one.double() * tail
            self.global_step += 1
        torch.cuda.synchronize()
        train_s = time.perf_counter() - t0
        loss = float(loss_sum.item()) / self.n
        # ---- epoch boundary: Eq. 2 averaging (periodic, optional), pruning, evolution
        if self.average_every_epoch and self.world > 1:
            average_model_(self.m, self.group)
        prune_s = evolve_s = 0.0
        pruned, removed = [], []
        if cfg.prune and epoch % cfg.prune_every == 0 and epoch >= cfg.prune_start:
            t1 = time.perf_counter()
            pruned, _ = self.m.prune_neurons(cfg.prune_percentile)
            torch.cuda.synchronize()
            prune_s = time.perf_counter() - t1
        if not last:
            t1 = time.perf_counter()
            removed = self.m.evolve_topology(cfg.zeta, epoch)
            torch.cuda.synchronize()
            evolve_s = time.perf_counter() - t1
        inf = self.m.info()
        return EpochRecord(epoch, loss, self.n, train_s, evolve_s, prune_s, inf["nnz"], inf["alive"], removed,
                           pruned)

    def fit(self, epochs: int) -> List[EpochRecord]:
        return [self.train_epoch(e, last=(e == epochs - 1)) for e in range(epochs)]

    def fit_wasap(self, phase1_epochs: int, phase2_epochs: int) -> List[EpochRecord]:
        """WASAP with the paper's phase 2 (Alg. 1):
        phase 1 = synchronous DP (one gradient allreduce per step, replicated evolution); phase 2 =
        every replica trains its own shard with NO per-step collective and evolves its topology
        with its own counter (rank-specific evolve index, DESIGN R21), so the K topologies diverge;
        at the end the K models are averaged over the union of their supports and re-sparsified
        to the phase-1 per-layer connection counts (dp.union_average_)."""
        recs = [self.train_epoch(e, last=False) for e in range(phase1_epochs)]
        targets = self.m.info()["nnz"][1:]
        world, use_graph = self.world, self.use_graph
        self.world, self.use_graph = 1, False            # local steps: no collective in phase 2
        try:
            for e in range(phase1_epochs, phase1_epochs + phase2_epochs):
                rec = self.train_epoch(e, last=True)       # local training, no replicated evolve
                t1 = time.perf_counter()
                # independent evolution: counter distinct per (epoch, rank)
                rec.removed = self.m.evolve_topology(self.cfg.zeta, (1 << 20) + e * max(1, world) + self.rank)
                self.torch.cuda.synchronize()
                rec.evolve_s = time.perf_counter() - t1
                recs.append(rec)
        finally:
            self.world, self.use_graph = world, use_graph
        union_average_(self.m, targets, self.group)
        return recs


# ---------------------------------------------------------------------------------- post-training
def evaluate(model: SparseMLP, X, Y, batch: int) -> float:
    """Test accuracy: inference forward (no dropout) in batches of <= batch rows, argmax of p."""
    import torch
    n = X.shape[0]
    correct = 0
    probs = torch.empty((batch, model.sizes[-1]), dtype=torch.float32, device=X.device)
    for s in range(0, n, batch):
        b = min(batch, n - s)
        model.forward(X[s:s + b], train=False, probs=probs)
        correct += int((probs[:b].argmax(1) == Y[s:s + b].long()).sum().item())
    return correct / n


def prune_sweep(model: SparseMLP, X, Y, batch: int, percentiles=(5.0, 10.0, 15.0, 20.0, 25.0)):
    """Importance Pruning applied ONCE after training (Supp. C, Table of
    post-training pruning): for every threshold percentile rho, prune the
    trained model's hidden neurons with sparse_mlp_prune_neurons, record the test accuracy and the
    number of remaining connections, then restore the trained model.  Each rho starts from the
    same trained model (one-shot, not cumulative).  Returns [(rho, accuracy, connections)] plus
    the unpruned (None, accuracy, connections) first."""
    L = model.L
    snap = {l: (model.export_layer(l), model.sparse_mlp_export_bias(l)) for l in range(2, L + 1)}
    alive = {l: model.sparse_mlp_export_alive(l) for l in range(1, L + 1)}
    out = [(None, evaluate(model, X, Y, batch), int(sum(model.info()["nnz"])))]
    for rho in percentiles:
        model.prune_neurons(float(rho))
        out.append((float(rho), evaluate(model, X, Y, batch), int(sum(model.info()["nnz"]))))
        for l in range(2, L + 1):                      # restore the trained model
            e, (b, vb) = snap[l]
            model.import_layer(l, e["row_ptr"], e["col"], e["w"], e["v"])
            model.sparse_mlp_import_bias(l, b, vb)
        for l in range(1, L + 1):
            model.sparse_mlp_import_alive(l, alive[l])
    return out
