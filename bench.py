#!/usr/bin/env python
"""Benchmark: training samples/s of the truly sparse MLP step on B200 (BASELINE.json "metric").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1: synchronous DP over NCCL)

A step is one pass of the whole hot path over one minibatch B per rank: input
staging (a1), forward SpMM + All-ReLU (a2, a3), softmax-CE, backward delta SpMM + SDDMM (a4, a5),
the Eq. 1 momentum / weight-decay update (a6; fused into the backward on one GPU), and for N > 1
the NCCL SUM allreduce of the grad view (a7) + the update kernel.  Inputs are resident in HBM
(C5: 100k x 65536 fp32 = 26.2 GB per rank, far larger than the 126 MB L2, so no L2 flush is
needed between steps).  Per-epoch SET evolution / pruning is measured separately ("epoch" key).

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training samples/sec per sparse-MLP step"
UNIT = "samples/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            P = json.load(f)
        return float(P["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def f1_bytes(sizes, nnz, B):
    """Formula F1: algorithmic HBM bytes of one fused 1-GPU step."""
    tot = 0.0
    for l in range(2, len(sizes) + 1):
        tot += 32.0 * nnz[l - 1] + 4.0 * B * (3 * sizes[l - 2] + 2 * sizes[l - 1])
    return tot - 4.0 * B * sizes[0]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------ data
def load_data(cfg, rank, world, device):
    """Resident per-rank shard (X [n x n_1] fp32, Y [n] int32) on the device."""
    import numpy as np
    import torch

    from paper_2102_01732_b200.dp import shard_bounds
    from synth.data import c5_device_dataset, make_dataset
    lo, hi = shard_bounds(cfg.n_samples, rank, world)
    if cfg.binary_input:
        return c5_device_dataset(cfg, hi - lo, device, seed_offset=rank)
    X, Y = make_dataset(cfg, n=hi)
    return (torch.from_numpy(np.ascontiguousarray(X[lo:hi])).to(device),
            torch.from_numpy(np.ascontiguousarray(Y[lo:hi])).to(device))


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_job(cfg_name: str, batch: int, steps: int, evolve: bool = False) -> dict:
    """The oracle as it stands (its test instrumentation -- the R24 error magnitudes and the R32
    kink count -- switched off), single-threaded on the host cores, over a bounded sample of the
    same workload: `steps` training steps (fwd + bwd + Eq. 1) at batch `batch`, optionally followed
    by one SET evolution of every sparse layer (timed separately)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("MKL_NUM_THREADS", "1")
    import numpy as np

    from oracle import model as M
    from oracle import topology as T
    from synth import get_config
    from synth.data import c5_host_rows, make_dataset
    M.INSTRUMENT = False
    cfg = get_config(cfg_name)
    t0 = time.perf_counter()
    st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed)
    t_init = time.perf_counter() - t0
    n = batch * steps
    X, Y = (c5_host_rows(cfg, np.arange(n)) if cfg.binary_input else make_dataset(cfg, n=n))
    t0 = time.perf_counter()
    for s in range(steps):
        sl = slice(s * batch, (s + 1) * batch)
        M.train_step(st, X[sl], Y[sl], cfg.lr, cfg.momentum, cfg.weight_decay, s)
    dt = time.perf_counter() - t0
    t_ev = None
    if evolve:
        t1 = time.perf_counter()
        T.evolve(st, cfg.zeta, 0)
        t_ev = time.perf_counter() - t1
    nz = sum(L.nnz for L in st.layers if not L.dense_capped)
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{steps} oracle training step(s) (fwd+bwd+Eq.1 update) of {cfg_name} at batch {batch} "
                      f"(of {cfg.batch}): {dt:.1f} s timed"
                      + (f"; one SET evolution of all sparse layers ({nz / 1e6:.1f}M connections): {t_ev:.1f} s"
                         if t_ev is not None else "")
                      + f"; {t_init:.1f} s untimed ER init; plain NumPy, 1 thread, test instrumentation off",
            "cpu_model": _cpu_model(), "host_cpu_count": os.cpu_count(),
            "evolve_s": None if t_ev is None else round(t_ev, 2), "step_s": round(dt / steps, 2)}


def gathered_bytes(rec, sizes, nnz, cb, cbf, bits_layer2=False, implicit_delta=False):
    """L2->SM gather bytes of one launch of a row kernel (SURVEY.md §8(d) second ceiling): one
    chunk-wide fp32 row per connection -- the forward gathers a_{l-1} rows (CBf columns), the
    backward delta_l rows (CB columns).  Narrow output layers stream instead (0).  With the
    binary-input path, W^(2)'s fp32 row kernels return at once (0) and the bit kernels gather one
    16-B bit row (128 batch columns) per connection.  With the implicit delta_{L-1}
    the backward of W^(L-1) gathers one 16-B record per connection instead of a delta row."""
    l, k = rec["layer"], rec["kernel"]
    if k in ("fwd_bits", "bwd_bits"):
        return float(nnz[l - 1]) * 16.0
    if k not in ("fwd", "bwd") or l < 2:
        return 0.0
    if l == 2 and bits_layer2:
        return 0.0
    if l == len(sizes) and sizes[-1] <= 32:
        return 0.0
    if implicit_delta and k == "bwd" and l == len(sizes) - 1:
        return float(nnz[l - 1]) * 16.0
    w = cbf if k == "fwd" else cb
    return float(nnz[l - 1]) * w * 4.0


# ------------------------------------------------------------------------------------------ reference arm
def run_reference(args):
    """The reference arm of this tier: the oracle as it stands on the host cores,
    rank 0 only.  Same workload, metric and config as our arm; each step is a bounded sample of the
    workload's minibatch (C5: 4 of the 128 rows, C3: all 5, others the full batch) so the whole
    --steps K --warmup W run stays within a few minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth import get_config
    cfg = get_config(args.config)
    sample_B = min(cfg.batch, 4) if cfg.binary_input else cfg.batch
    warm = max(0, min(args.warmup, 1))
    res = cpu_baseline_job(cfg.name, sample_B, args.steps + warm)
    res["sample"] = (f"each of the {args.steps + warm} timed steps runs {sample_B} of the {cfg.batch} rows of the "
                     f"minibatch; " + res["sample"])
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, args.gpus),
            "cpu_baseline": res,
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(cfg, world: int) -> dict:
    """The workload keys both arms report (BASELINE.json configs)."""
    return {"workload": cfg.name, "stand_in_for": cfg.stand_in_for, "global_batch": cfg.batch * world,
            "batch_per_rank": cfg.batch, "layer_sizes": list(cfg.sizes), "epsilon": cfg.epsilon,
            "parallelism": f"dp{world}"}


# ------------------------------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunk-batch", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-epoch", action="store_true")
    ap.add_argument("--profile-json", default="")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the timed steps as CUDA graphs (auto: on for the launch-bound C1-C4 on one GPU)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(3, args.warmup)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2102_01732_b200 import SGD, SparseMLP
    from paper_2102_01732_b200.dp import OverlappedAllreduce, init_process_group, replicas_identical, scaled_lr
    from synth import get_config

    rank, world, local = init_process_group()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    cfg = get_config(args.config)
    B = cfg.batch

    t0 = time.perf_counter()
    model = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed,
                      rank, B, args.chunk_batch, local, input_kind=2 if cfg.binary_input else 1)
    t_create = time.perf_counter() - t0
    X, Y = load_data(cfg, rank, world, device)
    n_local = X.shape[0]
    rng = np.random.default_rng([cfg.data_seed, 77, rank])
    total_steps = args.warmup + args.steps
    idx_all = torch.from_numpy(np.concatenate([rng.permutation(n_local)[: B] for _ in range(total_steps)])
                               .astype(np.int32)).to(device)
    loss = torch.zeros(1, device=device)
    info0 = model.info()
    nnz = info0["nnz"]
    warm_steps = max(1, (cfg.n_samples // (B * world)))    # one epoch of linear-scaling warmup

    # N > 1 (or SMLP_BENCH_DP=1 to exercise the same path on one GPU): unfused backward, per-layer
    # allreduce of the grad view overlapped on the backward (OverlappedAllreduce), Eq. 1 update
    dp_path = world > 1 or os.environ.get("SMLP_BENCH_DP") == "1"
    overlap = OverlappedAllreduce(model) if dp_path else None

    def one_step(s):
        idx = idx_all[s * B:(s + 1) * B]
        lr = scaled_lr(cfg.lr, world, s, warm_steps)
        model.forward(X, x_idx=idx, train=True, step=s)
        if not dp_path:
            model.backward(Y, y_idx=idx, loss=loss, fused=SGD(lr, cfg.momentum, cfg.weight_decay))
        else:
            model.backward(Y, y_idx=idx, loss=loss, fused=None)
            if world > 1:
                overlap()
            else:
                overlap(reduce=lambda t: None)               # one rank: the identity, same streams / events
            model.step(SGD(lr, cfg.momentum, cfg.weight_decay, 1.0 / world))

    for s in range(args.warmup):
        one_step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    use_graph = args.graph in ("on", "auto")
    graph_note = None
    if use_graph:
        # C1-C4 steps last ~0.1-0.3 ms: replay G captured steps per CUDA graph; the
        # step's sample indices go to a fixed window and the dropout step to a device counter before
        # every replay (both inside the timed region)
        G = max(d for d in range(1, 9) if args.steps % d == 0)
        idx_win = torch.zeros(G * B, dtype=torch.int32, device=device)
        counter = torch.zeros(1, dtype=torch.int64, device=device)
        model.sparse_mlp_set_step_counter(counter)
        # the DP path replays with the post-warmup learning rate K eta (R20: the warmup is a
        # schedule of the same kernels)
        lr_g = scaled_lr(cfg.lr, world, warm_steps, warm_steps) if dp_path else cfg.lr
        sgd_g = SGD(lr_g, cfg.momentum, cfg.weight_decay, 1.0 / world if dp_path else 1.0)
        cap_stream = torch.cuda.Stream(device=device)
        cap_stream.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        l_cap0 = model.info()["launches"]
        with torch.cuda.stream(cap_stream):
            with torch.cuda.graph(graph, stream=cap_stream):
                for k in range(G):
                    iw = idx_win[k * B:(k + 1) * B]
                    model.forward(X, x_idx=iw, train=True, step=0)
                    if not dp_path:
                        model.backward(Y, y_idx=iw, loss=loss, fused=sgd_g)
                    else:   # unfused backward, bucketed allreduce on the side stream, Eq. 1 (1/K)
                        model.backward(Y, y_idx=iw, loss=loss, fused=None)
                        overlap() if world > 1 else overlap(reduce=lambda t: None)
                        model.step(sgd_g)
                    counter.add_(1)
                model.join()                                 # the library's side-stream work rejoins the capture
        torch.cuda.current_stream().wait_stream(cap_stream)
        launches_per_step = (model.info()["launches"] - l_cap0) / G
        torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = model.info()["launches"]
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0.record(stream)
    if use_graph:
        for r in range(args.steps // G):
            s0 = args.warmup + r * G
            idx_win.copy_(idx_all[s0 * B:(s0 + G) * B])
            counter.fill_(s0)
            graph.replay()
    else:
        for s in range(args.warmup, total_steps):
            one_step(s)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if use_graph:
        launches = int(round(launches_per_step * args.steps))
        model.sparse_mlp_set_step_counter(None)
    else:
        launches = model.info()["launches"] - launches0
    # per-kernel times: the same number of steps again, eager, with the library's event pair around
    # every launch (the events cost ~3% of a C5 step, so they stay out of the headline region)
    torch.cuda.synchronize()
    model.sparse_mlp_profile(True)
    evp0, evp1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evp0.record(stream)
    for s in range(args.steps):
        one_step(args.warmup + s)
    evp1.record(stream)
    torch.cuda.synchronize()
    ms_prof = evp0.elapsed_time(evp1) / args.steps
    prof = model.sparse_mlp_profile_read()
    model.sparse_mlp_profile(False)
    profiled_steps = args.steps
    if use_graph:
        graph_note = f"timed region: {args.steps // G} CUDA-graph replays of {G} steps (no per-kernel events)"
    clk = clocks.stop()
    t_ms = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms = float(t_ms.item())
    ms_per_step = ms / args.steps
    value = B * world * args.steps / (ms / 1e3)

    # ---------------------------------------------------------------- roofline of the dominant kernel
    peak, peak_src = _peaks()
    dom = max(prof, key=lambda r: r["total_ms"]) if prof else None
    roof = None
    if dom:
        avg_ms = dom["total_ms"] / dom["launches"]
        achieved = dom["bytes_per_launch"] / (avg_ms * 1e-3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:
                T = json.load(open(tpath))
                traffic = T.get(cfg.name, {}).get(f"{dom['kernel']}:{dom['layer']}")
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": f"{dom['kernel']} W^({dom['layer']})", "avg_launch_ms": round(avg_ms, 4),
                "algorithmic_bytes_per_launch": dom["bytes_per_launch"], "peak_source": peak_src}
    # second ceiling: L2 -> SM random-row gathers (profiles/gather_ceiling.json, measured on the box)
    roof_g = None
    gpath = os.path.join(ROOT, "profiles", "gather_ceiling.json")
    if prof and os.path.exists(gpath):
        try:
            GC = json.load(open(gpath))
            gpeak = float(GC["ceiling_GBps"])
            per = []
            step_gb = 0.0
            bits2 = any(r["kernel"] == "fwd_bits" for r in prof)
            for r in prof:
                gb = gathered_bytes(r, cfg.sizes, nnz, info0["chunk_batch"], info0["fwd_chunk_batch"], bits2,
                                    bool(info0.get("implicit_delta")))
                if gb <= 0:
                    continue
                avg = r["total_ms"] / r["launches"]
                step_gb += gb * r["launches"] / profiled_steps
                per.append({"kernel": f"{r['kernel']} W^({r['layer']})", "gathered_bytes_per_launch": gb,
                            "avg_launch_ms": round(avg, 4), "achieved_GBps": round(gb / (avg * 1e-3) / 1e9, 1),
                            "frac": round(gb / (avg * 1e-3) / 1e9 / gpeak, 4)})
            if per:
                ach = step_gb / (ms_per_step * 1e-3) / 1e9
                roof_g = {"bound": "l2_gather", "peak": gpeak, "unit": "GB/s",
                          "peak_source": "profiles/gather_ceiling.json (tools/gather_ceiling.py, sm clock median "
                                         f"{GC.get('clocks', {}).get('sm_mhz_median')} MHz)",
                          "gathered_bytes_per_step": step_gb, "achieved_step_GBps": round(ach, 1),
                          "frac_step": round(ach / gpeak, 4), "kernels": per}
        except Exception as e:  # reported, not fatal
            roof_g = {"bound": "l2_gather", "error": str(e)}
    step_bytes = f1_bytes(cfg.sizes, nnz, B)
    step_roof = {"bytes_per_step_F1": step_bytes, "achieved_GBps": round(step_bytes / (ms_per_step * 1e-3) / 1e9, 1),
                 "frac": round(step_bytes / (ms_per_step * 1e-3) / 1e9 / peak, 4)}

    # ---------------------------------------------------------------- epoch-boundary ops (evolve / prune)
    epoch = None
    if not args.no_epoch:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if cfg.prune:
            model.prune_neurons(cfg.prune_percentile)
        model.evolve_topology(cfg.zeta, 0)
        torch.cuda.synchronize()
        t_ev = time.perf_counter() - t0
        steps_per_epoch = math.ceil(cfg.n_samples / (B * world))
        epoch = {"evolve_s": round(t_ev, 4), "steps_per_epoch": steps_per_epoch,
                 "epoch_samples_per_s_incl_evolve": cfg.n_samples / (steps_per_epoch * ms_per_step / 1e3 + t_ev),
                 "replicas_identical": bool(replicas_identical(model.param_view()[0])) if world > 1 else True}

    # ---------------------------------------------------------------- end to end through the host-buffer API
    e2e = None
    if not args.no_e2e:
        nb = 4
        if cfg.binary_input:
            from synth.data import c5_host_rows
            Xh, Yh = c5_host_rows(cfg, np.arange(rank * nb * B, (rank + 1) * nb * B))
        else:
            Xh = X[: nb * B].cpu().numpy()
            Yh = Y[: nb * B].cpu().numpy()
        xp = torch.from_numpy(Xh).pin_memory()
        yp = torch.from_numpy(Yh.astype(np.int32)).pin_memory()
        k2 = max(3, min(args.steps, 10))
        lossp = torch.zeros(k2 + 2, dtype=torch.float32).pin_memory()
        sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
        if dp_path:
            # N > 1: the synchronous DP step from host buffers -- H2D of x / y (pinned, on the
            # stream), forward, unfused backward, overlapped per-layer allreduce, Eq. 1, loss D2H
            xd = torch.empty((B, cfg.sizes[0]), dtype=torch.float32, device=device)
            yd = torch.empty(B, dtype=torch.int32, device=device)
            ld = torch.zeros(1, dtype=torch.float32, device=device)

            def host_step(j, step_idx, slot):
                xd.copy_(xp[j * B:(j + 1) * B], non_blocking=True)
                yd.copy_(yp[j * B:(j + 1) * B], non_blocking=True)
                model.forward(xd, train=True, step=step_idx)
                model.backward(yd, loss=ld, fused=None)
                if world > 1:
                    overlap()
                else:
                    overlap(reduce=lambda t: None)
                model.step(SGD(cfg.lr, cfg.momentum, cfg.weight_decay, 1.0 / world))
                lossp[slot:slot + 1].copy_(ld, non_blocking=True)
        else:
            def host_step(j, step_idx, slot):
                model.train_step_host_async(xp[j * B:(j + 1) * B], yp[j * B:(j + 1) * B], B, step_idx, sgd,
                                            lossp[slot:])
        for s in range(2):
            host_step(s, 10_000 + s, s)
        model.sync()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # every step: H2D of its x / y from pinned host memory (1 GPU: on a copy stream, overlapping
        # the previous step's compute), forward, backward + update, D2H of its loss; all timed
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(k2):
            host_step(s % nb, 20_000 + s, 2 + s)
        e1.record(stream)
        model.sync()
        torch.cuda.synchronize()
        assert np.all(np.isfinite(lossp.numpy()[2:2 + k2])), "e2e losses"
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": B * world * k2 / (float(et.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": B * cfg.sizes[0] * 4 + B * 4, "d2h_bytes_per_step": 4,
               "api": ("pinned host x, y -> device, forward, unfused backward, overlapped per-layer allreduce, "
                       "Eq. 1 step, loss -> pinned host" if dp_path else
                       "sparse_mlp_train_step_host_async (pinned host x, y -> device on a copy stream "
                       "overlapping the previous step, fwd, fused bwd, loss -> pinned host)")}

    # cpu_baseline (the oracle on the host cores), rank 0 at N = 1 only, after every GPU-timed
    # region: one full C5 step at the bench batch (B = 128) + one SET evolution; 20 steps otherwise
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import concurrent.futures as cf
        import multiprocessing as mp
        try:
            with cf.ProcessPoolExecutor(1, mp_context=mp.get_context("spawn")) as ex:
                cpu = ex.submit(cpu_baseline_job, cfg.name, B, 1 if cfg.binary_input else 20,
                                bool(cfg.binary_input)).result(timeout=1500)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {**config_dict(cfg, world),
                           "step_path": "dp: unfused bwd + per-layer overlapped allreduce + Eq.1 kernel" if dp_path
                           else "1 GPU: sparse_mlp_backward with SGD (gradient, then the streaming Eq.1 pass "
                           "and mirror refresh inside the same call)",
                           "nnz": sum(nnz), "chunk_batch": info0["chunk_batch"],
                           "fwd_chunk_batch": info0["fwd_chunk_batch"],
                           "l2_flush": "inputs larger than L2 (resident shard "
                           f"{X.numel() * 4 / 1e9:.1f} GB; per-step traffic {step_bytes / 1e9:.2f} GB)",
                           "create_s": round(t_create, 2), "cuda_graph": graph_note},
                "roofline": roof, "step_roofline": step_roof, "roofline_l2_gather": roof_g,
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk, "epoch": epoch, "profiled_steps": profiled_steps,
                "ms_per_step_profiled": round(ms_prof, 4),
                "kernels": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()} for r in prof]}
        print(json.dumps(line), flush=True)
        if args.profile_json:
            with open(args.profile_json, "w") as f:
                json.dump(line, f, indent=1)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
