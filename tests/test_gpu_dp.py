"""K >= 2 data-parallel parity of the CUDA path on ONE B200 (
WASSP phase 1 PAPER.md:320-323, Alg. 1; Eq. 2; phase-2 union
averaging PAPER.md:616-629).

K processes share cuda:0, each holding its own library replica (same seed -> same ER topology and
values; its rank in the dropout stream), joined by a gloo process group over the CUDA views (NCCL
refuses two ranks on one device; the collectives are host-side, so no rank's kernel waits on
another's).  Every process also runs the K-rank oracle (oracle/dp.py) on the same seeded batches
and checks, after every step:

* the synchronous step -- per-rank forward + unfused backward, SUM allreduce of the grad view
  (plain dp_train_step, or OverlappedAllreduce: per-layer slices released by the library's layer
  events to a side stream), Eq. 1 with grad_scale 1/K and the warmup-scaled learning rate (R20) --
  against oracle.dp.dp_step within R24 (1e-4 + the fp32 error bound), and the K replicas
  bit-identical (replicas_identical, the X3 hash all-gather);
* Eq. 2 averaging after K divergent local steps (dp.average_model_: SUM allreduce +
  sparse_mlp_params_averaged) against oracle.dp.average;
* phase-2 union averaging (dp.union_average_: all-gather of every replica's (position, value)
  lists, padded) after rank-specific evolutions, bit-exact against oracle.dp.average_union.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _kink_free_batches(st, X, Y, B, K, step, start):
    """K batches (one per rank, in rank order) that the oracle finds kink-free (R32) on state st,
    taken in order from the candidate pool starting at slice `start`; returns (batches, next)."""
    from oracle import model as M
    out, t = [], start
    for k in range(K):
        while True:
            assert (t + 1) * B <= len(X), "no kink-free batch among the candidates"
            x, y = X[t * B:(t + 1) * B], Y[t * B:(t + 1) * B]
            t += 1
            if sum(M.forward(st, x, True, step, rank=k).ambiguous) == 0:
                out.append((x, y))
                break
    return out, t


def _worker(rank, K, port, mode, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(K),
                          LOCAL_RANK="0")
        torch.cuda.set_device(0)
        from oracle import dp as ODP
        from oracle import model as M
        from oracle import topology as T
        from paper_2102_01732_b200 import SGD, SparseMLP
        from paper_2102_01732_b200 import dp as D
        from synth import get_config, make_dataset
        from tests.gpu_helpers import (TOL, assert_topology_equal, assert_values_close, load_oracle_state_into_gpu,
                                       to_dev)
        D.init_process_group(backend="gloo")
        assert dist.get_world_size() == K and dist.get_rank() == rank
        cfg = get_config("C1", dropout=0.2, n_samples=8000)
        B = cfg.batch
        g = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed,
                      rank, B)
        st = M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed)
        X, Y = make_dataset(cfg, n=8000)        # candidate pool: (3 + 1) x K kink-free batches
        ov = D.OverlappedAllreduce(g) if mode == "overlap" else None
        nxt = 0
        # ---- synchronous steps (WASSP phase 1)
        for s in range(3):
            lr = D.scaled_lr(cfg.lr * 10, K, s, 2)
            batches, nxt = _kink_free_batches(st, X, Y, B, K, s, nxt)
            ODP.dp_step(st, batches, lr, cfg.momentum, cfg.weight_decay, s)
            x, y = batches[rank]
            if ov is None:
                D.dp_train_step(g, to_dev(x), to_dev(y.astype(np.int32)), None, s, lr, cfg.momentum,
                                cfg.weight_decay, K)
            else:
                D.dp_train_step_overlapped(g, to_dev(x), to_dev(y.astype(np.int32)), None, s, lr, cfg.momentum,
                                           cfg.weight_decay, K, ov)
            torch.cuda.synchronize()
            assert_values_close(g, st, TOL, f"rank {rank} step {s}")
            p, _ = g.param_view()
            assert D.replicas_identical(p), f"replicas differ after step {s}"
            load_oracle_state_into_gpu(g, st)        # the next step from identical inputs (per-step parity)
        # ---- Eq. 2 averaging after divergent local steps (phase 2 without a per-step collective)
        states = [st.copy() for _ in range(K)]
        for k in range(K):                       # replica k draws the dropout stream of rank k
            states[k].rank = k
        batches, nxt = _kink_free_batches(st, X, Y, B, K, 3, nxt)
        sgd = SGD(cfg.lr * 10, cfg.momentum, cfg.weight_decay)
        for k in range(K):
            M.train_step(states[k], batches[k][0], batches[k][1], sgd.lr, sgd.momentum, sgd.weight_decay, 3)
        x, y = batches[rank]
        g.forward(to_dev(x), train=True, step=3)
        g.backward(to_dev(y.astype(np.int32)), fused=sgd)
        torch.cuda.synchronize()
        assert_values_close(g, states[rank], TOL, f"rank {rank} local step")
        for k in range(K):                       # Eq. 2 compared op by op: every replica's exact
            if k != rank:                        # pre-average state is the oracle's own
                states[k].reset_error()
        ODP.average(states)
        D.average_model_(g)
        torch.cuda.synchronize()
        for Ly in states[rank].layers:          # momentum stays local: compare w and b only
            Ly.vmag = None
        assert_values_close(g, _without_v(states[rank]), TOL, f"rank {rank} Eq. 2 average")
        p, _ = g.param_view()
        assert D.replicas_identical(p), "replicas differ after averaging"
        # the averaged model still trains (mirror copy refreshed by the library)
        x, y = X[-B:], Y[-B:]
        g.forward(to_dev(x), train=True, step=4)
        g.backward(to_dev(y.astype(np.int32)), fused=sgd)
        torch.cuda.synchronize()
        # ---- phase-2 union averaging after rank-specific evolutions (bit-exact, R31)
        gs = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, 0.0, cfg.init, cfg.model_seed, rank, B)
        ost = [M.create(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, 0.0, cfg.init, cfg.model_seed)
               for _ in range(K)]
        targets = [Ly.nnz for Ly in ost[0].layers]
        gs.evolve_topology(cfg.zeta, 100 + rank)
        for k in range(K):
            T.evolve(ost[k], cfg.zeta, 100 + k)
        kept = D.union_average_(gs, targets)
        kept_o = ODP.average_union(ost, targets)
        torch.cuda.synchronize()
        assert kept == kept_o, (kept, kept_o)
        assert_topology_equal(gs, ost[0], f"rank {rank} union average")
        for Ly in ost[0].layers:
            e = gs.export_layer(Ly.l)
            assert np.array_equal(e["w"].view(np.uint32), Ly.w.view(np.uint32)), Ly.l
            assert not np.any(e["v"])
        for l in range(2, cfg.n_layers + 1):
            b, _ = gs.sparse_mlp_export_bias(l)
            assert np.array_equal(b, ost[0].b[l - 2])
        q.put((rank, {"ok": True}))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # surfaced by the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))


def _without_v(st):
    """A copy of st whose momenta are all zero (assert_values_close skips v when it is zero):
    Eq. 2 averages (w, b); each replica keeps its own momentum."""
    s = st.copy()
    for Ly in s.layers:
        Ly.v = np.zeros_like(Ly.v)
    return s


@pytest.mark.parametrize("K,mode", [(2, "plain"), (2, "overlap"), (4, "plain")])
def test_dp_k_ranks_on_one_gpu_match_the_oracle(K, mode):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, K, port, mode, q)) for r in range(K)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(K))
    for p in ps:
        p.join(timeout=120)
    errs = {r: out[r]["error"] for r in range(K) if "error" in out[r]}
    # a rank whose peer failed first only reports the closed connection: show the root cause first
    root = sorted(errs.items(), key=lambda kv: "Connection closed" in kv[1])
    assert not errs, "\n".join(f"rank {r}: {e}" for r, e in root)
    assert all(out[r]["ok"] for r in range(K))


def _graph_worker(port, q):
    """One NCCL rank (world size 1: the collective is a real NCCL launch) -- the DP step (forward,
    unfused backward, bucketed OverlappedAllreduce on its side stream, Eq. 1 with 1/K) captured in
    ONE CUDA graph with its NCCL collectives, replayed, and compared bit for bit with the same
    steps run eagerly on a second replica."""
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        torch.cuda.set_device(0)
        from paper_2102_01732_b200 import SGD, SparseMLP
        from paper_2102_01732_b200 import dp as D
        from synth import get_config, make_dataset
        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
        cfg = get_config("C1", dropout=0.2)
        B = cfg.batch
        X, Y = make_dataset(cfg, n=4 * B)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y.astype(np.int32)).cuda()
        idx = torch.arange(4 * B, dtype=torch.int32, device="cuda")
        sgd = SGD(cfg.lr * 5, cfg.momentum, cfg.weight_decay, 1.0)
        mk = lambda: SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init,
                               cfg.model_seed, 0, B)
        ge, gg = mk(), mk()
        ove, ovg = D.OverlappedAllreduce(ge), D.OverlappedAllreduce(gg)
        assert len(ovg.buckets) == 1                      # C1's 0.08 MB view: one collective per step

        def step(g, ov, iw, s):
            g.forward(Xd, x_idx=iw, train=True, step=s)
            g.backward(Yd, y_idx=iw, fused=None)
            ov()
            g.step(sgd)

        for s in range(2):                                # eager warm-up of both (NCCL communicator up)
            step(ge, ove, idx[s * B:(s + 1) * B], s)
            step(gg, ovg, idx[s * B:(s + 1) * B], s)
        torch.cuda.synchronize()
        win = torch.zeros(B, dtype=torch.int32, device="cuda")
        counter = torch.zeros(1, dtype=torch.int64, device="cuda")
        gg.sparse_mlp_set_step_counter(counter)
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cs):
            with torch.cuda.graph(graph, stream=cs):
                step(gg, ovg, win, 0)
                gg.join()
        torch.cuda.current_stream().wait_stream(cs)
        for s in range(2, 4):
            win.copy_(idx[s * B:(s + 1) * B])
            counter.fill_(s)
            graph.replay()
            step(ge, ove, idx[s * B:(s + 1) * B], s)
        torch.cuda.synchronize()
        gg.sparse_mlp_set_step_counter(None)
        pe, _ = ge.param_view()
        pg, _ = gg.param_view()
        assert torch.equal(pe.view(torch.int32), pg.view(torch.int32)), "graph replay differs from eager"
        q.put({"ok": True})
        dist.destroy_process_group()
    except BaseException as e:  # surfaced by the parent
        import traceback
        q.put({"error": traceback.format_exc() + repr(e)})


def test_dp_step_with_nccl_collectives_in_a_cuda_graph():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_graph_worker, args=(_free_port(), q))
    p.start()
    out = q.get(timeout=600)
    p.join(timeout=120)
    assert "error" not in out, out.get("error")
