"""The N > 1 host path (paper_2102_01732_b200/dp.py) with a real torch.distributed process group:
world_size 2 over gloo on CPU.  Each rank is a separate process.

Checked per rank, on the same seeded inputs:
* shard_bounds partitions the sample range exactly (no overlap, no gap);
* allreduce_sum_ is the SUM over ranks;
* replicas_identical (the X3 hash allgather) is true for identical replicas and false as soon as
  one bit differs on one rank;
* a synchronous DP step wired exactly like bench.py / trainer.py (per-rank gradient of the local
  batch -> allreduce_sum_ of the flat grad view -> Eq. 1 with grad_scale 1/K) reproduces the
  single-process K-rank oracle step (oracle/dp.py), and leaves both replicas bit-identical.
The per-rank model here is the oracle (tests may use it); the CUDA library runs the same host path
with K = 2 and K = 4 ranks on one GPU in tests/test_gpu_dp.py (step, Eq. 2 averaging, union
averaging, against oracle/dp.py).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _flat(gr):
    return np.concatenate([g.ravel() for g in gr.g] + [g.ravel() for g in gr.gb]).astype(np.float32)


def _unflat(vec, like):
    out_g, out_gb, o = [], [], 0
    for g in like.g:
        out_g.append(vec[o:o + g.size].reshape(g.shape).astype(np.float32))
        o += g.size
    for g in like.gb:
        out_gb.append(vec[o:o + g.size].reshape(g.shape).astype(np.float32))
        o += g.size
    return out_g, out_gb


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                          LOCAL_RANK=str(rank))
        from oracle import dp as ODP
        from oracle import model as M
        from paper_2102_01732_b200 import dp as D
        r, w, _ = D.init_process_group(backend="gloo")
        assert (r, w) == (rank, world) and dist.get_backend() == "gloo"
        res = {}
        # shard bounds
        n = 1001
        lo, hi = D.shard_bounds(n, rank, world)
        got = [None] * world
        dist.all_gather_object(got, (lo, hi))
        res["shards"] = got
        # allreduce / average
        t = torch.arange(6, dtype=torch.float32) * (rank + 1)
        D.allreduce_sum_(t)
        res["sum"] = t.numpy().copy()
        # replica identity
        v = torch.linspace(-1, 1, 257)
        res["ident_same"] = D.replicas_identical(v)
        v2 = v.clone()
        if rank == 1:
            v2[100] = torch.nextafter(v2[100], torch.tensor(2.0))
        res["ident_diff"] = D.replicas_identical(v2)
        # one synchronous DP step through the dp.py plumbing, per-rank model = the oracle
        st = M.create((16, 12, 10, 3), 2.0, "all_relu", 0.5, 0.2, "he_uniform", 7)
        rng = np.random.default_rng(3)
        batches = [(rng.standard_normal((6, 16)).astype(np.float32), rng.integers(0, 3, 6)) for _ in range(world)]
        x, y = batches[rank]
        lr = D.scaled_lr(0.05, world, 5, 10)
        tr = M.forward(st, x, True, 0, rank=rank)
        gr = M.backward(st, tr, y)
        g = torch.from_numpy(_flat(gr))
        D.allreduce_sum_(g)                                  # X1: SUM of the grad views
        gg, ggb = _unflat(g.numpy(), gr)
        M.step(st, M.Grads(gg, ggb, gr.loss, gr.deltas), lr, 0.9, 1e-4, grad_scale=1.0 / world)
        ref = M.create((16, 12, 10, 3), 2.0, "all_relu", 0.5, 0.2, "he_uniform", 7)
        ODP.dp_step(ref, batches, lr, 0.9, 1e-4, 0)
        res["dp_err"] = max(float(np.max(np.abs(a.w - b.w))) for a, b in zip(st.layers, ref.layers))
        wv = torch.from_numpy(np.concatenate([L.w for L in st.layers]))
        res["dp_identical"] = D.replicas_identical(wv)
        q.put((rank, res))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surfaced by the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc() + str(e)}))


def test_dp_plumbing_world_size_2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in out[r], out[r].get("error")
    # shards: [0, 500), [500, 1001)
    assert out[0]["shards"] == [(0, 500), (500, 1001)]
    for r in range(world):
        assert np.array_equal(out[r]["sum"], np.arange(6, dtype=np.float32) * 3)
        assert out[r]["ident_same"] is True
        assert out[r]["ident_diff"] is False
        # the DP step equals the K-rank oracle step (summation order of the K = 2 gradients may
        # differ by one rounding: fp32 gloo SUM vs the oracle's fp64 sum rounded once)
        assert out[r]["dp_err"] < 1e-6
        assert out[r]["dp_identical"] is True


@pytest.mark.parametrize("bucket_bytes", [1, 4 << 20, 100 << 20, 1 << 40])
def test_overlapped_allreduce_buckets_cover_the_view_once(bucket_bytes):
    """OverlappedAllreduce.plan (host logic): the buckets are disjoint slices covering the whole
    grad view [0, param_count) exactly once, issued output layer first; a bucket waits for the
    lowest layer it holds; every bucket but the one reaching W^(2) holds >= bucket_bytes."""
    from paper_2102_01732_b200.dp import OverlappedAllreduce
    for caps in ([10304, 20000, 20000, 2016], [11310720, 20000000, 20000000, 1000000], [9000, 5000, 5000, 800]):
        L = len(caps) + 1
        layout, off = [], 0
        for c in caps:
            layout.append((off, c))
            off += (c + 31) // 32 * 32
        bias_base, total = off, off + 1000
        plan = OverlappedAllreduce.plan(layout, bias_base, L, bucket_bytes)
        cover = np.zeros(total, np.int32)
        for l, lo, hi in plan:
            cover[lo:(total if hi is None else hi)] += 1
        assert cover.max() == 1                           # disjoint
        for off_l, c in layout:                           # every value of every layer, once
            assert cover[off_l:off_l + c].min() == 1
        assert cover[bias_base:].min() == 1               # and the bias block
        waits = [l for l, _, _ in plan]
        assert waits == sorted(waits, reverse=True) and waits[-1] == 2
        for l, lo, hi in plan[:-1]:
            if l > 2 and hi is not None:
                assert 4 * (hi - lo) >= bucket_bytes
        if bucket_bytes >= 4 * total:
            assert plan == [(2, 0, None)]                # one collective of the whole view
