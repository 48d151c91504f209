"""The persistent step: for models of <= 4M parameters every forward / backward call
is ONE cooperative launch that runs the call's kernels as phases of a persistent kernel, separated
by grid-wide barriers, calling the same device bodies with the same virtual grids as the
per-kernel launches.  The two paths must therefore agree BIT FOR BIT -- every weight, momentum,
bias and loss -- through fused and unfused steps, dropout, the binary-input bit path, SET
evolution and importance pruning, and inside a CUDA graph.  (The per-kernel path's agreement with
the oracle is what the rest of the GPU suite checks; the persistent path is opt-in, SMLP_PERSIST=1,
because it measured slower than the CUDA-graph replay of the per-kernel step -- DESIGN.md §5.)
"""
import numpy as np
import pytest

from synth import get_config, make_dataset
from tests.gpu_helpers import to_dev

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _model(cfg, monkeypatch, persist, input_kind=0, max_batch=None):
    from paper_2102_01732_b200 import SparseMLP
    monkeypatch.setenv("SMLP_PERSIST", "1" if persist else "0")
    g = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed, 0,
                  max_batch or cfg.batch, input_kind=input_kind)
    monkeypatch.delenv("SMLP_PERSIST")
    return g


def _state(g, L):
    out = []
    for l in range(2, L + 1):
        e = g.export_layer(l)
        b, vb = g.sparse_mlp_export_bias(l)
        out.append((e["row_ptr"], e["col"], e["w"].view(np.uint32), e["v"].view(np.uint32),
                    np.asarray(b).view(np.uint32), np.asarray(vb).view(np.uint32)))
    return out


def _assert_same(a, b, what):
    for l, (x, y) in enumerate(zip(a, b)):
        for k, (u, v) in enumerate(zip(x, y)):
            assert np.array_equal(u, v), (what, l + 2, k)


def _binary_small():
    return get_config("C1", sizes=(300, 400, 350, 2), epsilon=10.0, alpha=0.5, dropout=0.2, init="he_uniform",
                      batch=128)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "binary"])
def test_persistent_matches_per_kernel_bitwise(name, monkeypatch):
    from paper_2102_01732_b200 import SGD
    torch = _torch()
    cfg = _binary_small() if name == "binary" else get_config(name)
    B = cfg.batch
    if name == "binary":
        rng = np.random.default_rng(7)
        X = (rng.random((8 * B, cfg.sizes[0])) < 0.05).astype(np.float32)
        Y = rng.integers(0, 2, size=8 * B).astype(np.int32)
    else:
        X, Y = make_dataset(cfg, n=8 * B)
        Y = Y.astype(np.int32)
    gp, gk = _model(cfg, monkeypatch, True), _model(cfg, monkeypatch, False)
    sgd = SGD(cfg.lr * 5, cfg.momentum, cfg.weight_decay)
    lp, lk = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")

    def fused(s):
        x, y = to_dev(X[s * B:(s + 1) * B]), to_dev(Y[s * B:(s + 1) * B])
        n0 = gp.info()["launches"]
        gp.forward(x, train=True, step=s)
        gp.backward(y, loss=lp, fused=sgd)
        assert gp.info()["launches"] - n0 == 2          # one persistent launch per call
        gk.forward(x, train=True, step=s)
        gk.backward(y, loss=lk, fused=sgd)
        torch.cuda.synchronize()
        assert lp.cpu().numpy().view(np.uint32) == lk.cpu().numpy().view(np.uint32), (name, s, lp.item(), lk.item())

    for s in range(3):
        fused(s)
    _assert_same(_state(gp, cfg.n_layers), _state(gk, cfg.n_layers), "fused steps")
    # unfused backward (the K > 1 path) + Eq. 1 with grad_scale 1/2
    x, y = to_dev(X[3 * B:4 * B]), to_dev(Y[3 * B:4 * B])
    for g in (gp, gk):
        g.forward(x, train=True, step=3)
        g.backward(y, fused=None)
    gv_p, _ = gp.grad_view()
    gv_k, _ = gk.grad_view()
    torch.cuda.synchronize()
    assert torch.equal(gv_p.view(torch.int32), gv_k.view(torch.int32)), "unfused gradient view"
    half = SGD(cfg.lr, cfg.momentum, cfg.weight_decay, 0.5)
    gp.step(half)
    gk.step(half)
    # an epoch boundary: pruning (C3's schedule) and SET evolution, then more steps on the new topology
    if cfg.prune:
        assert gp.prune_neurons(cfg.prune_percentile) == gk.prune_neurons(cfg.prune_percentile)
    assert gp.evolve_topology(cfg.zeta, 0) == gk.evolve_topology(cfg.zeta, 0)
    for s in range(4, 7):
        fused(s)
    _assert_same(_state(gp, cfg.n_layers), _state(gk, cfg.n_layers), "after evolve")
    # inference forward (no dropout): the same logits
    for g in (gp, gk):
        g.forward(to_dev(X[7 * B:8 * B]), train=False, step=7)
    torch.cuda.synchronize()
    zp, zk = gp.sparse_mlp_export_trace(0, cfg.n_layers, B), gk.sparse_mlp_export_trace(0, cfg.n_layers, B)
    assert np.array_equal(zp.view(np.uint32), zk.view(np.uint32))


def test_persistent_step_in_cuda_graph(monkeypatch):
    """A CUDA graph of G persistent training steps (cooperative launches inside the capture, the
    sample window and the dropout-step counter on the device) replays the eager per-kernel steps
    bit for bit."""
    from paper_2102_01732_b200 import SGD
    torch = _torch()
    cfg = get_config("C2")
    B, G = cfg.batch, 3
    X, Y = make_dataset(cfg, n=(1 + 2 * G) * B)
    Xd, Yd = to_dev(X), to_dev(Y.astype(np.int32))
    idx = torch.arange((1 + 2 * G) * B, dtype=torch.int32, device="cuda")
    gp, gk = _model(cfg, monkeypatch, True, input_kind=1), _model(cfg, monkeypatch, False, input_kind=1)
    sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
    win = torch.zeros(G * B, dtype=torch.int32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    gp.forward(Xd, x_idx=idx[:B], train=True, step=0)          # first call at max_batch outside the capture
    gp.backward(Yd, y_idx=idx[:B], fused=sgd)
    gk.forward(Xd, x_idx=idx[:B], train=True, step=0)
    gk.backward(Yd, y_idx=idx[:B], fused=sgd)
    torch.cuda.synchronize()
    gp.sparse_mlp_set_step_counter(counter)
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    n0 = gp.info()["launches"]
    with torch.cuda.stream(cs):
        with torch.cuda.graph(graph, stream=cs):
            for k in range(G):
                iw = win[k * B:(k + 1) * B]
                gp.forward(Xd, x_idx=iw, train=True, step=0)
                gp.backward(Yd, y_idx=iw, fused=sgd)
                counter.add_(1)
            gp.join()
    torch.cuda.current_stream().wait_stream(cs)
    assert gp.info()["launches"] - n0 == 2 * G
    for r in range(2):
        s0 = 1 + r * G
        win.copy_(idx[s0 * B:(s0 + G) * B])
        counter.fill_(s0)
        graph.replay()
        for k in range(G):
            iw = win[k * B:(k + 1) * B].clone()
            gk.forward(Xd, x_idx=iw, train=True, step=s0 + k)
            gk.backward(Yd, y_idx=iw, fused=sgd)
    torch.cuda.synchronize()
    gp.sparse_mlp_set_step_counter(None)
    _assert_same(_state(gp, cfg.n_layers), _state(gk, cfg.n_layers), "graph replay")
