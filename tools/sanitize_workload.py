"""Workload for compute-sanitizer: every kernel family of the
library on small shapes -- C1 (fwd rows, narrow output layer, fused step, evolve, prune), a
long-row / dense-capped layer with mixed chunk widths (multi-segment rows + finish kernels,
cp.async windows), eps = 1 short rows (row-streaming kernels), the binary-input bit path, the
union average and RetainValidUpdates.  Run by tools/sanitize.sh under each sanitizer tool."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2102_01732_b200 import SGD, SparseMLP  # noqa: E402
from synth import get_config, make_dataset  # noqa: E402


def run(g, X, Y, B, steps=2, sgd=SGD(0.01, 0.9, 2e-4)):
    for s in range(steps):
        x, y = X[s * B:(s + 1) * B], Y[s * B:(s + 1) * B]
        g.forward(torch.from_numpy(x).cuda(), train=True, step=s)
        g.backward(torch.from_numpy(y.astype(np.int32)).cuda(), fused=sgd)
    g.forward(torch.from_numpy(X[:B]).cuda(), train=True, step=9)
    g.backward(torch.from_numpy(Y[:B].astype(np.int32)).cuda())
    g.step(sgd)
    torch.cuda.synchronize()


def main():
    torch.cuda.set_device(0)
    cfg = get_config("C1", dropout=0.2)
    g = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed, 0, 128)
    X, Y = make_dataset(cfg, n=384)
    run(g, X, Y, 128)
    g.prune_neurons(10.0)
    g.evolve_topology(0.3, 0)
    run(g, X, Y, 128)
    pos, val = g.export_positions(3)
    g.union_average_layer(3, 1, pos, val, len(pos) - 10)
    # long rows + dense-capped layer, mixed chunk widths (64 backward / 32 forward), ragged batch
    os.environ["SMLP_FWD_CB"] = "32"
    c2 = get_config("C1", sizes=(30, 200, 150, 10), epsilon=40.0, alpha=0.6, dropout=0.3, batch=100)
    g2 = SparseMLP(c2.sizes, c2.epsilon, c2.activation, c2.alpha, c2.dropout, c2.init, 5, 0, 100, 64)
    rng = np.random.default_rng(1)
    X2 = rng.standard_normal((300, 30)).astype(np.float32)
    Y2 = rng.integers(0, 10, 300)
    run(g2, X2, Y2, 100)
    del os.environ["SMLP_FWD_CB"]
    # eps = 1: short rows, the row-streaming kernels
    os.environ["SMLP_SHORT_MIN_ROWS"] = "0"
    c3 = get_config("C1", sizes=(30, 600, 500, 10), epsilon=1.0, alpha=0.6, dropout=0.2, batch=128)
    g3 = SparseMLP(c3.sizes, c3.epsilon, c3.activation, c3.alpha, c3.dropout, c3.init, 6, 0, 128, 128)
    X3 = rng.standard_normal((384, 30)).astype(np.float32)
    Y3 = rng.integers(0, 10, 384)
    run(g3, X3, Y3, 128)
    del os.environ["SMLP_SHORT_MIN_ROWS"]
    # binary inputs: the bit path of W^(2)
    c4 = get_config("C1", sizes=(300, 400, 350, 2), epsilon=10.0, alpha=0.5, dropout=0.0, batch=128)
    g4 = SparseMLP(c4.sizes, c4.epsilon, c4.activation, c4.alpha, c4.dropout, c4.init, 7, 0, 128, 0, input_kind=2)
    X4 = (rng.random((384, 300)) < 0.05).astype(np.float32)
    Y4 = rng.integers(0, 2, 384)
    run(g4, X4, Y4, 128)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
