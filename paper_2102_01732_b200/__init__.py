"""paper_2102_01732_b200 — B200-native hot path of truly sparse MLP training (arXiv 2102.01732).

SET topology evolution + All-ReLU + Importance Pruning, as sm_100a CUDA kernels behind the C ABI
of ``include/sparse_mlp.h`` (``lib/libsparse_mlp.so``).  This package is the thin Python side:

  sparse_mlp.py   ctypes binding (argument marshalling only; same names as the C ABI)
  trainer.py      epoch driver (minibatch loop, CUDA-graph capture, evolve / prune schedule)
  dp.py           synchronous data parallelism over torch.distributed (NCCL on B200s)
  build.py        nvcc build of the library for sm_100a

There is no CPU fallback: importing ``sparse_mlp`` fails loudly if the library is not built.
"""
from .sparse_mlp import SGD, SparseMLP, SparseMLPError, from_config, load_library  # noqa: F401

__all__ = ["SGD", "SparseMLP", "SparseMLPError", "from_config", "load_library"]
