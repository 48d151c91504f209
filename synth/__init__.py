"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no forward, gradient, update,
topology or RNG-layout code).  It only defines the five workload configurations
(BASELINE.json ``configs``) and draws the stand-in datasets
with NumPy PCG64 (host) or a seeded torch generator (device, C5 only).
Both the oracle side and the CUDA side consume these inputs; neither side
imports the other.
"""
from .configs import CONFIGS, WorkloadConfig, get_config  # noqa: F401
from .data import make_dataset, make_batch_indices, c5_host_rows  # noqa: F401
