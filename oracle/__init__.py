"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct NumPy implementation of what the truly-sparse
SET-MLP training step computes (arXiv 2102.01732, /root/reference/PAPER.md),
written from the paper before any CUDA kernel existed.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it.  The product path (``paper_2102_01732_b200``)
never imports, calls or links anything here, and the oracle never imports the
product package; the two share no code.  The only shared module is ``synth``
(seeded inputs, no arithmetic of the method).

Modules (function names mirror the C-ABI so lockstep tests pair calls 1:1):
  philox.py    Philox4x32-10 (Salmon et al. 2011, Random123) and the stream layout
  model.py     create (ER init), forward, loss_grad, backward, step
  topology.py  evolve (SET prune/regrow), importance (Eq. 4), prune (Alg. 2)
  dp.py        K-rank synchronous data parallelism, model averaging (Eq. 2)
  compare.py   the comparison metric used by the parity tests

Precision: state (w, v, b) is float32, the paper's precision ("adopting 32-bit
float precision"); every stored tensor is computed in float64 and
rounded once to float32.  Topology arithmetic is integer / IEEE-bit based.

Parity pins: every function is pinned in tests/test_oracle_*.py against
something other than itself (closed forms, published Philox vectors, a dense
masked MLP, finite differences, brute force, SPEC worked examples).  Functions
with no such pin are listed as "parity unpinned" in DESIGN.md:
  * the regrowth / ER *positions* (the RNG layout is this build's own spec;
    pinned only structurally: counts, distinctness, exclusions, brute force).
"""
