"""CPU float64 oracle for the attention-template hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy float64, the reference algorithms of attnforge (AttentionEngine,
arXiv 2502.15349) that the sm_100a kernels replace.  Each function cites the reference file:line it
follows.  It exists to *check* the CUDA path: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it.  The product package
(``paper_2502_15349_b200``) never imports this package and has no CPU fallback.

Parity pinning: ``tests/golden/*.npz`` hold outputs of the reference itself (run in the build
container by ``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks this oracle
against every fixture, ``tests/test_oracle_reference.py`` re-runs the live reference when ``/root/reference`` is mounted,
and ``tests/test_oracle_gradcheck.py`` checks the closed-form VJPs against central differences.

Modules
  hooks      hook expressions evaluated on numpy arrays, with dual numbers for elementwise
             derivatives following the reference adjoint rules (graph.py:481-569)
  fills      deterministic problem instances (engine.py:326-388)
  parallel   parallel template: tiled online forward, dense forward, LSE, closed-form VJP
  recurrent  linear template: stepwise / chunked forward, chunked VJP
  gradcheck  central finite-difference check of the VJPs (engine.finite_diff_check restated)
"""

from .fills import generate, philox_key  # noqa: F401
from .parallel import (tiled_forward, naive_forward, forward_with_lse, parallel_vjp,  # noqa: F401
                       lse_rows)
from .recurrent import step_forward, chunk_forward, chunk_vjp  # noqa: F401
