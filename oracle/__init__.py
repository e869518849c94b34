"""Float64 CPU oracle for Fast Ordering ICA (arXiv 2408.17118).

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s cpu_baseline / `--impl reference` legs may import it.  The
product path (paper_2408_17118_b200) never imports it and shares no code with
it; the only common module is `datagen/` (seeded input recipe, no method
arithmetic).

Forms (each cites the passage it follows):
  rng       counter-based N(0,1) candidate generator (readings A7/A8)
  contrast  alpha eq. (2), Upsilon eq. (1), Gaussianity threshold
  whiten    centring + PCA whitening (readings A11/A12)
  ordering  O1 batched projection form of Alg. 2 -- the parity reference
  fastica   O2 Alg. 1 one candidate at a time
  reduced   O3 Alg. 2 with the §3.3 reduction of X
  select    argmax + cluster rule (reading A6), canonical sign (A17)
  metrics   cosine divergence, fluctuation, ordering error, Amari index

Parity pins: every function is pinned in tests/test_oracle_*.py.
"""
from . import contrast, fastica, metrics, ordering, reduced, rng, select, whiten  # noqa: F401
from .ordering import extract  # noqa: F401
