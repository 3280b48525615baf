"""CPU oracle for the Malleus hot path (arXiv 2410.13333).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import, call or execute anything under oracle/.  The product package
paper_2410_13333_b200 never imports it and fails loudly when its CUDA library is missing.

Modules:
  model     - unpartitioned fp64 training step (fwd, mean CE, manual bwd, AdamW)
  layout    - plan validation, holders / owners per element (R9), migration deltas (R10/R11)
  emulator  - fp64 partition emulator executing any plan's arithmetic member by member
  costmodel - closed forms (theoretic optimum P:848, cost model P:499-506, R7 split helper)

Parity status: every function is pinned by tests/test_oracle_*.py (finite differences, torch
fp64 autograd, closed-form special cases, paper-printed values, brute force).  No function is
"parity unpinned".
"""
