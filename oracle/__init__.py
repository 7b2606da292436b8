"""CPU oracle package: TEST INFRASTRUCTURE ONLY.

Restates the reference's grouped-GEMM semantics (C, oracle/tagg_oracle.c),
its planners (oracle/plan.py) and its FP8 codec / input recipe
(oracle/fp8.py).  Parity is pinned against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import it.
"""
