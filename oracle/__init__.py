"""CPU oracle for the LBM hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs import this package, and only as the checker or the
timed CPU baseline.  The product package (paper_1909_13772_b200) never imports
it and has no CPU fallback.

Parity status: pinned.  lbm_oracle.c restates the reference's numpy kernels
with identical operation order; tests/test_oracle_golden.py checks it bit for
bit against golden vectors produced by the reference itself
(tests/golden/make_golden.py, run in the container that holds
/root/reference).
"""
from .lbm_oracle import *  # noqa: F401,F403
