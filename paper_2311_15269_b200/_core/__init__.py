"""Decide-kernel seam — drop-in for ``repsched._core``
(/root/reference/pkg/src/repsched/_core/__init__.py:1-28).

``decide`` has the reference signature and return value
(kernel_c.pyx:23-37) and runs on the B200 through the C ABI
(include/tessel_b200.h: ``tsl_decide``).  The reference's selector accepted
``REPSCHED_KERNEL=auto|compiled|pure``; here ``auto``/``compiled``/``b200``
all select the sm_100a kernel and ``pure`` is rejected: this path has no CPU
implementation to fall back to.
"""

import os
import time

from .. import _native

_choice = os.environ.get("REPSCHED_KERNEL", "auto")
if _choice not in ("auto", "compiled", "b200", "pure"):
    raise RuntimeError(f"REPSCHED_KERNEL must be auto|compiled|b200, got {_choice!r}")
if _choice == "pure":
    raise RuntimeError("REPSCHED_KERNEL=pure: the B200 build has no CPU decide kernel")

KERNEL_NAME = "b200"
SAT = _native.SAT
UNSAT = _native.UNSAT
TIMEOUT = _native.TIMEOUT


def decide(n, dur, devmask, mem, edges, order, lo, hi, ndev, init_mem, cap,
           node_budget=0, deadline=0.0):
    """Return (status, starts or None, nodes explored) — kernel_c.decide semantics.

    ``edges`` may be an (m, 3) array or a flat list of 3m values (both caller
    layouts of the reference: repetend.py:171-185, solver.py:191-205).
    ``deadline`` is an absolute ``time.monotonic()`` value (0 = none).
    """
    budget_secs = 0.0
    if deadline:
        budget_secs = max(deadline - time.monotonic(), 1e-9)
    return _native.decide(n, dur, devmask, mem, edges, order, lo, hi, ndev, init_mem,
                          -1 if cap is None else cap, node_budget, budget_secs)


def decide_batch(problems, deadline=0.0):
    """Batched decide (no reference equivalent): list of problem dicts."""
    budget_secs = max(deadline - time.monotonic(), 1e-9) if deadline else 0.0
    return _native.decide_batch(problems, budget_secs)
