"""ORACLE — test infrastructure only; never imported by the product package.

CPU restatement of the reference schedule-search path, used as the checker by
tests/, by bench.py's `cpu_baseline` leg and by __graft_entry__.smoke():

* ``decide``       — ctypes binding of oracle/decide_port.c, the plain-C
                     restatement of /root/reference/pkg/src/repsched/_core/
                     kernel_c.pyx:23-508 (node-count exact).
* ``search_port``  — sequential Python restatement of the reference's
                     repetend.py / solver.py / completion.py driving ``decide``.
* ``_ref/``        — (git-ignored) the unmodified reference package built by
                     oracle/build_ref.sh; ``load_reference()`` imports it.

Pinned against the reference itself (tests/test_oracle.py) and against the
golden fixtures in tests/golden/ generated from the reference by
tests/golden/make_goldens.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle_decide.so"
REF_DIR = HERE / "_ref"

SAT, UNSAT, TIMEOUT = 1, 0, 2

_lib = None


def build(force: bool = False) -> Path:
    """Compile decide_port.c (gcc -O2, as the reference's default Cython build)."""
    src = HERE / "decide_port.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", str(LIB), str(src)])
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB))
        i64p = ctypes.POINTER(ctypes.c_int64)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        lib.oracle_decide.restype = ctypes.c_int
        lib.oracle_decide.argtypes = [
            ctypes.c_int, i64p, u64p, i64p, i64p, ctypes.c_int, i64p, i64p, i64p,
            ctypes.c_int, i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, i64p, i64p,
        ]
        _lib = lib
    return _lib


def _i64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64).reshape(-1))


def decide(n, dur, devmask, mem, edges, order, lo, hi, ndev, init_mem, cap,
           node_budget=0, deadline=0.0):
    """Same signature and return value as kernel_c.decide (kernel_c.pyx:23-37)."""
    lib = _load()
    dur_a, mem_a, order_a = _i64(dur), _i64(mem), _i64(order)
    lo_a, hi_a, init_a = _i64(lo), _i64(hi), _i64(init_mem)
    mask_a = np.ascontiguousarray(np.asarray(devmask, dtype=np.uint64).reshape(-1))
    e = _i64(edges)
    m = e.size // 3
    out = np.zeros(max(n, 1), dtype=np.int64)
    nodes = np.zeros(1, dtype=np.int64)
    P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    st = lib.oracle_decide(
        int(n), P(dur_a), mask_a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), P(mem_a),
        P(e), int(m), P(order_a), P(lo_a), P(hi_a), int(ndev), P(init_a), int(cap),
        int(node_budget), float(deadline), P(out), P(nodes))
    if st == SAT:
        return SAT, [int(v) for v in out[:n]], int(nodes[0])
    return st, None, int(nodes[0])


def load_reference():
    """Import the compiled reference package from oracle/_ref (or None)."""
    if not (REF_DIR / "repsched").is_dir():
        return None
    os.environ["REPSCHED_KERNEL"] = "compiled"
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import repsched._core  # noqa: F401
    import repsched.completion  # noqa: F401
    return sys.modules["repsched"]
