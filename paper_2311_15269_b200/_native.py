"""ctypes binding of the in-tree sm_100a library ``libtessel_b200.so``.

The library is the C ABI declared in include/tessel_b200.h.  It is built
in-tree by ``build()`` (nvcc, ``-gencode arch=compute_100a,code=sm_100a``) so
it travels with the repository snapshot to the GPU box.  There is no CPU
fallback anywhere on the product path: if the library is missing or no CUDA
device is visible, every compute call raises ``NativeError``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_PATH = PKG / "libtessel_b200.so"
SOURCES = [PKG / "csrc" / "tessel_b200.cu"]
HEADERS = sorted((PKG / "csrc").glob("*.cuh")) + sorted((PKG / "csrc").glob("*.inc")) + [
    PKG / "csrc" / "host_build.hpp", ROOT / "include" / "tessel_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared",
]

SAT, UNSAT, TIMEOUT, ABORT = 1, 0, 2, 3
ERRORS = {-1: "EINVAL", -2: "ENODEV", -3: "ECUDA", -4: "ERANGE"}


class NativeError(RuntimeError):
    """Failure reported by the native library (carries the TSL_E* code)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"tessel_b200 {ERRORS.get(code, code)}: {msg}")
        self.code = code


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile the library in-tree for sm_100a (no GPU needed)."""
    newest = max(p.stat().st_mtime for p in SOURCES + HEADERS)
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= newest:
        return LIB_PATH
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(LIB_PATH), *map(str, SOURCES)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd[cmd.index("-o") + 1] = str(tmp)
    subprocess.check_call(cmd, cwd=str(PKG))
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _Stats(ctypes.Structure):
    _fields_ = [("probes", ctypes.c_int64), ("root_refuted", ctypes.c_int64),
                ("nodes", ctypes.c_int64), ("capped", ctypes.c_int64), ("sat", ctypes.c_int64),
                ("deferred", ctypes.c_int64), ("dj_refuted", ctypes.c_int64),
                ("dj_nodes", ctypes.c_int64)]


class _Problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("m", ctypes.c_int), ("ndev", ctypes.c_int),
                ("dur", ctypes.c_void_p), ("mem", ctypes.c_void_p), ("edges", ctypes.c_void_p),
                ("order", ctypes.c_void_p), ("lo", ctypes.c_void_p), ("hi", ctypes.c_void_p),
                ("init_mem", ctypes.c_void_p), ("devmask", ctypes.c_void_p),
                ("cap", ctypes.c_int64), ("node_budget", ctypes.c_int64)]


_lib = None

EXPORTS = (
    "tsl_last_error", "tsl_version", "tsl_device_count", "tsl_set_device", "tsl_decide",
    "tsl_decide_batch", "tsl_engine_open", "tsl_engine_close", "tsl_engine_count",
    "tsl_engine_unrank", "tsl_engine_stage", "tsl_engine_probe", "tsl_engine_resolve",
    "tsl_engine_sat_rows", "tsl_engine_sat_next", "tsl_engine_take_deferred",
    "tsl_engine_add_active",
    "tsl_engine_verify", "tsl_engine_verify_stash", "tsl_engine_verify_launch",
    "tsl_engine_verify_wait", "tsl_engine_dj", "tsl_validate",
    "tsl_engine_last_kernel_ms", "tsl_engine_last_root_ms", "tsl_counters", "tsl_sp_stats",
)


def lib():
    """Load the library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeError(-2, f"{LIB_PATH.name} is not built; run __graft_entry__.build() "
                              "(there is no CPU fallback)")
    path = LIB_PATH
    variant = os.environ.get("TSL_LIB_VARIANT")  # experiments: an alternately compiled build
    if variant:
        path = PKG / f"libtessel_b200_{variant}.so"
    L = ctypes.CDLL(str(path))
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.tsl_last_error.restype = ctypes.c_char_p
    L.tsl_version.restype = i32
    L.tsl_device_count.restype = i32
    L.tsl_set_device.argtypes = [i32]
    L.tsl_decide.restype = i32
    L.tsl_decide.argtypes = [i32, vp, vp, vp, vp, i32, vp, vp, vp, i32, vp, i64, i64, dbl, vp, vp]
    L.tsl_decide_batch.restype = i32
    L.tsl_decide_batch.argtypes = [i32, vp, dbl, vp, vp, vp, i32]
    L.tsl_engine_open.restype = vp
    L.tsl_engine_open.argtypes = [i32, i32, vp, vp, vp, i32, vp, i32]
    L.tsl_engine_close.argtypes = [vp]
    L.tsl_engine_count.restype = i32
    L.tsl_engine_count.argtypes = [vp, i32, vp]
    L.tsl_engine_unrank.restype = i32
    L.tsl_engine_unrank.argtypes = [vp, i32, ctypes.c_uint64, vp]
    L.tsl_engine_stage.restype = i32
    L.tsl_engine_stage.argtypes = [vp, i32, ctypes.c_uint64, ctypes.c_uint64, i64, vp, vp]
    L.tsl_engine_probe.restype = i32
    L.tsl_engine_probe.argtypes = [vp, i32, i64, i64, i64, i64, dbl, i64, vp, vp, vp, vp, vp, vp]
    L.tsl_engine_resolve.restype = i32
    L.tsl_engine_resolve.argtypes = [vp, i32, i64, i64, i64, i64, i64, dbl, i64, vp, vp, vp,
                                     vp, vp, vp]
    L.tsl_engine_take_deferred.restype = i32
    L.tsl_engine_take_deferred.argtypes = [vp, i64, i64, vp, vp]
    L.tsl_engine_add_active.restype = i32
    L.tsl_engine_add_active.argtypes = [vp, i64, vp]
    L.tsl_engine_verify.restype = i32
    L.tsl_engine_verify.argtypes = [vp, i64, vp, vp, vp, i64, vp, vp, vp]
    L.tsl_engine_dj.restype = i32
    L.tsl_engine_dj.argtypes = [vp, i64, vp, vp, i64, i64, i32, vp, vp]
    L.tsl_engine_sat_rows.restype = i32
    L.tsl_engine_sat_rows.argtypes = [vp, i64, i64, vp, vp]
    L.tsl_engine_sat_next.restype = i32
    L.tsl_engine_sat_next.argtypes = [vp, i64, vp, vp]
    L.tsl_counters.restype = None
    L.tsl_counters.argtypes = [vp, vp, vp]
    L.tsl_engine_last_kernel_ms.restype = ctypes.c_float
    L.tsl_engine_last_kernel_ms.argtypes = [vp]
    L.tsl_engine_verify_stash.restype = i32
    L.tsl_engine_verify_stash.argtypes = [vp, i32, i64, vp]
    L.tsl_engine_verify_launch.restype = i32
    L.tsl_engine_verify_launch.argtypes = [vp, i32, i64, vp, vp, vp, vp, i64]
    L.tsl_engine_verify_wait.restype = i32
    L.tsl_engine_verify_wait.argtypes = [vp, i32, vp, vp, vp]
    L.tsl_validate.restype = i32
    L.tsl_validate.argtypes = [i32, i32, vp, vp, vp, i32, vp, i32, vp, vp, i64, i64, vp, vp, vp,
                               vp, vp, vp, vp]
    L.tsl_sp_stats.restype = None
    L.tsl_sp_stats.argtypes = [vp]
    L.tsl_engine_last_root_ms.restype = ctypes.c_float
    L.tsl_engine_last_root_ms.argtypes = [vp]
    _lib = L
    return L


def check(rc: int) -> int:
    if rc < 0:
        raise NativeError(rc, lib().tsl_last_error().decode(errors="replace"))
    return rc


def counters() -> dict:
    """Process-wide kernel launches and host<->device bytes of this library."""
    v = np.zeros(3, dtype=np.int64)
    lib().tsl_counters(_ptr(v[0:1]), _ptr(v[1:2]), _ptr(v[2:3]))
    return {"launches": int(v[0]), "h2d_bytes": int(v[1]), "d2h_bytes": int(v[2])}


def sp_stats() -> dict:
    """Counters of the subtree-parallel decide (csrc/sp_host.inc)."""
    a = np.zeros(12, dtype=np.float64)
    lib().tsl_sp_stats(_ptr(a))
    keys = ("solves", "rounds", "tasks", "replays", "subsolves", "master_nodes", "master_ms",
            "task_ms", "pieces", "undivided", "explored", "epochs")
    return {k: float(v) for k, v in zip(keys, a)}


def device_count() -> int:
    return lib().tsl_device_count()


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64).reshape(-1))


def _u64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64).reshape(-1))


def decide(n, dur, devmask, mem, edges, order, lo, hi, ndev, init_mem, cap,
           node_budget=0, budget_secs=0.0):
    """One decide problem on the GPU -> (status, starts | None, nodes)."""
    L = lib()
    a_dur, a_mem, a_edges = _i64(dur), _i64(mem), _i64(edges)
    a_order, a_lo, a_hi, a_init = _i64(order), _i64(lo), _i64(hi), _i64(init_mem)
    a_mask = _u64(devmask)
    if a_edges.size % 3:
        raise ValueError("edges must hold (src, dst, lag) triples")
    out = np.zeros(max(int(n), 1), dtype=np.int64)
    nodes = np.zeros(1, dtype=np.int64)
    st = check(L.tsl_decide(int(n), _ptr(a_dur), _ptr(a_mask), _ptr(a_mem), _ptr(a_edges),
                            a_edges.size // 3, _ptr(a_order), _ptr(a_lo), _ptr(a_hi), int(ndev),
                            _ptr(a_init), int(cap), int(node_budget), float(budget_secs),
                            _ptr(out), _ptr(nodes)))
    return st, ([int(v) for v in out[:n]] if st == SAT else None), int(nodes[0])


def decide_batch(problems, budget_secs=0.0):
    """Several independent decide problems in one launch.  Each problem is a
    dict with keys n, dur, devmask, mem, edges, order, lo, hi, ndev,
    init_mem, cap, node_budget.  Returns [(status, starts|None, nodes)]."""
    L = lib()
    count = len(problems)
    if count == 0:
        return []
    keep = []
    arr = (_Problem * count)()
    stride = 1
    for i, p in enumerate(problems):
        cols = dict(dur=_i64(p["dur"]), mem=_i64(p["mem"]), edges=_i64(p["edges"]),
                    order=_i64(p["order"]), lo=_i64(p["lo"]), hi=_i64(p["hi"]),
                    init_mem=_i64(p["init_mem"]), devmask=_u64(p["devmask"]))
        keep.append(cols)
        pr = arr[i]
        pr.n, pr.ndev = int(p["n"]), int(p["ndev"])
        pr.m = cols["edges"].size // 3
        for k, v in cols.items():
            setattr(pr, k, v.ctypes.data)
        pr.cap, pr.node_budget = int(p["cap"]), int(p.get("node_budget", 0))
        stride = max(stride, pr.n)
    status = np.zeros(count, dtype=np.int32)
    nodes = np.zeros(count, dtype=np.int64)
    starts = np.zeros(count * stride, dtype=np.int64)
    check(L.tsl_decide_batch(count, ctypes.cast(arr, ctypes.c_void_p), float(budget_secs),
                             _ptr(status), _ptr(nodes), _ptr(starts), stride))
    out = []
    for i, p in enumerate(problems):
        st = int(status[i])
        n = int(p["n"])
        s = [int(v) for v in starts[i * stride:i * stride + n]] if st == SAT else None
        out.append((st, s, int(nodes[i])))
    return out


class Engine:
    """Batched repetend-search engine over one placement (tsl_engine_*)."""

    def __init__(self, dur, mem, masks, deps, num_devices, device=0):
        L = lib()
        self.K = len(dur)
        self.D = int(num_devices)
        a_dur = np.ascontiguousarray(dur, dtype=np.int32)
        a_mem = np.ascontiguousarray(mem, dtype=np.int32)
        a_mask = np.ascontiguousarray(masks, dtype=np.uint64)
        a_deps = np.ascontiguousarray(np.asarray(sorted(deps), dtype=np.int32).reshape(-1))
        h = L.tsl_engine_open(self.K, self.D, _ptr(a_dur), _ptr(a_mem), _ptr(a_mask),
                              len(deps), _ptr(a_deps), int(device))
        if not h:
            raise NativeError(-1, L.tsl_last_error().decode(errors="replace"))
        self._h = ctypes.c_void_p(h)
        self._L = L
        self._a = np.zeros(self.K, dtype=np.int32)

    def close(self):
        if getattr(self, "_h", None):
            self._L.tsl_engine_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def count(self, n_r: int) -> int:
        out = np.zeros(1, dtype=np.uint64)
        check(self._L.tsl_engine_count(self._h, int(n_r), _ptr(out)))
        return int(out[0])

    def unrank(self, n_r: int, rank: int) -> tuple:
        check(self._L.tsl_engine_unrank(self._h, int(n_r), int(rank), _ptr(self._a)))
        return tuple(int(v) for v in self._a)

    def stage(self, n_r: int, r0: int, r1: int, cap, want_gate=False):
        n_act = np.zeros(1, dtype=np.int64)
        gate = np.zeros(max(r1 - r0, 1), dtype=np.uint8) if want_gate else None
        check(self._L.tsl_engine_stage(self._h, int(n_r), int(r0), int(r1),
                                       -1 if cap is None else int(cap), _ptr(n_act),
                                       _ptr(gate) if gate is not None else None))
        return int(n_act[0]), gate

    def probe(self, period: int, node_budget: int, small_budget: int, cap, widx_limit: int,
              budget_secs=0.0, max_sat=64):
        """Level pass -> (n_sat, widx[:k], rows[:k], n_active, n_deferred, stats)."""
        nsat = np.zeros(1, dtype=np.int64)
        n_act = np.zeros(1, dtype=np.int64)
        n_def = np.zeros(1, dtype=np.int64)
        widx = np.zeros(max(max_sat, 1), dtype=np.int64)
        rows = np.zeros(max(max_sat, 1) * self.K, dtype=np.int32)
        st = _Stats()
        check(self._L.tsl_engine_probe(self._h, int(period), int(node_budget), int(small_budget),
                                       -1 if cap is None else int(cap), int(widx_limit),
                                       float(budget_secs), int(max_sat), _ptr(nsat), _ptr(widx),
                                       _ptr(rows), _ptr(n_act), _ptr(n_def), ctypes.byref(st)))
        n = int(nsat[0])
        k = min(n, max_sat)
        return (n, widx[:k].copy(), rows[:k * self.K].reshape(k, self.K).copy(), int(n_act[0]),
                int(n_def[0]), {f: getattr(st, f) for f, _ in _Stats._fields_})

    def resolve(self, period: int, node_budget: int, stage_budget: int, dj_budget: int, cap,
                widx_limit: int, budget_secs=0.0, max_sat=64):
        """One stage of settling deferred probes ->
        (n_sat, widx[:k], rows[:k], n_active, n_deferred, stats)."""
        nsat = np.zeros(1, dtype=np.int64)
        n_act = np.zeros(1, dtype=np.int64)
        n_def = np.zeros(1, dtype=np.int64)
        widx = np.zeros(max(max_sat, 1), dtype=np.int64)
        rows = np.zeros(max(max_sat, 1) * self.K, dtype=np.int32)
        st = _Stats()
        check(self._L.tsl_engine_resolve(self._h, int(period), int(node_budget),
                                         int(stage_budget), int(dj_budget),
                                         -1 if cap is None else int(cap), int(widx_limit),
                                         float(budget_secs), int(max_sat), _ptr(nsat),
                                         _ptr(widx), _ptr(rows), _ptr(n_act), _ptr(n_def),
                                         ctypes.byref(st)))
        n = int(nsat[0])
        k = min(n, max_sat)
        return (n, widx[:k].copy(), rows[:k * self.K].reshape(k, self.K).copy(), int(n_act[0]),
                int(n_def[0]), {f: getattr(st, f) for f, _ in _Stats._fields_})

    def take_deferred(self, widx_limit: int, max_out: int):
        out = np.zeros(max(max_out, 1), dtype=np.int64)
        n = np.zeros(1, dtype=np.int64)
        check(self._L.tsl_engine_take_deferred(self._h, int(widx_limit), int(max_out),
                                               _ptr(out), _ptr(n)))
        return out[:int(n[0])].copy()

    def add_active(self, widx):
        a = np.ascontiguousarray(widx, dtype=np.int64)
        if a.size:
            check(self._L.tsl_engine_add_active(self._h, int(a.size), _ptr(a)))

    def verify(self, widx, periods, budgets, cap):
        """Exact probes for explicit (widx, period) pairs ->
        (status[], nodes[], starts[count, K])."""
        w = np.ascontiguousarray(widx, dtype=np.int64)
        per = np.ascontiguousarray(periods, dtype=np.int32)
        bud = np.ascontiguousarray(budgets, dtype=np.int64)
        n = int(w.size)
        st = np.zeros(max(n, 1), dtype=np.int32)
        nd = np.zeros(max(n, 1), dtype=np.int64)
        rows = np.zeros(max(n, 1) * self.K, dtype=np.int32)
        if n:
            check(self._L.tsl_engine_verify(self._h, n, _ptr(w), _ptr(per), _ptr(bud),
                                            -1 if cap is None else int(cap), _ptr(st), _ptr(nd),
                                            _ptr(rows)))
        return st[:n].copy(), nd[:n].copy(), rows[:n * self.K].reshape(n, self.K).copy()

    def verify_stash(self, slot: int, widx):
        """Keep the assignments of these window indices (row positions
        0..len-1) for asynchronous verification in `slot`."""
        w = np.ascontiguousarray(widx, dtype=np.int64)
        check(self._L.tsl_engine_verify_stash(self._h, int(slot), int(w.size), _ptr(w)))

    def verify_launch(self, slot: int, pos, widx, periods, budgets, cap):
        """Start verifying (row position, widx, period, cap) in `slot`."""
        self._vk = getattr(self, "_vk", {})
        arrs = [np.ascontiguousarray(pos, dtype=np.int64),
                np.ascontiguousarray(widx, dtype=np.int64),
                np.ascontiguousarray(periods, dtype=np.int32),
                np.ascontiguousarray(budgets, dtype=np.int64)]
        self._vk[slot] = (arrs, int(arrs[0].size))
        check(self._L.tsl_engine_verify_launch(self._h, int(slot), arrs[0].size, _ptr(arrs[0]),
                                               _ptr(arrs[1]), _ptr(arrs[2]), _ptr(arrs[3]),
                                               -1 if cap is None else int(cap)))

    def verify_wait(self, slot: int):
        """Results of the slot's launch -> (status[], nodes[], starts[count, K])."""
        n = self._vk[slot][1]
        st = np.zeros(max(n, 1), dtype=np.int32)
        nd = np.zeros(max(n, 1), dtype=np.int64)
        rows = np.zeros(max(n, 1) * self.K, dtype=np.int32)
        if n:
            check(self._L.tsl_engine_verify_wait(self._h, int(slot), _ptr(st), _ptr(nd),
                                                 _ptr(rows)))
        return st[:n].copy(), nd[:n].copy(), rows[:n * self.K].reshape(n, self.K).copy()

    def dj(self, assignments, periods, cap, budget, mode=1):
        """Diagnostic: disjunctive filter verdicts (0 infeasible, 1 feasible,
        2 undecided) and orientation nodes for explicit (assignment, period)
        pairs; mode 1 = warp filter, 0 = one-lane filter."""
        a = np.ascontiguousarray(assignments, dtype=np.int32).reshape(-1, self.K)
        per = np.ascontiguousarray(periods, dtype=np.int32)
        n = int(per.size)
        st = np.zeros(max(n, 1), dtype=np.int32)
        nd = np.zeros(max(n, 1), dtype=np.int64)
        if n:
            check(self._L.tsl_engine_dj(self._h, n, _ptr(a), _ptr(per),
                                        -1 if cap is None else int(cap), int(budget), int(mode),
                                        _ptr(st), _ptr(nd)))
        return st[:n].copy(), nd[:n].copy()

    def sat_next(self, after: int):
        """The level's SAT with the smallest window index above `after`
        (device argmin) -> (widx, starts[K]) or None."""
        w = np.zeros(1, dtype=np.int64)
        row = np.zeros(self.K, dtype=np.int32)
        check(self._L.tsl_engine_sat_next(self._h, int(after), _ptr(w), _ptr(row)))
        return None if w[0] < 0 else (int(w[0]), row)

    def sat_rows(self, first: int, count: int):
        widx = np.zeros(max(count, 1), dtype=np.int64)
        rows = np.zeros(max(count, 1) * self.K, dtype=np.int32)
        check(self._L.tsl_engine_sat_rows(self._h, int(first), int(count), _ptr(widx), _ptr(rows)))
        return widx[:count].copy(), rows[:count * self.K].reshape(count, self.K).copy()

    def last_kernel_ms(self) -> float:
        return float(self._L.tsl_engine_last_kernel_ms(self._h))

    def last_root_ms(self) -> float:
        return float(self._L.tsl_engine_last_root_ms(self._h))
