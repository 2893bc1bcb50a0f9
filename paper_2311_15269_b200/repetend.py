"""Repetend construction: candidate enumeration, per-candidate period scan, compaction.

API mirror of the reference ``repsched.repetend``
(/root/reference/pkg/src/repsched/repetend.py:24-328).  ``solve_repetend``
evaluates ONE candidate through the decide seam (``_core.decide`` on the
B200); the batched search over all candidates lives in ``engine.py`` and is
what ``completion.search`` uses.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Iterator, Optional

from . import _core
from .placement import BlockInstance, PlacementSpec
from .solver import SolveStats

PROBE_NODES = 400_000  # repetend.py:21: node cap for probes above the load bound


@dataclass(frozen=True)
class Repetend:
    placement: PlacementSpec
    assignment: tuple
    n_r: int
    internal: tuple
    period: int
    exec_spans: tuple
    waits: tuple
    entry_mem: tuple

    @property
    def t_r(self) -> int:
        return self.period

    def instances(self) -> list:
        return [(BlockInstance(st, n), self.internal[st]) for st, n in enumerate(self.assignment)]

    def tile_entries(self, copies: int, offset: int = 0) -> dict:
        """``copies`` consecutive copies: indices +k, starts +k * period."""
        return {BlockInstance(st, n + k): offset + self.internal[st] + k * self.period
                for k in range(copies) for st, n in enumerate(self.assignment)}


@dataclass
class RepetendOutcome:
    repetend: Optional[Repetend]
    status: str  # ok | infeasible | bound | timeout


def lower_bound(p: PlacementSpec) -> int:
    """Largest per-device load of one micro-batch (repetend.py:60-62)."""
    return max(p.device_load(d) for d in range(p.num_devices))


def iter_repetend_assignments(p: PlacementSpec, n_r: int) -> Iterator[tuple]:
    """Index vectors in [0, n_r)^K with n_i >= n_j on every edge i->j and
    minimum 0, in lexicographic order (repetend.py:65-90).  Explicit-stack
    odometer over stages in id order."""
    k = p.num_stages
    if k == 0:
        return
    lo_src = [[j for j in p.successors(st) if j < st] for st in range(k)]
    hi_src = [[i for i in p.predecessors(st) if i < st] for st in range(k)]
    vec = [0] * k
    top = [0] * k

    def arm(st):
        vec[st] = max([0] + [vec[j] for j in lo_src[st]]) - 1
        top[st] = min([n_r - 1] + [vec[i] for i in hi_src[st]])

    st = 0
    arm(0)
    while st >= 0:
        if vec[st] < top[st]:
            vec[st] += 1
            if st == k - 1:
                if 0 in vec:
                    yield tuple(vec)
            else:
                st += 1
                arm(st)
        else:
            st -= 1


def entry_memory(p: PlacementSpec, assignment) -> tuple:
    """Memory held on each device by the warmup blocks {B_i^n | n < n_i}."""
    out = [0] * p.num_devices
    for st, n in enumerate(assignment):
        blk = p.block(st)
        for d in blk.devices:
            out[d] += n * blk.mem_delta
    return tuple(out)


def steady_memory_ok(p: PlacementSpec) -> bool:
    """Repetition is memory-safe only if no device gains memory per copy."""
    return all(v <= 0 for v in p.net_mem_per_device())


class _CandidateModel:
    """Decide inputs of one placement; only lags and bounds depend on the
    candidate and the period (repetend.py:108-190)."""

    def __init__(self, p: PlacementSpec):
        self.p = p
        k = self.k = p.num_stages
        self.dur = [p.block(s).time_cost for s in range(k)]
        self.mask = [sum(1 << d for d in p.block(s).devices) for s in range(k)]
        self.mem = [p.block(s).mem_delta for s in range(k)]
        self.order = sorted(range(k), key=lambda s: (-len(p.block(s).devices), s))
        rows = sorted(p.deps)
        self.n_dep = len(rows)
        for d in range(p.num_devices):
            on = p.device_stages(d)
            rows += [(x, y) for x in on for y in on if x != y]
        self.rows = rows
        self.max_dur = max(self.dur) if k else 1
        self.coef = [1] * len(rows)

    def set_assignment(self, a):
        for r in range(self.n_dep):
            x, y = self.rows[r]
            self.coef[r] = a[x] - a[y]

    def edges(self, period):
        out = []
        for (x, y), c in zip(self.rows, self.coef):
            out += (x, y, self.dur[x] - c * period)
        return out

    def decide(self, period, cap, entry, deadline, stats=None, node_budget=0):
        anchor = (self.k - 1) * (period + self.max_dur)
        lo = [0] * self.k
        hi = [2 * anchor] * self.k
        if self.k:
            lo[0] = hi[0] = anchor
        t0 = time.monotonic()
        status, starts, nodes = _core.decide(
            self.k, self.dur, self.mask, self.mem, self.edges(period), self.order, lo, hi,
            self.p.num_devices, list(entry), -1 if cap is None else cap, node_budget, deadline)
        if stats is not None:
            stats.decides += 1
            stats.nodes += nodes
            stats.wall_secs += time.monotonic() - t0
        return status, starts


_MODELS: dict = {}


def _model_for(p: PlacementSpec) -> _CandidateModel:
    m = _MODELS.get(id(p))
    if m is None or m.p is not p:
        _MODELS.clear()
        m = _MODELS[id(p)] = _CandidateModel(p)
    return m


def device_spans(p: PlacementSpec, internal) -> tuple:
    spans = []
    for d in range(p.num_devices):
        on = p.device_stages(d)
        spans.append(max(internal[s] + p.block(s).time_cost for s in on)
                     - min(internal[s] for s in on) if on else 0)
    return tuple(spans)


def compact_period(p: PlacementSpec, internal_schedule, assignment) -> tuple:
    """Smallest period at which copies of the internal schedule tile validly:
    every device span and every cross-copy dependency lag
    ceil((s_i + t_i - s_j) / (n_i - n_j)) (repetend.py:220-250).  Waits are
    W_d = P - E_d on every device."""
    starts = dict(internal_schedule)
    spans = device_spans(p, starts)
    period = max(1, max(spans))
    for i, j in p.deps:
        delta = assignment[i] - assignment[j]
        if delta < 0:
            raise ValueError("assignment violates the descending-index property")
        if delta:
            need = starts[i] + p.block(i).time_cost - starts[j]
            if need > 0:
                period = max(period, -(-need // delta))
    return period, spans, tuple(period - e for e in spans)


def make_repetend(p: PlacementSpec, assignment, witness, scanned_period: int, entry=None,
                  monotone: bool = True) -> Repetend:
    """Repetend from a first-SAT witness (repetend.py:305-328)."""
    base = min(witness)
    internal = tuple(int(s) - base for s in witness)
    if monotone:
        period, spans, waits = compact_period(p, dict(enumerate(internal)), tuple(assignment))
    else:
        period, spans = scanned_period, device_spans(p, internal)
        waits = tuple(period - e for e in spans)
    if entry is None:
        entry = entry_memory(p, assignment)
    return Repetend(p, tuple(assignment), max(assignment) + 1, internal, period, spans, waits,
                    tuple(entry))


def solve_repetend(p: PlacementSpec, assignment, mem_capacity: Optional[int],
                   upper: Optional[int] = None, budget: Optional[float] = None,
                   stats: Optional[SolveStats] = None) -> RepetendOutcome:
    """Scan periods upward from the load bound; the first SAT period is
    minimal (repetend.py:253-328).  Probes above the bound carry the
    reference's 400k-node cap; a capped probe on a monotone assignment is
    skipped."""
    entry = entry_memory(p, assignment)
    if mem_capacity is not None and (any(e > mem_capacity for e in entry)
                                     or not steady_memory_ok(p)):
        return RepetendOutcome(None, "infeasible")
    lb = lower_bound(p)
    ub = sum(b.time_cost for b in p.blocks)
    if upper is not None:
        ub = min(ub, upper - 1)
    if ub < lb:
        return RepetendOutcome(None, "bound")
    deadline = time.monotonic() + budget if budget is not None else 0.0
    model = _model_for(p)
    model.set_assignment(assignment)
    monotone = all(assignment[i] >= assignment[j] for i, j in p.deps)
    for period in range(lb, ub + 1):
        status, starts = model.decide(period, mem_capacity, entry, deadline, stats,
                                      0 if period == lb else PROBE_NODES)
        if status == _core.TIMEOUT:
            if budget is not None and time.monotonic() > deadline:
                return RepetendOutcome(None, "timeout")
            if not monotone:
                return RepetendOutcome(None, "timeout")
            continue
        if status == _core.SAT:
            return RepetendOutcome(make_repetend(p, assignment, starts, period, entry, monotone),
                                   "ok")
    return RepetendOutcome(None, "bound" if upper is not None else "infeasible")
