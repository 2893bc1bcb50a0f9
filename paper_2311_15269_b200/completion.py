"""Warmup / cooldown completion and the two-phase schedule search (Algorithm 1).

API mirror of the reference ``repsched.completion``
(/root/reference/pkg/src/repsched/completion.py:41-396).  ``search`` keeps the
reference signature and results — improvements, chosen repetend, schedule,
candidate records — but evaluates candidates in GPU windows
(engine.BatchedRepetendSearch) and replays them in index order with the
reference's improvement rule.  Completion (warmup / cooldown min-makespan
and the lazy feasibility checks) runs its decide probes on the GPU too.
"""

from __future__ import annotations

import bisect
import os
from collections import deque
import time
from collections.abc import Sequence
from dataclasses import dataclass, field
from typing import Optional

from .engine import (VERIFY_SLOTS, WINDOW_FIRST, WINDOW_GROWTH, WINDOW_MAX,
                     BatchedRepetendSearch)
from .parallel import LevelSync, split_range
from .placement import BlockInstance, PlacementSpec
from .repetend import (Repetend, RepetendOutcome, entry_memory, lower_bound, make_repetend,
                       steady_memory_ok)
from .schedule import RepetendInfo, Schedule
from .solver import (SolveRequest, SolveStats, Status, default_budget, solve_decide,
                     solve_min_makespan)

DEFAULT_MAX_NR = 8
LAZY_CHECK_NODES = 2_000_000  # completion.py:178


class NoFeasibleSchedule(Exception):
    pass


class CompletionTimeout(Exception):
    """Time-optimal completion exceeded its budget (fatal, with diagnostic)."""


@dataclass
class CandidateRecord:
    n_r: int
    assignment: tuple
    t_r: Optional[int]
    status: str


class CandidateLog(Sequence):
    """``SearchReport.candidates`` without materialising one object per
    candidate (10^6..10^10 of them).  Records are rebuilt on access: rank
    windows are unranked on the host, gate-infeasible candidates are
    recomputed from their entry memory, and the few improved /
    completion-infeasible ones are stored explicitly.  Behaves like the
    reference's list (len, indexing, iteration, append)."""

    def __init__(self, p: PlacementSpec, cap: Optional[int], unrank):
        self._p, self._cap, self._unrank = p, cap, unrank
        self._starts: list = []   # global index of each segment's first record
        self._segs: list = []     # (n_r, r0, count)
        self._special: dict = {}  # global index -> CandidateRecord
        self._appended: list = []
        self._size = 0
        self.counts: dict = {}

    def add_segment(self, n_r: int, r0: int, count: int, special: dict, infeasible: int):
        if count <= 0:
            return
        base = self._size
        self._starts.append(base)
        self._segs.append((n_r, r0, count))
        for off, rec in special.items():
            self._special[base + off] = rec
            self.counts[rec.status] = self.counts.get(rec.status, 0) + 1
        if infeasible:
            self.counts["infeasible"] = self.counts.get("infeasible", 0) + infeasible
        bound = count - len(special) - infeasible
        if bound:
            self.counts["bound"] = self.counts.get("bound", 0) + bound
        self._size += count

    def append(self, rec: CandidateRecord):
        self._appended.append(rec)
        self.counts[rec.status] = self.counts.get(rec.status, 0) + 1

    def __len__(self):
        return self._size + len(self._appended)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        if i >= self._size:
            return self._appended[i - self._size]
        rec = self._special.get(i)
        if rec is not None:
            return rec
        s = bisect.bisect_right(self._starts, i) - 1
        n_r, r0, _ = self._segs[s]
        a = self._unrank(n_r, r0 + (i - self._starts[s]))
        if self._cap is not None and any(e > self._cap for e in entry_memory(self._p, a)):
            return CandidateRecord(n_r, a, None, "infeasible")
        return CandidateRecord(n_r, a, None, "bound")


@dataclass
class SearchReport:
    lower_bound: int
    max_nr: int
    inflights: int
    lazy: bool
    candidates: object = field(default_factory=list)
    improvements: list = field(default_factory=list)
    phase_secs: dict = field(default_factory=lambda: {"repetend": 0.0, "warmup": 0.0,
                                                      "cooldown": 0.0})
    stats: SolveStats = field(default_factory=SolveStats)
    timed_out: bool = False
    best_t_r: Optional[int] = None
    diagnostics: list = field(default_factory=list)
    engine: dict = field(default_factory=dict)  # GPU counters (B200 build only)

    def to_dict(self) -> dict:
        return {
            "lower_bound": self.lower_bound,
            "max_nr": self.max_nr,
            "inflights": self.inflights,
            "lazy": self.lazy,
            "timed_out": self.timed_out,
            "diagnostics": self.diagnostics,
            "best_t_r": self.best_t_r,
            "phase_secs": self.phase_secs,
            "solver": {"decides": self.stats.decides, "nodes": self.stats.nodes,
                       "wall_secs": self.stats.wall_secs},
            "candidates": [{"nr": c.n_r, "assignment": list(c.assignment), "t_r": c.t_r,
                            "status": c.status} for c in self.candidates],
        }


@dataclass
class SearchResult:
    schedule: Optional[Schedule]
    report: SearchReport


def warmup_blocks(rep: Repetend) -> set:
    """Eq. 5: {B_i^n | n < n_i}."""
    return {BlockInstance(st, n) for st, r in enumerate(rep.assignment) for n in range(r)}


def cooldown_blocks(rep: Repetend, n_r: Optional[int] = None) -> set:
    """Eq. 6: {B_i^n | n_i < n < N_R}."""
    top = rep.n_r if n_r is None else n_r
    return {BlockInstance(st, n) for st, r in enumerate(rep.assignment)
            for n in range(r + 1, top)}


def cooldown_entry_memory(p: PlacementSpec, rep: Repetend, n: int) -> tuple:
    """Memory when the cooldown starts with (n - N_R + 1) repetend copies."""
    reps = n - rep.n_r + 1
    net = p.net_mem_per_device()
    return tuple(e + reps * net[d] for d, e in enumerate(rep.entry_mem))


def cal_max_inflight(p: PlacementSpec, mem_capacity: Optional[int]) -> Optional[int]:
    """min over devices of floor(M / stage-order prefix peak) (completion.py:132-149)."""
    if mem_capacity is None:
        return None
    best = None
    for d in range(p.num_devices):
        run = peak = 0
        for st in p.device_stages(d):
            run += p.block(st).mem_delta
            peak = max(peak, run)
        if peak > 0:
            c = mem_capacity // peak
            best = c if best is None else min(best, c)
    return best


def _budget_left(deadline: float) -> float:
    return max(0.0, deadline - time.monotonic())


def _completion_feasible(p: PlacementSpec, rep: Repetend, cap: Optional[int], deadline: float,
                         report: SearchReport) -> bool:
    """Lazy check: warmup and cooldown each decidable within the serial
    horizon under a 2M-node cap (completion.py:156-182)."""
    phases = (
        (warmup_blocks(rep), (0,) * p.num_devices),
        (cooldown_blocks(rep),
         tuple(max(0, v) for v in cooldown_entry_memory(p, rep, rep.n_r))),
    )
    for insts, init in phases:
        if not insts:
            continue
        horizon = sum(p.block(b.stage).time_cost for b in insts)
        req = SolveRequest(p, tuple(sorted(insts)), init, cap, horizon, "decide")
        res = solve_decide(req, budget=_budget_left(deadline), probe_nodes=LAZY_CHECK_NODES)
        report.stats.merge(res.stats)
        if res.status != Status.SATISFIABLE:
            return False
    return True


def complete_schedule(p: PlacementSpec, rep: Repetend, cap: Optional[int], deadline: float,
                      report: Optional[SearchReport] = None) -> Schedule:
    """warmup || copy 0 at the warmup makespan || cooldown, at N = N_R
    (completion.py:185-274)."""
    report = report if report is not None else SearchReport(0, 0, 0, True)
    entries: dict = {}
    t0 = time.monotonic()
    wu = tuple(sorted(warmup_blocks(rep)))
    w_end = 0
    if wu:
        res = solve_min_makespan(SolveRequest(p, wu, (0,) * p.num_devices, cap),
                                 budget=_budget_left(deadline))
        report.stats.merge(res.stats)
        if res.status == Status.TIMEOUT and res.assignment is None:
            raise CompletionTimeout(f"warmup completion timed out ({len(wu)} blocks)")
        if res.status == Status.INFEASIBLE:
            raise NoFeasibleSchedule(f"warmup infeasible for assignment {rep.assignment}")
        if res.status == Status.TIMEOUT:
            report.diagnostics.append(
                f"warmup completed at {res.objective} but optimality is unproven")
        entries.update(res.assignment)
        w_end = res.objective
    report.phase_secs["warmup"] += time.monotonic() - t0

    offset = w_end
    span = max(rep.internal[st] + p.block(st).time_cost for st in range(p.num_stages))
    for st, n in enumerate(rep.assignment):
        entries[BlockInstance(st, n)] = offset + rep.internal[st]

    t0 = time.monotonic()
    cd = tuple(sorted(cooldown_blocks(rep)))
    if cd:
        window = {}
        for d in range(p.num_devices):
            on = p.device_stages(d)
            if on:
                window[d] = offset + min(rep.internal[st] for st in on)
        fences = tuple((b, max((window[d] for d in p.block(b.stage).devices), default=0))
                       for b in cd)
        res = solve_min_makespan(
            SolveRequest(p, cd, (0,) * p.num_devices, cap, fixed=tuple(sorted(entries.items())),
                         min_starts=fences),
            budget=_budget_left(deadline))
        report.stats.merge(res.stats)
        if res.status == Status.TIMEOUT and res.assignment is None:
            raise CompletionTimeout(f"cooldown completion timed out ({len(cd)} blocks)")
        if res.status == Status.INFEASIBLE:
            raise NoFeasibleSchedule(f"cooldown infeasible for assignment {rep.assignment}")
        if res.status == Status.TIMEOUT:
            report.diagnostics.append(
                f"cooldown completed at {res.objective} but optimality is unproven")
        entries.update(res.assignment)
    report.phase_secs["cooldown"] += time.monotonic() - t0
    info = RepetendInfo(start=offset, end=offset + span, period=rep.period, nr=rep.n_r)
    return Schedule(p, rep.n_r, entries, info)


class _Feasibility:
    """Completion check per assignment, evaluated at most once and replayed
    with its side effects (stats, diagnostics, eager schedules, exceptions)
    only where the reference itself would run it."""

    def __init__(self, p, cap, lazy, deadline):
        self.p, self.cap, self.lazy, self.deadline = p, cap, lazy, deadline
        self.memo: dict = {}

    def evaluate(self, rep: Repetend):
        key = rep.assignment
        if key not in self.memo:
            scratch = SearchReport(0, 0, 0, self.lazy)
            ok, sched, exc = False, None, None
            try:
                if self.lazy:
                    ok = _completion_feasible(self.p, rep, self.cap, self.deadline, scratch)
                else:
                    sched = complete_schedule(self.p, rep, self.cap, self.deadline, scratch)
                    ok = True
            except NoFeasibleSchedule:
                ok = False
            except CompletionTimeout as e:
                exc = e
            self.memo[key] = (ok, sched, exc, scratch)
        return self.memo[key]

    def ok(self, rep: Repetend) -> bool:
        ok, _, exc, _ = self.evaluate(rep)
        return ok and exc is None

    def replay(self, rep: Repetend, report: SearchReport):
        ok, sched, exc, scratch = self.evaluate(rep)
        report.stats.merge(scratch.stats)
        report.diagnostics.extend(scratch.diagnostics)
        for k, v in scratch.phase_secs.items():
            report.phase_secs[k] += v
        if exc is not None:
            raise exc
        return ok, sched


# scan window w+1 while window w's pending probes are verified (engine.py)
PIPELINE_WINDOWS = os.environ.get("TESSEL_PIPELINE_WINDOWS", "1") == "1"
# windows whose pending probes may be under verification at once (one
# verification slot each, plus the slot of the window being scanned)
PIPELINE_DEPTH = max(1, min(int(os.environ.get("TESSEL_PIPELINE_DEPTH", "3")), VERIFY_SLOTS - 1))


def search(p: PlacementSpec, mem_capacity: Optional[int] = None, max_nr: Optional[int] = None,
           lazy: bool = True, budget: Optional[float] = None, jobs: int = 1,
           device: Optional[int] = None, engine: Optional[BatchedRepetendSearch] = None,
           comm=None) -> SearchResult:
    """Two-phase schedule search: repetend construction, then completion
    (completion.py:284-396).  ``jobs`` is accepted for API compatibility;
    candidate parallelism comes from the GPU windows instead of a process
    pool.  ``device`` selects the CUDA device (default: current)."""
    cap = mem_capacity
    lb = lower_bound(p)
    total = sum(b.time_cost for b in p.blocks)
    inflights = cal_max_inflight(p, cap)
    limit = max_nr if max_nr is not None else DEFAULT_MAX_NR
    if inflights is not None:
        limit = min(limit, inflights)
    report = SearchReport(lower_bound=lb, max_nr=limit,
                          inflights=inflights if inflights is not None else -1, lazy=lazy)
    if cap is not None and not steady_memory_ok(p):
        raise NoFeasibleSchedule("per-device net memory of one micro-batch must be <= 0 to repeat")
    deadline = time.monotonic() + (budget if budget is not None else default_budget())

    eng = engine if engine is not None else BatchedRepetendSearch(p, device or 0)
    log = CandidateLog(p, cap, eng.unrank)
    report.candidates = log
    feas = _Feasibility(p, cap, lazy, deadline)

    def feasible(n_r, rank, period, starts):
        rep = make_repetend(p, eng.unrank(n_r, rank), [int(v) for v in starts], period)
        return feas.ok(rep)

    best: Optional[Repetend] = None
    best_completed: Optional[Schedule] = None
    optimal = total + 1
    done = False
    t_rep = time.monotonic()

    def windows():
        """(n_r, r0, r1) in the reference's candidate order, windows growing."""
        for n_r in range(1, max(limit, 1) + 1):
            count = eng.count(n_r)
            r0, width = 0, WINDOW_FIRST
            while r0 < count:
                r1 = min(count, r0 + width)
                yield n_r, r0, r1
                r0 = r1
                width = min(width * WINDOW_GROWTH, WINDOW_MAX)

    def replay(n_r, r0, r1, a0, win) -> bool:
        """Ordered replay of a window's first SATs (completion.py:351-382);
        True = the search ends (load bound reached)."""
        nonlocal best, best_completed, optimal
        first_sat = {a0 - r0 + w: v for w, v in win.first_sat.items()}
        if comm is not None:
            merged: dict = {}
            for part in comm.allgather(first_sat):
                merged.update(part)
            first_sat = merged
        special: dict = {}
        used = r1 - r0
        stop = False
        for widx in sorted(first_sat):
            period, starts = first_sat[widx]
            if period >= optimal:
                continue  # first SAT beyond this candidate's bound: "bound"
            a = eng.unrank(n_r, r0 + widx)
            rep = make_repetend(p, a, [int(v) for v in starts], period)
            ok, sched = feas.replay(rep, report)
            status = "completion-infeasible"
            if ok:
                best, optimal = rep, rep.period
                if not lazy:
                    best_completed = sched
                report.improvements.append((a, optimal))
                status = "improved"
            special[widx] = CandidateRecord(n_r, a, rep.period, status)
            if ok and optimal == lb:
                stop = True
                used = widx + 1
                break
        infeasible = 0
        if win.gate is not None:
            mine = max(0, min(win.count, r0 + used - a0))
            infeasible = int(mine - win.gate[:mine].sum())
            if comm is not None:
                infeasible = comm.allreduce_sum([infeasible])[0]
        log.add_segment(n_r, r0, used, special, infeasible)
        return stop

    def predicted_optimal(n_r, r0, win, opt) -> int:
        """The bound after replaying `win` from bound `opt` if its
        speculation holds: the replay rule run without side effects
        (memoised completion checks)."""
        for widx in sorted(win.first_sat):
            period, starts = win.first_sat[widx]
            if period >= opt:
                continue
            rep = make_repetend(p, eng.unrank(n_r, r0 + widx), [int(v) for v in starts], period)
            if feas.ok(rep):
                opt = rep.period
        return opt

    pipelined = comm is None and PIPELINE_WINDOWS and hasattr(eng, "begin_window")
    # windows scanned whose pending probes are being verified, oldest first:
    # [n_r, r0, r1, job, bound the window was scanned under]
    inflight: deque = deque()

    def settle_head() -> bool:
        """Finish and replay the oldest window in flight; True = the search
        ends (load bound reached or out of time)."""
        pn, p0, p1, pjob, _ = inflight.popleft()
        pwin = eng.finish_window(pjob, feasible)
        if pwin.timed_out:
            report.timed_out = True
            return True
        return replay(pn, p0, p1, p0, pwin)

    def redo_mispredicted() -> bool:
        """The next window in flight was scanned under a predicted bound; a
        true bound above it (a repaired / rescanned misprediction) means it
        missed periods: redo it and every later one, in order, exactly."""
        if not inflight or optimal <= inflight[0][4]:
            return False
        redo = list(inflight)
        inflight.clear()  # their verification results are dropped
        for rn, q0, q1, _, _ in redo:
            win = eng.evaluate_window(rn, q0, q1, cap, optimal, feasible, deadline)
            if win.timed_out:
                report.timed_out = True
                return True
            if replay(rn, q0, q1, q0, win):
                return True
        return False

    for n_r, r0, r1 in windows():
        if time.monotonic() > deadline:
            report.timed_out = True
            done = True
            break
        if comm is not None:  # rank-prefix shard of the window (parallel.py)
            a0, b0 = split_range(r0, r1, comm.rank, comm.size)
            win = eng.evaluate_window(n_r, a0, b0, cap, optimal, feasible, 0.0,
                                      LevelSync(comm, a0 - r0))
        elif not pipelined:
            a0 = r0
            win = eng.evaluate_window(n_r, r0, r1, cap, optimal, feasible, deadline)
        else:
            # Scan this window while the pending probes of up to
            # PIPELINE_DEPTH earlier windows are verified (one stream each),
            # under the bound their replays yield if their speculation holds
            # (else the true bound is lower: the scan only did extra work);
            # windows are settled and replayed strictly in order.
            bound = optimal
            for pn, p0, _, pjob, _ in inflight:
                bound = predicted_optimal(pn, p0, pjob.res, bound)
            busy = {e[3].slot for e in inflight}
            slot = next(k for k in range(VERIFY_SLOTS) if k not in busy)
            job = eng.begin_window(n_r, r0, r1, cap, bound, feasible, deadline, slot)
            inflight.append([n_r, r0, r1, job, bound])
            # settle the oldest while too many are in flight, and every head
            # with nothing to verify (it settles without waiting)
            while inflight and (len(inflight) > PIPELINE_DEPTH or not inflight[0][3].launched):
                if settle_head() or redo_mispredicted():
                    done = True
                    break
            if done:
                break
            continue
        if win.timed_out:
            report.timed_out = True
            done = True
            break
        if replay(n_r, r0, r1, a0, win):
            done = True
            break
    while inflight and not done:
        if settle_head() or redo_mispredicted():
            break
    report.phase_secs["repetend"] += time.monotonic() - t_rep
    c = eng.counters
    report.engine = dict(c.__dict__)
    report.stats.decides += c.probes
    report.stats.nodes += c.nodes

    report.best_t_r = best.period if best else None
    if best is None:
        if report.timed_out:
            return SearchResult(None, report)
        raise NoFeasibleSchedule("no repetend candidate is schedulable under memory")
    if lazy or best_completed is None:
        best_completed = complete_schedule(p, best, cap, deadline, report)
    return SearchResult(best_completed, report)
