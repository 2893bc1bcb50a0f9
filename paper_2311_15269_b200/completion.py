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
import gc
import os

import numpy as np
from collections import deque
import time
from collections.abc import Sequence
from dataclasses import dataclass, field
from typing import Optional

from .engine import TRACE as ENGINE_TRACE
from .engine import (VERIFY_SLOTS, WINDOW_FIRST, WINDOW_GROWTH, WINDOW_MAX,
                     BatchedRepetendSearch)
from .parallel import SoloComm, split_range
from .placement import BlockInstance, PlacementSpec
from .repetend import (Repetend, RepetendOutcome, entry_memory, lower_bound, make_repetend,
                       steady_memory_ok)
from .schedule import RepetendInfo, Schedule
from . import _core
from .solver import (Lowering, SolveRequest, SolveStats, Status, default_budget, solve_decide,
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
        self._pending: list = []  # (count, specials) of segments awaiting set_infeasible
        self._size = 0
        self.counts: dict = {}

    def add_segment(self, n_r: int, r0: int, count: int, special: dict,
                    infeasible: Optional[int]):
        """Window [r0, r0 + count) of n_r with its explicit records;
        ``infeasible`` = its gate-rejected count, or None when it is supplied
        later by ``set_infeasible`` (sharded windows: reduced at the end)."""
        self._pending.append((count, len(special)))
        if count > 0:
            self._starts.append(self._size)
            self._segs.append((n_r, r0, count))
            for off, rec in special.items():
                self._special[self._size + off] = rec
                self.counts[rec.status] = self.counts.get(rec.status, 0) + 1
            self._size += count
        if infeasible is not None:
            self.set_infeasible([infeasible])

    def set_infeasible(self, counts):
        """Gate-rejected counts of the segments added without one, in order."""
        for infeasible in counts:
            count, n_special = self._pending.pop(0)
            if infeasible:
                self.counts["infeasible"] = self.counts.get("infeasible", 0) + infeasible
            bound = count - n_special - infeasible
            if bound:
                self.counts["bound"] = self.counts.get("bound", 0) + bound

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
    horizon under a 2M-node cap (completion.py:156-182).  Both decides run in
    one batched launch; the cooldown's outcome and statistics only count when
    the warmup is SAT, as in the reference's sequential evaluation."""
    phases = (
        (warmup_blocks(rep), (0,) * p.num_devices),
        (cooldown_blocks(rep),
         tuple(max(0, v) for v in cooldown_entry_memory(p, rep, rep.n_r))),
    )
    probs = []  # per phase: the decide problem, or None (empty phase / bounds refute)
    for insts, init in phases:
        if not insts:
            probs.append("empty")
            continue
        horizon = sum(p.block(b.stage).time_cost for b in insts)
        low = Lowering(SolveRequest(p, tuple(sorted(insts)), init, cap, horizon, "decide"))
        probs.append(low.problem(horizon, LAZY_CHECK_NODES))
    batch = [q for q in probs if isinstance(q, dict)]
    t0 = time.monotonic()
    outs = iter(_core.decide_batch(batch, deadline) if batch else [])
    wall = time.monotonic() - t0
    for q in probs:
        if q == "empty":
            continue
        if q is None:  # a fixed block misses the horizon: UNSAT without a decide
            return False
        status, _, nodes = next(outs)
        report.stats.decides += 1
        report.stats.nodes += nodes
        report.stats.wall_secs += wall / len(batch)
        if status != _core.SAT:
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
        self.trace = None  # engine trace list (TESSEL_TRACE=1): one entry per evaluation

    def evaluate(self, rep: Repetend):
        # lazy checks depend on the assignment only (warmup / cooldown sets and
        # entry memory); an eager completion also places copy 0 from the
        # witness, so it is keyed by the whole repetend
        key = rep.assignment if self.lazy else (rep.assignment, rep.internal, rep.period)
        if key not in self.memo:
            t0 = time.perf_counter()
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
            if self.trace is not None:
                t1 = time.perf_counter()
                self.trace.append((rep.n_r, 0, rep.period, "feasible", round((t1 - t0) * 1e3, 3),
                                   {"ok": int(ok), "t": round(t1, 4)}))
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

_IMPROVED, _COMPLETION_INFEASIBLE = 1, 2


def search(p: PlacementSpec, mem_capacity: Optional[int] = None, max_nr: Optional[int] = None,
           lazy: bool = True, budget: Optional[float] = None, jobs: int = 1,
           device: Optional[int] = None, engine: Optional[BatchedRepetendSearch] = None,
           comm=None) -> SearchResult:
    """Two-phase schedule search: repetend construction, then completion
    (completion.py:284-396).  ``jobs`` is accepted for API compatibility;
    candidate parallelism comes from the GPU windows instead of a process
    pool.  ``device`` selects the CUDA device (default: current).  ``comm``
    (parallel.Comm) shards every window across the processes of a
    torch.distributed group, one GPU each; every rank returns the same
    result.

    ``report.stats.decides`` is the reference's decide count (every period
    probe its sequential scan would run, plus the completion decides);
    ``report.stats.nodes`` counts the completion decides' nodes exactly and
    the repetend probes' nodes as explored here (the root filter and the
    disjunctive refutation settle most probes without the reference's DFS,
    so its node total is not reproduced).  ``report.engine`` holds this
    search's GPU counters."""
    # the cyclic garbage collector stays off during the search: the scan
    # allocates many short-lived host objects per level and a full
    # collection over the caller's heap stalled single searches by
    # 0.2-0.6 s (profiles/r02i_e2e_var.log); reference counting frees them
    paused = gc.isenabled()
    if paused:
        gc.disable()
    try:
        return _search(p, mem_capacity, max_nr, lazy, budget, jobs, device, engine, comm)
    finally:
        if paused:
            gc.enable()


def _search(p, mem_capacity, max_nr, lazy, budget, jobs, device, engine, comm):
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

    coll = comm if comm is not None else SoloComm()
    root = coll.rank == 0
    eng = engine if engine is not None else BatchedRepetendSearch(p, device or 0)
    c_start = dict(eng.counters.__dict__)
    log = CandidateLog(p, cap, eng.unrank)
    report.candidates = log
    feas = _Feasibility(p, cap, lazy, deadline)
    if ENGINE_TRACE:
        feas.trace = eng.counters.trace
    k = p.num_stages

    def feasible(n_r, rank, period, starts):
        rep = make_repetend(p, eng.unrank(n_r, rank), [int(v) for v in starts], period)
        return feas.ok(rep)

    def span(opt: int) -> int:
        """Periods the reference's scan probes for a candidate with no SAT
        below ``opt`` (repetend.py:272-302)."""
        return max(0, min(total, opt - 1) - lb + 1)

    best: Optional[Repetend] = None
    best_completed: Optional[Schedule] = None
    optimal = total + 1
    done = False
    past_deadline = False       # agreed by every rank at each gather
    acct = {"decides": 0, "infeasible": []}  # this rank's share, reduced at the end
    t_rep = time.monotonic()

    def windows():
        """(n_r, r0, r1) in the reference's candidate order, windows growing
        (one window per rank at a time)."""
        for n_r in range(1, max(limit, 1) + 1):
            count = eng.count(n_r)
            r0, width = 0, WINDOW_FIRST * coll.size
            while r0 < count:
                r1 = min(count, r0 + width)
                yield n_r, r0, r1
                r0 = r1
                width = min(width * WINDOW_GROWTH, WINDOW_MAX * coll.size)

    def gather(r0, a0, win, optimal_now, launched=False):
        """All shards' first SATs of a window (window-relative index ->
        (period, starts)), the window prefix whose outcomes are known and
        whether any shard launched a verification."""
        nonlocal past_deadline
        rows = np.zeros((len(win.first_sat), k + 2), dtype=np.int64)
        for i, (w, (period, starts)) in enumerate(sorted(win.first_sat.items())):
            rows[i, 0], rows[i, 1] = a0 - r0 + w, period
            rows[i, 2:] = starts
        cut = a0 - r0 + win.determined_prefix(optimal_now)
        if not win.timed_out:
            cut = 1 << 62
        allrows, heads = coll.gather_rows(rows, [cut, int(time.monotonic() > deadline),
                                                 int(launched)])
        past_deadline = any(h[1] for h in heads)
        cut = min(h[0] for h in heads)
        first_sat = {int(r[0]): (int(r[1]), r[2:]) for r in allrows}
        return first_sat, cut, any(h[2] for h in heads)

    def replay(n_r, r0, r1, a0, win) -> bool:
        """Ordered replay of a window's first SATs (completion.py:351-382);
        True = the search ends (load bound reached or out of time)."""
        nonlocal best, best_completed, optimal
        opt0 = optimal
        first_sat, cut, _ = gather(r0, a0, win, optimal)
        timed_out = cut < (1 << 62)
        used = min(r1 - r0, cut)
        msg, error = None, None
        if root:  # the improvement rule and the completion checks, rank 0 only
            decisions, stop, opt = [], False, optimal
            try:
                for widx in sorted(first_sat):
                    if widx >= used:
                        break
                    period, starts = first_sat[widx]
                    if period >= opt:
                        continue  # first SAT beyond this candidate's bound: "bound"
                    rep = make_repetend(p, eng.unrank(n_r, r0 + widx),
                                        [int(v) for v in starts], period)
                    ok, sched = feas.replay(rep, report)
                    if ok:
                        opt = rep.period
                        if not lazy:
                            best_completed = sched
                    decisions += [widx, _IMPROVED if ok else _COMPLETION_INFEASIBLE]
                    if ok and opt == lb:
                        stop, used = True, widx + 1
                        break
            except CompletionTimeout as e:  # eager mode: fatal, as in the reference
                error = e
            msg = [used, int(stop), int(error is not None)] + decisions
        msg = coll.bcast_ints(msg)
        used, stop, decisions = msg[0], bool(msg[1]), msg[3:]
        if msg[2]:
            text = coll.bcast_obj(str(error) if root else None)
            raise error if error is not None else CompletionTimeout(text)
        special: dict = {}
        points = []  # (widx, bound from widx + 1 on) for the decide accounting
        for i in range(0, len(decisions), 2):
            widx, code = decisions[i], decisions[i + 1]
            period, starts = first_sat[widx]
            a = eng.unrank(n_r, r0 + widx)
            rep = make_repetend(p, a, [int(v) for v in starts], period)
            if root:  # the reference's probes for this candidate: lb..first SAT
                acct["decides"] += (period - lb + 1) - span(optimal)
            if code == _IMPROVED:
                best, optimal = rep, rep.period
                report.improvements.append((a, optimal))
                points.append((widx, optimal))
            special[widx] = CandidateRecord(n_r, a, rep.period,
                                            "improved" if code == _IMPROVED
                                            else "completion-infeasible")
        # this rank's share: reference decides of every candidate that
        # passes the memory gate, at the bound in force at its index
        lo_w, hi_w = a0 - r0, min(a0 - r0 + win.count, used)
        gate = win.gate  # 0/1 per candidate of this shard; None: no memory gate

        def n_pass(i0, i1):  # window-relative [i0, i1) within this shard
            i0, i1 = max(i0, lo_w), min(i1, hi_w)
            if i1 <= i0:
                return 0
            if gate is None:
                return i1 - i0
            return int(np.count_nonzero(gate[i0 - lo_w:i1 - lo_w]))

        opt, prev = opt0, 0
        for widx, new_opt in points:
            acct["decides"] += n_pass(prev, widx + 1) * span(opt)
            opt, prev = new_opt, widx + 1
        acct["decides"] += n_pass(prev, used) * span(opt)
        acct["infeasible"].append(max(0, hi_w - lo_w) - n_pass(lo_w, hi_w))
        log.add_segment(n_r, r0, used, special, None)
        if timed_out and not stop:
            report.timed_out = True
            return True
        return stop

    def predicted_optimal(n_r, r0, a0, job, opt):
        """The bound after replaying `job`'s window from bound `opt` if its
        speculation holds: the replay rule run without side effects
        (memoised completion checks); computed on rank 0 and broadcast.
        Also whether any shard has pending probes under verification."""
        first_sat, _, launched = gather(r0, a0, job.res, opt, job.launched)
        if root:
            for widx in sorted(first_sat):
                period, starts = first_sat[widx]
                if period >= opt:
                    continue
                rep = make_repetend(p, eng.unrank(n_r, r0 + widx), [int(v) for v in starts],
                                    period)
                if feas.ok(rep):
                    opt = rep.period
        return coll.bcast_ints([opt] if root else None)[0], launched

    pipelined = PIPELINE_WINDOWS and hasattr(eng, "begin_window")
    # windows scanned whose pending probes are being verified, oldest first:
    # [n_r, r0, r1, a0, job, bound the window was scanned under, predicted bound
    #  after it, any shard verifying]
    inflight: deque = deque()

    def settle_head() -> bool:
        """Finish and replay the oldest window in flight; True = the search
        ends (load bound reached or out of time)."""
        pn, p0, p1, pa, pjob, _, _, _ = inflight.popleft()
        pwin = eng.finish_window(pjob, feasible)
        return replay(pn, p0, p1, pa, pwin)

    def redo_mispredicted() -> bool:
        """The next window in flight was scanned under a predicted bound; a
        true bound above it (a repaired / rescanned misprediction) means it
        missed periods: redo it and every later one, in order, exactly."""
        if not inflight or optimal <= inflight[0][5]:
            return False
        redo = list(inflight)
        inflight.clear()  # their verification results are dropped
        for rn, q0, q1, qa, qjob, _, _, _ in redo:
            qb = qa + qjob.res.count
            win = eng.evaluate_window(rn, qa, qb, cap, optimal, feasible, deadline)
            if replay(rn, q0, q1, qa, win):
                return True
        return False

    for n_r, r0, r1 in windows():
        if past_deadline or (comm is None and time.monotonic() > deadline):
            report.timed_out = True
            break  # windows already scanned are still settled below
        a0, b0 = split_range(r0, r1, coll.rank, coll.size)
        if not pipelined:
            win = eng.evaluate_window(n_r, a0, b0, cap, optimal, feasible, deadline)
            if replay(n_r, r0, r1, a0, win):
                done = True
                break
            continue
        # Scan this window while the pending probes of up to PIPELINE_DEPTH
        # earlier windows are verified (one stream each), under the bound
        # their replays yield if their speculation holds (else the true bound
        # is lower: the scan only did extra work); windows are settled and
        # replayed strictly in order.
        bound = inflight[-1][6] if inflight else optimal
        busy = {e[4].slot for e in inflight}
        slot = next(s for s in range(VERIFY_SLOTS) if s not in busy)
        job = eng.begin_window(n_r, a0, b0, cap, bound, feasible, deadline, slot)
        after, launched = predicted_optimal(n_r, r0, a0, job, bound)
        inflight.append([n_r, r0, r1, a0, job, bound, after, launched])
        # settle the oldest while too many are in flight, and every head
        # with nothing to verify (it settles without waiting)
        while inflight and (len(inflight) > PIPELINE_DEPTH or not inflight[0][7]):
            if settle_head() or redo_mispredicted():
                done = True
                break
        if done:
            break
    while inflight and not done:
        if settle_head() or redo_mispredicted():
            break
    report.phase_secs["repetend"] += time.monotonic() - t_rep

    # reduce this rank's accounting: status counts per segment and decides
    red = coll.allreduce_sum([acct["decides"]] + acct["infeasible"])
    log.set_infeasible(red[1:])
    report.stats.decides += red[0]
    c = eng.counters
    report.engine = {key: (v - c_start[key] if isinstance(v, (int, float)) else v)
                     for key, v in c.__dict__.items() if key != "trace"}
    report.stats.nodes += c.nodes - c_start["nodes"]
    report.best_t_r = best.period if best else None

    def finish():
        nonlocal best_completed
        if best is None:
            if report.timed_out:
                return None
            raise NoFeasibleSchedule("no repetend candidate is schedulable under memory")
        if lazy or best_completed is None:
            best_completed = complete_schedule(p, best, cap, deadline, report)
        return best_completed

    if comm is None:
        return SearchResult(finish(), report)
    # rank 0 completes the schedule; every rank returns the same result
    out = None
    if root:
        try:
            s = finish()
            out = {"entries": None if s is None else [(b.stage, b.mb, t)
                                                      for b, t in s.entries.items()],
                   "info": None if s is None else s.repetend}
        except (NoFeasibleSchedule, CompletionTimeout) as e:
            out = {"error": (type(e).__name__, str(e))}
        out.update(diagnostics=report.diagnostics, phase_secs=report.phase_secs,
                   stats=(report.stats.decides, report.stats.nodes, report.stats.wall_secs),
                   timed_out=report.timed_out)
    out = coll.bcast_obj(out)
    report.diagnostics, report.phase_secs = out["diagnostics"], out["phase_secs"]
    report.stats.decides, report.stats.nodes, report.stats.wall_secs = out["stats"]
    report.timed_out = out["timed_out"]
    if "error" in out:
        name, msg = out["error"]
        raise (NoFeasibleSchedule if name == "NoFeasibleSchedule" else CompletionTimeout)(msg)
    if out["entries"] is None:
        return SearchResult(None, report)
    entries = {BlockInstance(st, mb): t for st, mb, t in out["entries"]}
    return SearchResult(Schedule(p, best.n_r, entries, out["info"]), report)
