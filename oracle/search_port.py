"""ORACLE — test infrastructure only (see oracle/__init__.py).

Sequential Python restatement of the reference search path on top of the C
decide restatement (oracle/decide_port.c):

* repetend probes and the period scan — repetend.py:60-328
* lowering, lower bound, decide / min-makespan binary search — solver.py:96-325
* lazy completion check, complete_schedule, Algorithm-1 search — completion.py:107-396

Semantics are the reference's, including node caps (400k per repetend probe
above the load bound, 8M per completion probe, 2M per lazy check); the wall
budget is not modelled (parity runs disable it).
Uses the product's placement/schedule *data model* only (pinned separately
against the reference's JSON).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional

from . import SAT, TIMEOUT, UNSAT, decide
from paper_2311_15269_b200.placement import BlockInstance
from paper_2311_15269_b200.schedule import RepetendInfo, Schedule

PROBE_NODES = 400_000          # repetend.py:21
COMPLETION_NODES = 8_000_000   # solver.py:29
LAZY_NODES = 2_000_000         # completion.py:178


# ---------------------------------------------------------------- repetend
def lower_bound(p):
    return max(p.device_load(d) for d in range(p.num_devices))   # repetend.py:60-62


def iter_assignments(p, n_r):
    """repetend.py:65-90 (lexicographic, n_i >= n_j on i->j, min index 0)."""
    k = p.num_stages
    succ = [p.successors(s) for s in range(k)]
    pred = [p.predecessors(s) for s in range(k)]
    vec = [0] * k

    def rec(st, cur_min):
        if st == k:
            if cur_min == 0:
                yield tuple(vec)
            return
        lo = max([0] + [vec[j] for j in succ[st] if j < st])
        hi = min([n_r - 1] + [vec[i] for i in pred[st] if i < st])
        for v in range(lo, hi + 1):
            vec[st] = v
            yield from rec(st + 1, min(cur_min, v))

    yield from rec(0, n_r)


def entry_memory(p, a):
    out = [0] * p.num_devices                                      # repetend.py:93-100
    for st, n in enumerate(a):
        b = p.block(st)
        for d in b.devices:
            out[d] += n * b.mem_delta
    return tuple(out)


def steady_memory_ok(p):
    return all(v <= 0 for v in p.net_mem_per_device())             # repetend.py:103-105


class ProbeModel:
    """repetend.py:108-190: per-placement arrays, lag = base - coef*P."""

    def __init__(self, p):
        k = p.num_stages
        self.p, self.k = p, k
        self.dur = [p.block(s).time_cost for s in range(k)]
        self.mask = [sum(1 << d for d in p.block(s).devices) for s in range(k)]
        self.mem = [p.block(s).mem_delta for s in range(k)]
        self.order = sorted(range(k), key=lambda s: (-len(p.block(s).devices), s))
        dep = sorted(p.deps)
        win = []
        for d in range(p.num_devices):
            sts = p.device_stages(d)
            win += [(x, y) for x in sts for y in sts if x != y]
        self.rows = dep + win
        self.n_dep = len(dep)
        self.max_dur = max(self.dur) if k else 1

    def edges(self, a, period):
        out = []
        for r, (x, y) in enumerate(self.rows):
            coef = a[x] - a[y] if r < self.n_dep else 1
            out += [x, y, self.dur[x] - coef * period]
        return out

    def bounds(self, period):
        anchor = (self.k - 1) * (period + self.max_dur)
        lo = [0] * self.k
        hi = [2 * anchor] * self.k
        lo[0] = hi[0] = anchor
        return lo, hi

    def probe(self, a, period, cap, entry, node_budget=0):
        lo, hi = self.bounds(period)
        return decide(self.k, self.dur, self.mask, self.mem, self.edges(a, period), self.order,
                      lo, hi, self.p.num_devices, list(entry), -1 if cap is None else cap,
                      node_budget, 0.0)


def compact_period(p, internal, a):
    """repetend.py:220-250."""
    spans = []
    for d in range(p.num_devices):
        sts = p.device_stages(d)
        if not sts:
            spans.append(0)
            continue
        spans.append(max(internal[s] + p.block(s).time_cost for s in sts) - min(internal[s] for s in sts))
    period = max(1, max(spans))
    for i, j in p.deps:
        delta = a[i] - a[j]
        if delta < 0:
            raise ValueError("assignment violates the descending-index property")
        if delta > 0:
            need = internal[i] + p.block(i).time_cost - internal[j]
            if need > 0:
                period = max(period, -(-need // delta))
    return period, tuple(spans), tuple(period - e for e in spans)


@dataclass
class RepOut:
    status: str
    assignment: tuple = ()
    internal: Optional[tuple] = None
    period: Optional[int] = None
    spans: tuple = ()
    waits: tuple = ()
    entry: tuple = ()
    n_r: int = 0
    probes: int = 0
    nodes: int = 0


def solve_repetend(p, a, cap, upper=None, model=None):
    """repetend.py:253-328 (monotone assignments; no wall budget)."""
    model = model or ProbeModel(p)
    entry = entry_memory(p, a)
    if cap is not None and (any(e > cap for e in entry) or not steady_memory_ok(p)):
        return RepOut("infeasible")
    lb = lower_bound(p)
    ub = sum(b.time_cost for b in p.blocks)
    if upper is not None:
        ub = min(ub, upper - 1)
    if ub < lb:
        return RepOut("bound")
    monotone = all(a[i] >= a[j] for i, j in p.deps)
    out = RepOut("bound" if upper is not None else "infeasible")
    for P in range(lb, ub + 1):
        st, w, nodes = model.probe(a, P, cap, entry, 0 if P == lb else PROBE_NODES)
        out.probes += 1
        out.nodes += nodes
        if st == TIMEOUT:
            if not monotone:
                out.status = "timeout"
                return out
            continue
        if st == SAT:
            base = min(w)
            internal = tuple(v - base for v in w)
            if monotone:
                per, spans, waits = compact_period(p, internal, a)
            else:
                per = P
                spans = []
                for d in range(p.num_devices):
                    sts = p.device_stages(d)
                    spans.append(max(internal[s] + p.block(s).time_cost for s in sts)
                                 - min(internal[s] for s in sts) if sts else 0)
                spans = tuple(spans)
                waits = tuple(per - e for e in spans)
            return RepOut("ok", tuple(a), internal, per, spans, waits, entry, max(a) + 1,
                          out.probes, out.nodes)
    return out


# ---------------------------------------------------------------- solver
class Lowered:
    """solver.py:96-167."""

    def __init__(self, p, instances, init, cap, fixed=(), min_starts=()):
        fixed_map = dict(fixed)
        free = sorted(instances)
        self.items = sorted(fixed_map) + free
        self.n_fixed = len(fixed_map)
        idx = {b: k for k, b in enumerate(self.items)}
        self.n = len(self.items)
        self.dur = [p.block(b.stage).time_cost for b in self.items]
        self.mem = [p.block(b.stage).mem_delta for b in self.items]
        self.mask = [sum(1 << d for d in p.block(b.stage).devices) for b in self.items]
        ms = dict(min_starts)
        self.lo = [fixed_map[b] if b in fixed_map else max(0, ms.get(b, 0)) for b in self.items]
        present = set(self.items)
        edges = []
        for i, j in sorted(p.deps):
            ti = p.block(i).time_cost
            for b in self.items:
                if b.stage == i and BlockInstance(j, b.mb) in present:
                    edges.append((idx[b], idx[BlockInstance(j, b.mb)], ti))
        by_stage = {}
        for b in free:
            by_stage.setdefault(b.stage, []).append(b)
        for st, insts in by_stage.items():
            t = p.block(st).time_cost
            insts.sort()
            for x, y in zip(insts, insts[1:]):
                if y.mb == x.mb + 1:
                    edges.append((idx[x], idx[y], t))
        self.edges = edges
        self.cap = -1 if cap is None else cap
        self.init = list(init)
        self.ndev = p.num_devices

    def fixed_max_end(self):
        return max([0] + [self.lo[k] + self.dur[k] for k in range(self.n_fixed)])

    def makespan(self, s):
        return max(a + d for a, d in zip(s, self.dur))


def run_decide(low, horizon, budget):
    """solver.py:191-209."""
    lo = list(low.lo)
    big = sum(low.dur) + max(lo, default=0) + 1
    hi = lo[:low.n_fixed] + [big] * (low.n - low.n_fixed)
    if horizon is not None:
        for k in range(low.n):
            c = horizon - low.dur[k]
            if k < low.n_fixed:
                if lo[k] > c:
                    return UNSAT, None, 0
            else:
                hi[k] = c
                if hi[k] < lo[k]:
                    return UNSAT, None, 0
    flat = [v for e in low.edges for v in e]
    return decide(low.n, low.dur, low.mask, low.mem, flat, list(range(low.n)), lo, hi,
                  low.ndev, low.init, low.cap, budget, 0.0)


def lowered_lower_bound(low):
    """solver.py:212-237."""
    lo = list(low.lo)
    changed, passes = True, 0
    while changed and passes <= low.n + 1:
        changed = False
        passes += 1
        for a, b, lag in low.edges:
            if lo[a] + lag > lo[b]:
                lo[b] = lo[a] + lag
                changed = True
    bound = max([0] + [lo[k] + low.dur[k] for k in range(low.n)])
    for d in range(low.ndev):
        c = 0
        for t0, du in sorted((lo[k], low.dur[k]) for k in range(low.n) if low.mask[k] >> d & 1):
            c = max(c, t0) + du
        bound = max(bound, c)
    return bound


def min_makespan(low, horizon=None, pn=COMPLETION_NODES):
    """solver.py:264-325 -> (status, starts|None) with status in
    optimal|infeasible|timeout."""
    lb = max(lowered_lower_bound(low), low.fixed_max_end())
    ub = low.fixed_max_end() + sum(low.dur[low.n_fixed:])
    for k in range(low.n):
        ub = max(ub, low.lo[k] + low.dur[k])
    if horizon is not None:
        ub = min(ub, horizon)
        if ub < lb:
            return "infeasible", None
    st, s, _ = run_decide(low, ub, pn)
    if st == UNSAT:
        return "infeasible", None
    if st == TIMEOUT:
        return "timeout", None
    best, hi, best_h, lo_h = s, low.makespan(s), None, lb
    best_h = hi
    while lo_h < hi:
        mid = (lo_h + hi) // 2
        st, s, _ = run_decide(low, mid, pn)
        if st == SAT:
            hi = low.makespan(s)
            best, best_h = s, mid
        elif st == UNSAT:
            lo_h = mid + 1
        else:
            return "timeout", best
    if best_h != hi:
        st, s, _ = run_decide(low, hi, pn)
        if st == SAT:
            best = s
        elif st == TIMEOUT:
            return "timeout", best
    return "optimal", best


# ---------------------------------------------------------------- completion
def warmup_blocks(a):
    return {BlockInstance(st, n) for st, r in enumerate(a) for n in range(r)}


def cooldown_blocks(a, n_r):
    return {BlockInstance(st, n) for st, r in enumerate(a) for n in range(r + 1, n_r)}


def completion_feasible(p, rep, cap):
    """completion.py:156-182."""
    net = p.net_mem_per_device()
    reps = 1
    cd_init = tuple(max(0, e + reps * net[d]) for d, e in enumerate(rep.entry))
    for inst, init in ((warmup_blocks(rep.assignment), (0,) * p.num_devices),
                       (cooldown_blocks(rep.assignment, rep.n_r), cd_init)):
        if not inst:
            continue
        horizon = sum(p.block(b.stage).time_cost for b in inst)
        if cap is not None and any(not 0 <= v <= cap for v in init):
            raise ValueError("initial_memory outside [0, cap]")
        low = Lowered(p, tuple(sorted(inst)), init, cap)
        st, _, _ = run_decide(low, horizon, LAZY_NODES)
        if st != SAT:
            return False
    return True


def complete_schedule(p, rep, cap, diagnostics=None):
    """completion.py:185-274."""
    diagnostics = diagnostics if diagnostics is not None else []
    entries = {}
    wu = tuple(sorted(warmup_blocks(rep.assignment)))
    w_end = 0
    if wu:
        low = Lowered(p, wu, (0,) * p.num_devices, cap)
        st, s = min_makespan(low)
        if st == "timeout" and s is None:
            raise RuntimeError("CompletionTimeout: warmup")
        if st == "infeasible":
            raise RuntimeError("NoFeasibleSchedule: warmup")
        if st == "timeout":
            diagnostics.append(f"warmup completed at {low.makespan(s)} but optimality is unproven")
        entries.update({low.items[k]: s[k] for k in range(low.n_fixed, low.n)})
        w_end = low.makespan(s)
    offset = w_end
    span = max(rep.internal[st] + p.block(st).time_cost for st in range(p.num_stages))
    for st, n in enumerate(rep.assignment):
        entries[BlockInstance(st, n)] = offset + rep.internal[st]
    cd = tuple(sorted(cooldown_blocks(rep.assignment, rep.n_r)))
    if cd:
        win = {}
        for d in range(p.num_devices):
            sts = p.device_stages(d)
            if sts:
                win[d] = offset + min(rep.internal[s] for s in sts)
        ms = tuple((b, max((win[d] for d in p.block(b.stage).devices), default=0)) for b in cd)
        low = Lowered(p, cd, (0,) * p.num_devices, cap, fixed=tuple(sorted(entries.items())),
                      min_starts=ms)
        st, s = min_makespan(low)
        if st == "timeout" and s is None:
            raise RuntimeError("CompletionTimeout: cooldown")
        if st == "infeasible":
            raise RuntimeError("NoFeasibleSchedule: cooldown")
        if st == "timeout":
            diagnostics.append(f"cooldown completed at {low.makespan(s)} but optimality is unproven")
        entries.update({low.items[k]: s[k] for k in range(low.n_fixed, low.n)})
    info = RepetendInfo(offset, offset + span, rep.period, rep.n_r)
    return Schedule(p, rep.n_r, entries, info)


@dataclass
class PortResult:
    schedule: Optional[Schedule]
    best: Optional[RepOut]
    improvements: list = field(default_factory=list)
    n_candidates: int = 0
    status_counts: dict = field(default_factory=dict)
    probes: int = 0
    nodes: int = 0
    diagnostics: list = field(default_factory=list)
    wall: float = 0.0


def search(p, mem_capacity=None, max_nr=None, time_limit=None):
    """completion.py:284-396, lazy mode, jobs=1.  ``time_limit`` (seconds)
    stops the candidate loop early for bounded CPU-baseline samples; the
    result is then partial and ``schedule`` is None."""
    t0 = time.perf_counter()
    cap = mem_capacity
    lb = lower_bound(p)
    total = sum(b.time_cost for b in p.blocks)
    limit = 8 if max_nr is None else max_nr
    if cap is not None:
        infl = None
        for d in range(p.num_devices):
            run = peak = 0
            for st in p.device_stages(d):
                run += p.block(st).mem_delta
                peak = max(peak, run)
            if peak > 0:
                infl = cap // peak if infl is None else min(infl, cap // peak)
        if infl is not None:
            limit = min(limit, infl)
        if not steady_memory_ok(p):
            raise RuntimeError("NoFeasibleSchedule: net memory > 0")
    model = ProbeModel(p)
    res = PortResult(None, None)
    optimal = total + 1
    done = False
    for n_r in range(1, max(limit, 1) + 1):
        for a in iter_assignments(p, n_r):
            if time_limit is not None and time.perf_counter() - t0 > time_limit:
                res.wall = time.perf_counter() - t0
                return res
            out = solve_repetend(p, a, cap, upper=optimal, model=model)
            res.n_candidates += 1
            res.probes += out.probes
            res.nodes += out.nodes
            status = out.status
            if out.period is not None and out.period < optimal:
                if completion_feasible(p, out, cap):
                    res.best = out
                    optimal = out.period
                    res.improvements.append((tuple(a), optimal))
                    status = "improved"
                    done = optimal == lb
                else:
                    status = "completion-infeasible"
            res.status_counts[status] = res.status_counts.get(status, 0) + 1
            if done:
                break
        if done:
            break
    if res.best is not None:
        res.schedule = complete_schedule(p, res.best, cap, res.diagnostics)
    res.wall = time.perf_counter() - t0
    return res
