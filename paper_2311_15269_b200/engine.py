"""Batched repetend search on the B200 (the hot loop of completion.search).

The reference evaluates candidates one at a time, each with a sequential
period scan (completion.py:318-349 -> repetend.py:253-302).  Here a WINDOW of
consecutive candidate ranks is staged on the GPU (unrank + memory gate,
kernel ``k_stage``) and scanned LEVEL-SYNCHRONOUSLY: at period P every
still-active candidate of the window is probed in one launch (``k_probe``,
reference-exact decide with the reference's node caps).  After each level the
host applies the safe bound rule: the lowest-index
candidate that is SAT at P and completion-feasible retires every
higher-index candidate (their sequential bound is <= P).  The window is then
REPLAYED in index order with the reference's improvement rule
(completion.py:351-382), so improvements, the chosen repetend and the
candidate records are exactly the reference's.

Why this is exact: a probe's outcome depends only on (candidate, P, node cap),
and the cap depends only on whether P is the load bound.  A candidate's
reference scan covers [lb, opt_seq - 1] and stops at the first SAT; the
level scan covers a superset of that range for every candidate that can still
matter, and stops a candidate only when its own first SAT is known or when a
lower-index completion-feasible SAT y at a period <= P bounds it
(opt_seq(x) <= p1_y).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native
from .placement import PlacementSpec
from .repetend import PROBE_NODES, lower_bound

WINDOW_FIRST = int(os.environ.get("TESSEL_WINDOW_FIRST", "2048"))
WINDOW_GROWTH = 4
WINDOW_MAX = 1 << 21
VERIFY_SLOTS = 8      # asynchronous verification slots (TSL_VERIFY_SLOTS)
SAT_CHUNK = 1        # SAT rows returned with a level (the rest: device argmin walk)
SMALL_BUDGET = 64     # first-pass RX-DFS nodes per probe (thread per probe) before deferral
# node cap of the concurrent verify pass; longer probes run one at a time
# through the decide path (subtree-parallel for unlimited / >= 1M caps).
# Default: off — capped repetend probes change their sticky sets too often
# for the speculation to pay (tests/native/sp_sim.cpp model), so they stay
# one warp each, all concurrently.
VERIFY_FIRST = int(os.environ.get("TESSEL_VERIFY_FIRST", str(1 << 40)))
DJ_BUDGET = int(os.environ.get("TESSEL_DJ_BUDGET", "200000"))  # disjunctive nodes per deferred probe
# escalation of deferred probes: (DJ budget, RX-DFS stage budget; 0 = the
# reference cap).  The retirement limit is re-applied between stages, so a
# probe above the lowest completion-feasible SAT never runs the full cap.
RESOLVE_STAGES = ((DJ_BUDGET, 32_768), (0, 0))
# with speculation the RX-DFS stages are replaced by pending probes verified
# once per window (one concurrent launch); -1 = disjunctive filter only.
# TESSEL_SPEC_STAGE overrides the RX budget of the single resolve stage.
SPEC_STAGES = ((DJ_BUDGET, int(os.environ.get("TESSEL_SPEC_STAGE", "65536"))),)


# latency mode of the speculative resolve stage: a level with few deferred
# probes (< SPEC_SMALL_NDEF, all resident at once) is bound by its longest
# probe's stage budget, so its DFS stage stops after SPEC_SMALL nodes and the
# rest goes to the window-end verification, which overlaps the next levels;
# a level with many deferred probes keeps the full stage budget (throughput:
# its early SATs retire the higher candidates)
SPEC_SMALL = int(os.environ.get("TESSEL_SPEC_SMALL", "1024"))
SPEC_SMALL_NDEF = int(os.environ.get("TESSEL_SPEC_SMALL_NDEF", "4096"))


def spec_stages(k: int):
    """The single resolve stage's DFS budget: 64k nodes when every stage fits
    one lane (K <= 32; cut to SPEC_SMALL on levels with few deferred probes),
    SPEC_SMALL when lanes carry two stages (K > 32, ~3x dearer nodes: their
    deferred probes are mostly 400k-node TIMEOUTs that the window-end
    verification settles concurrently; measured with 16k / 1k nodes: C4a@3
    4.5 / 3.0 s, C4a@4 5.3 / 3.6 s, C5@5 5.4 / 4.8 s)."""
    if "TESSEL_SPEC_STAGE" in os.environ:
        return SPEC_STAGES
    return ((DJ_BUDGET, 65536 if k <= 32 else SPEC_SMALL),)
TRACE = os.environ.get("TESSEL_TRACE", "0") == "1"


@dataclass
class EngineCounters:
    """GPU-side work counters (no reference equivalent beyond SolveStats)."""
    windows: int = 0
    levels: int = 0
    probes: int = 0
    root_refuted: int = 0
    nodes: int = 0
    capped: int = 0
    sat: int = 0
    deferred: int = 0
    dj_refuted: int = 0
    dj_nodes: int = 0
    verified: int = 0        # speculated probes verified at window ends
    redo: int = 0            # window rescans after a misprediction
    repaired: int = 0        # mispredictions settled without a rescan
    aborted: int = 0         # verifications cancelled by a lower SAT
    sp_probes: int = 0       # long probes settled by the subtree-parallel decide
    kernel_ms: float = 0.0
    root_ms: float = 0.0      # k_root (root filter, every probe of a level)
    probe_ms: float = 0.0     # survivors' small-budget DFS (k_resolve_warp, no filter)
    resolve_ms: float = 0.0   # k_resolve_warp (disjunctive filter + warp RX-DFS stages)
    verify_ms: float = 0.0    # k_verify_warp (pending speculated probes)
    stage_ms: float = 0.0     # k_stage (unrank + gate)
    launches: int = 0
    trace: list = field(default_factory=list)

    def add(self, st: dict, ms: float, level: bool, tag=None):
        if level:
            self.probe_ms += ms
        else:
            self.resolve_ms += ms
        if TRACE and tag is not None:
            self.trace.append((*tag, round(ms, 3), {**{k: v for k, v in st.items() if v},
                                                     "t": round(time.perf_counter(), 4)}))
        self.levels += level
        self.launches += 1
        for k in ("probes", "root_refuted", "nodes", "capped", "sat", "deferred", "dj_refuted",
                  "dj_nodes"):
            setattr(self, k, getattr(self, k) + st[k])
        self.kernel_ms += ms


@dataclass
class WindowJob:
    """A scanned window whose pending probes are being verified."""
    args: tuple
    res: "WindowResult"
    pending: list
    slot: int
    launched: bool


@dataclass
class WindowResult:
    n_r: int
    r0: int
    count: int
    first_sat: dict = field(default_factory=dict)  # widx -> (period, starts)
    gate: Optional[np.ndarray] = None               # 1 = passes the memory gate
    timed_out: bool = False
    first_feasible: Optional[int] = None            # lowest completion-feasible SAT widx
    retirers: set = field(default_factory=set)      # widx that lowered a retirement limit
    # set when the scan ran out of time: levels lb..level-1 are complete for
    # every candidate <= limit except the unverified (widx, period) pending
    level: int = 0
    limit: int = -1
    pending: list = field(default_factory=list)

    def determined_prefix(self, optimal: int) -> int:
        """Window indices [0, n) whose reference outcome is already known
        for a search whose bound before this window is ``optimal``: every
        candidate of the prefix is gated out, retired, has its first SAT
        with no unverified period below it, or was scanned through
        optimal - 1 (conservative: the bound only falls during the replay)."""
        if not self.timed_out:
            return self.count
        pend: dict = {}
        for w, q in self.pending:
            pend[w] = min(q, pend.get(w, q))
        for w in range(self.count):
            if self.gate is not None and not self.gate[w]:
                continue
            if w > self.limit:
                return self.count  # retired by a lower completion-feasible SAT
            fs = self.first_sat.get(w)
            q = pend.get(w)
            if fs is not None:
                if q is not None and q < fs[0]:
                    return w
            elif (q is not None and q < optimal) or self.level < optimal:
                return w
        return self.count


class BatchedRepetendSearch:
    """One placement resident on one GPU."""

    def __init__(self, p: PlacementSpec, device: int = 0, native=None):
        """``native`` substitutes the low-level engine (tests drive the level
        logic on CPU with an oracle-backed stand-in); default: the sm_100a
        library."""
        self.p = p
        k = p.num_stages
        dur = [p.block(s).time_cost for s in range(k)]
        mem = [p.block(s).mem_delta for s in range(k)]
        masks = [sum(1 << d for d in p.block(s).devices) for s in range(k)]
        self.eng = native if native is not None else _native.Engine(
            dur, mem, masks, sorted(p.deps), p.num_devices, device)
        self.lb = lower_bound(p)
        self.total = sum(dur)
        self.counters = EngineCounters()
        self.small_budget = int(os.environ.get("TESSEL_SMALL_BUDGET", SMALL_BUDGET))
        self.speculate = os.environ.get("TESSEL_SPECULATE", "1") == "1"
        self.resolve_stages = spec_stages(k) if self.speculate else RESOLVE_STAGES
        self.repair = os.environ.get("TESSEL_REPAIR", "1") == "1"
        self._last_ms = 0.0

    def _scan_sats(self, res, n_r, r0, period, n_sat, widx, rows, limit, feasible, extra=()):
        """Walk the level's SATs in window order — the device's ordered
        argmin (the first row comes with the level's result, each next one
        from ``sat_next``), merged with host-known SATs `extra` — up to the
        first completion-feasible one; it retires every higher index."""
        ex = sorted(extra, key=lambda r: r[0])
        xi = 0
        dev = (int(widx[0]), rows[0]) if n_sat and len(widx) else None
        fetch = n_sat > 0 and dev is None  # the next device SAT is still to be fetched
        last, taken = -1, 0
        while True:
            if fetch:
                dev = self.eng.sat_next(last) if taken < n_sat else None
                fetch = False
            if dev is None and xi >= len(ex):
                break
            if xi >= len(ex) or (dev is not None and dev[0] < ex[xi][0]):
                w, row = dev
                last, dev, fetch, taken = w, None, True, taken + 1
            else:
                w, row = ex[xi]
                xi += 1
            if w > limit:
                break
            res.first_sat[w] = (period, np.array(row, dtype=np.int32).copy())
            if feasible(n_r, r0 + w, period, row):
                res.first_feasible = w
                res.retirers.add(w)
                return w - 1
        return limit

    def count(self, n_r: int) -> int:
        return self.eng.count(n_r)

    def unrank(self, n_r: int, rank: int) -> tuple:
        return self.eng.unrank(n_r, rank)

    def close(self):
        self.eng.close()

    # ---- pipelined windows: scan window w+1 while window w is verified ----
    def begin_window(self, n_r: int, r0: int, r1: int, cap: Optional[int], bound: int,
                     feasible, deadline: float = 0.0, slot: int = 0) -> "WindowJob":
        """Scan a window and launch the verification of its pending probes
        asynchronously (its assignments stashed in `slot`), so that the next
        window can be staged and scanned meanwhile.  The scan may run under a
        stale (higher) bound than the exact sequential one: its outcomes are
        facts about (candidate, period) pairs and the ordered replay applies
        the true bound, so only work is added, never a different answer."""
        res, pending = self._scan_window(n_r, r0, r1, cap, bound, feasible, deadline, {})
        job = WindowJob((n_r, r0, r1, cap, bound, deadline), res, pending, slot, False)
        if pending and not res.timed_out:
            self.eng.verify_stash(slot, [x for x, _ in pending])
            self._launch_round(job, list(range(len(pending))))
            job.launched = True
        return job

    def _launch_round(self, job, positions):
        n_r, r0, r1, cap, bound, deadline = job.args
        w = [job.pending[i][0] for i in positions]
        per = [job.pending[i][1] for i in positions]
        bud = [0 if q == self.lb else PROBE_NODES for q in per]
        run_bud = [VERIFY_FIRST if (b == 0 or b > VERIFY_FIRST) else b for b in bud]
        self.eng.verify_launch(job.slot, positions, w, per, run_bud, cap)
        if TRACE:
            self.counters.trace.append((n_r, r0, 0, "vlaunch", 0.0,
                                        {"n": len(w), "slot": job.slot,
                                         "t": round(time.perf_counter(), 4)}))

    def finish_window(self, job: "WindowJob", feasible) -> WindowResult:
        n_r, r0, r1, cap, bound, deadline = job.args
        if job.res.timed_out:
            return job.res
        hints: dict = {}
        first = self.eng.verify_wait(job.slot) if job.launched else None
        index = {xq: i for i, xq in enumerate(job.pending)}

        def run(todo, w, per, run_bud):
            self._launch_round(job, [index[xq] for xq in todo])
            return self.eng.verify_wait(job.slot)

        sats = self._verify_pending(n_r, r0, cap, job.pending, feasible, hints, first=first,
                                    runner=run)
        res = job.res
        fix = self._first_sats(sats)
        if not fix:
            return res
        if not (set(fix) & res.retirers) and self.repair:
            for x, (q, row) in fix.items():
                res.first_sat[x] = (q, row)
            self.counters.repaired += len(fix)
            return res
        self.counters.redo += 1  # rescan (the window is staged again) with the hints
        return self.evaluate_window(n_r, r0, r1, cap, bound, feasible, deadline, hints)

    @staticmethod
    def _first_sats(sats) -> dict:
        fix: dict = {}
        for x, q, row in sats:
            if x not in fix or q < fix[x][0]:
                fix[x] = (q, row)
        return fix

    def evaluate_window(self, n_r: int, r0: int, r1: int, cap: Optional[int], bound: int,
                        feasible: Callable[[int, int, int, np.ndarray], bool],
                        deadline: float = 0.0, hints=None) -> WindowResult:
        """Level-synchronous period scan of ranks [r0, r1) at n_r under the
        sequential bound ``bound`` in force at the window start.
        ``feasible(n_r, rank, period, starts)`` is the completion check.

        Speculation: deferred probes that survive the disjunctive filter
        would need the reference-exact DFS up to the reference's 400k-node cap,
        one latency-bound launch per level.  They are instead assumed "not
        SAT" (the outcome for nearly all of them), the scan continues, and all
        pending probes of the window are verified together in ONE launch at
        the end.  A verified SAT (w, P) is a misprediction: w's first SAT is
        P.  Every other outcome the scan recorded is a fact about its own
        (candidate, period) and retirement only flows to higher indices, so
        unless w itself lowered a retirement limit (its later SAT would not
        exist in the exact scan) the window result is REPAIRED by recording
        (P, row) as w's first SAT: candidates the exact scan would have
        retired at P only carry first SATs at periods >= P, which the ordered
        replay skips once w's period is the bound.  Otherwise the window is
        scanned again with every verified outcome as a hint."""
        hints = {} if hints is None else hints
        for _ in range(1 + 4 * 64):
            res, pending = self._scan_window(n_r, r0, r1, cap, bound, feasible, deadline, hints)
            if res.timed_out:
                return res
            fix: dict = {}
            for x, q, row in self._verify_pending(n_r, r0, cap, pending, feasible, hints):
                if x not in fix or q < fix[x][0]:
                    fix[x] = (q, row)
            mispredicted = bool(fix)
            unsafe = bool(set(fix) & res.retirers)
            if not mispredicted:
                return res
            if not unsafe and self.repair:
                for x, (q, row) in fix.items():
                    res.first_sat[x] = (q, row)
                self.counters.repaired += len(fix)
                return res
            self.counters.redo += 1
        raise RuntimeError("speculation did not converge")

    def _verify_pending(self, n_r, r0, cap, pending, feasible, hints, first=None, runner=None):
        """Settle the window's pending (speculated) probes in concurrent
        launches.  The kernel lets a SAT (x, q) cancel pairs (x2, q2) with
        x2 > x and q2 >= q; a cancelled pair is re-run unless such a SAT
        passes its completion check (then the exact scan retires x2 at q and
        its outcome is never used).  Returns the verified SATs (x, q, row)."""
        sats = []
        todo = list(pending)

        def justified(x2, q2):
            return any(x < x2 and q <= q2 and feasible(n_r, r0 + x, q, row)
                       for x, q, row in sorted(sats, key=lambda r: r[:2]))

        while todo:
            w = [x for x, _ in todo]
            per = [q for _, q in todo]
            bud = [0 if q == self.lb else PROBE_NODES for q in per]
            # one concurrent launch settles the probes that end within
            # VERIFY_FIRST nodes; longer ones run one at a time through the
            # subtree-parallel decide (sp_dfs.cuh) below
            run_bud = [VERIFY_FIRST if (b == 0 or b > VERIFY_FIRST) else b for b in bud]
            if first is not None:  # round 1 already ran asynchronously (begin_window)
                st, nodes, rows = first
                first = None
            elif runner is not None:
                st, nodes, rows = runner(todo, w, per, run_bud)
            else:
                st, nodes, rows = self.eng.verify(w, per, run_bud, cap)
            self.counters.add({"probes": 0, "root_refuted": 0, "nodes": int(nodes.sum()),
                               "capped": int((st == _native.TIMEOUT).sum()),
                               "sat": int((st == _native.SAT).sum()), "deferred": 0,
                               "dj_refuted": 0, "dj_nodes": 0},
                              self.eng.last_kernel_ms(), False, (n_r, r0, 0, "verify"))
            self.counters.resolve_ms -= self.eng.last_kernel_ms()
            self.counters.verify_ms += self.eng.last_kernel_ms()
            self.counters.verified += len(w)
            again, long = [], []
            for i, (x, q) in enumerate(todo):
                s = int(st[i])
                if s == _native.ABORT:
                    again.append((x, q))
                    continue
                if s == _native.TIMEOUT and run_bud[i] != bud[i]:
                    long.append((x, q, bud[i]))
                    continue
                hints[(x, q)] = (s, rows[i].copy())
                if s == _native.SAT:
                    sats.append((x, q, rows[i].copy()))
            for x, q, b in sorted(long):
                if justified(x, q):
                    continue  # retired at q by a lower completion-feasible SAT
                s, row, nd = self._long_probe(n_r, r0 + x, q, cap, b)
                self.counters.add({"probes": 0, "root_refuted": 0, "nodes": nd,
                                   "capped": int(s == _native.TIMEOUT),
                                   "sat": int(s == _native.SAT), "deferred": 0,
                                   "dj_refuted": 0, "dj_nodes": 0},
                                  self._last_ms, False, (n_r, r0, q, "verify-sp"))
                self.counters.sp_probes += 1
                hints[(x, q)] = (s, row)
                if s == _native.SAT:
                    sats.append((x, q, row))
            self.counters.aborted += len(again)
            todo = [(x2, q2) for x2, q2 in again if not justified(x2, q2)]
        return sats

    def _long_probe(self, n_r, rank, period, cap, budget):
        """One repetend probe as a general reference decide (the lowering of
        repetend.py:108-190 in repetend._CandidateModel), which the decide
        path runs subtree-parallel when it is long."""
        from . import _core
        from .repetend import _model_for, entry_memory

        a = self.eng.unrank(n_r, rank)
        m = _model_for(self.p)
        m.set_assignment(a)
        anchor = (m.k - 1) * (period + m.max_dur)
        lo = [0] * m.k
        hi = [2 * anchor] * m.k
        if m.k:
            lo[0] = hi[0] = anchor
        t0 = time.perf_counter()
        status, starts, nodes = _core.decide(
            m.k, m.dur, m.mask, m.mem, m.edges(period), m.order, lo, hi, self.p.num_devices,
            list(entry_memory(self.p, a)), -1 if cap is None else cap, budget, 0.0)
        self._last_ms = (time.perf_counter() - t0) * 1e3
        row = np.array(starts if starts is not None else [0] * m.k, dtype=np.int32)
        return int(status), row, int(nodes)

    def _scan_window(self, n_r, r0, r1, cap, bound, feasible, deadline, hints):
        res = WindowResult(n_r, r0, r1 - r0)
        pending = []
        n_act, gate = self.eng.stage(n_r, r0, r1, cap, want_gate=cap is not None)
        self.counters.windows += 1
        self.counters.launches += 1  # k_stage
        self.counters.kernel_ms += self.eng.last_kernel_ms()
        self.counters.stage_ms += self.eng.last_kernel_ms()
        res.gate = gate
        limit = res.count - 1
        top = min(self.total, bound - 1)
        active = n_act > 0

        def out_of_time(level):
            res.timed_out, res.level, res.limit, res.pending = True, level, limit, pending
            return res, pending

        for period in range(self.lb, top + 1):
            if not active:
                break
            budget_secs = 0.0
            if deadline:
                left = deadline - time.monotonic()
                if left <= 0:
                    return out_of_time(period)
                budget_secs = left
            node_cap = 0 if period == self.lb else PROBE_NODES
            n_sat, widx, rows, n_act, n_def, st = self.eng.probe(
                period, node_cap, self.small_budget, cap, limit, budget_secs, SAT_CHUNK)
            self.counters.add(st, self.eng.last_kernel_ms(), True, (n_r, r0, period, "probe"))
            root = self.eng.last_root_ms()
            self.counters.root_ms += root
            self.counters.probe_ms -= root
            if deadline and st["capped"] and time.monotonic() > deadline:
                return out_of_time(period)
            limit = self._scan_sats(res, n_r, r0, period, n_sat, widx, rows, limit, feasible)
            si, reruns = 0, 0
            while n_def and si < len(self.resolve_stages):
                dj_budget, stage_budget = self.resolve_stages[si]
                if self.speculate and 0 < SPEC_SMALL < stage_budget and n_def < SPEC_SMALL_NDEF:
                    stage_budget = SPEC_SMALL
                n_sat, widx, rows, n_act, n_def, st = self.eng.resolve(
                    period, node_cap, stage_budget, dj_budget, cap, limit, budget_secs,
                    SAT_CHUNK)
                self.counters.add(st, self.eng.last_kernel_ms(), False,
                                  (n_r, r0, period, f"resolve{stage_budget}"))
                if deadline and st["capped"] and time.monotonic() > deadline:
                    return out_of_time(period)
                limit = self._scan_sats(res, n_r, r0, period, n_sat, widx, rows, limit,
                                        feasible)
                si += 1
                if (si == len(self.resolve_stages) and n_def and not self.speculate
                        and stage_budget == 0):
                    # the full-cap stage leaves only probes a lower SAT cancelled;
                    # re-run those its completion check did not retire
                    reruns += 1
                    if reruns > 64:
                        raise RuntimeError("deferred probes did not settle")
                    si -= 1
            if self.speculate and n_def:
                spec, known_sat, back = [], [], []
                for w in self.eng.take_deferred(limit, n_def):
                    h = hints.get((int(w), period))
                    if h is None:
                        spec.append(int(w))
                        back.append(int(w))
                    elif h[0] == _native.SAT:
                        known_sat.append((int(w), h[1]))
                    else:
                        back.append(int(w))
                self.eng.add_active(back)
                n_act += len(back)
                if known_sat:
                    limit = self._scan_sats(res, n_r, r0, period, n_sat, widx, rows, limit,
                                            feasible, extra=known_sat)
                pending += [(w, period) for w in spec if w <= limit]
            active = n_act > 0
        return res, pending
