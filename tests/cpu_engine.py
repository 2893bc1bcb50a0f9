"""TEST-ONLY stand-in for the native engine (paper_2311_15269_b200._native.Engine)
built on the oracle, so the host-side search logic — level-synchronous scan,
deferral stages, retirement limits, ordered replay and the multi-rank
protocol — can be exercised on a machine without a GPU.  Same interface and
result contract as the sm_100a engine; the disjunctive filter is skipped (it
only changes how fast "not SAT" is reached, never the outcome)."""

from __future__ import annotations

import numpy as np

import oracle
from oracle import search_port as SP

STATS = ("probes", "root_refuted", "nodes", "capped", "sat", "deferred", "dj_refuted", "dj_nodes")


class OracleEngine:
    def __init__(self, p):
        self.p = p
        self.K = p.num_stages
        self.model = SP.ProbeModel(p)
        self._lists = {}
        self.cands, self.active, self.deferred, self.sats = [], [], [], []
        self.cancel = True  # emulate the device's speculative cancellations

    def _list(self, n_r):
        if n_r not in self._lists:
            self._lists[n_r] = list(SP.iter_assignments(self.p, n_r))
        return self._lists[n_r]

    def close(self):
        pass

    def last_root_ms(self):
        return 0.0

    def last_kernel_ms(self):
        return 0.0

    def count(self, n_r):
        return len(self._list(n_r))

    def unrank(self, n_r, rank):
        return tuple(self._list(n_r)[rank])

    def stage(self, n_r, r0, r1, cap, want_gate=False):
        self.cands = self._list(n_r)[r0:r1]
        gate = [cap is None or all(e <= cap for e in SP.entry_memory(self.p, a))
                for a in self.cands]
        self.active = [w for w, g in enumerate(gate) if g]
        self.deferred, self.sats = [], []
        return len(self.active), (np.array(gate, dtype=np.uint8) if want_gate else None)

    def _probe(self, w, period, cap, budget):
        a = self.cands[w]
        return self.model.probe(a, period, cap, SP.entry_memory(self.p, a), budget)

    def _rows(self, max_sat):
        self.sats.sort(key=lambda r: r[0])
        k = min(len(self.sats), max_sat)
        widx = np.array([w for w, _ in self.sats[:k]], dtype=np.int64)
        rows = np.array([s for _, s in self.sats[:k]], dtype=np.int32).reshape(k, self.K)
        return len(self.sats), widx, rows

    def probe(self, period, node_budget, small_budget, cap, widx_limit, budget_secs=0.0,
              max_sat=64):
        first = small_budget if (node_budget == 0 or small_budget < node_budget) else node_budget
        st = dict.fromkeys(STATS, 0)
        act, dfr, self.sats = [], [], []
        for w in self.active:
            if w > widx_limit:
                continue
            s, starts, nodes = self._probe(w, period, cap, first)
            st["probes"] += 1
            if s == oracle.SAT:
                self.sats.append((w, starts))
                st["sat"] += 1
            elif s == oracle.TIMEOUT and first != node_budget:
                dfr.append(w)
                st["deferred"] += 1
            else:
                act.append(w)
                st["capped"] += s == oracle.TIMEOUT
                st["root_refuted"] += s == oracle.UNSAT and nodes == 0
            st["nodes"] += nodes
        self.active, self.deferred = act, dfr
        n, widx, rows = self._rows(max_sat)
        return n, widx, rows, len(act), len(dfr), st

    def resolve(self, period, node_budget, stage_budget, dj_budget, cap, widx_limit,
                budget_secs=0.0, max_sat=64):
        partial = stage_budget > 0 and (node_budget == 0 or stage_budget < node_budget)
        budget = stage_budget if partial else node_budget
        st = dict.fromkeys(STATS, 0)
        if stage_budget < 0:  # filter-only stage; the stand-in has no filter
            self.deferred = [w for w in self.deferred if w <= widx_limit]
            st["deferred"] = len(self.deferred)
            n, widx, rows = self._rows(max_sat)
            return n, widx, rows, len(self.active), len(self.deferred), st
        redo = []
        todo = sorted(w for w in self.deferred if w <= widx_limit)
        # the device cancels probes above a SAT of the same launch (speculative
        # retirement); emulate the maximal cancellation: everything above the
        # lowest SAT goes back to the deferred list
        first_sat = None
        for w in todo:
            s, _, _ = self._probe(w, period, cap, budget)
            if s == oracle.SAT:
                first_sat = w
                break
        for w in todo:
            if self.cancel and first_sat is not None and w > first_sat:
                redo.append(w)
                st["deferred"] += 1
                continue
            s, starts, nodes = self._probe(w, period, cap, budget)
            if s == oracle.SAT:
                self.sats.append((w, starts))
                st["sat"] += 1
            elif s == oracle.TIMEOUT and partial:
                redo.append(w)
                st["deferred"] += 1
            else:
                self.active.append(w)
                st["capped"] += s == oracle.TIMEOUT
            st["nodes"] += nodes
        self.deferred = redo
        n, widx, rows = self._rows(max_sat)
        return n, widx, rows, len(self.active), len(redo), st

    def take_deferred(self, widx_limit, max_out):
        out = sorted(w for w in self.deferred if w <= widx_limit)
        self.deferred = []
        return np.array(out, dtype=np.int64)

    def add_active(self, widx):
        self.active.extend(int(w) for w in widx)

    def verify(self, widx, periods, budgets, cap):
        st, nodes, rows = [], [], []
        for w, per, b in zip(widx, periods, budgets):
            s, starts, nd = self._probe(int(w), int(per), cap, int(b))
            st.append(s)
            nodes.append(nd)
            rows.append(starts if starts is not None else [0] * self.K)
        if self.cancel:  # maximal cancellation by SATs (x, q): x < x2, q <= q2
            sats = [(int(w), int(q)) for w, q, s in zip(widx, periods, st) if s == oracle.SAT]
            for i, (w, q) in enumerate(zip(widx, periods)):
                if any(x < int(w) and p <= int(q) for x, p in sats):
                    st[i], nodes[i] = 3, 0
        return (np.array(st, dtype=np.int32), np.array(nodes, dtype=np.int64),
                np.array(rows, dtype=np.int32).reshape(len(st), self.K))

    def verify_stash(self, slot, widx):
        self._stash = getattr(self, "_stash", {})
        self._stash[slot] = [self.cands[int(w)] for w in widx]

    def verify_launch(self, slot, pos, widx, periods, budgets, cap):
        # computed now, read at verify_wait (the device runs it meanwhile);
        # the stashed assignments, not the staged window, are probed
        saved, cancel = self.cands, self.cancel
        rows = self._stash[slot]
        self.cands, self.cancel = [rows[int(p)] for p in pos], False
        try:
            out = self.verify(list(range(len(pos))), periods, budgets, cap)
        finally:
            self.cands, self.cancel = saved, cancel
        st = out[0]
        if self.cancel:  # cancellation compares window indices, not positions
            sats = [(int(w), int(q)) for w, q, s in zip(widx, periods, st) if s == oracle.SAT]
            st = st.copy()
            for i, (w, q) in enumerate(zip(widx, periods)):
                if any(x < int(w) and p <= int(q) for x, p in sats):
                    st[i] = 3
        self._vres = getattr(self, "_vres", {})
        self._vres[slot] = (st, out[1], out[2])

    def verify_wait(self, slot):
        return self._vres[slot]

    def sat_next(self, after):
        later = sorted((w, s) for w, s in self.sats if w > after)
        return (later[0][0], np.array(later[0][1], dtype=np.int32)) if later else None

    def sat_rows(self, first, count):
        self.sats.sort(key=lambda r: r[0])
        part = self.sats[first:first + count]
        widx = np.array([w for w, _ in part], dtype=np.int64)
        rows = np.array([s for _, s in part], dtype=np.int32).reshape(len(part), self.K)
        return widx, rows


def oracle_decide(n, dur, devmask, mem, edges, order, lo, hi, ndev, init_mem, cap,
                  node_budget=0, deadline=0.0):
    """Stand-in for paper_2311_15269_b200._core.decide in CPU tests."""
    return oracle.decide(n, dur, devmask, mem, edges, order, lo, hi, ndev, init_mem, cap,
                         node_budget, 0.0)


def oracle_decide_batch(problems, deadline=0.0):
    """Stand-in for paper_2311_15269_b200._core.decide_batch in CPU tests."""
    return [oracle.decide(p["n"], p["dur"], p["devmask"], p["mem"], p["edges"], p["order"],
                          p["lo"], p["hi"], p["ndev"], p["init_mem"], p["cap"],
                          p.get("node_budget", 0), 0.0) for p in problems]
