"""Fixture for validating the disjunctive refutation filter (csrc/dj_solve.cuh).

Collects the repetend probes that the reference search node-caps (400k nodes
-> TIMEOUT) on several workloads, plus a sample of DFS-resolved probes, and
records their TRUE feasibility by running the oracle decide (C restatement of
the reference kernel, pinned against it in tests/test_oracle.py) without the
cap but with a large node budget.  truth: 1 SAT, 0 UNSAT, -1 unresolved.

Usage: python tests/golden/make_dj_fixture.py   (~10-20 min on 8 cores)
"""

from __future__ import annotations

import json
import sys
from multiprocessing import Pool
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import search_port as SP  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402

TRUTH_BUDGET = 40_000_000
CASES = ["C2@3", "C3@9", "C5@2", "C4a@3"]


def collect(wl):
    w = WORKLOADS[wl]
    p = w.placement()
    model = SP.ProbeModel(p)
    orig = model.probe
    rows = []

    def rec(a, P, cap, entry, node_budget=0):
        st, s, nodes = orig(a, P, cap, entry, node_budget)
        if st == SP.TIMEOUT or (nodes > 50 and len(rows) < 400):
            rows.append({"workload": wl, "a": list(a), "P": P, "cap": cap,
                         "ref_status": st, "ref_nodes": nodes})
        return st, s, nodes

    model.probe = rec
    optimal = sum(b.time_cost for b in p.blocks) + 1
    for n_r in range(1, (w.max_nr or 3) + 1):
        for a in SP.iter_assignments(p, n_r):
            out = SP.solve_repetend(p, a, w.mem_capacity, upper=optimal, model=model)
            if out.period is not None and out.period < optimal and SP.completion_feasible(p, out, w.mem_capacity):
                optimal = out.period
    return rows


def truth(row):
    p = WORKLOADS[row["workload"]].placement()
    model = SP.ProbeModel(p)
    st, s, nodes = model.probe(row["a"], row["P"], row["cap"], SP.entry_memory(p, row["a"]),
                               TRUTH_BUDGET)
    row["truth"] = {SP.SAT: 1, SP.UNSAT: 0}.get(st, -1)
    row["truth_nodes"] = nodes
    return row


def main():
    rows = []
    for wl in CASES:
        got = collect(wl)
        print(wl, len(got), "probes", flush=True)
        rows += got
    with Pool(8) as pool:
        rows = pool.map(truth, rows, chunksize=1)
    out = Path(__file__).resolve().parent / "dj_probes.json"
    out.write_text(json.dumps(rows) + "\n")
    from collections import Counter
    print(Counter((r["workload"], r["ref_status"], r["truth"]) for r in rows))


if __name__ == "__main__":
    main()
