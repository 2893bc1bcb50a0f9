"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs the unmodified reference package (built into oracle/_ref by
oracle/build_ref.sh) in this container — it cannot travel to the GPU box, so
its outputs are committed as small JSON fixtures:

* ``search_<name>.json``  — completion.search results per workload (SURVEY
  §8(d)) and per small/random placement: best t_R, improvements, chosen
  repetend, full schedule entries, makespan, candidate status counts, the
  non-"bound" candidate records and diagnostics;
* ``probes_<name>.json.gz`` — recorded decide() calls (inputs and
  status/witness/node count), covering root refutations, DFS-resolved probes,
  node-capped TIMEOUT probes and completion probes.

Reference settings: REPSCHED_KERNEL=compiled, TESSEL_BUDGET_SECS=1e9 (no wall
timeouts, deterministic), jobs=1, lazy=True.

Usage: python tests/golden/make_goldens.py [name ...]   (default: all)
"""

from __future__ import annotations

import copy
import gzip
import json
import os
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
os.environ["TESSEL_BUDGET_SECS"] = "1e9"
os.environ["REPSCHED_KERNEL"] = "compiled"

import oracle  # noqa: E402

R = oracle.load_reference()
if R is None:
    sys.exit("oracle/_ref missing: run oracle/build_ref.sh first")
import repsched._core as RC  # noqa: E402
from repsched import completion as Rcomp  # noqa: E402
from repsched import placement as Rplace  # noqa: E402

from paper_2311_15269_b200 import placement as P  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent


def _ref_placement(p):
    return Rplace.placement_from_dict(P.placement_to_dict(p))


class Recorder:
    """Wraps repsched._core.decide; keeps a bounded, stratified sample."""

    def __init__(self, seed=0, keep_root=300, keep_dfs=600, keep_capped=40, keep_completion=200):
        self.rng = random.Random(seed)
        self.lim = {"root": keep_root, "dfs": keep_dfs, "capped": keep_capped, "completion": keep_completion}
        self.seen = {k: 0 for k in self.lim}
        self.kept = {k: [] for k in self.lim}
        self.orig = RC.decide

    def __call__(self, *args):
        a = copy.deepcopy(args)
        st, w, nodes = self.orig(*args)
        caller = sys._getframe(1).f_code.co_name
        if caller == "_run_decide":
            kind = "completion"
        elif st == RC.TIMEOUT:
            kind = "capped"
        elif nodes == 0:
            kind = "root"
        else:
            kind = "dfs"
        self.seen[kind] += 1
        # reservoir sampling per stratum
        rows = self.kept[kind]
        if len(rows) < self.lim[kind]:
            rows.append((a, (st, w, nodes)))
        else:
            j = self.rng.randrange(self.seen[kind])
            if j < self.lim[kind]:
                rows[j] = (a, (st, w, nodes))
        return st, w, nodes

    def dump(self, path):
        recs = []
        for kind, rows in self.kept.items():
            for a, (st, w, nodes) in rows:
                n, dur, mask, mem, edges, order, lo, hi, ndev, init, cap, budget, _deadline = a
                recs.append({
                    "kind": kind, "n": int(n),
                    "dur": [int(x) for x in dur], "devmask": [int(x) for x in mask],
                    "mem": [int(x) for x in mem],
                    "edges": [int(x) for x in __import__("numpy").asarray(edges).reshape(-1)],
                    "order": [int(x) for x in order], "lo": [int(x) for x in lo],
                    "hi": [int(x) for x in hi], "ndev": int(ndev), "init": [int(x) for x in init],
                    "cap": int(cap), "budget": int(budget),
                    "status": int(st), "starts": w, "nodes": int(nodes),
                })
        with gzip.open(path, "wt") as f:
            json.dump({"seen": self.seen, "probes": recs}, f)


def run_search(name, p, cap, max_nr, record=False, lazy=True):
    rp = _ref_placement(p)
    rec = Recorder() if record else None
    if rec:
        RC.decide = rec
    try:
        t0 = time.perf_counter()
        res = Rcomp.search(rp, cap, max_nr=max_nr, lazy=lazy)
        wall = time.perf_counter() - t0
    finally:
        RC.decide = rec.orig if rec else RC.decide
    rep = res.report
    counts = {}
    records = []
    for c in rep.candidates:
        counts[c.status] = counts.get(c.status, 0) + 1
        if c.status != "bound":
            records.append([c.n_r, list(c.assignment), c.t_r, c.status])
    s = res.schedule
    doc = {
        "name": name,
        "placement": P.placement_to_dict(p),
        "mem_capacity": cap,
        "max_nr": max_nr,
        "lazy": lazy,
        "lower_bound": rep.lower_bound,
        "limit": rep.max_nr,
        "inflights": rep.inflights,
        "best_t_r": rep.best_t_r,
        "improvements": [[list(a), t] for a, t in rep.improvements],
        "n_candidates": len(rep.candidates),
        "status_counts": counts,
        "records": records,
        "diagnostics": rep.diagnostics,
        "timed_out": rep.timed_out,
        "schedule": None if s is None else {
            "N": s.num_microbatches,
            "entries": sorted([b.stage, b.mb, t] for b, t in s.entries.items()),
            "repetend": [s.repetend.start, s.repetend.end, s.repetend.period, s.repetend.nr],
            "makespan": s.makespan(),
        },
        "ref_stats": {"decides": rep.stats.decides, "nodes": rep.stats.nodes},
        "ref_wall_secs": wall,
        "ref_cpu": os.uname().machine,
    }
    (OUT / f"search_{name}.json").write_text(json.dumps(doc) + "\n")
    if rec:
        rec.dump(OUT / f"probes_{name}.json.gz")
    print(f"{name}: t_R={rep.best_t_r} makespan={doc['schedule'] and doc['schedule']['makespan']} "
          f"cands={len(rep.candidates)} wall={wall:.1f}s", flush=True)


SMALL = {
    "v4_unit_cap4": (lambda: P.make_shape("vshape", 4, P.CostModel(1, 1, 1, -1), mem_capacity=4), 4, 4),
    "v4_demo_cap4": (lambda: P.make_shape("vshape", 4, P.CostModel(1, 2, 1, -1)), 4, None),
    "x4_demo_k3": (lambda: P.make_shape("xshape", 4, P.CostModel(1, 2, 1, -1)), None, 3),
    "m4_cap8": (lambda: P.make_shape("mshape", 4), 8, None),
    "k4_k3": (lambda: P.make_shape("kshape", 4), None, 3),
    "nn4_k3": (lambda: P.make_shape("nnshape", 4), None, 3),
    "v2_k4": (lambda: P.make_shape("vshape", 2), None, 4),
}


def random_suite(count=60, seed=2311):
    """Random placements from the reference's own generator
    (tests/oracles.py:143-167), searched with and without a memory cap."""
    import oracles  # reference tests/oracles.py

    rng = random.Random(seed)
    out = []
    for i in range(count):
        rp = oracles.random_placement(rng, max_k=6, max_d=3)
        p = P.placement_from_dict(Rplace.placement_to_dict(rp))
        capped = i % 2 == 0 and all(v <= 0 for v in p.net_mem_per_device())
        cap = p.mem_capacity if capped else None
        t0 = time.perf_counter()
        try:
            res = Rcomp.search(rp, cap, max_nr=3)
            s = res.schedule
            row = {
                "placement": P.placement_to_dict(p), "mem_capacity": cap, "max_nr": 3,
                "best_t_r": res.report.best_t_r,
                "improvements": [[list(a), t] for a, t in res.report.improvements],
                "n_candidates": len(res.report.candidates),
                "diagnostics": res.report.diagnostics,
                "schedule": None if s is None else {
                    "entries": sorted([b.stage, b.mb, t] for b, t in s.entries.items()),
                    "repetend": [s.repetend.start, s.repetend.end, s.repetend.period, s.repetend.nr],
                    "makespan": s.makespan()},
                "error": None,
            }
        except Exception as exc:  # NoFeasibleSchedule etc. are part of the contract
            row = {"placement": P.placement_to_dict(p), "mem_capacity": cap, "max_nr": 3,
                   "error": type(exc).__name__}
        row["wall"] = time.perf_counter() - t0
        out.append(row)
    (OUT / "search_random.json").write_text(json.dumps(out) + "\n")
    print(f"random: {len(out)} placements", flush=True)


def main(names):
    todo = names or (list(SMALL) + ["random"] + list(WORKLOADS))
    for name in todo:
        if name == "random":
            random_suite()
        elif name in SMALL:
            mk, cap, k = SMALL[name]
            run_search(name, mk(), cap, k, record=True)
        elif name in WORKLOADS:
            w = WORKLOADS[name]
            if name in ("C2@5", "C5@4"):
                continue  # the CPU reference does not finish these
            run_search(name.replace("@", "_"), w.placement(), w.mem_capacity, w.max_nr,
                       record=os.environ.get("GOLDEN_NO_RECORD") != "1")
        else:
            raise SystemExit(f"unknown golden {name}")


if __name__ == "__main__":
    main(sys.argv[1:])
