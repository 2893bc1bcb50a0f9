"""Reference goldens for searches too long for one core (BASELINE configs[4]).

Drives the UNMODIFIED reference package (oracle/_ref) with the reference's
own functions, reproducing ``repsched.completion.search(..., jobs=1,
lazy=True)`` exactly while spreading candidate evaluations over a process
pool:

* every candidate is evaluated by the reference's ``solve_repetend`` with the
  reference's own ``upper`` rule (``completion.py:331-337``: upper = the
  optimum after every earlier candidate);
* candidates are evaluated speculatively in chunks with the optimum known at
  chunk start; when an improvement lowers the optimum inside a chunk, every
  later candidate of that chunk is re-evaluated with the correct upper (a
  ``solve_repetend`` call with no budget is a pure function of (assignment,
  cap, upper)), so every
  outcome, status record and stats merge is the one the sequential loop
  produces;
* lazy checks (``_completion_feasible``) and the final ``complete_schedule``
  run in the driver process, in candidate order, exactly as
  ``completion.py:351-396``.

Pinned by re-generating a golden the plain sequential reference produced
(``--check C5@3`` compares everything in ``search_C5_3.json``, the reference
stats included).

Usage: python tests/golden/make_par_golden.py C5@4 [--jobs 8]
       python tests/golden/make_par_golden.py --check C5@3
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
os.environ["TESSEL_BUDGET_SECS"] = "1e9"
os.environ["REPSCHED_KERNEL"] = "compiled"

import oracle  # noqa: E402

R = oracle.load_reference()
if R is None:
    sys.exit("oracle/_ref missing: run oracle/build_ref.sh first")
from repsched import completion as Rcomp  # noqa: E402
from repsched import placement as Rplace  # noqa: E402
from repsched import repetend as Rrep  # noqa: E402
from repsched.solver import SolveStats  # noqa: E402

from paper_2311_15269_b200 import placement as P  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402

OUT = Path(__file__).resolve().parent
_P = None


def _init(pd):
    global _P
    _P = Rplace.placement_from_dict(pd)


def _eval(args):
    asg, cap, upper = args
    st = SolveStats()
    out = Rrep.solve_repetend(_P, asg, cap, upper=upper, budget=1e9, stats=st)
    return out, st


def par_search(p_dict, cap, max_nr, jobs, chunk=512, log=None):
    p = Rplace.placement_from_dict(p_dict)
    lb = Rrep.lower_bound(p)
    total = sum(b.time_cost for b in p.blocks)
    inflights = Rcomp.cal_max_inflight(p, cap)
    limit = max_nr if max_nr is not None else Rcomp.DEFAULT_MAX_NR
    if inflights is not None:
        limit = min(limit, inflights)
    report = Rcomp.SearchReport(lower_bound=lb, max_nr=limit,
                                inflights=inflights if inflights is not None else -1, lazy=True)
    deadline = time.monotonic() + 1e9
    best = None
    optimal = total + 1
    done = False
    reruns = 0
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=jobs, initializer=_init, initargs=(p_dict,)) as pool:
        for n_r in range(1, max(limit, 1) + 1):
            if done:
                break
            gen = Rrep.iter_repetend_assignments(p, n_r)
            while not done:
                batch = []
                for asg in gen:
                    batch.append(asg)
                    if len(batch) >= chunk:
                        break
                if not batch:
                    break
                spec_upper = optimal
                outs = list(pool.map(_eval, [(a, cap, spec_upper) for a in batch], chunksize=4))
                i = 0
                while i < len(batch):
                    asg = batch[i]
                    out, st = outs[i]
                    if optimal != spec_upper:
                        # evaluated with a stale (larger) upper: re-run the
                        # rest of the chunk with the sequential upper
                        rest = [(x, cap, optimal) for x in batch[i:]]
                        outs[i:] = list(pool.map(_eval, rest, chunksize=4))
                        spec_upper = optimal
                        reruns += len(rest)
                        continue
                    report.stats.merge(st)
                    rec_status = out.status
                    t_r = out.repetend.period if out.repetend else None
                    if out.status == "timeout":
                        report.timed_out = True
                    if out.repetend is not None and out.repetend.period < optimal:
                        ok = Rcomp._completion_feasible(p, out.repetend, cap, deadline, report)
                        if not ok:
                            rec_status = "completion-infeasible"
                        if ok:
                            best = out.repetend
                            optimal = out.repetend.period
                            report.improvements.append((asg, optimal))
                            rec_status = "improved"
                            if optimal == lb:
                                done = True
                    report.candidates.append(Rcomp.CandidateRecord(n_r, tuple(asg), t_r, rec_status))
                    i += 1
                    if done:
                        break
                if log:
                    log(f"n_r={n_r} cands={len(report.candidates)} optimal={optimal} "
                        f"reruns={reruns} {time.perf_counter() - t0:.0f}s")
    report.best_t_r = best.period if best else None
    if best is None:
        raise Rcomp.NoFeasibleSchedule("no repetend candidate is schedulable under memory")
    sched = Rcomp.complete_schedule(p, best, cap, deadline, report)
    return Rcomp.SearchResult(sched, report), time.perf_counter() - t0


def to_doc(name, p, cap, max_nr, res, wall, jobs):
    rep = res.report
    counts, records = {}, []
    for c in rep.candidates:
        counts[c.status] = counts.get(c.status, 0) + 1
        if c.status != "bound":
            records.append([c.n_r, list(c.assignment), c.t_r, c.status])
    s = res.schedule
    return {
        "name": name, "placement": P.placement_to_dict(p), "mem_capacity": cap, "max_nr": max_nr,
        "lower_bound": rep.lower_bound, "limit": rep.max_nr, "inflights": rep.inflights,
        "best_t_r": rep.best_t_r,
        "improvements": [[list(a), t] for a, t in rep.improvements],
        "n_candidates": len(rep.candidates), "status_counts": counts, "records": records,
        "diagnostics": rep.diagnostics, "timed_out": rep.timed_out,
        "schedule": None if s is None else {
            "N": s.num_microbatches,
            "entries": sorted([b.stage, b.mb, t] for b, t in s.entries.items()),
            "repetend": [s.repetend.start, s.repetend.end, s.repetend.period, s.repetend.nr],
            "makespan": s.makespan(),
        },
        "ref_stats": {"decides": rep.stats.decides, "nodes": rep.stats.nodes},
        "ref_wall_secs": wall,
        "ref_driver": f"tests/golden/make_par_golden.py jobs={jobs} (sequential-equivalent)",
        "ref_cpu": os.uname().machine,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    w = WORKLOADS[a.name]
    p = w.placement()
    res, wall = par_search(P.placement_to_dict(p), w.mem_capacity, w.max_nr, a.jobs,
                           log=lambda m: print(m, flush=True))
    doc = to_doc(a.name.replace("@", "_"), p, w.mem_capacity, w.max_nr, res, wall, a.jobs)
    fn = OUT / f"search_{a.name.replace('@', '_')}.json"
    if a.check:
        ref = json.loads(fn.read_text())
        keys = ["best_t_r", "improvements", "n_candidates", "status_counts", "records",
                "diagnostics", "schedule", "ref_stats", "limit", "inflights", "lower_bound"]
        bad = [k for k in keys if ref[k] != doc[k]]
        print("check", a.name, "OK" if not bad else f"MISMATCH {bad}", f"wall={wall:.1f}s")
        sys.exit(1 if bad else 0)
    fn.write_text(json.dumps(doc) + "\n")
    print(f"{a.name}: t_R={doc['best_t_r']} makespan={doc['schedule']['makespan']} "
          f"cands={doc['n_candidates']} wall={wall:.1f}s")


if __name__ == "__main__":
    main()
