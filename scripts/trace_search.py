"""Run one search with per-launch tracing (TESSEL_TRACE=1) and summarise
where the GPU time goes.  Usage: python scripts/trace_search.py C2@4"""

import json
import os
import sys
import time
from collections import defaultdict
from pathlib import Path

os.environ["TESSEL_TRACE"] = "1"
os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2311_15269_b200.completion import search  # noqa: E402
from paper_2311_15269_b200.engine import BatchedRepetendSearch  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402


def main(name):
    w = WORKLOADS[name]
    p = w.placement()
    eng = BatchedRepetendSearch(p)
    search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)  # warm
    eng.counters.trace.clear()
    t0 = time.perf_counter()
    res = search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
    wall = time.perf_counter() - t0
    tr = eng.counters.trace
    by_kind = defaultdict(lambda: [0, 0.0])
    for n_r, r0, period, kind, ms, st in tr:
        by_kind[kind][0] += 1
        by_kind[kind][1] += ms
    kern = sum(ms for *_, ms, _ in tr)
    print(json.dumps({"workload": name, "wall_s": wall, "kernel_s": kern / 1e3,
                      "phase_secs": res.report.phase_secs, "best_t_r": res.report.best_t_r,
                      "candidates": len(res.report.candidates),
                      "by_kind": {k: {"launches": v[0], "ms": round(v[1], 2)}
                                  for k, v in by_kind.items()}}))
    for row in sorted(tr, key=lambda r: -r[4])[:15]:
        print("top", row)
    out = os.environ.get("TRACE_OUT")
    if out:
        Path(out).parent.mkdir(parents=True, exist_ok=True)
        Path(out).write_text(json.dumps({"workload": name, "wall_s": wall,
                                         "counters": {k: v for k, v in vars(eng.counters).items()
                                                      if k != "trace"},
                                         "trace": tr}))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2@4")
