"""Where the completion phase of a search spends its time: decide calls of
the lazy checks and the final completion, with SP-DFS counters.
usage: python scripts/phase_probe.py C2@8"""
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_15269_b200._core as core  # noqa: E402
from paper_2311_15269_b200 import _native  # noqa: E402
from paper_2311_15269_b200.completion import search  # noqa: E402
from paper_2311_15269_b200.engine import BatchedRepetendSearch  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402


def main(name):
    w = WORKLOADS[name]
    p = w.placement()
    eng = BatchedRepetendSearch(p)
    search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
    calls = []
    real = core.decide

    def rec(*a, **k):
        t0 = time.perf_counter()
        out = real(*a, **k)
        calls.append((a[0], k.get("node_budget", a[11] if len(a) > 11 else 0), out[0], out[2],
                      round(time.perf_counter() - t0, 4)))
        return out

    core.decide = rec
    s0 = _native.sp_stats()
    res = search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
    s1 = _native.sp_stats()
    print(json.dumps({"phase_secs": res.report.phase_secs,
                      "sp": {k: s1[k] - s0[k] for k in s1}}))
    for c in calls:
        print("decide n=%d budget=%d status=%d nodes=%d secs=%.4f" % c)


if __name__ == "__main__":
    main(sys.argv[1])
