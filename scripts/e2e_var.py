"""Run-to-run variation of fresh-engine vs resident-engine searches: wall,
phases, SP counters per search.  usage: python scripts/e2e_var.py C2@8 6"""
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15269_b200 import _native  # noqa: E402
from paper_2311_15269_b200.completion import search  # noqa: E402
from paper_2311_15269_b200.engine import BatchedRepetendSearch  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
w = WORKLOADS[name]
p = w.placement()
eng = BatchedRepetendSearch(p)
search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
for mode in ("resident", "fresh") * reps:
    s0 = _native.sp_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "resident":
        res = search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
    else:
        res = search(p, w.mem_capacity, max_nr=w.max_nr, device=0)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    s1 = _native.sp_stats()
    print(json.dumps({"mode": mode, "wall": round(wall, 4),
                      "phases": {k: round(v, 4) for k, v in res.report.phase_secs.items()},
                      "sp": {k: round(s1[k] - s0[k], 1) for k in ("task_ms", "master_ms", "pieces", "explored", "solves", "rounds")},
                      "kernel_ms": round(res.report.engine.get("kernel_ms", 0), 1)}))
