"""Fresh-engine searches as in bench.py's e2e leg, with per-step phase
times and the old engine's teardown timed separately, to localise the
occasional 0.5-1.5 s steps.  usage: python scripts/e2e_outlier.py C2@8 12"""
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15269_b200.completion import search  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
w = WORKLOADS[name]
p = w.placement()
res = search(p, w.mem_capacity, max_nr=w.max_nr, device=0)
buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(reps):
    buf.fill_(i & 255)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    new = search(p, w.mem_capacity, max_nr=w.max_nr, device=0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = new  # drops the previous result (and its engine)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"step": i, "search": round(t1 - t0, 4), "drop_old": round(t2 - t1, 4),
                      "phases": {k: round(v, 4) for k, v in new.report.phase_secs.items()},
                      "kernel_ms": round(new.report.engine.get("kernel_ms", 0), 1)}), flush=True)
