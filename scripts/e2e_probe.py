"""Where a fresh-engine search (bench.py's e2e leg) spends its time beyond
the resident-engine search: engine construction, the search itself, engine
teardown.  usage: python scripts/e2e_probe.py [workload] [reps]"""
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15269_b200.completion import search  # noqa: E402
from paper_2311_15269_b200.engine import BatchedRepetendSearch  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402


def main(name="C2@8", reps=3):
    w = WORKLOADS[name]
    p = w.placement()
    eng = BatchedRepetendSearch(p)
    search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
    rows = []
    for _ in range(int(reps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        e2 = BatchedRepetendSearch(p)
        t2 = time.perf_counter()
        search(p, w.mem_capacity, max_nr=w.max_nr, engine=e2)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        e2.eng.close()
        del e2
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        search(p, w.mem_capacity, max_nr=w.max_nr, device=0)
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        rows.append({"resident": t1 - t0, "create": t2 - t1, "fresh_search": t3 - t2,
                     "close": t4 - t3, "public_api": t5 - t4})
    print(json.dumps({"workload": name, "rows": rows}))


if __name__ == "__main__":
    main(*sys.argv[1:])
