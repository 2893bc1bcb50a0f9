"""DJ filter propagation statistics of one search (library built with
-DWDJ_COUNT_ROUNDS): propagate calls, rounds, row / pair chunks relaxed.
usage: python scripts/dj_rounds.py C2@8"""
import ctypes
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_15269_b200 import _native  # noqa: E402
from paper_2311_15269_b200.completion import search  # noqa: E402
from paper_2311_15269_b200.engine import BatchedRepetendSearch  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402

w = WORKLOADS[sys.argv[1]]
p = w.placement()
eng = BatchedRepetendSearch(p)
res = search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
out = (ctypes.c_ulonglong * 4)()
_native.lib().tsl_debug_wdj_rounds(out)
c = vars(eng.counters)
print(json.dumps({"workload": sys.argv[1], "rounds": out[0], "calls": out[1], "row_chunks": out[2],
                  "pair_chunks": out[3], "dj_nodes": c.get("dj_nodes")}))
