"""cProfile of one warm C2@8 search (host-side orchestration costs)."""
import cProfile
import os
import pstats
import sys
from pathlib import Path

os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_15269_b200.completion import search  # noqa: E402
from paper_2311_15269_b200.engine import BatchedRepetendSearch  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2@8"]
p = w.placement()
eng = BatchedRepetendSearch(p)
search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
pr = cProfile.Profile()
pr.enable()
search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
