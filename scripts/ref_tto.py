"""Time-to-optimal on the GPU box, both arms, per SURVEY §8(d) parity config:
the reference's own completion.search (oracle/_ref, compiled kernel,
TESSEL_BUDGET_SECS=1e9) with jobs=1 and jobs=nproc, and this package's
search on cuda:0 (warm engine, then a timed run; results checked against
the golden).  One JSON line per config.

Usage: python scripts/ref_tto.py C2@4 C3@9 ...   (default: all parity configs)
"""

import json
import os
import sys
import time
from pathlib import Path

os.environ["TESSEL_BUDGET_SECS"] = "1e9"
os.environ.setdefault("REPSCHED_KERNEL", "compiled")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

DEFAULT = ["C1", "C2@3", "C5@2", "C3@9", "C4b", "C3@12", "C4a@3", "C4a@4", "C2@4", "C5@3"]


def ref_time(p, w, jobs):
    import oracle

    oracle.load_reference()
    from repsched import completion as RC
    from repsched import placement as RP

    from paper_2311_15269_b200.placement import placement_to_dict

    rp = RP.placement_from_dict(placement_to_dict(p))
    t0 = time.perf_counter()
    res = RC.search(rp, w.mem_capacity, max_nr=w.max_nr, jobs=jobs)
    return time.perf_counter() - t0, res.report.best_t_r, res.schedule.makespan(), \
        len(res.report.candidates)


def gpu_time(p, w):
    from paper_2311_15269_b200.completion import search
    from paper_2311_15269_b200.engine import BatchedRepetendSearch

    t0 = time.perf_counter()
    res = search(p, w.mem_capacity, max_nr=w.max_nr)  # cold: fresh engine, first use
    cold = time.perf_counter() - t0
    eng = BatchedRepetendSearch(p)
    search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
    t0 = time.perf_counter()
    res = search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng)
    return cold, time.perf_counter() - t0, res


def main(names):
    from paper_2311_15269_b200.workloads import WORKLOADS

    nproc = os.cpu_count() or 1
    for name in names or DEFAULT:
        w = WORKLOADS[name]
        p = w.placement()
        g = json.loads((ROOT / "tests" / "golden" /
                        f"search_{name.replace('@', '_')}.json").read_text())
        cold, warm, res = gpu_time(p, w)
        ok = (res.report.best_t_r == g["best_t_r"]
              and res.schedule.makespan() == g["schedule"]["makespan"]
              and len(res.report.candidates) == g["n_candidates"])
        row = {"workload": name, "gpu_s": warm, "gpu_cold_s": cold, "parity": ok}
        for jobs in (1, nproc):
            wall, t_r, mk, n = ref_time(p, w, jobs)
            assert (t_r, mk, n) == (g["best_t_r"], g["schedule"]["makespan"], g["n_candidates"])
            row[f"ref_jobs{jobs}_s"] = wall
        best = min(row["ref_jobs1_s"], row[f"ref_jobs{nproc}_s"])
        row.update(ref_best_s=best, speedup_vs_best_cpu=best / warm,
                   speedup_cold=best / cold, nproc=nproc)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
