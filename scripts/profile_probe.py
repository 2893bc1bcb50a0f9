"""Run the heaviest recorded decide probe of a golden fixture through the
batched decide kernel (for ncu / timing).  Usage:
  python scripts/profile_probe.py <fixture> <kind> [node_budget] [copies]
e.g. python scripts/profile_probe.py C4a_3 capped 50000 1"""

import gzip
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2311_15269_b200 import _native  # noqa: E402


def main():
    name, kind = sys.argv[1], sys.argv[2]
    budget = int(sys.argv[3]) if len(sys.argv) > 3 else None
    copies = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    with gzip.open(ROOT / "tests" / "golden" / f"probes_{name}.json.gz", "rt") as f:
        probes = [p for p in json.load(f)["probes"] if p["kind"] == kind]
    p = max(probes, key=lambda q: (q["nodes"], q["n"]))
    prob = dict(n=p["n"], dur=p["dur"], devmask=p["devmask"], mem=p["mem"], edges=p["edges"],
                order=p["order"], lo=p["lo"], hi=p["hi"], ndev=p["ndev"], init_mem=p["init"],
                cap=p["cap"], node_budget=p["budget"] if budget is None else budget)
    _native.decide_batch([dict(prob, node_budget=10)])  # warm-up launch
    t0 = time.perf_counter()
    out = _native.decide_batch([prob] * copies)
    dt = time.perf_counter() - t0
    st, _, nodes = out[0]
    print(json.dumps({"fixture": name, "kind": kind, "n": p["n"], "ref_nodes": p["nodes"],
                      "ref_status": p["status"], "status": st, "nodes": nodes, "copies": copies,
                      "secs": dt, "us_per_node": 1e6 * dt / max(nodes, 1)}))


if __name__ == "__main__":
    main()
