"""Golden fixtures for the TO baseline (to_search.search_time_optimal) from
the REFERENCE itself (oracle/_ref, built by oracle/build_ref.sh): status,
makespan, every schedule entry and the decide count, for small shapes the
reference solves in seconds.  Also records every decide call (inputs and
status / witness / node count) as probes_to_<name>.json.gz.

Usage: python tests/golden/make_to_goldens.py
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
os.environ["TESSEL_BUDGET_SECS"] = "1e9"
os.environ["REPSCHED_KERNEL"] = "compiled"

import oracle  # noqa: E402

R = oracle.load_reference()
assert R is not None, "build oracle/_ref first (oracle/build_ref.sh)"
from repsched import _core  # noqa: E402
from repsched import placement as RP  # noqa: E402
from repsched import to_search as RT  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"

# (name, shape, devices, costs, N, mem_capacity)
CASES = [
    ("to_v4_n2", "vshape", 4, (1, 1, 1, -1), 2, None),
    ("to_v4_n3_cap3", "vshape", 4, (1, 1, 1, -1), 3, 3),
    ("to_v4_n4", "vshape", 4, (1, 2, 1, -1), 4, None),
    ("to_x4_n2", "xshape", 4, (1, 2, 1, -1), 2, None),
    ("to_m4_n2", "mshape", 4, (1, 2, 1, -1), 2, None),
    ("to_k4_n2", "kshape", 4, (1, 2, 1, -1), 2, None),
    ("to_v4_n6_cap4", "vshape", 4, (1, 2, 1, -1), 6, 4),
    ("to_v4_n8", "vshape", 4, (1, 1, 1, -1), 8, None),
    ("to_x4_n4", "xshape", 4, (1, 2, 1, -1), 4, None),
    ("to_m4_n3_cap6", "mshape", 4, (1, 2, 1, -1), 3, 6),
    ("to_k4_n3", "kshape", 4, (1, 2, 1, -1), 3, None),
    ("to_nn4_n2", "nnshape", 4, (1, 2, 1, -1), 2, None),
]


def main(only=()):
    for name, shape, d, costs, n, cap in CASES:
        if only and name not in only:
            continue
        p = RP.make_shape(shape, d, RP.CostModel(*costs))
        calls = []
        real = _core.decide

        def rec(*a, **k):
            out = real(*a, **k)
            args = list(a) + [k.get("node_budget", a[11] if len(a) > 11 else 0)]
            n_, dur, mask, mem, edges, order, lo, hi, ndev, init, cap_ = a[:11]
            flat = list(edges) if not hasattr(edges, "tolist") else edges.tolist()
            if flat and isinstance(flat[0], (list, tuple)):
                flat = [x for e in flat for x in e]
            calls.append({"n": int(n_), "dur": list(map(int, dur)), "devmask": list(map(int, mask)),
                          "mem": list(map(int, mem)), "edges": list(map(int, flat)),
                          "order": list(map(int, order)), "lo": list(map(int, lo)),
                          "hi": list(map(int, hi)), "ndev": int(ndev),
                          "init": list(map(int, init)), "cap": int(cap_),
                          "budget": int(args[-1] or 0), "status": int(out[0]),
                          "starts": None if out[1] is None else list(map(int, out[1])),
                          "nodes": int(out[2]), "kind": "to"})
            return out

        import repsched.solver as RS
        RS._core.decide = rec
        t0 = time.monotonic()
        res = RT.search_time_optimal(p, n, mem_capacity=cap)
        wall = time.monotonic() - t0
        RS._core.decide = real
        doc = {"name": name, "placement": RP.placement_to_dict(p), "n_microbatches": n,
               "mem_capacity": cap, "status": res.status.name,
               "makespan": None if res.schedule is None else res.schedule.makespan(),
               "entries": None if res.schedule is None else sorted(
                   [b.stage, b.mb, t] for b, t in res.schedule.entries.items()),
               "decides": res.stats.decides, "ref_wall_secs": wall}
        (GOLDEN / f"search_{name}.json").write_text(json.dumps(doc))
        with gzip.open(GOLDEN / f"probes_{name}.json.gz", "wt") as f:
            json.dump({"seen": len(calls), "probes": calls}, f)
        print(name, res.status.name, doc["makespan"], len(calls), f"{wall:.2f}s")


if __name__ == "__main__":
    main(tuple(sys.argv[1:]))
