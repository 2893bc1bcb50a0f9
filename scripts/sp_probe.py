"""Time one long golden decide probe on the B200 (subtree-parallel decide)
and print the SP-DFS counters.  usage: python scripts/sp_probe.py <fixture> <index>"""
import gzip
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_15269_b200 import _native  # noqa: E402


def main(name, idx):
    d = json.loads(gzip.open(Path(__file__).resolve().parents[1] / "tests" / "golden" /
                             f"probes_{name}.json.gz").read())["probes"]
    ps = [p for p in d if p["nodes"] >= 1_000_000 or (len(sys.argv) > 3 and p["nodes"] > 20_000)]
    p = ps[int(idx)]
    args = (p["n"], p["dur"], p["devmask"], p["mem"], p["edges"], p["order"], p["lo"], p["hi"],
            p["ndev"], p["init"], p["cap"], p["budget"])
    _native.decide(*args)  # warm (allocations)
    s0 = _native.sp_stats()
    t0 = time.perf_counter()
    st, starts, nodes = _native.decide(*args)
    wall = time.perf_counter() - t0
    s1 = _native.sp_stats()
    ok = (st, nodes) == (p["status"], p["nodes"])
    print(json.dumps({"probe": f"{name}[{idx}]", "n": p["n"], "status": st, "nodes": nodes,
                      "exact": ok, "wall_s": round(wall, 3),
                      "sp": {k: round(s1[k] - s0[k], 2) for k in s1}}))


if __name__ == "__main__":
    main(*sys.argv[1:3])
