"""Capped (400k-node) repetend probes of a golden fixture through the
subtree-parallel decide (TSL_SP_MIN_BUDGET lowered) vs one warp each:
exactness, wall time, SP counters.  usage: sp_capped.py <fixture> [max]"""
import gzip
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_15269_b200 import _native  # noqa: E402


def main(name, mx=6):
    d = json.loads(gzip.open(Path(__file__).resolve().parents[1] / "tests" / "golden" /
                             f"probes_{name}.json.gz").read())["probes"]
    ps = [p for p in d if p["kind"] == "capped" and p["nodes"] > 100_000][:int(mx)]
    for i, p in enumerate(ps):
        args = (p["n"], p["dur"], p["devmask"], p["mem"], p["edges"], p["order"], p["lo"], p["hi"],
                p["ndev"], p["init"], p["cap"], p["budget"])
        row = {"probe": f"{name}[{i}]", "n": p["n"], "status": p["status"], "nodes": p["nodes"]}
        for mode in ("warp", "sp", "sp_any"):
            os.environ.pop("TSL_SP_DONATE_ANY_S", None)
            if mode.startswith("sp"):
                os.environ["TSL_SP_MIN_BUDGET"] = "1"
            else:
                os.environ.pop("TSL_SP_MIN_BUDGET", None)
            if mode == "sp_any":
                os.environ["TSL_SP_DONATE_ANY_S"] = "1"
            _native.decide(*args)
            s0 = _native.sp_stats()
            t0 = time.perf_counter()
            st, starts, nodes = _native.decide(*args)
            wall = time.perf_counter() - t0
            s1 = _native.sp_stats()
            row[mode] = {"exact": (st, nodes) == (p["status"], p["nodes"]) and
                         (st != 1 or list(starts) == p["starts"]), "wall_s": round(wall, 4),
                         "undivided": s1["undivided"] - s0["undivided"],
                         "pieces": s1["pieces"] - s0["pieces"], "explored": s1["explored"] - s0["explored"], "epochs": s1["epochs"] - s0["epochs"]}
        print(json.dumps(row))


if __name__ == "__main__":
    main(*sys.argv[1:])
