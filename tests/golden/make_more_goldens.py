"""Round-2 reference fixtures (generated from the UNMODIFIED reference in
oracle/_ref; the reference cannot travel to the GPU box, so its outputs are
committed here):

* ``search_eager_<name>.json`` — ``completion.search(..., lazy=False)``
  (completion.py:359-368): every improvement completes the schedule eagerly;
* ``search_gate_<name>.json`` — placements whose entry-memory gate fires
  (repetend.py:264-266 "infeasible" outcomes within the inflight limit):
  three forward/backward pairs sharing devices, so a device's stage-order
  memory peak (cal_max_inflight, completion.py:132-149) stays below the
  entry memory of candidates with N_R at the limit;
* ``validate_ref.json.gz`` — ``schedule.validate_schedule`` violation lists
  (schedule.py:77-168) of extended and corrupted schedules, plus
  ``compute_metrics`` and ``plan_to_dict`` (schedule.py:171-296) documents.

Usage: python tests/golden/make_more_goldens.py
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
os.environ["TESSEL_BUDGET_SECS"] = "1e9"
os.environ["REPSCHED_KERNEL"] = "compiled"

import oracle  # noqa: E402

if oracle.load_reference() is None:
    sys.exit("oracle/_ref missing: run oracle/build_ref.sh first")
from repsched import extension as Rext  # noqa: E402
from repsched import placement as Rplace  # noqa: E402
from repsched import schedule as Rsched  # noqa: E402

import make_goldens as MG  # noqa: E402
from paper_2311_15269_b200 import placement as P  # noqa: E402
from paper_2311_15269_b200.placement import BlockSpec, PlacementSpec  # noqa: E402
from paper_2311_15269_b200.workloads import WORKLOADS  # noqa: E402

OUT = Path(__file__).resolve().parent


# Found by a seeded search over random "interleaved pairs" placements
# (two or three forward/backward pairs sharing devices plus "other" blocks)
# for ones where the reference records gate-"infeasible" candidates.
GATE_DOCS = {
    "pairs_a_cap4": {"devices": 3, "memory": 4, "blocks": [
        ["f0", "forward", [0, 1], 1, 1], ["b0", "backward", [0, 1], 3, -1],
        ["f1", "forward", [1, 2], 2, 1], ["b1", "backward", [1, 2], 1, -1],
        ["f2", "forward", [0, 2], 2, 1], ["b2", "backward", [0, 2], 3, -1],
        ["o0", "other", [2], 2, 0], ["o1", "other", [1], 3, 0]],
        "deps": [[0, 1], [2, 3], [4, 5], [4, 6], [4, 7]]},
    "pairs_b_cap3": {"devices": 3, "memory": 3, "blocks": [
        ["f0", "forward", [0, 2], 2, 1], ["b0", "backward", [0, 2], 2, -1],
        ["f1", "forward", [1, 2], 2, 1], ["b1", "backward", [1, 2], 2, -1],
        ["f2", "forward", [0, 1], 1, 1], ["b2", "backward", [0, 1], 1, -1],
        ["o0", "other", [0], 3, 0], ["o1", "other", [2], 1, 0]],
        "deps": [[0, 1], [2, 3], [4, 5], [4, 6], [6, 7]]},
    "pairs_c_cap5": {"devices": 3, "memory": 5, "blocks": [
        ["f0", "forward", [0, 1], 2, 1], ["b0", "backward", [0, 1], 1, -1],
        ["f1", "forward", [0, 2], 2, 1], ["b1", "backward", [0, 2], 1, -1],
        ["f2", "forward", [1, 2], 2, 1], ["b2", "backward", [1, 2], 1, -1],
        ["o0", "other", [1], 2, 0]],
        "deps": [[0, 1], [0, 6], [2, 3], [4, 5]]},
}


def gate_placements():
    """name -> (placement, mem_capacity, max_nr): the entry-memory gate fires
    for candidates within the inflight limit."""
    out = {}
    for name, d in GATE_DOCS.items():
        blocks = tuple(BlockSpec(i, lab, kind, frozenset(devs), t, m)
                       for i, (lab, kind, devs, t, m) in enumerate(d["blocks"]))
        p = PlacementSpec(d["devices"], d["memory"], blocks,
                          frozenset(tuple(e) for e in d["deps"]))
        out[name] = (p, d["memory"], None)
    return out


def run_eager():
    cases = {"C1": WORKLOADS["C1"], "C2_3": WORKLOADS["C2@3"], "C3_9": WORKLOADS["C3@9"]}
    for name, w in cases.items():
        MG.run_search(f"eager_{name}", w.placement(), w.mem_capacity, w.max_nr, lazy=False)
    for name in ("m4_cap8", "x4_demo_k3", "v4_demo_cap4"):
        mk, cap, k = MG.SMALL[name]
        MG.run_search(f"eager_{name}", mk(), cap, k, lazy=False)


def run_gate():
    for name, (p, cap, k) in gate_placements().items():
        MG.run_search(f"gate_{name}", p, cap, k)
        doc = json.loads((OUT / f"search_gate_{name}.json").read_text())
        assert doc["status_counts"].get("infeasible", 0) > 0, (name, doc["status_counts"])


def _ref_schedule(p, n, entries, rep):
    rp = Rplace.placement_from_dict(P.placement_to_dict(p))
    return Rsched.Schedule(rp, n, {Rplace.BlockInstance(a, m): t for (a, m), t in entries.items()},
                           None if rep is None else Rsched.RepetendInfo(*rep))


def run_validate():
    rng = random.Random(11)
    cases = []
    for name in ("C1", "C2_3", "C4b", "C5_2", "C3_9", "x4_demo_k3", "m4_cap8", "k4_k3"):
        doc = json.loads((OUT / f"search_{name}.json").read_text())
        p = P.placement_from_dict(doc["placement"])
        sd = doc["schedule"]
        rs = _ref_schedule(p, sd["N"], {(a, m): t for a, m, t in sd["entries"]}, sd["repetend"])
        for n in (sd["N"], 24, 96):
            ext = Rext.extend(rs, n)
            base = {(b.stage, b.mb): t for b, t in ext.entries.items()}
            rep = [ext.repetend.start, ext.repetend.end, ext.repetend.period, ext.repetend.nr]
            variants = [("extended", base, None)]
            for k in (1, 2, 4, 16):
                bad = dict(base)
                keys = sorted(bad)
                for _ in range(k):
                    key = rng.choice(keys)
                    bad[key] = bad[key] + rng.choice([-3, -2, -1, 1, 2, 3])
                variants.append((f"corrupt{k}", bad, None))
            # structure violations: a missing and an extra instance, a negative start
            miss = dict(base)
            miss.pop(sorted(miss)[0])
            variants.append(("missing", miss, None))
            extra = dict(base)
            extra[(0, n + 3)] = 0
            variants.append(("extra", extra, None))
            neg = dict(base)
            neg[sorted(neg)[1]] = -2
            variants.append(("negative", neg, None))
            init = [p.mem_capacity + 1] + [0] * (p.num_devices - 1)
            variants.append(("initmem", base, init))
            for tag, ent, im in variants:
                s = _ref_schedule(p, n, ent, rep)
                viol = Rsched.validate_schedule(s, im)
                row = {"name": name, "N": n, "tag": tag, "placement": doc["placement"],
                       "entries": sorted([a, m, t] for (a, m), t in ent.items()),
                       "repetend": rep, "initial_memory": im,
                       "violations": [[v.kind, v.message,
                                       [[b.stage, b.mb] for b in v.instances]] for v in viol]}
                if tag == "extended":
                    met = Rsched.compute_metrics(s)
                    row["metrics"] = {
                        "makespan": met.makespan, "per_device_busy": met.per_device_busy,
                        "peak_memory": met.peak_memory,
                        "bubble_rate_total": [met.bubble_rate_total.numerator,
                                              met.bubble_rate_total.denominator],
                        "bubble_rate_steady": None if met.bubble_rate_steady is None else
                        [met.bubble_rate_steady.numerator, met.bubble_rate_steady.denominator]}
                    row["plan"] = Rsched.plan_to_dict(s)
                    row["canonical"] = sorted(
                        [b.stage, b.mb, t]
                        for b, t in Rsched.canonicalize_microbatch_order(s).entries.items())
                cases.append(row)
    with gzip.open(OUT / "validate_ref.json.gz", "wt") as f:
        json.dump(cases, f)
    print(f"validate: {len(cases)} schedules", flush=True)


if __name__ == "__main__":
    todo = sys.argv[1:] or ["eager", "gate", "validate"]
    for t in todo:
        {"eager": run_eager, "gate": run_gate, "validate": run_validate}[t]()
