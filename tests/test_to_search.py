"""TO baseline (to_search.search_time_optimal) against
the reference's own results (tests/golden/make_to_goldens.py): status,
makespan, every schedule entry and the number of decide probes — including
cases whose 8M-node probes TIMEOUT (best-so-far schedule or none)."""

import json

import pytest

from conftest import GOLDEN

NAMES = sorted(p.stem[len("search_"):] for p in GOLDEN.glob("search_to_*.json"))
FAST = [n for n in NAMES if json.loads((GOLDEN / f"search_{n}.json").read_text())["status"]
        == "OPTIMAL"]


def _run(name):
    from paper_2311_15269_b200.placement import placement_from_dict
    from paper_2311_15269_b200.to_search import search_time_optimal

    doc = json.loads((GOLDEN / f"search_{name}.json").read_text())
    p = placement_from_dict(doc["placement"])
    res = search_time_optimal(p, doc["n_microbatches"], mem_capacity=doc["mem_capacity"])
    got = {"status": res.status.name,
           "makespan": None if res.schedule is None else res.schedule.makespan(),
           "entries": None if res.schedule is None else sorted(
               [b.stage, b.mb, t] for b, t in res.schedule.entries.items()),
           "decides": res.stats.decides}
    exp = {k: doc[k] for k in ("status", "makespan", "entries", "decides")}
    return got, exp


@pytest.mark.parametrize("name", FAST)
def test_to_search_matches_reference_on_cpu_oracle(monkeypatch, name):
    """Host logic (lowering, binary search, assembly) with the oracle decide."""
    from cpu_engine import oracle_decide

    import paper_2311_15269_b200._core as core

    monkeypatch.setattr(core, "decide", oracle_decide)
    got, exp = _run(name)
    assert got == exp


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_to_search_matches_reference_on_gpu(gpu, name):
    """Every probe on the B200 (8M-node probes subtree-parallel)."""
    got, exp = _run(name)
    assert got == exp
