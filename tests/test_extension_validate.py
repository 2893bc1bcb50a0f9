"""structural extension (extension.extend, reference
extension.py:22-75) and schedule validation on the device
(validate.validate_schedule_device == the reference's validate_schedule,
schedule.py:77-168, violation for violation)."""

import random

import pytest

from conftest import load_search

NAMES = ["C1", "C2_3", "C4b", "C5_2", "C3_9", "x4_demo_k3", "m4_cap8", "k4_k3"]


def _searched(name):
    from paper_2311_15269_b200.placement import BlockInstance, placement_from_dict
    from paper_2311_15269_b200.schedule import RepetendInfo, Schedule

    doc = load_search(name)
    p = placement_from_dict(doc["placement"])
    sd = doc["schedule"]
    entries = {BlockInstance(a, n): t for a, n, t in sd["entries"]}
    return p, Schedule(p, sd["N"], entries, RepetendInfo(*sd["repetend"]))


@pytest.mark.parametrize("name", NAMES)
def test_extension_matches_reference_and_stays_valid(name):
    """Extension vs the reference's own extend (oracle/_ref) and the host
    validity check, for several N."""
    import oracle
    from paper_2311_15269_b200.extension import extend
    from paper_2311_15269_b200.placement import placement_to_dict
    from paper_2311_15269_b200.schedule import validate_schedule

    from paper_2311_15269_b200.repetend import steady_memory_ok

    ref = oracle.load_reference()
    p, s = _searched(name)
    for n in (s.num_microbatches, s.num_microbatches + 1, s.num_microbatches + 7, 64):
        e = extend(s, n)
        if steady_memory_ok(p):  # else memory grows with every copy (e.g. inference C4b)
            assert validate_schedule(e) == []
        if ref is not None:
            from repsched import extension as RE
            from repsched import placement as RP
            from repsched import schedule as RS

            rp = RP.placement_from_dict(placement_to_dict(p))
            rs = RS.Schedule(rp, s.num_microbatches,
                             {RP.BlockInstance(b.stage, b.mb): t for b, t in s.entries.items()},
                             RS.RepetendInfo(s.repetend.start, s.repetend.end, s.repetend.period,
                                             s.repetend.nr))
            re_ = RE.extend(rs, n)
            assert sorted((b.stage, b.mb, t) for b, t in e.entries.items()) == sorted(
                (b.stage, b.mb, t) for b, t in re_.entries.items())
            assert (e.repetend.start, e.repetend.end) == (re_.repetend.start, re_.repetend.end)


def _corrupt(s, rng, k):
    from paper_2311_15269_b200.schedule import Schedule

    entries = dict(s.entries)
    keys = list(entries)
    for _ in range(k):
        b = rng.choice(keys)
        entries[b] = entries[b] + rng.choice([-3, -2, -1, 1, 2, 3])
    return Schedule(s.placement, s.num_microbatches, entries, s.repetend)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_validation_matches_host(gpu, name):
    from paper_2311_15269_b200.extension import extend
    from paper_2311_15269_b200.schedule import validate_schedule
    from paper_2311_15269_b200.validate import validate_schedule_device

    rng = random.Random(7)
    p, s = _searched(name)
    for n in (s.num_microbatches, 200, 2000):
        e = extend(s, n)
        assert validate_schedule_device(e) == validate_schedule(e)
    e = extend(s, 300)
    for k in (1, 3, 20):  # overlaps, memory and dependency violations
        bad = _corrupt(e, rng, k)
        assert validate_schedule_device(bad) == validate_schedule(bad)
    init = [p.mem_capacity + 1] + [0] * (p.num_devices - 1)
    assert validate_schedule_device(e, init) == validate_schedule(e, init)


# ---- pinned against the reference's own validate_schedule / metrics / plan
# documents (tests/golden/make_more_goldens.py, schedule.py:77-296) ----------

def _ref_cases():
    import gzip
    import json

    from conftest import GOLDEN

    with gzip.open(GOLDEN / "validate_ref.json.gz", "rt") as f:
        return json.load(f)


def _case_schedule(row):
    from paper_2311_15269_b200.placement import BlockInstance, placement_from_dict
    from paper_2311_15269_b200.schedule import RepetendInfo, Schedule

    p = placement_from_dict(row["placement"])
    entries = {BlockInstance(a, m): t for a, m, t in row["entries"]}
    return Schedule(p, row["N"], entries, RepetendInfo(*row["repetend"]))


def _viol(vs):
    return [[v.kind, v.message, [[b.stage, b.mb] for b in v.instances]] for v in vs]


def test_host_validation_matches_reference_fixtures():
    from paper_2311_15269_b200.schedule import validate_schedule

    rows = _ref_cases()
    assert len(rows) >= 200 and any(r["violations"] for r in rows)
    kinds = set()
    for row in rows:
        got = _viol(validate_schedule(_case_schedule(row), row["initial_memory"]))
        assert got == row["violations"], (row["name"], row["N"], row["tag"])
        kinds |= {v[0] for v in row["violations"]}
    assert kinds == {"structure", "overlap", "memory", "dependency"}


def test_metrics_and_plan_documents_match_reference_fixtures():
    from fractions import Fraction

    from paper_2311_15269_b200.schedule import (canonicalize_microbatch_order, compute_metrics,
                                                plan_from_dict, plan_to_dict)

    for row in _ref_cases():
        if row["tag"] != "extended":
            continue
        s = _case_schedule(row)
        m = compute_metrics(s)
        exp = row["metrics"]
        assert (m.makespan, list(m.per_device_busy), list(m.peak_memory)) == (
            exp["makespan"], exp["per_device_busy"], exp["peak_memory"])
        assert m.bubble_rate_total == Fraction(*exp["bubble_rate_total"])
        assert m.bubble_rate_steady == (None if exp["bubble_rate_steady"] is None
                                        else Fraction(*exp["bubble_rate_steady"]))
        assert plan_to_dict(s) == row["plan"]
        back = plan_from_dict(row["plan"])
        assert back.entries == s.entries and back.repetend == s.repetend
        assert sorted([b.stage, b.mb, t] for b, t in
                      canonicalize_microbatch_order(s).entries.items()) == row["canonical"]


@pytest.mark.gpu
def test_device_validation_matches_reference_fixtures(gpu):
    from paper_2311_15269_b200.validate import validate_schedule_device

    for row in _ref_cases():
        got = _viol(validate_schedule_device(_case_schedule(row), row["initial_memory"]))
        assert got == row["violations"], (row["name"], row["N"], row["tag"])
