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
