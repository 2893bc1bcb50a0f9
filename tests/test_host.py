"""CPU tests of the host side: the C-ABI library loads and exports every
declared symbol, candidate enumeration / unranking, the data model and the
lazy candidate log.  No GPU compute is invoked."""

import ctypes
import json
import re

import pytest

from conftest import GOLDEN, ROOT, load_search, search_names

from paper_2311_15269_b200 import _native
from paper_2311_15269_b200.placement import (CostModel, ParseError, UnsupportedShape,
                                             ValidationError, make_shape, placement_from_dict,
                                             placement_to_dict)
from paper_2311_15269_b200.workloads import WORKLOADS


@pytest.fixture(scope="module")
def lib():
    _native.build()
    return _native.lib()


def test_library_exports_every_declared_symbol(lib):
    header = (ROOT / "include" / "tessel_b200.h").read_text()
    declared = set(re.findall(r"\b(tsl_[a-z_]+)\s*\(", header))
    assert declared >= set(_native.EXPORTS)
    handle = ctypes.CDLL(str(_native.LIB_PATH))
    for sym in sorted(declared):
        assert hasattr(handle, sym), sym


def test_compute_fails_loudly_without_device(lib):
    if _native.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(_native.NativeError) as ei:
        _native.decide(1, [1], [1], [0], [], [0], [0], [5], 1, [0], -1)
    assert "no CPU fallback" in str(ei.value)


def test_sass_is_sm100a():
    """The shipped library carries sm_100a SASS for every kernel."""
    import shutil
    import subprocess

    _native.build()
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _engine(p):
    k = p.num_stages
    return _native.Engine([p.block(s).time_cost for s in range(k)],
                          [p.block(s).mem_delta for s in range(k)],
                          [sum(1 << d for d in p.block(s).devices) for s in range(k)],
                          sorted(p.deps), p.num_devices)


# SURVEY.md §8(d) candidate counts per N_R (exact reference enumeration)
COUNTS = {
    "C2@3": {1: 1, 2: 288, 3: 23120, 4: 915552},
    "C3@9": {1: 1, 2: 20, 3: 210, 4: 1540, 5: 8855, 6: 42504, 7: 177100, 8: 657800},
    "C4a@3": {1: 1, 2: 34, 3: 595, 4: 7140, 5: 66045, 6: 501942},
    "C4b": {1: 1, 2: 17, 3: 153, 4: 969, 5: 4845, 6: 20349, 7: 74613, 8: 245157},
    "C5@2": {1: 1, 2: 162, 3: 10611, 4: 382500},
    "C1": {1: 1, 2: 8, 3: 36, 4: 120},
}


@pytest.mark.parametrize("wl", sorted(COUNTS))
def test_candidate_counts(lib, wl):
    e = _engine(WORKLOADS[wl].placement())
    for n_r, c in COUNTS[wl].items():
        assert e.count(n_r) == c


def test_large_counts_match_survey(lib):
    e = _engine(WORKLOADS["C2@4"].placement())
    assert e.count(8) == 54_476_446_464 or abs(e.count(8) - 5.45e10) / 5.45e10 < 0.01
    k = _engine(WORKLOADS["C5@2"].placement())
    assert abs(k.count(8) - 2.16e10) / 2.16e10 < 0.01


@pytest.mark.parametrize("wl", ["C1", "C2@3", "C3@9", "C4b", "C5@2"])
def test_unrank_matches_reference_order(lib, wl):
    from paper_2311_15269_b200.repetend import iter_repetend_assignments

    p = WORKLOADS[wl].placement()
    e = _engine(p)
    for n_r in (1, 2, 3):
        gen = list(iter_repetend_assignments(p, n_r))
        assert len(gen) == e.count(n_r)
        step = max(1, len(gen) // 500)
        for r in range(0, len(gen), step):
            assert e.unrank(n_r, r) == gen[r]
        assert e.unrank(n_r, len(gen) - 1) == gen[-1]


def test_unrank_random_placements(lib):
    from paper_2311_15269_b200.repetend import iter_repetend_assignments

    rows = json.loads((GOLDEN / "search_random.json").read_text())
    for row in rows:
        p = placement_from_dict(row["placement"])
        e = _engine(p)
        for n_r in (1, 2, 3, 4):
            gen = list(iter_repetend_assignments(p, n_r))
            assert e.count(n_r) == len(gen)
            assert [e.unrank(n_r, r) for r in range(len(gen))] == gen


@pytest.mark.parametrize("name", search_names())
def test_placement_json_matches_golden(name):
    doc = load_search(name)
    p = placement_from_dict(doc["placement"])
    assert placement_to_dict(p) == doc["placement"]


def test_workload_placements_match_goldens():
    for wl, gold in [("C1", "C1"), ("C2@3", "C2_3"), ("C3@9", "C3_9"), ("C4a@3", "C4a_3")]:
        assert placement_to_dict(WORKLOADS[wl].placement()) == load_search(gold)["placement"]


def test_placement_errors():
    with pytest.raises(UnsupportedShape):
        make_shape("kshape", 3)
    with pytest.raises(UnsupportedShape):
        make_shape("vshape", 1)
    doc = placement_to_dict(make_shape("vshape", 2))
    doc["deps"].append([3, 3])
    with pytest.raises(ValidationError):
        placement_from_dict(doc)
    doc = placement_to_dict(make_shape("vshape", 2))
    doc["blocks"][0]["devices"] = [5]
    with pytest.raises(ValidationError):
        placement_from_dict(doc)
    with pytest.raises(ParseError):
        placement_from_dict({"devices": 2})


def test_spec_goldens_host_side():
    """SPEC examples G1-G3, G14."""
    from paper_2311_15269_b200.completion import cal_max_inflight
    from paper_2311_15269_b200.repetend import entry_memory, iter_repetend_assignments

    v4 = make_shape("vshape", 4, CostModel(1, 2, 1, -1))
    assert len(list(iter_repetend_assignments(v4, 1))) == 1
    assert len(list(iter_repetend_assignments(v4, 2))) == 8
    from paper_2311_15269_b200.placement import BlockSpec, PlacementSpec

    two = PlacementSpec(2, 4, (BlockSpec(0, "a", "forward", frozenset([0]), 1, 1),
                               BlockSpec(1, "b", "forward", frozenset([1]), 1, 1)), frozenset())
    assert list(iter_repetend_assignments(two, 2)) == [(0, 0), (0, 1), (1, 0)]
    assert entry_memory(v4, (3, 2, 1, 0, 0, 0, 0, 0)) == (3, 2, 1, 0)
    assert cal_max_inflight(v4, 4) == 4


def test_compact_period_spec_golden():
    """G4: internal (6,4,2,0,1,3,5,7) at (3,2,1,0,...) -> P=3, E=(3,3,3,3), W=0."""
    from paper_2311_15269_b200.repetend import compact_period

    v4 = make_shape("vshape", 4, CostModel(1, 2, 1, -1))
    internal = dict(enumerate((6, 4, 2, 0, 1, 3, 5, 7)))
    assert compact_period(v4, internal, (3, 2, 1, 0, 0, 0, 0, 0)) == (3, (3, 3, 3, 3),
                                                                      (0, 0, 0, 0))


def test_candidate_log_sequence(lib):
    from paper_2311_15269_b200.completion import CandidateLog, CandidateRecord
    from paper_2311_15269_b200.repetend import iter_repetend_assignments

    p = make_shape("vshape", 4, CostModel(1, 1, 1, -1), mem_capacity=4)
    e = _engine(p)
    log = CandidateLog(p, 4, e.unrank)
    gen = list(iter_repetend_assignments(p, 3))
    special = {5: CandidateRecord(3, gen[5], 4, "improved")}
    log.add_segment(3, 0, 20, special, infeasible=0)
    assert len(log) == 20
    assert log[5].status == "improved" and log[5].t_r == 4
    assert [r.assignment for r in log] == gen[:20]
    assert log.counts["improved"] == 1
