"""CPU tests: pin the oracle against the reference's golden fixtures, and check
the device DFS routine's logic (compiled for the host by a test harness)
against the same fixtures.  No GPU needed."""

import subprocess
from pathlib import Path

import pytest

from conftest import GOLDEN, ROOT, load_probes, load_search, probe_names

import oracle
from oracle import search_port as SP
from paper_2311_15269_b200.placement import placement_from_dict


def _expected(p):
    return (p["status"], p["starts"], p["nodes"])


@pytest.mark.parametrize("name", probe_names())
def test_oracle_decide_matches_reference_probes(name):
    """oracle/decide_port.c == reference kernel_c on recorded probes
    (root refutations, DFS, 400k-capped TIMEOUTs, completion probes)."""
    for p in load_probes(name):
        got = oracle.decide(p["n"], p["dur"], p["devmask"], p["mem"], p["edges"], p["order"],
                            p["lo"], p["hi"], p["ndev"], p["init"], p["cap"], p["budget"])
        assert got == _expected(p), (name, p["kind"])


@pytest.fixture(scope="module")
def rx_host(tmp_path_factory):
    exe = tmp_path_factory.mktemp("rx") / "rx_host_check"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", str(exe),
                           str(ROOT / "tests" / "native" / "rx_host_check.cpp")])
    return exe


def _gen_line(p):
    m = len(p["edges"]) // 3
    vals = [p["n"], m, p["ndev"], p["cap"], p["budget"], *p["dur"], *p["mem"], *p["devmask"],
            *p["edges"], *p["order"], *p["lo"], *p["hi"], *p["init"]]
    return "G " + " ".join(map(str, vals))


@pytest.mark.parametrize("name", probe_names())
def test_device_dfs_logic_matches_reference_probes(rx_host, name):
    """rx_dfs.cuh (trail-based undo, int32) reproduces status, witness and
    node count of the reference on every recorded probe."""
    probes = load_probes(name)
    out = subprocess.run([str(rx_host)], input="\n".join(map(_gen_line, probes)) + "\n",
                         capture_output=True, text=True, check=True).stdout.split("\n")
    for p, line in zip(probes, out):
        t = list(map(int, line.split()))
        assert t[0] == p["status"] and t[1] == p["nodes"], (name, p["kind"], t[:2])
        if p["status"] == 1:
            assert t[2:] == p["starts"]


def _rep_block(placement, queries):
    K = placement.num_stages
    dur = [placement.block(s).time_cost for s in range(K)]
    mem = [placement.block(s).mem_delta for s in range(K)]
    mask = [sum(1 << d for d in placement.block(s).devices) for s in range(K)]
    deps = sorted(placement.deps)
    head = ["R", K, placement.num_devices, len(deps), *dur, *mem, *mask,
            *[v for e in deps for v in e], len(queries)]
    body = []
    for a, P, cap, budget in queries:
        body += [P, cap, budget, *a]
    return " ".join(map(str, head + body))


@pytest.mark.parametrize("wl", ["C1", "C2@3", "C3@9", "C4b", "C5@2"])
def test_device_repetend_view_matches_oracle(rx_host, wl):
    """RepView (period-parametric lags, anchored bounds, entry memory)
    == the oracle's repetend probe on sampled candidates and periods."""
    import random

    from paper_2311_15269_b200.workloads import WORKLOADS

    w = WORKLOADS[wl]
    p = w.placement()
    model = SP.ProbeModel(p)
    rng = random.Random(7)
    cands = list(SP.iter_assignments(p, 2)) + list(SP.iter_assignments(p, 3))
    rng.shuffle(cands)
    lb = SP.lower_bound(p)
    queries = []
    for a in cands[:60]:
        for P in (lb, lb + 1, lb + 3):
            queries.append((a, P, -1 if w.mem_capacity is None else w.mem_capacity,
                            0 if P == lb else 20000))
    out = subprocess.run([str(rx_host)], input=_rep_block(p, queries) + "\n",
                         capture_output=True, text=True, check=True).stdout.split("\n")
    for (a, P, cap, budget), line in zip(queries, out):
        st, w_, nodes = model.probe(a, P, None if cap < 0 else cap,
                                    SP.entry_memory(p, a), budget)
        t = list(map(int, line.split()))
        assert t[:2] == [st, nodes], (a, P)
        if st == 1:
            assert t[2:] == w_


SMALL = ["v4_unit_cap4", "v4_demo_cap4", "x4_demo_k3", "m4_cap8", "k4_k3", "v2_k4", "C1",
         "nn4_k3", "C3_9"]


def _check_port(doc, res):
    assert [[list(a), t] for a, t in res.improvements] == doc["improvements"]
    assert res.n_candidates == doc["n_candidates"]
    assert res.diagnostics == doc["diagnostics"]
    s = res.schedule
    assert sorted([b.stage, b.mb, t] for b, t in s.entries.items()) == doc["schedule"]["entries"]
    r = s.repetend
    assert [r.start, r.end, r.period, r.nr] == doc["schedule"]["repetend"]
    assert s.makespan() == doc["schedule"]["makespan"]
    counts = dict(res.status_counts)
    assert counts == doc["status_counts"]


@pytest.mark.parametrize("name", SMALL)
def test_search_port_matches_reference(name):
    doc = load_search(name)
    p = placement_from_dict(doc["placement"])
    res = SP.search(p, doc["mem_capacity"], doc["max_nr"])
    _check_port(doc, res)


def test_search_port_random_placements():
    import json

    rows = json.loads((GOLDEN / "search_random.json").read_text())
    assert len(rows) >= 50
    for row in rows:
        p = placement_from_dict(row["placement"])
        if row.get("error"):
            with pytest.raises(Exception):
                SP.search(p, row["mem_capacity"], row["max_nr"])
            continue
        res = SP.search(p, row["mem_capacity"], row["max_nr"])
        assert [[list(a), t] for a, t in res.improvements] == row["improvements"]
        assert sorted([b.stage, b.mb, t] for b, t in res.schedule.entries.items()) == \
            row["schedule"]["entries"]


def test_reference_crosscheck_when_available():
    """When the compiled reference (oracle/_ref) is present, the oracle
    matches it on freshly generated random probes too."""
    ref = oracle.load_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    import random

    import repsched._core as RC

    rng = random.Random(11)
    for _ in range(300):
        n = rng.randint(1, 7)
        ndev = rng.randint(1, 3)
        dur = [rng.randint(1, 3) for _ in range(n)]
        mem = [rng.choice((-1, 0, 1)) for _ in range(n)]
        mask = [rng.randint(1, (1 << ndev) - 1) for _ in range(n)]
        edges = []
        for i in range(n):
            for j in range(n):
                if i != j and rng.random() < 0.2:
                    edges += [i, j, rng.randint(-4, 3)]
        order = list(range(n))
        rng.shuffle(order)
        lo = [rng.randint(0, 3) for _ in range(n)]
        hi = [v + rng.randint(0, 10) for v in lo]
        init = [rng.randint(0, 2) for _ in range(ndev)]
        cap = rng.choice((-1, 2, 3, 5))
        budget = rng.choice((0, 0, 5, 50))
        args = (n, dur, mask, mem, edges, order, lo, hi, ndev, init, cap, budget, 0.0)
        assert oracle.decide(*args) == RC.decide(*args)


def test_disjunctive_filter_never_refutes_a_feasible_probe(rx_host):
    """DJ (csrc/dj_solve.cuh) is used only to prove repetend probes
    infeasible.  On the probes the reference node-caps (plus DFS-heavy ones)
    it must never answer UNSAT when the probe is feasible, and it must agree
    with the oracle's exact verdict whenever it decides."""
    import json
    from collections import defaultdict

    from paper_2311_15269_b200.workloads import WORKLOADS

    path = GOLDEN / "dj_probes.json"
    if not path.exists():
        pytest.skip("dj_probes.json not generated")
    rows = json.loads(path.read_text())
    by_wl = defaultdict(list)
    for r in rows:
        by_wl[r["workload"]].append(r)
    decided = refuted_capped = capped = 0
    for wl, rs in by_wl.items():
        p = WORKLOADS[wl].placement()
        qs = [(r["a"], r["P"], -1 if r["cap"] is None else r["cap"], 200_000) for r in rs]
        out = subprocess.run([str(rx_host)], input=_rep_block(p, qs).replace("R ", "J ", 1) + "\n",
                             capture_output=True, text=True, check=True).stdout.split("\n")
        for r, line in zip(rs, out):
            verdict, _ = map(int, line.split())
            if r["truth"] == 1:
                assert verdict != 0, (wl, r["a"], r["P"])
            if verdict != 2 and r["truth"] != -1:
                decided += 1
                assert verdict == r["truth"], (wl, r["a"], r["P"])
            if r["ref_status"] == 2:
                capped += 1
                refuted_capped += verdict == 0
    assert decided > 0
    # the filter is only useful if it settles most reference-capped probes
    assert capped == 0 or refuted_capped / capped > 0.5
