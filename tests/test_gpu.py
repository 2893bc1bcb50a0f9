"""GPU parity tests (run on a B200 with ``-m gpu``): every compute call goes
through the in-tree sm_100a library via the C ABI; results are compared
bit-exactly with the reference's golden fixtures and with the oracle."""

import json
import os
import random

import pytest

from conftest import GOLDEN, load_probes, load_search, probe_names

pytestmark = pytest.mark.gpu

SLOW = os.environ.get("TESSEL_SLOW", "0") == "1"


def _problem(p):
    return dict(n=p["n"], dur=p["dur"], devmask=p["devmask"], mem=p["mem"], edges=p["edges"],
                order=p["order"], lo=p["lo"], hi=p["hi"], ndev=p["ndev"], init_mem=p["init"],
                cap=p["cap"], node_budget=p["budget"])


@pytest.mark.parametrize("name", probe_names())
def test_decide_batch_matches_reference_probes(gpu, name):
    """k_decide_batch == reference kernel_c: status, lex-min witness, node
    count — including 400k-node capped TIMEOUT probes and completion probes."""
    probes = load_probes(name)
    got = gpu.decide_batch([_problem(p) for p in probes])
    for p, (st, s, nodes) in zip(probes, got):
        assert (st, s, nodes) == (p["status"], p["starts"], p["nodes"]), (name, p["kind"])


@pytest.mark.parametrize("name", ["C1", "C2_3", "nn4_k3", "C5_2"])
def test_decide_thread_kernel_matches_reference_probes(gpu, name, monkeypatch):
    """The one-thread-per-problem DFS kernel (TSL_DFS_MODE=thread) is kept as
    a cross-check of the default warp-cooperative kernel."""
    monkeypatch.setenv("TSL_DFS_MODE", "thread")
    probes = [p for p in load_probes(name) if p["kind"] != "capped"]
    got = gpu.decide_batch([_problem(p) for p in probes])
    for p, r in zip(probes, got):
        assert r == (p["status"], p["starts"], p["nodes"]), (name, p["kind"])


def test_decide_single_and_core_seam(gpu):
    from paper_2311_15269_b200 import _core

    assert _core.KERNEL_NAME == "b200"
    probes = load_probes("C1")[:20]
    for p in probes:
        r = _core.decide(p["n"], p["dur"], p["devmask"], p["mem"], p["edges"], p["order"],
                         p["lo"], p["hi"], p["ndev"], p["init"], p["cap"], p["budget"])
        assert r == (p["status"], p["starts"], p["nodes"])


def test_decide_edge_cases(gpu):
    import oracle

    cases = [
        (0, [], [], [], [], [], [], [], 2, [0, 0], -1, 0),          # empty
        (0, [], [], [], [], [], [], [], 1, [5], 3, 0),              # init > cap, no items
        (1, [2], [1], [1], [], [0], [0], [0], 1, [0], 0, 0),        # memory cap violated
        (2, [1, 1], [1, 1], [0, 0], [0, 1, 5, 1, 0, -3], [0, 1], [0, 0], [9, 9], 1, [0], -1, 0),
        (3, [2, 2, 2], [1, 1, 1], [0, 0, 0], [], [2, 0, 1], [0, 0, 0], [3, 3, 3], 1, [0], -1, 0),
        (3, [1, 1, 1], [3, 1, 2], [1, -1, 0], [0, 2, 1], [1, 0, 2], [0, 0, 0], [4, 4, 4], 2,
         [1, 0], 2, 1),                                              # node cap 1
    ]
    for c in cases:
        exp = oracle.decide(*c)
        got = gpu.decide(*c)
        assert got == exp, c


def test_decide_random_vs_oracle(gpu):
    import oracle

    rng = random.Random(5)
    probs, exps = [], []
    for _ in range(400):
        n = rng.randint(1, 9)
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
        hi = [v + rng.randint(0, 12) for v in lo]
        init = [rng.randint(0, 2) for _ in range(ndev)]
        cap = rng.choice((-1, 2, 3, 5))
        budget = rng.choice((0, 0, 5, 50))
        exps.append(oracle.decide(n, dur, mask, mem, edges, order, lo, hi, ndev, init, cap,
                                  budget))
        probs.append(dict(n=n, dur=dur, devmask=mask, mem=mem, edges=edges, order=order, lo=lo,
                          hi=hi, ndev=ndev, init_mem=init, cap=cap, node_budget=budget))
    assert gpu.decide_batch(probs) == exps


def _check(doc, res):
    assert res.report.best_t_r == doc["best_t_r"]
    assert [[list(a), t] for a, t in res.report.improvements] == doc["improvements"]
    assert len(res.report.candidates) == doc["n_candidates"]
    assert res.report.diagnostics == doc["diagnostics"]
    s = res.schedule
    assert sorted([b.stage, b.mb, t] for b, t in s.entries.items()) == doc["schedule"]["entries"]
    r = s.repetend
    assert [r.start, r.end, r.period, r.nr] == doc["schedule"]["repetend"]
    assert s.makespan() == doc["schedule"]["makespan"]
    counts = dict(res.report.candidates.counts)
    assert counts == doc["status_counts"]
    # the reference's decide count (every period probe of its sequential
    # scans plus the completion decides), reproduced exactly
    assert res.report.stats.decides == doc["ref_stats"]["decides"]
    nonbound = [[c.n_r, list(c.assignment), c.t_r, c.status]
                for c in (res.report.candidates[i] for i in range(len(res.report.candidates)))
                if c.status != "bound"] if doc["n_candidates"] <= 30000 else None
    if nonbound is not None:
        assert nonbound == doc["records"]


FAST = ["v4_unit_cap4", "v4_demo_cap4", "x4_demo_k3", "m4_cap8", "k4_k3", "v2_k4", "nn4_k3",
        "C1", "C2_3", "C3_9", "C5_2",
        # the full-size parity configs — seconds each on the B200
        "C2_4", "C3_12", "C4a_3", "C4a_4", "C4b", "C5_3",
        # BASELINE configs[4] (K16) at N_R <= 4 and <= 5 (9.4 M candidates):
        # reference goldens from tests/golden/make_par_golden.py (the
        # reference's own functions, sequential-equivalent, 13.6 min and
        # 3.7 h on the CPU container's cores)
        "C5_4", "C5_5",
        # eager completion (completion.py:359-368) and the entry-memory gate
        "eager_C1", "eager_C2_3", "eager_C3_9", "eager_m4_cap8", "eager_x4_demo_k3",
        "eager_v4_demo_cap4", "gate_pairs_a_cap4", "gate_pairs_b_cap3", "gate_pairs_c_cap5"]
# BASELINE configs[1] (8 micro-batches): its reference golden takes the CPU
# reference hours; checked when tests/golden/search_C2_8.json is present
SLOW_CASES = ["C2_8"]


@pytest.mark.parametrize("name", FAST)
def test_search_matches_reference(gpu, name):
    from paper_2311_15269_b200.completion import search
    from paper_2311_15269_b200.placement import placement_from_dict

    doc = load_search(name)
    p = placement_from_dict(doc["placement"])
    _check(doc, search(p, doc["mem_capacity"], max_nr=doc["max_nr"], lazy=doc.get("lazy", True)))


@pytest.mark.parametrize("name", SLOW_CASES)
def test_search_matches_reference_full_configs(gpu, name):
    if not (GOLDEN / f"search_{name}.json").exists():
        pytest.skip("golden not generated")
    from paper_2311_15269_b200.completion import search
    from paper_2311_15269_b200.placement import placement_from_dict

    doc = load_search(name)
    p = placement_from_dict(doc["placement"])
    _check(doc, search(p, doc["mem_capacity"], max_nr=doc["max_nr"]))


def test_search_random_placements(gpu):
    from paper_2311_15269_b200.completion import NoFeasibleSchedule, search
    from paper_2311_15269_b200.placement import placement_from_dict

    rows = json.loads((GOLDEN / "search_random.json").read_text())
    for row in rows:
        p = placement_from_dict(row["placement"])
        if row.get("error"):
            with pytest.raises((NoFeasibleSchedule, ValueError)):
                search(p, row["mem_capacity"], max_nr=row["max_nr"])
            continue
        res = search(p, row["mem_capacity"], max_nr=row["max_nr"])
        assert res.report.best_t_r == row["best_t_r"]
        assert [[list(a), t] for a, t in res.report.improvements] == row["improvements"]
        assert sorted([b.stage, b.mb, t] for b, t in res.schedule.entries.items()) == \
            row["schedule"]["entries"]
        assert len(res.report.candidates) == row["n_candidates"]


def test_solve_repetend_and_solver_spec_goldens(gpu):
    """SPEC examples G4, G5, G7, G8, G9 through the single-candidate API."""
    from paper_2311_15269_b200.completion import cooldown_blocks, warmup_blocks
    from paper_2311_15269_b200.placement import CostModel, make_shape
    from paper_2311_15269_b200.repetend import solve_repetend
    from paper_2311_15269_b200.solver import (SolveRequest, Status, full_request, solve_decide,
                                              solve_min_makespan)

    v4 = make_shape("vshape", 4, CostModel(1, 2, 1, -1))
    out = solve_repetend(v4, (3, 2, 1, 0, 0, 0, 0, 0), 4)
    r = out.repetend
    assert out.status == "ok" and r.period == 3
    assert r.internal == (6, 4, 2, 0, 1, 3, 5, 7)
    assert r.exec_spans == (3, 3, 3, 3) and r.waits == (0, 0, 0, 0)
    assert len(warmup_blocks(r)) == 6 and len(cooldown_blocks(r)) == 18
    z = solve_repetend(v4, (0,) * 8, 4).repetend
    assert z.period == 12 and z.internal == (0, 1, 2, 3, 4, 6, 8, 10)
    assert solve_min_makespan(full_request(v4, 1)).objective == 12
    assert solve_min_makespan(full_request(v4, 2)).objective == 15
    req = full_request(v4, 1, horizon=12, mode="decide")
    assert solve_decide(req).status == Status.SATISFIABLE
    req = full_request(v4, 1, horizon=11, mode="decide")
    assert solve_decide(req).status == Status.INFEASIBLE


def test_solve_repetend_matches_oracle(gpu):
    from oracle import search_port as SP
    from paper_2311_15269_b200.repetend import solve_repetend
    from paper_2311_15269_b200.workloads import WORKLOADS

    rng = random.Random(3)
    for wl in ("C2@3", "C3@9", "C5@2"):
        w = WORKLOADS[wl]
        p = w.placement()
        cands = list(SP.iter_assignments(p, 2))
        for a in rng.sample(cands, min(8, len(cands))):
            exp = SP.solve_repetend(p, a, w.mem_capacity, upper=None)
            got = solve_repetend(p, a, w.mem_capacity)
            assert got.status == exp.status
            if exp.status == "ok":
                assert got.repetend.internal == exp.internal
                assert got.repetend.period == exp.period


@pytest.mark.parametrize("mode", [1, 0])
def test_disjunctive_filter_on_device_never_refutes_a_feasible_probe(gpu, mode):
    """The device disjunctive filters (warp: wdj_solve.cuh, one-lane:
    dj_solve.cuh) on the reference-capped / DFS-heavy probes of
    tests/golden/dj_probes.json: never 'infeasible' for a probe whose exact
    verdict is SAT, agreement whenever they decide, and most capped probes
    refuted (the filter's purpose)."""
    from collections import defaultdict

    import numpy as np

    from paper_2311_15269_b200 import _native
    from paper_2311_15269_b200.workloads import WORKLOADS

    rows = json.loads((GOLDEN / "dj_probes.json").read_text())
    by = defaultdict(list)
    for r in rows:
        by[(r["workload"], r["cap"])].append(r)
    decided = capped = refuted_capped = 0
    for (wl, cap), rs in by.items():
        p = WORKLOADS[wl].placement()
        k = p.num_stages
        eng = _native.Engine([p.block(s).time_cost for s in range(k)],
                             [p.block(s).mem_delta for s in range(k)],
                             [sum(1 << d for d in p.block(s).devices) for s in range(k)],
                             sorted(p.deps), p.num_devices, 0)
        try:
            st, _ = eng.dj(np.array([r["a"] for r in rs]), np.array([r["P"] for r in rs]), cap,
                           200_000, mode)
        finally:
            eng.close()
        for r, v in zip(rs, st.tolist()):
            if r["truth"] == 1:
                assert v != 0, (wl, r["a"], r["P"])
            if v != 2 and r["truth"] != -1:
                decided += 1
                assert v == r["truth"], (wl, r["a"], r["P"])
            if r["ref_status"] == 2:
                capped += 1
                refuted_capped += v == 0
    assert decided > 0
    assert capped == 0 or refuted_capped / capped > 0.5


def _sharded_worker(rank, world, port, names, out_dir):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        from paper_2311_15269_b200 import _native
        from paper_2311_15269_b200.completion import search
        from paper_2311_15269_b200.parallel import Comm
        from paper_2311_15269_b200.placement import placement_from_dict

        _native.lib().tsl_set_device(0)
        comm = Comm()
        for name in names:
            doc = json.loads((root / "tests" / "golden" / f"search_{name}.json").read_text())
            p = placement_from_dict(doc["placement"])
            res = search(p, doc["mem_capacity"], max_nr=doc["max_nr"], comm=comm)
            s = res.schedule
            out = {"best_t_r": res.report.best_t_r,
                   "improvements": [[list(a), t] for a, t in res.report.improvements],
                   "n_candidates": len(res.report.candidates),
                   "entries": sorted([b.stage, b.mb, t] for b, t in s.entries.items()),
                   "makespan": s.makespan()}
            Path(out_dir, f"{name}_{rank}.json").write_text(json.dumps(out))
    finally:
        dist.destroy_process_group()


def test_sharded_search_two_ranks_on_device(gpu):
    """world_size 2 (gloo plumbing, both ranks' engines on cuda:0): rank-prefix
    windows, per-level bound exchange, all-gathered SAT rows — the real
    kernels, identical results on both ranks and equal to the reference."""
    import socket
    import tempfile
    from pathlib import Path

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    names = ["C2_3", "C5_2", "C4b"]
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_sharded_worker, args=(2, port, names, out), nprocs=2, join=True)
        for name in names:
            doc = load_search(name)
            exp = {"best_t_r": doc["best_t_r"], "improvements": doc["improvements"],
                   "n_candidates": doc["n_candidates"], "entries": doc["schedule"]["entries"],
                   "makespan": doc["schedule"]["makespan"]}
            r0 = json.loads(Path(out, f"{name}_0.json").read_text())
            r1 = json.loads(Path(out, f"{name}_1.json").read_text())
            assert r0 == r1 == exp, name


@pytest.mark.parametrize("helpers", ["0", "4"])
def test_subtree_parallel_nested_runs_exact(gpu, monkeypatch, helpers):
    """Small per-round task budgets force oversized subtree tasks into nested
    runs — one at a time, or concurrently on helper workers — on the long
    (8M-capped) golden probes: status, witness and node count still exact."""
    monkeypatch.setenv("TSL_SP_TASK_NODES", "16384")
    monkeypatch.setenv("TSL_SP_HELPERS", helpers)
    probes = [p for name in ("C3_12", "to_m4_n3_cap6", "C4a_4") for p in load_probes(name)
              if p["budget"] >= 1_000_000 and p["nodes"] > 100_000]
    assert probes
    for p in probes:
        got = gpu.decide_batch([_problem(p)])[0]
        assert got == (p["status"], p["starts"], p["nodes"]), p["n"]


@pytest.mark.parametrize("env", [{"TSL_DJ_SPLIT": "1"}, {"TSL_SP_PIPELINE": "0"},
                                 {"TSL_ROOT_FILTER": "0"}])
def test_search_variants_match_reference(gpu, monkeypatch, env):
    """The non-default execution variants kept for cross-validation (split
    disjunctive-filter launch, no pipelined SP master walk, thread-per-probe
    level pass) give the same searches."""
    from paper_2311_15269_b200.completion import search
    from paper_2311_15269_b200.placement import placement_from_dict

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for name in ("C2_3", "C5_2", "C3_9", "m4_cap8"):
        doc = load_search(name)
        p = placement_from_dict(doc["placement"])
        _check(doc, search(p, doc["mem_capacity"], max_nr=doc["max_nr"]))


def _probe_inputs(p, a, period):
    """The reference's probe for (assignment, period): repetend.py:160-190."""
    from paper_2311_15269_b200.repetend import _model_for, entry_memory

    m = _model_for(p)
    m.set_assignment(a)
    anchor = (m.k - 1) * (period + m.max_dur)
    lo, hi = [0] * m.k, [2 * anchor] * m.k
    if m.k:
        lo[0] = hi[0] = anchor
    return (m.k, m.dur, m.mask, m.mem, m.edges(period), m.order, lo, hi, p.num_devices,
            list(entry_memory(p, a)))


@pytest.mark.parametrize("kernel", ["strong", "wrr", "wrx"])
def test_repetend_probe_kernel_matches_oracle(gpu, monkeypatch, kernel):
    """k_verify_warp's per-warp decide — the register-resident exact DFS
    (wrr_dfs.cuh, TSL_REP_STRONG=0), the shared-memory one (wrx_dfs.cuh,
    TSL_REP_DFS=wrx) and the default strong search with the exact DFS only
    for SATs within a cap (wst_dfs.cuh) — against the oracle's kernel_c
    restatement on random (candidate, period) probes of every shape (single-
    and multi-device blocks, K = 8..34, with and without a memory cap), with
    node caps that end probes mid-search.  Exact kernels: status, node count
    and witness.  Strong: the repetend scan's verdict — SAT with the
    reference's witness, or not SAT exactly when the reference is UNSAT or
    TIMEOUT (repetend.py:294-299)."""
    import numpy as np

    import oracle
    from paper_2311_15269_b200 import _native
    from paper_2311_15269_b200.placement import placement_from_dict
    from paper_2311_15269_b200.workloads import WORKLOADS

    if kernel == "wrx":
        monkeypatch.setenv("TSL_REP_DFS", "wrx")
    if kernel == "wrr":
        monkeypatch.setenv("TSL_REP_STRONG", "0")
    rng = random.Random(17)
    cases = [(WORKLOADS[w].placement(), WORKLOADS[w].mem_capacity, n_r)
             for w, n_r in (("C2@8", 4), ("C3@9", 3), ("C4a@4", 3), ("C4b", 5), ("C5@4", 3),
                            ("C1", 3))]
    for name in ("m4_cap8", "x4_demo_k3", "k4_k3", "nn4_k3", "gate_pairs_a_cap4"):
        doc = load_search(name)
        cases.append((placement_from_dict(doc["placement"]), doc["mem_capacity"], 3))
    for row in json.loads((GOLDEN / "search_random.json").read_text())[:24]:
        cases.append((placement_from_dict(row["placement"]), row["mem_capacity"], 3))
    checked = timeouts = sats = 0
    for p, cap, n_r in cases:
        k = p.num_stages
        eng = _native.Engine([p.block(s).time_cost for s in range(k)],
                             [p.block(s).mem_delta for s in range(k)],
                             [sum(1 << d for d in p.block(s).devices) for s in range(k)],
                             sorted(p.deps), p.num_devices, 0)
        try:
            count = eng.count(n_r)
            if count == 0:
                continue
            r1 = min(count, 4096)
            eng.stage(n_r, 0, r1, cap)
            lb = max(p.device_load(d) for d in range(p.num_devices))
            total = sum(b.time_cost for b in p.blocks)
            widx, per, bud = [], [], []
            for _ in range(48):
                widx.append(rng.randrange(r1))
                per.append(rng.choice((lb, lb, lb + 1, rng.randint(lb, min(total, lb + 5)))))
                bud.append(rng.choice((3, 12, 60, 700, 5000, 40000)))
            st, nd, rows = eng.verify(widx, per, bud, cap)
            # a SAT (w, q) cancels pairs (w2 > w, q2 >= q) of the same launch
            # (the engine's speculative retirement): re-run those alone
            for i in np.nonzero(st == _native.ABORT)[0]:
                s1, n1, r1 = eng.verify([widx[i]], [per[i]], [bud[i]], cap)
                st[i], nd[i], rows[i] = s1[0], n1[0], r1[0]
            for i, (w, q, b) in enumerate(zip(widx, per, bud)):
                a = eng.unrank(n_r, w)
                exp = oracle.decide(*_probe_inputs(p, a, q), -1 if cap is None else cap, b)
                got = (int(st[i]), [int(v) for v in rows[i]] if st[i] == 1 else None, int(nd[i]))
                if kernel == "strong":
                    assert (got[0] == 1) == (exp[0] == 1), (k, a, q, b, got[0], exp[0])
                    assert got[1] == exp[1], (k, a, q, b)
                else:
                    assert got == (exp[0], exp[1], exp[2]), (k, a, q, b)
                checked += 1
                timeouts += exp[0] == 2
                sats += exp[0] == 1
        finally:
            eng.close()
    assert checked > 1000 and timeouts > 100 and sats > 100, (checked, timeouts, sats)


def test_decide_k16_sixteen_microbatches_vs_oracle(gpu):
    """BASELINE configs[4] at 16 micro-batches: the monolithic lowering of
    the K16 placement's 34 x 16 = 544 blocks (solver.py:96-167) exceeds the
    round-1 item limit; the decide runs on the device (one warp: problems
    above the subtree-parallel limit) with the reference's status, witness
    and node count at several horizons and node caps."""
    import oracle
    from paper_2311_15269_b200.solver import Lowering, full_request
    from paper_2311_15269_b200.workloads import WORKLOADS

    p = WORKLOADS["C5@4"].placement()
    low = Lowering(full_request(p, 16))
    assert low.n == 544
    lb = low.lower_bound()
    total = low.sum_free_dur()
    for horizon, budget in ((total, 0), (lb + 40, 3000), (lb + 8, 20000), (lb, 5000)):
        prob = low.problem(horizon, budget)
        if prob is None:
            continue
        got = gpu.decide_batch([prob])[0]
        exp = oracle.decide(prob["n"], prob["dur"], prob["devmask"], prob["mem"], prob["edges"],
                            prob["order"], prob["lo"], prob["hi"], prob["ndev"],
                            prob["init_mem"], prob["cap"], budget)
        assert got == (exp[0], exp[1], exp[2]), (horizon, budget, got[0], got[2], exp[0], exp[2])


@pytest.mark.parametrize("env", [{"TSL_SP_DONATE": "0"},
                                 {"TSL_SP_DONATE_FORCE": "1", "TSL_SP_DONATE_EVERY": "16"},
                                 {"TSL_SP_DONATE_FORCE": "1", "TSL_SP_DONATE_EVERY": "1"},
                                 {"TSL_SP_DONATE_EVERY": "8", "TSL_SP_PAUSE": "4096"},
                                 {"TSL_SP_DONATE_WINDOW": "-1"}, {"TSL_SP_DONATE_WINDOW": "0"}])
def test_subtree_parallel_donation_exact(gpu, monkeypatch, env):
    """Task launches that split their subtrees dynamically (idle warps take
    the shallowest untried siblings of running pieces; forced donation at
    every check builds deep piece trees and fills the piece queue) settle
    every long golden probe exactly: status, lex-min witness, node count."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    probes = [p for name in probe_names() for p in load_probes(name)
              if (p["budget"] >= 1_000_000 or p["budget"] == 0) and p["nodes"] > 20_000]
    assert len(probes) >= 10
    for p in probes:
        got = gpu.decide_batch([_problem(p)])[0]
        assert got == (p["status"], p["starts"], p["nodes"]), (p["n"], p["status"], p["nodes"])


@pytest.mark.parametrize("env", [{}, {"TSL_SP_DONATE_FORCE": "1", "TSL_SP_DONATE_EVERY": "16"},
                                 {"TSL_SP_DONATE_ANY_S": "1"},
                                 {"TSL_SP_DONATE_ANY_S": "1", "TSL_SP_DONATE_FORCE": "1",
                                  "TSL_SP_DONATE_EVERY": "16"}])
def test_subtree_parallel_sticky_set_epochs_exact(gpu, monkeypatch, env):
    """400k-capped repetend probes whose sticky sets change many times, run
    subtree-parallel: after each change the rest of the task is re-run on
    the new set (epochs) — status, witness and node count stay exact."""
    monkeypatch.setenv("TSL_SP_MIN_BUDGET", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    probes = [p for name in ("C3_9", "C4a_3", "nn4_k3") for p in load_probes(name)
              if p["kind"] == "capped" and p["nodes"] > 50_000][:10]
    assert len(probes) >= 6
    for p in probes:
        got = gpu.decide_batch([_problem(p)])[0]
        assert got == (p["status"], p["starts"], p["nodes"]), (p["n"], p["status"], p["nodes"])
