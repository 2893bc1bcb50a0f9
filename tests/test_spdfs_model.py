"""CPU test of the subtree-parallel decide ALGORITHM (csrc/sp_dfs.cuh +
csrc/sp_host.inc): tests/native/sp_sim.cpp runs the same master walk /
speculative subtree tasks / in-order verification / replay / nested
sub-solve scheme sequentially on the host (with the host build of the DFS
steps) and must reproduce the reference's status, lex-min witness and node
count on the golden decide probes for any split depth and round sizes.  The
parameters are deliberately tiny so every mechanism (many rounds, sticky-set
mispredictions and replays, oversized tasks solved as nested runs, split
depth adaptation) is exercised.  The CUDA implementation itself is checked
against the same fixtures on the GPU (tests/test_gpu.py)."""

import gzip
import json
import subprocess

import pytest

from conftest import GOLDEN, ROOT


@pytest.fixture(scope="module")
def sp_sim(tmp_path_factory):
    exe = tmp_path_factory.mktemp("sp") / "sp_sim"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", str(exe),
                           str(ROOT / "tests" / "native" / "sp_sim.cpp")])
    return exe


def _toks(p):
    e = p["edges"]
    flat = [x for t in e for x in t] if e and isinstance(e[0], list) else e
    return (["G", p["n"], len(flat) // 3, p["ndev"], p["cap"], p["budget"]] + p["dur"] + p["mem"]
            + p["devmask"] + flat + p["order"] + p["lo"] + p["hi"] + p["init"])


def _probes(name, lo, hi, limit):
    d = json.loads(gzip.open(GOLDEN / f"probes_{name}.json.gz").read())["probes"]
    ps = [p for p in d if lo <= p["nodes"] <= hi]
    return ps[:limit]


@pytest.mark.parametrize("ck", ["64", "1"])  # replay checkpoint interval (tasks)
@pytest.mark.parametrize("params", [
    (256, 64, 1024, 2048, 0),     # histogram split depth, small rounds
    (128, 16, 512, 512, 3),       # shallow split: big tasks -> nested runs
    (512, 256, 4096, 1 << 20, 8), # deep split, large tasks
])
def test_subtree_parallel_scheme_is_exact(sp_sim, params, ck):
    import os

    probes = []
    for name in ("C2_3", "C3_9", "C4a_3", "C5_2", "C3_12", "nn4_k3"):
        probes += _probes(name, 300, 60_000, 6)
    assert len(probes) >= 20
    inp = []
    for p in probes:
        inp += ["P", *params] + _toks(p)
    out = subprocess.run([str(sp_sim)], input=" ".join(map(str, inp)), capture_output=True,
                         text=True, check=True, timeout=600,
                         env={**os.environ, "SP_CK": ck}).stdout.split("\n")
    replays = subsolves = 0
    for p, line in zip(probes, out):
        r = list(map(int, line.split()))
        st, nodes = r[0], r[1]
        starts = r[7:] if st == 1 else None
        assert (st, nodes, starts) == (p["status"], p["nodes"], p["starts"]), (p["kind"], p["n"])
        replays += r[4]
        subsolves += r[5]
    if params[1] <= 64:
        assert replays > 0
    if params[3] <= 512:
        assert subsolves > 0
