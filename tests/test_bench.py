"""bench.py's multi-GPU launcher path on CPU: ``python bench.py --gpus 2``
without a rank environment starts two ranks under torch.distributed.run
(127.0.0.1 rendezvous), the ranks run the sharded search (gloo here, NCCL on
the B200 box) and rank 0 prints ONE JSON line with n_gpus = 2 and parity
against the reference golden.

The engine has no CPU implementation, so a sitecustomize in a scratch
directory (put first on PYTHONPATH, for every process torchrun starts)
swaps in the oracle-backed stand-in of tests/cpu_engine.py — test
infrastructure only; bench.py itself is unchanged."""

import json
import os
import subprocess
import sys
from pathlib import Path

from conftest import ROOT

SHIM = r'''
import os, runpy, sys
_sys_site = "/usr/lib/python3.12/sitecustomize.py"
if os.path.exists(_sys_site):
    runpy.run_path(_sys_site)
if os.environ.get("TESSEL_BENCH_CPU_SHIM") == "1":
    sys.path.insert(0, os.environ["TESSEL_REPO"])
    sys.path.insert(0, os.path.join(os.environ["TESSEL_REPO"], "tests"))
    import paper_2311_15269_b200._core as core
    import paper_2311_15269_b200.engine as E
    from cpu_engine import OracleEngine, oracle_decide, oracle_decide_batch
    core.decide = oracle_decide
    core.decide_batch = oracle_decide_batch
    _init = E.BatchedRepetendSearch.__init__
    def _patched(self, p, device=0, native=None):
        _init(self, p, device, native if native is not None else OracleEngine(p))
    E.BatchedRepetendSearch.__init__ = _patched
'''


def _run(tmp_path, gpus):
    (tmp_path / "sitecustomize.py").write_text(SHIM)
    env = dict(os.environ, TESSEL_BENCH_CPU_SHIM="1", TESSEL_REPO=str(ROOT),
               PYTHONPATH=f"{tmp_path}{os.pathsep}{ROOT}", CUDA_VISIBLE_DEVICES="")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    proc = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(gpus),
                           "--steps", "2", "--warmup", "1", "--workload", "C1",
                           "--no-cpu-baseline"], env=env, capture_output=True, text=True,
                          timeout=900, cwd=str(ROOT))
    assert proc.returncode == 0, proc.stderr[-3000:]
    lines = [l for l in proc.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, proc.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_launcher_two_ranks_on_cpu(tmp_path):
    line = _run(tmp_path, 2)
    assert line["n_gpus"] == 2
    assert line["parity_vs_reference"] is True
    assert line["config"]["parallelism"].startswith("sharded2")
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["candidates_per_step"] == 90


def test_bench_single_rank_on_cpu(tmp_path):
    line = _run(tmp_path, 1)
    assert line["n_gpus"] == 1 and line["parity_vs_reference"] is True
