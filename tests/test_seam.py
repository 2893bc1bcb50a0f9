"""The drop-in boundary: the UNMODIFIED reference package
(oracle/_ref) runs its own ``solve_repetend``, ``solve_min_makespan`` and
``search`` with its decide seam routed to the B200 kernel, exactly as
INTEGRATION.md §2 tells a maintainer to do.

The test copies oracle/_ref/repsched to a scratch directory, applies the
documented edit to ``repsched/_core/__init__.py`` (reference
_core/__init__.py:9-23: the selector whitelist, the ``b200`` branch and
``KERNEL_NAME``) and imports that copy in a subprocess with
``REPSCHED_KERNEL=b200``.  Every result — including the reference's own
``SolveStats`` decide and node totals — must equal the golden the reference
produced with its compiled CPU kernel.
"""

import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import GOLDEN, ROOT

REF = ROOT / "oracle" / "_ref"

# the three edits of INTEGRATION.md §2, applied verbatim
WHITELIST_OLD = '("auto", "compiled", "pure")'
WHITELIST_NEW = '("auto", "compiled", "pure", "b200")'
BRANCH_OLD = "kernel = None\n"
BRANCH_NEW = ("kernel = None\n"
              "if _choice == \"b200\":\n"
              "    from paper_2311_15269_b200 import _core as kernel\n")
NAME_OLD = 'KERNEL_NAME = "compiled" if kernel.__name__.endswith("kernel_c") else "pure"'
NAME_NEW = ('KERNEL_NAME = "b200" if _choice == "b200" else (\n'
            '    "compiled" if kernel.__name__.endswith("kernel_c") else "pure")')


def patched_reference(dst: Path) -> Path:
    """Copy oracle/_ref's repsched to `dst` with INTEGRATION.md §2 applied."""
    shutil.copytree(REF / "repsched", dst / "repsched")
    init = dst / "repsched" / "_core" / "__init__.py"
    src = init.read_text()
    for old, new in ((WHITELIST_OLD, WHITELIST_NEW), (BRANCH_OLD, BRANCH_NEW),
                     (NAME_OLD, NAME_NEW)):
        assert src.count(old) == 1, old
        src = src.replace(old, new)
    init.write_text(src)
    return dst


def test_integration_doc_states_the_tested_patch():
    doc = (ROOT / "INTEGRATION.md").read_text()
    for snippet in (WHITELIST_NEW, "from paper_2311_15269_b200 import _core as kernel",
                    'KERNEL_NAME = "b200" if _choice == "b200"'):
        assert snippet in doc, snippet


def test_patched_reference_seam_imports_and_exports(tmp_path):
    """CPU: the patched selector loads the B200 seam (no compute call)."""
    if not (REF / "repsched").is_dir():
        pytest.skip("oracle/_ref not built")
    patched_reference(tmp_path)
    code = ("import repsched._core as c, paper_2311_15269_b200._core as b;"
            "assert c.KERNEL_NAME == 'b200' and c.decide is b.decide;"
            "assert (c.SAT, c.UNSAT, c.TIMEOUT) == (1, 0, 2); print('ok')")
    env = dict(os.environ, REPSCHED_KERNEL="b200",
               PYTHONPATH=f"{tmp_path}{os.pathsep}{ROOT}")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr[-2000:]


DRIVER = r"""
import json, sys, os
from repsched import _core, completion, placement, repetend, solver
assert _core.KERNEL_NAME == "b200"
out = {}
for name in sys.argv[1:]:
    doc = json.load(open(os.path.join(os.environ["GOLDEN"], f"search_{name}.json")))
    p = placement.placement_from_dict(doc["placement"])
    res = completion.search(p, doc["mem_capacity"], max_nr=doc["max_nr"],
                            lazy=doc.get("lazy", True))
    s = res.schedule
    counts = {}
    for c in res.report.candidates:
        counts[c.status] = counts.get(c.status, 0) + 1
    # single-candidate API on the golden's best repetend and its completion
    best = doc["improvements"][-1][0]
    st = solver.SolveStats()
    rep = repetend.solve_repetend(p, tuple(best), doc["mem_capacity"], stats=st)
    wu = tuple(sorted(completion.warmup_blocks(rep.repetend)))
    mk = solver.solve_min_makespan(solver.SolveRequest(
        placement=p, instances=wu, initial_memory=(0,) * p.num_devices,
        mem_capacity=doc["mem_capacity"])) if wu else None
    out[name] = {
        "best_t_r": res.report.best_t_r,
        "improvements": [[list(a), t] for a, t in res.report.improvements],
        "n_candidates": len(res.report.candidates), "status_counts": counts,
        "entries": sorted([b.stage, b.mb, t] for b, t in s.entries.items()),
        "makespan": s.makespan(), "diagnostics": res.report.diagnostics,
        "stats": [res.report.stats.decides, res.report.stats.nodes],
        "rep": [rep.status, rep.repetend.period, list(rep.repetend.internal)],
        "rep_decides": st.decides,
        "warmup": None if mk is None else [mk.status.name if hasattr(mk.status, "name")
                                            else str(mk.status), mk.objective],
    }
print("RESULT " + json.dumps(out))
"""


@pytest.mark.gpu
def test_reference_package_runs_on_the_b200_seam(gpu, tmp_path):
    """GPU: the reference's own search / solve_repetend / solve_min_makespan
    through the patched seam equal the reference's goldens — results, status
    counts and the reference's SolveStats (decides AND nodes: the B200 decide
    reproduces kernel_c's node counts)."""
    if not (REF / "repsched").is_dir():
        pytest.skip("oracle/_ref not built")
    names = ["C1", "C5_2", "x4_demo_k3", "m4_cap8", "eager_m4_cap8", "gate_pairs_b_cap3",
             "C2_3"]
    patched_reference(tmp_path)
    env = dict(os.environ, REPSCHED_KERNEL="b200", GOLDEN=str(GOLDEN),
               TESSEL_BUDGET_SECS="1e9", PYTHONPATH=f"{tmp_path}{os.pathsep}{ROOT}")
    proc = subprocess.run([sys.executable, "-c", DRIVER, *names], env=env, capture_output=True,
                          text=True, timeout=1800)
    assert proc.returncode == 0, proc.stderr[-3000:]
    line = next(l for l in proc.stdout.splitlines() if l.startswith("RESULT "))
    got = json.loads(line[len("RESULT "):])
    for name in names:
        doc = json.loads((GOLDEN / f"search_{name}.json").read_text())
        g = got[name]
        assert g["best_t_r"] == doc["best_t_r"], name
        assert g["improvements"] == doc["improvements"], name
        assert g["n_candidates"] == doc["n_candidates"], name
        assert g["status_counts"] == doc["status_counts"], name
        assert g["entries"] == doc["schedule"]["entries"], name
        assert g["makespan"] == doc["schedule"]["makespan"], name
        assert g["diagnostics"] == doc["diagnostics"], name
        assert g["stats"] == [doc["ref_stats"]["decides"], doc["ref_stats"]["nodes"]], name
        assert g["rep"][0] == "ok" and g["rep"][1] == doc["best_t_r"], name
        if g["warmup"] is not None:  # the warmup makespan is copy 0's offset
            assert g["warmup"][1] == doc["schedule"]["repetend"][0], name
