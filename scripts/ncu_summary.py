"""Summarise an ncu --metrics launch list (CSV) of `scripts/trace_search.py
<workload>` (2 searches) into per-kernel, per-search-step aggregates:
profiles/inst_counts.json (read by bench.py's roofline) and a markdown table.

usage: python scripts/ncu_summary.py gpurun_out/metrics.csv C2@4 [steps=2]
"""
import collections
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main(path, workload, steps=2):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    for r in rows:
        per[(int(r[ii]), r[ki].split("(")[0])][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    for (_, k), m in per.items():
        a = agg[k]
        a["launches"] += 1.0 / steps
        a["warp_inst"] += m.get("smsp__inst_executed.sum", 0) / steps
        a["thread_inst"] += m.get("smsp__thread_inst_executed.sum", 0) / steps
        a["alu_warp_inst"] += m.get("smsp__inst_executed_pipe_alu.sum", 0) / steps
        a["fma_warp_inst"] += m.get("smsp__inst_executed_pipe_fma.sum", 0) / steps
        a["lsu_warp_inst"] += m.get("smsp__inst_executed_pipe_lsu.sum", 0) / steps
        a["dram_bytes"] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / steps
        a["ncu_time_us"] += m.get("gpu__time_duration.sum", 0) / 1e3 / steps
    total = sum(a["ncu_time_us"] for a in agg.values()) or 1.0
    out = {"workload": workload,
           "basis": f"ncu --metrics ... --clock-control none over scripts/trace_search.py {workload} "
                    f"({steps} searches; values are per search step); {Path(path).name}",
           "per_step": {k: dict(v) for k, v in agg.items()}}
    (ROOT / "profiles" / "inst_counts.json").write_text(json.dumps(out, indent=1))
    print("| kernel | launches/step | ncu time/step (ms) | share | warp-inst/step | "
          "active lanes/inst | DRAM bytes/step |")
    print("|---|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ncu_time_us"]):
        lanes = a["thread_inst"] / a["warp_inst"] if a["warp_inst"] else 0
        print(f"| {k} | {a['launches']:.0f} | {a['ncu_time_us'] / 1e3:.2f} | "
              f"{100 * a['ncu_time_us'] / total:.1f}% | {a['warp_inst']:.3e} | {lanes:.1f} | "
              f"{a['dram_bytes'] / 1e6:.1f} MB |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 2)
