"""Key metrics of a one-kernel `ncu --set full` report (raw page): duration,
instructions, launch shape, occupancy, issue activity, DRAM bytes and the
top warp-stall reasons.  usage: ncu_rep_summary.py <report.ncu-rep>"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print("kernel", d.get("Kernel Name", "?")[:60])
    for k in KEYS:
        print(k, d.get(k), u.get(k, ""))
    stalls = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    for v, k in sorted(stalls, reverse=True)[:8]:
        print("stall", k, round(v, 3))


if __name__ == "__main__":
    main(sys.argv[1])
