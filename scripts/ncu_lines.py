"""Top CUDA source lines of an ncu report by warp-stall samples and executed
instructions (cuda,sass source view).  usage: ncu_lines.py <report> [top]"""
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows, path, hdr = [], None, None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].rsplit("/", 1)[-1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and r[0].isdigit():
            d = dict(zip(hdr[2:], r[2:]))
            try:
                s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                i = int(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            rows.append((s, i, f"{path}:{r[0]}", r[1].strip()[:90]))
    ts = sum(r[0] for r in rows) or 1
    ti = sum(r[1] for r in rows) or 1
    print(f"total samples {ts}  warp-inst {ti}")
    for s, i, loc, src in sorted(rows, reverse=True)[:int(top)]:
        print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% inst  {loc:22s} {src}")


if __name__ == "__main__":
    main(*sys.argv[1:])
