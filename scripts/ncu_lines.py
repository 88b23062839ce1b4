#!/usr/bin/env python
"""Top source lines by warp-stall samples of an ncu report (all files):
  python scripts/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, res = list(csv.reader(io.StringIO(out))), None, []
    h = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            h = r
        elif h and len(r) == len(h) and r[0].isdigit():
            try:
                s = int(r[4] or 0)
            except ValueError:
                continue
            if s:
                res.append((s, f"{fname}:{r[0]}", r[1][:100]))
    tot = sum(x[0] for x in res) or 1
    for s, loc, src in sorted(res, reverse=True)[:top]:
        print(f"{s / tot:6.1%}  {loc:18s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
