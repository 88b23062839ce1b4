#!/usr/bin/env python
"""Summarise ncu reports (gpurun_out/prof_<tag>_cfg<c>_<kernel>.ncu-rep) and
launch lists into profiles/<tag>_ncu_summary.md and profiles/ncu_traffic.json.

  python scripts/ncu_summary.py <tag>
"""
import csv
import glob
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("NCU_SUMMARY_DIR", os.path.join(ROOT, "profiles"))
sys.path.insert(0, ROOT)
from bench import build_id  # noqa: E402

# the build the reports were captured on: NCU_BUILD (written by the profiling
# script on the box), else the current sources
BUILD = os.environ.get("NCU_BUILD") or build_id()

DETAILS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput",
           "L2 Hit Rate", "L1/TEX Hit Rate", "Achieved Occupancy", "Registers Per Thread", "Grid Size",
           "Block Size", "Warp Cycles Per Issued Instruction"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def ncu_csv(rep, page):
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * scale


def summarise(rep):
    rows = ncu_csv(rep, "details")
    h = rows[0]
    det = {}
    for row in rows[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in DETAILS and d.get("Section Name") != "PM Sampling":
            det.setdefault(d["Metric Name"], f"{d['Metric Value']} {d['Metric Unit']}".strip())
    raw = ncu_csv(rep, "raw")
    rh, ru, rv = raw[0], raw[1], raw[2]
    rd = {}
    for name in RAW:
        if name in rh:
            i = rh.index(name)
            rd[name] = (rv[i], ru[i])
    traffic = None
    if "dram__bytes_read.sum" in rd and "dram__bytes_write.sum" in rd:
        traffic = to_bytes(*rd["dram__bytes_read.sum"]) + to_bytes(*rd["dram__bytes_write.sum"])
    return det, rd, traffic


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        k = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
        m = d["Metric Name"]
        v = to_bytes(d["Metric Value"], d["Metric Unit"]) if "bytes" in m else float(d["Metric Value"].replace(",", ""))
        a = agg.setdefault(k, {})
        a.setdefault(m, []).append(v)
    return agg


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary — {tag}", "",
             "Captured with `scripts/profile.sh` under gpurun on one B200 (`ncu --set full "
             "--clock-control none`, cold cache: ncu flushes caches before each replay).  "
             "Per-launch figures; `traffic` = dram read + write bytes.", ""]
    tj_path = os.path.join(PROF, "ncu_traffic.json")
    tj = json.load(open(tj_path)) if os.path.exists(tj_path) else {}
    for rep in sorted(glob.glob(os.path.join(OUT, f"prof_{tag}_cfg*_k_*.ncu-rep"))):
        m = re.search(r"cfg(\d+(?:-corr\d+)?(?:-dt)?(?:-dic)?(?:-gamg)?(?:-rcm)?)_(k_\w+)\.ncu-rep", rep)
        cfg, kern = m.group(1), m.group(2)
        det, rd, traffic = summarise(rep)
        lines.append(f"## config {cfg} — `{kern}`")
        lines.append("")
        for k in DETAILS:
            if k in det:
                lines.append(f"- {k}: {det[k]}")
        for k, (v, u) in rd.items():
            lines.append(f"- `{k}`: {v} {u}")
        if traffic is not None:
            lines.append(f"- traffic (DRAM read+write): {traffic / 1e6:.1f} MB per launch")
            # tied to the device-code build it was captured on (bench.py drops stale figures)
            tj.setdefault(f"config{cfg}", {})[kern] = {"bytes": traffic, "build": BUILD, "tag": tag}
        lines.append("")
    for path in sorted(glob.glob(os.path.join(OUT, f"launches_{tag}_cfg*.csv"))):
        cfg = re.search(r"cfg(\d+(?:-corr\d+)?(?:-dt)?(?:-dic)?(?:-gamg)?(?:-rcm)?)", path).group(1)
        agg = launch_table(path)
        lines.append(f"## config {cfg} — launch list (`--metrics gpu__time_duration.sum,dram__bytes_*`)")
        lines.append("")
        lines.append("| kernel | launches | mean time (us) | share of listed time | mean DRAM MB |")
        lines.append("|---|---|---|---|---|")
        tot = sum(sum(a.get("gpu__time_duration.sum", [])) for a in agg.values())
        for k, a in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", []))):
            t = a.get("gpu__time_duration.sum", [])
            dr = [x + y for x, y in zip(a.get("dram__bytes_read.sum", []), a.get("dram__bytes_write.sum", []))]
            lines.append(f"| `{k}` | {len(t)} | {sum(t) / max(len(t), 1) / 1e3:.2f} | "
                         f"{sum(t) / tot:.1%} | {sum(dr) / max(len(dr), 1) / 1e6:.1f} |")
        lines.append("")
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(tj_path, "w") as f:
        json.dump(tj, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1])
