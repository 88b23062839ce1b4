#!/usr/bin/env python
"""Build (here) / run (GPU box) kernel tuning variants of liblfoam.

  python scripts/variants.py build            # nvcc all variants in-tree
  python scripts/variants.py run [cfg ...]    # bench each variant, print a table
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {
    "base": [],
    "pf0": ["LF_PF=0"],
    "pf2": ["LF_PF=2"],
    "mg4": ["LF_MINB_G=4"],
    "mg6": ["LF_MINB_G=6"],
}


def build():
    from paper_2507_18268_b200 import build as B
    for name, defs in VARIANTS.items():
        print(name, B.build(force=True, defines=defs or ["LF_VARIANT_BASE=1"], out=f"liblfoam_{name}.so"), flush=True)


def run(cfgs):
    rows = []
    for cfg in cfgs:
        for name in VARIANTS:
            env = dict(os.environ, LFOAM_LIB=f"liblfoam_{name}.so")
            r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "10", "--warmup", "3",
                                "--config", str(cfg), "--no-cpu-baseline"], capture_output=True, text=True, env=env,
                               timeout=900)
            line = [l for l in r.stdout.splitlines() if l.startswith("{")]
            if not line:
                print(name, cfg, "FAILED", r.stderr[-2000:], flush=True)
                continue
            d = json.loads(line[-1])
            rf = d["roofline"]
            row = dict(variant=name, cfg=cfg, ms_step=round(d["ms_per_step"], 3), value=f"{d['value']:.3e}",
                       it=d["config"]["pcg_iterations_per_step"]["mean"],
                       p1_us=round(rf["avg_launch_ms"] * 1e3, 2), p1_GBs=round(rf["achieved"] or 0),
                       p2_us=round(rf["phase2"]["avg_launch_ms"] * 1e3, 2),
                       p2_GBs=round(rf["phase2"]["achieved"] or 0),
                       inst_ms=round(rf["instrumented_ms_per_step"], 3))
            rows.append(row)
            print(json.dumps(row), flush=True)
    return rows


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run([int(c) for c in sys.argv[2:]] or [2])
