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

# name -> (-D defines, bench --mode[, bench --precond])
VARIANTS = {
    "fit1": ([], "persistent"),
    "fit0": (["LF_STASH_FIT=0"], "persistent"),
    "fit1-dic": ([], "persistent", "DIC"),
    "fit0-dic": (["LF_STASH_FIT=0"], "persistent", "DIC"),
}


def libname(name):
    return f"liblfoam_{name}.so"


def build():
    from paper_2507_18268_b200 import build as B
    built = {}
    for name, (defs, *_) in VARIANTS.items():
        key = tuple(defs)
        if key in built:  # same defines: reuse
            continue
        built[key] = B.build(force=True, defines=list(defs) or ["LF_VARIANT_BASE=1"], out=libname(name))
        print(name, built[key], flush=True)


def lib_for(name):
    defs = tuple(VARIANTS[name][0])
    for other, (d, *_) in VARIANTS.items():
        if tuple(d) == defs:
            return libname(other)


def run(cfgs, steps=10):
    rows = []
    for cfg in cfgs:
        for name, (_, mode, *pc) in VARIANTS.items():
            env = dict(os.environ, LFOAM_LIB=lib_for(name))
            r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(steps), "--warmup", "3",
                                "--config", str(cfg), "--no-cpu-baseline", "--mode", mode,
                                "--precond", pc[0] if pc else "diagonal",
                                "--variant", str(pc[1] if len(pc) > 1 else 0)],
                               capture_output=True, text=True, env=env, timeout=1800)
            line = [l for l in r.stdout.splitlines() if l.startswith("{")]
            if not line:
                print(name, cfg, "FAILED", r.stderr[-2000:], flush=True)
                continue
            d = json.loads(line[-1])
            rf = d["roofline"]
            row = dict(variant=name, cfg=cfg, ms_step=round(d["ms_per_step"], 3), value=f"{d['value']:.3e}",
                       it=d["config"]["pcg_iterations_per_step"]["mean"], kernel=rf["kernel"],
                       k_us=round(rf["avg_launch_ms"] * 1e3, 2), k_GBs=round(rf["achieved"] or 0),
                       frac=round(rf["frac"] or 0, 3),
                       p1_us=round(rf["phase1"]["avg_launch_ms"] * 1e3, 2), p2_us=round(rf["phase2"]["avg_launch_ms"] * 1e3, 2),
                       inst_ms=round(rf["instrumented_ms_per_step"], 3), e2e=f"{d['e2e']['value']:.3e}")
            rows.append(row)
            print(json.dumps(row), flush=True)
    return rows


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run([int(c) for c in sys.argv[2:]] or [2])
