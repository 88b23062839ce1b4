#!/usr/bin/env python
"""Per-step solve time over a long run (warm-up trend), config 3 by default.

  python scripts/step_trend.py [n_steps] [cfg] [key=value options ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_2507_18268_b200 as P  # noqa: E402
CONFIGS = meshgen.CONFIGS

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg = sys.argv[2] if len(sys.argv) > 2 else "3"  # config number, or N<edge> for an N^3 cube
opts = dict(a.split("=") for a in sys.argv[3:])
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = P.Context(0, stream=stream)
for k, v in opts.items():
    ctx.set_option(k, int(v))
m = meshgen.block_mesh(int(cfg[1:]) if cfg.startswith("N") else CONFIGS[int(cfg)]["N"])
mesh = P.Mesh(ctx, m)
mesh.set_T(meshgen.canonical_field(m))
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ms = []
clk = []
for k in range(n):
    flush.fill_(float(k))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    p = mesh.step(1, 1.0, 0.2, tol=1e-10)
    b.record(stream)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b) / p[0]["n_iterations"] * 1e3)
    if k % 5 == 0:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        clk.append(r.stdout.strip())
print(opts, "us/iteration per step:", " ".join(f"{x:.1f}" for x in ms))
print(opts, "clocks/power/temp every 5 steps:", clk)
