#!/usr/bin/env python
"""Paper-protocol harness (Table 3).

The paper times 100 s of simulated time at dt = 0.2 s (500 laplacianFoam
steps), PCG + diagonal preconditioner, on Mesh-S/M/L/XL (100^3 ... 400^3
cells, Table 1), five repeats each, and reports three intervals: assembly,
solver and total execution (which includes reading the initial data).  This
script runs the same protocol on one B200 through the public API:

  Execution (s)  wall clock of mesh_create (upload + addressing build) +
                 field_set + 500 steps + field_get (+ optional field writes)
  Assembly (s)   summed CUDA-event time of the assembly kernels
  Solver (s)     summed CUDA-event time of the PCG kernels (+ sum kernels)

Workload: the hot plate (xmin 1, xmax 0, other walls zeroGradient, T0 = 0)
with DT = 1e-3 so the transient spans the whole 100 s (meshgen.PROTOCOL;
the decaying sine would underflow, reading A30).  Tolerance 1e-10 as the
bench (OpenFOAM tutorials use 1e-6; --tol to change).

  python scripts/protocol.py [--meshes S,M,L,XL] [--repeats 5] [--write-interval K] [--tol 1e-10]
Prints one JSON line per mesh and writes a Table-3-like markdown summary
(--out).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import meshgen  # noqa: E402

# Table 3, Grace-Hopper (GH200) "GPU+ALL" column: context only
# (other hardware, unstated tolerance).
PAPER_GH200 = {"S": (0.56, 1.93, 6.78), "M": (2.04, 12.53, 50.83), "L": (5.90, 48.76, 183.95),
               "XL": (13.31, 144.92, 458.93)}


def run_once(P, ctx, m, t_gen, steps, DT, dt, tol, write_interval, precond="diagonal", renumber=0):
    import torch
    torch.cuda.synchronize()
    ctx.set_instrumentation(True)
    w0 = time.perf_counter()
    mesh = P.Mesh(ctx, m, renumber=renumber)    # "read initial data": upload + build
    mesh.set_T(np.zeros(m.n_cells))
    perfs = []
    tmp = tempfile.mkdtemp(prefix="lfoam_protocol_") if write_interval else None
    host = np.zeros(m.n_cells)
    for k in range(steps):
        perfs += mesh.step(1, DT, dt, tol=tol, precond=precond)
        if write_interval and (k + 1) % write_interval == 0:
            mesh.get_T(host)
            np.save(os.path.join(tmp, f"T_{k + 1}.npy"), host)
    T = mesh.get_T()
    wall = time.perf_counter() - w0
    asm = ctx.kernel_stats("assemble")[1] / 1e3
    solver = sum(ctx.kernel_stats(k)[1] for k in ("pcg", "pcg_dic", "precond", "phase1", "phase2", "setup",
                                                   "sumpsi", "pack")) / 1e3
    ctx.set_instrumentation(False)
    mesh.close()
    if tmp:
        for f in os.listdir(tmp):
            os.remove(os.path.join(tmp, f))
        os.rmdir(tmp)
    its = [p["n_iterations"] for p in perfs]
    return dict(execution_s=wall, assembly_s=asm, solver_s=solver, meshgen_s=t_gen,
                iterations=dict(min=min(its), max=max(its), total=sum(its)),
                all_converged=all(p["converged"] for p in perfs), T=T, m=m)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--meshes", default="S,M,L,XL")
    ap.add_argument("--repeats", type=int, default=meshgen.PROTOCOL["repeats"])
    ap.add_argument("--steps", type=int, default=meshgen.PROTOCOL["steps"])
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--write-interval", type=int, default=0, help="write T to disk every K steps (0 = never)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "protocol.md"))
    ap.add_argument("--precond", default="diagonal", choices=["diagonal", "DIC"])
    ap.add_argument("--renumber", type=int, default=-1, help="default: 2 (multicolour) with DIC, else 0")
    args = ap.parse_args()

    import torch
    import paper_2507_18268_b200 as P
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream=stream)
    DT, dt = meshgen.PROTOCOL["DT"], meshgen.PROTOCOL["dt"]
    rows = []
    for name in args.meshes.split(","):
        t0 = time.perf_counter()
        mg = meshgen.protocol_mesh(name)          # host-side generator, not timed (no file I/O here)
        t_gen = time.perf_counter() - t0
        rn = args.renumber if args.renumber >= 0 else (2 if args.precond != "diagonal" else 0)
        runs = [run_once(P, ctx, mg, t_gen, args.steps, DT, dt, args.tol, args.write_interval, args.precond, rn)
                for _ in range(args.repeats)]
        T, m = runs[-1]["T"], runs[-1]["m"]
        # 1-D check of the last run: every x-line equals the same profile
        nx = m.dims[0]
        prof = T.reshape(-1, nx)
        line_spread = float(np.max(np.abs(prof - prof[0])))
        stat = lambda k: (statistics.mean(r[k] for r in runs), statistics.pstdev(r[k] for r in runs))
        row = {"mesh": f"Mesh-{name}", "N": m.dims[0], "n_cells": m.n_cells, "steps": args.steps,
               "repeats": args.repeats, "DT": DT, "dt": dt, "tol": args.tol, "precond": args.precond,
               "write_interval": args.write_interval,
               "assembly_s": stat("assembly_s"), "solver_s": stat("solver_s"),
               "execution_s": stat("execution_s"), "meshgen_s_host": stat("meshgen_s"),
               "iterations": runs[-1]["iterations"], "all_converged": all(r["all_converged"] for r in runs),
               "x_line_spread": line_spread,
               "cell_updates_per_s_execution": m.n_cells * args.steps / stat("execution_s")[0],
               "paper_gh200_gpu_all": PAPER_GH200.get(name)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del runs
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        f.write("# Paper protocol on one B200 (SURVEY §8(f) row 4)\n\n")
        f.write(f"Hot plate, DT = {DT}, dt = {dt} s, {args.steps} steps (100 s), PCG + {args.precond}, tol {args.tol}, "
                f"{args.repeats} repeats (mean ± std), field writes every {args.write_interval or 'never'}.  "
                "Assembly / Solver = summed CUDA-event kernel time; Execution = wall clock of "
                "mesh_create + field_set + steps + field_get (the paper's 'Execution' includes reading "
                "the initial data).  Paper column: Table 3 GH200 GPU+ALL (other hardware, unstated "
                "tolerance) — context only.\n\n")
        f.write("| mesh | cells | Assembly (s) | Solver (s) | Execution (s) | PCG its/step | paper GH200 A / S / E (s) |\n")
        f.write("|---|---|---|---|---|---|---|\n")
        for r in rows:
            a, s_, e = r["assembly_s"], r["solver_s"], r["execution_s"]
            its = r["iterations"]
            pap = r["paper_gh200_gpu_all"]
            f.write(f"| {r['mesh']} | {r['n_cells']:,} | {a[0]:.3f} ± {a[1]:.3f} | {s_[0]:.2f} ± {s_[1]:.2f} | "
                    f"{e[0]:.2f} ± {e[1]:.2f} | {its['min']}-{its['max']} (total {its['total']}) | "
                    f"{' / '.join(str(x) for x in pap) if pap else '-'} |\n")
    ctx.close()


if __name__ == "__main__":
    main()
