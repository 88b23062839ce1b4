#!/usr/bin/env python
"""Cost of the multi-rank machinery measured on ONE GPU (no second GPU in
this sandbox): the config mesh cut at its mid z-plane into a pair of
self-coupled processor patches (reading A32), solved through
  * no processor patches (the single-rank persistent solve),
  * the peer-memory transport with one rank (halo puts + system fences of
    the pushing blocks + the mailbox allreduce inside the persistent kernel),
  * NCCL with one rank, per-phase launches in CUDA graphs, the w halo
    overlapped with the interior Amul (LF_OPT_OVERLAP_HALO) or serial.
The difference to the uncut solve is the overhead a real decomposed run pays
per rank on top of its share of the work.  CUDA events on the library
stream, inputs resident, 2 warm-up steps.

  python scripts/p2p_overhead.py [N] [steps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_2507_18268_b200 as P  # noqa: E402
from paper_2507_18268_b200 import decompose  # noqa: E402


def run(mesh_in, setup, steps):
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream=stream)
    setup(ctx)
    mesh = P.Mesh(ctx, mesh_in)
    if getattr(ctx, "_p2p", False):
        mesh.p2p_connect([mesh.p2p_export()], 0)
    T0 = meshgen.canonical_field(mesh_in)
    mesh.set_T(T0)
    mesh.step(2)
    mesh.set_T(T0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    perfs = mesh.step(steps)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    its = sum(p["n_iterations"] for p in perfs) / len(perfs)
    mesh.close()
    ctx.close()
    return ms, its


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    m = meshgen.block_mesh(N)
    c = decompose.cut_mesh(m, decompose.z_plane_faces(m, N // 2))

    def p2p(ctx):
        ctx.p2p_init(1, 0)

    def nccl(overlap):
        def f(ctx):
            ctx.comm_init(P.Context.unique_id(), 1, 0)
            ctx.set_option("overlap_halo", overlap)
        return f

    rows = {}
    rows["uncut"] = run(m, lambda ctx: None, steps)
    rows["cut-p2p"] = run(c, p2p, steps)
    rows["cut-nccl-overlap"] = run(c, nccl(True), steps)
    rows["cut-nccl-serial"] = run(c, nccl(False), steps)
    base = rows["uncut"][0]
    out = {k: {"ms_per_step": round(v[0], 3), "its_per_step": v[1], "overhead_vs_uncut": round(v[0] / base - 1, 4)}
           for k, v in rows.items()}
    print(json.dumps({"N": N, "steps": steps, "halo_faces": N * N, "rows": out}), flush=True)


if __name__ == "__main__":
    main()
