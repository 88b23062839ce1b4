"""Diagnostic: per-step PCG iteration counts and residuals, GPU vs oracle."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import meshgen, oracle
import paper_2507_18268_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
m = meshgen.block_mesh(N)
s = meshgen.canonical_field(m)
To, _, po = oracle.laplacian_foam(m, s, steps)
ctx = P.Context(0)
mesh = P.Mesh(ctx, m)
mesh.set_T(s)
pg = mesh.step(steps)
T = mesh.get_T()
print("rel Linf", np.max(np.abs(T - To)) / np.max(np.abs(To)))
for i, (a, b) in enumerate(zip(pg, po)):
    if a["n_iterations"] != b["n_iterations"]:
        print(i, a["n_iterations"], b["n_iterations"], "%.4e %.4e" % (a["final_residual"], b["final_residual"]),
              "init %.4e %.4e" % (a["initial_residual"], b["initial_residual"]))
print("gpu", [p["n_iterations"] for p in pg])
print("orc", [p["n_iterations"] for p in po])
mesh.close(); ctx.close()
