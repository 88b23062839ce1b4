"""Probe: can two processes share one GPU through the library's NCCL path?
Rank r builds slab r of a 2-way decomposed 40^3 cube; compares with the
undecomposed oracle.  Launch: torchrun --nproc-per-node 2 scripts/two_rank_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch, torch.distributed as dist
import meshgen, oracle
import paper_2507_18268_b200 as P
from paper_2507_18268_b200 import decompose
rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("PROBE_DEVICE", os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
ctx = P.Context(dev)
uid = [P.Context.unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
try:
    ctx.comm_init(uid[0], ws, rank)
except Exception as e:
    print(f"rank {rank}: comm_init failed: {e}", flush=True)
    sys.exit(0)
g = meshgen.block_mesh(40)
s = meshgen.multimode_field(g)
part = decompose.slab_partition(g, ws)
m, cells = decompose.local_mesh(g, part, rank)
mesh = P.Mesh(ctx, m)
mesh.set_T(s[cells])
perfs = mesh.step(3)
T = mesh.get_T()
out = [None] * ws
dist.all_gather_object(out, (cells, T, [p["n_iterations"] for p in perfs]))
if rank == 0:
    Tg = np.zeros(g.n_cells)
    for c, t, _ in out:
        Tg[c] = t
    To, _, po = oracle.laplacian_foam(g, s, 3)
    print("its", [o[2] for o in out], [p["n_iterations"] for p in po])
    print("rel Linf vs oracle", np.max(np.abs(Tg - To)) / np.max(np.abs(To)), flush=True)
mesh.close(); ctx.close()
dist.destroy_process_group()
