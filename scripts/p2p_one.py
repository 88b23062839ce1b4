"""One cut-mesh (self-coupled processor patches) solve over the peer-memory
transport with one rank, for ncu: python scripts/p2p_one.py [N]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen
import paper_2507_18268_b200 as P
from paper_2507_18268_b200 import decompose
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
m = meshgen.block_mesh(N)
c = decompose.cut_mesh(m, decompose.z_plane_faces(m, N // 2))
ctx = P.Context(0)
ctx.p2p_init(1, 0)
mesh = P.Mesh(ctx, c)
mesh.p2p_connect([mesh.p2p_export()], 0)
mesh.set_T(meshgen.canonical_field(m))
print(mesh.step(3))
