"""Host-side domain decomposition for the multi-GPU path.

The paper runs "1 MPI process for each GPU" (§6.2) on OpenFOAM's
decomposed meshes; here each rank builds its own subdomain from the global
LDU mesh (reading A26: contiguous cell blocks in library numbering — z-slabs
on the blockMesh cube).  Faces between ranks become processor patches
(fvPatch "processor"), ordered by ascending global face id on both sides so
that the i-th face of rank r's patch towards s is the i-th face of s's patch
towards r (the halo exchange relies on it).  No arithmetic of the method is
done here: only index bookkeeping.

`cut_mesh` builds the single-rank loopback variant (reading A32): chosen
internal faces are replaced by a pair of self-coupled processor patches; the
system solved is unchanged, which tests every processor-patch code path and
the NCCL send/recv path on one GPU.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

import numpy as np


def slab_partition(mesh, nranks: int) -> np.ndarray:
    """Rank of every cell: contiguous blocks [r*n/P, (r+1)*n/P)."""
    n = mesh.n_cells
    bounds = (np.arange(nranks + 1, dtype=np.int64) * n) // nranks
    part = np.empty(n, dtype=np.int32)
    for r in range(nranks):
        part[bounds[r]:bounds[r + 1]] = r
    return part


def _patch_cls(mesh):
    return type(mesh.patches[0]) if mesh.patches else None


def local_mesh(mesh, part: np.ndarray, rank: int):
    """Subdomain of `rank`: (local mesh, global ids of its cells).

    Local cell order = ascending global id; internal faces keep the global
    (upper-triangular) order; processor patches follow the global patches,
    one per neighbour rank in ascending rank order."""
    import meshgen  # input container type only (dataclasses Mesh/Patch)
    cells = np.nonzero(part == rank)[0].astype(np.int64)
    loc = np.full(mesh.n_cells, -1, dtype=np.int64)
    loc[cells] = np.arange(cells.shape[0])
    po, pn = part[mesh.owner], part[mesh.neighbour]
    inner = (po == rank) & (pn == rank)
    owner = loc[mesh.owner[inner]].astype(np.int32)
    neighbour = loc[mesh.neighbour[inner]].astype(np.int32)
    geo = mesh.Sf is not None
    patches = []
    for p in mesh.patches:
        sel = part[p.face_cells] == rank
        extra = {}
        if geo and p.Sf is not None:
            extra = dict(Sf=p.Sf[sel], Cf=None if p.Cf is None else p.Cf[sel])
        patches.append(dataclasses.replace(
            p, face_cells=loc[p.face_cells[sel]].astype(np.int32), mag_sf=p.mag_sf[sel],
            delta=p.delta[sel], value=p.value[sel], **extra))
    cut = (po == rank) ^ (pn == rank)
    fidx = np.nonzero(cut)[0]
    mine_is_owner = po[fidx] == rank
    other = np.where(mine_is_owner, pn[fidx], po[fidx])
    mine = np.where(mine_is_owner, mesh.owner[fidx], mesh.neighbour[fidx])
    theirs = np.where(mine_is_owner, mesh.neighbour[fidx], mesh.owner[fidx])
    for s in np.unique(other):
        sel = other == s
        f = fidx[sel]                                   # ascending global face id
        extra = {}
        if geo:
            # outward from this rank's cell; the coupled cell's centre (Cn)
            sgn = np.where(mine_is_owner[sel], 1.0, -1.0)[:, None]
            extra = dict(Sf=mesh.Sf[f] * sgn, Cf=mesh.Cf[f].copy(), Cn=mesh.C[theirs[sel]].copy())
        patches.append(meshgen.Patch(f"procBoundary{rank}to{int(s)}", "processor",
                                     loc[mine[sel]].astype(np.int32), mesh.mag_sf[f], mesh.delta[f],
                                     np.zeros(f.shape[0]), neighb_rank=int(s), global_faces=f, **extra))
    gkw = {}
    if geo:
        gkw = dict(Sf=mesh.Sf[inner], Cf=mesh.Cf[inner], C=mesh.C[cells], affine=mesh.affine,
                   grid_lines=mesh.grid_lines)
    if mesh.DT_field is not None:
        gkw["DT_field"] = mesh.DT_field[cells]
    sub = meshgen.Mesh(int(cells.shape[0]), owner, neighbour, mesh.mag_sf[inner], mesh.delta[inner],
                       mesh.V[cells], patches, dims=mesh.dims, extent=mesh.extent,
                       cell_global=mesh.block_labels()[cells].astype(np.int64), **gkw)
    return sub, cells


def cut_mesh(mesh, face_mask: np.ndarray, rank: int = 0):
    """Single-rank loopback: internal faces in `face_mask` become the pair of
    self-coupled processor patches (owner side, then neighbour side)."""
    import meshgen
    keep = ~face_mask
    f = np.nonzero(face_mask)[0]
    patches = list(mesh.patches)
    ga, gb, gkw = {}, {}, {}
    if mesh.Sf is not None:  # geometry of the coupled faces (outward Sf, Cf, coupled cell centre)
        ga = dict(Sf=mesh.Sf[f].copy(), Cf=mesh.Cf[f].copy(), Cn=mesh.C[mesh.neighbour[f]].copy())
        gb = dict(Sf=-mesh.Sf[f], Cf=mesh.Cf[f].copy(), Cn=mesh.C[mesh.owner[f]].copy())
        gkw = dict(Sf=mesh.Sf[keep], Cf=mesh.Cf[keep])
    patches.append(meshgen.Patch("procSelfA", "processor", mesh.owner[f].astype(np.int32), mesh.mag_sf[f],
                                 mesh.delta[f], np.zeros(f.shape[0]), neighb_rank=rank, global_faces=f, **ga))
    patches.append(meshgen.Patch("procSelfB", "processor", mesh.neighbour[f].astype(np.int32), mesh.mag_sf[f],
                                 mesh.delta[f], np.zeros(f.shape[0]), neighb_rank=rank, global_faces=f, **gb))
    return dataclasses.replace(mesh, owner=mesh.owner[keep], neighbour=mesh.neighbour[keep],
                               mag_sf=mesh.mag_sf[keep], delta=mesh.delta[keep], patches=patches, **gkw)


def z_plane_faces(mesh, k: int) -> np.ndarray:
    """Mask of the internal faces between z-layers k-1 and k of a block mesh."""
    nx, ny, _ = mesh.dims
    layer = nx * ny
    return (mesh.owner // layer == k - 1) & (mesh.neighbour // layer == k)


def check_pairing(local_meshes: List) -> List[Tuple[int, int, int]]:
    """Host check that processor patches pair up face by face across ranks:
    returns (r, s, n_faces) for every matched pair; raises on mismatch."""
    out = []
    by = {}
    for r, m in enumerate(local_meshes):
        for p in m.patches:
            if p.type == "processor":
                by[(r, p.neighb_rank)] = p
    for (r, s), p in by.items():
        q = by.get((s, r))
        if q is None or not np.array_equal(p.global_faces, q.global_faces):
            raise ValueError(f"processor patches {r}->{s} do not match")
        if r < s:
            out.append((r, s, p.n_faces))
    return out
