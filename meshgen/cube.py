"""blockMesh-style hex meshes in OpenFOAM LDU face addressing (input generator).

Citations (PAPER.md = P, SPEC.md = S):
  * owner/neighbour face addressing, boundary faces have an owner only:
    P:158-174 (§4.1, "Owner and neighbour lists").
  * Table 1 meshes Mesh-S/M/L/XL = 100^3..400^3: P:563-580 (§6).
  * counting formulas internal = 3N^2(N-1), total = 3N^2(N+1),
    points = (N+1)^3: S:50.
  * permuted variant (cells pi_c seed 1, faces pi_f seed 2,
    owner = min, neighbour = max): SURVEY.md §8(c.2) reading A24.

Geometry is written in closed form (uniform box cells): |Sf| = face area,
internal deltaCoeffs = 1/h (distance between the two cell centres), boundary
deltaCoeffs = 2/h (1/|n.(Cf - C_P)|, reading A5), V = hx*hy*hz.  The oracle
recomputes these from ``mesh_points_faces`` as an independent self-check.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

PATCH_NAMES = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")
PATCH_TYPES = ("fixedValue", "zeroGradient", "processor")


@dataclasses.dataclass
class Patch:
    name: str
    type: str                      # "fixedValue" | "zeroGradient" | "processor"
    face_cells: np.ndarray         # int32 [nf]
    mag_sf: np.ndarray             # f64 [nf]
    delta: np.ndarray              # f64 [nf]  deltaCoeffs
    value: np.ndarray              # f64 [nf]  fixedValue T_b (ignored otherwise)
    neighb_rank: int = -1          # processor patches only
    global_faces: Optional[np.ndarray] = None  # processor: global face ids (ordering key)

    @property
    def n_faces(self) -> int:
        return int(self.face_cells.shape[0])


@dataclasses.dataclass
class Mesh:
    n_cells: int
    owner: np.ndarray              # int32 [F]
    neighbour: np.ndarray          # int32 [F]
    mag_sf: np.ndarray             # f64 [F]
    delta: np.ndarray              # f64 [F]
    V: np.ndarray                  # f64 [n]
    patches: List[Patch]
    dims: tuple = (0, 0, 0)        # (nx, ny, nz) of the generating block
    extent: tuple = (1.0, 1.0, 1.0)
    old_of_new: Optional[np.ndarray] = None   # permuted meshes: block label of each cell
    face_old_of_new: Optional[np.ndarray] = None
    cell_global: Optional[np.ndarray] = None  # decomposed meshes: global (block) label per local cell

    @property
    def n_faces(self) -> int:
        return int(self.owner.shape[0])

    @property
    def n_boundary_faces(self) -> int:
        return sum(p.n_faces for p in self.patches)

    def block_labels(self) -> np.ndarray:
        """Label of each cell in the generating block (c = i + nx*j + nx*ny*k)."""
        lab = np.arange(self.n_cells, dtype=np.int64)
        if self.old_of_new is not None:
            lab = self.old_of_new.astype(np.int64)
        if self.cell_global is not None:
            lab = self.cell_global.astype(np.int64)
        return lab

    def cell_centres(self) -> np.ndarray:
        nx, ny, nz = self.dims
        hx, hy, hz = (self.extent[0] / nx, self.extent[1] / ny, self.extent[2] / nz)
        lab = self.block_labels()
        i = lab % nx
        j = (lab // nx) % ny
        k = lab // (nx * ny)
        return np.stack([(i + 0.5) * hx, (j + 0.5) * hy, (k + 0.5) * hz], axis=1)


def cube_counts(N: int) -> Dict[str, int]:
    """S:50/S:68 counting formulas for an N^3 block."""
    return {"cells": N ** 3, "internal": 3 * N * N * (N - 1),
            "total": 3 * N * N * (N + 1), "points": (N + 1) ** 3,
            "boundary": 6 * N * N}


def block_mesh(nx: int, ny: Optional[int] = None, nz: Optional[int] = None,
               extent: Sequence[float] = (1.0, 1.0, 1.0),
               bc: Optional[Dict[str, object]] = None) -> Mesh:
    """Structured hex block, faces internal-first in upper-triangular order.

    ``bc`` maps patch name -> ("fixedValue", T_b) | "zeroGradient".  Default:
    fixedValue 0 on all six walls (reading A6).
    """
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    if min(nx, ny, nz) < 1:
        raise ValueError("block dimensions must be >= 1")
    n = nx * ny * nz
    if n >= 2 ** 31 - 1:
        raise ValueError("int32 labels")
    Lx, Ly, Lz = (float(e) for e in extent)
    hx, hy, hz = Lx / nx, Ly / ny, Lz / nz
    area = np.array([hy * hz, hx * hz, hx * hy])
    dint = np.array([1.0 / hx, 1.0 / hy, 1.0 / hz])
    dbnd = np.array([2.0 / hx, 2.0 / hy, 2.0 / hz])

    c = np.arange(n, dtype=np.int32)
    i = c % nx
    j = (c // nx) % ny
    k = c // (nx * ny)
    # owner ascending, then neighbour ascending: c+1 < c+nx < c+nx*ny
    nb = np.stack([c + 1, c + nx, c + nx * ny], axis=1)
    mask = np.stack([i < nx - 1, j < ny - 1, k < nz - 1], axis=1)
    dirs = np.broadcast_to(np.arange(3, dtype=np.int8), (n, 3))
    mflat = mask.ravel()
    owner = np.repeat(c, 3)[mflat]
    neighbour = nb.ravel()[mflat]
    d = dirs.ravel()[mflat]
    del nb, mask, dirs, mflat
    mag_sf = area[d]
    delta = dint[d]
    del d
    V = np.full(n, hx * hy * hz)

    bc = dict(bc or {})
    patches = []
    sel = [i == 0, i == nx - 1, j == 0, j == ny - 1, k == 0, k == nz - 1]
    for p, name in enumerate(PATCH_NAMES):
        fc = np.nonzero(sel[p])[0].astype(np.int32)
        spec = bc.get(name, ("fixedValue", 0.0))
        if isinstance(spec, str):
            ptype, val = spec, 0.0
        else:
            ptype, val = spec[0], float(spec[1])
        if ptype not in ("fixedValue", "zeroGradient"):
            raise ValueError(f"unknown bc {ptype}")
        ax = p // 2
        patches.append(Patch(name, ptype, fc, np.full(fc.shape[0], area[ax]),
                             np.full(fc.shape[0], dbnd[ax]),
                             np.full(fc.shape[0], val if ptype == "fixedValue" else 0.0)))
    return Mesh(n, owner, neighbour, mag_sf, delta, V, patches,
                dims=(nx, ny, nz), extent=(Lx, Ly, Lz))


def permute_mesh(mesh: Mesh, cell_seed: int = 1, face_seed: int = 2) -> Mesh:
    """Reading A24: random cell labels pi_c, random face order pi_f,
    owner = min(pi_c(P), pi_c(N)), neighbour = max."""
    n, F = mesh.n_cells, mesh.n_faces
    new_of_old = np.random.Generator(np.random.PCG64(cell_seed)).permutation(n).astype(np.int32)
    fperm = np.random.Generator(np.random.PCG64(face_seed)).permutation(F).astype(np.int64)
    a = new_of_old[mesh.owner[fperm]]
    b = new_of_old[mesh.neighbour[fperm]]
    owner = np.minimum(a, b).astype(np.int32)
    neighbour = np.maximum(a, b).astype(np.int32)
    V = np.empty_like(mesh.V)
    V[new_of_old] = mesh.V
    old_of_new = np.empty(n, dtype=np.int32)
    old_of_new[new_of_old] = np.arange(n, dtype=np.int32)
    base = mesh.block_labels()
    patches = [dataclasses.replace(p, face_cells=new_of_old[p.face_cells].astype(np.int32))
               for p in mesh.patches]
    return Mesh(n, owner, neighbour, mesh.mag_sf[fperm], mesh.delta[fperm], V, patches,
                dims=mesh.dims, extent=mesh.extent,
                old_of_new=base[old_of_new].astype(np.int32), face_old_of_new=fperm)


# ----------------------------------------------------------------- fields
def sine_field(mesh: Mesh, k=(1, 1, 1), amp: float = 1.0) -> np.ndarray:
    """T0 = amp * prod_d sin(k_d pi x_d / L_d) at cell centres (reading A6)."""
    C = mesh.cell_centres()
    out = np.full(mesh.n_cells, amp)
    for d in range(3):
        out = out * np.sin(k[d] * np.pi * C[:, d] / mesh.extent[d])
    return out


# Reading A30: the decaying sine case loses a factor g ~ 1/6.9
# per step (g^100 ~ 1e-84 at dt = 0.2).  OpenFOAM's normFactor carries an
# absolute floor (solverPerformance::small_ = 1e-20); once the field falls
# to ~1e-20 the solver "converges" with ~0 iterations and the run degenerates
# into empty steps.  The problem is linear and homogeneous (T_b = 0), so the
# canonical bench/full-run field is the same mode scaled by 1e80: the decay is
# identical (T^n = g^n T0) and the field ends at ~1e-4 after 100 steps, far
# above the floor; squares stay < 1e170.
CANONICAL_AMPLITUDE = 1e80


def canonical_field(mesh: Mesh) -> np.ndarray:
    return sine_field(mesh, amp=CANONICAL_AMPLITUDE)


def cosine_field(mesh: Mesh, k=(1, 2, 0), amp: float = 1.0, offset: float = 0.0) -> np.ndarray:
    """offset + amp * prod_d cos(k_d pi x_d / L_d): the zeroGradient eigenmode."""
    C = mesh.cell_centres()
    out = np.full(mesh.n_cells, amp)
    for d in range(3):
        out = out * np.cos(k[d] * np.pi * C[:, d] / mesh.extent[d])
    return offset + out


MULTIMODE = (((1, 1, 1), 1.0), ((2, 3, 1), 0.5), ((5, 2, 7), 0.25), ((11, 13, 3), 0.125))


def multimode_field(mesh: Mesh, modes=MULTIMODE) -> np.ndarray:
    """SURVEY §8(d) richer-spectrum option: superposition of sine modes."""
    out = np.zeros(mesh.n_cells)
    for k, a in modes:
        out += sine_field(mesh, k, a)
    return out


def random_field(mesh: Mesh, seed: int = 0, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return np.random.Generator(np.random.PCG64(seed)).uniform(lo, hi, mesh.n_cells)


def hot_plate(N: int) -> Mesh:
    """S:469 hot plate: xmin fixedValue 1, xmax fixedValue 0, others zeroGradient."""
    bc = {"xmin": ("fixedValue", 1.0), "xmax": ("fixedValue", 0.0),
          "ymin": "zeroGradient", "ymax": "zeroGradient",
          "zmin": "zeroGradient", "zmax": "zeroGradient"}
    return block_mesh(N, bc=bc)


# ----------------------------------------------------------- points/faces
def mesh_points_faces(mesh: Mesh):
    """Vertices and quad faces (internal in LDU order, then patches) of an
    unpermuted block, for the oracle's geometry self-check (small meshes only).
    Quads are ordered so the right-hand normal points owner -> neighbour
    (outward on boundaries)."""
    if mesh.old_of_new is not None or mesh.cell_global is not None:
        raise ValueError("points/faces only for unpermuted blocks")
    nx, ny, nz = mesh.dims
    hx, hy, hz = (mesh.extent[0] / nx, mesh.extent[1] / ny, mesh.extent[2] / nz)
    I, J, K = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    pts = np.zeros(((nx + 1) * (ny + 1) * (nz + 1), 3))
    pid = lambda i, j, k: i + (nx + 1) * (j + (ny + 1) * k)
    pts[pid(I, J, K).ravel()] = np.stack([I.ravel() * hx, J.ravel() * hy, K.ravel() * hz], axis=1)

    def quad(ax, i, j, k, outward_positive):
        # face of cell (i,j,k) on its +ax side
        if ax == 0:
            q = [pid(i + 1, j, k), pid(i + 1, j + 1, k), pid(i + 1, j + 1, k + 1), pid(i + 1, j, k + 1)]
        elif ax == 1:
            q = [pid(i, j + 1, k), pid(i, j + 1, k + 1), pid(i + 1, j + 1, k + 1), pid(i + 1, j + 1, k)]
        else:
            q = [pid(i, j, k + 1), pid(i + 1, j, k + 1), pid(i + 1, j + 1, k + 1), pid(i, j + 1, k + 1)]
        return q if outward_positive else q[::-1]

    faces = []
    for f in range(mesh.n_faces):
        o, nb = int(mesh.owner[f]), int(mesh.neighbour[f])
        i, j, k = o % nx, (o // nx) % ny, o // (nx * ny)
        ax = 0 if nb == o + 1 and nx > 1 else (1 if nb == o + nx and ny > 1 else 2)
        faces.append(quad(ax, i, j, k, True))
    for p, patch in enumerate(mesh.patches):
        ax, hi = p // 2, p % 2
        for c in patch.face_cells:
            c = int(c)
            i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
            if hi:
                faces.append(quad(ax, i, j, k, True))
            else:
                ii, jj, kk = (i - 1, j, k) if ax == 0 else ((i, j - 1, k) if ax == 1 else (i, j, k - 1))
                faces.append(quad(ax, ii, jj, kk, False))
    return pts, np.array(faces, dtype=np.int64)


# ---------------------------------------------------------------- configs
CONFIGS = {
    1: dict(N=10, steps=10, permuted=False),
    2: dict(N=100, steps=100, permuted=False),
    3: dict(N=200, steps=100, permuted=False),
    4: dict(N=400, steps=50, permuted=False),
    5: dict(N=200, steps=100, permuted=True),
}


def config_mesh(cfg: int) -> Mesh:
    c = CONFIGS[cfg]
    m = block_mesh(c["N"])
    return permute_mesh(m) if c["permuted"] else m
