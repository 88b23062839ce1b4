"""Oracle geometry self-check — TEST INFRASTRUCTURE ONLY.

Recomputes, from points and face vertex lists alone, the geometric inputs
the generator writes in closed form:
  * face area vector Sf (triangle fan about the vertex average, oriented by
    the vertex order: owner -> neighbour, outward on boundaries),
    face centre Cf (area-weighted triangle centroids);
  * cell volume V = (1/3) sum_f Cf . Sf_out (divergence theorem) and cell
    centre by pyramid decomposition;
  * internal deltaCoeffs 1/|C_N - C_P|; boundary 1/|n.(Cf - C_P)| (A5).
"""
from __future__ import annotations

import numpy as np


def face_geometry(points: np.ndarray, faces: np.ndarray):
    P = points[faces]                                   # [F, k, 3]
    est = P.mean(axis=1)                                # [F, 3]
    k = P.shape[1]
    Sf = np.zeros_like(est)
    Cf = np.zeros_like(est)
    atot = np.zeros(est.shape[0])
    for i in range(k):
        a, b = P[:, i], P[:, (i + 1) % k]
        s = 0.5 * np.cross(b - a, est - a)   # = 0.5 (a-est) x (b-est)
        c = (a + b + est) / 3.0
        mag = np.linalg.norm(s, axis=1)
        Sf += s
        Cf += c * mag[:, None]
        atot += mag
    Cf /= atot[:, None]
    return Sf, Cf


def cell_geometry(points, faces, owner_all, neighbour, n_cells):
    """owner_all: owner of every face (internal then boundary);
    neighbour: internal faces only."""
    Sf, Cf = face_geometry(points, faces)
    F = neighbour.shape[0]
    # estimated centre: average of face centres
    cnt = np.zeros(n_cells)
    est = np.zeros((n_cells, 3))
    np.add.at(est, owner_all, Cf)
    np.add.at(cnt, owner_all, 1.0)
    np.add.at(est, neighbour, Cf[:F])
    np.add.at(cnt, neighbour, 1.0)
    est /= cnt[:, None]
    V = np.zeros(n_cells)
    C = np.zeros((n_cells, 3))

    def add(cells, sf_out, cf):
        pyr = np.einsum("ij,ij->i", sf_out, cf - est[cells]) / 3.0
        np.add.at(V, cells, pyr)
        np.add.at(C, cells, pyr[:, None] * (0.75 * cf + 0.25 * est[cells]))

    add(owner_all, Sf, Cf)
    add(neighbour, -Sf[:F], Cf[:F])
    C /= V[:, None]
    return Sf, Cf, V, C


def mesh_geometry(mesh, points, faces):
    """Returns dict(mag_sf, delta, V, b_mag_sf, b_delta, closure) in mesh order."""
    F = mesh.n_faces
    b_cells = np.concatenate([p.face_cells for p in mesh.patches]).astype(np.int64)
    owner_all = np.concatenate([mesh.owner.astype(np.int64), b_cells])
    nb = mesh.neighbour.astype(np.int64)
    Sf, Cf, V, C = cell_geometry(points, faces, owner_all, nb, mesh.n_cells)
    magSf = np.linalg.norm(Sf, axis=1)
    d = C[nb] - C[mesh.owner]
    delta = 1.0 / np.linalg.norm(d, axis=1)
    n_b = Sf[F:] / magSf[F:, None]
    b_delta = 1.0 / np.abs(np.einsum("ij,ij->i", n_b, Cf[F:] - C[b_cells]))
    closure = np.zeros((mesh.n_cells, 3))
    np.add.at(closure, owner_all, Sf)
    np.add.at(closure, nb, -Sf[:F])
    return dict(mag_sf=magSf[:F], delta=delta, V=V, b_mag_sf=magSf[F:], b_delta=b_delta,
                closure=closure, Sf=Sf, Cf=Cf, C=C)
