"""CPU oracle for the laplacianFoam hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and the ``--impl reference`` arm) may import this
package.  The product (``paper_2507_18268_b200``) never imports it and
shares no code with it; ``oracle/lfoam_oracle.c`` is compiled on its own
(gcc -O2 -ffp-contract=off) into ``oracle/liboracle.so``.

Functions follow SURVEY.md §8(c.1) / PAPER.md Listing 1, §5.2
 and §6; see the C file header for per-function
citations.  ``geometry`` recomputes mesh geometry from points/faces.
Parity pins: tests/test_oracle_*.py.  Unpinned beyond oracle agreement
("parity unpinned"): PCG iteration counts and residual values after step 0
(no closed form exists).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Callable, List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lfoam_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_TYPES = {"fixedValue": 0, "zeroGradient": 1, "processor": 2}
# preconditioners (OpenFOAM fvSolution names): diagonal (the paper's),
# DIC and GAMG
PRECONDITIONERS = {"diagonal": 0, "DIC": 1, "GAMG": 3}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Mesh(C.Structure):
    _fields_ = [("n_cells", C.c_int32), ("n_faces", C.c_int32), ("n_patches", C.c_int32),
                ("n_bfaces", C.c_int32), ("owner", C.c_void_p), ("neighbour", C.c_void_p),
                ("mag_sf", C.c_void_p), ("delta", C.c_void_p), ("V", C.c_void_p),
                ("patch_type", C.c_void_p), ("patch_start", C.c_void_p), ("b_cells", C.c_void_p),
                ("b_mag_sf", C.c_void_p), ("b_delta", C.c_void_p),
                ("Sf", C.c_void_p), ("Cf", C.c_void_p), ("C", C.c_void_p), ("b_Sf", C.c_void_p),
                ("gamma", C.c_void_p), ("b_gamma", C.c_void_p)]


class Perf(C.Structure):
    _fields_ = [("initial_residual", C.c_double), ("final_residual", C.c_double),
                ("n_iterations", C.c_int32), ("converged", C.c_int32),
                ("singular", C.c_int32), ("pad", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k in ("initial_residual", "final_residual",
                                              "n_iterations", "converged", "singular")}


GSUM = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.c_int32)
HALO = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double))

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        vp = C.c_void_p
        _lib.orc_group.argtypes = [vp, C.c_int64, C.c_int32, vp, vp]
        _lib.orc_assemble.argtypes = [C.POINTER(_Mesh), C.c_double, C.c_double, vp, vp, vp, vp, vp, vp, vp]
        _lib.orc_amul.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp, vp, vp]
        _lib.orc_sumA.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp]
        _lib.orc_pcg.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp, vp, C.c_double, C.c_double,
                                 C.c_int32, C.c_int32, GSUM, HALO, vp, C.POINTER(Perf)]
        _lib.orc_laplacian_foam.argtypes = [C.POINTER(_Mesh), C.c_double, C.c_double, vp, vp,
                                            C.c_int32, C.c_double, C.c_double, C.c_int32,
                                            C.c_int32, GSUM, HALO, vp, C.POINTER(Perf)]
        _lib.orc_pcg_p.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp, vp, C.c_double, C.c_double,
                                   C.c_int32, C.c_int32, C.c_int32, GSUM, HALO, vp, C.POINTER(Perf)]
        _lib.orc_laplacian_foam_p.argtypes = [C.POINTER(_Mesh), C.c_double, C.c_double, vp, vp,
                                              C.c_int32, C.c_double, C.c_double, C.c_int32,
                                              C.c_int32, C.c_int32, GSUM, HALO, vp, C.POINTER(Perf)]
        _lib.orc_dic.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp, vp]
        _lib.orc_gamg.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp, vp, vp, vp]
        _lib.orc_gamg_level.argtypes = [C.POINTER(_Mesh), vp, vp, C.c_int32, vp, vp, vp, vp]
        _lib.orc_patch_values.argtypes = [C.POINTER(_Mesh), vp, vp]
        _lib.orc_weights.argtypes = [C.POINTER(_Mesh), vp]
        _lib.orc_corr_vectors.argtypes = [C.POINTER(_Mesh), vp]
        _lib.orc_grad.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp]
        _lib.orc_grad_bc.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp]
        _lib.orc_lap_correction.argtypes = [C.POINTER(_Mesh), C.c_double, vp, vp, vp, vp]
        _lib.orc_face_gamma.argtypes = [C.POINTER(_Mesh), vp, vp, vp, vp]
        _lib.orc_laplacian_foam_corrected.argtypes = [C.POINTER(_Mesh), C.c_double, C.c_double, vp, vp,
                                                      C.c_int32, C.c_int32, C.c_double, C.c_double,
                                                      C.c_int32, C.c_int32, C.POINTER(Perf)]
        _lib.orc_laplacian_foam_corrected_p.argtypes = [C.POINTER(_Mesh), C.c_double, C.c_double, vp, vp,
                                                        C.c_int32, C.c_int32, C.c_double, C.c_double,
                                                        C.c_int32, C.c_int32, C.c_int32, C.POINTER(Perf)]
    return _lib


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


class OMesh:
    """Flattened view of a meshgen.Mesh (keeps the numpy buffers alive)."""

    def __init__(self, mesh):
        self.src = mesh
        self.owner = np.ascontiguousarray(mesh.owner, dtype=np.int32)
        self.neighbour = np.ascontiguousarray(mesh.neighbour, dtype=np.int32)
        self.mag_sf = np.ascontiguousarray(mesh.mag_sf, dtype=np.float64)
        self.delta = np.ascontiguousarray(mesh.delta, dtype=np.float64)
        self.V = np.ascontiguousarray(mesh.V, dtype=np.float64)
        self.patch_type = np.array([_TYPES[p.type] for p in mesh.patches], dtype=np.int32)
        sizes = [p.n_faces for p in mesh.patches]
        self.patch_start = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        cat = lambda name, dt: (np.concatenate([getattr(p, name) for p in mesh.patches]).astype(dt)
                                if mesh.patches else np.zeros(0, dt))
        self.b_cells = cat("face_cells", np.int32)
        self.b_mag_sf = cat("mag_sf", np.float64)
        self.b_delta = cat("delta", np.float64)
        self.b_value = cat("value", np.float64)
        self.n_cells, self.n_faces = int(mesh.n_cells), int(self.owner.shape[0])
        self.n_bfaces = int(self.b_cells.shape[0])
        g = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        self.Sf, self.Cf = g(getattr(mesh, "Sf", None)), g(getattr(mesh, "Cf", None))
        self.C = g(getattr(mesh, "C", None))
        if all(getattr(p, "Sf", None) is not None for p in mesh.patches):
            self.b_Sf = (np.ascontiguousarray(np.concatenate([p.Sf for p in mesh.patches]), dtype=np.float64)
                         if mesh.patches else np.zeros((0, 3)))
        else:
            self.b_Sf = None
        self.s = _Mesh(self.n_cells, self.n_faces, len(sizes), self.n_bfaces,
                       _p(self.owner), _p(self.neighbour), _p(self.mag_sf), _p(self.delta),
                       _p(self.V), _p(self.patch_type), _p(self.patch_start), _p(self.b_cells),
                       _p(self.b_mag_sf), _p(self.b_delta), _p(self.Sf), _p(self.Cf), _p(self.C),
                       _p(self.b_Sf), None, None)
        # spatially varying DT (mesh.DT_field): face
        # diffusivities by linear interpolation with the geometric weights
        self.DT_field = getattr(mesh, "DT_field", None)
        self.gamma = self.b_gamma = None
        if self.DT_field is not None:
            if not self.has_geometry:
                raise ValueError("a DT field needs the full geometry (interpolation weights)")
            self.DT_field = np.ascontiguousarray(self.DT_field, dtype=np.float64)
            w = np.zeros(self.n_faces)
            lib().orc_weights(C.byref(self.s), _p(w))
            self.gamma, self.b_gamma = np.zeros(self.n_faces), np.zeros(self.n_bfaces)
            lib().orc_face_gamma(C.byref(self.s), _p(w), _p(self.DT_field), _p(self.gamma), _p(self.b_gamma))
            self.s.gamma, self.s.b_gamma = _p(self.gamma), _p(self.b_gamma)

    @property
    def has_geometry(self):
        return self.Sf is not None and self.Cf is not None and self.C is not None and self.b_Sf is not None

    def patch_slices(self):
        return [slice(int(self.patch_start[i]), int(self.patch_start[i + 1]))
                for i in range(len(self.patch_start) - 1)]


def _om(mesh):
    return mesh if isinstance(mesh, OMesh) else OMesh(mesh)


def group(keys: np.ndarray, n_groups: int):
    """Stable cell->face grouping (items, starts[n_groups+1])."""
    keys = np.ascontiguousarray(keys, dtype=np.int32)
    items = np.zeros(keys.shape[0], np.int32)
    starts = np.zeros(n_groups + 1, np.int32)
    rc = lib().orc_group(_p(keys), keys.shape[0], n_groups, _p(items), starts.ctypes.data)
    if rc:
        raise ValueError("key out of range")
    return items, starts


def assemble(mesh, DT: float, dt: float, T0: np.ndarray, b_value: Optional[np.ndarray] = None):
    """Returns dict(diag, upper, source, internal_coeffs, boundary_coeffs)."""
    om = _om(mesh)
    T0 = np.ascontiguousarray(T0, dtype=np.float64)
    bv = om.b_value if b_value is None else np.ascontiguousarray(b_value, np.float64)
    out = dict(diag=np.zeros(om.n_cells), upper=np.zeros(om.n_faces), source=np.zeros(om.n_cells),
               internal_coeffs=np.zeros(om.n_bfaces), boundary_coeffs=np.zeros(om.n_bfaces))
    rc = lib().orc_assemble(C.byref(om.s), DT, dt, _p(T0), _p(bv), _p(out["diag"]),
                            _p(out["upper"]), _p(out["source"]), _p(out["internal_coeffs"]),
                            _p(out["boundary_coeffs"]))
    if rc:
        raise MemoryError
    return out


def amul(mesh, diag, upper, x, boundary_coeffs=None, x_remote=None):
    om = _om(mesh)
    bc = np.zeros(om.n_bfaces) if boundary_coeffs is None else np.ascontiguousarray(boundary_coeffs, np.float64)
    xr = np.zeros(om.n_bfaces) if x_remote is None else np.ascontiguousarray(x_remote, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(om.n_cells)
    lib().orc_amul(C.byref(om.s), _p(np.ascontiguousarray(diag, np.float64)),
                   _p(np.ascontiguousarray(upper, np.float64)), _p(bc), _p(x), _p(xr), _p(y))
    return y


def sumA(mesh, diag, upper, boundary_coeffs=None):
    om = _om(mesh)
    bc = np.zeros(om.n_bfaces) if boundary_coeffs is None else np.ascontiguousarray(boundary_coeffs, np.float64)
    out = np.zeros(om.n_cells)
    lib().orc_sumA(C.byref(om.s), _p(np.ascontiguousarray(diag, np.float64)),
                   _p(np.ascontiguousarray(upper, np.float64)), _p(bc), _p(out))
    return out


def _callbacks(gsum: Optional[Callable], halo: Optional[Callable], n_cells: int, n_bfaces: int):
    g = GSUM(0)
    h = HALO(0)
    if gsum is not None:
        def _g(ctx, vals, k):
            arr = np.ctypeslib.as_array(vals, shape=(k,))
            arr[:] = gsum(arr.copy())
        g = GSUM(_g)
    if halo is not None:
        def _h(ctx, x, xr):
            xa = np.ctypeslib.as_array(x, shape=(max(n_cells, 1),))[:n_cells].copy()
            xra = np.ctypeslib.as_array(xr, shape=(max(n_bfaces, 1),))
            halo(xa, xra[:n_bfaces])
        h = HALO(_h)
    return g, h


def pcg(mesh, sys: dict, psi: np.ndarray, tol=1e-10, rel_tol=0.0, max_iter=1000, min_iter=0,
        gsum=None, halo=None, precond="diagonal"):
    """OpenFOAM PCG (diagonal or DIC preconditioner). Returns (psi, perf dict)."""
    om = _om(mesh)
    psi = np.array(psi, dtype=np.float64, copy=True)
    perf = Perf()
    g, h = _callbacks(gsum, halo, om.n_cells, om.n_bfaces)
    bc = sys.get("boundary_coeffs")
    bc = np.zeros(om.n_bfaces) if bc is None else np.ascontiguousarray(bc, np.float64)
    rc = lib().orc_pcg_p(C.byref(om.s), _p(np.ascontiguousarray(sys["diag"], np.float64)),
                         _p(np.ascontiguousarray(sys["upper"], np.float64)), _p(bc),
                         _p(np.ascontiguousarray(sys["source"], np.float64)), _p(psi),
                         tol, rel_tol, max_iter, min_iter, PRECONDITIONERS[precond], g, h, None,
                         C.byref(perf))
    if rc:
        raise MemoryError
    return psi, perf.as_dict()


def laplacian_foam(mesh, T0, n_steps, DT=1.0, dt=0.2, tol=1e-10, rel_tol=0.0, max_iter=1000,
                   min_iter=0, gsum=None, halo=None, b_value=None, precond="diagonal"):
    """Listing 1 time loop. Returns (T, b_value, [perf dicts])."""
    om = _om(mesh)
    T = np.array(T0, dtype=np.float64, copy=True)
    bv = np.array(om.b_value if b_value is None else b_value, dtype=np.float64, copy=True)
    perfs = (Perf * max(n_steps, 1))()
    g, h = _callbacks(gsum, halo, om.n_cells, om.n_bfaces)
    rc = lib().orc_laplacian_foam_p(C.byref(om.s), DT, dt, _p(T), _p(bv), n_steps, tol, rel_tol,
                                    max_iter, min_iter, PRECONDITIONERS[precond], g, h, None, perfs)
    if rc:
        raise MemoryError
    return T, bv, [perfs[i].as_dict() for i in range(n_steps)]


def dic(mesh, diag, upper, r=None):
    """OpenFOAM DICPreconditioner: the reciprocal DIC
    diagonal rD and, if r is given, w = M^-1 r.  Returns (rD, w or None)."""
    om = _om(mesh)
    rD = np.zeros(om.n_cells)
    w = None if r is None else np.zeros(om.n_cells)
    rr = None if r is None else np.ascontiguousarray(r, np.float64)
    rc = lib().orc_dic(C.byref(om.s), _p(np.ascontiguousarray(diag, np.float64)),
                       _p(np.ascontiguousarray(upper, np.float64)), _p(rr), _p(rD), _p(w))
    if rc:
        raise MemoryError
    return rD, w


GAMG_MAXL = 30


def gamg(mesh, diag=None, upper=None, r=None):
    """GAMG hierarchy of a mesh (reading A43): dict(n=[cells per level],
    nf=[faces per level], agg=[level l -> l+1 maps]) and, with (diag, upper,
    r), w = M^-1 r (one V-cycle)."""
    om = _om(mesh)
    n = np.zeros(GAMG_MAXL + 1, np.int32)
    nf = np.zeros(GAMG_MAXL + 1, np.int32)
    aggs = np.zeros(max(2 * om.n_cells, 1), np.int32)
    w = np.zeros(om.n_cells) if r is not None else None
    d = None if diag is None else np.ascontiguousarray(diag, np.float64)
    u = None if upper is None else np.ascontiguousarray(upper, np.float64)
    rr = None if r is None else np.ascontiguousarray(r, np.float64)
    L = lib().orc_gamg(C.byref(om.s), _p(d), _p(u), n.ctypes.data, nf.ctypes.data, aggs.ctypes.data,
                       _p(rr), _p(w))
    if L < 0:
        raise ValueError(f"GAMG oracle failed ({L})")
    sizes = [int(x) for x in n[:L + 1]]
    out, off = [], 0
    for l in range(L):
        out.append(aggs[off:off + sizes[l]].copy())
        off += sizes[l]
    res = dict(n=sizes, nf=[int(x) for x in nf[:L + 1]], agg=out)
    if w is not None:
        res["w"] = w
    return res


def gamg_level(mesh, diag, upper, level):
    """Coarse matrix of `level`: dict(D, U, l, u) (faces upper-triangular)."""
    om = _om(mesh)
    info = gamg(mesh)
    n, nf = info["n"][level], info["nf"][level]
    D, U = np.zeros(n), np.zeros(max(nf, 1))
    fl, fu = np.zeros(max(nf, 1), np.int32), np.zeros(max(nf, 1), np.int32)
    rc = lib().orc_gamg_level(C.byref(om.s), _p(np.ascontiguousarray(diag, np.float64)),
                              _p(np.ascontiguousarray(upper, np.float64)), level, D.ctypes.data,
                              U.ctypes.data, fl.ctypes.data, fu.ctypes.data)
    if rc:
        raise ValueError(f"GAMG oracle failed ({rc})")
    return dict(D=D, U=U[:nf], l=fl[:nf], u=fu[:nf])


def self_halo(mesh):
    """Halo callback for a mesh whose processor patches couple to the same
    rank (pairs of consecutive self-processor patches, matched face by face)."""
    om = _om(mesh)
    sl = om.patch_slices()
    procs = [i for i, p in enumerate(mesh.patches) if p.type == "processor"]
    pairs = [(procs[i], procs[i + 1]) for i in range(0, len(procs), 2)]

    def halo(x, xr):
        for a, b in pairs:
            xr[sl[a]] = x[om.b_cells[sl[b]]]
            xr[sl[b]] = x[om.b_cells[sl[a]]]
    return halo


# ------------------------------------------- non-orthogonal correction path
def _need_geom(om):
    if not om.has_geometry:
        raise ValueError("mesh has no full geometry (Sf, Cf, C, patch Sf)")


def weights(mesh):
    """Owner interpolation weights (Listing 'weights parallel loop')."""
    om = _om(mesh)
    _need_geom(om)
    w = np.zeros(om.n_faces)
    lib().orc_weights(C.byref(om.s), _p(w))
    return w


def corr_vectors(mesh):
    om = _om(mesh)
    _need_geom(om)
    cv = np.zeros((om.n_faces, 3))
    lib().orc_corr_vectors(C.byref(om.s), _p(cv))
    return cv


def grad(mesh, x, b_value=None):
    """Green-Gauss cell gradient [n,3] (gaussGrad::gradf) and the
    corrected boundary gradient [B,3] (correctBoundaryConditions)."""
    om = _om(mesh)
    _need_geom(om)
    x = np.ascontiguousarray(x, np.float64)
    bv = om.b_value if b_value is None else np.ascontiguousarray(b_value, np.float64)
    w = weights(om)
    g = np.zeros((om.n_cells, 3))
    lib().orc_grad(C.byref(om.s), _p(w), _p(x), _p(bv), _p(g))
    bg = np.zeros((om.n_bfaces, 3))
    lib().orc_grad_bc(C.byref(om.s), _p(x), _p(bv), _p(g), _p(bg))
    return g, bg


def lap_correction(mesh, DT, g):
    """Source contribution -V*div(gammaMagSf*(corr & interpolate(grad)))."""
    om = _om(mesh)
    _need_geom(om)
    w, cv = weights(om), corr_vectors(om)
    out = np.zeros(om.n_cells)
    lib().orc_lap_correction(C.byref(om.s), DT, _p(w), _p(cv), _p(np.ascontiguousarray(g, np.float64)), _p(out))
    return out


def laplacian_foam_corrected(mesh, T0, n_steps, n_corr=1, DT=1.0, dt=0.2, tol=1e-10, rel_tol=0.0,
                             max_iter=1000, min_iter=0, b_value=None, precond="diagonal"):
    """Listing 1 with Gauss linear corrected laplacian and n_corr non-orthogonal
    correctors per step.  Returns (T, b_value, [perf per corrector solve])."""
    om = _om(mesh)
    _need_geom(om)
    T = np.array(T0, dtype=np.float64, copy=True)
    bv = np.array(om.b_value if b_value is None else b_value, dtype=np.float64, copy=True)
    perfs = (Perf * max(n_steps * (n_corr + 1), 1))()
    rc = lib().orc_laplacian_foam_corrected_p(C.byref(om.s), DT, dt, _p(T), _p(bv), n_steps, n_corr, tol,
                                              rel_tol, max_iter, min_iter, PRECONDITIONERS[precond], perfs)
    if rc:
        raise MemoryError
    return T, bv, [perfs[i].as_dict() for i in range(n_steps * (n_corr + 1))]


def face_gamma(mesh, DT_field):
    """Face / boundary diffusivities of a cell DT field (linear interpolation
    with the weights of P:321-334; boundary DT[faceCell])."""
    om = _om(mesh)
    _need_geom(om)
    w = weights(om)
    g, gb = np.zeros(om.n_faces), np.zeros(om.n_bfaces)
    lib().orc_face_gamma(C.byref(om.s), _p(w), _p(np.ascontiguousarray(DT_field, np.float64)), _p(g), _p(gb))
    return g, gb
