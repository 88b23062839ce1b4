"""Thin ctypes binding of liblfoam.so (include/lfoam.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module
only converts numpy/torch arguments to pointers and status codes to
exceptions.  If liblfoam.so is missing it raises ImportError: there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LFOAM_LIB selects an in-tree build variant (perf experiments); default liblfoam.so
LIB_PATH = os.path.join(_HERE, os.environ.get("LFOAM_LIB", "liblfoam.so"))

LF_OK = 0
STATUS = {0: "LF_OK", 1: "LF_ERR_INVALID_ARG", 2: "LF_ERR_STATE", 3: "LF_ERR_OOM",
          4: "LF_ERR_CUDA", 5: "LF_ERR_NCCL", 6: "LF_ERR_INTERNAL"}
PATCH_TYPES = {"fixedValue": 0, "zeroGradient": 1, "processor": 2}
FIELD_T, FIELD_PATCH_VALUE, FIELD_DT = 0, 1, 2
KERNELS = {"assemble": 0, "setup": 1, "phase1": 2, "phase2": 3, "amul": 4, "sumpsi": 5, "pack": 6, "pcg": 7,
           "nonorth": 8, "pcg_dic": 9, "precond": 10, "pcg_gamg": 11}
# lf_preconditioner (OpenFOAM fvSolution names)
PRECONDITIONERS = {"diagonal": 0, "DIC": 1, "DILU": 2, "GAMG": 3}
GAMG_MAXL = 30
# lf_mesh_desc.renumber
RENUMBER = {False: 0, True: 1, 0: 0, 1: 1, 2: 2, "none": 0, "rcm": 1, "colour": 2}
OPTIONS = {"persistent": 0, "graphs": 1, "variant": 2, "compressed_labels": 3, "overlap_halo": 4, "l2_prefetch": 5, "dynamic_trips": 6}


class LfoamError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class PatchDesc(C.Structure):
    _fields_ = [("type", C.c_int), ("n_faces", C.c_int32), ("face_cells", C.c_void_p),
                ("mag_sf", C.c_void_p), ("delta_coeffs", C.c_void_p), ("value", C.c_void_p),
                ("neighb_rank", C.c_int32), ("sf", C.c_void_p), ("cf", C.c_void_p), ("cn", C.c_void_p)]


class MeshDesc(C.Structure):
    _fields_ = [("n_cells", C.c_int32), ("n_faces", C.c_int32), ("n_patches", C.c_int32),
                ("owner", C.c_void_p), ("neighbour", C.c_void_p), ("mag_sf", C.c_void_p),
                ("delta_coeffs", C.c_void_p), ("V", C.c_void_p), ("patches", C.POINTER(PatchDesc)),
                ("renumber", C.c_int32), ("sf", C.c_void_p), ("cf", C.c_void_p), ("c", C.c_void_p)]


class Params(C.Structure):
    _fields_ = [("DT", C.c_double), ("dt", C.c_double), ("corrected", C.c_int32),
                ("n_non_orth_correctors", C.c_int32), ("variable_DT", C.c_int32)]


class Controls(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("rel_tol", C.c_double),
                ("max_iter", C.c_int32), ("min_iter", C.c_int32),
                ("preconditioner", C.c_int32), ("reserved", C.c_int32)]


class Perf(C.Structure):
    _fields_ = [("initial_residual", C.c_double), ("final_residual", C.c_double),
                ("n_iterations", C.c_int32), ("converged", C.c_int32), ("singular", C.c_int32),
                ("reserved", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k in ("initial_residual", "final_residual",
                                              "n_iterations", "converged", "singular")}


# name -> (restype, argtypes); every function declared in include/lfoam.h
_vp, _i32, _i64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
SIGNATURES = {
    "lf_status_string": (C.c_char_p, [C.c_int]),
    "lf_last_error": (C.c_char_p, []),
    "lf_version": (C.c_int, []),
    "lf_context_create": (C.c_int, [C.c_int, _vp, C.POINTER(_vp)]),
    "lf_context_destroy": (C.c_int, [_vp]),
    "lf_comm_unique_id": (C.c_int, [_vp]),
    "lf_comm_init": (C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    "lf_comm_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "mesh_create": (C.c_int, [_vp, C.POINTER(MeshDesc), C.POINTER(_vp)]),
    "mesh_destroy": (C.c_int, [_vp]),
    "lf_mesh_info": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i64)]),
    "lf_mesh_layout": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "lf_mesh_export_addressing": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "lf_permute": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "field_set": (C.c_int, [_vp, C.c_int, _i32, _vp, _i64, C.c_int]),
    "field_get": (C.c_int, [_vp, C.c_int, _i32, _vp, _i64, C.c_int]),
    "laplacian_assemble": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(_vp)]),
    "lf_ldu_export": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "lf_fvc_grad": (C.c_int, [_vp, _vp, _vp, _vp]),
    "ldu_amul": (C.c_int, [_vp, _vp, _vp]),
    "ldu_precondition": (C.c_int, [_vp, _i32, _vp, _vp, _vp]),
    "pcg_solve": (C.c_int, [_vp, _vp, C.POINTER(Controls), C.POINTER(Perf)]),
    "laplacianFoam_step": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Controls), _i32, C.POINTER(Perf)]),
    "lf_set_instrumentation": (C.c_int, [_vp, C.c_int]),
    "lf_kernel_stats": (C.c_int, [_vp, C.c_int, C.POINTER(_i64), C.POINTER(_d)]),
    "lf_launch_count": (C.c_int, [_vp, C.POINTER(_i64)]),
    "lf_set_option": (C.c_int, [_vp, C.c_int, C.c_int]),
    "lf_p2p_init": (C.c_int, [_vp, C.c_int, C.c_int]),
    "lf_p2p_export": (C.c_int, [_vp, _vp]),
    "lf_p2p_connect": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
    "lf_gamg_hierarchy": (C.c_int, [_vp, C.POINTER(_i32), _vp, _vp, _vp]),
    "lf_gamg_export": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _vp]),
}
P2P_HANDLE_BYTES = 1024

_lib = None


def lib():
    """Load liblfoam.so (loud failure if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None:  # older experiment variant (LFOAM_LIB); the shipped build exports all
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(st: int):
    if st != LF_OK:
        raise LfoamError(st, lib().lf_last_error().decode(errors="replace"))


def _host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _vec3(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data if a.size else None
    return a.data_ptr()  # torch tensor


def _is_device(a) -> bool:
    return not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)


def _device_sync():
    """Order torch's work and the library stream around a call on device
    vectors (the context may own a private stream): device-wide sync."""
    import torch
    torch.cuda.synchronize()


def _check_dev(t, n):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
            and t.is_contiguous() and t.numel() == n):
        raise ValueError(f"expected a contiguous float64 CUDA tensor with {n} elements")


def _check_host_out(a, n):
    """A host output buffer must be a writable C-contiguous float64 array of n."""
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
            and a.flags.writeable and a.size == n):
        raise ValueError(f"expected a writable C-contiguous float64 numpy array with {n} elements")


class Context:
    def __init__(self, device: int = 0, stream=None):
        h = C.c_void_p()
        s = None
        if stream is not None:
            s = stream if isinstance(stream, int) else stream.cuda_stream
        _check(lib().lf_context_create(device, s, C.byref(h)))
        self.h = h
        self.device = device
        self._meshes = weakref.WeakSet()  # destroyed before the context

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().lf_comm_unique_id(buf))
        return buf.raw

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(uid), 128)
        _check(lib().lf_comm_init(self.h, buf, nranks, rank))

    def p2p_init(self, nranks: int, rank: int):
        """Peer-memory transport (CUDA IPC); call before creating meshes."""
        _check(lib().lf_p2p_init(self.h, nranks, rank))
        self._p2p = True

    def comm_info(self):
        n, r = C.c_int(), C.c_int()
        _check(lib().lf_comm_info(self.h, C.byref(n), C.byref(r)))
        return n.value, r.value

    def set_option(self, name: str, value):
        """persistent / graphs: bool; variant: 0 auto, 1 L2-resident, 2 HBM-bound."""
        _check(lib().lf_set_option(self.h, OPTIONS[name], int(value)))

    def set_instrumentation(self, on: bool):
        _check(lib().lf_set_instrumentation(self.h, 1 if on else 0))

    def kernel_stats(self, kind: str):
        n, ms = C.c_int64(), C.c_double()
        _check(lib().lf_kernel_stats(self.h, KERNELS[kind], C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(lib().lf_launch_count(self.h, C.byref(n)))
        return n.value

    def close(self):
        if self.h:
            for m in list(self._meshes):
                m.close()
            _check(lib().lf_context_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def controls(tol=1e-10, rel_tol=0.0, max_iter=1000, min_iter=0, precond="diagonal") -> Controls:
    return Controls(tol, rel_tol, max_iter, min_iter, PRECONDITIONERS[precond], 0)


class Mesh:
    """A device mesh built from a meshgen-like description (duck-typed:
    n_cells, owner, neighbour, mag_sf, delta, V, patches[type, face_cells,
    mag_sf, delta, value, neighb_rank])."""

    def __init__(self, ctx: Context, m, renumber=False, geometry: Optional[bool] = None):
        """renumber: False/0 keep, True/1/"rcm" reverse Cuthill-McKee, 2/"colour"
        multicolour (the DIC levels); geometry: pass the full geometry (Sf, Cf,
        C, patch Sf) for the non-orthogonal correction path; default: when the
        description has it."""
        self.ctx = ctx
        if geometry is None:
            geometry = getattr(m, "Sf", None) is not None
        keep = []
        own = _host(m.owner, np.int32); nb = _host(m.neighbour, np.int32)
        ms = _host(m.mag_sf, np.float64); de = _host(m.delta, np.float64); V = _host(m.V, np.float64)
        keep += [own, nb, ms, de, V]
        pds = (PatchDesc * max(len(m.patches), 1))()
        self.patch_sizes = []
        self.patch_types = []
        for i, p in enumerate(m.patches):
            fc = _host(p.face_cells, np.int32); pm = _host(p.mag_sf, np.float64)
            pd = _host(p.delta, np.float64); pv = _host(p.value, np.float64)
            psf = _vec3(getattr(p, "Sf", None)) if geometry else None
            # processor patches of a geometry mesh: face centres and coupled cell centres
            cpl = geometry and p.type == "processor" and getattr(p, "Cn", None) is not None
            pcf = _vec3(p.Cf) if cpl else None
            pcn = _vec3(p.Cn) if cpl else None
            keep += [fc, pm, pd, pv, psf, pcf, pcn]
            pds[i] = PatchDesc(PATCH_TYPES[p.type], fc.shape[0], _ptr(fc), _ptr(pm), _ptr(pd), _ptr(pv),
                               int(getattr(p, "neighb_rank", -1)), _ptr(psf), _ptr(pcf), _ptr(pcn))
            self.patch_sizes.append(int(fc.shape[0]))
            self.patch_types.append(p.type)
        g = [None, None, None]
        if geometry:
            g = [_vec3(m.Sf), _vec3(m.Cf), _vec3(m.C)]  # a missing one -> NULL -> INVALID_ARG
            keep += g
        desc = MeshDesc(int(m.n_cells), int(own.shape[0]), len(m.patches), _ptr(own), _ptr(nb), _ptr(ms),
                        _ptr(de), _ptr(V), pds, RENUMBER[renumber], _ptr(g[0]), _ptr(g[1]), _ptr(g[2]))
        h = C.c_void_p()
        _check(lib().mesh_create(ctx.h, C.byref(desc), C.byref(h)))
        self.h = h
        ctx._meshes.add(self)
        self.n_cells = int(m.n_cells)
        self.n_faces = int(own.shape[0])
        self.n_bfaces = int(sum(self.patch_sizes))
        self.renumber = renumber
        self.variable_dt = False
        self._pending_dt = None
        if getattr(m, "DT_field", None) is not None:
            if getattr(ctx, "_p2p", False) and any(p.type == "processor" for p in m.patches):
                self._pending_dt = m.DT_field   # its halo needs the transport: set in p2p_connect
            else:
                self.set_DT_field(m.DT_field)

    def info(self):
        n, F, B, b = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        _check(lib().lf_mesh_info(self.h, C.byref(n), C.byref(F), C.byref(B), C.byref(b)))
        return dict(n_cells=n.value, n_faces=F.value, n_boundary_faces=B.value, device_bytes=b.value)

    def layout(self):
        """Gather layout of the mesh (lf_mesh_layout)."""
        k, ks, esc = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().lf_mesh_layout(self.h, C.byref(k), C.byref(ks), C.byref(esc)))
        return dict(ell_width=k.value, row_width=ks.value, label_escapes=esc.value)

    def gamg_hierarchy(self):
        """GAMG levels of the mesh (lf_gamg_hierarchy): dict(n=[cells per
        level], nf=[faces per level], agg=[level l -> l+1 maps])."""
        nl = C.c_int32()
        cells = np.zeros(GAMG_MAXL + 1, np.int32)
        faces = np.zeros(GAMG_MAXL + 1, np.int32)
        _check(lib().lf_gamg_hierarchy(self.h, C.byref(nl), cells.ctypes.data, faces.ctypes.data, None))
        L = nl.value
        agg = np.zeros(max(int(cells[:L - 1].sum()), 1), np.int32)
        _check(lib().lf_gamg_hierarchy(self.h, C.byref(nl), None, None, agg.ctypes.data))
        maps, off = [], 0
        for l in range(L - 1):
            maps.append(agg[off:off + cells[l]].copy())
            off += int(cells[l])
        return dict(n=[int(x) for x in cells[:L]], nf=[int(x) for x in faces[:L]], agg=maps)

    def p2p_export(self) -> bytes:
        buf = C.create_string_buffer(P2P_HANDLE_BYTES)
        _check(lib().lf_p2p_export(self.h, buf))
        return buf.raw

    def p2p_connect(self, handles, rank: int):
        """handles: list of every rank's p2p_export() bytes, in rank order."""
        blob = b"".join(bytes(h) for h in handles)
        buf = C.create_string_buffer(blob, len(blob))
        _check(lib().lf_p2p_connect(self.h, len(handles), rank, buf))
        if self._pending_dt is not None:   # collective: every rank connects, then sets its DT
            self.set_DT_field(self._pending_dt)
            self._pending_dt = None

    def export_addressing(self):
        os_ = np.zeros(self.n_cells + 1, np.int32); lo = np.zeros(self.n_faces, np.int32)
        ls = np.zeros(self.n_cells + 1, np.int32); fo = np.zeros(self.n_faces, np.int32)
        co = np.zeros(self.n_cells, np.int32)
        _check(lib().lf_mesh_export_addressing(self.h, _ptr(os_), _ptr(lo), _ptr(ls), _ptr(fo), _ptr(co)))
        return dict(owner_start=os_, losort=lo, losort_start=ls, face_order=fo, cell_order=co)

    # ---------------------------------------------------------- fields
    def set_T(self, v):
        if _is_device(v):
            _check_dev(v, self.n_cells)
            _device_sync()
            _check(lib().field_set(self.h, FIELD_T, -1, _ptr(v), self.n_cells, 1))
        else:
            a = _host(v, np.float64)
            _check(lib().field_set(self.h, FIELD_T, -1, _ptr(a), a.shape[0], 0))

    def get_T(self, out=None):
        if out is not None and _is_device(out):
            _check_dev(out, self.n_cells)
            _check(lib().field_get(self.h, FIELD_T, -1, _ptr(out), self.n_cells, 1))
            _device_sync()
            return out
        a = np.zeros(self.n_cells) if out is None else out
        _check_host_out(a, self.n_cells)
        _check(lib().field_get(self.h, FIELD_T, -1, _ptr(a), self.n_cells, 0))
        return a

    def set_DT_field(self, v):
        """Spatially varying DT (cell values, caller numbering); later solves
        use it unless called with variable_DT=False."""
        if _is_device(v):
            _check_dev(v, self.n_cells)
            _device_sync()   # torch's producer stream before the library reads v
            _check(lib().field_set(self.h, FIELD_DT, -1, _ptr(v), self.n_cells, 1))
        else:
            a = _host(v, np.float64)
            _check(lib().field_set(self.h, FIELD_DT, -1, _ptr(a), a.shape[0], 0))
        self.variable_dt = True

    def get_DT_field(self):
        a = np.zeros(self.n_cells)
        _check(lib().field_get(self.h, FIELD_DT, -1, _ptr(a), self.n_cells, 0))
        return a

    def set_patch_value(self, patch: int, v):
        a = _host(v, np.float64)
        _check(lib().field_set(self.h, FIELD_PATCH_VALUE, patch, _ptr(a), a.shape[0], 0))

    def get_patch_value(self, patch: int):
        a = np.zeros(self.patch_sizes[patch])
        _check(lib().field_get(self.h, FIELD_PATCH_VALUE, patch, _ptr(a), a.shape[0], 0))
        return a

    def permute(self, to_internal: bool, x, y):
        _check(lib().lf_permute(self.h, 1 if to_internal else 0, _ptr(x), _ptr(y)))

    # ------------------------------------------------------------ ops
    def _var(self, variable_DT):
        return int(self.variable_dt if variable_DT is None else variable_DT)

    def assemble(self, DT: float = 1.0, dt: float = 0.2, corrected: bool = False,
                 variable_DT: Optional[bool] = None) -> "Ldu":
        h = C.c_void_p()
        prm = Params(DT, dt, int(corrected), 0, self._var(variable_DT))
        _check(lib().laplacian_assemble(self.h, C.byref(prm), C.byref(h)))
        return Ldu(self, h)

    def step(self, n_steps: int, DT: float = 1.0, dt: float = 0.2, corrected: bool = False,
             n_non_orth_correctors: int = 0, variable_DT: Optional[bool] = None, **ctl) -> List[Dict]:
        """n_steps time steps; one perf dict per solve (n_steps * (1 +
        n_non_orth_correctors) when corrected)."""
        nsol = n_steps * (1 + (n_non_orth_correctors if corrected else 0))
        perfs = (Perf * max(nsol, 1))()
        prm = Params(DT, dt, int(corrected), int(n_non_orth_correctors), self._var(variable_DT))
        _check(lib().laplacianFoam_step(self.h, C.byref(prm), C.byref(controls(**ctl)), n_steps, perfs))
        return [perfs[i].as_dict() for i in range(nsol)]

    def fvc_grad(self, x, grad=None, bgrad=None):
        """grad(x) (gaussGrad, linear) into device grad[n_cells, 3] and, if
        given, the corrected boundary gradient bgrad[n_boundary_faces, 3];
        internal numbering.  Returns grad."""
        import torch
        _check_dev(x, self.n_cells)
        if grad is None:
            grad = torch.empty((self.n_cells, 3), dtype=torch.float64, device=x.device)
        _check_dev(grad, 3 * self.n_cells)
        if bgrad is not None:
            _check_dev(bgrad, 3 * self.n_bfaces)
        _device_sync()
        _check(lib().lf_fvc_grad(self.h, _ptr(x), _ptr(grad), _ptr(bgrad)))
        _device_sync()
        return grad

    def close(self):
        if getattr(self, "h", None):
            _check(lib().mesh_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Ldu:
    def __init__(self, mesh: Mesh, h):
        self.mesh = mesh
        self.h = h

    def export(self) -> Dict[str, np.ndarray]:
        m = self.mesh
        out = dict(diag=np.zeros(m.n_cells), upper=np.zeros(m.n_faces), source=np.zeros(m.n_cells),
                   internal_coeffs=np.zeros(m.n_bfaces), boundary_coeffs=np.zeros(m.n_bfaces))
        _check(lib().lf_ldu_export(self.h, _ptr(out["diag"]), _ptr(out["upper"]), _ptr(out["source"]),
                                   _ptr(out["internal_coeffs"]), _ptr(out["boundary_coeffs"])))
        return out

    def amul(self, x, y):
        _check_dev(x, self.mesh.n_cells)
        _check_dev(y, self.mesh.n_cells)
        _device_sync()
        _check(lib().ldu_amul(self.h, _ptr(x), _ptr(y)))
        _device_sync()
        return y

    def precondition(self, r, w, precond: str = "DIC", rD=None):
        """w = M^-1 r (device vectors, internal numbering); rD (optional
        device vector) receives the reciprocal preconditioner diagonal."""
        _check_dev(r, self.mesh.n_cells)
        _check_dev(w, self.mesh.n_cells)
        if rD is not None:
            _check_dev(rD, self.mesh.n_cells)
        _device_sync()
        _check(lib().ldu_precondition(self.h, PRECONDITIONERS[precond], _ptr(r), _ptr(w), _ptr(rD)))
        _device_sync()
        return w

    def gamg_level(self, level: int) -> Dict[str, np.ndarray]:
        """Galerkin matrix of GAMG level `level` from the last GAMG use
        (lf_gamg_export): dict(D, U, l, u)."""
        h = self.mesh.gamg_hierarchy()
        n, nf = h["n"][level], h["nf"][level]
        D, U = np.zeros(n), np.zeros(max(nf, 1))
        fl, fu = np.zeros(max(nf, 1), np.int32), np.zeros(max(nf, 1), np.int32)
        _check(lib().lf_gamg_export(self.h, level, D.ctypes.data, U.ctypes.data, fl.ctypes.data, fu.ctypes.data))
        return dict(D=D, U=U[:nf], l=fl[:nf], u=fu[:nf])

    def pcg_solve(self, psi, **ctl) -> Dict:
        _check_dev(psi, self.mesh.n_cells)
        _device_sync()
        perf = Perf()
        _check(lib().pcg_solve(self.h, _ptr(psi), C.byref(controls(**ctl)), C.byref(perf)))
        return perf.as_dict()
