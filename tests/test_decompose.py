"""Multi-GPU host logic on CPU (-m "not gpu"): slab decomposition, processor
patch pairing, and the decomposed solve over a world-size-2 gloo group
(oracle per rank, gloo allreduce for gSum, gloo send/recv for the halo)
against the undecomposed oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import meshgen
import oracle
from paper_2507_18268_b200 import decompose


def _mesh():
    return meshgen.block_mesh(6, 5, 8, bc={"xmin": ("fixedValue", 1.0), "zmax": "zeroGradient"})


@pytest.mark.parametrize("P", [2, 3, 4])
def test_partition_covers_mesh(P):
    m = _mesh()
    part = decompose.slab_partition(m, P)
    subs = [decompose.local_mesh(m, part, r) for r in range(P)]
    assert sum(s.n_cells for s, _ in subs) == m.n_cells
    assert np.array_equal(np.sort(np.concatenate([c for _, c in subs])), np.arange(m.n_cells))
    inner = sum(s.n_faces for s, _ in subs)
    pairs = decompose.check_pairing([s for s, _ in subs])
    assert inner + sum(n for _, _, n in pairs) == m.n_faces
    for s, cells in subs:      # local LDU stays upper-triangular
        key = s.owner.astype(np.int64) * s.n_cells + s.neighbour
        assert np.all(np.diff(key) > 0)
        for p in s.patches[:6]:
            assert p.n_faces == np.isin(m.patches[s.patches.index(p)].face_cells, cells).sum()


def test_cube_slabs_are_z_planes():
    m = meshgen.block_mesh(8)
    part = decompose.slab_partition(m, 4)
    k = np.arange(m.n_cells) // 64
    assert np.array_equal(part, k // 2)
    s, _ = decompose.local_mesh(m, part, 1)
    procs = [p for p in s.patches if p.type == "processor"]
    assert [p.neighb_rank for p in procs] == [0, 2] and all(p.n_faces == 64 for p in procs)


def test_cut_mesh_loopback_equals_undecomposed():
    """Reading A32: self-coupled processor patches solve the same system."""
    m = meshgen.block_mesh(6, 6, 6)
    s = meshgen.sine_field(m)
    T_ref, _, p_ref = oracle.laplacian_foam(m, s, 4)
    c = decompose.cut_mesh(m, decompose.z_plane_faces(m, 3))
    T, _, p = oracle.laplacian_foam(c, s, 4, halo=oracle.self_halo(c))
    # interface terms are summed after the face loop: rounding-level change,
    # amplified to solver-tolerance level through the PCG iterates
    assert np.max(np.abs(T - T_ref)) <= 1e-9 * np.max(np.abs(T_ref))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(p, p_ref))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def gloo_oracle_callbacks(sub):
    """gSum (gloo allreduce) and processor-patch halo (gloo send/recv) for
    the oracle's decomposed mode on this rank's subdomain `sub`."""
    om = oracle.OMesh(sub)
    sl = om.patch_slices()
    procs = [(i, p) for i, p in enumerate(sub.patches) if p.type == "processor"]

    def gsum(vals):
        t = torch.from_numpy(vals.copy())
        dist.all_reduce(t)
        return t.numpy()

    def halo(x, xr):
        reqs, bufs = [], []
        for i, p in procs:
            send = torch.from_numpy(np.ascontiguousarray(x[om.b_cells[sl[i]]]))
            recv = torch.empty(p.n_faces, dtype=torch.float64)
            reqs.append(dist.isend(send, p.neighb_rank))
            reqs.append(dist.irecv(recv, p.neighb_rank))
            bufs.append((i, recv, send))
        for r in reqs:
            r.wait()
        for i, recv, _ in bufs:
            xr[sl[i]] = recv.numpy()
    return gsum, halo


def _worker(rank, world, port, out, precond="diagonal"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = _mesh()
    part = decompose.slab_partition(m, world)
    sub, cells = decompose.local_mesh(m, part, rank)
    gsum, halo = gloo_oracle_callbacks(sub)
    T0 = meshgen.multimode_field(m)[cells]
    T, _, perfs = oracle.laplacian_foam(sub, T0, 3, gsum=gsum, halo=halo, precond=precond)
    out[rank] = (cells, T, [p["n_iterations"] for p in perfs])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_decomposed_solve_matches_undecomposed(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    m = _mesh()
    T_ref, _, p_ref = oracle.laplacian_foam(m, meshgen.multimode_field(m), 3)
    T = np.zeros(m.n_cells)
    for r in range(world):
        cells, Tr, its = out[r]
        T[cells] = Tr
        assert all(abs(a - b["n_iterations"]) <= 1 for a, b in zip(its, p_ref))
    assert np.max(np.abs(T - T_ref)) <= 1e-9 * np.max(np.abs(T_ref))


def test_gloo_decomposed_dic():
    """Decomposed DIC is block-Jacobi IC(0) (processor-local, reading A42):
    the same converged T as the undecomposed solve within the solver
    tolerance, identical stopping decisions on both ranks, fewer iterations
    than the decomposed diagonal preconditioner."""
    world = 2
    mgr = mp.Manager()
    out, outd = mgr.dict(), mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, "DIC"), nprocs=world, join=True)
    mp.spawn(_worker, args=(world, _free_port(), outd, "diagonal"), nprocs=world, join=True)
    m = _mesh()
    T_ref, _, _ = oracle.laplacian_foam(m, meshgen.multimode_field(m), 3, precond="DIC")
    T = np.zeros(m.n_cells)
    for r in range(world):
        cells, Tr, _ = out[r]
        T[cells] = Tr
    assert out[0][2] == out[1][2]
    assert all(a < b for a, b in zip(out[0][2], outd[0][2])), (out[0][2], outd[0][2])
    assert np.max(np.abs(T - T_ref)) <= 1e-8 * np.max(np.abs(T_ref))
