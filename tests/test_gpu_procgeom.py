"""Non-orthogonal correction and spatially varying DT ACROSS processor
patches (SURVEY §8(f) rows 1-2 on the decomposed path; the paper's multi-GPU
runs are MPI decompositions of the whole application, §6.2, and its
gradient kernels carry the coupled-patch handling, §5.2) — CUDA vs
the CPU oracle of the UNDECOMPOSED mesh through the C ABI (-m gpu).

A coupled face interpolates with the neighbour rank's value (T halo for the
gradient, gradient halo for the correction, DT halo for the face
diffusivity) with weights and correction vectors formed from the coupled
cell's centre, so the decomposed system is the undecomposed one up to
rounding: gradients 1e-12 relative, T after the steps 1e-8, iterations +-1.

* loopback: one process, an internal plane cut into a pair of self-coupled
  processor patches (reading A32), host-copy halos or the peer-memory
  transport with one rank;
* two processes sharing the GPU over CUDA IPC, each owning a slab.
"""
import dataclasses
import os
import socket

import numpy as np
import pytest

import meshgen
import oracle
from paper_2507_18268_b200 import decompose

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2507_18268_b200 as _P
    return _P


def mixed_bc():
    return {"xmin": ("fixedValue", 1.5), "xmax": "zeroGradient", "ymin": ("fixedValue", -0.5),
            "zmax": "zeroGradient"}


def skewed(nx=10, ny=9, nz=12, dt_field=False, seed=4):
    m = meshgen.skewed_block_mesh(nx, ny, nz, shear=(0.3, 0.1, 0.2), grading=(1.15, 0.9, 1.05), bc=mixed_bc())
    if dt_field:
        m = dataclasses.replace(m, DT_field=np.random.default_rng(seed).uniform(0.2, 3.0, m.n_cells))
    return m


def loopback_ctx(P, transport):
    ctx = P.Context(0)
    if transport == "p2p":
        ctx.p2p_init(1, 0)
    return ctx


def connect(mesh, transport):
    if transport == "p2p":
        mesh.p2p_connect([mesh.p2p_export()], 0)


@pytest.mark.parametrize("transport", ["copy", "p2p"])
def test_loopback_fvc_grad(P, transport):
    m = skewed()
    c = decompose.cut_mesh(m, decompose.z_plane_faces(m, 6))
    x = meshgen.random_field(m, seed=3)
    g_ref, _ = oracle.grad(m, x)
    ctx = loopback_ctx(P, transport)
    mesh = P.Mesh(ctx, c)
    connect(mesh, transport)
    g = mesh.fvc_grad(torch.as_tensor(x, device="cuda")).cpu().numpy()
    scale = np.max(np.abs(g_ref))
    assert np.max(np.abs(g - g_ref)) <= 1e-12 * scale
    ctx.close()


@pytest.mark.parametrize("transport", ["copy", "p2p"])
@pytest.mark.parametrize("dt_field,corrected", [(False, True), (True, False), (True, True)])
def test_loopback_steps(P, transport, dt_field, corrected):
    m = skewed(dt_field=dt_field)
    c = decompose.cut_mesh(m, decompose.z_plane_faces(m, 6))
    T0 = meshgen.sine_field(m) + 0.1 * meshgen.random_field(m, seed=2)
    if corrected:
        To, _, po = oracle.laplacian_foam_corrected(m, T0, 3, n_corr=1)
    else:
        To, _, po = oracle.laplacian_foam(m, T0, 3)
    ctx = loopback_ctx(P, transport)
    mesh = P.Mesh(ctx, c)
    connect(mesh, transport)
    if dt_field:
        np.testing.assert_array_equal(mesh.get_DT_field(), m.DT_field)
        # the coupled faces' diffusivity: the assembled diagonal equals the uncut one
        mesh.set_T(T0)
        d = mesh.assemble(1.0, 0.2).export()["diag"]
        d_ref = oracle.assemble(m, 1.0, 0.2, T0)["diag"]
        assert np.max(np.abs(d - d_ref)) <= 1e-12 * np.max(np.abs(d_ref))
    mesh.set_T(T0)
    pg = mesh.step(3, corrected=corrected, n_non_orth_correctors=1 if corrected else 0)
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    ctx.close()


def test_processor_patches_without_cn_refused(P):
    """A geometry mesh whose processor patches lack cf/cn keeps the old
    refusal (INVALID_ARG) for the corrected path and DT fields."""
    m = skewed(6, 5, 6)
    c = decompose.cut_mesh(m, decompose.z_plane_faces(m, 3))
    c = dataclasses.replace(c, patches=[dataclasses.replace(p, Cn=None) if p.type == "processor" else p
                                        for p in c.patches])
    ctx = P.Context(0)
    mesh = P.Mesh(ctx, c)
    mesh.set_T(np.ones(c.n_cells))
    with pytest.raises(P.LfoamError) as e:
        mesh.step(1, corrected=True)
    assert e.value.status == 1
    with pytest.raises(P.LfoamError) as e:
        mesh.set_DT_field(np.ones(c.n_cells))
    assert e.value.status == 1
    ctx.close()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _rank_main(rank, world, port, out):
    import torch.distributed as dist
    import paper_2507_18268_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        g = skewed(10, 9, 14, dt_field=True)
        part = decompose.slab_partition(g, world)
        m, cells = decompose.local_mesh(g, part, rank)
        T0 = (meshgen.sine_field(g) + 0.1 * meshgen.random_field(g, seed=2))[cells]
        ctx = P.Context(0)
        ctx.p2p_init(world, rank)
        mesh = P.Mesh(ctx, m)
        hs = [None] * world
        dist.all_gather_object(hs, mesh.p2p_export())
        mesh.p2p_connect(hs, rank)          # sets the DT field (its halo) afterwards
        x = torch.as_tensor(meshgen.random_field(g, seed=3)[cells], device="cuda")
        grad = mesh.fvc_grad(x).cpu().numpy()
        mesh.set_T(T0)
        perfs = mesh.step(3, corrected=True, n_non_orth_correctors=1)
        out[rank] = ("ok", cells, mesh.get_T(), [p["n_iterations"] for p in perfs], grad)
        dist.barrier()
        ctx.close()
    except Exception as e:  # report instead of hanging the peer
        out[rank] = ("error", repr(e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_processes_corrected_dt_field(P, world):
    import torch.multiprocessing as mp
    mctx = mp.get_context("spawn")
    out = mctx.Manager().dict()
    port = _free_port()
    procs = [mctx.Process(target=_rank_main, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    for p in procs:
        if p.is_alive():
            p.kill()
    res = dict(out)
    assert len(res) == world, res
    for r in range(world):
        assert res[r][0] == "ok", res[r]
    g = skewed(10, 9, 14, dt_field=True)
    T0 = meshgen.sine_field(g) + 0.1 * meshgen.random_field(g, seed=2)
    To, _, po = oracle.laplacian_foam_corrected(g, T0, 3, n_corr=1)
    g_ref, _ = oracle.grad(g, meshgen.random_field(g, seed=3))
    T = np.zeros(g.n_cells)
    G = np.zeros((g.n_cells, 3))
    for r in range(world):
        _, cells, Tr, its, gr = res[r]
        T[cells] = Tr
        G[cells] = gr
        assert all(abs(a - b["n_iterations"]) <= 1 for a, b in zip(its, po)), (its, po)
    assert all(res[r][3] == res[0][3] for r in range(world))
    assert np.max(np.abs(G - g_ref)) <= 1e-12 * np.max(np.abs(g_ref))
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
