"""Peer-memory (CUDA IPC) transport (-m gpu).

* one process, self-coupled processor patches, P2P with nranks = 1: the
  kernels' halo stores and mailbox allreduce on their own buffers;
* TWO processes sharing the one GPU (CUDA IPC within a device), each owning
  a slab of the cube, handles exchanged over a gloo group: the real
  multi-rank code path (kernel-side halo puts into the other process's
  memory, rank-ordered mailbox allreduce), compared with the undecomposed
  oracle.  Watchdog: a missing peer traps after 30 s instead of hanging.
"""
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


@pytest.mark.parametrize("persistent,variant", [(True, 0), (False, 0), (True, 2)])
def test_p2p_loopback_single_process(P, persistent, variant):
    m = meshgen.block_mesh(14, 12, 16, bc={"ymin": ("fixedValue", 1.0)})
    c = decompose.cut_mesh(m, decompose.z_plane_faces(m, 7))
    s = meshgen.multimode_field(m)
    To, _, po = oracle.laplacian_foam(m, s, 4)
    ctx = P.Context(0)
    ctx.set_option("persistent", persistent)
    ctx.set_option("variant", variant)
    ctx.p2p_init(1, 0)
    mesh = P.Mesh(ctx, c)
    mesh.p2p_connect([mesh.p2p_export()], 0)
    mesh.set_T(s)
    pg = mesh.step(4)
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po))
    n_pcg, _ = ctx.kernel_stats("pcg")
    assert (n_pcg > 0) == persistent
    # standalone Amul through the peer-memory halo
    ldu = mesh.assemble(1.0, 0.2)
    x = meshgen.random_field(m, seed=2)
    ref = oracle.assemble(m, 1.0, 0.2, T)
    y_ref = oracle.amul(m, ref["diag"], ref["upper"], x)
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    ldu.amul(xd, yd)
    scale = np.abs(ref["diag"] * x) + 6 * np.abs(ref["upper"]).max() * np.abs(x).max()
    assert np.max(np.abs(yd.cpu().numpy() - y_ref) / scale) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("renumber", [0, 2])
def test_p2p_loopback_dic(P, renumber):
    """DIC through the peer-memory transport (processor-local factor and
    sweeps, halo w puts, mailbox allreduce) vs the oracle on the same cut
    mesh with its self halo, in the same numbering (A41, A42)."""
    m = meshgen.block_mesh(10, 9, 12, bc={"ymin": ("fixedValue", 1.0)})
    c = decompose.cut_mesh(m, decompose.z_plane_faces(m, 6))
    s = meshgen.multimode_field(m)
    order = meshgen.colour_order(c) if renumber == 2 else np.arange(c.n_cells)
    co = meshgen.relabel_mesh(c, order) if renumber == 2 else c
    To, _, po = oracle.laplacian_foam(co, s[order], 4, halo=oracle.self_halo(co), precond="DIC")
    ctx = P.Context(0)
    ctx.p2p_init(1, 0)
    mesh = P.Mesh(ctx, c, renumber=renumber)
    mesh.p2p_connect([mesh.p2p_export()], 0)
    mesh.set_T(s)
    pg = mesh.step(4, precond="DIC")
    T = mesh.get_T()[order]
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    ctx.close()


def test_dic_needs_peer_memory_with_processor_patches(P):
    m = meshgen.block_mesh(6)
    c = decompose.cut_mesh(m, decompose.z_plane_faces(m, 3))
    ctx = P.Context(0)
    mesh = P.Mesh(ctx, c)
    mesh.set_T(np.ones(c.n_cells))
    with pytest.raises(P.LfoamError) as e:
        mesh.step(1, precond="DIC")
    assert e.value.status == 1
    ctx.close()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _rank_main(rank, world, port, persistent, out, precond="diagonal", variant=0):
    import torch.distributed as dist
    import paper_2507_18268_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        g = meshgen.block_mesh(18, 16, 20, bc={"xmax": "zeroGradient"})
        part = decompose.slab_partition(g, world)
        m, cells = decompose.local_mesh(g, part, rank)
        ctx = P.Context(0)
        ctx.set_option("persistent", persistent)
        ctx.set_option("variant", variant)
        ctx.p2p_init(world, rank)
        mesh = P.Mesh(ctx, m)
        hs = [None] * world
        dist.all_gather_object(hs, mesh.p2p_export())
        mesh.p2p_connect(hs, rank)
        T0 = meshgen.multimode_field(g)[cells]
        mesh.set_T(T0)
        perfs = mesh.step(3, precond=precond)
        ref = None
        if precond != "diagonal":
            # the decomposed oracle on the same subdomain (gloo gSum / halo):
            # block-Jacobi DIC, processor-local like OpenFOAM's
            from test_decompose import gloo_oracle_callbacks
            gsum, halo = gloo_oracle_callbacks(m)
            To, _, po = oracle.laplacian_foam(m, T0, 3, gsum=gsum, halo=halo, precond=precond)
            ref = (To, [p["n_iterations"] for p in po])
        out[rank] = ("ok", cells, mesh.get_T(), [p["n_iterations"] for p in perfs], ref)
        dist.barrier()
        ctx.close()
    except Exception as e:  # report instead of hanging the peer
        out[rank] = ("error", repr(e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("persistent,world,variant", [(False, 2, 0), (True, 2, 0), (True, 3, 0), (True, 2, 2)])
def test_p2p_two_processes_one_gpu(P, persistent, world, variant):
    """world = 3: the middle rank has two processor patches (an interior slab);
    variant = 2 forces the HBM-bound persistent variant on the halo path (the
    small test meshes otherwise take the L2-resident one)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, persistent, out, "diagonal", variant))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    res = dict(out)
    assert len(res) == world, res
    for r in range(world):
        assert res[r][0] == "ok", res[r]
    g = meshgen.block_mesh(18, 16, 20, bc={"xmax": "zeroGradient"})
    s = meshgen.multimode_field(g)
    To, _, po = oracle.laplacian_foam(g, s, 3)
    T = np.zeros(g.n_cells)
    for r in range(world):
        _, cells, Tr, its, _ = res[r]
        T[cells] = Tr
        assert all(abs(a - b["n_iterations"]) <= 1 for a, b in zip(its, po)), (its, po)
    assert all(res[r][3] == res[0][3] for r in range(world))  # identical stopping decisions on all ranks
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))


def test_p2p_two_processes_one_gpu_dic(P):
    """Two ranks, DIC (block-Jacobi IC(0) across the slab interface): each
    rank against the decomposed oracle run in the same process over gloo."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, True, out, "DIC")) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    res = dict(out)
    assert len(res) == world, res
    for r in range(world):
        assert res[r][0] == "ok", res[r]
        _, cells, Tr, its, (To, its_o) = res[r]
        assert np.max(np.abs(Tr - To)) <= 1e-8 * np.max(np.abs(To))
        assert all(abs(a - b) <= 1 for a, b in zip(its, its_o)), (its, its_o)
    assert res[0][3] == res[1][3]


def _amul_rank_main(rank, world, port, out):
    """Back-to-back standalone ldu_amul calls with different x through the
    peer-memory halo (the T halo of call i+1 must not overwrite
    the one a slower rank still reads in call i — recvT is double-buffered by
    push parity).  Rank 1 is slowed down between calls."""
    import time
    import torch.distributed as dist
    import paper_2507_18268_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        g = meshgen.block_mesh(24, 20, 22, bc={"xmax": "zeroGradient"})
        part = decompose.slab_partition(g, world)
        m, cells = decompose.local_mesh(g, part, rank)
        ctx = P.Context(0)
        ctx.p2p_init(world, rank)
        mesh = P.Mesh(ctx, m)
        hs = [None] * world
        dist.all_gather_object(hs, mesh.p2p_export())
        mesh.p2p_connect(hs, rank)
        T0 = meshgen.multimode_field(g)[cells]
        mesh.set_T(T0)
        ldu = mesh.assemble(1.0, 0.2)
        ys = []
        for i in range(12):
            x = torch.as_tensor(meshgen.random_field(g, seed=100 + i)[cells], device="cuda")
            y = torch.empty_like(x)
            if rank == 1 and i % 2:
                time.sleep(0.02)
            ldu.amul(x, y)
            ys.append(y.cpu().numpy())
        # and a solve right after an Amul (same halo buffers)
        psi = torch.as_tensor(T0, device="cuda")
        perf = ldu.pcg_solve(psi)
        out[rank] = ("ok", cells, ys, psi.cpu().numpy(), perf["n_iterations"])
        dist.barrier()
        ctx.close()
    except Exception as e:
        out[rank] = ("error", repr(e))
    finally:
        dist.destroy_process_group()


def test_p2p_two_processes_back_to_back_amul(P):
    import torch.multiprocessing as mp
    world = 2
    mctx = mp.get_context("spawn")
    out = mctx.Manager().dict()
    port = _free_port()
    procs = [mctx.Process(target=_amul_rank_main, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    res = dict(out)
    assert len(res) == world, res
    for r in range(world):
        assert res[r][0] == "ok", res[r]
    g = meshgen.block_mesh(24, 20, 22, bc={"xmax": "zeroGradient"})
    T0 = meshgen.multimode_field(g)
    ref = oracle.assemble(g, 1.0, 0.2, T0)
    for i in range(12):
        x = meshgen.random_field(g, seed=100 + i)
        y_ref = oracle.amul(g, ref["diag"], ref["upper"], x)
        scale = np.abs(ref["diag"] * x) + 6 * np.abs(ref["upper"]).max() * np.abs(x).max()
        for r in range(world):
            _, cells, ys, _, _ = res[r]
            assert np.max(np.abs(ys[i] - y_ref[cells]) / scale[cells]) <= 1e-12, (i, r)
    x_ref, p_ref = oracle.pcg(g, ref, T0)
    for r in range(world):
        _, cells, _, psi, it = res[r]
        assert np.max(np.abs(psi - x_ref[cells])) <= 1e-8 * np.max(np.abs(x_ref))
        assert abs(it - p_ref["n_iterations"]) <= 1
