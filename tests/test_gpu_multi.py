"""Processor-patch path on one GPU (-m gpu): self-coupled processor patches
(reading A32) exercise the interface term in assembly/Amul/PCG, the halo pack
kernels and — with a 1-rank NCCL communicator — ncclSend/ncclRecv and the
NCCL allreduce of the PCG sums; results must equal the undecomposed oracle."""
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


def cut(N=12, k=None, bc=None):
    m = meshgen.block_mesh(N, bc=bc)
    return m, decompose.cut_mesh(m, decompose.z_plane_faces(m, k or N // 2))


@pytest.mark.parametrize("use_nccl", [False, True])
def test_loopback_assembly_and_amul(P, use_nccl):
    m, c = cut(10, bc={"xmin": ("fixedValue", 2.0)})
    ctx = P.Context(0)
    if use_nccl:
        ctx.comm_init(P.Context.unique_id(), 1, 0)
    T0 = meshgen.random_field(m, seed=3)
    ref = oracle.assemble(c, 1.0, 0.2, T0)
    mesh = P.Mesh(ctx, c)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    got = ldu.export()
    for k in ("diag", "upper", "source", "internal_coeffs", "boundary_coeffs"):
        assert np.array_equal(got[k], ref[k]), k
    x = meshgen.random_field(m, seed=7)
    o = oracle.OMesh(c)
    xr = np.zeros(o.n_bfaces)
    oracle.self_halo(c)(x, xr)
    y_ref = oracle.amul(c, ref["diag"], ref["upper"], x, ref["boundary_coeffs"], xr)
    # the same product on the undecomposed mesh (the cut is transparent)
    ref_full = oracle.assemble(m, 1.0, 0.2, T0)
    y_full = oracle.amul(m, ref_full["diag"], ref_full["upper"], x)
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    ldu.amul(xd, yd)
    y = yd.cpu().numpy()
    scale = np.abs(ref_full["diag"] * x) + 6 * np.abs(ref_full["upper"]).max() * np.abs(x).max()
    assert np.max(np.abs(y - y_ref) / scale) <= 1e-12
    assert np.max(np.abs(y - y_full) / scale) <= 1e-12
    mesh.close()
    ctx.close()


@pytest.mark.parametrize("use_nccl", [False, True])
def test_loopback_steps_equal_undecomposed(P, use_nccl):
    m, c = cut(12)
    s = meshgen.multimode_field(m)
    T_ref, _, p_ref = oracle.laplacian_foam(m, s, 4)
    ctx = P.Context(0)
    if use_nccl:
        ctx.comm_init(P.Context.unique_id(), 1, 0)
        assert ctx.comm_info() == (1, 0)
    mesh = P.Mesh(ctx, c)
    mesh.set_T(s)
    pg = mesh.step(4)
    T = mesh.get_T()
    assert np.max(np.abs(T - T_ref)) <= 1e-8 * np.max(np.abs(T_ref))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, p_ref))
    # standalone pcg_solve through the halo path
    ldu = mesh.assemble(1.0, 0.2)
    sy = oracle.assemble(c, 1.0, 0.2, T)
    x_ref, pr = oracle.pcg(c, sy, T, halo=oracle.self_halo(c))
    psi = torch.as_tensor(T.copy(), device="cuda")
    perf = ldu.pcg_solve(psi)
    assert abs(perf["n_iterations"] - pr["n_iterations"]) <= 1
    assert np.max(np.abs(psi.cpu().numpy() - x_ref)) <= 1e-8 * np.max(np.abs(x_ref))
    mesh.close()
    ctx.close()


def test_multiple_cuts_and_orders(P):
    """Two self pairs (z and x cuts) in one mesh."""
    m = meshgen.block_mesh(9, 8, 10)
    mask = decompose.z_plane_faces(m, 4)
    c = decompose.cut_mesh(m, mask)
    nx = 9
    xmask = (c.owner % nx == 4) & (c.neighbour == c.owner + 1)
    c2 = decompose.cut_mesh(c, xmask)
    s = meshgen.sine_field(m, k=(1, 2, 1))
    T_ref, _, _ = oracle.laplacian_foam(m, s, 3)
    ctx = P.Context(0)
    mesh = P.Mesh(ctx, c2)
    mesh.set_T(s)
    mesh.step(3)
    T = mesh.get_T()
    assert np.max(np.abs(T - T_ref)) <= 1e-8 * np.max(np.abs(T_ref))
    mesh.close()
    ctx.close()


def test_unpaired_processor_patch_rejected(P):
    m, c = cut(6)
    c.patches = c.patches[:-1]       # drop one side of the pair
    ctx = P.Context(0)
    with pytest.raises(P.LfoamError) as e:
        P.Mesh(ctx, c)
    assert e.value.status == 1
    ctx.close()


@pytest.mark.parametrize("overlap,graphs", [(True, True), (True, False), (False, True)])
def test_nccl_halo_overlap(P, overlap, graphs):
    """NCCL transport (1-rank communicator, self pairs): the w halo on the
    split communicator / comm stream, overlapped with the Amul phase of the
    cells without processor faces (LF_OPT_OVERLAP_HALO), CUDA-graph chunks or
    direct launches — against the undecomposed oracle, and the launch count
    (two phase-1 launches per iteration when overlapped)."""
    m, c = cut(12)
    s = meshgen.multimode_field(m)
    T_ref, _, p_ref = oracle.laplacian_foam(m, s, 4)
    ctx = P.Context(0)
    ctx.comm_init(P.Context.unique_id(), 1, 0)
    ctx.set_option("overlap_halo", overlap)
    ctx.set_option("graphs", graphs)
    mesh = P.Mesh(ctx, c)
    mesh.set_T(s)
    ctx.set_instrumentation(not graphs)
    pg = mesh.step(4)
    T = mesh.get_T()
    assert np.max(np.abs(T - T_ref)) <= 1e-8 * np.max(np.abs(T_ref))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, p_ref)), (pg, p_ref)
    if not graphs:
        n1, _ = ctx.kernel_stats("phase1")
        n2, _ = ctx.kernel_stats("phase2")
        assert (n1 >= 2 * n2) if overlap else (n1 < 2 * n2), (n1, n2)
    mesh.close()
    ctx.close()
