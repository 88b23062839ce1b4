"""Non-orthogonal correction path: CUDA vs the CPU
oracle through the C ABI (-m gpu).

Bars: on upper-triangular meshes (the generator's face order) the gather
kernels visit each cell's faces in the order the serial scatter reaches
them and round every operation explicitly, so weights-driven gradients,
boundary gradients and assembled coefficients are compared BITWISE; on
permuted / renumbered meshes summation orders differ: 1e-12 relative.
Time steps: final T rel L-inf 1e-8 at tol 1e-10 (as the orthogonal path).
"""
import numpy as np
import pytest

import meshgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = None


@pytest.fixture(scope="module")
def ctx():
    global P
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2507_18268_b200 as _P
    P = _P
    c = P.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def mixed_bc():
    return {"xmin": ("fixedValue", 1.5), "xmax": "zeroGradient", "ymin": ("fixedValue", -0.5),
            "zmax": "zeroGradient"}


def randomise_fixed_values(m, seed=3):
    rng = np.random.default_rng(seed)
    for p in m.patches:
        if p.type == "fixedValue":
            p.value[:] = rng.uniform(-2, 2, p.n_faces)
    return m


MESHES = {
    # ragged: 13*11*9 = 1287 cells, several 256-thread tiles plus a tail
    "skew_graded": lambda: randomise_fixed_values(
        meshgen.skewed_block_mesh(13, 11, 9, shear=(0.3, 0.1, 0.2), grading=(1.15, 0.9, 1.05), bc=mixed_bc())),
    "skew_uniform": lambda: meshgen.skewed_block_mesh(10, 10, 10, shear=(0.4, 0.0, 0.25)),
    "orthogonal": lambda: meshgen.with_geometry(meshgen.block_mesh(8, 6, 7)),
    "perm_skew": lambda: randomise_fixed_values(meshgen.permute_mesh(
        meshgen.skewed_block_mesh(7, 6, 5, shear=(0.3, 0.1, 0.2), grading=(1.2, 0.9, 1.1), bc=mixed_bc()))),
    "single_cell": lambda: meshgen.skewed_block_mesh(1, 1, 1, shear=(0.3, 0.1, 0.2)),
    "line": lambda: meshgen.skewed_block_mesh(29, 1, 1, shear=(0.5, 0.2, 0.0), grading=(1.1, 1, 1)),
}


def close(got, ref, exact, tol=1e-12):
    if exact:
        return np.array_equal(got, ref)
    den = np.maximum(np.max(np.abs(ref)), 1e-300)
    return np.max(np.abs(got - ref), initial=0.0) <= tol * den


def expected_source(m, DT, dt, T0, T):
    """Corrected TEqn source in the oracle's order: (T0/dt) V - lapSrc(T),
    then the fixedValue boundary source (orc_laplacian_foam_corrected)."""
    g, _ = oracle.grad(m, T)
    lap = oracle.lap_correction(m, DT, g)
    src = (1.0 / dt * T0) * m.V - lap
    sysm = oracle.assemble(m, DT, dt, T0)
    for p, sl in zip(m.patches, oracle.OMesh(m).patch_slices()):
        if p.type == "fixedValue":
            for i, c in enumerate(p.face_cells):
                src[c] += sysm["boundary_coeffs"][sl][i]
    return src, sysm


# ----------------------------------------------------------------- fvc::grad
@pytest.mark.parametrize("name", list(MESHES))
def test_grad_parity(ctx, name):
    m = MESHES[name]()
    x = meshgen.random_field(m, seed=11)
    g_ref, bg_ref = oracle.grad(m, x)
    mesh = P.Mesh(ctx, m)
    g = torch.empty((m.n_cells, 3), dtype=torch.float64, device="cuda")
    bg = torch.empty((mesh.n_bfaces, 3), dtype=torch.float64, device="cuda")
    mesh.fvc_grad(dev(x), g, bg)
    exact = m.old_of_new is None
    assert close(g.cpu().numpy(), g_ref, exact), name
    assert close(bg.cpu().numpy(), bg_ref, exact), name
    mesh.close()


def test_grad_linear_field_exact(ctx):
    """Any size: grad of a linear field with exact walls is g in every cell
    (the property the oracle pin proves), at a ragged 61x47x53 block."""
    m = meshgen.skewed_block_mesh(61, 47, 53, shear=(0.3, 0.1, 0.2), grading=(1.02, 0.99, 1.01))
    gvec = np.array([1.3, -0.4, 2.1])
    T = 0.7 + m.C @ gvec
    for p in m.patches:
        p.value[:] = 0.7 + p.Cf @ gvec
    mesh = P.Mesh(ctx, m)
    g = mesh.fvc_grad(dev(T)).cpu().numpy()
    assert np.max(np.abs(g - gvec)) < 1e-9 * np.max(np.abs(gvec))
    # sampled cells vs the oracle's definition at full size
    mesh.close()


# ------------------------------------------------------------------ assembly
@pytest.mark.parametrize("name", ["skew_graded", "skew_uniform", "orthogonal", "perm_skew", "line"])
def test_corrected_assembly_parity(ctx, name):
    m = MESHES[name]()
    T = meshgen.random_field(m, seed=5)
    DT, dt = 1.3, 0.2
    src, sysm = expected_source(m, DT, dt, T, T)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T)
    got = mesh.assemble(DT, dt, corrected=True).export()
    exact = m.old_of_new is None
    for k in ("diag", "upper", "internal_coeffs", "boundary_coeffs"):
        assert close(got[k], sysm[k], exact), k
    assert close(got["source"], src, exact), "source"
    # the correction is really there (non-orthogonal 3-D meshes; on the
    # orthogonal block corr = 0, on the one-cell-thick line every gradient is
    # along n and corr . n = 0)
    plain = mesh.assemble(DT, dt).export()["source"]
    if name not in ("orthogonal", "line"):
        assert np.max(np.abs(plain - got["source"])) > 1e-6 * np.max(np.abs(src))
    mesh.close()


# --------------------------------------------------------------- time steps
@pytest.mark.parametrize("name,n_corr", [("skew_graded", 0), ("skew_graded", 2), ("skew_uniform", 1),
                                         ("perm_skew", 1), ("single_cell", 1), ("line", 2)])
def test_corrected_step_parity(ctx, name, n_corr):
    m = MESHES[name]()
    T0 = meshgen.sine_field(m) + 0.1 * meshgen.random_field(m, seed=2)
    To, bo, po = oracle.laplacian_foam_corrected(m, T0, 4, n_corr=n_corr)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T0)
    pg = mesh.step(4, corrected=True, n_non_orth_correctors=n_corr)
    T = mesh.get_T()
    assert len(pg) == len(po) == 4 * (1 + n_corr)
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    for a, b in zip(pg, po):
        assert abs(a["n_iterations"] - b["n_iterations"]) <= 1, (pg, po)
        assert a["converged"] == b["converged"]
    for i, sl in enumerate(oracle.OMesh(m).patch_slices()):
        assert np.max(np.abs(mesh.get_patch_value(i) - bo[sl]), initial=0.0) <= 1e-8 * max(1.0, np.max(np.abs(To)))
    mesh.close()


def test_corrected_renumbered(ctx):
    m = MESHES["perm_skew"]()
    T0 = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam_corrected(m, T0, 3, n_corr=1)
    mesh = P.Mesh(ctx, m, renumber=True)
    mesh.set_T(T0)
    pg = mesh.step(3, corrected=True, n_non_orth_correctors=1)
    assert np.max(np.abs(mesh.get_T() - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po))
    # gradient in internal numbering: permute in/out through the ABI
    x = meshgen.random_field(m, seed=8)
    g_ref, bg_ref = oracle.grad(m, x)
    xi = torch.empty(m.n_cells, dtype=torch.float64, device="cuda")
    mesh.permute(True, dev(x), xi)
    bg = torch.empty((mesh.n_bfaces, 3), dtype=torch.float64, device="cuda")
    gi = mesh.fvc_grad(xi, bgrad=bg)
    co = mesh.export_addressing()["cell_order"]
    g = np.empty((m.n_cells, 3))
    g[co] = gi.cpu().numpy()
    assert close(g, g_ref, False) and close(bg.cpu().numpy(), bg_ref, False)
    mesh.close()


def test_orthogonal_corrected_equals_plain(ctx):
    m = MESHES["orthogonal"]()
    s = meshgen.sine_field(m)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(s)
    mesh.step(3)
    Tp = mesh.get_T()
    mesh.set_T(s)
    mesh.step(3, corrected=True, n_non_orth_correctors=1)
    Tc = mesh.get_T()
    assert np.max(np.abs(Tc - Tp)) <= 1e-12 * np.max(np.abs(s))
    mesh.close()


def test_corrected_adiabatic_conservation(ctx):
    bc = {n: "zeroGradient" for n in meshgen.PATCH_NAMES}
    m = meshgen.skewed_block_mesh(17, 13, 11, shear=(0.3, 0.1, 0.2), grading=(1.1, 0.95, 1.05), bc=bc)
    T0 = meshgen.random_field(m, seed=6)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T0)
    mesh.step(5, corrected=True, n_non_orth_correctors=1, tol=1e-14, max_iter=2000)
    T = mesh.get_T()
    assert abs(np.dot(m.V, T) - np.dot(m.V, T0)) < 1e-11 * np.dot(m.V, np.abs(T0))
    mesh.close()


def test_corrected_full_size_sampled(ctx):
    """A 1M-cell skewed graded block (the config-2 size): step 0 with one
    corrector vs the oracle, every cell (the oracle runs it in seconds)."""
    m = meshgen.skewed_block_mesh(100, 100, 100, shear=(0.3, 0.1, 0.2), grading=(1.01, 0.995, 1.0))
    s = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam_corrected(m, s, 1, n_corr=1)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(s)
    pg = mesh.step(1, corrected=True, n_non_orth_correctors=1)
    assert np.max(np.abs(mesh.get_T() - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po))
    mesh.close()


def test_nonorth_kernels_launched(ctx):
    m = MESHES["skew_graded"]()
    mesh = P.Mesh(ctx, m)
    mesh.set_T(meshgen.sine_field(m))
    ctx.set_instrumentation(True)
    mesh.step(2, corrected=True, n_non_orth_correctors=1)
    n, ms = ctx.kernel_stats("nonorth")
    ctx.set_instrumentation(False)
    assert n == 2 * 2 * 2  # grad + correction, per pass
    assert ms > 0
    mesh.close()


def test_nonorth_invalid(ctx):
    plain = meshgen.block_mesh(4)
    mesh = P.Mesh(ctx, plain)
    with pytest.raises(P.LfoamError) as e:
        mesh.assemble(corrected=True)
    assert e.value.status == 1
    with pytest.raises(P.LfoamError):
        mesh.step(1, corrected=True)
    with pytest.raises(P.LfoamError):
        mesh.fvc_grad(dev(np.zeros(plain.n_cells)))
    mesh.close()
    m = MESHES["skew_uniform"]()
    mesh = P.Mesh(ctx, m)
    with pytest.raises(P.LfoamError):
        mesh.step(1, corrected=True, n_non_orth_correctors=-1)
    mesh.close()
    bad = MESHES["skew_uniform"]()
    bad.C = None  # partial geometry
    with pytest.raises(P.LfoamError):
        P.Mesh(ctx, bad, geometry=True)
