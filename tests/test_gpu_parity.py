"""CUDA path vs the CPU oracle, element by element, through the C ABI (-m gpu).

Tolerances (north_star / SURVEY §8(c.4)): coefficients and one Amul 1e-12
relative (row-scaled for Amul), final T rel L-inf 1e-8 at tol 1e-10,
iterations within +-1; integer addressing bit-exact.
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


def zg_all():
    return {n: "zeroGradient" for n in meshgen.cube.PATCH_NAMES}


def mixed_bc():
    return {"xmin": ("fixedValue", 1.5), "xmax": "zeroGradient", "ymin": ("fixedValue", -0.5),
            "zmax": "zeroGradient"}


def randomise_fixed_values(m, seed=3):
    rng = np.random.default_rng(seed)
    for p in m.patches:
        if p.type == "fixedValue":
            p.value[:] = rng.uniform(-2, 2, p.n_faces)
    return m


def row_scale(m, diag, upper, x):
    s = np.abs(diag * x)
    np.add.at(s, m.owner, np.abs(upper * x[m.neighbour]))
    np.add.at(s, m.neighbour, np.abs(upper * x[m.owner]))
    return s


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


MESHES = {
    "cube10": lambda: randomise_fixed_values(meshgen.block_mesh(10)),
    "box_mixed": lambda: randomise_fixed_values(meshgen.block_mesh(7, 5, 4, extent=(1.0, 0.6, 1.3), bc=mixed_bc())),
    "perm6": lambda: randomise_fixed_values(meshgen.permute_mesh(meshgen.block_mesh(6, bc=mixed_bc()))),
    "single_cell": lambda: meshgen.block_mesh(1),
    "line": lambda: meshgen.block_mesh(37, 1, 1),
}


# --------------------------------------------------------------- addressing
@pytest.mark.parametrize("name", ["cube10", "perm6", "line", "single_cell"])
@pytest.mark.parametrize("renumber", [False, True])
def test_addressing_bitexact(ctx, name, renumber):
    m = MESHES[name]()
    mesh = P.Mesh(ctx, m, renumber=renumber)
    a = mesh.export_addressing()
    co, fo = a["cell_order"], a["face_order"]
    inv = np.empty_like(co)
    inv[co] = np.arange(m.n_cells, dtype=co.dtype)
    lo = np.minimum(inv[m.owner], inv[m.neighbour])[fo]
    hi = np.maximum(inv[m.owner], inv[m.neighbour])[fo]
    # internal faces upper-triangular: sorted by (owner, neighbour)
    key = lo.astype(np.int64) * m.n_cells + hi
    assert np.all(np.diff(key) >= 0)
    assert np.array_equal(np.sort(fo), np.arange(m.n_faces))
    items, starts = oracle.group(lo, m.n_cells)
    assert np.array_equal(items, np.arange(m.n_faces))
    assert np.array_equal(a["owner_start"], starts)
    items, starts = oracle.group(hi, m.n_cells)
    assert np.array_equal(a["losort"], items)
    assert np.array_equal(a["losort_start"], starts)
    if not renumber:
        assert np.array_equal(co, np.arange(m.n_cells))
    mesh.close()


# ----------------------------------------------------------------- assembly
@pytest.mark.parametrize("name", ["cube10", "box_mixed", "perm6", "single_cell", "line"])
def test_assembly_parity(ctx, name):
    m = MESHES[name]()
    T0 = meshgen.random_field(m, seed=9)
    DT, dt = 1.3, 0.2
    ref = oracle.assemble(m, DT, dt, T0)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T0)
    got = mesh.assemble(DT, dt).export()
    exact = m.old_of_new is None  # upper-triangular input: same op order as the definition
    for k in ("diag", "upper", "source", "internal_coeffs", "boundary_coeffs"):
        if exact:
            assert np.array_equal(got[k], ref[k]), k
        else:
            den = np.maximum(np.abs(ref[k]), 1e-300)
            assert np.max(np.abs(got[k] - ref[k]) / den, initial=0.0) <= 1e-12, k
    mesh.close()


def test_assembly_renumbered(ctx):
    m = MESHES["perm6"]()
    T0 = meshgen.random_field(m, seed=2)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    mesh = P.Mesh(ctx, m, renumber=True)
    mesh.set_T(T0)
    got = mesh.assemble(1.0, 0.2).export()
    for k in ("diag", "upper", "source"):
        assert np.max(np.abs(got[k] - ref[k]) / np.abs(ref[k])) <= 1e-12, k
    np.testing.assert_array_equal(mesh.get_T(), T0)
    mesh.close()


# --------------------------------------------------------------------- Amul
@pytest.mark.parametrize("name", ["cube10", "box_mixed", "perm6", "line"])
def test_amul_parity(ctx, name):
    m = MESHES[name]()
    T0 = meshgen.random_field(m, seed=1)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    x = meshgen.random_field(m, seed=5)
    y_ref = oracle.amul(m, ref["diag"], ref["upper"], x)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    xd = dev(x)
    yd = torch.empty_like(xd)
    ldu.amul(xd, yd)
    y = yd.cpu().numpy()
    assert np.max(np.abs(y - y_ref) / row_scale(m, ref["diag"], ref["upper"], x)) <= 1e-12
    mesh.close()


@pytest.mark.parametrize("N", [100, 200])
def test_amul_eigenmode_full_size(ctx, N):
    """A s = mu s at the bench sizes (no oracle needed: closed form)."""
    m = meshgen.block_mesh(N)
    s = meshgen.sine_field(m)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(s)
    ldu = mesh.assemble(1.0, 0.2)
    sd = dev(s)
    yd = torch.empty_like(sd)
    ldu.amul(sd, yd)
    h = 1.0 / N
    lam = 3 * 4 * np.sin(np.pi * h / 2) ** 2 / h ** 2
    mu = h ** 3 / 0.2 + h ** 3 * lam
    scale = np.abs(s) * (h ** 3 / 0.2 + 12 * h)   # |diag s| + sum |upper s_nb| ~ 2*6h|s|
    err = np.abs(yd.cpu().numpy() - mu * s)
    assert np.max(err / np.maximum(scale, 1e-300)) <= 1e-12
    mesh.close()


# ---------------------------------------------------------------------- PCG
@pytest.mark.parametrize("name", ["cube10", "box_mixed", "perm6"])
def test_pcg_parity(ctx, name):
    m = MESHES[name]()
    T0 = meshgen.random_field(m, seed=4)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    x_ref, p_ref = oracle.pcg(m, ref, T0)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    psi = dev(T0)
    perf = ldu.pcg_solve(psi)
    x = psi.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref)) <= 1e-8
    assert abs(perf["n_iterations"] - p_ref["n_iterations"]) <= 1
    assert perf["converged"] == p_ref["converged"] == 1
    assert abs(perf["initial_residual"] - p_ref["initial_residual"]) <= 1e-10 * p_ref["initial_residual"]
    mesh.close()


def test_pcg_controls(ctx):
    m = meshgen.block_mesh(8)
    T0 = meshgen.sine_field(m)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    for kw in [dict(max_iter=3), dict(min_iter=40), dict(tol=0.0, rel_tol=1e-3), dict(max_iter=0)]:
        x_ref, p_ref = oracle.pcg(m, ref, T0, **kw)
        psi = dev(T0)
        perf = ldu.pcg_solve(psi, **kw)
        assert perf["n_iterations"] == p_ref["n_iterations"], kw
        assert perf["converged"] == p_ref["converged"], kw
        assert np.max(np.abs(psi.cpu().numpy() - x_ref)) <= 1e-8 * np.max(np.abs(x_ref)), kw
    mesh.close()


def test_pcg_zero_rhs_zero_iterations(ctx):
    """b = 0, x0 = 0 -> 0 iterations (T0 = 0, walls 0)."""
    m = meshgen.block_mesh(6)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(np.zeros(m.n_cells))
    perfs = mesh.step(2)
    assert all(p["n_iterations"] == 0 and p["converged"] for p in perfs)
    assert np.all(mesh.get_T() == 0.0)
    mesh.close()


# -------------------------------------------------------------- full steps
@pytest.mark.parametrize("name", ["cube10", "box_mixed", "perm6", "single_cell", "line"])
def test_step_parity(ctx, name):
    m = MESHES[name]()
    T0 = meshgen.sine_field(m) if name != "single_cell" else np.array([0.3])
    To, bo, po = oracle.laplacian_foam(m, T0, 5)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T0)
    pg = mesh.step(5)
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    for a, b in zip(pg, po):
        assert abs(a["n_iterations"] - b["n_iterations"]) <= 1, (pg, po)
        assert a["converged"] == b["converged"]
    o = oracle.OMesh(m)
    for i, sl in enumerate(o.patch_slices()):
        got = mesh.get_patch_value(i)
        assert np.max(np.abs(got - bo[sl]), initial=0.0) <= 1e-8 * max(1.0, np.max(np.abs(To)))
    mesh.close()


def test_config1_parity_and_closed_form(ctx, canonical_constants):
    """BASELINE config 1: 10^3, 10 steps, tol 1e-10 vs oracle and g^10 s."""
    m = meshgen.block_mesh(10)
    s = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam(m, s, 10)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(s)
    pg = mesh.step(10)
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po))
    g = canonical_constants["rows"][0]["g"]
    assert np.max(np.abs(T - g ** 10 * s)) <= 1e-8 * np.max(np.abs(g ** 10 * s))
    mesh.close()


def test_config2_two_steps_full_field(ctx):
    """BASELINE config 2 mesh (1M cells), first 2 steps vs the oracle, every cell."""
    m = meshgen.block_mesh(100)
    s = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam(m, s, 2)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(s)
    pg = mesh.step(2)
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po))
    mesh.close()


def test_config2_full_run_closed_form(ctx, canonical_constants):
    """The bench workload (100^3, 100 steps) vs T^100 = g^100 s (any size)."""
    row = [r for r in canonical_constants["rows"] if r["N"] == 100][0]
    m = meshgen.block_mesh(100)
    s = meshgen.canonical_field(m)     # amplitude 1e80 (reading A30)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(s)
    pg = mesh.step(100)
    T = mesh.get_T()
    ref = row["g"] ** 100 * s
    assert np.max(np.abs(T - ref)) <= 1e-8 * np.max(np.abs(ref))
    its = [p["n_iterations"] for p in pg]
    assert all(p["converged"] for p in pg)
    assert 90 <= min(its) and max(its) <= 130, its   # SCRATCH 96-97 early on (indicative)
    mesh.close()


@pytest.mark.slow
def test_config2_full_run_vs_oracle(ctx):
    """Config 2 exactly as bench.py times it (100^3, 100 steps, canonical
    field) against the oracle: every cell and every step's iteration count."""
    m = meshgen.block_mesh(100)
    s = meshgen.canonical_field(m)
    To, _, po = oracle.laplacian_foam(m, s, 100)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(s)
    pg = mesh.step(100)
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    check_iterations(pg, po, tol=1e-10)
    mesh.close()


def check_iterations(pg, po, tol):
    """Iterations within +-1 per step, except criterion flips: OpenFOAM's L1
    residual is not monotone in CG, so when one side stops with a residual
    within 10% below tol the other side may need to ride out a bump
    (observed 97 vs 109 at 100^3).  Such a step and the one after it (which
    starts from a slightly different T) are exempt; totals must agree to 2%."""
    flip = [max(a["final_residual"], b["final_residual"]) >= 0.9 * tol for a, b in zip(pg, po)]
    bad = []
    for i, (a, b) in enumerate(zip(pg, po)):
        exempt = flip[i] or (i > 0 and flip[i - 1])
        if abs(a["n_iterations"] - b["n_iterations"]) > 1 and not exempt:
            bad.append((i, a["n_iterations"], b["n_iterations"]))
    assert not bad, bad
    tg = sum(p["n_iterations"] for p in pg)
    to = sum(p["n_iterations"] for p in po)
    assert abs(tg - to) <= max(2, 0.02 * to), (tg, to)


@pytest.mark.parametrize("mode", ["graphs", "direct"])
def test_loop_modes_agree(mode):
    """Persistent cooperative kernel vs per-phase launches (graph / direct):
    same algorithm, different reduction grids -> equal within tolerance."""
    import paper_2507_18268_b200 as _P
    m = meshgen.block_mesh(24, 20, 16, bc=mixed_bc())
    s = meshgen.multimode_field(m)
    To, _, po = oracle.laplacian_foam(m, s, 4)
    c = _P.Context(0)
    c.set_option("persistent", False)
    c.set_option("graphs", mode == "graphs")
    mesh = _P.Mesh(c, m)
    mesh.set_T(s)
    pg = mesh.step(4)
    assert np.max(np.abs(mesh.get_T() - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po))
    n_phase1, _ = c.kernel_stats("phase1")
    n_pcg, _ = c.kernel_stats("pcg")
    assert n_phase1 > 0 and n_pcg == 0
    c.close()


def test_determinism_bitwise(ctx):
    m = meshgen.block_mesh(30)
    s = meshgen.multimode_field(m)
    out = []
    for _ in range(2):
        mesh = P.Mesh(ctx, m)
        mesh.set_T(s)
        pg = mesh.step(3)
        out.append((mesh.get_T(), [p["n_iterations"] for p in pg]))
        mesh.close()
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]


def test_hot_plate_and_zero_gradient_values(ctx):
    m = meshgen.hot_plate(20)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(np.zeros(m.n_cells))
    mesh.step(40)
    T = mesh.get_T()
    x = m.cell_centres()[:, 0]
    assert np.max(np.abs(T - (1 - x))) < 1e-8
    np.testing.assert_array_equal(mesh.get_patch_value(2), T[m.patches[2].face_cells])
    np.testing.assert_array_equal(mesh.get_patch_value(0), 1.0)
    mesh.close()


def test_adiabatic_conservation(ctx):
    m = meshgen.block_mesh(10, bc=zg_all())
    T = meshgen.cosine_field(m, k=(1, 2, 0), offset=1.0)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T)
    for _ in range(6):
        mesh.step(1)
        T1 = mesh.get_T()
        assert abs((m.V * T1).sum() - (m.V * T).sum()) <= 1e-9 * (m.V * np.abs(T)).sum()
        T = T1
    mesh.close()


def test_renumbered_step_parity(ctx):
    """BASELINE config 5 shape (permuted numbering) at 12^3, renumber 0 and 1."""
    m = meshgen.permute_mesh(meshgen.block_mesh(12))
    s = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam(m, s, 4)
    for rn in (False, True):
        mesh = P.Mesh(ctx, m, renumber=rn)
        mesh.set_T(s)
        pg = mesh.step(4)
        T = mesh.get_T()
        assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To)), rn
        assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po))
        mesh.close()


def test_invalid_arguments(ctx):
    m = meshgen.block_mesh(3)
    bad = meshgen.block_mesh(3)
    bad.neighbour = bad.neighbour.copy()
    bad.neighbour[0] = bad.owner[0]
    with pytest.raises(P.LfoamError) as e:
        P.Mesh(ctx, bad)
    assert e.value.status == 1
    bad2 = meshgen.block_mesh(3)
    bad2.V = bad2.V.copy()
    bad2.V[3] = 0.0
    with pytest.raises(P.LfoamError):
        P.Mesh(ctx, bad2)
    mesh = P.Mesh(ctx, m)
    with pytest.raises(P.LfoamError) as e:
        mesh.assemble(DT=-1.0)
    assert e.value.status == 1
    with pytest.raises(P.LfoamError):
        mesh.set_T(np.zeros(5))
    mesh.close()


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("dims", [(10, 10, 10), (37, 23, 19), (7, 5, 4), (64, 32, 24)])
def test_solve_variants(ctx, variant, dims):
    """The persistent solve's L2-resident variant (psi update in the beta-
    barrier wait) and HBM-bound variant (psi update deferred into the Amul
    phase), forced on meshes of several sizes and ragged tails, against the
    oracle."""
    c = P.Context(0)
    c.set_option("variant", variant)
    m = randomise_fixed_values(meshgen.block_mesh(*dims, bc=mixed_bc()))
    T0 = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam(m, T0, 4)
    mesh = P.Mesh(c, m)
    mesh.set_T(T0)
    pg = mesh.step(4)
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    # pcg_solve from a standalone assembly through the same variant
    x_ref, p_ref = oracle.pcg(m, oracle.assemble(m, 1.0, 0.2, T), T)
    ldu = mesh.assemble(1.0, 0.2)
    psi = dev(T)
    perf = ldu.pcg_solve(psi)
    assert np.max(np.abs(psi.cpu().numpy() - x_ref)) <= 1e-8 * np.max(np.abs(x_ref))
    assert abs(perf["n_iterations"] - p_ref["n_iterations"]) <= 1
    mesh.close()
    c.close()


def k4_mesh(n=9):
    """A block mesh plus one extra 'diagonal' internal face per cell
    ((i,j,k)-(i+1,j+1,k)): up to 4 owned and 4 neighbour-side faces per cell,
    so the 4-slot ELL kernels run (hex meshes use 3 slots; permuted meshes
    the CSR gather).  Any LDU mesh with positive coefficients is a valid
    input of the method (SPD, diagonally dominant)."""
    import dataclasses
    m = meshgen.block_mesh(n, bc=mixed_bc())
    c = np.arange(m.n_cells)
    i, j = c % n, (c // n) % n
    sel = (i < n - 1) & (j < n - 1)
    o = c[sel].astype(np.int32)
    nb = (o + 1 + n).astype(np.int32)
    owner = np.concatenate([m.owner, o])
    neighbour = np.concatenate([m.neighbour, nb])
    key = np.lexsort((neighbour, owner))
    h = 1.0 / n
    extra = np.full(o.shape[0], 0.5 * h * h)
    return dataclasses.replace(m, owner=owner[key], neighbour=neighbour[key],
                               mag_sf=np.concatenate([m.mag_sf, extra])[key],
                               delta=np.concatenate([m.delta, np.full(o.shape[0], 1.0 / (h * np.sqrt(2.0)))])[key])


@pytest.mark.parametrize("variant", [1, 2])
def test_k4_ell_mesh(ctx, variant):
    c = P.Context(0)
    c.set_option("variant", variant)
    m = k4_mesh()
    T0 = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam(m, T0, 3)
    mesh = P.Mesh(c, m)
    mesh.set_T(T0)
    pg = mesh.step(3)
    assert np.max(np.abs(mesh.get_T() - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    ref = oracle.assemble(m, 1.0, 0.2, mesh.get_T())
    ldu = mesh.assemble(1.0, 0.2)
    got = ldu.export()
    assert np.array_equal(got["diag"], ref["diag"]) and np.array_equal(got["upper"], ref["upper"])
    x = meshgen.random_field(m, seed=5)
    y = ldu.amul(dev(x), dev(np.zeros(m.n_cells))).cpu().numpy()
    y_ref = oracle.amul(m, ref["diag"], ref["upper"], x)
    assert np.max(np.abs(y - y_ref) / row_scale(m, ref["diag"], ref["upper"], x)) <= 1e-12
    mesh.close()
    c.close()


def test_constant_field_A29(ctx):
    """Reading A29: T = T_b everywhere is the exact solution; normFactor
    collapses to ~1e-20, so the normalised residual is rounding noise and PCG
    may iterate (to max_iter) — checked through the field and A.1 directly,
    not through iteration counts."""
    N = 10
    m = meshgen.block_mesh(N, bc={n: ("fixedValue", 1.0) for n in meshgen.cube.PATCH_NAMES})
    mesh = P.Mesh(ctx, m)
    mesh.set_T(np.ones(m.n_cells))
    perfs = mesh.step(2, max_iter=50)
    assert np.max(np.abs(mesh.get_T() - 1.0)) <= 1e-12
    assert all(p["n_iterations"] <= 50 for p in perfs)
    # A.1 = V/dt + sum of the fixedValue boundary coefficients of the row
    ldu = mesh.assemble(1.0, 0.2)
    y = ldu.amul(dev(np.ones(m.n_cells)), dev(np.zeros(m.n_cells))).cpu().numpy()
    h = 1.0 / N
    nbf = np.zeros(m.n_cells)
    for p in m.patches:
        np.add.at(nbf, p.face_cells, 1.0)
    expect = h ** 3 / 0.2 + nbf * (1.0 * h * h * 2.0 / h)
    assert np.max(np.abs(y - expect) / expect) <= 1e-13
    mesh.close()
