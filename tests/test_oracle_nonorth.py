"""Pins for the oracle's non-orthogonal correction path (
-m "not gpu").

What fixes each expected value:
  * SPEC worked examples (tests/golden/spec_examples.json "weights",
    "interpolate", "grad_bc"), evaluated on hand-built one/two-cell meshes;
  * Green-Gauss exactness for linear fields on planar-faced cells whose
    owner-neighbour line passes through the face centre (the sheared, graded
    block: every such line runs along one mapped grid direction), checked
    against the field's own gradient g;
  * the corrected face flux is exact for linear fields
    (delta (T_N - T_P) + (n - delta d).g = n.g), so the full discrete
    laplacian of a linear field vanishes in every interior cell — and does
    NOT without the correction (the test sees the term matter);
  * orthogonal meshes: the correction vectors vanish, corrected == plain;
  * conservation with zeroGradient walls (the correction is a flux
    difference: sum over cells is zero);
  * geometry recomputed from points/faces (oracle.geometry) for Sf, C, Cf.
"""
import numpy as np
import pytest

import meshgen
import oracle
from oracle import geometry


def linear_field(m, a=0.7, g=(1.3, -0.4, 2.1)):
    g = np.asarray(g, float)
    T = a + m.C @ g
    for p in m.patches:
        if p.type == "fixedValue":
            p.value[:] = a + p.Cf @ g
    return T, g


def two_cell(Sf, C_own, C_nei, Cf, V=(1.0, 1.0)):
    Sf = np.array([Sf], float)
    return meshgen.Mesh(2, np.array([0], np.int32), np.array([1], np.int32),
                        np.linalg.norm(Sf, axis=1), np.ones(1), np.array(V, float), [],
                        dims=(2, 1, 1), Sf=Sf, Cf=np.array([Cf], float), C=np.array([C_own, C_nei], float))


# ------------------------------------------------------ worked examples
def test_weights_spec_example(spec_examples):
    ex = spec_examples["weights"][0]
    m = two_cell(ex["Sf"], ex["C_own"], ex["C_nei"], ex["Cf"])
    assert oracle.weights(m)[0] == ex["w"]
    co = spec_examples["weights"][1]
    m = two_cell([1, 0, 0], [0.5, 0, 0], [0.5, 0, 0], [0.5, 0, 0])
    assert oracle.weights(m)[0] == co["w"]


def test_interpolation_spec_examples(spec_examples):
    """Face value lambda (x_P - x_N) + x_N seen through the gradient of a
    two-cell mesh with one face: grad_P = Sf * x_f / V_P."""
    for ex in spec_examples["interpolate"]:
        w = ex["w"]
        # geometry with SfdNei / (SfdOwn + SfdNei) = w: Cf at 1 - w between C_P = 0 and C_N = 1
        m = two_cell([1, 0, 0], [0, 0, 0], [1, 0, 0], [1 - w, 0, 0])
        assert oracle.weights(m)[0] == w
        g, _ = oracle.grad(m, np.array([ex["v_owner"], ex["v_neighbour"]]))
        assert g[0, 0] == ex["face"] and g[1, 0] == -ex["face"]
        assert np.all(g[:, 1:] == 0)


def test_grad_bc_spec_examples(spec_examples):
    """One cell, V = 1: a fixedValue face Sf = (0,0,1) (value T_b) and a
    zeroGradient face Sf = (1,0,0) give grad = (x, 0, T_b); snGrad =
    delta (T_b - x).  Listing CorrectBoundaryConditions."""
    for ex in spec_examples["grad_bc"]:
        gb, sng = np.array(ex["gb"], float), ex["snGrad"]
        x, Tb = gb[0], gb[2]
        delta = sng / (Tb - x)
        pf = meshgen.Patch("top", "fixedValue", np.array([0], np.int32), np.ones(1), np.array([delta]),
                           np.array([Tb]), Sf=np.array([[0.0, 0.0, 1.0]]))
        pz = meshgen.Patch("side", "zeroGradient", np.array([0], np.int32), np.ones(1), np.ones(1),
                           np.zeros(1), Sf=np.array([[1.0, 0.0, 0.0]]))
        m = meshgen.Mesh(1, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros(0),
                         np.ones(1), [pf, pz], dims=(1, 1, 1), Sf=np.zeros((0, 3)), Cf=np.zeros((0, 3)),
                         C=np.zeros((1, 3)))
        g, bg = oracle.grad(m, np.array([x]))
        assert np.array_equal(g[0], gb)
        assert np.array_equal(bg[0], np.array(ex["out"], float))
        # zeroGradient face: normal component removed, tangential kept
        assert np.array_equal(bg[1], np.array([0.0, 0.0, gb[2]]))


def test_grad_bc_fixed_point():
    """snGrad = n.gb leaves gb unchanged (orthogonal graded block,
    linear field: d || n on every wall, so snGrad = n.g exactly)."""
    m = meshgen.skewed_block_mesh(5, 4, 3, shear=(0, 0, 0), grading=(1.3, 0.8, 1.1))
    T, gvec = linear_field(m)
    _, bg = oracle.grad(m, T)
    assert np.max(np.abs(bg - gvec)) < 1e-11 * np.max(np.abs(gvec))


# ------------------------------------------------------------- geometry
@pytest.mark.parametrize("shear,grading", [((0.3, 0.0, 0.2), (1.0, 1.0, 1.0)),
                                           ((0.3, 0.1, 0.2), (1.25, 0.85, 1.1))])
def test_skewed_geometry_from_points(shear, grading):
    """The closed-form geometry of skewed_block_mesh equals the geometry
    recomputed from its points and faces (triangle decomposition)."""
    m = meshgen.skewed_block_mesh(4, 3, 5, shear=shear, grading=grading)
    pts, faces = meshgen.mesh_points_faces(m)
    g = geometry.mesh_geometry(m, pts, faces)
    F = m.n_faces
    assert np.max(np.abs(g["Sf"][:F] - m.Sf)) < 1e-13
    assert np.max(np.abs(g["Cf"][:F] - m.Cf)) < 1e-13
    assert np.max(np.abs(g["C"] - m.C)) < 1e-13
    assert np.max(np.abs(g["V"] - m.V)) < 1e-15
    bsf = np.concatenate([p.Sf for p in m.patches])
    assert np.max(np.abs(g["Sf"][F:] - bsf)) < 1e-13


def test_weights_graded():
    """On a graded block the weight of an x-face is h_{i+1} / (h_i + h_{i+1})
    (SfdNei/(SfdOwn+SfdNei) with SfdOwn = |Sf| h_i/2, SfdNei = |Sf| h_{i+1}/2),
    shear-invariant (Sf.(A u) = det A (A^-T Sf0).(A u) = Sf0.u)."""
    m = meshgen.skewed_block_mesh(6, 1, 1, shear=(0.3, 0.1, 0.2), grading=(1.4, 1, 1))
    h = np.diff(m.grid_lines[0])
    w = oracle.weights(m)
    expect = h[1:] / (h[:-1] + h[1:])
    assert np.max(np.abs(w - expect)) < 1e-14
    assert not np.allclose(w, 0.5)


def test_corr_vectors_orthogonal_zero():
    m = meshgen.with_geometry(meshgen.block_mesh(4, 3, 2))
    cv = oracle.corr_vectors(m)
    assert np.max(np.abs(cv)) < 1e-14


def test_corr_vectors_orthogonal_to_d():
    """n - delta d with delta = 1/(n.d): (n - delta d).n = 1 - 1 = 0 ... on
    the plane of the face, i.e. corr . n = 0 whenever n.d >= 0.05|d|."""
    m = meshgen.skewed_block_mesh(4, 4, 4, shear=(0.3, 0.1, 0.2), grading=(1.2, 1, 0.9))
    cv = oracle.corr_vectors(m)
    n = m.Sf / m.mag_sf[:, None]
    assert np.max(np.abs(np.einsum("ij,ij->i", cv, n))) < 1e-14
    assert np.max(np.abs(cv)) > 0.1  # genuinely non-orthogonal


# -------------------------------------------------------------- gradient
@pytest.mark.parametrize("shear,grading", [((0, 0, 0), (1, 1, 1)), ((0.3, 0.0, 0.2), (1, 1, 1)),
                                           ((0.3, 0.1, 0.2), (1.25, 0.85, 1.1))])
def test_grad_linear_exact(shear, grading):
    """Green-Gauss + linear interpolation reproduces g for T = a + g.x with
    exact fixedValue walls (S:328 'exact for linear fields')."""
    m = meshgen.skewed_block_mesh(5, 4, 6, shear=shear, grading=grading)
    T, gvec = linear_field(m)
    g, _ = oracle.grad(m, T)
    assert np.max(np.abs(g - gvec)) < 1e-10 * np.max(np.abs(gvec))


def test_grad_constant_zero():
    """grad of a constant is zero (closure), zeroGradient walls."""
    bc = {n: "zeroGradient" for n in meshgen.PATCH_NAMES}
    m = meshgen.skewed_block_mesh(4, 5, 3, shear=(0.3, 0.1, 0.2), grading=(1.2, 0.9, 1.1), bc=bc)
    g, bg = oracle.grad(m, np.full(m.n_cells, 3.5))
    scale = 3.5 * np.max(np.abs(m.Sf)) / np.min(m.V)
    assert np.max(np.abs(g)) < 1e-13 * scale and np.max(np.abs(bg)) < 1e-13 * scale


def test_grad_bc_closed_form_skewed():
    """Skewed fixedValue walls, linear field (cell gradient exact): gb = g +
    n (g.d/(n.d) - n.g), d = Cf - C, since snGrad = deltaCoeffs (T_b - T_c)
    with deltaCoeffs = 1/(n.d) (nonOrthDeltaCoeffs; n.d >= 0.05|d| here)."""
    m = meshgen.skewed_block_mesh(4, 3, 5, shear=(0.3, 0.1, 0.2), grading=(1.1, 0.9, 1.2))
    T, gvec = linear_field(m)
    _, bg = oracle.grad(m, T)
    exp = []
    for p in m.patches:
        n = p.Sf / p.mag_sf[:, None]
        d = p.Cf - m.C[p.face_cells]
        sn = (d @ gvec) / np.einsum("ij,ij->i", n, d)
        exp.append(gvec + n * (sn - n @ gvec)[:, None])
    exp = np.concatenate(exp)
    assert np.max(np.abs(bg - exp)) < 1e-10 * np.max(np.abs(gvec))
    assert np.max(np.abs(bg - gvec)) > 0.1  # the correction acts on skewed walls


def test_grad_bc_zero_gradient_walls():
    """zeroGradient walls: the corrected boundary gradient has no normal
    component and keeps the cell gradient's tangential part."""
    bc = {"xmin": "zeroGradient", "ymax": "zeroGradient"}
    m = meshgen.skewed_block_mesh(4, 3, 5, shear=(0.3, 0.1, 0.2), grading=(1.1, 0.9, 1.2), bc=bc)
    T, _ = linear_field(m)
    g, bg = oracle.grad(m, T)
    off = 0
    for p in m.patches:
        sl = slice(off, off + p.n_faces)
        off += p.n_faces
        if p.type != "zeroGradient":
            continue
        n = p.Sf / p.mag_sf[:, None]
        gc = g[p.face_cells]
        assert np.max(np.abs(np.einsum("ij,ij->i", bg[sl], n))) < 1e-14
        tang = gc - n * np.einsum("ij,ij->i", gc, n)[:, None]
        assert np.max(np.abs(bg[sl] - tang)) < 1e-14


# ---------------------------------------------------- corrected laplacian
def full_laplacian(m, T, DT, corrected):
    """source - A T with T0 = T: the integrated discrete laplacian of T
    (implicit two-point part + explicit correction + boundary terms)."""
    sysm = oracle.assemble(m, DT, 1.0, T)
    y = oracle.amul(m, sysm["diag"], sysm["upper"], T)
    src = sysm["source"].copy()
    if corrected:
        g, _ = oracle.grad(m, T)
        src -= oracle.lap_correction(m, DT, g)
    return src - y


def interior_cells(m):
    nx, ny, nz = m.dims
    lab = np.arange(m.n_cells)
    i, j, k = lab % nx, (lab // nx) % ny, lab // (nx * ny)
    return (i > 0) & (i < nx - 1) & (j > 0) & (j < ny - 1) & (k > 0) & (k < nz - 1)


def test_assemble_boundary_source_convention():
    """oracle.assemble's source includes the fixedValue boundary source, so
    source - A T of a constant field with equal wall values is zero."""
    m = meshgen.skewed_block_mesh(3, 3, 3, shear=(0, 0, 0))
    T = np.ones(m.n_cells)
    for p in m.patches:
        p.value[:] = 1.0
    r = full_laplacian(m, T, 1.0, corrected=False)
    assert np.max(np.abs(r)) < 1e-13


@pytest.mark.parametrize("grading", [(1, 1, 1), (1.25, 0.85, 1.1)])
def test_corrected_laplacian_linear_exact(grading):
    """Corrected face flux of a linear field = DT Sf.g exactly (the cell
    gradients are exact), so the discrete laplacian vanishes in interior
    cells."""
    m = meshgen.skewed_block_mesh(6, 5, 6, shear=(0.3, 0.1, 0.2), grading=grading)
    T, gvec = linear_field(m)
    DT = 0.7
    inner = interior_cells(m)
    scale = DT * np.max(m.mag_sf) * np.linalg.norm(gvec)
    rc = full_laplacian(m, T, DT, corrected=True)
    assert np.max(np.abs(rc[inner])) < 1e-12 * scale


def test_corrected_laplacian_quadratic_exact():
    """Uniform sheared block, T = x.Q x: the Gauss gradient is exact in every
    cell off the walls (midpoint interpolation errors cancel on opposite
    faces), its face interpolation is exact (grad T is linear), and T_N - T_P
    = grad T(Cf).d, so the corrected flux is DT Sf.grad T(Cf) = the exact
    face integral: the discrete laplacian equals DT 2 tr(Q) V in cells two
    layers in.  The uncorrected two-point flux DT |Sf| d.Q2d/(n.d) differs
    (non-orthogonal d), and the test sees that."""
    m = meshgen.skewed_block_mesh(7, 7, 7, shear=(0.3, 0.1, 0.2))
    Q = np.array([[1.0, 0.3, -0.2], [0.3, -0.5, 0.4], [-0.2, 0.4, 0.8]])
    T = np.einsum("ij,jk,ik->i", m.C, Q, m.C)
    for p in m.patches:
        p.value[:] = np.einsum("ij,jk,ik->i", p.Cf, Q, p.Cf)
    DT = 0.7
    nx, ny, nz = m.dims
    lab = np.arange(m.n_cells)
    ijk = np.stack([lab % nx, (lab // nx) % ny, lab // (nx * ny)], 1)
    deep = np.all((ijk >= 2) & (ijk <= np.array(m.dims) - 3), axis=1)
    assert deep.sum() == 27
    exact = DT * 2 * np.trace(Q) * m.V
    rc = full_laplacian(m, T, DT, corrected=True)
    ru = full_laplacian(m, T, DT, corrected=False)
    scale = np.max(np.abs(exact))
    assert np.max(np.abs(rc[deep] - exact[deep])) < 1e-10 * scale
    assert np.max(np.abs(ru[deep] - exact[deep])) > 1e-2 * scale


def test_corrected_equals_plain_on_orthogonal():
    m = meshgen.with_geometry(meshgen.block_mesh(5, 4, 3))
    s = meshgen.sine_field(m)
    Tp, _, pp = oracle.laplacian_foam(m, s, 3, tol=1e-12)
    Tc, _, pc = oracle.laplacian_foam_corrected(m, s, 3, n_corr=1, tol=1e-12)
    assert np.max(np.abs(Tc - Tp)) < 1e-13 * np.max(np.abs(s))
    assert len(pc) == 6
    # second pass of each step starts from the converged first pass
    assert all(pc[2 * k + 1]["n_iterations"] <= 1 for k in range(3))
    assert [p["n_iterations"] for p in pp] == [pc[2 * k]["n_iterations"] for k in range(3)]


def test_corrected_conservation_adiabatic():
    """All walls zeroGradient: sum V T is conserved by every corrected step."""
    bc = {n: "zeroGradient" for n in meshgen.PATCH_NAMES}
    m = meshgen.skewed_block_mesh(5, 4, 6, shear=(0.3, 0.1, 0.2), grading=(1.2, 0.9, 1.1), bc=bc)
    rng = np.random.default_rng(3)
    T0 = rng.uniform(-1, 1, m.n_cells)
    T, _, _ = oracle.laplacian_foam_corrected(m, T0, 4, n_corr=2, tol=1e-14)
    assert abs(np.dot(m.V, T) - np.dot(m.V, T0)) < 1e-12 * np.dot(m.V, np.abs(T0))
    assert np.std(T) < np.std(T0)


def test_corrector_fixed_point():
    """With many correctors the last pass of a step solves A T = b(T0) with
    the correction of its own result: the full-corrected residual of the
    final T is at solver tolerance (the loop converges to the implicit
    corrected scheme)."""
    m = meshgen.skewed_block_mesh(6, 6, 6, shear=(0.3, 0.1, 0.2), grading=(1.2, 1, 0.9))
    s = meshgen.sine_field(m)
    T1, _, perfs = oracle.laplacian_foam_corrected(m, s, 1, n_corr=12, tol=1e-14, dt=0.01)
    sysm = oracle.assemble(m, 1.0, 0.01, s)
    g, _ = oracle.grad(m, T1)
    src = sysm["source"] - oracle.lap_correction(m, 1.0, g)
    r = src - oracle.amul(m, sysm["diag"], sysm["upper"], T1)
    assert np.max(np.abs(r)) < 1e-9 * np.max(np.abs(src))
    its = [p["n_iterations"] for p in perfs]
    assert its[-1] <= 2 < its[0]


def test_permutation_invariance():
    """Relabelling cells / reordering and re-orienting faces (reading A24)
    changes only the summation order: grad and the corrected steps agree."""
    m = meshgen.skewed_block_mesh(5, 4, 3, shear=(0.3, 0.1, 0.2), grading=(1.2, 0.9, 1.1))
    pm = meshgen.permute_mesh(m)
    new_of_old = np.argsort(pm.old_of_new)  # block label -> new label
    x = meshgen.random_field(m, seed=4)
    xp = np.empty_like(x)
    xp[new_of_old] = x
    g, bg = oracle.grad(m, x)
    gp, bgp = oracle.grad(pm, xp)
    assert np.max(np.abs(gp[new_of_old] - g)) < 1e-12 * np.max(np.abs(g))
    assert np.max(np.abs(bgp - bg)) < 1e-12 * np.max(np.abs(bg))
    T, _, _ = oracle.laplacian_foam_corrected(m, x, 2, n_corr=1, tol=1e-13)
    Tp, _, _ = oracle.laplacian_foam_corrected(pm, xp, 2, n_corr=1, tol=1e-13)
    assert np.max(np.abs(Tp[new_of_old] - T)) < 1e-10 * np.max(np.abs(T))
