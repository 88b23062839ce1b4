"""Spatially varying DT: CUDA vs the CPU oracle through
the C ABI (-m gpu).  Coefficients bitwise on upper-triangular meshes (same
rounded operations, same order), 1e-12 when renumbered; steps T rel L-inf
1e-8 at tol 1e-10, iterations +-1; the two-material slab closed form."""
import dataclasses

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


def mixed_bc():
    return {"xmin": ("fixedValue", 1.5), "xmax": "zeroGradient", "ymin": ("fixedValue", -0.5),
            "zmax": "zeroGradient"}


def with_random_dt(m, seed=4, lo=0.2, hi=3.0):
    rng = np.random.default_rng(seed)
    return dataclasses.replace(m, DT_field=rng.uniform(lo, hi, m.n_cells))


MESHES = {
    "skew_graded": lambda: with_random_dt(meshgen.skewed_block_mesh(13, 11, 9, shear=(0.3, 0.1, 0.2),
                                                                    grading=(1.15, 0.9, 1.05), bc=mixed_bc())),
    "orthogonal": lambda: with_random_dt(meshgen.with_geometry(meshgen.block_mesh(9, 7, 8))),
    "perm_skew": lambda: meshgen.permute_mesh(with_random_dt(meshgen.skewed_block_mesh(
        7, 6, 5, shear=(0.3, 0.1, 0.2), grading=(1.2, 0.9, 1.1), bc=mixed_bc()))),
}


def close(got, ref, exact, tol=1e-12):
    if exact:
        return np.array_equal(got, ref)
    den = np.maximum(np.max(np.abs(ref)), 1e-300)
    return np.max(np.abs(got - ref), initial=0.0) <= tol * den


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("corrected", [False, True])
def test_dtfield_assembly_parity(ctx, name, corrected):
    m = MESHES[name]()
    T = meshgen.random_field(m, seed=5)
    DT, dt = 99.0, 0.2          # the scalar DT must be ignored
    ref = oracle.assemble(m, DT, dt, T)
    if corrected:
        g, _ = oracle.grad(m, T)
        src = (1.0 / dt * T) * m.V - oracle.lap_correction(m, DT, g)
        for p, sl in zip(m.patches, oracle.OMesh(m).patch_slices()):
            if p.type == "fixedValue":
                for i, c in enumerate(p.face_cells):
                    src[c] += ref["boundary_coeffs"][sl][i]
        ref["source"] = src
    mesh = P.Mesh(ctx, m)
    assert mesh.variable_dt
    np.testing.assert_array_equal(mesh.get_DT_field(), m.DT_field)
    mesh.set_T(T)
    got = mesh.assemble(DT, dt, corrected=corrected).export()
    exact = m.old_of_new is None
    for k in ("diag", "upper", "source", "internal_coeffs", "boundary_coeffs"):
        assert close(got[k], ref[k], exact), k
    mesh.close()


@pytest.mark.parametrize("name,corrected", [("skew_graded", True), ("orthogonal", False), ("perm_skew", True)])
def test_dtfield_step_parity(ctx, name, corrected):
    m = MESHES[name]()
    T0 = meshgen.sine_field(m) + 0.1 * meshgen.random_field(m, seed=2)
    if corrected:
        To, _, po = oracle.laplacian_foam_corrected(m, T0, 4, n_corr=1)
    else:
        To, _, po = oracle.laplacian_foam(m, T0, 4)
    for rn in (False, True):
        mesh = P.Mesh(ctx, m, renumber=rn)
        mesh.set_T(T0)
        pg = mesh.step(4, corrected=corrected, n_non_orth_correctors=1 if corrected else 0)
        assert np.max(np.abs(mesh.get_T() - To)) <= 1e-8 * np.max(np.abs(To)), rn
        assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
        mesh.close()


def test_two_material_slab(ctx):
    """Steady state of a two-material slab = the series-resistance closed
    form (see tests/test_oracle_dtfield.py), 1000 cells along x."""
    N, DT1, DT2 = 1000, 0.3, 4.0
    bc = {"xmin": ("fixedValue", 0.0), "xmax": ("fixedValue", 1.0),
          "ymin": "zeroGradient", "ymax": "zeroGradient", "zmin": "zeroGradient", "zmax": "zeroGradient"}
    m = meshgen.skewed_block_mesh(N, 1, 1, shear=(0, 0, 0), bc=bc)
    m = dataclasses.replace(m, DT_field=np.where(np.arange(N) < N // 2, DT1, DT2))
    h = 1.0 / N
    R = [h / (2 * DT1)] + [h / DT1] * (N // 2 - 1) + [2 * h / (DT1 + DT2)] + [h / DT2] * (N // 2 - 1) \
        + [h / (2 * DT2)]
    Texact = np.cumsum(R)[:-1] / sum(R)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(np.zeros(N))
    mesh.step(4, dt=1e8, tol=1e-15, max_iter=5000)
    assert np.max(np.abs(mesh.get_T() - Texact)) < 1e-9
    mesh.close()


def test_uniform_field_equals_scalar(ctx):
    m = meshgen.skewed_block_mesh(12, 10, 9, shear=(0.3, 0.1, 0.2), grading=(1.2, 0.9, 1.1))
    s = meshgen.sine_field(m)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(s)
    mesh.step(3, DT=1.7, corrected=True, n_non_orth_correctors=1)
    a = mesh.get_T()
    mesh.set_DT_field(np.full(m.n_cells, 1.7))
    mesh.set_T(s)
    mesh.step(3, DT=55.0, corrected=True, n_non_orth_correctors=1)
    assert np.array_equal(mesh.get_T(), a)
    mesh.close()


def test_dtfield_errors(ctx):
    plain = meshgen.block_mesh(4)
    mesh = P.Mesh(ctx, plain)
    with pytest.raises(P.LfoamError) as e:
        mesh.set_DT_field(np.ones(plain.n_cells))
    assert e.value.status == 1
    with pytest.raises(P.LfoamError) as e:
        mesh.step(1, variable_DT=True)
    assert e.value.status == 2
    mesh.close()
    g = meshgen.skewed_block_mesh(4, 4, 4)
    mesh = P.Mesh(ctx, g)
    with pytest.raises(P.LfoamError):
        mesh.get_DT_field()
    with pytest.raises(P.LfoamError):
        mesh.set_DT_field(np.zeros(g.n_cells))
    with pytest.raises(P.LfoamError):
        mesh.set_DT_field(np.ones(3))
    mesh.close()
