"""DIC preconditioner: CUDA path vs the CPU oracle through
the C ABI (-m gpu).

Bars: the multicolour numbering bit-exact against meshgen's (an independent
implementation of the same first-fit rule); the reciprocal DIC diagonal and
one preconditioner application BITWISE equal to the oracle's sequential face
loops (the level-scheduled gather visits a cell's faces in the loop order
with explicit _rn operations); solves and steps T rel L-inf 1e-8, iterations
+-1 (criterion flips exempt, A33); the full config-2 run against the discrete
closed form g^n s.
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


MESHES = {
    "cube8": lambda: meshgen.block_mesh(8),                                   # 22 levels
    "box_mixed": lambda: meshgen.block_mesh(7, 5, 4, extent=(1.0, 0.6, 1.3), bc=mixed_bc()),
    "perm6": lambda: meshgen.permute_mesh(meshgen.block_mesh(6, bc=mixed_bc())),  # scattered levels
    "colour9": lambda: meshgen.colour_mesh(meshgen.block_mesh(9, bc=mixed_bc())),  # 2 levels, contiguous
    "skewed": lambda: meshgen.skewed_block_mesh(6, 5, 7, shear=(0.3, 0.1, 0.2), grading=(2.0, 1.0, 0.5)),
    "line": lambda: meshgen.block_mesh(37, 1, 1),
    "single_cell": lambda: meshgen.block_mesh(1),
}


@pytest.mark.parametrize("name", ["cube8", "box_mixed", "perm6", "skewed", "line"])
def test_colour_renumber_matches_meshgen(ctx, name):
    m = MESHES[name]()
    mesh = P.Mesh(ctx, m, renumber="colour", geometry=False)
    co = mesh.export_addressing()["cell_order"]
    np.testing.assert_array_equal(co, meshgen.colour_order(m))
    mesh.close()


@pytest.mark.parametrize("name", list(MESHES))
def test_precondition_bitwise(ctx, name):
    m = MESHES[name]()
    T0 = meshgen.random_field(m, seed=2)
    ref = oracle.assemble(m, 0.7, 0.1, T0)
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(T0)
    ldu = mesh.assemble(0.7, 0.1)
    r = meshgen.random_field(m, seed=11)
    rD_o, w_o = oracle.dic(m, ref["diag"], ref["upper"], r)
    w, rD = dev(np.zeros(m.n_cells)), dev(np.zeros(m.n_cells))
    ldu.precondition(dev(r), w, "DIC", rD)
    np.testing.assert_array_equal(rD.cpu().numpy(), rD_o)
    np.testing.assert_array_equal(w.cpu().numpy(), w_o)
    # the diagonal preconditioner: w = (1/diag) r
    ldu.precondition(dev(r), w, "diagonal", rD)
    np.testing.assert_array_equal(rD.cpu().numpy(), 1.0 / ref["diag"])
    np.testing.assert_array_equal(w.cpu().numpy(), (1.0 / ref["diag"]) * r)
    mesh.close()


@pytest.mark.parametrize("name", ["cube8", "box_mixed"])
def test_precondition_bitwise_library_colouring(ctx, name):
    """renumber = 2 inside the library == the oracle on meshgen's colour mesh."""
    m = MESHES[name]()
    mc = meshgen.colour_mesh(m)
    T0 = meshgen.random_field(m, seed=5)
    order = meshgen.colour_order(m)
    ref = oracle.assemble(mc, 1.0, 0.2, T0[order])
    r = meshgen.random_field(mc, seed=6)
    rD_o, w_o = oracle.dic(mc, ref["diag"], ref["upper"], r)
    mesh = P.Mesh(ctx, m, renumber="colour", geometry=False)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    w, rD = dev(np.zeros(m.n_cells)), dev(np.zeros(m.n_cells))
    ldu.precondition(dev(r), w, "DIC", rD)       # internal numbering == mc's
    np.testing.assert_array_equal(rD.cpu().numpy(), rD_o)
    np.testing.assert_array_equal(w.cpu().numpy(), w_o)
    mesh.close()


@pytest.mark.parametrize("name", ["cube8", "box_mixed", "perm6", "colour9", "skewed"])
def test_pcg_dic_parity(ctx, name):
    m = MESHES[name]()
    T0 = meshgen.random_field(m, seed=4)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    x_ref, p_ref = oracle.pcg(m, ref, T0, precond="DIC")
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    psi = dev(T0)
    perf = ldu.pcg_solve(psi, precond="DIC")
    x = psi.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref)) <= 1e-8
    assert abs(perf["n_iterations"] - p_ref["n_iterations"]) <= 1, (perf, p_ref)
    assert perf["converged"] == p_ref["converged"] == 1
    assert abs(perf["initial_residual"] - p_ref["initial_residual"]) <= 1e-10 * p_ref["initial_residual"]
    mesh.close()


def test_pcg_dic_controls(ctx):
    m = meshgen.colour_mesh(meshgen.block_mesh(8))
    T0 = meshgen.sine_field(m)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    for kw in [dict(max_iter=3), dict(min_iter=30), dict(tol=0.0, rel_tol=1e-3), dict(max_iter=0)]:
        x_ref, p_ref = oracle.pcg(m, ref, T0, precond="DIC", **kw)
        psi = dev(T0)
        perf = ldu.pcg_solve(psi, precond="DIC", **kw)
        assert perf["n_iterations"] == p_ref["n_iterations"], kw
        assert perf["converged"] == p_ref["converged"], kw
        assert np.max(np.abs(psi.cpu().numpy() - x_ref)) <= 1e-8 * np.max(np.abs(x_ref)), kw
    mesh.close()


@pytest.mark.parametrize("name", ["cube8", "box_mixed", "perm6", "line", "single_cell"])
@pytest.mark.parametrize("colour", [False, True])
def test_step_dic_parity(ctx, name, colour):
    m = MESHES[name]()
    T0 = meshgen.sine_field(m) if name != "single_cell" else np.array([0.3])
    mo = meshgen.colour_mesh(m) if colour else m
    order = meshgen.colour_order(m) if colour else np.arange(m.n_cells)
    To, _, po = oracle.laplacian_foam(mo, T0[order], 5, precond="DIC")
    mesh = P.Mesh(ctx, m, renumber="colour" if colour else False, geometry=False)
    mesh.set_T(T0)
    pg = mesh.step(5, precond="DIC")
    T = mesh.get_T()[order]
    assert np.max(np.abs(T - To)) <= 1e-8 * max(np.max(np.abs(To)), 1e-300)
    for a, b in zip(pg, po):
        assert abs(a["n_iterations"] - b["n_iterations"]) <= 1, (pg, po)
        assert a["converged"] == b["converged"]
    mesh.close()


def test_dilu_is_dic(ctx):
    """DILU on this symmetric matrix runs the DIC recurrences: identical bits."""
    m = MESHES["box_mixed"]()
    T0 = meshgen.sine_field(m)
    out = {}
    for pc in ("DIC", "DILU"):
        mesh = P.Mesh(ctx, m, renumber="colour")
        mesh.set_T(T0)
        out[pc] = (mesh.step(3, precond=pc), mesh.get_T())
        mesh.close()
    assert [p["n_iterations"] for p in out["DIC"][0]] == [p["n_iterations"] for p in out["DILU"][0]]
    np.testing.assert_array_equal(out["DIC"][1], out["DILU"][1])


def test_dic_determinism_and_launches(ctx):
    m = meshgen.block_mesh(20)
    T0 = meshgen.canonical_field(m)
    res = []
    for _ in range(2):
        mesh = P.Mesh(ctx, m, renumber="colour")
        mesh.set_T(T0)
        ctx.set_instrumentation(True)
        pg = mesh.step(4, precond="DIC")
        n, ms = ctx.kernel_stats("pcg_dic")
        ctx.set_instrumentation(False)
        assert n == 4 and ms > 0.0          # one persistent launch per step
        res.append(([p["n_iterations"] for p in pg], mesh.get_T()))
        mesh.close()
    assert res[0][0] == res[1][0]
    np.testing.assert_array_equal(res[0][1], res[1][1])


def test_dic_fewer_iterations(ctx):
    m = meshgen.block_mesh(40)
    T0 = meshgen.canonical_field(m)
    its = {}
    for pc in ("diagonal", "DIC"):
        mesh = P.Mesh(ctx, m, renumber="colour")
        mesh.set_T(T0)
        its[pc] = [p["n_iterations"] for p in mesh.step(3, precond=pc)]
        mesh.close()
    assert all(a < b for a, b in zip(its["DIC"], its["diagonal"])), its


def test_config2_dic_two_steps_vs_oracle(ctx):
    """The DIC bench mesh (100^3, multicolour numbering), first 2 steps vs the
    oracle on meshgen's colour mesh, every cell."""
    m = meshgen.block_mesh(100)
    order = meshgen.colour_order(m)
    mo = meshgen.relabel_mesh(m, order)
    s = meshgen.canonical_field(m)
    To, _, po = oracle.laplacian_foam(mo, s[order], 2, precond="DIC")
    mesh = P.Mesh(ctx, m, renumber="colour")
    mesh.set_T(s)
    pg = mesh.step(2, precond="DIC")
    T = mesh.get_T()[order]
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    mesh.close()


def test_config2_dic_full_run_closed_form(ctx, canonical_constants):
    """The DIC bench workload (100^3, 100 steps) vs T^100 = g^100 s."""
    row = [r for r in canonical_constants["rows"] if r["N"] == 100][0]
    m = meshgen.block_mesh(100)
    s = meshgen.canonical_field(m)
    mesh = P.Mesh(ctx, m, renumber="colour")
    mesh.set_T(s)
    pg = mesh.step(100, precond="DIC")
    T = mesh.get_T()
    ref = row["g"] ** 100 * s
    assert np.max(np.abs(T - ref)) <= 1e-8 * np.max(np.abs(ref))
    assert all(p["converged"] for p in pg)
    mesh.close()


def test_dic_invalid(ctx):
    m = meshgen.block_mesh(4)
    mesh = P.Mesh(ctx, m)
    mesh.set_T(np.ones(m.n_cells))
    ldu = mesh.assemble()
    with pytest.raises(P.LfoamError) as e:
        ldu.pcg_solve(dev(np.ones(m.n_cells)), precond="DIC", max_iter=-1)
    assert e.value.status == 1
    mesh.close()
    # processor patches: the DIC is single-rank
    from paper_2507_18268_b200 import decompose
    base = meshgen.block_mesh(6)
    loop = decompose.cut_mesh(base, decompose.z_plane_faces(base, 3))
    mp = P.Mesh(ctx, loop)
    mp.set_T(np.ones(loop.n_cells))
    with pytest.raises(P.LfoamError) as e:
        mp.step(1, precond="DIC")
    assert e.value.status == 1
    mp.close()


@pytest.mark.parametrize("colour", [False, True])
def test_dic_corrected_laplacian(ctx, colour):
    """DIC with the non-orthogonal correction loop (§8(f) rows 1 + 3) on a
    sheared graded mesh: 1 corrector, vs the oracle in the same numbering."""
    m = meshgen.skewed_block_mesh(9, 8, 7, shear=(0.3, 0.1, 0.2), grading=(2.0, 1.0, 0.5),
                                  bc={"xmin": ("fixedValue", 1.0), "zmax": "zeroGradient"})
    order = meshgen.colour_order(m) if colour else np.arange(m.n_cells)
    mo = meshgen.relabel_mesh(m, order) if colour else m
    T0 = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam_corrected(mo, T0[order], 3, n_corr=1, precond="DIC")
    mesh = P.Mesh(ctx, m, renumber="colour" if colour else False)
    mesh.set_T(T0)
    pg = mesh.step(3, corrected=True, n_non_orth_correctors=1, precond="DIC")
    T = mesh.get_T()[order]
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert len(pg) == len(po) == 6
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    mesh.close()


def test_dic_dt_field(ctx):
    """DIC with a two-material DT field (§8(f) rows 2 + 3), colour numbering."""
    import dataclasses
    base = meshgen.with_geometry(meshgen.block_mesh(10, 9, 8))
    m = dataclasses.replace(base, DT_field=meshgen.layered_dt_field(base))
    order = meshgen.colour_order(m)
    mo = meshgen.relabel_mesh(m, order)
    T0 = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam(mo, T0[order], 4, precond="DIC")
    mesh = P.Mesh(ctx, m, renumber="colour")
    mesh.set_T(T0)
    pg = mesh.step(4, precond="DIC")
    T = mesh.get_T()[order]
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    mesh.close()


def test_dic_multicolour_8_neighbours(ctx):
    """Block + diagonal faces: up to 8 neighbours per cell (the 8-slot rows)
    and a first-fit colouring with 4 colours, i.e. 4 contiguous levels under
    renumber = 2 (several forward and backward level passes) — bitwise
    preconditioner and step parity."""
    from test_gpu_parity import k4_mesh
    m = k4_mesh(8)
    order = meshgen.colour_order(m)
    mc = meshgen.relabel_mesh(m, order)
    deg = np.bincount(mc.owner, minlength=mc.n_cells) + np.bincount(mc.neighbour, minlength=mc.n_cells)
    assert deg.max() == 8
    T0 = meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam(mc, T0[order], 3, precond="DIC")
    mesh = P.Mesh(ctx, m, renumber="colour")
    mesh.set_T(T0)
    pg = mesh.step(3, precond="DIC")
    assert np.max(np.abs(mesh.get_T()[order] - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    ref = oracle.assemble(mc, 1.0, 0.2, mesh.get_T()[order])
    ldu = mesh.assemble(1.0, 0.2)
    r = meshgen.random_field(mc, seed=3)
    rD_o, w_o = oracle.dic(mc, ref["diag"], ref["upper"], r)
    w, rD = dev(np.zeros(m.n_cells)), dev(np.zeros(m.n_cells))
    ldu.precondition(dev(r), w, "DIC", rD)
    np.testing.assert_array_equal(rD.cpu().numpy(), rD_o)
    np.testing.assert_array_equal(w.cpu().numpy(), w_o)
    mesh.close()


@pytest.mark.parametrize("name", ["cube8", "box_mixed", "colour9"])
@pytest.mark.parametrize("variant", [1, 2])
def test_step_dic_forced_variants(name, variant):
    """Both persistent DIC variants forced on small colour-numbered meshes:
    variant 2 is the HBM-bound one (two contiguous colours interleaved in the
    Amul phase, the `pair` path the 200^3/400^3 benches run), variant 1 the
    L2-resident one (stash) — 5 steps vs the oracle in the same numbering."""
    import paper_2507_18268_b200 as _P
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m = MESHES[name]()
    order = meshgen.colour_order(m)
    mo = meshgen.relabel_mesh(m, order)
    T0 = meshgen.multimode_field(m)
    To, _, po = oracle.laplacian_foam(mo, T0[order], 5, precond="DIC")
    c = _P.Context(0)
    c.set_option("variant", variant)
    mesh = _P.Mesh(c, m, renumber="colour")
    mesh.set_T(T0)
    pg = mesh.step(5, precond="DIC")
    T = mesh.get_T()[order]
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    assert all(a["converged"] == b["converged"] for a, b in zip(pg, po))
    mesh.close()
    c.close()


def test_config3_dic_hbm_vs_oracle_and_closed_form(ctx, canonical_constants):
    """The DIC bench workload at config 3 (200^3, colour numbering) through the
    HBM-bound DIC path it is benched with: step 0 against the oracle on every
    cell (same numbering), then 5 steps against T^5 = g^5 s."""
    row = [r for r in canonical_constants["rows"] if r["N"] == 200][0]
    m = meshgen.block_mesh(200)
    order = meshgen.colour_order(m)
    mo = meshgen.relabel_mesh(m, order)
    s = meshgen.canonical_field(m)
    To, _, po = oracle.laplacian_foam(mo, s[order], 1, precond="DIC")
    mesh = P.Mesh(ctx, m, renumber="colour")
    mesh.set_T(s)
    pg = mesh.step(1, precond="DIC")
    T = mesh.get_T()
    assert np.max(np.abs(T[order] - To)) <= 1e-8 * np.max(np.abs(To))
    assert abs(pg[0]["n_iterations"] - po[0]["n_iterations"]) <= 1, (pg, po)
    pg += mesh.step(4, precond="DIC")
    ref = row["g"] ** 5 * s
    assert np.max(np.abs(mesh.get_T() - ref)) <= 1e-8 * np.max(np.abs(ref))
    assert all(p["converged"] for p in pg)
    mesh.close()
