"""GAMG preconditioner (reading A43): CUDA path vs
the CPU oracle through the C ABI (-m gpu).

Bars: the agglomeration hierarchy (level sizes, face counts, every
aggregate map) BIT-EXACT against the oracle's (an independent host
implementation of the same pairing rule); the Galerkin coarse matrices and
one V-cycle application BITWISE equal to the oracle (the device passes sum
in the oracle's order with explicit _rn operations), with the single-block
tail of the V-cycle at its default threshold and at both extremes; solves
and steps T rel L-inf 1e-8, iterations +-1; the 100^3 and 200^3 workloads
against the oracle's first steps and the discrete closed form g^n s.
"""
import os

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
    "cube8": lambda: meshgen.block_mesh(8),
    "box_mixed": lambda: meshgen.block_mesh(17, 9, 11, extent=(1.0, 0.6, 1.3), bc=mixed_bc()),
    "perm9": lambda: meshgen.permute_mesh(meshgen.block_mesh(9, bc=mixed_bc())),
    "colour10": lambda: meshgen.colour_mesh(meshgen.block_mesh(10, bc=mixed_bc())),
    "skewed": lambda: meshgen.skewed_block_mesh(12, 10, 9, shear=(0.3, 0.1, 0.2), grading=(2.0, 1.0, 0.5)),
    "line": lambda: meshgen.block_mesh(300, 1, 1),
    "small": lambda: meshgen.block_mesh(4, 4, 3),          # 48 cells: one level (L = 0)
    "single_cell": lambda: meshgen.block_mesh(1),
    "cube40": lambda: meshgen.block_mesh(40),             # grid levels + single-block tail
}


@pytest.mark.parametrize("name", list(MESHES))
def test_hierarchy_matches_oracle(ctx, name):
    m = MESHES[name]()
    mesh = P.Mesh(ctx, m, geometry=False)
    h = mesh.gamg_hierarchy()
    o = oracle.gamg(m)
    assert h["n"] == o["n"] and h["nf"] == o["nf"], (h["n"], o["n"])
    for a, b in zip(h["agg"], o["agg"]):
        np.testing.assert_array_equal(a, b)
    mesh.close()


@pytest.mark.parametrize("tail", [None, "0", "100000000"])
@pytest.mark.parametrize("name", list(MESHES))
def test_galerkin_and_vcycle_bitwise(ctx, name, tail, monkeypatch):
    if tail is not None:
        monkeypatch.setenv("LF_GAMG_TAIL", tail)   # read when the hierarchy is built
    m = MESHES[name]()
    T0 = meshgen.random_field(m, seed=2)
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(T0)
    ldu = mesh.assemble(0.7, 0.1)
    sy = ldu.export()
    ref = oracle.assemble(m, 0.7, 0.1, T0)
    np.testing.assert_array_equal(sy["diag"], ref["diag"])
    r = meshgen.random_field(m, seed=11)
    w, rD = dev(np.zeros(m.n_cells)), dev(np.zeros(m.n_cells))
    ldu.precondition(dev(r), w, "GAMG", rD)
    o = oracle.gamg(m, ref["diag"], ref["upper"], r)
    np.testing.assert_array_equal(rD.cpu().numpy(), 1.0 / ref["diag"])
    for lev in range(1, len(o["n"])):
        g = ldu.gamg_level(lev)
        ol = oracle.gamg_level(m, ref["diag"], ref["upper"], lev)
        np.testing.assert_array_equal(g["l"], ol["l"])
        np.testing.assert_array_equal(g["u"], ol["u"])
        np.testing.assert_array_equal(g["D"], ol["D"])
        np.testing.assert_array_equal(g["U"], ol["U"])
    np.testing.assert_array_equal(w.cpu().numpy(), o["w"])
    mesh.close()


@pytest.mark.parametrize("name", ["cube8", "box_mixed", "perm9", "colour10", "skewed", "small", "cube40"])
def test_pcg_gamg_parity(ctx, name):
    m = MESHES[name]()
    T0 = meshgen.multimode_field(m) if name.startswith("cube") else meshgen.random_field(m, seed=4)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    x_ref, p_ref = oracle.pcg(m, ref, T0, precond="GAMG")
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    psi = dev(T0)
    perf = ldu.pcg_solve(psi, precond="GAMG")
    assert abs(perf["n_iterations"] - p_ref["n_iterations"]) <= 1, (perf, p_ref)
    assert perf["converged"] == p_ref["converged"] == 1
    x = psi.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) <= 1e-8 * np.max(np.abs(x_ref))
    mesh.close()


@pytest.mark.parametrize("kw", [dict(max_iter=1), dict(max_iter=2), dict(max_iter=3), dict(min_iter=12),
                                dict(tol=0.0, rel_tol=1e-4)])
def test_pcg_gamg_controls(ctx, kw):
    m = meshgen.block_mesh(16, 12, 10, bc=mixed_bc())
    T0 = meshgen.random_field(m, seed=7)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    x_ref, p_ref = oracle.pcg(m, ref, T0, precond="GAMG", **kw)
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    psi = dev(T0)
    perf = ldu.pcg_solve(psi, precond="GAMG", **kw)
    assert perf["n_iterations"] == p_ref["n_iterations"], (kw, perf, p_ref)
    assert perf["converged"] == p_ref["converged"]
    x = psi.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) <= 1e-8 * np.max(np.abs(x_ref)), kw
    mesh.close()


@pytest.mark.parametrize("name", ["box_mixed", "perm9", "cube40"])
def test_step_gamg_parity(ctx, name):
    m = MESHES[name]()
    T0 = meshgen.multimode_field(m) if name.startswith("cube") else meshgen.random_field(m, seed=5)
    To, _, po = oracle.laplacian_foam(m, T0, 5, precond="GAMG")
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(T0)
    pg = mesh.step(5, precond="GAMG")
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    mesh.close()


def test_gamg_singular_branch(ctx):
    """T = 0, fixedValue-0 walls, min_iter = 1: r = 0, w = M^-1 0 = 0,
    wApA = 0 -> singular at iteration 0, LF_OK."""
    m = meshgen.block_mesh(9)
    z = np.zeros(m.n_cells)
    _, _, po = oracle.laplacian_foam(m, z, 1, min_iter=1, precond="GAMG")
    assert po[0]["singular"] == 1
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(z)
    pg = mesh.step(1, min_iter=1, precond="GAMG")
    assert pg[0]["singular"] == 1 and pg[0]["n_iterations"] == po[0]["n_iterations"] == 0
    np.testing.assert_array_equal(mesh.get_T(), 0.0)
    mesh.close()


def test_gamg_determinism_and_launches(ctx):
    m = meshgen.block_mesh(30)
    T0 = meshgen.multimode_field(m)
    out = []
    for _ in range(2):
        mesh = P.Mesh(ctx, m, geometry=False)
        mesh.set_T(T0)
        ctx.set_instrumentation(True)
        pg = mesh.step(3, precond="GAMG")
        n, _ = ctx.kernel_stats("pcg_gamg")
        assert n == 3                       # one persistent launch per solve
        out.append((mesh.get_T(), [p["n_iterations"] for p in pg]))
        ctx.set_instrumentation(False)
        mesh.close()
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


def test_gamg_fewer_iterations(ctx):
    m = meshgen.block_mesh(48)
    T0 = meshgen.canonical_field(m)
    its = {}
    for pc in ("diagonal", "GAMG"):
        mesh = P.Mesh(ctx, m, geometry=False)
        mesh.set_T(T0)
        its[pc] = mesh.step(1, precond=pc)[0]["n_iterations"]
        mesh.close()
    assert its["GAMG"] * 2 < its["diagonal"], its


def test_gamg_invalid(ctx):
    from paper_2507_18268_b200 import decompose
    base = meshgen.block_mesh(6)
    loop = decompose.cut_mesh(base, decompose.z_plane_faces(base, 3))
    mp = P.Mesh(ctx, loop)
    mp.set_T(np.ones(loop.n_cells))
    with pytest.raises(P.LfoamError) as e:
        mp.step(1, precond="GAMG")
    assert e.value.status == 1
    with pytest.raises(P.LfoamError) as e:
        mp.gamg_hierarchy()
    assert e.value.status == 1
    mp.close()
    m = meshgen.block_mesh(5)
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(np.ones(m.n_cells))
    ldu = mesh.assemble()
    with pytest.raises(P.LfoamError) as e:
        ldu.gamg_level(1)                   # before any GAMG use
    assert e.value.status == 2
    mesh.close()


def test_config2_gamg_vs_oracle_and_closed_form(ctx, canonical_constants):
    """The GAMG bench workload at 100^3: 2 steps against the oracle on every
    cell, then 20 steps against T^20 = g^20 s."""
    row = [r for r in canonical_constants["rows"] if r["N"] == 100][0]
    m = meshgen.block_mesh(100)
    s = meshgen.canonical_field(m)
    To, _, po = oracle.laplacian_foam(m, s, 2, precond="GAMG")
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(s)
    pg = mesh.step(2, precond="GAMG")
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
    pg += mesh.step(18, precond="GAMG")
    ref = row["g"] ** 20 * s
    assert np.max(np.abs(mesh.get_T() - ref)) <= 1e-8 * np.max(np.abs(ref))
    assert all(p["converged"] for p in pg)
    mesh.close()


def test_config3_gamg_vs_oracle_and_closed_form(ctx, canonical_constants):
    """The GAMG bench workload at config 3 (200^3): step 0 against the
    oracle on every cell, then 5 steps against T^5 = g^5 s."""
    row = [r for r in canonical_constants["rows"] if r["N"] == 200][0]
    m = meshgen.block_mesh(200)
    s = meshgen.canonical_field(m)
    To, _, po = oracle.laplacian_foam(m, s, 1, precond="GAMG")
    mesh = P.Mesh(ctx, m, geometry=False)
    mesh.set_T(s)
    pg = mesh.step(1, precond="GAMG")
    T = mesh.get_T()
    assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
    assert abs(pg[0]["n_iterations"] - po[0]["n_iterations"]) <= 1, (pg, po)
    pg += mesh.step(4, precond="GAMG")
    ref = row["g"] ** 5 * s
    assert np.max(np.abs(mesh.get_T() - ref)) <= 1e-8 * np.max(np.abs(ref))
    assert all(p["converged"] for p in pg)
    mesh.close()
