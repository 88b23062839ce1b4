"""The HBM-bound persistent solve (88n variant: w recomputed from r/diag, psi
written every second iteration, 16-bit compressed gather labels) against the
CPU oracle through the C ABI (-m gpu); plus the singular branch and the
lockstep diagnostic of SURVEY §8(c.4).

Bars: T rel L-inf 1e-8 and iterations +-1 against the oracle (north_star);
compressed labels decode to the int32 labels, so a solve with them is
BITWISE the solve without them; the forced-iteration (lockstep) rerun of a
step agrees with the oracle's step to ~1e-12 (kernel rounding only).
"""
import numpy as np
import pytest

import meshgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = None


@pytest.fixture(scope="module")
def P_():
    global P
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2507_18268_b200 as _P
    P = _P
    return _P


def context(variant=0, compressed=True, l2_prefetch=0):
    c = P.Context(0)
    c.set_option("variant", variant)
    c.set_option("compressed_labels", compressed)
    c.set_option("l2_prefetch", l2_prefetch)
    return c


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def mixed_bc():
    return {"xmin": ("fixedValue", 1.5), "xmax": "zeroGradient", "ymin": ("fixedValue", -0.5),
            "zmax": "zeroGradient"}


MESHES = {
    "cube12": lambda: meshgen.block_mesh(12),
    "box_mixed": lambda: meshgen.block_mesh(37, 23, 19, bc=mixed_bc()),
    # N_x N_y = 40000 > 2^15: the +N_x N_y offsets escape to the int32 labels
    "wide_plate": lambda: meshgen.block_mesh(200, 200, 3),
    "perm_rcm": lambda: meshgen.permute_mesh(meshgen.block_mesh(14, bc=mixed_bc())),
}


@pytest.mark.parametrize("name", list(MESHES))
def test_compressed_labels_bitwise_and_oracle(P_, name):
    """HBM-bound variant forced: compressed vs int32 labels bitwise equal;
    both against the oracle (5 steps, T 1e-8, iterations +-1)."""
    m = MESHES[name]()
    T0 = meshgen.multimode_field(m) if name != "wide_plate" else meshgen.sine_field(m)
    To, _, po = oracle.laplacian_foam(m, T0, 5)
    out = {}
    for comp in (True, False):
        c = context(variant=2, compressed=comp)
        mesh = P.Mesh(c, m, renumber=1 if name == "perm_rcm" else 0)
        lay = mesh.layout()
        assert lay["ell_width"] in (3, 4)
        assert (lay["label_escapes"] >= 0) == comp
        if comp and name == "wide_plate":
            assert lay["label_escapes"] > 0          # the escape path is exercised
        if comp and name == "cube12":
            assert lay["label_escapes"] == 0
        mesh.set_T(T0)
        pg = mesh.step(5)
        out[comp] = (mesh.get_T(), [p["n_iterations"] for p in pg])
        T = out[comp][0]
        assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
        assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
        mesh.close()
        c.close()
    np.testing.assert_array_equal(out[True][0], out[False][0])
    assert out[True][1] == out[False][1]


@pytest.mark.parametrize("name", ["box_3trips", "perm_rcm_3trips"])
def test_l2_prefetch_bitwise_and_oracle(P_, name):
    """Next-trip L2 prefetch (LF_OPT_L2_PREFETCH) in the HBM-bound variant on
    meshes of 2+ full grid-stride trips and a ragged tail (~420K cells: the
    prefetch runs, and stops before the tail trip): prefetch on and off give
    BITWISE the same T and iteration counts (pure prefetch), both match the
    oracle (4 steps, T 1e-8, iterations +-1)."""
    m = meshgen.block_mesh(81, 67, 77, bc=mixed_bc())
    if name == "perm_rcm_3trips":
        m = meshgen.permute_mesh(m)
    T0 = meshgen.multimode_field(m)
    To, _, po = oracle.laplacian_foam(m, T0, 4)
    out = {}
    for pf in (1, 2):
        c = context(variant=2, compressed=False, l2_prefetch=pf)
        mesh = P.Mesh(c, m, renumber=1 if name == "perm_rcm_3trips" else 0)
        assert mesh.layout()["ell_width"] in (3, 4)
        mesh.set_T(T0)
        pg = mesh.step(4)
        out[pf] = (mesh.get_T(), [p["n_iterations"] for p in pg])
        T = out[pf][0]
        assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
        assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
        mesh.close()
        c.close()
    np.testing.assert_array_equal(out[1][0], out[2][0])
    assert out[1][1] == out[2][1]


@pytest.mark.parametrize("pct", [25, 100])
def test_runtime_trips_deterministic_and_oracle(P_, pct):
    """Run-time scheduled phase-1 trips (LF_OPT_DYNAMIC_TRIPS; in builds with
    -DLF_DYN=1 — the default build keeps the static schedule) on a mesh of
    several grid-stride trips with a ragged tail (~420K cells, mixed
    patches): T matches the oracle (4 steps, T 1e-8, iterations +-1) and a
    second run is BITWISE identical (per-unit sums, added in unit order)."""
    m = meshgen.block_mesh(81, 67, 77, bc=mixed_bc())
    T0 = meshgen.multimode_field(m)
    To, _, po = oracle.laplacian_foam(m, T0, 4)
    res = []
    for rep in range(2):
        c = context(variant=2, compressed=False, l2_prefetch=1)
        c.set_option("dynamic_trips", pct)
        mesh = P.Mesh(c, m)
        mesh.set_T(T0)
        pg = mesh.step(4)
        T = mesh.get_T()
        assert np.max(np.abs(T - To)) <= 1e-8 * np.max(np.abs(To))
        assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po)), (pg, po)
        res.append((T, [p["n_iterations"] for p in pg]))
        mesh.close()
        c.close()
    np.testing.assert_array_equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1]


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("kw", [dict(max_iter=1), dict(max_iter=2), dict(max_iter=5), dict(max_iter=6),
                                dict(min_iter=41), dict(min_iter=42), dict(tol=0.0, rel_tol=1e-3)])
def test_psi_every_second_iteration_controls(P_, variant, kw):
    """psi is written every second iteration in the HBM-bound variant: a stop
    after an odd or an even number of iterations (max_iter, min_iter) must
    flush the pending update(s) — iteration count exact, psi 1e-8."""
    m = meshgen.block_mesh(16, 12, 10, bc=mixed_bc())
    T0 = meshgen.random_field(m, seed=7)
    ref = oracle.assemble(m, 1.0, 0.2, T0)
    x_ref, p_ref = oracle.pcg(m, ref, T0, **kw)
    c = context(variant=variant)
    mesh = P.Mesh(c, m)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 0.2)
    psi = dev(T0)
    perf = ldu.pcg_solve(psi, **kw)
    assert perf["n_iterations"] == p_ref["n_iterations"], (kw, perf, p_ref)
    assert perf["converged"] == p_ref["converged"]
    x = psi.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) <= 1e-8 * np.max(np.abs(x_ref)), kw
    mesh.close()
    c.close()


@pytest.mark.parametrize("variant", [1, 2])
def test_singular_branch_zero_field(P_, variant):
    """T = 0 with fixedValue-0 walls: b = r = 0, normFactor = 1e-20; with
    min_iter = 1 the loop is entered and wApA = 0 -> checkSingularity stops
    at iteration 0 with singular = 1 and LF_OK (SURVEY §8(b) errors)."""
    m = meshgen.block_mesh(9)
    z = np.zeros(m.n_cells)
    _, _, po = oracle.laplacian_foam(m, z, 1, min_iter=1)
    assert po[0]["singular"] == 1
    c = context(variant=variant)
    mesh = P.Mesh(c, m)
    mesh.set_T(z)
    pg = mesh.step(1, min_iter=1)
    assert pg[0]["singular"] == 1 and pg[0]["n_iterations"] == po[0]["n_iterations"] == 0
    assert pg[0]["converged"] == po[0]["converged"]
    np.testing.assert_array_equal(mesh.get_T(), 0.0)
    mesh.close()
    c.close()


@pytest.mark.parametrize("variant", [1, 2])
def test_singular_after_exact_first_iteration(P_, variant):
    """Two cells, zeroGradient walls, V/dt = 1, face coefficient 1: A = [[2,-1],
    [-1,2]] and r0 = (1,1) is an eigenvector, so iteration 0 solves exactly
    (r1 = 0 in floating point); min_iter = 3 forces iteration 1, where
    wArA = 0 -> p = 0 -> wApA = 0: singular at the ODD iteration 1, after the
    HBM-bound variant deferred psi's update — the flush must still apply
    alpha_0 p_0 (psi = (1,1), the exact solution)."""
    zg = {n: "zeroGradient" for n in meshgen.cube.PATCH_NAMES}
    m = meshgen.block_mesh(2, 1, 1, extent=(2.0, 1.0, 1.0), bc=zg)
    T0 = np.ones(2)
    ref = oracle.assemble(m, 1.0, 1.0, T0)
    np.testing.assert_array_equal(ref["diag"], [2.0, 2.0])
    x_ref, p_ref = oracle.pcg(m, ref, np.zeros(2), min_iter=3)
    assert p_ref["singular"] == 1 and p_ref["n_iterations"] == 1
    c = context(variant=variant)
    mesh = P.Mesh(c, m)
    mesh.set_T(T0)
    ldu = mesh.assemble(1.0, 1.0)
    psi = dev(np.zeros(2))
    perf = ldu.pcg_solve(psi, min_iter=3)
    assert perf["singular"] == 1 and perf["n_iterations"] == 1, perf
    np.testing.assert_array_equal(psi.cpu().numpy(), x_ref)
    np.testing.assert_array_equal(x_ref, [1.0, 1.0])
    mesh.close()
    c.close()


def test_lockstep_diagnostic_config2(P_):
    """SURVEY §8(c.4) lockstep diagnostic on config 2 (100^3, canonical field):
    every step of the first 20 rerun on the GPU from the ORACLE's state with
    min_iter = max_iter = the oracle's iteration count.  This removes the
    criterion flips of reading A33 (|dit| > 1 on some steps of the free run)
    and leaves only the kernels' rounding against the oracle's: per-step T
    within 1e-11 relative (measured ~1e-13), including the flip steps."""
    m = meshgen.block_mesh(100)
    T = meshgen.canonical_field(m)
    c = context()
    mesh = P.Mesh(c, m)
    worst = 0.0
    flips = 0
    for step in range(20):
        To, _, po = oracle.laplacian_foam(m, T, 1)
        it = po[0]["n_iterations"]
        mesh.set_T(T)
        free = mesh.step(1)[0]["n_iterations"]
        flips += abs(free - it) > 1
        mesh.set_T(T)
        pg = mesh.step(1, min_iter=it, max_iter=it)
        assert pg[0]["n_iterations"] == it
        err = np.max(np.abs(mesh.get_T() - To)) / np.max(np.abs(To))
        worst = max(worst, err)
        assert err <= 1e-11, (step, err)
        T = To
    print(f"lockstep: worst per-step rel Linf {worst:.2e}, free-run flip steps {flips}")
    mesh.close()
    c.close()
