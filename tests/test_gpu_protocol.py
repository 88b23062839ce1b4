"""Paper-protocol workload: hot plate, DT = 1e-3,
dt = 0.2 s, 500 steps.  The case is one-dimensional (zeroGradient y/z
walls), so every x-line of the 3-D solution equals the implicit-Euler
solution of the 1-D two-point system, computed here with a banded direct
solve (scipy) — a property that holds at the full Mesh-S size."""
import numpy as np
import pytest
from scipy.linalg import solve_banded

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


def hot_plate_1d(N, DT, dt, steps):
    """(h/dt) T_i + (DT/h) sum_nb (T_i - T_nb) + (2 DT/h)(T_i - T_wall) = (h/dt) T0_i
    per unit cross-section; T_wall = 1 at x = 0, 0 at x = 1."""
    h = 1.0 / N
    a, ab = DT / h, 2 * DT / h
    diag = np.full(N, h / dt + 2 * a)
    diag[0] = diag[-1] = h / dt + a + ab
    ab_m = np.zeros((3, N))
    ab_m[0, 1:] = -a
    ab_m[1] = diag
    ab_m[2, :-1] = -a
    T = np.zeros(N)
    for _ in range(steps):
        b = h / dt * T
        b[0] += ab * 1.0
        T = solve_banded((1, 1), ab_m, b)
    return T


def test_protocol_mesh_s_vs_1d(ctx):
    pr = meshgen.PROTOCOL
    m = meshgen.protocol_mesh("S")
    mesh = P.Mesh(ctx, m)
    mesh.set_T(np.zeros(m.n_cells))
    perfs = mesh.step(pr["steps"], pr["DT"], pr["dt"], tol=1e-10)
    T = mesh.get_T().reshape(-1, m.dims[0])
    ref = hot_plate_1d(m.dims[0], pr["DT"], pr["dt"], pr["steps"])
    assert np.max(np.abs(T - ref)) < 1e-7
    assert all(p["converged"] for p in perfs)
    # the transient spans the whole 100 s: far from both the start and the steady state
    x = (np.arange(m.dims[0]) + 0.5) / m.dims[0]
    assert 0.05 < np.max(np.abs(ref - (1 - x))) < 0.9
    mesh.close()


def test_protocol_small_vs_oracle(ctx):
    pr = meshgen.PROTOCOL
    m = meshgen.protocol_mesh(12)
    To, _, po = oracle.laplacian_foam(m, np.zeros(m.n_cells), 50, DT=pr["DT"], dt=pr["dt"])
    mesh = P.Mesh(ctx, m)
    mesh.set_T(np.zeros(m.n_cells))
    pg = mesh.step(50, pr["DT"], pr["dt"])
    assert np.max(np.abs(mesh.get_T() - To)) <= 1e-8 * np.max(np.abs(To))
    assert all(abs(a["n_iterations"] - b["n_iterations"]) <= 1 for a, b in zip(pg, po))
    mesh.close()
