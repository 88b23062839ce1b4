"""Pins for the oracle's DIC preconditioner against
things other than itself (-m "not gpu").

What fixes each expected value:
  * the defining property of an incomplete Cholesky factorisation with no
    fill, M = (D*+L) D*^-1 (D*+U): diag(M) = diag(A) and M = A on A's
    off-diagonal pattern (a dropped term or wrong index in calcReciprocalD
    breaks the diagonal identity);
  * the preconditioner solves M w = r (dense matrix product; a transposed
    sweep or wrong neighbour breaks it);
  * on a graph without cycles (a 1-D chain) IC(0) has no fill, M = A, and
    DIC-PCG converges in ONE iteration to the dense solution (textbook);
  * SPEC's worked PCG examples with DIC;
  * closed forms on the 2-colour numbered cube (red rD = 1/diag; an interior
    black cell 1/(d - 6a^2/d));
  * the dense LU / Cholesky solution of the assembled system;
  * the multicolour numbering: a valid colouring, first fit, parity on a block.
"""
import numpy as np
import pytest

import meshgen
import oracle

from test_oracle_pins import dense_from_ldu, raw_mesh


def dense_L_U(m, upper):
    n = m.n_cells
    lo = np.minimum(m.owner, m.neighbour)
    hi = np.maximum(m.owner, m.neighbour)
    Lm = np.zeros((n, n))
    Lm[hi, lo] = upper
    return Lm, Lm.T.copy()


def dic_M(m, upper, rD):
    Lm, Um = dense_L_U(m, upper)
    Ds = np.diag(1.0 / rD)
    return (Ds + Lm) @ np.diag(rD) @ (Ds + Um)


def meshes():
    yield "block", meshgen.block_mesh(4, 3, 5, bc={"zmax": "zeroGradient"})
    yield "permuted", meshgen.permute_mesh(meshgen.block_mesh(4))
    yield "skewed-graded", meshgen.skewed_block_mesh(4, 5, 3, shear=(0.3, 0.1, 0.2), grading=(2.0, 1.0, 0.5))
    yield "colour", meshgen.colour_mesh(meshgen.block_mesh(5))


@pytest.mark.parametrize("name,m", list(meshes()))
def test_dic_is_incomplete_cholesky(name, m):
    T0 = meshgen.random_field(m, seed=3)
    sy = oracle.assemble(m, 1.0, 0.2, T0)
    A = dense_from_ldu(m.n_cells, m.owner, m.neighbour, sy["diag"], sy["upper"])
    rD, _ = oracle.dic(m, sy["diag"], sy["upper"])
    M = dic_M(m, sy["upper"], rD)
    scale = np.max(np.abs(A))
    np.testing.assert_allclose(np.diag(M), np.diag(A), rtol=1e-13, atol=1e-15 * scale)
    pattern = A != 0
    np.fill_diagonal(pattern, False)
    assert np.max(np.abs((M - A)[pattern])) <= 1e-13 * scale
    # and M differs from A (fill outside the pattern) on meshes with cycles
    assert np.max(np.abs(M - A)) > 1e-6 * scale


@pytest.mark.parametrize("name,m", list(meshes()))
def test_dic_precondition_solves_M(name, m):
    sy = oracle.assemble(m, 0.7, 0.05, meshgen.random_field(m, seed=1))
    r = meshgen.random_field(m, seed=9)
    rD, w = oracle.dic(m, sy["diag"], sy["upper"], r)
    M = dic_M(m, sy["upper"], rD)
    assert np.max(np.abs(M @ w - r)) <= 1e-13 * np.max(np.abs(r))


def test_dic_chain_is_exact_cholesky():
    """1-D chain: no fill, M = A; DIC-PCG converges in one iteration."""
    m = meshgen.block_mesh(40, 1, 1, bc={"xmin": ("fixedValue", 1.0)})
    T0 = meshgen.random_field(m, seed=2)
    sy = oracle.assemble(m, 1.0, 0.2, T0)
    A = dense_from_ldu(m.n_cells, m.owner, m.neighbour, sy["diag"], sy["upper"])
    rD, _ = oracle.dic(m, sy["diag"], sy["upper"])
    np.testing.assert_allclose(dic_M(m, sy["upper"], rD), A, rtol=0, atol=1e-13 * np.max(np.abs(A)))
    x, perf = oracle.pcg(m, sy, T0, tol=1e-12, precond="DIC")
    assert perf["n_iterations"] == 1 and perf["converged"]
    ref = np.linalg.solve(A, sy["source"])
    assert np.max(np.abs(x - ref)) / np.max(np.abs(ref)) < 1e-12
    # the diagonal preconditioner needs many
    _, pd = oracle.pcg(m, sy, T0, tol=1e-12)
    assert pd["n_iterations"] > 10


def test_dic_spec_examples(spec_examples):
    for ex in spec_examples["pcg"]:
        A = np.array(ex["A"], float)
        if A[0, 1] != 0:
            m = raw_mesh(2, [0], [1])
            sys = dict(diag=np.diag(A).copy(), upper=np.array([A[0, 1]]), source=np.array(ex["b"], float))
        else:
            m = raw_mesh(2)
            sys = dict(diag=np.diag(A).copy(), upper=np.zeros(0), source=np.array(ex["b"], float))
        x, perf = oracle.pcg(m, sys, np.zeros(2), precond="DIC")
        np.testing.assert_allclose(x, ex["x"], rtol=1e-12, atol=1e-14)
        expect = ex.get("iterations", 1)  # 2 cells, one face: DIC is exact
        assert perf["n_iterations"] == expect and perf["converged"]


def test_dic_red_black_closed_form():
    """2-colour numbered cube, DT=1, dt=0.2, fixedValue walls: red cells
    (colour 0, the first half) have no lower neighbours, rD = 1/diag; an
    interior black cell has six interior red neighbours: rD = 1/(d - 6a^2/d),
    d = V/dt + 6a, a = DT h."""
    N = 6
    base = meshgen.block_mesh(N)
    m = meshgen.colour_mesh(base)
    sy = oracle.assemble(m, 1.0, 0.2, np.zeros(m.n_cells))
    rD, _ = oracle.dic(m, sy["diag"], sy["upper"])
    lab = m.old_of_new.astype(np.int64)            # block label of every new cell
    i, j, k = lab % N, (lab // N) % N, lab // (N * N)
    red = (i + j + k) % 2 == 0
    assert np.all(red[: m.n_cells // 2]) and not np.any(red[m.n_cells // 2:])
    np.testing.assert_array_equal(rD[red], 1.0 / sy["diag"][red])
    h = 1.0 / N
    a, d = h, h ** 3 / 0.2 + 6 * h
    deep = (~red) & (i >= 2) & (i <= N - 3) & (j >= 2) & (j <= N - 3) & (k >= 2) & (k <= N - 3)
    assert deep.sum() > 0
    np.testing.assert_allclose(rD[deep], 1.0 / (d - 6 * a * a / d), rtol=1e-14)


@pytest.mark.parametrize("N,colour", [(5, False), (6, True), (5, "perm")])
def test_dic_pcg_dense_solve(N, colour):
    m = meshgen.block_mesh(N, bc={"zmax": "zeroGradient", "xmin": ("fixedValue", 1.0)})
    if colour is True:
        m = meshgen.colour_mesh(m)
    elif colour == "perm":
        m = meshgen.permute_mesh(m)
    T0 = meshgen.random_field(m, seed=N)
    sy = oracle.assemble(m, 1.0, 0.2, T0)
    A = dense_from_ldu(m.n_cells, m.owner, m.neighbour, sy["diag"], sy["upper"])
    Lc = np.linalg.cholesky(A)
    ref = np.linalg.solve(Lc.T, np.linalg.solve(Lc, sy["source"]))
    x, perf = oracle.pcg(m, sy, T0, tol=1e-14, precond="DIC")
    assert perf["converged"] and not perf["singular"]
    assert np.max(np.abs(x - ref)) / np.max(np.abs(ref)) < 1e-10
    assert perf["n_iterations"] <= m.n_cells


def test_dic_fewer_iterations_than_diagonal():
    """IC(0) is a better preconditioner than Jacobi on the Laplacian, in the
    natural and in the multicolour numbering (fewer CG iterations)."""
    base = meshgen.block_mesh(20)
    for m in (base, meshgen.colour_mesh(base)):
        T0 = meshgen.sine_field(m)
        _, _, pd = oracle.laplacian_foam(m, T0, 2)
        _, _, pc = oracle.laplacian_foam(m, T0, 2, precond="DIC")
        for a, b in zip(pc, pd):
            assert a["converged"] and a["n_iterations"] < b["n_iterations"]


def test_dic_step_matches_discrete_decay(canonical_constants):
    """The full step with DIC reaches the same exact linear-solve result
    g^n s as with the diagonal preconditioner."""
    N = 10
    key = [k for k in canonical_constants if k != "_about"][0]
    c = [row for row in canonical_constants[key] if row["N"] == N][0]
    for m in (meshgen.block_mesh(N), meshgen.colour_mesh(meshgen.block_mesh(N))):
        s = meshgen.sine_field(m)
        T, _, perf = oracle.laplacian_foam(m, s, 10, precond="DIC")
        expect = float(c["g"]) ** 10 * s
        assert np.max(np.abs(T - expect)) / np.max(np.abs(expect)) < 1e-8
        assert all(p["converged"] for p in perf)


def test_colour_order_first_fit():
    """meshgen's multicolour numbering: a permutation, a valid colouring
    (no face inside a colour), first fit (each colour is the smallest not
    used by a lower-labelled neighbour, brute force), parity on a block."""
    for m in (meshgen.block_mesh(5, 4, 3), meshgen.permute_mesh(meshgen.block_mesh(4)),
              meshgen.skewed_block_mesh(3, 4, 5)):
        order = meshgen.colour_order(m)
        n = m.n_cells
        assert sorted(order.tolist()) == list(range(n))
        nbrs = [set() for _ in range(n)]
        for a, b in zip(m.owner, m.neighbour):
            nbrs[a].add(int(b))
            nbrs[b].add(int(a))
        col = [0] * n
        for c in range(n):
            used = {col[j] for j in nbrs[c] if j < c}
            col[c] = min(set(range(len(used) + 1)) - used)
        col = np.array(col)
        assert np.all(np.diff(col[order]) >= 0)                       # sorted by colour
        for k in np.unique(col):
            cells = order[col[order] == k]
            assert np.all(np.diff(cells) > 0)
        assert all(col[a] != col[b] for a, b in zip(m.owner, m.neighbour))
    m = meshgen.block_mesh(6, 5, 4)
    order = meshgen.colour_order(m)
    lab = np.arange(m.n_cells)
    par = (lab % 6 + (lab // 6) % 5 + lab // 30) % 2
    assert np.all(par[order[: (par == 0).sum()]] == 0)


def test_relabel_mesh_preserves_the_system():
    """relabel_mesh is a pure renumbering: the assembled system and the
    diagonal-PCG solution are the same up to the permutation."""
    base = meshgen.block_mesh(5, bc={"xmax": ("fixedValue", 2.0), "ymin": "zeroGradient"})
    order = np.random.default_rng(5).permutation(base.n_cells)
    m = meshgen.relabel_mesh(base, order)
    T0 = meshgen.random_field(base, seed=4)
    s0 = oracle.assemble(base, 1.0, 0.2, T0)
    s1 = oracle.assemble(m, 1.0, 0.2, T0[order])
    np.testing.assert_array_equal(s1["diag"], s0["diag"][order])
    np.testing.assert_array_equal(s1["source"], s0["source"][order])
    x0, _ = oracle.pcg(base, s0, T0, tol=1e-13)
    x1, _ = oracle.pcg(m, s1, T0[order], tol=1e-13)
    assert np.max(np.abs(x1 - x0[order])) < 1e-11 * np.max(np.abs(x0))
