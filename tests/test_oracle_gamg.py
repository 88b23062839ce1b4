"""Pins for the oracle's GAMG preconditioner (
reading A43 in DESIGN.md) against things other than itself (-m "not gpu").

What fixes each expected value:
  * agglomeration on a uniform block: every face weight is equal, so the
    first pairing pass (ascending) pairs cells along x and the second
    (descending) pairs the x-pairs along z (coarse faces in z and y carry
    two fine faces, z has the lower label) — the level-1 aggregate of cell
    (i, j, k) is the 2x1x2 block (i//2, j, k//2), numbered in the descending
    pass's creation order: a closed form from the geometry;
  * any mesh: the maps are partitions into CONNECTED aggregates, level sizes
    shrink, the coarsest has at most 64 cells (or coarsening stalled);
  * Galerkin coarse matrices = P^T A P with dense matrices (numpy matmul of
    the piecewise-constant prolongation built from the maps);
  * the V-cycle = the multigrid error-propagation operator of textbook
    theory, computed with dense matrices level by level:
      M_L^-1 = A_L^-1,
      E_l = (I - S_l A_l)(I - P_l M_{l+1}^-1 P_l^T A_l)(I - S_l A_l),
      M_l^-1 = (I - E_l) A_l^-1,   S_l = omega D_l^-1
    (a wrong smoother weight, a dropped residual term, a transposed
    restriction or a wrong coarse index changes M^-1);
  * M^-1 is symmetric positive definite (a PCG preconditioner);
  * a mesh with at most 64 cells has one level: M^-1 = A^-1 exactly, so
    GAMG-PCG converges in ONE iteration;
  * GAMG-PCG converges to the dense Cholesky solution and needs fewer
    iterations than DIC and diagonal on a cube;
  * a full step reaches the exact discrete decay g^n s.
"""
import numpy as np
import pytest

import meshgen
import oracle

from test_oracle_pins import dense_from_ldu

OMEGA = 0.9   # reading A43: weighted-Jacobi smoother weight
NMIN = 64     # reading A43: coarsening stops at <= 64 cells


def meshes():
    yield "block", meshgen.block_mesh(9, 7, 6, bc={"zmax": "zeroGradient"})
    yield "permuted", meshgen.permute_mesh(meshgen.block_mesh(7))
    yield "skewed-graded", meshgen.skewed_block_mesh(8, 6, 7, shear=(0.3, 0.1, 0.2), grading=(2.0, 1.0, 0.5))
    yield "colour", meshgen.colour_mesh(meshgen.block_mesh(8))


def prolongations(info):
    """Dense piecewise-constant prolongations P_l (n_l x n_{l+1})."""
    Ps = []
    for l, agg in enumerate(info["agg"]):
        P = np.zeros((info["n"][l], info["n"][l + 1]))
        P[np.arange(info["n"][l]), agg] = 1.0
        Ps.append(P)
    return Ps


def system(m, seed=3):
    T0 = meshgen.random_field(m, seed=seed)
    sy = oracle.assemble(m, 1.0, 0.2, T0)
    A = dense_from_ldu(m.n_cells, m.owner, m.neighbour, sy["diag"], sy["upper"])
    return sy, A


def test_block_agglomeration_closed_form():
    """Uniform 8^3 block: level-1 aggregates are the 2x1x2 blocks, numbered
    in creation order of the descending second pass; 512 -> 128 -> 32 cells;
    the coarse graphs are the block graphs of 4x8x4 and (level 2) 32 cells."""
    N = 8
    m = meshgen.block_mesh(N)
    g = oracle.gamg(m)
    assert g["n"] == [512, 128, 32]
    assert g["nf"][0] == 3 * N * N * (N - 1)
    assert g["nf"][1] == 3 * 8 * 4 + 4 * 7 * 4 + 4 * 8 * 3      # a 4 x 8 x 4 block
    c = np.arange(m.n_cells)
    i, j, k = c % N, (c // N) % N, c // (N * N)
    expect = (3 - k // 2) * 32 + (7 - j) * 4 + (3 - i // 2)
    np.testing.assert_array_equal(g["agg"][0], expect)


def test_chain_pairs():
    """1-D chain: at most 64 cells is one level; with 200 cells pass 1 pairs
    (0,1),(2,3),... and pass 2 (descending) pairs neighbouring pairs, so the
    level-1 aggregates are runs of 4 consecutive cells: 200 -> 50."""
    m = meshgen.block_mesh(10, 1, 1)
    assert oracle.gamg(m)["n"] == [10]
    m = meshgen.block_mesh(200, 1, 1)
    g = oracle.gamg(m)
    assert g["n"][:2] == [200, 50]
    # aggregates are runs of 4 consecutive cells (pairs of pairs)
    a = g["agg"][0]
    for s in range(0, 200, 4):
        assert len(set(a[s:s + 4].tolist())) == 1
    assert len(set(a.tolist())) == 50


@pytest.mark.parametrize("name,m", list(meshes()))
def test_aggregates_are_connected_partitions(name, m):
    g = oracle.gamg(m)
    n = g["n"]
    assert n[0] == m.n_cells
    assert n[-1] <= NMIN or len(n) == 1
    assert all(b < a for a, b in zip(n, n[1:]))
    lo, hi = np.minimum(m.owner, m.neighbour), np.maximum(m.owner, m.neighbour)
    for l, agg in enumerate(g["agg"]):
        assert agg.shape == (n[l],)
        assert agg.min() == 0 and agg.max() == n[l + 1] - 1
        assert len(np.unique(agg)) == n[l + 1]        # onto: no empty aggregate
        # connectivity of every aggregate through faces internal to it
        par = np.arange(n[l])

        def find(x):
            while par[x] != x:
                par[x] = par[par[x]]
                x = par[x]
            return x
        for a, b in zip(lo, hi):
            if agg[a] == agg[b]:
                ra, rb = find(a), find(b)
                if ra != rb:
                    par[ra] = rb
        roots = {}
        for c in range(n[l]):
            roots.setdefault(agg[c], set()).add(find(c))
        assert all(len(v) == 1 for v in roots.values())
        # next level's graph: adjacent aggregates
        pairs = {(min(agg[a], agg[b]), max(agg[a], agg[b])) for a, b in zip(lo, hi) if agg[a] != agg[b]}
        assert len(pairs) == g["nf"][l + 1]
        lo, hi = np.array(sorted(pairs)).T if pairs else (np.zeros(0, int), np.zeros(0, int))


@pytest.mark.parametrize("name,m", list(meshes()))
def test_galerkin_coarse_matrices(name, m):
    sy, A = system(m)
    g = oracle.gamg(m)
    Ps = prolongations(g)
    Al = A
    for l in range(1, len(g["n"])):
        Al = Ps[l - 1].T @ Al @ Ps[l - 1]
        lev = oracle.gamg_level(m, sy["diag"], sy["upper"], l)
        Ad = dense_from_ldu(g["n"][l], lev["l"], lev["u"], lev["D"], lev["U"])
        assert np.all(lev["l"] < lev["u"])
        assert np.max(np.abs(Ad - Al)) <= 1e-13 * np.max(np.abs(Al))


def vcycle_dense(A, Ps, omega=OMEGA):
    """M^-1 of the symmetric V-cycle by the error-propagation operator."""
    As = [A]
    for P in Ps:
        As.append(P.T @ As[-1] @ P)

    def minv(l):
        Al = As[l]
        if l == len(Ps):
            return np.linalg.inv(Al)
        n = Al.shape[0]
        I = np.eye(n)
        S = omega * np.diag(1.0 / np.diag(Al))
        Mc = minv(l + 1)
        E = (I - S @ Al) @ (I - Ps[l] @ Mc @ Ps[l].T @ Al) @ (I - S @ Al)
        return (I - E) @ np.linalg.inv(Al)
    return minv(0)


@pytest.mark.parametrize("name,m", list(meshes()))
def test_vcycle_is_the_multigrid_operator(name, m):
    sy, A = system(m)
    g = oracle.gamg(m)
    assert len(g["n"]) >= 2
    Minv = vcycle_dense(A, prolongations(g))
    rng = np.random.default_rng(11)
    for _ in range(3):
        r = rng.uniform(-1, 1, m.n_cells)
        w = oracle.gamg(m, sy["diag"], sy["upper"], r)["w"]
        ref = Minv @ r
        assert np.max(np.abs(w - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_preconditioner_spd():
    m = meshgen.skewed_block_mesh(7, 6, 5, shear=(0.2, 0.1, 0.3), grading=(1.5, 1.0, 0.7))
    sy, A = system(m)
    n = m.n_cells
    Mi = np.zeros((n, n))
    for c in range(n):
        e = np.zeros(n)
        e[c] = 1.0
        Mi[:, c] = oracle.gamg(m, sy["diag"], sy["upper"], e)["w"]
    assert np.max(np.abs(Mi - Mi.T)) <= 1e-13 * np.max(np.abs(Mi))
    assert np.min(np.linalg.eigvalsh(0.5 * (Mi + Mi.T))) > 0


def test_single_level_is_exact():
    """<= 64 cells: no coarsening, the coarsest solve is the whole solve —
    M^-1 = A^-1, GAMG-PCG converges in one iteration to the dense solution."""
    m = meshgen.block_mesh(4, 4, 4, bc={"xmin": ("fixedValue", 1.0), "zmax": "zeroGradient"})
    assert oracle.gamg(m)["n"] == [64]
    sy, A = system(m, seed=5)
    x, perf = oracle.pcg(m, sy, meshgen.random_field(m, seed=5), tol=1e-12, precond="GAMG")
    ref = np.linalg.solve(A, sy["source"])
    assert perf["n_iterations"] == 1 and perf["converged"]
    assert np.max(np.abs(x - ref)) / np.max(np.abs(ref)) < 1e-12


@pytest.mark.parametrize("N,kind", [(9, "block"), (8, "perm"), (10, "colour")])
def test_gamg_pcg_dense_solve(N, kind):
    m = meshgen.block_mesh(N, bc={"zmax": "zeroGradient", "xmin": ("fixedValue", 1.0)})
    m = {"block": m, "perm": meshgen.permute_mesh(m), "colour": meshgen.colour_mesh(m)}[kind]
    sy, A = system(m, seed=N)
    Lc = np.linalg.cholesky(A)
    ref = np.linalg.solve(Lc.T, np.linalg.solve(Lc, sy["source"]))
    x, perf = oracle.pcg(m, sy, meshgen.random_field(m, seed=N), tol=1e-14, precond="GAMG")
    assert perf["converged"] and not perf["singular"]
    assert np.max(np.abs(x - ref)) / np.max(np.abs(ref)) < 1e-10


def test_gamg_fewer_iterations():
    """Multigrid beats the one-level preconditioners on a 24^3 cube."""
    m = meshgen.block_mesh(24)
    T0 = meshgen.sine_field(m)
    its = {}
    for pc in ("diagonal", "DIC", "GAMG"):
        _, _, p = oracle.laplacian_foam(m, T0, 1, precond=pc)
        assert p[0]["converged"]
        its[pc] = p[0]["n_iterations"]
    assert its["GAMG"] < its["DIC"] < its["diagonal"], its


def test_gamg_step_matches_discrete_decay(canonical_constants):
    N = 10
    key = [k for k in canonical_constants if k != "_about"][0]
    c = [row for row in canonical_constants[key] if row["N"] == N][0]
    m = meshgen.block_mesh(N)
    s = meshgen.sine_field(m)
    T, _, perf = oracle.laplacian_foam(m, s, 10, precond="GAMG")
    expect = float(c["g"]) ** 10 * s
    assert np.max(np.abs(T - expect)) / np.max(np.abs(expect)) < 1e-8
    assert all(p["converged"] for p in perf)


def test_gamg_spec_pcg_examples(spec_examples):
    """SPEC's 2x2 PCG examples: two cells <= 64, one level, exact."""
    from test_oracle_pins import raw_mesh
    for ex in spec_examples["pcg"]:
        A = np.array(ex["A"], float)
        if A[0, 1] != 0:
            m = raw_mesh(2, [0], [1])
            sys = dict(diag=np.diag(A).copy(), upper=np.array([A[0, 1]]), source=np.array(ex["b"], float))
        else:
            m = raw_mesh(2)
            sys = dict(diag=np.diag(A).copy(), upper=np.zeros(0), source=np.array(ex["b"], float))
        x, perf = oracle.pcg(m, sys, np.zeros(2), precond="GAMG")
        np.testing.assert_allclose(x, ex["x"], rtol=1e-12, atol=1e-14)
        assert perf["converged"]
