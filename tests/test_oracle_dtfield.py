"""Pins for the oracle's spatially varying diffusivity (
-m "not gpu").

gamma_f = lambda (DT_P - DT_N) + DT_N (P:293-299 interpolation with the
weights of P:321-334), boundary DT[faceCell] (reading A38); the laplacian
uses gammaMagSf = gamma_f |Sf| in place of DT |Sf|.  Fixed by: the SPEC
interpolation example carried into a coefficient; the discrete steady state
of a two-material slab (series resistances, closed form); uniform fields
reduce to the scalar-DT oracle bitwise; conservation.
"""
import dataclasses

import numpy as np
import pytest

import meshgen
import oracle


def with_dt(m, DTc):
    return dataclasses.replace(m, DT_field=np.asarray(DTc, dtype=np.float64))


def test_gamma_spec_interpolation(spec_examples):
    """w = 0.25, (DT_P, DT_N) = (2, 4) -> gamma_f = 3.5, so
    upper = -delta * (3.5 |Sf|)."""
    ex = spec_examples["interpolate"][1]
    Sf = np.array([[1.0, 0.0, 0.0]])
    m = meshgen.Mesh(2, np.array([0], np.int32), np.array([1], np.int32), np.ones(1), np.array([2.0]),
                     np.ones(2), [], dims=(2, 1, 1), Sf=Sf, Cf=np.array([[1 - ex["w"], 0, 0]]),
                     C=np.array([[0.0, 0, 0], [1.0, 0, 0]]))
    g, _ = oracle.face_gamma(m, [ex["v_owner"], ex["v_neighbour"]])
    assert g[0] == ex["face"]
    sysm = oracle.assemble(with_dt(m, [ex["v_owner"], ex["v_neighbour"]]), 1.0, 1e300, np.zeros(2))
    assert sysm["upper"][0] == -2.0 * ex["face"]


@pytest.mark.parametrize("N,DT1,DT2", [(10, 1.0, 5.0), (16, 0.2, 3.0)])
def test_two_material_slab_steady_state(N, DT1, DT2):
    """1-D slab, T = 0 at x = 0 and 1 at x = 1, DT1 in the left half, DT2 in
    the right: the discrete steady state carries one flux q through a chain
    of face resistances R = 1/(gamma |Sf| delta): h/(2 DT1) at the wall,
    h/DT1 inside, 2h/(DT1 + DT2) at the interface (arithmetic mean = linear
    interpolation with w = 1/2), h/DT2, h/(2 DT2)."""
    bc = {"xmin": ("fixedValue", 0.0), "xmax": ("fixedValue", 1.0),
          "ymin": "zeroGradient", "ymax": "zeroGradient", "zmin": "zeroGradient", "zmax": "zeroGradient"}
    m = meshgen.skewed_block_mesh(N, 1, 1, shear=(0, 0, 0), bc=bc)
    DTc = np.where(np.arange(N) < N // 2, DT1, DT2)
    h = 1.0 / N
    R = [h / (2 * DT1)] + [h / DT1] * (N // 2 - 1) + [2 * h / (DT1 + DT2)] + [h / DT2] * (N // 2 - 1) \
        + [h / (2 * DT2)]
    q = 1.0 / sum(R)
    Texact = q * np.cumsum(R)[:-1]
    T, _, _ = oracle.laplacian_foam(with_dt(m, DTc), np.zeros(N), 6, dt=1e8, tol=1e-15)
    assert np.max(np.abs(T - Texact)) < 1e-10
    # a uniform DT gives the straight line: the variable-DT path is really used
    assert np.max(np.abs(Texact - (np.arange(N) + 0.5) * h)) > 1e-2


@pytest.mark.parametrize("corrected", [False, True])
def test_uniform_field_equals_scalar(corrected):
    """gamma = w (DT - DT) + DT = DT exactly: bitwise the scalar-DT run."""
    m = meshgen.skewed_block_mesh(6, 5, 4, shear=(0.3, 0.1, 0.2), grading=(1.2, 0.9, 1.1))
    s = meshgen.sine_field(m)
    mv = with_dt(m, np.full(m.n_cells, 1.7))
    if corrected:
        a = oracle.laplacian_foam_corrected(m, s, 2, n_corr=1, DT=1.7)[0]
        b = oracle.laplacian_foam_corrected(mv, s, 2, n_corr=1, DT=123.0)[0]
    else:
        a = oracle.laplacian_foam(m, s, 2, DT=1.7)[0]
        b = oracle.laplacian_foam(mv, s, 2, DT=123.0)[0]
    assert np.array_equal(a, b)


def test_conservation_random_field():
    bc = {n: "zeroGradient" for n in meshgen.PATCH_NAMES}
    m = meshgen.skewed_block_mesh(6, 5, 7, shear=(0.3, 0.1, 0.2), grading=(1.2, 0.9, 1.1), bc=bc)
    rng = np.random.default_rng(5)
    mv = with_dt(m, rng.uniform(0.1, 3.0, m.n_cells))
    T0 = rng.uniform(-1, 1, m.n_cells)
    T, _, _ = oracle.laplacian_foam_corrected(mv, T0, 3, n_corr=1, tol=1e-14)
    assert abs(np.dot(m.V, T) - np.dot(m.V, T0)) < 1e-12 * np.dot(m.V, np.abs(T0))
    assert np.std(T) < np.std(T0)


def test_gamma_bounds_and_symmetry():
    """gamma_f is a convex combination (weights in [0,1]): between the two
    cell values; boundary values equal the face cell's DT."""
    m = meshgen.skewed_block_mesh(7, 6, 5, shear=(0.3, 0.1, 0.2), grading=(1.3, 0.8, 1.1))
    rng = np.random.default_rng(9)
    DTc = rng.uniform(0.5, 4.0, m.n_cells)
    g, gb = oracle.face_gamma(m, DTc)
    lo = np.minimum(DTc[m.owner], DTc[m.neighbour])
    hi = np.maximum(DTc[m.owner], DTc[m.neighbour])
    assert np.all(g >= lo - 1e-15) and np.all(g <= hi + 1e-15)
    bc = np.concatenate([p.face_cells for p in m.patches])
    assert np.array_equal(gb, DTc[bc])
