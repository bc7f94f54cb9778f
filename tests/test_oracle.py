"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference.

Runs without a GPU.  The goldens come from cbctkit itself
(tests/golden/make_golden.py); the oracle is a C restatement of its Numba
kernels, so agreement is expected to fp64 rounding.
"""

import numpy as np
import pytest

from _helpers import geom_from_golden, load_golden, rel_l2

from oracle import oracle as O


@pytest.fixture(scope="module")
def small():
    d = load_golden("small_instance")
    vg, tr = geom_from_golden(d)
    return d, O.OracleOperator(vg, tr, workers=3)


def test_small_instance_operator_outputs(small):
    d, op = small
    np.testing.assert_allclose(op.project(d["x"]), d["Ax"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(op.backproject(d["y"]), d["ATy"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(op.row_sums(), d["row_sums"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(op.col_sums(), d["col_sums"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(op.normal_diagonal(), d["normal_diagonal"], rtol=1e-13, atol=1e-13)


def test_small_instance_dense_matrix(small):
    # the reference's independent dense Siddon (tests/oracle.py:47-63) vs our walk
    d, op = small
    A = np.zeros((op.m, op.n))
    A[d["dense_rows"], d["dense_cols"]] = d["dense_vals"]
    x = d["x"]
    assert rel_l2(op.project(x), A @ x) <= 1e-10
    assert rel_l2(op.backproject(d["y"]), A.T @ d["y"]) <= 1e-10


def test_single_pixel_and_segments(small):
    d, op = small
    y = np.zeros(op.m)
    y[137] = 2.5
    np.testing.assert_allclose(op.backproject(y), d["pixel137_backprojection"], rtol=1e-12, atol=0)
    view, rem = divmod(137, 64)
    v, u = divmod(rem, 8)
    idx, ln = op.ray_segments(view, u, v)
    np.testing.assert_array_equal(idx, d["seg137_idx"])
    np.testing.assert_allclose(ln, d["seg137_len"], rtol=1e-13)


def test_adjoint_instance(golden):
    d = golden("adjoint_instance")
    vg, tr = geom_from_golden(d)
    op = O.OracleOperator(vg, tr, workers=8)
    np.testing.assert_allclose(op.project(d["x"]), d["Ax"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(op.backproject(d["y"]), d["ATy"], rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(op.normal_diagonal(), d["normal_diagonal"], rtol=1e-12, atol=1e-12)


def test_known_answers(golden):
    from paper_2110_13526_b200.geometry import DetectorGeometry, VolumeGeometry, make_circular_trajectory

    k = golden("known_answers")
    vg = VolumeGeometry(5, 5, 5, (2.0, 2.0, 2.0))
    tr = make_circular_trajectory(100.0, 200.0, 1, 0.0, 2 * np.pi, DetectorGeometry(1, 1, (1.0, 1.0)))
    chord = O.OracleOperator(vg, tr).project(np.ones(125))[0]
    assert chord == pytest.approx(10.0, rel=1e-9)  # test_operator.py:30-36
    assert chord == pytest.approx(float(k["axial_chord"]), rel=1e-15)
    vg2 = VolumeGeometry(2, 2, 2, (1.0, 1.0, 1.0))
    tr2 = make_circular_trajectory(50.0, 100.0, 2, 0.05, 2 * np.pi, DetectorGeometry(32, 32, (2.0, 2.0)))
    rows = O.OracleOperator(vg2, tr2).row_sums()
    np.testing.assert_allclose(rows, k["miss_rows"], rtol=1e-13, atol=0)
    assert rows.reshape(2, 32, 32)[0, 0, 0] == 0.0
    vg3 = VolumeGeometry(16, 16, 16, (1.0, 1.0, 1.0))
    tr3 = make_circular_trajectory(50.0, 100.0, 12, 0.04, 2 * np.pi, DetectorGeometry(24, 12, (1.5, 1.5)))
    np.testing.assert_allclose(O.OracleOperator(vg3, tr3).normal_diagonal(), k["cone_diag"], rtol=1e-12, atol=1e-12)


def test_desk_projection_and_solvers(golden):
    d = golden("desk")
    vg, tr = geom_from_golden(d)
    op = O.OracleOperator(vg, tr, workers=8)
    truth = O.shepp_logan_phantom(vg)
    np.testing.assert_array_equal(truth.astype(np.float32), d["truth"])
    b = op.project(truth)
    np.testing.assert_allclose(b[d["b_idx"]], d["b_val"], rtol=1e-12, atol=1e-12)
    assert np.linalg.norm(b) == pytest.approx(float(d["b_norm"]), rel=1e-13)
    ycheck = np.random.default_rng(1).standard_normal(op.m)
    np.testing.assert_allclose(op.backproject(ycheck)[d["aty_idx"]], d["aty_val"], rtol=1e-11, atol=1e-10)
    x, hist = O.cgls(op, b, 10)
    np.testing.assert_allclose(hist, d["cgls10_hist"], rtol=1e-8)
    assert rel_l2(x, d["cgls10_x"]) <= 1e-8
    scale = O.jacobi_scale(op)
    xl, hl = O.lsqr(op, b, 10, scale=scale)
    np.testing.assert_allclose(hl, d["lsqrj10_hist"], rtol=1e-7)
    assert rel_l2(xl, d["lsqrj10_x"]) <= 1e-7
    xp, hp = O.psirt(op, b, 10)
    np.testing.assert_allclose(hp, d["psirt10_hist"], rtol=1e-9)
    assert rel_l2(xp, d["psirt10_x"]) <= 1e-9


def test_small_instance_solvers(small):
    d, op = small
    b = d["solver_b"]
    x, h = O.cgls(op, b, 25)
    np.testing.assert_allclose(h, d["cgls25_hist"], rtol=1e-8)
    assert rel_l2(x, d["cgls25_x"]) <= 1e-8
    x, h = O.lsqr(op, b, 25)
    np.testing.assert_allclose(h, d["lsqr25_hist"], rtol=1e-7)
    x, h = O.lsqr(op, b, 25, scale=O.jacobi_scale(op))
    np.testing.assert_allclose(h, d["lsqrj25_hist"], rtol=1e-7)
    x, h = O.psirt(op, b, 7)
    np.testing.assert_allclose(h, d["psirt7_hist"], rtol=1e-10)
    assert rel_l2(x, d["psirt7_x"]) <= 1e-10
    assert O.normal_spectral_radius(op) == pytest.approx(float(d["rho"]), rel=1e-12)


def test_config1_cgls(golden):
    from _helpers import baseline_geometry

    d = golden("config1")
    vg, tr = baseline_geometry(64, 90, 128, 96)
    assert vg.voxel_size[0] == pytest.approx(float(d["voxel_size"][0]))
    op = O.OracleOperator(vg, tr, workers=8)
    b = op.project(O.shepp_logan_phantom(vg))
    np.testing.assert_allclose(b[d["b_idx"]], d["b_val"], rtol=1e-12, atol=1e-12)
    x, hist = O.cgls(op, b, 10)
    np.testing.assert_allclose(hist, d["cgls10_hist"], rtol=1e-8)
    np.testing.assert_allclose(x[d["cgls10_x_idx"]], d["cgls10_x_val"], rtol=1e-7, atol=1e-9)
