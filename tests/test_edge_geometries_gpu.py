"""Degenerate and boundary shapes through the CUDA pair, against the fp64 oracle: a single z slab,
a single cell column, fewer slabs than one 31-voxel boundary group and just over one, a two-row
detector, one view, and a detector shifted so that every ray misses the volume (A = 0, A^T = 0
exactly).  Tolerance as in test_operator_gpu.py (max relative 1e-4)."""

import numpy as np
import pytest

from _helpers import max_rel

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _geom(nx, ny, nz, nu, nv, views, pix=(1.5, 1.5), offset=(0.0, 0.0), voxel=(1.0, 1.0, 1.0)):
    import paper_2110_13526_b200 as P

    vg = P.VolumeGeometry(nx, ny, nz, voxel)
    det = P.DetectorGeometry(nu, nv, pix, offset)
    return vg, P.make_circular_trajectory(60.0, 120.0, views, 0.1, 2 * np.pi, det)


SHAPES = {
    "one_slab": dict(nx=12, ny=10, nz=1, nu=24, nv=8, views=6),
    "one_cell_column": dict(nx=1, ny=1, nz=9, nu=6, nv=20, views=5),
    "one_row_of_cells": dict(nx=17, ny=1, nz=4, nu=30, nv=10, views=7),
    "nz_below_one_group": dict(nx=8, ny=8, nz=30, nu=16, nv=40, views=4),
    "nz_just_over_one_group": dict(nx=8, ny=8, nz=32, nu=16, nv=40, views=4),
    "two_detector_rows": dict(nx=10, ny=9, nz=6, nu=20, nv=2, views=5),
    "one_view": dict(nx=10, ny=12, nz=8, nu=24, nv=16, views=1),
}


@pytest.mark.parametrize("name", sorted(SHAPES))
def test_edge_shapes_against_oracle(name):
    import paper_2110_13526_b200 as P

    vg, tr = _geom(**SHAPES[name])
    op, ref = P.CbctOperator(vg, tr), O.OracleOperator(vg, tr)
    rng = np.random.default_rng(len(name))
    x = rng.random(op.n).astype(np.float32).astype(np.float64)
    y = rng.standard_normal(op.m).astype(np.float32).astype(np.float64)
    got, want = op.project(P.Volume(vg, x)).data, ref.project(x)
    assert max_rel(got, want) <= TOL, ("A", max_rel(got, want))
    got, want = op.backproject(P.ProjectionStack(tr, y)).data, ref.backproject(y)
    assert max_rel(got, want) <= TOL, ("A^T", max_rel(got, want))
    for kind in ("row_sums", "col_sums", "normal_diagonal"):
        got, want = getattr(op, kind)().data, getattr(ref, kind)()
        assert max_rel(got, want) <= TOL, (kind, max_rel(got, want))


def test_all_rays_miss_the_volume():
    import paper_2110_13526_b200 as P

    # detector shifted far above the volume's z extent: no ray meets a voxel
    vg, tr = _geom(8, 8, 4, nu=12, nv=6, views=5, offset=(0.0, 400.0))
    op = P.CbctOperator(vg, tr)
    assert not np.any(O.OracleOperator(vg, tr).row_sums())  # the oracle agrees nothing is hit
    x = np.random.default_rng(0).random(op.n)
    y = np.random.default_rng(1).standard_normal(op.m)
    assert not np.any(op.project(P.Volume(vg, x)).data)
    assert not np.any(op.backproject(P.ProjectionStack(tr, y)).data)
    assert not np.any(op.row_sums().data) and not np.any(op.col_sums().data)
