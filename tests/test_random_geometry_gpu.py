"""Seeded random geometries against the fp64 oracle: every plan choice the geometry drives.

Each seed draws a circular-orbit geometry the reference accepts (geometry.py:144-164): unequal
nx/ny/nz, anisotropic voxels, a shifted volume (half the seeds with a voxel boundary exactly on the
source plane z = 0, which selects the sided backprojector), a detector with odd or even row count
(odd with no vertical offset puts a row at the source height: the flat-ray path), a principal-point offset and a partial
or full angular span.  A, A^T and diag(A^T A) are held to the north-star 1e-4 max-rel
(operator.py:190-233, 353-362), and the plan's kernel choices are recorded in the failure message.
"""

import numpy as np
import pytest

from _helpers import max_rel, rel_l2

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _geometry(seed):
    import paper_2110_13526_b200 as P

    g = np.random.default_rng(1000 + seed)
    even = seed % 2 == 0
    nx, ny, nz = (int(v) for v in g.integers(24, 120, size=3))
    # even seeds: voxels short against the source distance (the closed-form straddle, eps <= 3e-3),
    # z pitch a multiple of 1/64 mm so the boundary placed on z = 0 is exact; odd seeds: anything
    vox = [float(v) for v in g.uniform(0.5, 1.1, size=3)] if even else [float(v) for v in g.uniform(0.6, 1.6, size=3)]
    if even:
        vox[2] = round(vox[2] * 64.0) / 64.0
    vox = tuple(vox)
    shift_xy = g.uniform(-0.15, 0.15, size=2) * np.array([nx * vox[0], ny * vox[1]])
    if even:
        # a voxel boundary on z = 0: the lower corner at -k voxels for an integer k inside the volume
        k = int(g.integers(0, nz + 1))
        zc = -k * vox[2] + 0.5 * nz * vox[2]
    else:
        zc = float(g.uniform(-0.3, 0.3) * nz * vox[2])
    vg = P.VolumeGeometry(nx, ny, nz, vox, (float(shift_xy[0]), float(shift_xy[1]), zc))
    if even:
        assert vg.corner()[2] + k * vox[2] == 0.0
    nu = int(g.integers(32, 260))
    nv = int(g.integers(16, 200)) | (1 if seed % 3 == 0 else 0)
    sid = float(g.uniform(700.0, 1000.0) if even else g.uniform(500.0, 900.0))
    sdd = sid * float(g.uniform(1.3, 1.9))
    # the detector sees the whole volume (plus margin), as in every BASELINE config
    half = 0.5 * np.sqrt((nx * vox[0]) ** 2 + (ny * vox[1]) ** 2) + np.abs(shift_xy).max()
    pu = float(2.2 * half * sdd / sid / nu)
    hz = 0.5 * nz * vox[2] + abs(zc)
    pv = float(2.2 * hz * sdd / (sid - half) / nv)
    off_v = float(g.uniform(-2.0, 2.0))
    off = (float(g.uniform(-2.0, 2.0)), 0.0 if nv % 2 else off_v)  # odd nv, no v offset: a flat row
    det = P.DetectorGeometry(nu, nv, (pu, pv), off)
    nviews = int(g.integers(1, 5))
    span = float(g.uniform(0.2, 2 * np.pi))
    tr = P.make_circular_trajectory(sid, sdd, nviews, float(g.uniform(0, 2 * np.pi)), span, det)
    return vg, tr


@pytest.mark.parametrize("seed", range(24))
def test_random_geometry_against_oracle(seed, monkeypatch):
    """Even seeds (a boundary on z = 0) force the sided backprojector with GS = 2 or 3 (the plan
    would otherwise pick it only where few group slots are wasted); odd seeds take the plan's own
    choice (k_bp_boundary: z = 0 cuts a voxel)."""
    from paper_2110_13526_b200.operator import CbctOperator, ProjectionStack
    from paper_2110_13526_b200.phantom import Volume

    vg, tr = _geometry(seed)
    if seed % 2 == 0:
        monkeypatch.setenv("CBCT_BP_GS", str(2 + (seed // 2) % 2))
    op, ref = CbctOperator(vg, tr), O.OracleOperator(vg, tr)
    i = op.info
    if seed % 2 == 0 and i.bp_fast_path:
        assert i.bp_sided_gs == 2 + (seed // 2) % 2, seed
    plan = (f"seed {seed}: vol {vg.nx}x{vg.ny}x{vg.nz} det {tr.detector.nu}x{tr.detector.nv} V {tr.n_views}; "
            f"proj_chunk {i.proj_chunk} bp_fast {i.bp_fast_path} closed {i.bp_closed_form} "
            f"groups {i.bp_groups} sided {i.bp_sided_gs}")
    x = np.random.default_rng(seed).random(op.n).astype(np.float32).astype(np.float64)
    y = np.random.default_rng(seed + 1).standard_normal(op.m).astype(np.float32).astype(np.float64)
    got, want = op.project(Volume(vg, x)).data, ref.project(x)
    assert max_rel(got, want) <= TOL, (plan, "A", max_rel(got, want))
    got, want = op.backproject(ProjectionStack(tr, y)).data, ref.backproject(y)
    assert max_rel(got, want) <= TOL, (plan, "A^T", max_rel(got, want))
    assert rel_l2(got, want) <= 2e-5, (plan, "A^T rel-L2", rel_l2(got, want))
    got, want = op.normal_diagonal().data, ref.normal_diagonal()
    assert max_rel(got, want) <= TOL, (plan, "normal_diagonal", max_rel(got, want))


@pytest.mark.parametrize("seed", range(0, 24, 3))
def test_random_geometry_f64_path(seed):
    """The reference-precision path (csrc/f64.cu) on the same geometries: A bit for bit the
    oracle's (the reference's fp64 Siddon sum, operator.py:190-206), A^T and diag(A^T A) to
    fp64 summation-order rounding."""
    from paper_2110_13526_b200.operator import CbctOperator, ProjectionStack
    from paper_2110_13526_b200.phantom import Volume

    vg, tr = _geometry(seed)
    op, ref = CbctOperator(vg, tr, precision="f64"), O.OracleOperator(vg, tr)
    x = np.random.default_rng(seed).random(op.n)
    y = np.random.default_rng(seed + 1).standard_normal(op.m)
    got, want = op.project(Volume(vg, x)).data, ref.project(x)
    assert np.array_equal(got, want), (seed, max_rel(got, want))
    got, want = op.backproject(ProjectionStack(tr, y)).data, ref.backproject(y)
    assert max_rel(got, want) <= 1e-13, (seed, max_rel(got, want))
    got, want = op.normal_diagonal().data, ref.normal_diagonal()
    assert max_rel(got, want) <= 1e-13, (seed, max_rel(got, want))


@pytest.mark.parametrize("case", ["nv2048", "nz2048", "nu1_one_view", "thin_slab_wide_det"])
def test_size_limits_against_oracle(case):
    """The largest detector height and volume depth the plan accepts (nv, nz <= 2048: four rays / voxels
    per thread), a single detector column in a single view, and a one-slice volume under a wide
    detector: A, A^T and diag(A^T A) against the oracle."""
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.operator import CbctOperator, ProjectionStack
    from paper_2110_13526_b200.phantom import Volume

    if case == "nv2048":
        vg = P.VolumeGeometry(12, 10, 40, (2.0, 2.0, 2.0))
        det = P.DetectorGeometry(16, 2048, (2.0, 0.07))
        tr = P.make_circular_trajectory(400.0, 700.0, 2, 0.3, 1.0, det)
    elif case == "nz2048":
        vg = P.VolumeGeometry(6, 7, 2048, (2.0, 2.0, 0.05))
        det = P.DetectorGeometry(20, 300, (1.5, 0.6))
        tr = P.make_circular_trajectory(400.0, 700.0, 2, 0.3, 1.0, det)
    elif case == "nu1_one_view":
        vg = P.VolumeGeometry(30, 30, 30, (1.0, 1.0, 1.0), (0.4, -0.3, 0.2))
        det = P.DetectorGeometry(1, 64, (1.0, 1.0), (0.3, 0.0))
        tr = P.make_circular_trajectory(300.0, 500.0, 1, 0.7, 0.0, det)
    else:
        vg = P.VolumeGeometry(50, 40, 1, (1.0, 1.0, 1.0))
        det = P.DetectorGeometry(120, 101, (0.8, 0.8))
        tr = P.make_circular_trajectory(300.0, 500.0, 3, 0.0, 2.0, det)
    op, ref = CbctOperator(vg, tr), O.OracleOperator(vg, tr)
    x = np.random.default_rng(5).random(op.n).astype(np.float32).astype(np.float64)
    y = np.random.default_rng(6).standard_normal(op.m).astype(np.float32).astype(np.float64)
    got, want = op.project(Volume(vg, x)).data, ref.project(x)
    assert max_rel(got, want) <= TOL, (case, "A", max_rel(got, want))
    got, want = op.backproject(ProjectionStack(tr, y)).data, ref.backproject(y)
    assert max_rel(got, want) <= TOL, (case, "A^T", max_rel(got, want))
    got, want = op.normal_diagonal().data, ref.normal_diagonal()
    assert max_rel(got, want) <= TOL, (case, "normal_diagonal", max_rel(got, want))
