"""Generate golden vectors from the REFERENCE implementation (cbctkit 0.1.0).

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

It imports the reference from a scratch copy (``baseline/_ref/pkg`` or
``/tmp``) with ``NUMBA_CACHE_DIR`` pointed at /tmp, so nothing is written
into the read-only reference tree.  Outputs
``tests/golden/*.npz``; large vectors are stored as seeded index samples plus
norms so the fixtures stay small.
"""

from __future__ import annotations

import os
import pathlib
import shutil
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF = pathlib.Path("/root/reference/pkg")


def _import_reference():
    scratch = REPO / "baseline" / "_ref" / "pkg"
    if not scratch.exists():
        scratch.parent.mkdir(parents=True, exist_ok=True)
        shutil.copytree(REF, scratch)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.path.insert(0, str(scratch / "src"))
    import cbctkit  # noqa: F401

    return scratch


def _sample(vec, k=4096, seed=12345):
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(vec.size, size=min(k, vec.size), replace=False)).astype(np.int64)
    return idx, vec[idx].copy()


def main():
    scratch = _import_reference()
    from cbctkit.geometry import DetectorGeometry, VolumeGeometry, load_config, make_circular_trajectory
    from cbctkit.operator import CbctOperator, ProjectionStack
    from cbctkit.phantom import Volume, generate_phantom, shepp_logan_3d
    from cbctkit.solvers import SolverConfig, cgls, lsqr, normal_spectral_radius, psirt

    sys.path.insert(0, str(scratch / "tests"))
    from oracle import assemble_matrix  # the reference's own dense oracle (tests/oracle.py)

    def geom_dict(vg, tr):
        d = tr.detector
        return dict(
            vol=np.array([vg.nx, vg.ny, vg.nz], dtype=np.int64),
            voxel_size=np.array(vg.voxel_size, dtype=np.float64),
            center_offset=np.array(vg.center_offset, dtype=np.float64),
            det=np.array([d.nu, d.nv], dtype=np.int64),
            pixel_size=np.array(d.pixel_size, dtype=np.float64),
            principal_point_offset=np.array(d.principal_point_offset, dtype=np.float64),
            traj=np.array([tr.sid, tr.sdd, tr.n_views, tr.start_angle, tr.angular_span], dtype=np.float64),
        )

    # 1. small_instance (tests/conftest.py:41-51) -- full vectors + dense A
    vg = VolumeGeometry(6, 6, 6, voxel_size=(2.0, 2.0, 2.0))
    det = DetectorGeometry(8, 8, pixel_size=(3.0, 3.0))
    tr = make_circular_trajectory(100.0, 200.0, 8, 0.1, 2 * np.pi, det)
    op = CbctOperator(vg, tr, workers=3)
    A = assemble_matrix(vg, tr)
    x = np.random.default_rng(0).standard_normal(op.n)
    y = np.random.default_rng(1).standard_normal(op.m)
    rows, cols = np.nonzero(A)
    b1 = ProjectionStack(tr)
    b1.data[137] = 2.5
    seg_idx, seg_len = op.ray_segments(*(lambda r: (r // 64, r % 8, (r % 64) // 8))(137))
    xt = np.random.default_rng(2024).random(op.n)
    bb = ProjectionStack(tr, A @ xt)
    rep = cgls(op, bb, SolverConfig(method="cgls", max_iterations=25))
    rep_l = lsqr(op, bb, SolverConfig(method="lsqr", max_iterations=25))
    rep_lj = lsqr(op, bb, SolverConfig(method="lsqr", max_iterations=25, jacobi_precondition=True))
    rep_p = psirt(op, bb, SolverConfig(method="psirt", max_iterations=7))
    np.savez_compressed(
        HERE / "small_instance.npz", **geom_dict(vg, tr),
        x=x, Ax=op.project(Volume(vg, x)).data, y=y,
        ATy=op.backproject(ProjectionStack(tr, y)).data,
        row_sums=op.row_sums().data, col_sums=op.col_sums().data,
        normal_diagonal=op.normal_diagonal().data,
        dense_rows=rows.astype(np.int32), dense_cols=cols.astype(np.int32), dense_vals=A[rows, cols],
        pixel137_backprojection=op.backproject(b1).data,
        seg137_idx=seg_idx, seg137_len=seg_len,
        solver_xtrue=xt, solver_b=bb.data,
        cgls25_x=rep.final_x.data, cgls25_hist=np.array([r.rel_discrepancy for r in rep.history]),
        lsqr25_x=rep_l.final_x.data, lsqr25_hist=np.array([r.rel_discrepancy for r in rep_l.history]),
        lsqrj25_x=rep_lj.final_x.data, lsqrj25_hist=np.array([r.rel_discrepancy for r in rep_lj.history]),
        psirt7_x=rep_p.final_x.data, psirt7_hist=np.array([r.rel_discrepancy for r in rep_p.history]),
        rho=np.array(normal_spectral_radius(op)),
    )

    # 2. adjoint_instance (tests/test_acceptance.py:40-45) -- full vectors
    vg = VolumeGeometry(32, 32, 16, voxel_size=(5.0, 5.0, 10.0))
    det = DetectorGeometry(48, 32, pixel_size=(6.0, 6.0))
    tr = make_circular_trajectory(749.0, 1198.0, 16, 0.05, 2 * np.pi, det)
    op = CbctOperator(vg, tr, workers=8)
    x = np.random.default_rng(0).random(op.n)
    y = np.random.default_rng(1).standard_normal(op.m)
    np.savez_compressed(
        HERE / "adjoint_instance.npz", **geom_dict(vg, tr),
        x=x, Ax=op.project(Volume(vg, x)).data, y=y, ATy=op.backproject(ProjectionStack(tr, y)).data,
        row_sums=op.row_sums().data, col_sums=op.col_sums().data, normal_diagonal=op.normal_diagonal().data,
    )

    # 3. known answers: axial chord (test_operator.py:30-36), ray miss (115-124),
    #    cone-boundary diagonal (127-136), off-centre shift (157-176)
    vg = VolumeGeometry(5, 5, 5, voxel_size=(2.0, 2.0, 2.0))
    det = DetectorGeometry(1, 1, pixel_size=(1.0, 1.0))
    tr = make_circular_trajectory(100.0, 200.0, 1, 0.0, 2 * np.pi, det)
    chord = CbctOperator(vg, tr).project(Volume(vg, np.ones(125))).data[0]
    vg2 = VolumeGeometry(2, 2, 2, voxel_size=(1.0, 1.0, 1.0))
    det2 = DetectorGeometry(32, 32, pixel_size=(2.0, 2.0))
    tr2 = make_circular_trajectory(50.0, 100.0, 2, 0.05, 2 * np.pi, det2)
    miss_rows = CbctOperator(vg2, tr2).row_sums().data
    vg3 = VolumeGeometry(16, 16, 16, voxel_size=(1.0, 1.0, 1.0))
    det3 = DetectorGeometry(24, 12, pixel_size=(1.5, 1.5))
    tr3 = make_circular_trajectory(50.0, 100.0, 12, 0.04, 2 * np.pi, det3)
    diag3 = CbctOperator(vg3, tr3).normal_diagonal().data
    np.savez_compressed(HERE / "known_answers.npz", axial_chord=np.array(chord), miss_rows=miss_rows,
                        cone_diag=diag3)

    # 4. desk scale (configs/desk_scale.cfg) -- b = A phantom, CGLS/LSQR/PSIRT histories
    vg, tr = load_config(scratch / "configs" / "desk_scale.cfg")
    op = CbctOperator(vg, tr, workers=8)
    truth = generate_phantom(shepp_logan_3d(), vg)
    b = op.project(truth)
    ycheck = np.random.default_rng(1).standard_normal(op.m)
    aty = op.backproject(ProjectionStack(tr, ycheck)).data
    c10 = cgls(op, b, SolverConfig(method="cgls", max_iterations=10, true_discrepancy_every=10))
    l10 = lsqr(op, b, SolverConfig(method="lsqr", max_iterations=10, jacobi_precondition=True))
    p10 = psirt(op, b, SolverConfig(method="psirt", max_iterations=10))
    bi, bv = _sample(b.data)
    ai, av = _sample(aty)
    np.savez_compressed(
        HERE / "desk.npz", **geom_dict(vg, tr),
        truth=truth.data.astype(np.float32),
        b_idx=bi, b_val=bv, b_norm=np.array(np.linalg.norm(b.data)), b_sum=np.array(b.data.sum()),
        aty_idx=ai, aty_val=av, aty_norm=np.array(np.linalg.norm(aty)),
        cgls10_hist=np.array([r.rel_discrepancy for r in c10.history]), cgls10_x=c10.final_x.data,
        cgls10_true10=np.array(c10.history[10].true_rel_discrepancy),
        lsqrj10_hist=np.array([r.rel_discrepancy for r in l10.history]), lsqrj10_x=l10.final_x.data,
        psirt10_hist=np.array([r.rel_discrepancy for r in p10.history]), psirt10_x=p10.final_x.data,
    )

    # 5. BASELINE config 1 (SURVEY.md 8d geometry rule): 64^3, 90 views, 128x96, CGLS 10
    N, V, nu, nv = 64, 90, 128, 96
    vg = VolumeGeometry(N, N, N, voxel_size=(220.16 / N,) * 3)
    det = DetectorGeometry(nu, nv, pixel_size=(379.456 / nu, 379.456 / nu))
    tr = make_circular_trajectory(749.0, 1198.0, V, 0.0, 2 * np.pi, det)
    op = CbctOperator(vg, tr, workers=8)
    truth = generate_phantom(shepp_logan_3d(), vg)
    b = op.project(truth)
    c10 = cgls(op, b, SolverConfig(method="cgls", max_iterations=10))
    bi, bv = _sample(b.data)
    xi, xv = _sample(c10.final_x.data)
    np.savez_compressed(
        HERE / "config1.npz", **geom_dict(vg, tr),
        b_idx=bi, b_val=bv, b_norm=np.array(np.linalg.norm(b.data)),
        cgls10_hist=np.array([r.rel_discrepancy for r in c10.history]),
        cgls10_x_idx=xi, cgls10_x_val=xv, cgls10_x_norm=np.array(np.linalg.norm(c10.final_x.data)),
    )
    for f in sorted(HERE.glob("*.npz")):
        print(f"{f.name}: {f.stat().st_size / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
