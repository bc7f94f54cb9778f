"""The sided boundary backprojector (csrc/backproject.cu k_bp_sided) against the fp64 oracle.

The plan selects it by waste (config 3: GS = 3, config 5: GS = 2); here it is forced with
CBCT_BP_GS on centred BASELINE-geometry view subsets, on a detector with a flat row (odd nv,
the reference's axis-parallel ray, operator.py:87-89) and with a principal-point offset (an
arbitrary fractional row centre), at both GS values, for A^T (mode 1) and diag(A^T A) (mode 2, the
squared-weight boundary form).  Bar: the north star's 1e-4 max-rel (operator.py:209-233, 353-362),
bitwise-deterministic reruns, and the norm partials of the epilogue.
"""

import numpy as np
import pytest

from _helpers import baseline_geometry, max_rel, rel_l2

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _geoms():
    import paper_2110_13526_b200 as P

    out = {
        "config2_views": baseline_geometry(256, 360, 512, 384, views=(87, 5)),
        "config3_views": baseline_geometry(512, 720, 616, 480, views=(300, 2)),
        "flat_row": baseline_geometry(256, 360, 512, 383, views=(40, 3)),
        # config-5 cells (0.215 mm) and detector on a 32-slice slab centred on the source plane
        "config5_slab": baseline_geometry(1024, 1440, 1024, 768, views=(700, 2), zslab=(496, 32)),
    }
    vg, tr0 = baseline_geometry(256, 360, 512, 384, views=(200, 3))
    det = P.DetectorGeometry(512, 384, tr0.detector.pixel_size, (0.37, -1.13))
    out["principal_offset"] = (vg, P.make_circular_trajectory(tr0.sid, tr0.sdd, 3, tr0.start_angle,
                                                              tr0.angular_span, det))
    return out


@pytest.mark.parametrize("gs", [2, 3])
@pytest.mark.parametrize("name", ["config2_views", "config3_views", "flat_row", "principal_offset", "config5_slab"])
def test_sided_against_oracle(name, gs, monkeypatch):
    import torch

    from paper_2110_13526_b200.operator import CbctOperator, ProjectionStack

    monkeypatch.setenv("CBCT_BP_GS", str(gs))
    vg, tr = _geoms()[name]
    op = CbctOperator(vg, tr)
    assert op.info.bp_closed_form == 1 and op.info.bp_sided_gs == gs
    y = np.random.default_rng(1).standard_normal(op.m).astype(np.float32).astype(np.float64)
    got = op.backproject(ProjectionStack(tr, y)).data
    want = O.OracleOperator(vg, tr).backproject(y)
    assert max_rel(got, want) <= 1e-4, (name, gs, max_rel(got, want))
    assert rel_l2(got, want) <= 2e-5, (name, gs, rel_l2(got, want))
    # mode 2: diag(A^T A) in the squared-weight boundary form (operator.py:166-167, 353-362)
    got, want = op.normal_diagonal().data, O.OracleOperator(vg, tr).normal_diagonal()
    assert max_rel(got, want) <= 1e-4, (name, gs, "normal_diagonal", max_rel(got, want))
    # squared weights double the straddle fraction's relative error (config-5 cells, 2 views: 2.8e-5)
    assert rel_l2(got, want) <= 5e-5, (name, gs, "normal_diagonal", rel_l2(got, want))
    # determinism and the fused norm: same device buffers twice, ||A^T y||^2 from the epilogue
    yi = op.proj_to_internal(y)
    r1, r2 = op.new_volume(), op.new_volume()
    n1 = op.backproject_internal(yi, r1, norm2=True)
    op.backproject_internal(yi, r2)
    assert torch.equal(r1, r2)
    assert n1 == pytest.approx(float((r1.double() ** 2).sum()), rel=1e-12)


def test_sided_matches_boundary_kernel_closely(monkeypatch):
    """The two boundary kernels evaluate the same closed form with different fp32 rounding (sign
    blend and two-word z vs compile-time side and exact integer z): rare boundary
    classifications differ by a sliver (3e-5 of the maximum at worst), the bulk agrees to 1e-6."""
    import torch

    from paper_2110_13526_b200.operator import CbctOperator

    vg, tr = baseline_geometry(512, 720, 616, 480, views=(0, 4))
    monkeypatch.setenv("CBCT_BP_SIDED_OFF", "1")
    a = CbctOperator(vg, tr)
    assert a.info.bp_sided_gs == 0
    monkeypatch.delenv("CBCT_BP_SIDED_OFF")
    b = CbctOperator(vg, tr)
    assert b.info.bp_sided_gs == 3
    y = a.proj_to_internal(np.random.default_rng(7).standard_normal(a.m))
    ra, rb = a.new_volume(), b.new_volume()
    a.backproject_internal(y, ra)
    b.backproject_internal(y, rb)
    assert float((ra - rb).abs().max() / ra.abs().max()) <= 1e-4
    assert float(torch.linalg.norm(ra - rb) / torch.linalg.norm(ra)) <= 2e-6


@pytest.mark.parametrize("gs", [2, 3])
@pytest.mark.parametrize("zslab", [(300, 64), (100, 64)])
def test_sided_one_sided_slabs(zslab, gs, monkeypatch):
    """A z slab entirely above (k0 = 0) or below (k0 = nz + 1) the source plane at config-3 cell
    sizes: only one side's groups carry voxels, the boundary heights start at z_off != 0 (folded
    into the per-crossing row offsets), mode 1 and mode 2 against the oracle."""
    from paper_2110_13526_b200.operator import CbctOperator, ProjectionStack

    monkeypatch.setenv("CBCT_BP_GS", str(gs))
    vg, tr = baseline_geometry(512, 720, 616, 480, views=(50, 2), zslab=zslab)
    op = CbctOperator(vg, tr)
    assert op.info.bp_closed_form == 1 and op.info.bp_sided_gs == gs
    ref = O.OracleOperator(vg, tr)
    y = np.random.default_rng(3).standard_normal(op.m).astype(np.float32).astype(np.float64)
    got, want = op.backproject(ProjectionStack(tr, y)).data, ref.backproject(y)
    assert max_rel(got, want) <= 1e-4, (zslab, gs, max_rel(got, want))
    got, want = op.normal_diagonal().data, ref.normal_diagonal()
    assert max_rel(got, want) <= 1e-4, (zslab, gs, "normal_diagonal", max_rel(got, want))


def test_sided_not_used_when_the_source_plane_cuts_a_voxel(monkeypatch):
    """Both sides present but z = 0 inside a voxel (an off-centre slab): the plan must keep
    k_bp_boundary even when GS is forced, and the result still matches the oracle."""
    from paper_2110_13526_b200.operator import CbctOperator, ProjectionStack
    from paper_2110_13526_b200.geometry import VolumeGeometry

    monkeypatch.setenv("CBCT_BP_GS", "3")
    vg0, tr = baseline_geometry(512, 720, 616, 480, views=(10, 2))
    p = vg0.voxel_size[2]
    vg = VolumeGeometry(vg0.nx, vg0.ny, 40, vg0.voxel_size, (0.0, 0.0, 0.37 * p))
    op = CbctOperator(vg, tr)
    assert op.info.bp_closed_form == 1 and op.info.bp_sided_gs == 0
    y = np.random.default_rng(4).standard_normal(op.m).astype(np.float32).astype(np.float64)
    got, want = op.backproject(ProjectionStack(tr, y)).data, O.OracleOperator(vg, tr).backproject(y)
    assert max_rel(got, want) <= 1e-4, max_rel(got, want)
