"""View-batched backprojector (plan.bp_vbatch, backproject.cu): A^T split into several launches
over contiguous runs of each cell's view-ordered entries, later launches accumulating.  The test
geometries are too small for the plan to batch by itself, so the batch count is forced through
CBCT_BP_VBATCH and compared with the single launch, the oracle and the norm partials that only
the last launch writes, for both straddle forms."""

import numpy as np
import pytest
import torch

from _helpers import baseline_geometry, max_rel

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _op(vg, tr, nb, monkeypatch):
    from paper_2110_13526_b200.operator import CbctOperator

    monkeypatch.setenv("CBCT_BP_VBATCH", str(nb))
    try:
        return CbctOperator(vg, tr)
    finally:
        monkeypatch.delenv("CBCT_BP_VBATCH")


GEOMS = {
    # config-2 cells (closed-form straddle fraction)
    "closed": lambda: baseline_geometry(256, 360, 512, 384, views=(87, 5)),
    # config-3 cells and full columns: the sided kernel (k_bp_sided, GS = 3, four crossings per shuffle)
    "sided": lambda: baseline_geometry(512, 720, 616, 480, views=(200, 3)),
    # config-1 cells are long against the source distance: the 1/rz-table straddle form
    "table": lambda: baseline_geometry(64, 90, 128, 96, views=(0, 12)),
}


@pytest.mark.parametrize("form", ["closed", "table", "sided"])
@pytest.mark.parametrize("nb", [2, 3, 7])
def test_view_batches_match_single_launch_and_oracle(form, nb, monkeypatch):
    from paper_2110_13526_b200.operator import ProjectionStack

    vg, tr = GEOMS[form]()
    one, many = _op(vg, tr, 1, monkeypatch), _op(vg, tr, nb, monkeypatch)
    assert one.info.bp_fast_path == 1 and one.info.bp_closed_form == (0 if form == "table" else 1)
    assert one.info.bp_sided_gs == (3 if form == "sided" else 0)
    y = np.random.default_rng(nb).standard_normal(one.m).astype(np.float32).astype(np.float64)
    a = one.backproject(ProjectionStack(tr, y)).data
    b = many.backproject(ProjectionStack(tr, y)).data
    # same per-entry terms, summed per batch then added: fp32 reassociation only (the sided kernel
    # also regroups the crossings that share a shuffle at each batch boundary)
    assert max_rel(b, a) <= (5e-6 if form == "sided" else 1e-6), max_rel(b, a)
    want = O.OracleOperator(vg, tr).backproject(y)
    assert max_rel(b, want) <= TOL, max_rel(b, want)
    # ||A^T y||^2 from the partials of the last launch equals the sum over the accumulated volume
    yi = many.proj_to_internal(y)
    r = many.new_volume()
    n2 = many.backproject_internal(yi, r, norm2=True)
    direct = float((many.volume_from_internal(r, torch.float64) ** 2).sum())
    assert abs(n2 - direct) <= 1e-6 * direct, (n2, direct)
    # deterministic: a rerun is bitwise equal
    r2 = many.new_volume()
    many.backproject_internal(yi, r2)
    assert torch.equal(r, r2)
