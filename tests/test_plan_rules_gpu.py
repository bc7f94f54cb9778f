"""Launch shapes the plan picks at the BASELINE sizes (csrc/plan.cu; the measurements behind each
rule are in profiles/history.md): prefix-projector chunk C = 16 unless two such CTAs no longer fit
an SM (then 8), boundary groups per warp from {3, 4, 6} by least waste with ties to the larger G,
view batches of the backprojector growing with the ray-prefix table, and the sided boundary kernel
(GS = 3, else 2, below + above groups per warp) where at most 10% of its group slots are wasted."""

import gc

import pytest
import torch

from _helpers import baseline_geometry

pytestmark = pytest.mark.gpu

# config: (N, V, nu, nv) -> (chunk, groups, view batches, sided GS)
CASES = {
    1: ((64, 90, 128, 96), (16, 3, 1, 0)),     # table-form straddle: k_bp_boundary
    2: ((256, 360, 512, 384), (16, 3, 2, 0)),  # 5 + 5 groups: 2 of 12 sided slots wasted
    3: ((512, 720, 616, 480), (16, 6, 2, 3)),
    5: ((1024, 1440, 1024, 768), (8, 6, 4, 3)),
}


@pytest.mark.parametrize("cfg", sorted(CASES))
def test_plan_launch_shapes(cfg, monkeypatch):
    from paper_2110_13526_b200.operator import CbctOperator

    for var in ("CBCT_PROJ_Q_C", "CBCT_BP_G", "CBCT_BP_VBATCH", "CBCT_PROJ_Q", "CBCT_BP_TABLE", "CBCT_BP_GS",
                "CBCT_BP_SIDED_OFF"):
        monkeypatch.delenv(var, raising=False)
    (n, v, nu, nv), want = CASES[cfg]
    op = CbctOperator(*baseline_geometry(n, v, nu, nv))
    info = op.info
    assert (info.proj_chunk, info.bp_groups, info.bp_view_batches, info.bp_sided_gs) == want
    assert info.bp_fast_path == 1 and info.bp_closed_form == (0 if cfg == 1 else 1)
    del op, info
    gc.collect()
    torch.cuda.empty_cache()
