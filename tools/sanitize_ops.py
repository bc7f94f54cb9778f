"""Drive every libcbct kernel family once on small geometries, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize_ops.py.  Not a test."""
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from _helpers import baseline_geometry  # noqa: E402
import paper_2110_13526_b200 as P  # noqa: E402


def run(vg, tr, label, precision="f32", solver=True):
    op = P.CbctOperator(vg, tr, precision=precision)
    x = op.phantom_internal(P.shepp_logan_3d())
    p = op.new_projections()
    op.project_internal(x, p, norm2=True)
    r = op.new_volume()
    op.backproject_internal(p, r, norm2=True, scratch=op.new_bp_scratch() if precision == "f32" else None)
    op.backproject_internal(None, r, mode=2)
    if solver:
        b = P.operator.InternalProjections(tr, p)
        P.cgls(op, b, P.SolverConfig(method="cgls", max_iterations=2))
        P.lsqr(op, b, P.SolverConfig(method="lsqr", max_iterations=2, jacobi_precondition=True))
    torch.cuda.synchronize()
    print(f"{label} ({precision}): ok, info sided={op.info.bp_sided_gs} closed={op.info.bp_closed_form}", flush=True)


run(*baseline_geometry(64, 90, 128, 96, views=(0, 6)), "config1 6 views (table-form A^T)")
run(*baseline_geometry(256, 360, 512, 384, views=(10, 2), zslab=(120, 16)), "config2 slab (k_bp_boundary)")
os.environ["CBCT_BP_GS"] = "2"
run(*baseline_geometry(256, 360, 512, 384, views=(87, 1)), "config2 1 view (k_bp_sided GS=2)", solver=False)
os.environ["CBCT_BP_GS"] = "3"
run(*baseline_geometry(256, 360, 512, 383, views=(40, 1)), "flat row 1 view (k_bp_sided GS=3, FLAT)", solver=False)
del os.environ["CBCT_BP_GS"]
run(*baseline_geometry(64, 90, 128, 96, views=(0, 4)), "config1 4 views", precision="f64")
print("sanitize_ops done")
