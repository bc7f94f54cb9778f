"""Locate the worst A^T voxels of the boundary-form kernel vs the oracle and the direct kernel."""
import os, sys, pathlib
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
from _helpers import baseline_geometry, max_rel
from oracle import oracle as O
import paper_2110_13526_b200 as P

vg, tr = baseline_geometry(256, 360, 512, 384, views=(0, 6))
op, ref = P.CbctOperator(vg, tr), O.OracleOperator(vg, tr)
print("fast path:", op.info.bp_fast_path)
y = np.random.default_rng(1).standard_normal(op.m).astype(np.float32).astype(np.float64)
want = ref.backproject(y)
fast = op.backproject(P.ProjectionStack(tr, y)).data
os.environ["CBCT_BP_PRECISE"] = "1"
direct = op.backproject(P.ProjectionStack(tr, y)).data
del os.environ["CBCT_BP_PRECISE"]
mx = np.abs(want).max()
for name, got in (("fast", fast), ("direct", direct)):
    err = np.abs(got - want)
    order = np.argsort(err)[::-1][:8]
    print(name, "max_rel", err.max() / mx, "l2", np.linalg.norm(got - want) / np.linalg.norm(want))
    for j in order:
        iz, rem = divmod(j, 256 * 256); iy, ix = divmod(rem, 256)
        print(f"   voxel ({ix},{iy},{iz}) ref {want[j]: .6e} got {got[j]: .6e} err {err[j] / mx:.2e}")
