"""A^T of the small golden instance vs the oracle (max-rel, worst voxels): python tools/diag_small.py"""
import pathlib, sys
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
from _helpers import geom_from_golden, load_golden
import paper_2110_13526_b200 as P
from oracle import oracle as O

d = load_golden("small_instance")
vg, tr = geom_from_golden(d)
op = P.CbctOperator(vg, tr)
ref = O.OracleOperator(vg, tr)
rng = np.random.default_rng(0)
print("geometry", vg.nx, vg.ny, vg.nz, tr.n_views, tr.detector.nu, tr.detector.nv, "bp_fast", op.info.bp_fast_path if hasattr(op, "info") else "?")
for trial in range(3):
    y = rng.standard_normal(ref.m)
    a = op.backproject(P.ProjectionStack(tr, y)).data
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b = ref.backproject(y)
    err = np.abs(a.ravel() - b.ravel())
    print(f"trial {trial}: maxrel {err.max() / np.abs(b).max():.3e} l2 {np.linalg.norm(err) / np.linalg.norm(b):.3e}")
    idx = np.argsort(err)[::-1][:4]
    for i in idx:
        print("   ", np.unravel_index(i, a.shape), f"{b.ravel()[i]:.6e} {a.ravel()[i]:.6e} {err[i]:.2e}")
