"""A and A^T max-rel vs the oracle on a BASELINE config view subset:
python tools/diag_subset.py N V nu nv view0 nviews [z0 nzs]"""
import pathlib, sys
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
from _helpers import baseline_geometry, max_rel
import paper_2110_13526_b200 as P
from oracle import oracle as O

N, V, nu, nv, v0, k = (int(a) for a in sys.argv[1:7])
zslab = (int(sys.argv[7]), int(sys.argv[8])) if len(sys.argv) > 8 else None
vg, tr = baseline_geometry(N, V, nu, nv, views=(v0, k), zslab=zslab)
op, ref = P.CbctOperator(vg, tr), O.OracleOperator(vg, tr)
x = np.random.default_rng(0).random(op.n).astype(np.float32).astype(np.float64)
y = np.random.default_rng(1).standard_normal(op.m).astype(np.float32).astype(np.float64)
xa = op.project(P.Volume(vg, x)).data
xa = xa.cpu().numpy() if hasattr(xa, "cpu") else np.asarray(xa)
ya = op.backproject(P.ProjectionStack(tr, y)).data
ya = ya.cpu().numpy() if hasattr(ya, "cpu") else np.asarray(ya)
rp, rb = ref.project(x), ref.backproject(y)
e = np.abs(ya.ravel() - rb.ravel())
i = int(np.argmax(e))
print(f"closed={op.info.bp_closed_form} A maxrel {max_rel(xa, rp):.3e}  AT maxrel {max_rel(ya, rb):.3e} "
      f"l2 {np.linalg.norm(e) / np.linalg.norm(rb):.3e} worst voxel (z, y, x) {tuple(int(v) for v in np.unravel_index(i, (vg.nz, vg.ny, vg.nx)))} "
      f"ref {rb.ravel()[i]:.5e} got {ya.ravel()[i]:.5e}")
# z-neighbours of the worst voxel (reference layout (nz, ny, nx), x fastest)
iz_, iy_, ix_ = np.unravel_index(i, (vg.nz, vg.ny, vg.nx))
for dz in range(-2, 3):
    z2 = iz_ + dz
    if 0 <= z2 < vg.nz:
        j = (z2 * vg.ny + iy_) * vg.nx + ix_
        print(f"   z {z2:4d}: ref {rb.ravel()[j]: .6e} got {ya.ravel()[j]: .6e} err {ya.ravel()[j] - rb.ravel()[j]: .3e}")
