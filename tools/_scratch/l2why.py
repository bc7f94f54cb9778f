import pathlib, sys
ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
from _helpers import geom_from_golden, load_golden, rel_l2
from oracle import oracle as O
import paper_2110_13526_b200 as P
t = load_golden("config2_lsqrj_trajectory")
vg, tr = geom_from_golden(t)
st = int(t["x_stride"])
op64 = P.CbctOperator(vg, tr, precision="f64")
b = op64.project(P.Volume(vg, O.shepp_logan_phantom(vg))).data.astype(np.float32).astype(np.float64)
diag = op64.normal_diagonal().data[::st]
op = P.CbctOperator(vg, tr)
d32 = op.normal_diagonal().data[::st]
print("diag f32 vs f64 max-rel", np.abs(d32 - diag).max() / diag.max(), "rel-l2", np.linalg.norm(d32 - diag) / np.linalg.norm(diag))
rep = P.solve(op, P.ProjectionStack(tr, b), P.SolverConfig(method="lsqr", max_iterations=10, jacobi_precondition=True))
g = t["lsqrj_w8_x10_sample"].astype(np.float64)
d = rep.final_x.data[::st] - g
tot = np.sum(d * d)
mx = diag.max()
for thr in (1e-6, 1e-4, 1e-3, 1e-2, 1e-1):
    m = diag < thr * mx
    print(f"diag < {thr:g} max: {m.mean()*100:.2f}% of voxels, {np.sum(d[m]**2)/tot*100:.1f}% of the error^2")
rel = np.abs(d) / (np.abs(g) + 1e-12)
i = np.argsort(-np.abs(d))[:5]
print("largest |d|:", d[i], "golden", g[i], "diag/max", diag[i] / mx)
print("rel_l2", np.linalg.norm(d) / np.linalg.norm(g))
