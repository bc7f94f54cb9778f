import pathlib, sys
ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
from _helpers import geom_from_golden, load_golden, rel_l2
from oracle import oracle as O
import paper_2110_13526_b200 as P
t = load_golden("config2_lsqrj_trajectory")
vg, tr = geom_from_golden(t)
op64 = P.CbctOperator(vg, tr, precision="f64")
b = op64.project(P.Volume(vg, O.shepp_logan_phantom(vg))).data.astype(np.float32).astype(np.float64)
for prec in ("f64", "f32"):
    op = op64 if prec == "f64" else P.CbctOperator(vg, tr)
    for K in (10, 20, 30, 40):
        rep = P.solve(op, P.ProjectionStack(tr, b), P.SolverConfig(method="lsqr", max_iterations=K, jacobi_precondition=True))
        h = np.array([r.rel_discrepancy for r in rep.history])
        hr = t["lsqrj_w8_hist"][: K + 1]
        rel = rel_l2(rep.final_x.data[:: int(t["x_stride"])], t[f"lsqrj_w8_x{K}_sample"])
        print(prec, K, "x", f"{rel:.3e}", "hist maxdev", f"{np.abs(h / hr - 1).max():.2e}", "h[:11]", f"{np.abs(h[:11] / hr[:11] - 1).max():.2e}", "e", h[-1], hr[-1], flush=True)
