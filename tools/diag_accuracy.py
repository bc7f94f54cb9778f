"""Accuracy diagnostic: GPU operator errors vs the fp64 oracle and CGLS drift (desk, config 1)."""
import os, sys, pathlib
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
from _helpers import load_golden, geom_from_golden, baseline_geometry, max_rel, rel_l2
from oracle import oracle as O
import paper_2110_13526_b200 as P
import paper_2110_13526_b200.solvers as S

def report(name, vg, tr, golden_hist=None, K=10):
    op, ref = P.CbctOperator(vg, tr), O.OracleOperator(vg, tr)
    x = np.random.default_rng(0).random(op.n)
    y = np.random.default_rng(1).standard_normal(op.m)
    ax, axr = op.project(P.Volume(vg, x)).data, ref.project(x)
    aty, atyr = op.backproject(P.ProjectionStack(tr, y)).data, ref.backproject(y)
    pe = np.abs(aty - atyr) / np.maximum(np.abs(atyr), 1e-30)
    print(f"{name}: A maxrel {max_rel(ax, axr):.2e} l2 {rel_l2(ax, axr):.2e} | AT maxrel {max_rel(aty, atyr):.2e} "
          f"l2 {rel_l2(aty, atyr):.2e} per-voxel rel p50 {np.median(pe):.1e} p99 {np.quantile(pe, .99):.1e}")
    b = ref.project(O.shepp_logan_phantom(vg))
    rep = S.cgls(op, P.ProjectionStack(tr, b), S.SolverConfig(method="cgls", max_iterations=K))
    h = np.array([r.rel_discrepancy for r in rep.history])
    xr, hr = O.cgls(ref, b, K)
    print(f"   CGLS{K}: hist maxdev {np.abs(h / np.array(hr) - 1).max():.2e}  x rel {rel_l2(rep.final_x.data, xr):.2e}")

d = load_golden("desk"); vg, tr = geom_from_golden(d)
report("desk", vg, tr)
report("config1", *baseline_geometry(64, 90, 128, 96))
d = load_golden("adjoint_instance"); report("adjoint", *geom_from_golden(d))
