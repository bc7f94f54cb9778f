"""Probe: GPU solvers (fp32 and fp64 paths) vs the reference iterates on the committed config
goldens, next to the reference's own floor (workers 8 vs 5).  Diagnostic, not a test."""
import sys, pathlib, time
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
from _helpers import load_golden, geom_from_golden, rel_l2, max_rel
from oracle import oracle as O
import paper_2110_13526_b200 as P
import paper_2110_13526_b200.solvers as S

name = sys.argv[1] if len(sys.argv) > 1 else "config34_subset"
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["f32", "f64"]
d = load_golden(name)
tpath = ROOT / "tests" / "golden" / f"{name}_trajectory.npz"
traj = load_golden(f"{name}_trajectory") if tpath.exists() else None
vg, tr = geom_from_golden(d)
ref = O.OracleOperator(vg, tr)
t = time.time()
b = ref.project(O.shepp_logan_phantom(vg)).astype(np.float32).astype(np.float64)
print("oracle b", f"{time.time() - t:.1f}s", "b sample maxrel", max_rel(b[::int(d["b_stride"])], d["b_sample"]), flush=True)
st = int(d["x_stride"])
if traj is not None:
    for key in ("cgls", "lsqrj"):
        if f"{key}_w8_hist" in traj:
            fl = [float(traj[f"{key}_x{k}_floor"]) for k in (10, 20, 30, 40)]
            print(f"reference floor {key} (w5 vs w8) x rel at 10/20/30/40:", " ".join(f"{v:.2e}" for v in fl))
for prec in precs:
    t = time.time()
    op = P.CbctOperator(vg, tr, precision=prec)
    print(f"--- precision {prec}: plan {time.time() - t:.1f}s", flush=True)
    bs = P.ProjectionStack(tr, b)
    x = np.random.default_rng(0).random(op.n)
    t = time.time()
    ax = op.project(P.Volume(vg, x)).data
    t_a = time.time() - t
    ax_ref = ref.project(x)
    y = np.random.default_rng(1).standard_normal(op.m)
    t = time.time()
    aty = op.backproject(P.ProjectionStack(tr, y)).data
    t_at = time.time() - t
    aty_ref = ref.backproject(y)
    print(f"A maxrel {max_rel(ax, ax_ref):.2e} bitwise-equal frac {np.mean(ax == ax_ref):.4f} ({t_a:.2f}s)  "
          f"A^T maxrel {max_rel(aty, aty_ref):.2e} rel_l2 {rel_l2(aty, aty_ref):.2e} ({t_at:.2f}s)", flush=True)
    nd = op.normal_diagonal().data
    print(f"normal_diagonal maxrel {max_rel(nd, ref.normal_diagonal()):.2e}", flush=True)
    for key, method, kw in (("cgls40", "cgls", {}), ("lsqrj40", "lsqr", {"jacobi_precondition": True}),
                            ("psirt40", "psirt", {})):
        if f"{key}_hist" not in d:
            continue
        for K in ((10, 20, 30, 40) if traj is not None and method != "psirt" else (40,)):
            t = time.time()
            rep = S.solve(op, bs, S.SolverConfig(method=method, max_iterations=K, **kw))
            h = np.array([r.rel_discrepancy for r in rep.history])
            xs = rep.final_x.data[::st]
            if K == 40:
                xr, hr = d[key + "_x_sample"], d[key + "_hist"]
            else:
                tk = "cgls_w8" if method == "cgls" else "lsqrj_w8"
                xr, hr = traj[f"{tk}_x{K}_sample"], traj[f"{tk}_hist"][: K + 1]
            print(f"{key} K={K}: {time.time()-t:.1f}s hist maxdev {np.abs(h/hr-1).max():.2e} "
                  f"x rel {rel_l2(xs, xr):.2e}  e {h[-1]:.6e} vs {hr[-1]:.6e}", flush=True)
