"""Kernel-only timing of A and A^T (CUDA events) for a BASELINE config: python tools/time_ops.py [cfg] [reps] [A|AT]."""
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2110_13526_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
vg, tr = bench.geometry(cfg)
op = P.CbctOperator(vg, tr, precision=os.environ.get("PREC", "f32"))
x = op.phantom_internal(P.shepp_logan_3d())
p = op.new_projections()
r = op.new_volume()
scr = op.new_bp_scratch()
y = torch.randn(op.m, device="cuda", dtype=op.dtype)


def t(fn):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


only = sys.argv[3] if len(sys.argv) > 3 else ""  # "A" or "AT": time one operator only; "D": diag(A^T A)
if only == "D":
    td = t(lambda: op.backproject_internal(None, r, mode=2))
    print(f"cfg{cfg} {os.environ.get('PREC', 'f32')}: diag(A^T A) {td:.3f} ms", flush=True)
    sys.exit(0)
ta = t(lambda: op.project_internal(x, p)) if only != "AT" else float("nan")
tat = t(lambda: op.backproject_internal(y, r, scratch=scr)) if only != "A" else float("nan")
N, V = vg.nx, tr.n_views
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("CBCT_") or k == "PREC")
print(f"cfg{cfg} {tag or 'default'}: A {ta:.3f} ms ({N**3*V/ta/1e6:.0f} GUPS)  AT {tat:.3f} ms ({N**3*V/tat/1e6:.0f} GUPS)",
      flush=True)
