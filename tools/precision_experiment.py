"""Which precision does the Krylov iterate need to follow the reference's?  Diagnostic, not a test.

CGLS-K (the restated loop of tests/golden/make_golden_trajectory.py, solvers.py:269-358) on the
config-3/4 subset golden with every combination of
  operator: f64 (csrc/f64.cu) | f32 (the fast kernels) | f64 with fp32-rounded input and output
  vectors: fp64 | fp32
and the iterate / history compared with the reference's (workers = 8) at K = 10, 20, 30, 40.
"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import torch

from _helpers import geom_from_golden, load_golden, rel_l2
from oracle import oracle as O
import paper_2110_13526_b200 as P

d = load_golden("config34_subset")
t = load_golden("config34_subset_trajectory")
vg, tr = geom_from_golden(d)
b = O.OracleOperator(vg, tr).project(O.shepp_logan_phantom(vg)).astype(np.float32).astype(np.float64)
op64 = P.CbctOperator(vg, tr, precision="f64")
op32 = P.CbctOperator(vg, tr, precision="f32")
assert op64.vol_elems == op32.vol_elems
scr = op32.new_bp_scratch()
dev = op64.device


def A(kind, x):
    if kind == "f32":
        out = torch.empty(op32.m, device=dev)
        op32.project_internal(x.float().contiguous(), out)
        return out
    xin = x.double()
    if kind == "f64io32":
        xin = xin.float().double()
    out = torch.empty(op64.m, dtype=torch.float64, device=dev)
    op64.project_internal(xin.contiguous(), out)
    return out.float().double() if kind == "f64io32" else out


def AT(kind, y):
    if kind == "f32":
        out = torch.empty(op32.vol_elems, device=dev)
        op32.backproject_internal(y.float().contiguous(), out, scratch=scr)
        return out
    yin = y.double()
    if kind == "f64io32":
        yin = yin.float().double()
    out = torch.empty(op64.vol_elems, dtype=torch.float64, device=dev)
    op64.backproject_internal(yin.contiguous(), out)
    return out.float().double() if kind == "f64io32" else out


def cgls(kind, vdt, K=40, snaps=(10, 20, 30, 40)):
    b_int = op64.proj_to_internal(b).to(vdt)
    nb0 = float(torch.linalg.norm(b_int.double()))
    x = torch.zeros(op64.vol_elems, dtype=vdt, device=dev)
    e = b_int - A(kind, x).to(vdt)
    r = AT(kind, e).to(vdt)
    nr2_old = float((r.double() ** 2).sum())
    dd = r.clone()
    p = A(kind, dd).to(vdt)
    alpha = nr2_old / float((p.double() ** 2).sum())
    x += alpha * dd
    e -= alpha * p
    hist = [float(torch.linalg.norm(e.double())) / nb0]
    xs = {}
    for i in range(1, K + 1):
        r = AT(kind, e).to(vdt)
        nr2 = float((r.double() ** 2).sum())
        beta = nr2 / nr2_old
        dd = dd * beta + r
        nr2_old = nr2
        p = A(kind, dd).to(vdt)
        alpha = nr2_old / float((p.double() ** 2).sum())
        x += alpha * dd
        e -= alpha * p
        hist.append(float(torch.linalg.norm(e.double())) / nb0)
        if i in snaps:
            xs[i] = op64.volume_from_internal(x.double(), torch.float64).cpu().numpy()
    return np.array(hist), xs


st = int(d["x_stride"])
for kind in ("f64", "f64io32", "f32"):
    for vdt in (torch.float64, torch.float32):
        h, xs = cgls(kind, vdt)
        hr = t["cgls_w8_hist"]
        msg = " ".join(f"K{k}: x {rel_l2(xs[k][::st], t[f'cgls_w8_x{k}_sample']):.2e} "
                       f"h {np.abs(h[:k + 1] / hr[:k + 1] - 1).max():.1e}" for k in (10, 20, 30, 40))
        print(f"op {kind:8s} vec {str(vdt)[6:]:8s} e40 {h[-1]:.6e} (ref {hr[-1]:.6e}) | {msg}", flush=True)
