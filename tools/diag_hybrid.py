"""Isolate CGLS drift: fp64 numpy CGLS with GPU/oracle operators mixed."""
import sys, pathlib
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
from _helpers import load_golden, geom_from_golden
from oracle import oracle as O
import paper_2110_13526_b200 as P

d = load_golden("desk"); vg, tr = geom_from_golden(d)
op, ref = P.CbctOperator(vg, tr), O.OracleOperator(vg, tr)
A_g = lambda x: op.project(P.Volume(vg, x)).data
AT_g = lambda y: op.backproject(P.ProjectionStack(tr, y)).data
b = ref.project(O.shepp_logan_phantom(vg))
def cgls(A, AT, K=10):
    nb0=np.linalg.norm(b); x=np.zeros(op.n); p=A(x); e=b-p; r=AT(e); nr2=r@r; dd=r.copy(); p=A(dd); a=nr2/(p@p)
    x=x+a*dd; e=e-a*p; h=[np.linalg.norm(e)/nb0]
    for _ in range(K):
        r=AT(e); n2=r@r; beta=n2/nr2; dd=beta*dd+r; nr2=n2; p=A(dd); a=nr2/(p@p); x=x+a*dd; e=e-a*p; h.append(np.linalg.norm(e)/nb0)
    return x, np.array(h)
xr, hr = cgls(ref.project, ref.backproject)
print("ref vs golden", np.abs(hr/d["cgls10_hist"]-1).max())
for name, A, AT in (("A_gpu,AT_ref", A_g, ref.backproject), ("A_ref,AT_gpu", ref.project, AT_g), ("A_gpu,AT_gpu", A_g, AT_g)):
    x, h = cgls(A, AT)
    print(name, "hist dev", np.abs(h/hr-1).max(), "x rel", np.linalg.norm(x-xr)/np.linalg.norm(xr))
    print("   per-iter dev", np.array2string(np.abs(h/hr-1), precision=1))
# operator consistency: adjointness of the gpu pair vs ref pair
rng = np.random.default_rng(0)
for _ in range(3):
    x = rng.standard_normal(op.n); y = rng.standard_normal(op.m)
    g = abs(A_g(x) @ y - x @ AT_g(y)) / (np.linalg.norm(A_g(x)) * np.linalg.norm(y))
    print("adjoint gap gpu", g)
