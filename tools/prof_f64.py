"""Run the fp64 A and A^T once at a BASELINE config (for ncu): python tools/prof_f64.py cfg."""
import pathlib, sys
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import torch
import bench
import paper_2110_13526_b200 as P
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
vg, tr = bench.geometry(cfg)
op = P.CbctOperator(vg, tr, precision="f64")
x = op.phantom_internal(P.shepp_logan_3d())
p = op.new_projections(); r = op.new_volume()
op.project_internal(x, p)
op.backproject_internal(p, r)
torch.cuda.synchronize()
print("ok", flush=True)
