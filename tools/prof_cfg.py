"""Run A and A^T a few times at a BASELINE config (for ncu captures): python tools/prof_cfg.py cfg."""
import pathlib, sys
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import torch
import bench
import paper_2110_13526_b200 as P
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
vg, tr = bench.geometry(cfg)
op = P.CbctOperator(vg, tr)
x = op.phantom_internal(P.shepp_logan_3d())
p = op.new_projections(); r = op.new_volume(); scr = op.new_bp_scratch()
for _ in range(2):
    op.project_internal(x, p)
    op.backproject_internal(p, r, scratch=scr)
torch.cuda.synchronize()
print("ok", flush=True)
