"""Config 5 (1024^3, 1440 views of 1024x768) on one GPU: plan size, voxelizer, one A and A^T."""
import pathlib, sys, time
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import torch
import bench
import paper_2110_13526_b200 as P

vg, tr = bench.geometry(5)
t0 = time.perf_counter()
op = P.CbctOperator(vg, tr)
torch.cuda.synchronize()
print(f"plan {time.perf_counter() - t0:.1f} s, tables {op.info.table_bytes / 1e9:.1f} GB, "
      f"scratch {op.info.bp_scratch_floats * 4 / 1e9:.1f} GB, closed={op.info.bp_closed_form}", flush=True)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); x = op.phantom_internal(P.shepp_logan_3d()); e.record(); torch.cuda.synchronize()
print(f"voxelizer 1024^3: {s.elapsed_time(e):.1f} ms", flush=True)
p = op.new_projections(); r = op.new_volume(); scr = op.new_bp_scratch()
for name, fn in (("A", lambda: op.project_internal(x, p)), ("AT", lambda: op.backproject_internal(p, r, scratch=scr))):
    fn(); torch.cuda.synchronize()
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"{name}: {ms:.1f} ms ({1024 ** 3 * 1440 / ms / 1e6:.0f} GUPS)", flush=True)
print(f"peak mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB (torch) ", flush=True)
