"""KPRJ / KVOL I/O throughput, device pipeline vs host path (config 3 projections, fp32 file):
python tools/bench_io.py [cfg]"""
import os, pathlib, sys, tempfile, time
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import numpy as np
import torch
import bench
import paper_2110_13526_b200 as P
from paper_2110_13526_b200 import io as kio

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
vg, tr = bench.geometry(cfg)
op = P.CbctOperator(vg, tr)
d = tempfile.mkdtemp()
path = os.path.join(d, "b.kprj")
y = op.new_projections().normal_()
kio.write_internal(path, op, y, "projections", dtype=np.float32)
nbytes = os.path.getsize(path)


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best, out


t_dev, yi = timed(lambda: kio.read_projections_internal(path, op))
t_host, yh = timed(lambda: op.proj_to_internal(kio.read_projections(path, tr).data))
assert torch.equal(yi, yh)
t_wdev, _ = timed(lambda: kio.write_internal(path + "2", op, yi, "projections", dtype=np.float32))
t_whost, _ = timed(lambda: kio.write_projections(path + "3", P.ProjectionStack(tr, op.proj_from_internal(yi, torch.float64).cpu().numpy()), dtype=np.float32))
gb = nbytes / 1e9
print(f"cfg{cfg} KPRJ fp32 {gb:.2f} GB (page-cached): read -> device layout: pinned pipeline {gb / t_dev:.1f} GB/s "
      f"({t_dev * 1e3:.0f} ms), host path {gb / t_host:.1f} GB/s ({t_host * 1e3:.0f} ms); "
      f"write from device layout: {gb / t_wdev:.1f} GB/s vs host path {gb / t_whost:.1f} GB/s")
