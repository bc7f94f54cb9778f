"""Times the reference (Numba, from the build container's /root/reference) and the C oracle port on the same
config-3 view samples; the numbers are quoted in DESIGN.md section 3.  Build container only."""
import sys, time, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests/golden')
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
import numpy as np
from make_golden import _import_reference
_import_reference()
from cbctkit.geometry import DetectorGeometry, VolumeGeometry, make_circular_trajectory
from cbctkit.operator import CbctOperator, ProjectionStack
from cbctkit.phantom import Volume
import bench
for k in (16, 32):
    N, V, nu, nv = 512, 720, 616, 480
    p = 220.16 / N
    vg = VolumeGeometry(N, N, N, voxel_size=(p, p, p))
    det = DetectorGeometry(nu, nv, pixel_size=(379.456/nu, 379.456/nu))
    tr = make_circular_trajectory(749.0, 1198.0, k, 0.0, k * 2*np.pi / V, det)
    op = CbctOperator(vg, tr, workers=8)
    x = np.random.default_rng(0).random(op.n); y = np.random.default_rng(1).standard_normal(op.m)
    if k == 16:  # JIT warm-up on a tiny instance
        small = CbctOperator(VolumeGeometry(8,8,8), make_circular_trajectory(749.0,1198.0,2,0.0,1.0,DetectorGeometry(8,8)), workers=2)
        small.project(Volume(small.vol_geom, np.ones(small.n))); small.backproject(ProjectionStack(small.trajectory, np.ones(small.m)))
    t0 = time.perf_counter(); op.project(Volume(vg, x)); ta = time.perf_counter() - t0
    t0 = time.perf_counter(); op.backproject(ProjectionStack(tr, y)); tat = time.perf_counter() - t0
    oa, oat = bench.cpu_time_views(3, k, 8, 8)
    print(f"k={k}: reference A {ta:.2f} s A^T {tat:.2f} s | oracle port A {oa:.2f} s A^T {oat:.2f} s", flush=True)
