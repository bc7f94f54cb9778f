"""End-to-end breakdown of cgls() on host fp64 data: python tools/e2e_probe.py [cfg] [K]."""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
import paper_2110_13526_b200 as P
from paper_2110_13526_b200 import solvers as S
cfg_n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
vg, tr = bench.geometry(cfg_n)
op = P.CbctOperator(vg, tr)
x = op.phantom_internal(P.shepp_logan_3d()); b_int = op.new_projections(); op.project_internal(x, b_int)
b_host = op.proj_from_internal(b_int, torch.float64).cpu().numpy()
bs = P.ProjectionStack(tr, b_host)
cfg = S.SolverConfig(method="cgls", max_iterations=K)
for mode in ("device", "host", "device", "host"):
    orig = S.CglsRun.device_capable
    if mode == "host":
        S.CglsRun.device_capable = lambda self: False
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rep = S.cgls(op, bs, cfg)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    S.CglsRun.device_capable = orig
    print(mode, f"{t*1e3:.1f} ms", rep.iterations, f"{rep.history[-1].rel_discrepancy:.6e}")
# breakdown of the device solve
torch.cuda.synchronize(); t0 = time.perf_counter()
run = S.CglsRun(op, bs, cfg); torch.cuda.synchronize(); t1 = time.perf_counter()
while run.should_continue():
    run.run_device(min(8, K - run.i))
torch.cuda.synchronize(); t2 = time.perf_counter()
rep = run.report(); t3 = time.perf_counter()
print(f"init {1e3*(t1-t0):.1f} loop {1e3*(t2-t1):.1f} report {1e3*(t3-t2):.1f}")
# pieces of init: upload of b alone, pre-loop operators alone
torch.cuda.synchronize(); t0 = time.perf_counter()
bi = op.proj_to_internal(b_host); torch.cuda.synchronize(); t1 = time.perf_counter()
xx = op.new_volume(); pp = op.new_projections(); op.project_internal(xx, pp); torch.cuda.synchronize(); t2 = time.perf_counter()
xr = op.volume_from_internal(x, torch.float64); torch.cuda.synchronize(); t3 = time.perf_counter()
from paper_2110_13526_b200 import hostcopy
h = hostcopy.to_host(xr); t4 = time.perf_counter()
print(f"upload b {1e3*(t1-t0):.1f} A(0) {1e3*(t2-t1):.1f} x->ref fp64 {1e3*(t3-t2):.1f} D2H x {1e3*(t4-t3):.1f}")
