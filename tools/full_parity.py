"""Operator parity at a FULL BASELINE configuration (not a subset) against the fp64 oracle.

python tools/full_parity.py [cfg] > profiles/full_parity_config{cfg}.json
(SKIP_F64=1 skips the fp64 path, SKIP_AT=1 stops after A: config 5's oracle A^T takes over 40 minutes)

A x (phantom + uniform noise), A^T y (standard normal) and diag(A^T A) from the fp32 fast path, and A x from
the fp64 path (bitwise check), against oracle/ (the C restatement of operator.py, all host threads).  The
inputs are fp32-representable so both sides see the same numbers.  Minutes of CPU: a measurement, not a test.
"""
import json
import os
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2110_13526_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
vg, tr = bench.geometry(cfg)
threads = os.cpu_count() or 8
ref = O.OracleOperator(vg, tr, workers=min(8, threads), threads=threads)
op = P.CbctOperator(vg, tr)
rng = np.random.default_rng(11)
x = (P.generate_phantom(P.shepp_logan_3d(), vg).data + 0.1 * rng.random(op.n)).astype(np.float32).astype(np.float64)
y = rng.standard_normal(op.m).astype(np.float32).astype(np.float64)


def cmp(got, want):
    d = got - want
    return {"max_rel": float(np.abs(d).max() / np.abs(want).max()),
            "rel_l2": float(np.linalg.norm(d) / np.linalg.norm(want))}


out = {"config": cfg, "n": op.n, "m": op.m, "oracle_threads": threads, "oracle_workers": ref.workers}
t = time.perf_counter()
want = ref.project(x)
out["oracle_A_s"] = time.perf_counter() - t
out["A_f32"] = cmp(op.project(P.Volume(vg, x)).data, want)
del op
if os.environ.get("SKIP_F64") is None:
    op64 = P.CbctOperator(vg, tr, precision="f64")
    got64 = op64.project(P.Volume(vg, x)).data
    out["A_f64_bitwise"] = bool(np.array_equal(got64, want))
    out["A_f64"] = cmp(got64, want)
    del op64, got64
del want
print(json.dumps(out), file=sys.stderr, flush=True)  # partial results (long oracle runs)
if os.environ.get("SKIP_AT") is not None:  # config 5: the oracle's A^T alone takes over 40 minutes
    print(json.dumps(out, indent=1))
    sys.exit(0)
op = P.CbctOperator(vg, tr)
t = time.perf_counter()
want = ref.backproject(y)
out["oracle_AT_s"] = time.perf_counter() - t
out["AT_f32"] = cmp(op.backproject(P.ProjectionStack(tr, y)).data, want)
if os.environ.get("SKIP_F64") is None:
    op64 = P.CbctOperator(vg, tr, precision="f64")
    out["AT_f64"] = cmp(op64.backproject(P.ProjectionStack(tr, y)).data, want)
    del op64
del want
t = time.perf_counter()
want = ref.normal_diagonal()
out["oracle_diag_s"] = time.perf_counter() - t
out["normal_diagonal_f32"] = cmp(op.normal_diagonal().data, want)
out["north_star_bar"] = "operator max-rel <= 1e-4 (operator.py:209-233)"
print(json.dumps(out, indent=1))
