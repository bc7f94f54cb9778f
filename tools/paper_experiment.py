"""The reference's CGLS-vs-PSIRT experiment on B200 (the reference's acceptance
criterion 3, test_acceptance.py / test_output.txt:166): iterations to 1 % relative discrepancy and
e(40) for CGLS and PSIRT, plus LSQR with Jacobi preconditioning (BASELINE config 4), at desk scale
and at BASELINE config 3.  Writes one JSON document:

    python tools/paper_experiment.py [out.json]
"""
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2110_13526_b200 as P  # noqa: E402
from paper_2110_13526_b200.analysis import iterations_to_tolerance  # noqa: E402
from paper_2110_13526_b200.operator import InternalProjections  # noqa: E402


def run(op, b, method, K, **kw):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = P.solve(op, b, P.SolverConfig(method=method, max_iterations=K, **kw))
    torch.cuda.synchronize()
    h = [r.rel_discrepancy for r in rep.history]
    return {"iterations": rep.iterations, "seconds": time.perf_counter() - t0, "e_final": h[-1],
            "e40": h[40] if len(h) > 40 else None,
            "iters_to_1pct": iterations_to_tolerance(rep.history, 0.01)}


def case(name, vg, tr, psirt_cap, precision="f32"):
    op = P.CbctOperator(vg, tr, precision=precision)
    x = op.phantom_internal(P.shepp_logan_3d())
    b_int = op.new_projections()
    op.project_internal(x, b_int)
    b = InternalProjections(tr, b_int)
    out = {"geometry": f"{vg.nx}x{vg.ny}x{vg.nz}, {tr.n_views} views of {tr.detector.nu}x{tr.detector.nv}",
           "precision": precision}
    out["cgls_40"] = run(op, b, "cgls", 40)
    out["psirt_to_1pct"] = run(op, b, "psirt", psirt_cap, rel_discrepancy_tol=0.01)
    out["psirt_40"] = run(op, b, "psirt", 40)
    out["lsqr_jacobi_40"] = run(op, b, "lsqr", 40, jacobi_precondition=True)
    print(name, json.dumps(out), flush=True)
    return out


def main():
    doc = {"device": torch.cuda.get_device_name(0), "note": "inverse-crime b = A phantom (fp32, device); "
           "seconds include each solver's setup (PSIRT: 13 A + 12 A^T power iteration)"}
    sys.path.insert(0, str(ROOT / "tests"))
    from _helpers import geom_from_golden, load_golden

    vg, tr = geom_from_golden(load_golden("desk"))  # the reference's configs/desk_scale.cfg geometry
    doc["desk"] = case("desk", vg, tr, 1500)
    doc["desk_f64"] = case("desk_f64", vg, tr, 1500, precision="f64")
    vg, tr = bench.geometry(3)
    doc["config3"] = case("config3", vg, tr, 400)
    out = pathlib.Path(sys.argv[1]) if len(sys.argv) > 1 else None
    if out:
        out.write_text(json.dumps(doc, indent=2) + "\n")


if __name__ == "__main__":
    main()
