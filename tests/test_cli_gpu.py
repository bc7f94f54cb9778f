"""GPU CLI and device I/O against the reference's CLI contract
(tests/test_cli.py) and the oracle: file-to-file project/backproject, reconstruct,
compare, breakdown exit code, bitwise reruns, and the pinned device read/write paths."""

import json
import pathlib

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture
def geom():
    import paper_2110_13526_b200 as P

    vg = P.VolumeGeometry(24, 20, 16, (2.0, 2.0, 2.0))
    tr = P.make_circular_trajectory(300.0, 500.0, 12, 0.1, 2 * np.pi, P.DetectorGeometry(32, 24, (2.0, 2.0)))
    return vg, tr


@pytest.fixture
def config(tmp_path, geom):
    import paper_2110_13526_b200 as P

    path = tmp_path / "geom.cfg"
    P.save_config(path, *geom)
    return str(path)


def _main(argv):
    from paper_2110_13526_b200.cli import main

    return main(argv)


@pytest.fixture
def phantom_file(tmp_path, config):
    out = str(tmp_path / "phantom.kvol")
    assert _main(["phantom", config, "--out", out]) == 0
    return out


@pytest.fixture
def projection_file(tmp_path, config, phantom_file):
    out = str(tmp_path / "data.kprj")
    assert _main(["project", config, "--vol", phantom_file, "--out", out]) == 0
    return out


def test_phantom_file_is_the_host_generators_bytes(tmp_path, config, geom, phantom_file):
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200 import io as kio

    host = tmp_path / "host.kvol"
    kio.write_volume(host, P.generate_phantom(P.shepp_logan_3d(), geom[0]))
    assert pathlib.Path(phantom_file).read_bytes() == host.read_bytes()
    table = tmp_path / "t.txt"
    table.write_text("0.1 -0.2 0.05  0.5 0.3 0.4  0.7 0.2 -0.4  0.3333333\n# comment\n")
    out = tmp_path / "t.kvol"
    assert _main(["phantom", config, "--out", str(out), "--ellipsoids", str(table)]) == 0
    kio.write_volume(host, P.generate_phantom(P.load_ellipsoids(table), geom[0]))
    assert out.read_bytes() == host.read_bytes()  # fp64 device sums: bit-identical for any table
    empty = tmp_path / "e.txt"
    empty.write_text("# nothing\n")
    assert _main(["phantom", config, "--out", str(out), "--ellipsoids", str(empty)]) == 0
    assert not np.any(kio.read_volume(out).data)
    assert json.loads((tmp_path / "phantom.kvol.manifest.json").read_text())["command"] == "phantom"


def test_project_backproject_files_match_oracle_and_are_adjoint(tmp_path, config, geom):
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200 import io as kio

    vg, tr = geom
    rng = np.random.default_rng(17)
    x = rng.standard_normal(vg.nx * vg.ny * vg.nz)
    y = rng.standard_normal(tr.detector.nu * tr.detector.nv * tr.n_views)
    kio.write_volume(tmp_path / "x.kvol", P.Volume(vg, x))
    kio.write_projections(tmp_path / "y.kprj", P.ProjectionStack(tr, y), dtype=np.float32)
    assert _main(["project", config, "--vol", str(tmp_path / "x.kvol"), "--out", str(tmp_path / "ax.kprj")]) == 0
    assert _main(["backproject", config, "--prj", str(tmp_path / "y.kprj"), "--out", str(tmp_path / "aty.kvol")]) == 0
    ax = kio.read_projections(tmp_path / "ax.kprj", tr).data
    aty = kio.read_volume(tmp_path / "aty.kvol", geometry=vg).data
    ref = O.OracleOperator(vg, tr)
    y32 = y.astype(np.float32).astype(np.float64)
    assert np.abs(ax - ref.project(x)).max() / np.abs(ax).max() <= 1e-4
    assert np.abs(aty - ref.backproject(y32)).max() / np.abs(aty).max() <= 1e-4
    # fp32 operator (the reference's fp64 bar is 1e-10)
    assert abs(ax @ y32 - x @ aty) / (np.linalg.norm(ax) * np.linalg.norm(y32)) <= 1e-6


def test_reconstruct_history_box_and_breakdown(tmp_path, config, phantom_file, projection_file):
    from paper_2110_13526_b200 import io as kio

    out, csv = tmp_path / "rec.kvol", tmp_path / "hist.csv"
    assert _main(["reconstruct", config, "--prj", projection_file, "--method", "cgls", "--iters", "5",
                  "--out", str(out), "--csv", str(csv)]) == 0
    assert len(csv.read_text().splitlines()) == 1 + 6  # header + pre-loop record + 5 iterations
    man = json.loads((tmp_path / "rec.kvol.manifest.json").read_text())
    assert man["command"] == "reconstruct" and man["parameters"]["method"] == "cgls" and man["worker_count"] == 8
    assert _main(["reconstruct", config, "--prj", projection_file, "--method", "psirt", "--iters", "5",
                  "--box", "0,1", "--out", str(out)]) == 0
    v = kio.read_volume(out).data
    assert v.min() >= 0.0 and v.max() <= 1.0
    # the exact solution as x0: zero residual at the start -> breakdown exit code, x0 returned
    assert _main(["reconstruct", config, "--prj", projection_file, "--method", "cgls", "--iters", "5",
                  "--x0", phantom_file, "--out", str(out)]) == 4
    np.testing.assert_array_equal(kio.read_volume(out).data, kio.read_volume(phantom_file).data)


def test_reconstruct_reference_precision(tmp_path, config, geom, projection_file):
    """--precision f64 runs the reference-precision path: the written iterate equals the fp64
    solver's on the same file data, bit for bit."""
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200 import io as kio

    out = tmp_path / "rec64.kvol"
    assert _main(["--precision", "f64", "reconstruct", config, "--prj", projection_file, "--method", "lsqr",
                  "--jacobi", "--iters", "6", "--out", str(out)]) == 0
    vg, tr = geom
    b = kio.read_projections(projection_file, tr)
    rep = P.lsqr(P.CbctOperator(vg, tr, precision="f64"), b,
                 P.SolverConfig(method="lsqr", max_iterations=6, jacobi_precondition=True))
    np.testing.assert_array_equal(kio.read_volume(out).data, rep.final_x.data)


def test_compare_outputs_and_bitwise_reruns(tmp_path, config, phantom_file, projection_file):
    outdir = tmp_path / "cmp"
    assert _main(["compare", config, "--prj", projection_file, "--iters", "3", "--tol", "0.5",
                  "--outdir", str(outdir)]) == 0
    for name in ("cgls.csv", "psirt.csv", "cgls_center_slice.pgm", "psirt_center_slice.pgm", "summary.txt",
                 "manifest.json"):
        assert (outdir / name).exists()
    summary = dict(line.split(" = ", 1) for line in (outdir / "summary.txt").read_text().splitlines())
    assert {"e_cgls", "e_psirt", "iters_to_tol_cgls", "iteration_ratio_psirt_over_cgls"} <= set(summary)
    a, b = tmp_path / "a.kprj", tmp_path / "b.kprj"
    assert _main(["project", config, "--vol", phantom_file, "--out", str(a)]) == 0
    assert _main(["project", config, "--vol", phantom_file, "--out", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()


def test_device_io_paths_equal_host_paths(tmp_path, geom):
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200 import io as kio

    vg, tr = geom
    op = P.CbctOperator(vg, tr)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(op.n)
    y = rng.standard_normal(op.m)
    kio.write_volume(tmp_path / "x.kvol", P.Volume(vg, x))
    kio.write_projections(tmp_path / "y32.kprj", P.ProjectionStack(tr, y), dtype=np.float32)
    old = kio._STAGE_BYTES
    kio._STAGE_BYTES = 4096  # force many double-buffered chunks
    try:
        xi = kio.read_volume_internal(tmp_path / "x.kvol", op)
        yi = kio.read_projections_internal(tmp_path / "y32.kprj", op)
        xd = kio.read_volume(tmp_path / "x.kvol", geometry=vg, device="cuda").data
    finally:
        kio._STAGE_BYTES = old
    assert torch.equal(xi, op.volume_to_internal(x))
    assert torch.equal(yi, op.proj_to_internal(y.astype(np.float32)))
    assert torch.equal(xd, torch.from_numpy(x).float().cuda())
    kio.write_internal(tmp_path / "w.kprj", op, yi, "projections", dtype=np.float32)
    assert (tmp_path / "w.kprj").read_bytes() == (tmp_path / "y32.kprj").read_bytes()
    kio.write_internal(tmp_path / "w.kvol", op, xi, "volume")
    np.testing.assert_array_equal(kio.read_volume(tmp_path / "w.kvol").data, x.astype(np.float32))
