"""CLI contract that needs no GPU (the reference's tests/test_cli.py usage and IO cases):
arguments, config and input files are validated before the device plan is built."""

import numpy as np
import pytest


@pytest.fixture
def config(tmp_path):
    import paper_2110_13526_b200 as P

    vg = P.VolumeGeometry(12, 10, 8, (2.0, 2.0, 2.0))
    tr = P.make_circular_trajectory(300.0, 500.0, 6, 0.0, 2 * np.pi, P.DetectorGeometry(16, 12, (2.0, 2.0)))
    path = tmp_path / "geom.cfg"
    P.save_config(path, vg, tr)
    return str(path)


def _main(argv):
    from paper_2110_13526_b200.cli import main

    return main(argv)


def test_usage_errors_exit_2(tmp_path, config):
    with pytest.raises(SystemExit) as exc:
        _main(["phantom", "--out", "x.kvol"])
    assert exc.value.code == 2
    with pytest.raises(SystemExit) as exc:
        _main(["reconstruct", config, "--prj", "b.kprj", "--method", "fbp", "--iters", "5", "--out", "r.kvol"])
    assert exc.value.code == 2
    assert _main(["phantom", str(tmp_path / "absent.cfg"), "--out", str(tmp_path / "x.kvol")]) == 2
    assert _main(["compare", config, "--prj", "b.kprj", "--iters", "0", "--outdir", str(tmp_path / "c")]) == 2
    # SIRT-family box bounds only (solvers.py validation): CGLS with --box is a config error
    assert _main(["reconstruct", config, "--prj", "b.kprj", "--method", "cgls", "--iters", "5", "--box", "0,1",
                  "--out", str(tmp_path / "r.kvol")]) == 2


def test_io_errors_exit_3(tmp_path, config):
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200 import io as kio

    bad = tmp_path / "corrupt.kvol"
    bad.write_bytes(b"XVOL" + b"\x00" * 40)
    assert _main(["project", config, "--vol", str(bad), "--out", str(tmp_path / "o.kprj")]) == 3
    wrong = tmp_path / "wrong.kvol"
    kio.write_volume(wrong, P.Volume(P.VolumeGeometry(5, 6, 6)))
    assert _main(["project", config, "--vol", str(wrong), "--out", str(tmp_path / "o.kprj")]) == 3
    assert _main(["backproject", config, "--prj", str(tmp_path / "missing.kprj"), "--out",
                  str(tmp_path / "o.kvol")]) == 3
