"""Golden KVOL / KPRJ / PGM files written by the REFERENCE's own io module (cbctkit.io).

Run in the development container (the reference is not on the GPU box):

    python tests/golden/make_io_golden.py

It imports the reference from the same scratch copy as make_golden.py and writes
small files under tests/golden/io/, which tests/test_io_cpu.py compares our
writer against byte for byte (and reads back with our reader).
"""

from __future__ import annotations

import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import _import_reference  # noqa: E402

OUT = HERE / "io"


def payloads():
    """Deterministic test payloads shared with tests/test_io_cpu.py."""
    vol = np.arange(3 * 4 * 5, dtype=np.float64) * 0.1234567891234 - 2.5  # (nz=5, ny=4, nx=3) x fastest
    prj = np.sin(np.arange(4 * 3 * 2, dtype=np.float64)) * 1e3            # (views=2, nv=3, nu=4) u fastest
    pgm = np.linspace(-0.25, 1.25, 6 * 5 * 4)                              # values across and beyond [0, 1]
    return vol, prj, pgm


def main():
    _import_reference()
    from cbctkit import io as kio
    from cbctkit.geometry import DetectorGeometry, VolumeGeometry, make_circular_trajectory
    from cbctkit.operator import ProjectionStack
    from cbctkit.phantom import Volume

    OUT.mkdir(parents=True, exist_ok=True)
    vol, prj, pgm = payloads()
    vg = VolumeGeometry(3, 4, 5)
    tr = make_circular_trajectory(500.0, 900.0, 2, 0.0, np.pi, DetectorGeometry(4, 3))
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        kio.write_volume(OUT / f"vol_{tag}.kvol", Volume(vg, vol), dtype=dt)
        kio.write_projections(OUT / f"prj_{tag}.kprj", ProjectionStack(tr, prj), dtype=dt)
    pv = Volume(VolumeGeometry(4, 5, 6), pgm)
    for axis, index in (("x", 1), ("y", 2), ("z", 3)):
        kio.export_slice_pgm(pv, axis, index, (0.0, 1.0), OUT / f"slice_{axis}{index}.pgm")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
