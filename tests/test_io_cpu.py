"""KVOL / KPRJ / PGM host I/O (paper_2110_13526_b200.io) against the reference's file
format: byte-for-byte equal to files the reference's own writer produced
(tests/golden/io, made by tests/golden/make_io_golden.py), plus the contract of the
reference's tests/test_io.py (round trips, sizes, every malformed-file error)."""

import pathlib
import struct

import numpy as np
import pytest

GOLD = pathlib.Path(__file__).resolve().parent / "golden" / "io"


def _payloads():  # = tests/golden/make_io_golden.py:payloads()
    vol = np.arange(3 * 4 * 5, dtype=np.float64) * 0.1234567891234 - 2.5
    prj = np.sin(np.arange(4 * 3 * 2, dtype=np.float64)) * 1e3
    pgm = np.linspace(-0.25, 1.25, 6 * 5 * 4)
    return vol, prj, pgm


def _mods():
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200 import io as kio

    return P, kio


def _geoms(P):
    vg = P.VolumeGeometry(3, 4, 5)
    tr = P.make_circular_trajectory(500.0, 900.0, 2, 0.0, np.pi, P.DetectorGeometry(4, 3))
    return vg, tr


@pytest.mark.parametrize("tag,dt", [("f64", np.float64), ("f32", np.float32)])
def test_writer_matches_reference_files_bytewise(tmp_path, tag, dt):
    P, kio = _mods()
    vg, tr = _geoms(P)
    vol, prj, _ = _payloads()
    kio.write_volume(tmp_path / "v.kvol", P.Volume(vg, vol), dtype=dt)
    kio.write_projections(tmp_path / "p.kprj", P.ProjectionStack(tr, prj), dtype=dt)
    assert (tmp_path / "v.kvol").read_bytes() == (GOLD / f"vol_{tag}.kvol").read_bytes()
    assert (tmp_path / "p.kprj").read_bytes() == (GOLD / f"prj_{tag}.kprj").read_bytes()
    v = kio.read_volume(GOLD / f"vol_{tag}.kvol", geometry=vg)
    p = kio.read_projections(GOLD / f"prj_{tag}.kprj", tr)
    np.testing.assert_array_equal(v.data, vol.astype(dt).astype(np.float64))
    np.testing.assert_array_equal(p.data, prj.astype(dt).astype(np.float64))
    assert v.data.dtype == np.float64 and p.data.dtype == np.float64


def test_pgm_export_matches_reference_files_bytewise(tmp_path):
    P, kio = _mods()
    _, _, pgm = _payloads()
    pv = P.Volume(P.VolumeGeometry(4, 5, 6), pgm)
    for axis, index in (("x", 1), ("y", 2), ("z", 3)):
        kio.export_slice_pgm(pv, axis, index, (0.0, 1.0), tmp_path / "s.pgm")
        assert (tmp_path / "s.pgm").read_bytes() == (GOLD / f"slice_{axis}{index}.pgm").read_bytes()


def test_round_trips_sizes_and_default_geometry(tmp_path):
    P, kio = _mods()
    vg, tr = _geoms(P)
    vol, prj, _ = _payloads()
    kio.write_volume(tmp_path / "v.kvol", P.Volume(vg, vol))
    assert (tmp_path / "v.kvol").stat().st_size == 20 + vol.size * 8
    back = kio.read_volume(tmp_path / "v.kvol")  # unit-voxel geometry synthesized
    assert (back.geometry.nx, back.geometry.ny, back.geometry.nz) == (3, 4, 5)
    assert np.array_equal(back.data, vol)
    kio.write_projections(tmp_path / "p.kprj", P.ProjectionStack(tr, prj), dtype=np.float32)
    assert (tmp_path / "p.kprj").stat().st_size == 20 + prj.size * 4


def _raw(path, magic=b"KVOL", version=1, code=1, dims=(2, 2, 2), payload=None):
    n = dims[0] * dims[1] * dims[2]
    body = payload if payload is not None else np.zeros(n, "<f8" if code == 1 else "<f4").tobytes()
    path.write_bytes(struct.pack("<4sBBxxIII", magic, version, code, *dims) + body)
    return path


def test_malformed_files_raise_the_reference_errors(tmp_path):
    P, kio = _mods()
    vg, tr = _geoms(P)
    with pytest.raises(kio.BadMagicError):
        kio.read_volume(_raw(tmp_path / "a", magic=b"KPRJ"))
    with pytest.raises(kio.UnsupportedVersionError):
        kio.read_volume(_raw(tmp_path / "b", version=2))
    with pytest.raises(kio.UnknownDtypeError):
        kio.read_volume(_raw(tmp_path / "c", code=7, payload=b""))
    with pytest.raises(kio.TruncatedFileError):
        kio.read_volume(_raw(tmp_path / "d", payload=b"\0" * 63))
    (tmp_path / "e").write_bytes(b"KVOL\x01")
    with pytest.raises(kio.TruncatedFileError):
        kio.read_volume(tmp_path / "e")
    with pytest.raises(kio.FormatError):
        kio.read_volume(_raw(tmp_path / "f", payload=b"\0" * 65))
    with pytest.raises(kio.DimensionMismatchError):
        kio.read_volume(_raw(tmp_path / "g"), geometry=vg)
    with pytest.raises(kio.DimensionMismatchError):
        kio.read_projections(_raw(tmp_path / "h", magic=b"KPRJ"), tr)
    with pytest.raises(kio.UnknownDtypeError):
        kio.write_volume(tmp_path / "i", P.Volume(vg), dtype=np.int32)
    assert issubclass(kio.FormatError, ValueError)


def test_pgm_window_rounding_and_errors(tmp_path):
    P, kio = _mods()
    v = P.Volume(P.VolumeGeometry(2, 2, 1), np.array([1.0, 0.5, -3.0, 2.0]))
    kio.export_slice_pgm(v, "z", 0, (0.0, 1.0), tmp_path / "s.pgm")
    raw = (tmp_path / "s.pgm").read_bytes()
    assert raw.startswith(b"P5\n2 2\n255\n") and list(raw[-4:]) == [255, 128, 0, 255]  # 127.5 rounds up
    with pytest.raises(ValueError):
        kio.export_slice_pgm(v, "z", 0, (1.0, 1.0), tmp_path / "t.pgm")
    with pytest.raises(IndexError):
        kio.export_slice_pgm(v, "z", 1, (0.0, 1.0), tmp_path / "t.pgm")
    with pytest.raises(ValueError):
        kio.export_slice_pgm(v, "w", 0, (0.0, 1.0), tmp_path / "t.pgm")
