"""KVOL / KPRJ binary files and PGM slice export (API of cbctkit.io, io.py:1-168),
with device paths for the GPU operator.

File format (io.py:39-41): a 20-byte little-endian header ``<4sBBxxIII`` -- magic
(b"KVOL" / b"KPRJ"), version 1, dtype code (0 = float32, 1 = float64), two pad
bytes, three uint32 dimensions (nx, ny, nz resp. nu, nv, n_views) -- then the
payload, fastest axis first (x resp. u).  Geometry travels in the sidecar config.

Host functions keep the reference's semantics exactly (fp64 containers, the same
error classes and checks).  The device functions stream the payload through two
pinned staging buffers on a side stream, so disk reads overlap the H2D copies, and
convert on the GPU: ``read_volume_internal`` / ``read_projections_internal`` land
directly in the solver's device layout (csrc/layout.cu), ``write_volume`` /
``write_projections`` accept device containers and ``write_internal`` writes a
device-layout vector without a host-side layout pass.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .geometry import VolumeGeometry
from .operator import ProjectionStack
from .phantom import Volume

__all__ = ["FormatError", "BadMagicError", "UnsupportedVersionError", "UnknownDtypeError", "TruncatedFileError",
           "DimensionMismatchError", "write_volume", "read_volume", "write_projections", "read_projections",
           "export_slice_pgm", "read_volume_internal", "read_projections_internal", "write_internal", "check_file"]

_HDR = struct.Struct("<4sBBxxIII")  # io.py:39 (20 bytes; the reference docstring's "16" is wrong)
_VERSION = 1
_CODES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}
_STAGE_BYTES = 64 << 20  # per pinned staging buffer


class FormatError(ValueError):
    """Malformed volume / projection file (io.py:44-66)."""


class BadMagicError(FormatError):
    pass


class UnsupportedVersionError(FormatError):
    pass


class UnknownDtypeError(FormatError):
    pass


class TruncatedFileError(FormatError):
    pass


class DimensionMismatchError(FormatError):
    """File dimensions disagree with the expected geometry."""


def _code_of(dtype) -> int:
    dt = np.dtype(dtype)
    for code, cand in _CODES.items():
        if cand == dt.newbyteorder("<"):
            return code
    raise UnknownDtypeError(f"unsupported dtype {dtype!r} (use float32 or float64)")


def _header(path, magic: bytes, fh):
    raw = fh.read(_HDR.size)
    if len(raw) < _HDR.size:
        raise TruncatedFileError(f"{path}: header truncated")
    got, version, code, d0, d1, d2 = _HDR.unpack(raw)
    if got != magic:
        raise BadMagicError(f"{path}: bad magic {got!r}, expected {magic!r}")
    if version != _VERSION:
        raise UnsupportedVersionError(f"{path}: version {version}, expected {_VERSION}")
    if code not in _CODES:
        raise UnknownDtypeError(f"{path}: unknown dtype code {code}")
    return (d0, d1, d2), code


def _check_payload(path, fh, dims, code):
    """Payload length against the header (io.py:96-101), without reading it."""
    expected = dims[0] * dims[1] * dims[2] * _CODES[code].itemsize
    have = os.fstat(fh.fileno()).st_size - _HDR.size
    if have < expected:
        raise TruncatedFileError(f"{path}: payload is {have} bytes, header promises {expected}")
    if have > expected:
        raise FormatError(f"{path}: {have - expected} trailing bytes")
    return expected


def _open_checked(path, magic: bytes):
    fh = open(path, "rb")
    try:
        dims, code = _header(path, magic, fh)
        nbytes = _check_payload(path, fh, dims, code)
    except BaseException:
        fh.close()
        raise
    return fh, dims, code, nbytes


def _host_payload(data):
    """Host fp64 view of a container's data (device tensors are copied back)."""
    try:
        import torch

        if isinstance(data, torch.Tensor):
            return data.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(data)


def _write(path, magic: bytes, dims, data, dtype) -> None:
    code = _code_of(dtype)
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(magic, _VERSION, code, *dims))
        fh.write(np.ascontiguousarray(_host_payload(data), dtype=_CODES[code]).tobytes())


def _read_host(path, magic: bytes):
    fh, dims, code, nbytes = _open_checked(path, magic)
    with fh:
        payload = fh.read(nbytes)
    return dims, np.frombuffer(payload, dtype=_CODES[code]).astype(np.float64)


def write_volume(path, vol: Volume, dtype=np.float64) -> None:
    """KVOL writer (io.py:107-109); device volumes are copied back first."""
    g = vol.geometry
    _write(path, b"KVOL", (g.nx, g.ny, g.nz), vol.data, dtype)


def read_volume(path, geometry: VolumeGeometry | None = None, device=None) -> Volume:
    """KVOL reader (io.py:112-123).  ``device``: an fp32 device Volume via the pinned pipeline."""
    if device is not None:
        fh, dims, code, nbytes = _open_checked(path, b"KVOL")
        with fh:
            geometry = _vol_geom_for(path, dims, geometry)
            raw = _stream_to_device(fh, nbytes, device)
        return Volume(geometry=geometry, data=_raw_as(raw, code).float())
    dims, data = _read_host(path, b"KVOL")
    return Volume(geometry=_vol_geom_for(path, dims, geometry), data=data)


def _vol_geom_for(path, dims, geometry):
    nx, ny, nz = dims
    if geometry is None:
        return VolumeGeometry(nx, ny, nz)
    if (geometry.nx, geometry.ny, geometry.nz) != (nx, ny, nz):
        raise DimensionMismatchError(f"{path}: file is {nx}x{ny}x{nz}, geometry expects "
                                     f"{geometry.nx}x{geometry.ny}x{geometry.nz}")
    return geometry


def _check_traj(path, dims, trajectory):
    nu, nv, nviews = dims
    det = trajectory.detector
    if (det.nu, det.nv, trajectory.n_views) != (nu, nv, nviews):
        raise DimensionMismatchError(f"{path}: file is {nu}x{nv}x{nviews}, trajectory expects "
                                     f"{det.nu}x{det.nv}x{trajectory.n_views}")


def write_projections(path, proj: ProjectionStack, dtype=np.float64) -> None:
    """KPRJ writer (io.py:126-128); device stacks are copied back first."""
    det = proj.trajectory.detector
    _write(path, b"KPRJ", (det.nu, det.nv, proj.trajectory.n_views), proj.data, dtype)


def read_projections(path, trajectory, device=None) -> ProjectionStack:
    """KPRJ reader (io.py:131-140).  ``device``: an fp32 device stack via the pinned pipeline."""
    if device is not None:
        fh, dims, code, nbytes = _open_checked(path, b"KPRJ")
        with fh:
            _check_traj(path, dims, trajectory)
            raw = _stream_to_device(fh, nbytes, device)
        return ProjectionStack(trajectory=trajectory, data=_raw_as(raw, code).float())
    dims, data = _read_host(path, b"KPRJ")
    _check_traj(path, dims, trajectory)
    return ProjectionStack(trajectory=trajectory, data=data)


def check_file(path, magic: bytes, geometry=None, trajectory=None):
    """Validate a KVOL / KPRJ header, payload length and (optionally) dimensions without
    reading the payload; returns (dims, dtype).  Raises the same errors as the readers."""
    fh, dims, code, _ = _open_checked(path, magic)
    fh.close()
    if geometry is not None:
        _vol_geom_for(path, dims, geometry)
    if trajectory is not None:
        _check_traj(path, dims, trajectory)
    return dims, _CODES[code]


# ------------------------------------------------------------------ device paths --
def _stream_to_device(fh, nbytes: int, device):
    """Payload bytes -> a uint8 device tensor, double-buffered through pinned memory:
    the next chunk's read overlaps the previous chunk's H2D copy on a side stream."""
    import torch

    dev = torch.device(device)
    out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    if nbytes == 0:
        return out
    chunk = min(_STAGE_BYTES, nbytes)
    stages = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [None, None]
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))  # `out` is allocated on the current stream
    off, k = 0, 0
    while off < nbytes:
        n = min(chunk, nbytes - off)
        buf = stages[k & 1]
        if done[k & 1] is not None:
            done[k & 1].synchronize()  # the copy that last used this staging buffer has finished
        got = fh.readinto(memoryview(buf.numpy())[:n])
        if got != n:
            raise TruncatedFileError(f"{getattr(fh, 'name', '?')}: short read")
        with torch.cuda.stream(side):
            out[off:off + n].copy_(buf[:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        done[k & 1] = ev
        off += n
        k += 1
    torch.cuda.current_stream(dev).wait_stream(side)
    out.record_stream(side)
    return out


def _raw_as(raw, code):
    import torch

    return raw.view(torch.float32 if code == 0 else torch.float64)


def read_volume_internal(path, op):
    """KVOL straight into ``op``'s device volume layout (fp32, guards zeroed):
    pinned-pipeline H2D of the raw payload, then the layout/precision conversion on the GPU."""
    fh, dims, code, nbytes = _open_checked(path, b"KVOL")
    with fh:
        _vol_geom_for(path, dims, op.vol_geom)
        raw = _stream_to_device(fh, nbytes, op.device)
    return op.volume_to_internal(_raw_as(raw, code))


def read_projections_internal(path, op):
    """KPRJ straight into ``op``'s device projection layout (fp32)."""
    fh, dims, code, nbytes = _open_checked(path, b"KPRJ")
    with fh:
        _check_traj(path, dims, op.trajectory)
        raw = _stream_to_device(fh, nbytes, op.device)
    return op.proj_to_internal(_raw_as(raw, code))


def write_internal(path, op, t, kind: str, dtype=np.float64) -> None:
    """Write a device-layout vector (``kind`` "volume" or "projections") as KVOL / KPRJ:
    layout and precision conversion on the GPU, one D2H of the payload."""
    import torch

    code = _code_of(dtype)
    tdt = torch.float32 if code == 0 else torch.float64
    if kind == "volume":
        g = op.vol_geom
        magic, dims, ref = b"KVOL", (g.nx, g.ny, g.nz), op.volume_from_internal(t, tdt)
    elif kind == "projections":
        det = op.trajectory.detector
        magic, dims, ref = b"KPRJ", (det.nu, det.nv, op.trajectory.n_views), op.proj_from_internal(t, tdt)
    else:
        raise ValueError(f"kind must be 'volume' or 'projections', got {kind!r}")
    host = torch.empty(ref.numel(), dtype=tdt, pin_memory=True)
    host.copy_(ref)
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(magic, _VERSION, code, *dims))
        fh.write(memoryview(host.numpy()).cast("B"))


# ------------------------------------------------------------------ PGM export --
def export_slice_pgm(vol: Volume, axis: str, index: int, window, path) -> None:
    """One slice as binary P5 PGM, [lo, hi] -> [0, 255] with round-half-up (io.py:143-168)."""
    lo, hi = float(window[0]), float(window[1])
    if not lo < hi:
        raise ValueError("window must satisfy lo < hi")
    g = vol.geometry
    cube = _host_payload(vol.data).reshape(g.nz, g.ny, g.nx)
    limits = {"x": g.nx, "y": g.ny, "z": g.nz}
    if axis not in limits:
        raise ValueError(f"axis must be one of x, y, z, got {axis!r}")
    if not 0 <= index < limits[axis]:
        raise IndexError(f"{axis} index {index} out of range [0, {limits[axis]})")
    img = {"x": lambda: cube[:, :, index], "y": lambda: cube[:, index, :], "z": lambda: cube[index, :, :]}[axis]()
    pixels = np.clip(np.floor((img - lo) / (hi - lo) * 255.0 + 0.5), 0, 255).astype(np.uint8)
    with open(path, "wb") as fh:
        fh.write(f"P5\n{pixels.shape[1]} {pixels.shape[0]}\n255\n".encode("ascii"))
        fh.write(pixels.tobytes())
