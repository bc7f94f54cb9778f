"""The system matrix A as a CUDA projector pair (API of cbctkit.operator).

``CbctOperator`` is a drop-in for the reference's ``CbctOperator``
(operator.py:284-374): same constructor, ``project``/``backproject``,
``row_sums``/``col_sums``/``normal_diagonal``, ``ray_segments``, ``n``/``m``,
``vol_geom``/``trajectory``/``workers``, ``GeometryMismatchError`` raised before
any compute.  The work runs in libcbct.so (hand-written sm_100a CUDA, see
``csrc/``) on fp32 device buffers; there is no CPU fallback.

Containers passed in decide what comes back:

* host numpy data (the reference's containers) -> fp64 numpy out, aliasing
  ``out`` when given (operator.py:320-326, 332-341);
* torch CUDA data in the reference layout -> fp32 torch out;
* containers flagged ``internal=True`` hold the operator's device layout
  (volume z-fastest with zero guard slices, projections v-fastest) and are
  what the solvers iterate on: no layout conversion per call.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, hostcopy
from ._lib import CBCT_ZPAD, call, zstride
from .geometry import TrajectoryGeometry, VolumeGeometry, geometry_key, view_tables
from .phantom import Volume, coerce_data

__all__ = ["GeometryMismatchError", "ProjectionStack", "CbctOperator", "InternalVolume", "InternalProjections",
           "PRECISIONS"]

PRECISIONS = ("f32", "f64")


class GeometryMismatchError(ValueError):
    """Input volume/projection geometry does not match the operator's."""


@dataclass
class ProjectionStack:
    """Line integrals, flat u-fastest then v then view (operator.py:30-50)."""

    trajectory: TrajectoryGeometry
    data: object = field(default=None)

    def __post_init__(self):
        m = self.trajectory.n_rays
        if self.data is None:
            self.data = np.zeros(m, dtype=np.float64)
        else:
            self.data = coerce_data(self.data, m, "nu*nv*n_views")

    def as_3d(self):
        t = self.trajectory
        return self.data.reshape(t.n_views, t.detector.nv, t.detector.nu)


@dataclass
class InternalVolume:
    """A volume in the device layout [ny][nx][nz + 2*ZPAD] (fp32, zero guards)."""

    geometry: VolumeGeometry
    data: torch.Tensor
    internal: bool = True

    def as_3d(self):
        g = self.geometry
        zs = zstride(g.nz)
        return self.data.view(g.ny, g.nx, zs)[:, :, CBCT_ZPAD:CBCT_ZPAD + g.nz].permute(2, 0, 1)


@dataclass
class InternalProjections:
    """Projections in the device layout [n_views][nu][nv] (fp32)."""

    trajectory: TrajectoryGeometry
    data: torch.Tensor
    internal: bool = True

    def as_3d(self):
        t = self.trajectory
        return self.data.view(t.n_views, t.detector.nu, t.detector.nv).permute(0, 2, 1)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class CbctOperator:
    """Matched Siddon projector pair on one CUDA device.

    Immutable after construction.  ``workers`` is kept for API parity
    (operator.py:292-298, solvers.py:312): the CUDA backprojector is a
    deterministic gather, so results are bitwise reproducible for any value.
    """

    def __init__(self, vol_geom, trajectory, workers: int = 8, device=None, precision: str = "f32", _shard=None):
        if workers < 1:
            raise ValueError("workers must be >= 1")
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}, got {precision!r}")
        if not torch.cuda.is_available():
            raise RuntimeError("CbctOperator needs a CUDA device (libcbct.so has no CPU path)")
        self.vol_geom = vol_geom
        self.trajectory = trajectory
        self.workers = int(workers)
        # "f32": the fast path (fp32 buffers, csrc/project.cu + backproject.cu + vec.cu).
        # "f64": the reference-precision path (fp64 buffers and arithmetic, csrc/f64.cu), which
        # follows the reference's fp64 Krylov iterates to its own reproducibility floor.
        self.precision = precision
        self.dtype = torch.float64 if precision == "f64" else torch.float32
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._vkey = geometry_key(vol_geom)
        self._tkey = geometry_key(trajectory)
        srcs, det00, ustep, vstep = (np.ascontiguousarray(a) for a in view_tables(trajectory))
        self._tables = (srcs, det00, ustep, vstep)
        lo = np.asarray(vol_geom.corner(), dtype=np.float64) if hasattr(vol_geom, "corner") else None
        det = trajectory.detector
        g = _lib.Geometry()
        g.nx, g.ny, g.nz = vol_geom.nx, vol_geom.ny, vol_geom.nz
        for a in range(3):
            g.lo[a] = float(lo[a])
            g.pitch[a] = float(vol_geom.voxel_size[a])
        g.nu, g.nv, g.n_views = det.nu, det.nv, trajectory.n_views
        g.srcs, g.det00, g.ustep, g.vstep = (a.ctypes.data for a in self._tables)
        plan = ctypes.c_void_p()
        # _shard = (view0, view1, row0, row1): a rank-local plan of the sharded operator
        # (distributed.ShardedOperator), which only supports A on those views and A^T on those
        # cell rows (cbct_plan_create_shard)
        self.shard = None if _shard is None else tuple(int(v) for v in _shard)
        if self.shard is not None and precision != "f32":
            raise ValueError("a shard plan has no fp64 path")
        with torch.cuda.device(self.device):
            if self.shard is None:
                call("cbct_plan_create", ctypes.byref(plan), ctypes.byref(g), self._stream())
            else:
                call("cbct_plan_create_shard", ctypes.byref(plan), ctypes.byref(g), *self.shard, self._stream())
        self._plan = plan
        if self.f64:
            with torch.cuda.device(self.device):
                call("cbct_plan_enable_f64", plan, self._stream())
        info = _lib.PlanInfo()
        call("cbct_plan_get_info", plan, ctypes.byref(info))
        self.info = info
        self.vol_elems = int(info.vol_elems)
        self.zstride = int(info.zstride)
        self._nred = max(int(info.proj_blocks), int(info.bp_blocks),
                         _lib.lib().cbct_vec_blocks(max(self.vol_elems, int(info.n_rays))),
                         _lib.lib().cbct_f64_vec_blocks(max(self.vol_elems, int(info.n_rays))),
                         _lib.lib().cbct_f64_proj_blocks(plan))
        self._tls = threading.local()

    # Norm-reduction scratch (per-CTA fp64 partials, the reduced device scalar and its host
    # copy) is per thread: the reference documents its operator as safe to share across
    # threads (operator.py:284-290), and two solves on one operator must not read each
    # other's partials.
    def _scratch(self):
        s = getattr(self._tls, "s", None)
        if s is None:
            s = (torch.empty(self._nred, dtype=torch.float64, device=self.device),
                 torch.empty(1, dtype=torch.float64, device=self.device), ctypes.c_double(0.0))
            self._tls.s = s
        return s

    @property
    def _partials(self) -> torch.Tensor:
        return self._scratch()[0]

    @property
    def _red(self) -> torch.Tensor:
        return self._scratch()[1]

    @property
    def _host(self) -> ctypes.c_double:
        return self._scratch()[2]

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                _lib.lib().cbct_plan_destroy(plan)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._plan = None

    def __deepcopy__(self, memo):
        # sklearn.clone deep-copies estimators (test_estimators.py:35-43): rebuild the plan.
        return CbctOperator(self.vol_geom, self.trajectory, self.workers, self.device, self.precision, self.shard)

    def __reduce__(self):
        # pickling (joblib workers of sklearn model selection) carries the geometry; the device
        # plan is rebuilt on load
        return (CbctOperator, (self.vol_geom, self.trajectory, self.workers, str(self.device), self.precision,
                               self.shard))

    @property
    def f64(self) -> bool:
        return self.precision == "f64"

    # ------------------------------------------------------------ properties --
    @property
    def n(self) -> int:
        g = self.vol_geom
        return g.nx * g.ny * g.nz

    @property
    def m(self) -> int:
        return self.trajectory.n_rays

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    # ------------------------------------------------- device-layout helpers --
    def new_volume(self) -> torch.Tensor:
        return torch.zeros(self.vol_elems, dtype=self.dtype, device=self.device)

    def new_bp_scratch(self) -> torch.Tensor:
        """Workspace of cbct_backproject (per-column prefix sums; the fp64 path needs none)."""
        n = 1 if self.f64 else int(self.info.bp_scratch_floats)
        return torch.empty(n, dtype=torch.float32, device=self.device)

    def fill_volume(self, vol: torch.Tensor, value: float) -> None:
        """Interior = value, guard slices = 0."""
        if self.f64:
            call("cbct_fill_volume_f64", self._plan, _ptr(vol), ctypes.c_double(value), self._stream())
        else:
            call("cbct_fill_volume", self._plan, _ptr(vol), ctypes.c_float(value), self._stream())

    def new_projections(self) -> torch.Tensor:
        return torch.zeros(self.m, dtype=self.dtype, device=self.device)

    def volume_to_internal(self, data, out=None) -> torch.Tensor:
        """Reference-layout volume (numpy fp64 or torch) -> device layout."""
        out = self.new_volume() if out is None else out
        src, f64 = self._device_src(data, self.n)
        if self.f64:
            call("cbct_volume_to_internal_f64", self._plan, _ptr(src), _ptr(out), self._stream())
        else:
            call("cbct_volume_to_internal", self._plan, _ptr(src), int(f64), _ptr(out), self._stream())
        return out

    def phantom_internal(self, ellipsoids, out=None) -> torch.Tensor:
        """generate_phantom(ellipsoids, vol_geom) voxelized on the device straight into the
        device layout (csrc/phantom.cu; bit-identical to the host generator rounded to fp32)."""
        from .phantom import _device_params

        ellipsoids = list(ellipsoids)
        out = self.new_volume() if out is None else out
        params = _device_params(ellipsoids, self.device)
        if self.f64:  # fp64 sums in the reference layout, then the device layout
            g = self.vol_geom
            ref = torch.empty(self.n, dtype=torch.float64, device=self.device)
            call("cbct_phantom_ref_f64", g.nx, g.ny, g.nz, _ptr(params) if ellipsoids else None, len(ellipsoids),
                 _ptr(ref), self._stream())
            return self.volume_to_internal(ref, out)
        call("cbct_phantom", self._plan, _ptr(params) if ellipsoids else None, len(ellipsoids), _ptr(out),
             self._stream())
        return out

    def volume_from_internal(self, t: torch.Tensor, dtype=torch.float32) -> torch.Tensor:
        if self.f64:
            out = torch.empty(self.n, dtype=torch.float64, device=self.device)
            call("cbct_volume_from_internal_f64", self._plan, _ptr(t), _ptr(out), self._stream())
            return out if dtype == torch.float64 else out.to(dtype)
        out = torch.empty(self.n, dtype=dtype, device=self.device)
        call("cbct_volume_from_internal", self._plan, _ptr(t), _ptr(out), int(dtype == torch.float64),
             self._stream())
        return out

    def proj_to_internal(self, data, out=None) -> torch.Tensor:
        out = self.new_projections() if out is None else out
        src, f64 = self._device_src(data, self.m)
        if self.f64:
            call("cbct_proj_to_internal_f64", self._plan, _ptr(src), _ptr(out), self._stream())
        else:
            call("cbct_proj_to_internal", self._plan, _ptr(src), int(f64), _ptr(out), self._stream())
        return out

    def proj_from_internal(self, t: torch.Tensor, dtype=torch.float32) -> torch.Tensor:
        if self.f64:
            out = torch.empty(self.m, dtype=torch.float64, device=self.device)
            call("cbct_proj_from_internal_f64", self._plan, _ptr(t), _ptr(out), self._stream())
            return out if dtype == torch.float64 else out.to(dtype)
        out = torch.empty(self.m, dtype=dtype, device=self.device)
        call("cbct_proj_from_internal", self._plan, _ptr(t), _ptr(out), int(dtype == torch.float64),
             self._stream())
        return out

    def _device_src(self, data, size):
        if isinstance(data, torch.Tensor):
            t = data.reshape(-1)
            if self.f64:
                t = t.to(self.device, torch.float64)
            elif t.device != self.device or t.dtype not in (torch.float32, torch.float64):
                t = t.to(self.device, torch.float32)
            t = t.contiguous()
        else:
            arr = np.ascontiguousarray(data, dtype=np.float64).ravel()
            # pinned-staged, threaded (hostcopy.py); the fp32 path narrows to fp32 on the host,
            # bit-identical to the device conversion and half the PCIe bytes
            t = hostcopy.to_device(arr, self.device, dtype=np.float64 if self.f64 else np.float32)
        if t.numel() != size:
            raise ValueError(f"data length {t.numel()} != {size}")
        return t, t.dtype == torch.float64

    # ------------------------------------------------------- device kernels --
    def project_internal(self, x: torch.Tensor, out: torch.Tensor, norm2: bool = False, norm_out=None):
        """out = A x on device layouts; returns ||out||^2 (fp64, deterministic) if norm2.
        With ``norm_out`` (a 1-element fp64 device tensor) the norm is reduced into it on the
        device instead, with no host round trip (device-resident solver loops)."""
        part = self._partials if (norm2 or norm_out is not None) else None
        if self.f64:
            call("cbct_project_f64", self._plan, _ptr(x), _ptr(out), _ptr(part), self._stream())
            nparts = _lib.lib().cbct_f64_proj_blocks(self._plan)
        else:
            call("cbct_project", self._plan, _ptr(x), _ptr(out), _ptr(part), self._stream())
            nparts = int(self.info.proj_blocks)
        if norm_out is not None:
            return self.reduce_to(nparts, norm_out)
        return self.reduce(nparts) if norm2 else None

    def backproject_internal(self, y, out: torch.Tensor, mode: int = 1, norm2: bool = False, col_scale=None,
                             scratch=None, norm_out=None):
        """out = A^T y (mode 1) or diag(A^T A) (mode 2, y ignored); ||out||^2 if norm2 (or, with
        ``norm_out``, reduced on the device into that 1-element fp64 tensor)."""
        part = self._partials if (norm2 or norm_out is not None) else None
        if self.f64:
            call("cbct_backproject_f64", self._plan, _ptr(y) if mode == 1 else None, _ptr(out), int(mode),
                 _ptr(col_scale), _ptr(part), self._stream())
        else:
            scratch = self.new_bp_scratch() if scratch is None else scratch
            call("cbct_backproject", self._plan, _ptr(y) if mode == 1 else None, _ptr(out), int(mode),
                 _ptr(scratch), _ptr(col_scale), _ptr(part), self._stream())
        if norm_out is not None:
            return self.reduce_to(int(self.info.bp_blocks), norm_out)
        return self.reduce(int(self.info.bp_blocks)) if norm2 else None

    def reduce_to(self, n_partials: int, out: torch.Tensor) -> None:
        """Deterministic sum of the first n partials into the fp64 device scalar ``out`` (no sync)."""
        call("cbct_reduce_partials", _ptr(self._partials), int(n_partials), _ptr(out), None, self._stream())

    def reduce(self, n_partials: int) -> float:
        """Deterministic sum of the first n partials (synchronises the stream)."""
        partials, red, host = self._scratch()
        call("cbct_reduce_partials", _ptr(partials), int(n_partials), _ptr(red), ctypes.byref(host),
             self._stream())
        return float(host.value)

    # ------------------------------------------------------------ public API --
    def _check_vol(self, x):
        if geometry_key(x.geometry) != self._vkey:
            raise GeometryMismatchError("volume geometry does not match operator")

    def _check_proj(self, b):
        if geometry_key(b.trajectory) != self._tkey:
            raise GeometryMismatchError("projection trajectory does not match operator")

    def project(self, x, out=None, internal: bool = False):
        """A x: forward projection (operator.py:316-326)."""
        self._check_vol(x)
        if getattr(x, "internal", False):
            dst = out if out is not None else self.new_projections()
            self.project_internal(x.data, dst)
            return InternalProjections(self.trajectory, dst)
        xin = self.volume_to_internal(x.data)
        p = self.new_projections()
        self.project_internal(xin, p)
        if internal:
            return InternalProjections(self.trajectory, p)
        return ProjectionStack(self.trajectory, self._emit(self.proj_from_internal, p, x.data, out, self.m))

    def backproject(self, b, out=None, internal: bool = False):
        """A^T b: exact adjoint of project (operator.py:328-341)."""
        self._check_proj(b)
        if getattr(b, "internal", False):
            dst = out if out is not None else self.new_volume()
            self.backproject_internal(b.data, dst)
            return InternalVolume(self.vol_geom, dst)
        yin = self.proj_to_internal(b.data)
        v = self.new_volume()
        self.backproject_internal(yin, v)
        if internal:
            return InternalVolume(self.vol_geom, v)
        return Volume(self.vol_geom, self._emit(self.volume_from_internal, v, b.data, out, self.n))

    def _emit(self, convert, t_int, like, out, size):
        """Convert a device-layout result back to the caller's kind of container."""
        if isinstance(like, torch.Tensor):
            res = convert(t_int, self.dtype)
            if out is not None:
                out.reshape(-1).copy_(res.to(out.dtype))
                return out
            return res
        res = hostcopy.to_host(convert(t_int, torch.float64))
        if out is not None:
            out[:] = res
            return out
        return res

    def row_sums(self, internal: bool = False):
        """A 1: per-ray chord length through the volume box, mm (operator.py:343-346)."""
        ones = self.new_volume()
        self.fill_volume(ones, 1.0)
        p = self.new_projections()
        self.project_internal(ones, p)
        if internal:
            return InternalProjections(self.trajectory, p)
        return ProjectionStack(self.trajectory, hostcopy.to_host(self.proj_from_internal(p, torch.float64)))

    def col_sums(self, internal: bool = False):
        """A^T 1: per-voxel total traversal length, mm (operator.py:348-351)."""
        ones = torch.ones(self.m, dtype=self.dtype, device=self.device)
        v = self.new_volume()
        self.backproject_internal(ones, v)
        if internal:
            return InternalVolume(self.vol_geom, v)
        return Volume(self.vol_geom, hostcopy.to_host(self.volume_from_internal(v, torch.float64)))

    def normal_diagonal(self, internal: bool = False):
        """diag(A^T A): per-voxel sum of squared intersection lengths (operator.py:353-362)."""
        v = self.new_volume()
        self.backproject_internal(None, v, mode=2)
        if internal:
            return InternalVolume(self.vol_geom, v)
        return Volume(self.vol_geom, hostcopy.to_host(self.volume_from_internal(v, torch.float64)))

    def ray_segments(self, view: int, u: int, v: int):
        """(voxel indices, lengths mm) of the ray through pixel (u, v): A^T of a unit
        impulse, computed by the same CUDA gather (operator.py:364-374)."""
        det = self.trajectory.detector
        if not (0 <= view < self.trajectory.n_views and 0 <= u < det.nu and 0 <= v < det.nv):
            raise IndexError("pixel out of range")
        y = self.new_projections()
        y[(view * det.nu + u) * det.nv + v] = 1.0
        out = self.new_volume()
        self.backproject_internal(y, out)
        ref = hostcopy.to_host(self.volume_from_internal(out, torch.float64))
        idx = np.flatnonzero(ref).astype(np.int64)
        return idx, ref[idx]
