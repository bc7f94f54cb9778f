"""CPU oracle for the cone-beam projector pair and its Krylov drivers.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) import this
module, and only as the checker / the timed CPU baseline -- never as part of
the product path, which fails loudly without its CUDA library.

Contents (each a restatement of the reference, cited by file:line under
``/root/reference/pkg/src/cbctkit``):

* ``view_tables``        <- operator.py:262-281 and geometry.py:138-179
* ``OracleOperator``     <- operator.py:284-374 (kernels in siddon_oracle.c)
* ``cgls``               <- solvers.py:269-358
* ``lsqr``               <- solvers.py:361-459 (with _JacobiChain solvers.py:158-193)
* ``psirt``/``normal_spectral_radius`` <- solvers.py:462-569
* ``shepp_logan_phantom`` <- phantom.py:78-141 and data/shepp_logan_3d.txt

Pinned: ``tests/test_oracle.py`` checks every function here against the
golden vectors that the reference itself produced (``tests/golden/``).
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB = None


def build(force: bool = False) -> pathlib.Path:
    """Compile liboracle.so with the committed Makefile (gcc + OpenMP)."""
    so = _HERE / "liboracle.so"
    src = _HERE / "siddon_oracle.c"
    if force or not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        so = _HERE / "liboracle.so"
        if not so.exists():
            build()
        L = ctypes.CDLL(str(so))
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        P = ctypes.c_void_p
        L.oracle_project.argtypes = [P, P, P, P, P, P, i64, i64, i64, d, d, d, d, d, d, i64, i64, i64, i32]
        L.oracle_project.restype = None
        L.oracle_backproject.argtypes = [P, P, P, P, P, P, i64, i64, i64, d, d, d, d, d, d, i64, i64, i64,
                                         i64, i32, i32]
        L.oracle_backproject.restype = i32
        L.oracle_ray_segments.argtypes = [d, d, d, d, d, d, d, d, d, d, d, d, i64, i64, i64, P, P]
        L.oracle_ray_segments.restype = i64
        L.oracle_count_nnz.argtypes = [P, P, P, P, i64, i64, i64, i64, d, d, d, d, d, d, i64, i64, i64, i32]
        L.oracle_count_nnz.restype = i64
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = i32
        _LIB = L
    return _LIB


# ----------------------------------------------------------------- geometry --
def view_angle(traj, view):  # geometry.py:138-141
    return traj.start_angle + view * traj.angular_span / traj.n_views


def source_position(traj, view):  # geometry.py:144-149
    theta = view_angle(traj, view)
    return np.array([-traj.sid * np.cos(theta), -traj.sid * np.sin(theta), 0.0], dtype=np.float64)


def detector_frame(traj, view):  # geometry.py:152-164
    theta = view_angle(traj, view)
    c, s = np.cos(theta), np.sin(theta)
    center = np.array([(traj.sdd - traj.sid) * c, (traj.sdd - traj.sid) * s, 0.0])
    return center, np.array([-s, c, 0.0]), np.array([0.0, 0.0, 1.0])


def detector_pixel_center(traj, view, u, v):  # geometry.py:167-179
    det = traj.detector
    center, ua, va = detector_frame(traj, view)
    pu, pv = det.pixel_size
    ou, ov = det.principal_point_offset
    du = (u + 0.5 - det.nu / 2.0) * pu + ou
    dv = (v + 0.5 - det.nv / 2.0) * pv + ov
    return center + du * ua + dv * va


def view_tables(traj):  # operator.py:262-281
    det = traj.detector
    V = traj.n_views
    srcs = np.empty((V, 3))
    det00 = np.empty((V, 3))
    ustep = np.empty((V, 3))
    vstep = np.empty((V, 3))
    pu, pv = det.pixel_size
    ou, ov = det.principal_point_offset
    for k in range(V):
        srcs[k] = source_position(traj, k)
        center, ua, va = detector_frame(traj, k)
        det00[k] = center + ((0.5 - det.nu / 2.0) * pu + ou) * ua + ((0.5 - det.nv / 2.0) * pv + ov) * va
        ustep[k] = pu * ua
        vstep[k] = pv * va
    return srcs, det00, ustep, vstep


def corner(vol):  # geometry.py:61-74
    ext = (vol.nx * vol.voxel_size[0], vol.ny * vol.voxel_size[1], vol.nz * vol.voxel_size[2])
    return np.array([vol.center_offset[a] - 0.5 * ext[a] for a in range(3)], dtype=np.float64)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


class OracleOperator:
    """fp64 CPU operator with the reference's semantics (operator.py:284-374).

    Works on flat numpy arrays in the reference layouts: volume x-fastest
    ``(nz, ny, nx)``, projections u-fastest ``(n_views, nv, nu)``.
    """

    def __init__(self, vol_geom, trajectory, workers=8, threads=0):
        if workers < 1:
            raise ValueError("workers must be >= 1")
        self.vol_geom = vol_geom
        self.trajectory = trajectory
        self.workers = int(workers)
        self.threads = int(threads)
        self._tables = [np.ascontiguousarray(t) for t in view_tables(trajectory)]
        self._lo = corner(vol_geom)
        self._pitch = np.asarray(vol_geom.voxel_size, dtype=np.float64)

    @property
    def n(self):
        return self.vol_geom.nx * self.vol_geom.ny * self.vol_geom.nz

    @property
    def m(self):
        d = self.trajectory.detector
        return d.nu * d.nv * self.trajectory.n_views

    def _grid(self):
        g, lo, p = self.vol_geom, self._lo, self._pitch
        return (lo[0], lo[1], lo[2], p[0], p[1], p[2], g.nx, g.ny, g.nz)

    def project(self, x, out=None):
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        assert x.size == self.n
        if out is None:
            out = np.empty(self.m)
        d = self.trajectory.detector
        s, d0, us, vs = self._tables
        lib().oracle_project(_ptr(x), _ptr(out), _ptr(s), _ptr(d0), _ptr(us), _ptr(vs),
                             self.trajectory.n_views, d.nu, d.nv, *self._grid(), self.threads)
        return out

    def _bp(self, y, mode):
        out = np.zeros(self.n)
        d = self.trajectory.detector
        s, d0, us, vs = self._tables
        yp = None if y is None else np.ascontiguousarray(y, dtype=np.float64).ravel()
        rc = lib().oracle_backproject(None if yp is None else _ptr(yp), _ptr(out), _ptr(s), _ptr(d0),
                                      _ptr(us), _ptr(vs), self.trajectory.n_views, d.nu, d.nv,
                                      *self._grid(), self.workers, mode, self.threads)
        if rc != 0:
            raise MemoryError(f"oracle_backproject failed ({rc})")
        return out

    def backproject(self, y):
        return self._bp(y, 1)

    def row_sums(self):  # operator.py:343-346
        return self.project(np.ones(self.n))

    def col_sums(self):  # operator.py:348-351
        return self._bp(np.ones(self.m), 1)

    def normal_diagonal(self):  # operator.py:353-362
        return self._bp(np.ones(self.m), 2)

    def ray_segments(self, view, u, v):  # operator.py:364-374
        src = source_position(self.trajectory, view)
        dst = detector_pixel_center(self.trajectory, view, u, v)
        idx = np.empty(self.n, dtype=np.int64)
        ln = np.empty(self.n)
        c = lib().oracle_ray_segments(src[0], src[1], src[2], dst[0], dst[1], dst[2], *self._grid(),
                                      _ptr(idx), _ptr(ln))
        return idx[:c].copy(), ln[:c].copy()

    def count_nnz(self, view0=0, view1=None):
        view1 = self.trajectory.n_views if view1 is None else view1
        d = self.trajectory.detector
        s, d0, us, vs = self._tables
        return int(lib().oracle_count_nnz(_ptr(s), _ptr(d0), _ptr(us), _ptr(vs), view0, view1, d.nu, d.nv,
                                          *self._grid(), self.threads))


# ------------------------------------------------------------------ solvers --
def cgls(op, b, K, x0=None, scale=None):
    """solvers.py:269-358 (delayed residual, d = r + beta d).  ``scale`` is the
    optional Jacobi column scaling (solvers.py:158-193).  Returns (x, history)."""
    n, m = op.n, op.m
    apply = (lambda z: op.project(z * scale)) if scale is not None else op.project
    applyT = (lambda y: op.backproject(y) * scale) if scale is not None else op.backproject
    x = np.zeros(n) if x0 is None else (x0 / scale if scale is not None else x0.copy())
    nb0 = float(np.linalg.norm(b))
    rel = lambda v: v / nb0 if nb0 > 0 else 0.0
    hist = []
    p = apply(x)
    e = b - p
    r = applyT(e)
    nr2_old = float(r @ r)
    if nr2_old == 0.0:
        return (x * scale if scale is not None else x), [rel(float(np.linalg.norm(e)))]
    d = r.copy()
    p = apply(d)
    np2 = float(p @ p)
    alpha = nr2_old / np2
    x += alpha * d
    e -= alpha * p
    hist.append(rel(float(np.linalg.norm(e))))
    for _ in range(K):
        r = applyT(e)
        nr2 = float(r @ r)
        beta = nr2 / nr2_old
        d = beta * d + r
        nr2_old = nr2
        p = apply(d)
        np2 = float(p @ p)
        alpha = nr2_old / np2
        x += alpha * d
        e -= alpha * p
        hist.append(rel(float(np.linalg.norm(e))))
    return (x * scale if scale is not None else x), hist


def jacobi_scale(op, floor_frac=1e-6):  # solvers.py:158-171
    diag = op.normal_diagonal()
    dmax = float(diag.max())
    return 1.0 / np.sqrt(np.maximum(diag, floor_frac * dmax))


def lsqr(op, b, K, scale=None):
    """solvers.py:361-459 with x0 = 0; returns (x, history of rel(phibar))."""
    apply = (lambda z: op.project(z * scale)) if scale is not None else op.project
    applyT = (lambda y: op.backproject(y) * scale) if scale is not None else op.backproject
    nb0 = float(np.linalg.norm(b))
    x = np.zeros(op.n)
    u = b - apply(x)
    beta = float(np.linalg.norm(u))
    u /= beta
    v = applyT(u)
    alpha = float(np.linalg.norm(v))
    v /= alpha
    w = v.copy()
    phibar, rhobar = beta, alpha
    hist = []
    for _ in range(K + 1):
        u = apply(v) - alpha * u
        beta = float(np.linalg.norm(u))
        if beta > 0:
            u /= beta
            v = applyT(u) - beta * v
            alpha = float(np.linalg.norm(v))
            if alpha > 0:
                v /= alpha
        rho = np.hypot(rhobar, beta)
        c, s = rhobar / rho, beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        x += (phi / rho) * w
        w = v - (theta / rho) * w
        hist.append(phibar / nb0)
        if beta == 0.0 or alpha == 0.0:
            break
    return (x * scale if scale is not None else x), hist


def normal_spectral_radius(op, power_iterations=10):  # solvers.py:462-489
    row = op.row_sums()
    inv_row = np.where(row > 0, 1.0 / np.where(row > 0, row, 1.0), 0.0)
    v = np.ones(op.n)
    for _ in range(power_iterations):
        w = op.backproject(op.project(v) * inv_row)
        v = w / float(np.linalg.norm(w))
    w = op.backproject(op.project(v) * inv_row)
    return float(v @ w)


def psirt(op, b, K, relaxation=1.0, box=None):
    """solvers.py:505-569 (method 'psirt'); returns (x, history)."""
    row = op.row_sums()
    inv_row = np.where(row > 0, 1.0 / np.where(row > 0, row, 1.0), 0.0)
    step = 2.0 * relaxation / (1.05 * normal_spectral_radius(op))
    x = np.zeros(op.n)
    nb0 = float(np.linalg.norm(b))
    resid = b - op.project(x)
    hist = [float(np.linalg.norm(resid)) / nb0]
    for _ in range(K):
        x += step * op.backproject(resid * inv_row)
        if box is not None:
            np.clip(x, box[0], box[1], out=x)
        resid = b - op.project(x)
        hist.append(float(np.linalg.norm(resid)) / nb0)
    return x, hist


# ------------------------------------------------------------------ phantom --
# data/shepp_logan_3d.txt:8-17 (cx cy cz a b c phi theta psi intensity)
SHEPP_LOGAN_3D = [
    (0.00, 0.000, 0.00, 0.690, 0.920, 0.810, 0.0, 0.0, 0.0, 1.0),
    (0.00, -0.0184, 0.00, 0.6624, 0.874, 0.780, 0.0, 0.0, 0.0, -0.75),
    (0.22, 0.000, 0.00, 0.110, 0.310, 0.220, -0.3141592653589793, 0.0, 0.1745329251994330, -0.25),
    (-0.22, 0.000, 0.00, 0.160, 0.410, 0.280, 0.3141592653589793, 0.0, 0.1745329251994330, -0.25),
    (0.00, 0.350, -0.15, 0.210, 0.250, 0.410, 0.0, 0.0, 0.0, 0.125),
    (0.00, 0.100, 0.25, 0.046, 0.046, 0.050, 0.0, 0.0, 0.0, 0.125),
    (0.00, -0.100, 0.25, 0.046, 0.046, 0.050, 0.0, 0.0, 0.0, 0.125),
    (-0.08, -0.605, 0.00, 0.046, 0.023, 0.050, 0.0, 0.0, 0.0, 0.125),
    (0.00, -0.606, 0.00, 0.023, 0.023, 0.020, 0.0, 0.0, 0.0, 0.125),
    (0.06, -0.605, 0.00, 0.023, 0.046, 0.020, 0.0, 0.0, 0.0, 0.125),
]


def _rot_z(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, s, 0.0], [-s, c, 0.0], [0.0, 0.0, 1.0]])


def _rot_x(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[1.0, 0.0, 0.0], [0.0, c, s], [0.0, -s, c]])


def shepp_logan_phantom(vol):
    """phantom.py:78-106: point-sampled sum of ellipsoids, x-fastest flat."""
    cx = (2.0 * np.arange(vol.nx) + 1.0 - vol.nx) / vol.nx
    cy = (2.0 * np.arange(vol.ny) + 1.0 - vol.ny) / vol.ny
    cz = (2.0 * np.arange(vol.nz) + 1.0 - vol.nz) / vol.nz
    X, Y, Z = cx[None, None, :], cy[None, :, None], cz[:, None, None]
    out = np.zeros((vol.nz, vol.ny, vol.nx))
    for e in SHEPP_LOGAN_3D:
        phi, theta, psi = e[6:9]
        R = _rot_z(psi) @ _rot_x(theta) @ _rot_z(phi)
        dx, dy, dz = X - e[0], Y - e[1], Z - e[2]
        px = (R[0, 0] * dx + R[0, 1] * dy + R[0, 2] * dz) / e[3]
        py = (R[1, 0] * dx + R[1, 1] * dy + R[1, 2] * dz) / e[4]
        pz = (R[2, 0] * dx + R[2, 1] * dy + R[2, 2] * dz) / e[5]
        out += np.where(px * px + py * py + pz * pz <= 1.0, e[9], 0.0)
    return out.ravel()


if os.environ.get("CBCT_ORACLE_AUTOBUILD", "1") == "1":
    try:
        build()
    except Exception:  # pragma: no cover - reported at first lib() call
        pass
