"""Shared test helpers: golden fixtures, geometries, error metrics."""

from __future__ import annotations

import pathlib

import numpy as np

from paper_2110_13526_b200.geometry import DetectorGeometry, VolumeGeometry, make_circular_trajectory

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def geom_from_golden(d):
    n = d["vol"]
    vg = VolumeGeometry(int(n[0]), int(n[1]), int(n[2]), tuple(float(v) for v in d["voxel_size"]),
                        tuple(float(v) for v in d["center_offset"]))
    det = DetectorGeometry(int(d["det"][0]), int(d["det"][1]), tuple(float(v) for v in d["pixel_size"]),
                           tuple(float(v) for v in d["principal_point_offset"]))
    t = d["traj"]
    tr = make_circular_trajectory(float(t[0]), float(t[1]), int(t[2]), float(t[3]), float(t[4]), det)
    return vg, tr


def baseline_geometry(N: int, V: int, nu: int, nv: int, views=None, zslab=None):
    """BASELINE.json configs under the SURVEY.md 8(d) geometry rule: SID 749, SDD 1198,
    full 2*pi from 0, N^3 at 220.16/N mm, detector pitch 379.456/nu mm.

    ``views=(k0, k)`` keeps a contiguous view subset (still a valid trajectory);
    ``zslab=(z0, nzs)`` keeps a z slab (a shifted VolumeGeometry)."""
    p = 220.16 / N
    vg = VolumeGeometry(N, N, N, (p, p, p))
    if zslab is not None:
        z0, nzs = zslab
        zc = -0.5 * N * p + (z0 + 0.5 * nzs) * p
        vg = VolumeGeometry(N, N, nzs, (p, p, p), (0.0, 0.0, zc))
    pu = 379.456 / nu
    det = DetectorGeometry(nu, nv, (pu, pu))
    span = 2 * np.pi
    if views is None:
        return vg, make_circular_trajectory(749.0, 1198.0, V, 0.0, span, det)
    k0, k = views
    return vg, make_circular_trajectory(749.0, 1198.0, k, k0 * span / V, k * span / V, det)


def max_rel(got, ref) -> float:
    """max|got - ref| / max|ref| (the north-star operator tolerance metric)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max()
    return float(np.abs(got - ref).max() / den) if den > 0 else float(np.abs(got).max())


def rel_l2(got, ref) -> float:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / den) if den > 0 else float(np.linalg.norm(got))
