"""ctypes binding of libcbct.so (the C ABI declared in include/cbct.h).

There is no fallback: if the shared library is missing or cannot be loaded,
importing the operator raises, so a GPU run can never silently route through
a CPU path.  Build it with ``__graft_entry__.build()`` or
``make -C paper_2110_13526_b200/csrc``.
"""

from __future__ import annotations

import ctypes
import os
import pathlib

# CBCT_LIBRARY: load another build of the same ABI (A/B timing of kernel variants); default in-tree
_SO = pathlib.Path(os.environ.get("CBCT_LIBRARY") or pathlib.Path(__file__).resolve().parent / "libcbct.so")

c_i64, c_i32, c_f64, c_f32, c_p = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_float, ctypes.c_void_p

CBCT_ZPAD = 4


def zstride(nz: int) -> int:
    """Padded z length of the device volume layout (include/cbct.h)."""
    return (nz + 2 * CBCT_ZPAD + 3) // 4 * 4


class CbctError(RuntimeError):
    """A libcbct call returned a non-zero status."""


class Geometry(ctypes.Structure):
    _fields_ = [
        ("nx", c_i64), ("ny", c_i64), ("nz", c_i64),
        ("lo", c_f64 * 3), ("pitch", c_f64 * 3),
        ("nu", c_i64), ("nv", c_i64), ("n_views", c_i64),
        ("srcs", c_p), ("det00", c_p), ("ustep", c_p), ("vstep", c_p),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_voxels", c_i64), ("n_rays", c_i64), ("vol_elems", c_i64), ("zstride", c_i64),
        ("n_columns", c_i64), ("n_intervals", c_i64), ("max_intervals", c_i64),
        ("max_cell_entries", c_i64), ("table_bytes", c_i64),
        ("proj_blocks", c_i32), ("bp_blocks", c_i32),
        ("bp_scratch_floats", c_i64), ("bp_fast_path", c_i32), ("bp_closed_form", c_i32),
        ("proj_chunk", c_i32), ("bp_groups", c_i32), ("bp_view_batches", c_i32), ("bp_sided_gs", c_i32),
    ]


# name -> (restype, argtypes); every symbol of include/cbct.h
SIGNATURES = {
    "cbct_plan_create": (c_i32, [ctypes.POINTER(c_p), ctypes.POINTER(Geometry), c_p]),
    "cbct_plan_create_shard": (c_i32, [ctypes.POINTER(c_p), ctypes.POINTER(Geometry), c_i64, c_i64, c_i64, c_i64,
                                       c_p]),
    "cbct_plan_destroy": (c_i32, [c_p]),
    "cbct_plan_get_info": (c_i32, [c_p, ctypes.POINTER(PlanInfo)]),
    "cbct_project": (c_i32, [c_p, c_p, c_p, c_p, c_p]),
    "cbct_backproject": (c_i32, [c_p, c_p, c_p, c_i32, c_p, c_p, c_p, c_p]),
    "cbct_project_views": (c_i32, [c_p, c_p, c_p, c_i64, c_i64, c_p, c_p]),
    "cbct_backproject_rows": (c_i32, [c_p, c_p, c_p, c_i64, c_i64, c_i32, c_p, c_p, c_p, c_p]),
    "cbct_volume_to_internal": (c_i32, [c_p, c_p, c_i32, c_p, c_p]),
    "cbct_volume_from_internal": (c_i32, [c_p, c_p, c_p, c_i32, c_p]),
    "cbct_proj_to_internal": (c_i32, [c_p, c_p, c_i32, c_p, c_p]),
    "cbct_proj_from_internal": (c_i32, [c_p, c_p, c_p, c_i32, c_p]),
    "cbct_vec_blocks": (c_i32, [c_i64]),
    "cbct_cgls_volume_update": (c_i32, [c_i64, c_p, c_p, c_p, c_f64, c_i32, c_f64, c_p]),
    "cbct_cgls_proj_update": (c_i32, [c_i64, c_p, c_p, c_f64, c_p, c_p]),
    "cbct_axpby": (c_i32, [c_i64, c_f64, c_p, c_f64, c_p, c_p, c_p]),
    "cbct_sub": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "cbct_dot": (c_i32, [c_i64, c_p, c_p, c_p, c_p]),
    "cbct_reduce_partials": (c_i32, [c_p, c_i32, c_p, c_p, c_p]),
    "cbct_mul": (c_i32, [c_i64, c_p, c_p, c_p, c_p]),
    "cbct_clip": (c_i32, [c_p, c_p, c_f32, c_f32, c_p]),
    "cbct_fill": (c_i32, [c_i64, c_p, c_f32, c_p]),
    "cbct_fill_volume": (c_i32, [c_p, c_p, c_f32, c_p]),
    "cbct_phantom": (c_i32, [c_p, c_p, c_i32, c_p, c_p]),
    "cbct_cgls_scalars": (c_i32, [c_p, c_i32, c_p]),
    "cbct_cgls_volume_update_dev": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "cbct_cgls_proj_update_dev": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "cbct_sum_ranks": (c_i32, [c_p, c_i32, c_p, c_p]),
    "cbct_lsqr_u_update": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "cbct_lsqr_v_update": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
    "cbct_lsqr_scalars": (c_i32, [c_p, c_i32, c_p]),
    "cbct_lsqr_flush": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "cbct_psirt_volume_update": (c_i32, [c_p, c_p, c_p, c_p, c_f32, c_i32, c_f32, c_f32, c_p, c_p]),
    "cbct_psirt_proj_update": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
    "cbct_psirt_scalars": (c_i32, [c_p, c_p]),
    "cbct_cgls_volume_update_p2p": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p, c_i32, c_i64, c_p]),
    "cbct_cgls_proj_update_p2p": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p, c_i32, c_i64, c_p]),
    "cbct_phantom_ref": (c_i32, [c_i64, c_i64, c_i64, c_p, c_i32, c_p, c_p]),
    "cbct_phantom_ref_f64": (c_i32, [c_i64, c_i64, c_i64, c_p, c_i32, c_p, c_p]),
    "cbct_ref_project": (c_i32, [c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_i64, c_i64,
                                 c_f64, c_f64, c_f64, c_f64, c_f64, c_f64, c_i64, c_i64, c_i64]),
    "cbct_ref_backproject": (c_i32, [c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_i64, c_i64,
                                     c_f64, c_f64, c_f64, c_f64, c_f64, c_f64, c_i64, c_i64, c_i64,
                                     c_i64, c_i32]),
    "cbct_plan_enable_f64": (c_i32, [c_p, c_p]),
    "cbct_f64_proj_blocks": (c_i32, [c_p]),
    "cbct_project_f64": (c_i32, [c_p, c_p, c_p, c_p, c_p]),
    "cbct_backproject_f64": (c_i32, [c_p, c_p, c_p, c_i32, c_p, c_p, c_p]),
    "cbct_volume_to_internal_f64": (c_i32, [c_p, c_p, c_p, c_p]),
    "cbct_volume_from_internal_f64": (c_i32, [c_p, c_p, c_p, c_p]),
    "cbct_proj_to_internal_f64": (c_i32, [c_p, c_p, c_p, c_p]),
    "cbct_proj_from_internal_f64": (c_i32, [c_p, c_p, c_p, c_p]),
    "cbct_f64_vec_blocks": (c_i32, [c_i64]),
    "cbct_axpby_f64": (c_i32, [c_i64, c_f64, c_p, c_f64, c_p, c_p, c_p]),
    "cbct_scale_div_f64": (c_i32, [c_i64, c_p, c_f64, c_p, c_p]),
    "cbct_sub_f64": (c_i32, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "cbct_dot_f64": (c_i32, [c_i64, c_p, c_p, c_p, c_p]),
    "cbct_mul_f64": (c_i32, [c_i64, c_p, c_p, c_p, c_p]),
    "cbct_cgls_volume_update_f64": (c_i32, [c_i64, c_p, c_p, c_p, c_f64, c_i32, c_f64, c_p]),
    "cbct_fill_volume_f64": (c_i32, [c_p, c_p, c_f64, c_p]),
    "cbct_clip_f64": (c_i32, [c_p, c_p, c_f64, c_f64, c_p]),
    "cbct_last_error": (ctypes.c_char_p, []),
    "cbct_version": (c_i32, []),
    "cbct_launch_count": (c_i64, []),
}

_lib = None


def so_path() -> pathlib.Path:
    return _SO


def lib():
    """Load libcbct.so (raises if it is absent -- there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not _SO.exists():
            raise ImportError(
                f"{_SO} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        L = ctypes.CDLL(str(_SO))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().cbct_last_error().decode(errors="replace")
        raise CbctError(f"{what or 'libcbct'} failed (status {rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
