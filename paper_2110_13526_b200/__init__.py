"""paper_2110_13526_b200 -- B200-native cone-beam projector pair + Krylov drivers.

Drop-in for the hot path of cbctkit 0.1.0 (arXiv 2110.13526's matrix-free
CGLS / LSQR / PSIRT reconstruction): the same operator/solver API, with the
projector ``A``, the backprojector ``A^T`` and the fused solver vector updates
running as hand-written sm_100a CUDA in libcbct.so.  See DESIGN.md.
"""

from .geometry import (ConfigError, DetectorGeometry, GeometryError, TrajectoryGeometry, VolumeGeometry,
                       detector_pixel_center, load_config, make_circular_trajectory, save_config, shifted,
                       source_position, view_angle)
from .phantom import Ellipsoid, Volume, generate_phantom, load_ellipsoids, shepp_logan_3d

__version__ = "0.1.0"


_LAZY = ("hostcopy", "operator", "solvers", "analysis", "estimators", "io", "cli")


def __getattr__(name):
    # The CUDA-backed modules are imported on first use so that geometry and
    # phantom helpers stay importable while the library is being built.
    import importlib

    if name.startswith("_"):
        raise AttributeError(name)
    if name in _LAZY:
        return importlib.import_module(f"{__name__}.{name}")
    for sub in _LAZY:
        mod = importlib.import_module(f"{__name__}.{sub}")
        if hasattr(mod, name):
            return getattr(mod, name)
    raise AttributeError(name)
