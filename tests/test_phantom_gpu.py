"""Device phantom voxelizer (csrc/phantom.cu) against the
reference generator: bit-identical voxels (phantom.py:78-106), pinned to the
reference's own desk phantom in tests/golden/desk.npz."""

import numpy as np
import pytest
import torch

from _helpers import geom_from_golden, load_golden

pytestmark = pytest.mark.gpu


def _mods():
    import paper_2110_13526_b200 as P

    return P


@pytest.mark.parametrize("dims", [(64, 64, 64), (33, 47, 29), (96, 80, 72), (1, 5, 130)])
def test_device_phantom_equals_host(dims):
    P = _mods()
    nx, ny, nz = dims
    vg = P.VolumeGeometry(nx, ny, nz, (0.9, 1.3, 0.7))
    host = P.generate_phantom(P.shepp_logan_3d(), vg).data
    dev = P.generate_phantom(P.shepp_logan_3d(), vg, device="cuda").data
    assert dev.dtype == torch.float32 and dev.is_cuda
    np.testing.assert_array_equal(dev.cpu().numpy().astype(np.float64), host)  # dyadic table: exact in fp32


def test_device_phantom_pinned_to_reference_golden():
    P = _mods()
    d = load_golden("desk")
    vg, _ = geom_from_golden(d)
    dev = P.generate_phantom(P.shepp_logan_3d(), vg, device="cuda").data.cpu().numpy()
    np.testing.assert_array_equal(dev, d["truth"])


def test_random_rotated_ellipsoids_round_like_the_host():
    P = _mods()
    rng = np.random.default_rng(7)
    ells = [P.Ellipsoid(tuple(rng.uniform(-0.5, 0.5, 3)), tuple(rng.uniform(0.1, 0.7, 3)),
                        tuple(rng.uniform(-np.pi, np.pi, 3)), float(rng.normal())) for _ in range(12)]
    vg = P.VolumeGeometry(40, 36, 44, (1.0, 1.0, 1.0))
    host = P.generate_phantom(ells, vg).data
    dev = P.generate_phantom(ells, vg, device="cuda").data.cpu().numpy()
    # same fp64 membership decisions and sum order, one rounding to fp32
    np.testing.assert_array_equal(dev, host.astype(np.float32))
    assert np.count_nonzero(host) > 1000


def test_phantom_internal_layout_and_guards():
    P = _mods()
    vg = P.VolumeGeometry(48, 40, 36, (1.0, 1.0, 1.0))
    tr = P.make_circular_trajectory(500.0, 900.0, 6, 0.0, 2 * np.pi, P.DetectorGeometry(64, 48, (1.0, 1.0)))
    op = P.CbctOperator(vg, tr)
    host = P.generate_phantom(P.shepp_logan_3d(), vg).data
    want = op.volume_to_internal(host)
    got = op.phantom_internal(P.shepp_logan_3d())
    assert torch.equal(got, want)
    g = got.view(vg.ny, vg.nx, op.zstride)
    assert torch.count_nonzero(g[:, :, :4]) == 0 and torch.count_nonzero(g[:, :, 4 + vg.nz:]) == 0
    assert torch.count_nonzero(op.phantom_internal([])) == 0
