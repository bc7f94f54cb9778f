"""Pinned-staged threaded host copies (hostcopy.py): byte-exact against the plain torch copies
across chunk edges, for the dtypes the solver boundary moves (fp64 inputs/results, fp32)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture
def small_stages():
    from paper_2110_13526_b200 import hostcopy as H

    old = (H._CHUNK, H._MIN_BYTES, H._stages[:])
    H._CHUNK, H._MIN_BYTES = 4096, 0  # many chunks, staged path even for small arrays
    H._stages.clear()
    yield H
    H._CHUNK, H._MIN_BYTES = old[0], old[1]
    H._stages[:] = old[2]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("n", [1, 511, 512, 513, 4096 * 3 + 7, 300_000])
def test_round_trip_is_exact(small_stages, dtype, n):
    H = small_stages
    a = np.random.default_rng(n).standard_normal(n).astype(dtype)
    d = H.to_device(a, "cuda")
    assert d.dtype == torch.from_numpy(a).dtype and d.is_cuda
    assert torch.equal(d, torch.from_numpy(a).cuda())
    h = H.to_host(d * 2)  # a producer kernel on the current stream right before the copy
    assert h.dtype == a.dtype
    np.testing.assert_array_equal(h, a * 2)


def test_large_default_path_and_solver_boundary():
    """Default stage size (multi-chunk at this size) and the solver's host fp64 result."""
    from paper_2110_13526_b200 import hostcopy as H

    a = np.random.default_rng(5).standard_normal(5_000_000)  # 40 MB: two 32 MB stages
    d = H.to_device(a, "cuda")
    assert torch.equal(d, torch.from_numpy(a).cuda())
    np.testing.assert_array_equal(H.to_host(d), a)
    np.testing.assert_array_equal(H.to_host(d[:10]), a[:10])  # below the staging threshold


def test_back_to_back_uploads_do_not_share_in_flight_stages(small_stages):
    """Consecutive uploads reuse the pinned stages: the previous upload's DMAs must have drained."""
    H = small_stages
    arrs = [np.full(4096 * 5 + 3, float(i)) for i in range(6)]
    outs = [H.to_device(a, "cuda") for a in arrs]
    for a, d in zip(arrs, outs):
        np.testing.assert_array_equal(d.cpu().numpy(), a)


def test_host_narrowing_is_bitwise_the_device_conversion(small_stages):
    """fp64 -> fp32 in the threaded host copy (the operator's upload path) equals the device's
    cvt.rn.f32.f64 bit for bit, across the fp32 subnormal range, overflow and signed zeros."""
    H = small_stages
    rng = np.random.default_rng(11)
    a = np.concatenate([
        rng.standard_normal(20000),
        rng.standard_normal(3000) * 1e-40,              # fp32 subnormal range
        rng.standard_normal(3000) * 1e-46,              # below it: rounds to +-0 / smallest subnormal
        rng.standard_normal(1000) * 1e39,               # beyond fp32 max: +-inf
        np.array([0.0, -0.0, np.inf, -np.inf, 3.4028235677973366e38, 1.0 + 2.0 ** -24]),
    ])
    got = H.to_device(a, "cuda", dtype=np.float32)
    want = torch.from_numpy(a).cuda().float()
    assert got.dtype == torch.float32
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))
