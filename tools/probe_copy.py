"""Pageable vs pinned-staged threaded host copies (hostcopy.py) at config-2 solver sizes."""
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_13526_b200 import hostcopy as H  # noqa: E402

b = np.random.default_rng(0).standard_normal(360 * 512 * 384)  # fp64 projections, 566 MB
x = torch.randn(256 ** 3, dtype=torch.float64, device="cuda")  # fp64 volume, 134 MB


def tm(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts), r


for _ in range(2):
    t0, d0 = tm(lambda: torch.from_numpy(b).to("cuda"))
    t1, d1 = tm(lambda: H.to_device(b, "cuda"))
    assert torch.equal(d0, d1)
    print(f"H2D {b.nbytes / 1e6:.0f} MB: pageable {t0 * 1e3:.1f} ms ({b.nbytes / t0 / 1e9:.1f} GB/s), "
          f"staged {t1 * 1e3:.1f} ms ({b.nbytes / t1 / 1e9:.1f} GB/s), threads {H._THREADS}", flush=True)
    t0, h0 = tm(lambda: x.cpu().numpy())
    t1, h1 = tm(lambda: H.to_host(x))
    assert np.array_equal(h0, h1)
    nb = x.numel() * 8
    print(f"D2H {nb / 1e6:.0f} MB: pageable {t0 * 1e3:.1f} ms ({nb / t0 / 1e9:.1f} GB/s), "
          f"staged {t1 * 1e3:.1f} ms ({nb / t1 / 1e9:.1f} GB/s)", flush=True)
