"""Pageable vs pinned-pipelined H2D of a large fp64 numpy array (config-2 projections)."""
import time, numpy as np, torch
n = 360 * 512 * 384
a = np.random.default_rng(0).standard_normal(n)
dev = torch.device("cuda")
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter(); t = torch.from_numpy(a).to(dev); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"pageable .to(): {a.nbytes / 1e9 / (t1 - t0):.1f} GB/s ({(t1 - t0) * 1e3:.0f} ms)")

def piped(arr, chunk=16 << 20):
    out = torch.empty(arr.size, dtype=torch.float64, device=dev)
    flat = arr.reshape(-1)
    per = chunk // 8
    bufs = [torch.empty(per, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    evs = [None, None]
    side = torch.cuda.Stream()
    k = 0
    for off in range(0, flat.size, per):
        m = min(per, flat.size - off)
        b = bufs[k & 1]
        if evs[k & 1] is not None:
            evs[k & 1].synchronize()
        np.copyto(b.numpy()[:m], flat[off:off + m])
        with torch.cuda.stream(side):
            out[off:off + m].copy_(b[:m], non_blocking=True)
            e = torch.cuda.Event(); e.record(side)
        evs[k & 1] = e
        k += 1
    torch.cuda.current_stream().wait_stream(side)
    return out
for chunk in (4 << 20, 16 << 20, 64 << 20):
    for _ in range(2):
        t0 = time.perf_counter(); t2 = piped(a, chunk); torch.cuda.synchronize(); t1 = time.perf_counter()
    assert torch.equal(t, t2)
    print(f"pinned pipeline chunk {chunk >> 20} MB: {a.nbytes / 1e9 / (t1 - t0):.1f} GB/s ({(t1 - t0) * 1e3:.0f} ms)")
