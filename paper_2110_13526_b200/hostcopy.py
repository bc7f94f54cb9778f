"""Host <-> device copies of large numpy arrays through pinned staging buffers.

A pageable ``torch.from_numpy(a).to("cuda")`` / ``t.cpu()`` runs at the driver's staging rate
(~11 GB/s H2D, ~2-5 GB/s D2H into fresh memory, single-threaded).  Here the host side of each
chunk is copied by several threads (numpy releases the GIL for plain-dtype copies, which also
spreads the page faults of a fresh result array) into / out of pinned buffers, while the
previous chunk's DMA runs on a side stream.  Used for the solver inputs (host fp64 projections)
and the reported volume, i.e. the host boundary of ``cgls()`` / ``lsqr()`` / ``sirt()``.
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

_CHUNK = 32 << 20  # bytes per pinned stage
_THREADS = max(1, min(8, os.cpu_count() or 1))
_MIN_BYTES = 8 << 20  # below this the plain pageable copy is as fast
_pool: ThreadPoolExecutor | None = None
_stages: list[torch.Tensor] = []
_lock = threading.Lock()  # the stages are shared: one staged copy at a time per process


def _workers() -> ThreadPoolExecutor:
    global _pool
    if _pool is None:
        _pool = ThreadPoolExecutor(max_workers=_THREADS, thread_name_prefix="cbct-copy")
    return _pool


def _stage(i: int) -> torch.Tensor:
    while len(_stages) <= i:
        _stages.append(torch.empty(_CHUNK, dtype=torch.uint8, pin_memory=True))
    return _stages[i]


def _copy(dst: np.ndarray, src: np.ndarray) -> None:
    # a narrowing float cast overflows to +-inf silently, as the device's cvt.rn does
    # (np.errstate is per thread, so it is set in the worker)
    with np.errstate(over="ignore"):
        np.copyto(dst, src, "same_kind")


def _par_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src, split across the worker threads (both 1-D, same length)."""
    n = src.size
    if n * src.itemsize < (1 << 20) or _THREADS == 1:
        _copy(dst, src)
        return
    step = -(-n // _THREADS)
    futs = [_workers().submit(_copy, dst[i:i + step], src[i:i + step]) for i in range(0, n, step)]
    for f in futs:
        f.result()


def to_device(arr: np.ndarray, device, dtype=None) -> torch.Tensor:
    """1-D numpy array -> device tensor, of ``dtype`` if given (a float narrowing such as fp64 ->
    fp32 happens in the threaded host copy, round-to-nearest-even like the device's cvt.rn,
    and halves the bytes that cross PCIe), else of the array's dtype."""
    arr = np.ascontiguousarray(arr).reshape(-1)
    dt = np.dtype(dtype) if dtype is not None else arr.dtype
    dev = torch.device(device)
    if arr.nbytes < _MIN_BYTES or dev.type != "cuda":
        with np.errstate(over="ignore"):
            return torch.from_numpy(arr.astype(dt, copy=False)).to(dev)
    with _lock:
        return _to_device_staged(arr, dt, dev)


def _to_device_staged(arr: np.ndarray, dt: np.dtype, dev: torch.device) -> torch.Tensor:
    out = torch.empty(arr.size, dtype=torch.from_numpy(np.empty(0, dt)).dtype, device=dev)
    per = _CHUNK // max(arr.itemsize, dt.itemsize)
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))  # `out` is allocated on the current stream
    done = [None, None]
    for k, off in enumerate(range(0, arr.size, per)):
        m = min(per, arr.size - off)
        if done[k & 1] is not None:
            done[k & 1].synchronize()  # the DMA that last read this stage has finished
        stage = _stage(k & 1)[: m * dt.itemsize].view(out.dtype)
        _par_copy(stage.numpy(), arr[off:off + m])
        with torch.cuda.stream(side):
            out[off:off + m].copy_(stage, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        done[k & 1] = ev
    for ev in done:  # the stages are reused by the next call: their last DMAs must have read them
        if ev is not None:
            ev.synchronize()
    torch.cuda.current_stream(dev).wait_stream(side)
    out.record_stream(side)
    return out


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> new 1-D numpy array of the same dtype."""
    t = t.reshape(-1)
    if t.device.type != "cuda" or t.numel() * t.element_size() < _MIN_BYTES:
        return t.cpu().numpy()
    with _lock:
        return _to_host_staged(t)


def _to_host_staged(t: torch.Tensor) -> np.ndarray:
    res = np.empty(t.numel(), dtype=t.new_empty(0).cpu().numpy().dtype)
    per = _CHUNK // t.element_size()
    dev = t.device
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))  # t's producer
    chunks = list(range(0, t.numel(), per))
    evs = [None, None]

    def issue(k):
        off = chunks[k]
        m = min(per, t.numel() - off)
        stage = _stage(k & 1)[: m * t.element_size()].view(t.dtype)
        with torch.cuda.stream(side):
            stage.copy_(t[off:off + m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        evs[k & 1] = (ev, stage, off, m)

    issue(0)
    for k in range(len(chunks)):
        ev, stage, off, m = evs[k & 1]
        ev.synchronize()
        if k + 1 < len(chunks):
            issue(k + 1)  # next DMA into the other stage overlaps this copy-out
        _par_copy(res[off:off + m], stage.numpy())
    t.record_stream(side)
    return res
