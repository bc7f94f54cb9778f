"""Device-resident CGLS / LSQR / SIRT / PSIRT (API of cbctkit.solvers).

Same configuration, validation, history convention, operator budgets,
breakdown guards and reports as the reference (solvers.py:1-609); the work
vectors are fp32 tensors on the GPU in the operator's device layouts and every
vector update is one of libcbct's fused kernels:

  CGLS iteration = A^T (with ||r||^2 in its epilogue)
                 + volume update  x += a_prev*d ; d = r + beta*d   (one pass)
                 + A (with ||p||^2 in its epilogue)
                 + projection update  e -= alpha*p ; ||e||^2      (one pass)

The x update is deferred by one iteration so it fuses with the d update; it is
flushed before anything reads x.  Scalars (alpha, beta, Givens rotations) are
fp64 on the host exactly as in the reference; the norms they need come from
deterministic fp64 device reductions.

Solvers touch the operator only through ``project``/``backproject`` (and
``normal_diagonal``/``row_sums``/``col_sums``), so instrumented wrappers that
forward other attributes work as with the reference (test_solvers.py:20-37).
When the operator is a bare ``CbctOperator`` the norm reductions fuse into the
A / A^T epilogues.
"""

from __future__ import annotations

import csv
import ctypes
import functools
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import hostcopy
from ._lib import call
from .operator import CbctOperator, InternalProjections, InternalVolume
from .phantom import Volume

__all__ = ["SolverConfigError", "DegenerateOperatorError", "SolverConfig", "ConvergenceRecord", "SolverReport",
           "cgls", "lsqr", "sirt", "psirt", "solve", "write_history_csv", "normal_spectral_radius",
           "psirt_step_scale", "KRYLOV_METHODS", "CLASSICAL_METHODS"]

KRYLOV_METHODS = ("cgls", "lsqr")
CLASSICAL_METHODS = ("sirt", "psirt")


class SolverConfigError(ValueError):
    """Invalid solver configuration."""


class DegenerateOperatorError(RuntimeError):
    """The operator never touches the volume (all-zero row or column sums)."""


@dataclass
class SolverConfig:  # reference solvers.py:56-97
    method: str = "cgls"
    max_iterations: int = 40
    rel_discrepancy_tol: float = 0.0
    initial_x0: object = None
    tikhonov_lambda: float = 0.0
    jacobi_precondition: bool = False
    jacobi_floor: float = 1e-6
    box_bounds: tuple = None
    relaxation: float = 1.0
    true_discrepancy_every: int = 0

    def validate(self) -> None:
        if self.method not in KRYLOV_METHODS + CLASSICAL_METHODS:
            raise SolverConfigError(f"unknown method {self.method!r}")
        if self.max_iterations < 1:
            raise SolverConfigError("max_iterations must be >= 1")
        if not 0.0 <= self.rel_discrepancy_tol <= 1.0:
            raise SolverConfigError("rel_discrepancy_tol must lie in [0, 1]")
        if self.tikhonov_lambda < 0:
            raise SolverConfigError("tikhonov_lambda must be >= 0")
        if self.jacobi_floor <= 0:
            raise SolverConfigError("jacobi_floor must be > 0")
        if self.relaxation <= 0:
            raise SolverConfigError("relaxation must be > 0")
        if self.true_discrepancy_every < 0:
            raise SolverConfigError("true_discrepancy_every must be >= 0")
        if self.box_bounds is not None:
            lo, hi = self.box_bounds
            if lo > hi:
                raise SolverConfigError("box_bounds must satisfy lo <= hi")
            if self.method in KRYLOV_METHODS:
                raise SolverConfigError("box constraints are incompatible with Krylov methods "
                                        "(the clamped iterate leaves the Krylov subspace)")
        if self.method in CLASSICAL_METHODS:
            if self.tikhonov_lambda != 0.0:
                raise SolverConfigError("tikhonov_lambda applies to cgls/lsqr only")
            if self.jacobi_precondition:
                raise SolverConfigError("jacobi_precondition applies to cgls/lsqr only")


@dataclass
class ConvergenceRecord:
    iteration: int
    wall_seconds: float
    rel_discrepancy: float
    true_rel_discrepancy: float = None


@dataclass
class SolverReport:
    final_x: Volume
    iterations: int
    final_discrepancy_norm: float
    history: list
    worker_count: int
    breakdown: bool = False


def _alloc(size: int, physical: int = None, device=None, dtype=torch.float32) -> torch.Tensor:
    """Allocation funnel for the solver work vectors (auditable, solvers.py:118-120).
    ``size`` is the logical length (n or m); ``physical`` the padded device length; ``dtype``
    the operator's precision (fp32 fast path, fp64 reference-precision path)."""
    return torch.zeros(physical if physical is not None else size, dtype=dtype, device=device)


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class _Dev:
    """Fused vector kernels of libcbct bound to an operator's stream and partials.  An fp64
    operator (``precision="f64"``) gets the fp64 kernels of csrc/f64.cu, which round like the
    reference's NumPy updates."""

    def __init__(self, op):
        self.op = op
        self.base = op if isinstance(op, CbctOperator) else None
        self.plan = op._plan
        self.partials = op._partials
        self.vol_elems = op.vol_elems
        self.device = op.device
        self.dtype = getattr(op, "dtype", torch.float32)
        self.f64 = self.dtype == torch.float64
        self._sfx = "_f64" if self.f64 else ""

    def s(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def empty(self, n):
        return torch.empty(n, dtype=self.dtype, device=self.device)

    def reduce(self, nparts: int) -> float:
        return self.op.reduce(nparts)

    def nblocks(self, n):
        from ._lib import lib

        return lib().cbct_f64_vec_blocks(n) if self.f64 else lib().cbct_vec_blocks(n)

    def axpby(self, a, x, b, y, norm2=False):
        call("cbct_axpby" + self._sfx, y.numel(), float(a), _p(x), float(b), _p(y),
             _p(self.partials) if norm2 else None, self.s())
        return self.reduce(self.nblocks(y.numel())) if norm2 else None

    def div(self, y, d, norm2=False):
        """y /= d (u /= beta and friends, solvers.py:407-441); the fp32 path multiplies by 1/d."""
        if not self.f64:
            return self.axpby(0.0, None, 1.0 / d, y, norm2=norm2)
        call("cbct_scale_div_f64", y.numel(), _p(y), float(d), _p(self.partials) if norm2 else None, self.s())
        return self.reduce(self.nblocks(y.numel())) if norm2 else None

    def sumsq(self, y):
        return self.axpby(0.0, None, 1.0, y, norm2=True)

    def sub(self, a, b, out, norm2=False):
        call("cbct_sub" + self._sfx, out.numel(), _p(a), _p(b), _p(out), _p(self.partials) if norm2 else None,
             self.s())
        return self.reduce(self.nblocks(out.numel())) if norm2 else None

    def dot(self, x, y):
        call("cbct_dot" + self._sfx, x.numel(), _p(x), _p(y), _p(self.partials), self.s())
        return self.reduce(self.nblocks(x.numel()))

    def mul(self, a, b, out):
        call("cbct_mul" + self._sfx, out.numel(), _p(a), _p(b), _p(out), self.s())

    def update2(self, x, d, r, a_prev, do_x, beta):
        """x += a_prev*d (if do_x); d = r + beta*d  -- one fused pass."""
        call("cbct_cgls_volume_update" + self._sfx, d.numel(), _p(x), _p(d), _p(r), float(a_prev), int(do_x),
             float(beta), self.s())

    def clip(self, vol, lo, hi):
        if self.f64:
            call("cbct_clip_f64", self.plan, _p(vol), ctypes.c_double(lo), ctypes.c_double(hi), self.s())
        else:
            call("cbct_clip", self.plan, _p(vol), ctypes.c_float(lo), ctypes.c_float(hi), self.s())

    def fill_volume(self, vol, value):
        if self.f64:
            call("cbct_fill_volume_f64", self.plan, _p(vol), ctypes.c_double(value), self.s())
        else:
            call("cbct_fill_volume", self.plan, _p(vol), ctypes.c_float(value), self.s())


def _as_internal_volume(op, vol) -> torch.Tensor:
    if getattr(vol, "internal", False):
        return vol.data
    return op.volume_to_internal(vol.data)


def _as_internal_proj(op, stack) -> torch.Tensor:
    if getattr(stack, "internal", False):
        return stack.data
    return op.proj_to_internal(stack.data)


def _call_sums(op, name):
    fn = getattr(op, name)
    try:
        return fn(internal=True)
    except TypeError:  # wrapper with the reference signature
        return fn()


class _Chain:
    """Flat device-layout view of the operator (solvers.py:123-155)."""

    def __init__(self, op, dev: _Dev):
        self.op, self.dev = op, dev
        self.n, self.m, self.m_orig = op.n, op.m, op.m
        self.n_phys, self.m_phys = dev.vol_elems, op.m
        self._fused = dev.base is not None

    def apply(self, x, out, norm2=False):
        if self._fused:
            return self.op.project_internal(x, out, norm2=norm2)
        res = self.op.project(InternalVolume(self.op.vol_geom, x), out=out)
        if res.data is not out:
            out.copy_(_as_internal_proj(self.op, res))
        return self.dev.sumsq(out) if norm2 else None

    def applyT(self, y, out, norm2=False):
        if self._fused:
            return self.op.backproject_internal(y, out, norm2=norm2, scratch=self._scratch())
        res = self.op.backproject(InternalProjections(self.op.trajectory, y), out=out)
        if res.data is not out:
            out.copy_(_as_internal_volume(self.op, res))
        return self.dev.sumsq(out) if norm2 else None

    def _scratch(self):
        if not hasattr(self, "_scr"):
            self._scr = self.op.new_bp_scratch()
        return self._scr

    def z_of(self, x0):
        return x0

    def x_of(self, z):
        return z

    def rhs(self, b):
        return b

    def head(self, e):
        return e[: self.m_orig]


class _JacobiChain(_Chain):
    """min ||b - A D^-1/2 z||, x = D^-1/2 z, diag floored (solvers.py:158-193)."""

    def __init__(self, inner: _Chain, diag: torch.Tensor, floor_frac: float):
        self.inner, self.op, self.dev = inner, inner.op, inner.dev
        self.n, self.m, self.m_orig = inner.n, inner.m, inner.m_orig
        self.n_phys, self.m_phys = inner.n_phys, inner.m_phys
        dmax = float(diag.max())
        if dmax <= 0:
            raise DegenerateOperatorError("normal-equation diagonal is identically zero")
        floored = torch.clamp(diag.double(), min=floor_frac * dmax)
        scale = (1.0 / torch.sqrt(floored)).to(self.dev.dtype)
        # zero the scale on the guard slices so scaled volumes keep zero guards
        mask = torch.zeros_like(scale)
        self.dev.fill_volume(mask, 1.0)
        self.scale = scale * mask
        self._tmp = torch.empty_like(self.scale)

    def apply(self, z, out, norm2=False):
        self.dev.mul(z, self.scale, self._tmp)
        return self.inner.apply(self._tmp, out, norm2=norm2)

    def applyT(self, y, out, norm2=False):
        inner = self.inner
        if inner._fused:
            return inner.op.backproject_internal(y, out, norm2=norm2, col_scale=self.scale, scratch=inner._scratch())
        inner.applyT(y, out)
        self.dev.mul(out, self.scale, out)
        return self.dev.sumsq(out) if norm2 else None

    def z_of(self, x0):
        safe = torch.where(self.scale > 0, self.scale, torch.ones_like(self.scale))
        return torch.where(self.scale > 0, x0 / safe, torch.zeros_like(x0))

    def x_of(self, z):
        out = torch.empty_like(z)
        self.dev.mul(z, self.scale, out)
        return out

    def rhs(self, b):
        return self.inner.rhs(b)

    def head(self, e):
        return self.inner.head(e)


class _TikhonovChain(_Chain):
    """Stacked [A; lambda I] with data [b; 0] (solvers.py:196-230)."""

    def __init__(self, inner: _Chain, lam: float):
        self.inner, self.op, self.dev = inner, inner.op, inner.dev
        self.lam = float(lam)
        self.n, self.m_orig = inner.n, inner.m_orig
        self.m = inner.m + inner.n
        self.n_phys = inner.n_phys
        self.m_phys = inner.m_phys + inner.n_phys

    def apply(self, x, out, norm2=False):
        mi = self.inner.m_phys
        a = self.inner.apply(x, out[:mi], norm2=norm2)
        tail = out[mi:]
        tail.zero_()
        b = self.dev.axpby(self.lam, x, 0.0, tail, norm2=norm2)
        return a + b if norm2 else None

    def applyT(self, y, out, norm2=False):
        mi = self.inner.m_phys
        self.inner.applyT(y[:mi], out)
        return self.dev.axpby(self.lam, y[mi:], 1.0, out, norm2=norm2)

    def z_of(self, x0):
        return self.inner.z_of(x0)

    def x_of(self, z):
        return self.inner.x_of(z)

    def rhs(self, b):
        out = torch.zeros(self.m_phys, dtype=self.dev.dtype, device=self.dev.device)
        out[: self.inner.m_phys] = self.inner.rhs(b)
        return out

    def head(self, e):
        return self.inner.head(e)


def _build_chain(op, cfg: SolverConfig, dev: _Dev) -> _Chain:  # solvers.py:233-240
    chain = _Chain(op, dev)
    if cfg.jacobi_precondition:
        diag = _as_internal_volume(op, op.normal_diagonal())
        chain = _JacobiChain(chain, diag, cfg.jacobi_floor)
    if cfg.tikhonov_lambda > 0.0:
        chain = _TikhonovChain(chain, cfg.tikhonov_lambda)
    return chain


def _geom_eq(a, b):
    from .geometry import geometry_key

    return geometry_key(a) == geometry_key(b)


def _check_inputs(op, b, cfg: SolverConfig, method: str) -> None:  # solvers.py:243-250
    cfg.validate()
    if cfg.method != method:
        raise SolverConfigError(f"cfg.method is {cfg.method!r}, expected {method!r}")
    if not _geom_eq(b.trajectory, op.trajectory):
        raise SolverConfigError("projection data does not match the operator trajectory")
    if cfg.initial_x0 is not None and not _geom_eq(cfg.initial_x0.geometry, op.vol_geom):
        raise SolverConfigError("initial_x0 geometry does not match the operator")


def _x0_internal(op, cfg: SolverConfig, dev: _Dev) -> torch.Tensor:
    if cfg.initial_x0 is None:
        return torch.zeros(dev.vol_elems, dtype=dev.dtype, device=dev.device)
    return _as_internal_volume(op, cfg.initial_x0).clone()


def _norm(dev: _Dev, v) -> float:
    return float(np.sqrt(dev.sumsq(v)))


def _final_volume(op, x_int, like):
    """Report the solution in the caller's container kind (numpy fp64 for host b)."""
    if isinstance(like, torch.Tensor) and getattr(like, "is_cuda", False):
        return Volume(op.vol_geom, op.volume_from_internal(x_int, getattr(op, "dtype", torch.float32)))
    return Volume(op.vol_geom, hostcopy.to_host(op.volume_from_internal(x_int, torch.float64)))


def _true_rel(op, chain, x_int, b_int, nb0, dev):  # solvers.py:259-261
    p = torch.empty_like(b_int)
    res = op.project(InternalVolume(op.vol_geom, chain.x_of(x_int)), out=p)
    p = _as_internal_proj(op, res)
    r = torch.empty_like(b_int)
    return float(np.sqrt(dev.sub(b_int, p, r, norm2=True))) / nb0 if nb0 > 0 else 0.0


def _want_true(cfg, iteration):
    k = cfg.true_discrepancy_every
    return k > 0 and iteration % k == 0


def _nvtx(name):
    """NVTX range around a public solver call (the kernels inside carry the C library's ranges:
    cbct_project / cbct_backproject / cbct_normal_diagonal)."""
    def deco(fn):
        @functools.wraps(fn)
        def wrapped(*args, **kwargs):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.nvtx.range_pop()
        return wrapped
    return deco


class CglsRun:
    """Device-resident CGLS state (solvers.py:269-358), split into the pre-loop
    (``__init__``: 2 A + 1 A^T, first update folded in) and one loop iteration
    (``step``: 1 A^T + 1 A + two fused vector passes).  ``cgls`` drives it; the
    benchmark times ``step`` directly."""

    def __init__(self, op, b, cfg: SolverConfig):
        self.op, self.b, self.cfg = op, b, cfg
        self.dev = dev = _Dev(op)
        self.chain = chain = _build_chain(op, cfg, dev)
        self.t0 = time.perf_counter()
        self.x = _alloc(chain.n, chain.n_phys, dev.device, dev.dtype)
        self.x.copy_(chain.z_of(_x0_internal(op, cfg, dev)))
        self.d = _alloc(chain.n, chain.n_phys, dev.device, dev.dtype)
        self.r = _alloc(chain.n, chain.n_phys, dev.device, dev.dtype)
        self.e = _alloc(chain.m, chain.m_phys, dev.device, dev.dtype)
        self.p = _alloc(chain.m, chain.m_phys, dev.device, dev.dtype)
        self.history = []
        self.pending = 0.0  # deferred x += alpha*d
        self.i = 0
        self.done = False
        self.breakdown = False
        x, d, r, e, p = self.x, self.d, self.r, self.e, self.p
        chain.apply(x, p)  # A x0 needs no b: queued first, it overlaps b's host upload
        self.b_int = _as_internal_proj(op, b)
        self.b_eff = chain.rhs(self.b_int)
        self.nb0 = _norm(dev, self.b_int)
        dev.sub(self.b_eff, p, e)
        self.nr2_old = chain.applyT(e, r, norm2=True)
        if self.nr2_old == 0.0:
            self._stop_at_start()
            return
        d.copy_(r)
        np2 = chain.apply(d, p, norm2=True)
        if np2 == 0.0:
            self._stop_at_start()
            return
        alpha = self.nr2_old / np2
        self.pending = alpha
        self._set_norms(*_proj_update(dev, chain, e, p, alpha))
        self._record(0)

    def _set_norms(self, head2, full2):
        self.nb = float(np.sqrt(head2))       # history / final_discrepancy_norm (report_norm)
        self.nb_full = float(np.sqrt(full2))  # the stop test (norm of the stacked e_b)

    def _stop_at_start(self):
        self.nb = self.nb_full = _norm(self.dev, self.chain.head(self.e))
        self._record(0)
        self.done = self.breakdown = True

    def rel(self, v):
        return v / self.nb0 if self.nb0 > 0 else 0.0

    def flush(self):
        if self.pending != 0.0:
            self.dev.axpby(self.pending, self.d, 1.0, self.x)
            self.pending = 0.0

    def _record(self, i):
        true_e = None
        if _want_true(self.cfg, i):
            self.flush()
            true_e = _true_rel(self.op, self.chain, self.x, self.b_int, self.nb0, self.dev)
        self.history.append(ConvergenceRecord(i, time.perf_counter() - self.t0, self.rel(self.nb), true_e))

    def should_continue(self) -> bool:
        return (not self.done) and self.rel(self.nb_full) > self.cfg.rel_discrepancy_tol and \
            self.i < self.cfg.max_iterations

    @_nvtx("cbct_cgls_iteration")
    def step(self, record: bool = True) -> bool:
        """One loop iteration; returns False on breakdown (state left as the reference leaves it)."""
        dev, chain = self.dev, self.chain
        nr2 = chain.applyT(self.e, self.r, norm2=True)
        if nr2 == 0.0:
            self.done = self.breakdown = True
            return False
        beta = nr2 / self.nr2_old
        dev.update2(self.x, self.d, self.r, self.pending, self.pending != 0.0, beta)  # x += a d ; d = r + b d
        self.pending = 0.0
        self.nr2_old = nr2
        np2 = chain.apply(self.d, self.p, norm2=True)
        if np2 == 0.0:
            self.done = self.breakdown = True
            return False
        alpha = self.nr2_old / np2
        self.pending = alpha
        self._set_norms(*_proj_update(dev, chain, self.e, self.p, alpha))
        self.i += 1
        if record:
            self._record(self.i)
        return True

    # ------------------------------------------------- device-resident iterations --
    def device_capable(self) -> bool:
        """The plain fused chain (no Jacobi/Tikhonov stacking) without true-discrepancy
        monitoring can run with every scalar on the device (``run_device``)."""
        c = self.chain
        return type(c) is _Chain and c._fused and self.cfg.true_discrepancy_every <= 0 and not self.dev.f64

    def _device_scalars(self) -> torch.Tensor:
        """The fp64 scalar array of include/cbct.h cbct_cgls_scalars, loaded from the host state."""
        if getattr(self, "_S", None) is None:
            self._S = torch.zeros(16 + self.cfg.max_iterations + 2, dtype=torch.float64, device=self.dev.device)
        host = torch.tensor([self.nr2_old, 0.0, 0.0, self.pending, 0.0, 0.0, 0.0, float(self.i), self.nb0,
                             float(self.cfg.rel_discrepancy_tol), 0.0], dtype=torch.float64)
        self._S[:11].copy_(host)
        return self._S

    def _device_iteration(self, S):
        op, dev, st = self.op, self.dev, self.dev.s
        op.backproject_internal(self.e, self.r, scratch=self.chain._scratch(), norm_out=S[1:2])
        call("cbct_cgls_scalars", _p(S), 1, st())                                   # beta
        call("cbct_cgls_volume_update_dev", self.d.numel(), _p(self.x), _p(self.d), _p(self.r), _p(S), st())
        op.project_internal(self.d, self.p, norm_out=S[2:3])
        call("cbct_cgls_scalars", _p(S), 2, st())                                   # alpha
        call("cbct_cgls_proj_update_dev", self.e.numel(), _p(self.e), _p(self.p), _p(S), _p(dev.partials), st())
        op.reduce_to(dev.nblocks(self.e.numel()), S[5:6])
        call("cbct_cgls_scalars", _p(S), 3, st())                                   # history, tolerance

    @_nvtx("cbct_cgls_device_iterations")
    def run_device(self, k: int, graph: bool = False, collect: bool = True) -> None:
        """Up to k loop iterations with alpha, beta, the norms and the stop tests on the device
        (csrc/vec.cu cbct_cgls_scalars): no host round trip inside, one synchronisation at the end,
        and iterates bit-identical to k calls of ``step``.  Iterations after a breakdown or after
        reaching the tolerance are no-ops for the iterate.  ``graph`` replays one captured CUDA
        graph of the iteration instead of issuing its launches from Python (``graph_launches`` is
        then the number of kernels per replay).  ``collect=False`` leaves the batch in flight;
        ``collect()`` synchronises and reads the history back.  History records of a batch share
        its end time."""
        if self.done or k <= 0:
            return
        S = self._device_scalars()
        self._i0 = self.i
        if graph:
            if getattr(self, "_graph", None) is None:
                from ._lib import lib

                self.chain._scratch()
                g = torch.cuda.CUDAGraph()
                n0 = lib().cbct_launch_count()
                with torch.cuda.graph(g):
                    self._device_iteration(S)
                self.graph_launches = lib().cbct_launch_count() - n0
                self._graph = g
            for _ in range(k):
                self._graph.replay()
        else:
            for _ in range(k):
                self._device_iteration(S)
        if collect:
            self.collect()

    def collect(self) -> None:
        """Synchronise with the device loop and fold its scalars and history into the host state."""
        h = self._S.cpu().numpy()
        self.nr2_old, self.pending = float(h[0]), float(h[3])
        it = int(h[7])
        now = time.perf_counter() - self.t0
        for j in range(self._i0 + 1, it + 1):
            self.nb = self.nb_full = float(np.sqrt(h[16 + j]))  # plain chain: no stacked tail
            self.history.append(ConvergenceRecord(j, now, self.rel(self.nb), None))
        self.i = it
        if h[6] == 1.0:
            self.done = self.breakdown = True

    def report(self) -> SolverReport:
        self.flush()
        op = self.op
        return SolverReport(_final_volume(op, self.chain.x_of(self.x), self.b.data), self.i, self.nb,
                            self.history, getattr(op, "workers", 1), self.breakdown)


@_nvtx("cbct_cgls")
def cgls(op, b, cfg: SolverConfig) -> SolverReport:
    """CGLS with delayed residual (solvers.py:269-358): K+2 A, K+1 A^T."""
    _check_inputs(op, b, cfg, "cgls")
    run = CglsRun(op, b, cfg)
    if run.device_capable():
        # batches of device-resident iterations (one host synchronisation per batch)
        while run.should_continue():
            run.run_device(min(_DEVICE_BATCH, cfg.max_iterations - run.i))
        return run.report()
    while run.should_continue():
        if not run.step():
            break
    return run.report()


_DEVICE_BATCH = 8


def _proj_update(dev, chain, e, p, alpha):
    """e -= alpha*p over the whole (possibly stacked) vector.  Returns (||head(e)||^2,
    ||e||^2): the reference records the data-block norm (report_norm, solvers.py:152-155)
    but stops on the full stacked norm (solvers.py:334, 339, 355)."""
    mo = chain.head(e).numel()
    nb2 = dev.axpby(-alpha, p[:mo], 1.0, e[:mo], norm2=True)
    if e.numel() > mo:
        return nb2, nb2 + dev.axpby(-alpha, p[mo:], 1.0, e[mo:], norm2=True)
    return nb2, nb2


class LsqrRun:
    """LSQR state (solvers.py:361-459): the pre-loop (``__init__``: u = b - A x0, beta, 1 A^T,
    alpha) and one loop iteration (``step``: 1 A + 1 A^T, the normalisations and the Givens
    update).  ``lsqr`` drives it; the benchmark times ``step``."""

    def __init__(self, op, b, cfg: SolverConfig):
        self.op, self.b, self.cfg = op, b, cfg
        self.dev = dev = _Dev(op)
        self.chain = chain = _build_chain(op, cfg, dev)
        self.t0 = time.perf_counter()
        self.b_int = _as_internal_proj(op, b)
        self.x = chain.z_of(_x0_internal(op, cfg, dev)).clone()
        b_eff = chain.rhs(self.b_int)
        self.nb0 = _norm(dev, self.b_int)
        self.history = []
        self.updates = 0
        self.done = False
        self.breakdown = False
        self.u = u = dev.empty(chain.m_phys)
        chain.apply(self.x, u)
        beta = float(np.sqrt(dev.sub(b_eff, u, u, norm2=True)))
        self.phibar = beta
        if beta == 0.0:
            self._record(0, 0.0)
            self.done = self.breakdown = True
            return
        dev.div(u, beta)
        self.v = v = dev.empty(chain.n_phys)
        alpha = float(np.sqrt(chain.applyT(u, v, norm2=True)))
        if alpha == 0.0:
            self._record(0, self.rel(beta))
            self.done = self.breakdown = True
            return
        dev.div(v, alpha)
        self.w = v.clone()
        self.alpha, self.rhobar = alpha, alpha
        self.tmp_m = torch.empty_like(u)
        self.tmp_n = torch.empty_like(v)

    def rel(self, v):
        return v / self.nb0 if self.nb0 > 0 else 0.0

    def _record(self, i, e):
        true_e = None
        if _want_true(self.cfg, i):
            true_e = _true_rel(self.op, self.chain, self.x, self.b_int, self.nb0, self.dev)
        self.history.append(ConvergenceRecord(i, time.perf_counter() - self.t0, e, true_e))

    def should_continue(self) -> bool:
        return not self.done and self.updates < self.cfg.max_iterations + 1

    @_nvtx("cbct_lsqr_iteration")
    def step(self) -> None:
        """One bidiagonalisation step + Givens update + record (solvers.py:427-458)."""
        dev, chain, u, v = self.dev, self.chain, self.u, self.v
        alpha = self.alpha
        chain.apply(v, self.tmp_m)
        beta = float(np.sqrt(dev.axpby(1.0, self.tmp_m, -alpha, u, norm2=True)))  # u = A v - alpha u
        if beta > 0.0:
            dev.div(u, beta)
            chain.applyT(u, self.tmp_n)
            alpha = float(np.sqrt(dev.axpby(1.0, self.tmp_n, -beta, v, norm2=True)))  # v = A^T u - beta v
            if alpha > 0.0:
                dev.div(v, alpha)
        rho = float(np.hypot(self.rhobar, beta))
        c, s = self.rhobar / rho, beta / rho
        theta = s * alpha
        self.rhobar = -c * alpha
        phi = c * self.phibar
        self.phibar = s * self.phibar
        self.alpha = alpha
        dev.update2(self.x, self.w, v, phi / rho, True, -(theta / rho))  # x += (phi/rho) w ; w = v - (theta/rho) w
        self._record(self.updates, self.rel(self.phibar))
        self.updates += 1
        err = self.cfg.rel_discrepancy_tol
        if beta == 0.0 or alpha == 0.0:
            self.done = self.breakdown = True
        elif err > 0.0 and self.rel(self.phibar) <= err:
            self.done = True

    def report(self) -> SolverReport:
        op = self.op
        if getattr(self, "_S", None) is not None:  # device-resident iterations: apply the pending update
            call("cbct_lsqr_flush", self.x.numel(), _p(self.x), _p(self.w), _p(self.v), _p(self._S), self.dev.s())
            self._S = None
        return SolverReport(_final_volume(op, self.chain.x_of(self.x), self.b.data), len(self.history) - 1,
                            self.phibar, self.history, getattr(op, "workers", 1), self.breakdown)

    # ------------------------------------------------- device-resident iterations --
    def device_capable(self) -> bool:
        """The fp32 fused chain, plain or Jacobi-preconditioned (no Tikhonov stacking, no true-discrepancy
        monitoring), runs with every scalar on the device (``run_device``)."""
        c = self.chain
        inner = c.inner if isinstance(c, _JacobiChain) else c
        return (type(c) in (_Chain, _JacobiChain) and type(inner) is _Chain and inner._fused and
                self.cfg.true_discrepancy_every <= 0 and not self.dev.f64 and not self.done)

    def _device_state(self):
        """Scalar array of include/cbct.h cbct_lsqr_scalars, loaded from the host state after the
        pre-loop (u and v normalised: nu = nv = 1; w = v, no update pending)."""
        if getattr(self, "_S", None) is None:
            K = self.cfg.max_iterations
            self._S = torch.zeros(24 + K + 2, dtype=torch.float64, device=self.dev.device)
            host = torch.tensor([self.alpha, 0.0, self.rhobar, self.phibar, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0,
                                 float(self.updates), self.nb0, float(self.cfg.rel_discrepancy_tol), float(K + 1),
                                 0.0], dtype=torch.float64)
            self._S[:17].copy_(host)
            self._jac = self.chain.scale if isinstance(self.chain, _JacobiChain) else None
            self._sv = torch.empty_like(self.v) if self._jac is not None else None
            if self._jac is not None:
                self.dev.mul(self.v, self._jac, self._sv)
            self._inner = self.chain.inner if self._jac is not None else self.chain
        return self._S

    def _device_iteration(self, S):
        op, dev, st = self.op, self.dev, self.dev.s
        inner = self._inner
        op.project_internal(self._sv if self._jac is not None else self.v, self.tmp_m)
        call("cbct_lsqr_u_update", self.u.numel(), _p(self.u), _p(self.tmp_m), _p(S), _p(dev.partials), st())
        op.reduce_to(dev.nblocks(self.u.numel()), S[9:10])
        call("cbct_lsqr_scalars", _p(S), 1, st())
        op.backproject_internal(self.u, self.tmp_n, scratch=inner._scratch(), col_scale=self._jac)
        call("cbct_lsqr_v_update", self.v.numel(), _p(self.x), _p(self.w), _p(self.v), _p(self.tmp_n),
             _p(self._sv), _p(self._jac), _p(S), _p(dev.partials), st())
        op.reduce_to(dev.nblocks(self.v.numel()), S[10:11])
        call("cbct_lsqr_scalars", _p(S), 2, st())

    @_nvtx("cbct_lsqr_device_iterations")
    def run_device(self, k: int, graph: bool = False, collect: bool = True) -> None:
        """Up to k LSQR iterations with the scalars on the device: one A, one A^T and two fused
        vector passes each (include/cbct.h cbct_lsqr_*), no host round trip inside; ``graph`` replays
        one captured CUDA graph of the iteration.  Once used, the run stays on the device (its
        vectors are kept unnormalised); ``report`` applies the pending update."""
        if self.done or k <= 0:
            return
        S = self._device_state()
        self._i0 = self.updates
        if graph:
            if getattr(self, "_graph", None) is None:
                from ._lib import lib

                g = torch.cuda.CUDAGraph()
                n0 = lib().cbct_launch_count()
                with torch.cuda.graph(g):
                    self._device_iteration(S)
                self.graph_launches = lib().cbct_launch_count() - n0
                self._graph = g
            for _ in range(k):
                self._graph.replay()
        else:
            for _ in range(k):
                self._device_iteration(S)
        if collect:
            self.collect()

    def collect(self) -> None:
        h = self._S.cpu().numpy()
        it = int(h[12])
        now = time.perf_counter() - self.t0
        for j in range(self._i0, it):
            self.history.append(ConvergenceRecord(j, now, self.rel(float(h[24 + j])), None))
        self.updates = it
        self.phibar = float(h[3])
        if h[11] != 0.0:
            self.done = True
            self.breakdown = h[11] == 1.0


@_nvtx("cbct_lsqr")
def lsqr(op, b, cfg: SolverConfig) -> SolverReport:
    """LSQR (solvers.py:361-459): Golub-Kahan bidiagonalisation + Givens.  The fp32 fused chain runs
    device-resident (two fused vector passes per iteration, no host round trip); the fp64 path,
    wrapped operators, Tikhonov stacking and true-discrepancy monitoring use the host loop."""
    _check_inputs(op, b, cfg, "lsqr")
    run = LsqrRun(op, b, cfg)
    if run.device_capable():
        while run.should_continue():
            run.run_device(min(_DEVICE_BATCH, cfg.max_iterations + 1 - run.updates))
        return run.report()
    while run.should_continue():
        run.step()
    return run.report()


def _inv_positive(t):
    return torch.where(t > 0, 1.0 / torch.where(t > 0, t, torch.ones_like(t)), torch.zeros_like(t))


def normal_spectral_radius(op, power_iterations: int = 10) -> float:
    """rho(A^T R^-1 A) by power iteration from all-ones (solvers.py:462-489)."""
    if power_iterations < 1:
        raise ValueError("power_iterations must be >= 1")
    dev = _Dev(op)
    row = _as_internal_proj(op, _call_sums(op, "row_sums"))
    inv_row = _inv_positive(row)
    return _spectral(op, dev, inv_row, power_iterations)


def _spectral(op, dev, inv_row, iters):
    proj = dev.empty(op.m)
    w = dev.empty(dev.vol_elems)
    v = torch.empty_like(w)
    dev.fill_volume(v, 1.0)
    chain = _Chain(op, dev)
    for _ in range(iters):
        chain.apply(v, proj)
        dev.mul(proj, inv_row, proj)
        norm = float(np.sqrt(chain.applyT(proj, w, norm2=True)))
        if norm == 0.0:
            raise DegenerateOperatorError("operator never intersects the volume")
        v.copy_(w)
        dev.div(v, norm)
    chain.apply(v, proj)
    dev.mul(proj, inv_row, proj)
    chain.applyT(proj, w)
    return dev.dot(v, w)


_PSIRT_SPECTRAL_SAFETY = 1.05  # solvers.py:496


def psirt_step_scale(op, relaxation: float = 1.0) -> float:
    return 2.0 * relaxation / (_PSIRT_SPECTRAL_SAFETY * normal_spectral_radius(op))


class ClassicalRun:
    """SIRT / PSIRT state (solvers.py:505-569): the setup (``__init__``: row and column sums,
    the PSIRT step from the spectral radius, r = b - A x0) and one iteration (``step``:
    x += step A^T R^-1 r, optional clip, r = b - A x)."""

    def __init__(self, op, b, cfg: SolverConfig, method: str):
        self.op, self.b, self.cfg, self.method = op, b, cfg, method
        self.dev = dev = _Dev(op)
        self.t0 = time.perf_counter()
        row = _as_internal_proj(op, _call_sums(op, "row_sums"))
        col = _as_internal_volume(op, _call_sums(op, "col_sums"))
        if not bool((row > 0).any()) or not bool((col > 0).any()):
            raise DegenerateOperatorError("operator never intersects the volume")
        self.inv_row = _inv_positive(row)
        del row
        if method == "sirt":
            self.step_vec = (cfg.relaxation * _inv_positive(col)).to(dev.dtype)
            self.step_size = None
        else:
            self.step_vec = None
            self.step_size = 2.0 * cfg.relaxation / (_PSIRT_SPECTRAL_SAFETY * _spectral(op, dev, self.inv_row, 10))
        del col
        self.b_int = _as_internal_proj(op, b)
        self.x = _x0_internal(op, cfg, dev)
        self.nb0 = _norm(dev, self.b_int)
        self.lo, self.hi = cfg.box_bounds if cfg.box_bounds is not None else (None, None)
        self.history = []
        self.chain = _Chain(op, dev)
        self.resid = dev.empty(op.m)
        self.weighted = torch.empty_like(self.resid)
        self.upd = dev.empty(dev.vol_elems)
        self.chain.apply(self.x, self.resid)
        self.e = self.rel(float(np.sqrt(dev.sub(self.b_int, self.resid, self.resid, norm2=True))))
        self._record(0)
        self.i = 0

    def rel(self, v):
        return v / self.nb0 if self.nb0 > 0 else 0.0

    def _record(self, i):
        e = self.e
        self.history.append(ConvergenceRecord(i, time.perf_counter() - self.t0, e,
                                              e if _want_true(self.cfg, i) else None))

    def should_continue(self) -> bool:
        err = self.cfg.rel_discrepancy_tol
        return (err == 0.0 or self.e > err) and self.i < self.cfg.max_iterations

    @_nvtx("cbct_classical_iteration")
    def step(self) -> None:
        dev, chain = self.dev, self.chain
        dev.mul(self.resid, self.inv_row, self.weighted)
        chain.applyT(self.weighted, self.upd)
        if self.step_vec is not None:
            dev.mul(self.upd, self.step_vec, self.upd)
            dev.axpby(1.0, self.upd, 1.0, self.x)
        else:
            dev.axpby(self.step_size, self.upd, 1.0, self.x)
        if self.lo is not None:
            dev.clip(self.x, self.lo, self.hi)
        chain.apply(self.x, self.resid)
        self.e = self.rel(float(np.sqrt(dev.sub(self.b_int, self.resid, self.resid, norm2=True))))
        self.i += 1
        self._record(self.i)

    def report(self) -> SolverReport:
        op = self.op
        return SolverReport(_final_volume(op, self.x, self.b.data), self.i, self.e * self.nb0, self.history,
                            getattr(op, "workers", 1), False)

    # ------------------------------------------------- device-resident iterations --
    def device_capable(self) -> bool:
        """The fp32 fused operator without true-discrepancy monitoring runs with the stop tests on the
        device (``run_device``): A^T, one fused volume pass, A, one fused projection pass; bitwise the
        host loop's values (same kernels' arithmetic and reduction grids)."""
        return self.chain._fused and not self.dev.f64 and self.cfg.true_discrepancy_every <= 0

    @_nvtx("cbct_classical_device_iterations")
    def run_device(self, k: int, graph: bool = False, collect: bool = True) -> None:
        if k <= 0 or not self.should_continue():
            return
        dev, op = self.dev, self.op
        if getattr(self, "_S", None) is None:
            self._S = torch.zeros(8 + self.cfg.max_iterations + 2, dtype=torch.float64, device=dev.device)
            self._S[:6].copy_(torch.tensor([0.0, 0.0, float(self.i), self.nb0, float(self.cfg.rel_discrepancy_tol),
                                            float(self.cfg.max_iterations)], dtype=torch.float64))
            dev.mul(self.resid, self.inv_row, self.weighted)
            self._inv_row32 = self.inv_row.to(dev.dtype).contiguous()
            self._step_vec = self.step_vec.contiguous() if self.step_vec is not None else None
        S = self._S
        self._i0 = self.i
        clip = self.lo is not None
        lo = float(self.lo) if clip else 0.0
        hi = float(self.hi) if clip else 0.0

        def iteration():
            st = dev.s()
            op.backproject_internal(self.weighted, self.upd, scratch=self.chain._scratch())
            call("cbct_psirt_volume_update", self.dev.plan, _p(self.x), _p(self.upd), _p(self._step_vec),
                 ctypes.c_float(self.step_size if self.step_size is not None else 0.0), int(clip),
                 ctypes.c_float(lo), ctypes.c_float(hi), _p(S), st)
            op.project_internal(self.x, self.tmp_p)
            call("cbct_psirt_proj_update", self.resid.numel(), _p(self.resid), _p(self.weighted), _p(self.b_int),
                 _p(self.tmp_p), _p(self._inv_row32), _p(S), _p(dev.partials), st)
            op.reduce_to(dev.nblocks(self.resid.numel()), S[0:1])
            call("cbct_psirt_scalars", _p(S), st)

        if not hasattr(self, "tmp_p"):
            self.tmp_p = torch.empty_like(self.resid)
        if graph:
            if getattr(self, "_graph", None) is None:
                from ._lib import lib

                g = torch.cuda.CUDAGraph()
                n0 = lib().cbct_launch_count()
                with torch.cuda.graph(g):
                    iteration()
                self.graph_launches = lib().cbct_launch_count() - n0
                self._graph = g
            for _ in range(k):
                self._graph.replay()
        else:
            for _ in range(k):
                iteration()
        if collect:
            self.collect()

    def collect(self) -> None:
        h = self._S.cpu().numpy()
        it = int(h[2])
        now = time.perf_counter() - self.t0
        for j in range(self._i0 + 1, it + 1):
            self.e = float(h[8 + j])
            self.history.append(ConvergenceRecord(j, now, self.e, None))
        self.i = it


def _classical(op, b, cfg: SolverConfig, method: str) -> SolverReport:  # solvers.py:505-569
    _check_inputs(op, b, cfg, method)
    run = ClassicalRun(op, b, cfg, method)
    err = cfg.rel_discrepancy_tol
    if run.device_capable():
        while run.should_continue():
            run.run_device(min(_DEVICE_BATCH, cfg.max_iterations - run.i))
        return run.report()
    while run.should_continue():
        run.step()
        if err > 0.0 and run.e <= err:
            break
    return run.report()


@_nvtx("cbct_sirt")
def sirt(op, b, cfg: SolverConfig) -> SolverReport:
    """SIRT: x += relaxation C^-1 A^T R^-1 (b - A x), optionally clamped (solvers.py:572-578)."""
    return _classical(op, b, cfg, "sirt")


@_nvtx("cbct_psirt")
def psirt(op, b, cfg: SolverConfig) -> SolverReport:
    """PSIRT: scalar step 2*omega/(1.05*rho) (solvers.py:581-587)."""
    return _classical(op, b, cfg, "psirt")


_SOLVERS = {"cgls": cgls, "lsqr": lsqr, "sirt": sirt, "psirt": psirt}


def solve(op, b, cfg: SolverConfig) -> SolverReport:
    cfg.validate()
    return _SOLVERS[cfg.method](op, b, cfg)


def write_history_csv(history, path) -> None:
    """iter,seconds,rel_discrepancy,true_rel_discrepancy (solvers.py:599-609)."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["iter", "seconds", "rel_discrepancy", "true_rel_discrepancy"])
        for rec in history:
            t = "" if rec.true_rel_discrepancy is None else repr(rec.true_rel_discrepancy)
            w.writerow([rec.iteration, f"{rec.wall_seconds:.6f}", repr(rec.rel_discrepancy), t])
