"""Multi-GPU CGLS: projection space sharded by view, volume space by cell rows.

One process per GPU (torchrun), NCCL over NVLink for the exchanges (SURVEY.md 8(e),
DESIGN.md section 5):

* rank r owns the view block [v0, v1) of every projection-space vector (b, e, p) --
  contiguous in the [V][nu][nv] device layout -- and applies A to those views;
* rank r owns the cell rows [y0, y1) of every volume-space vector (x, d, r) --
  contiguous in the [ny][nx][zs] device layout -- and applies A^T to those cells
  (gathering over all views);
* per CGLS iteration: all_gather(d) before A, all_gather(e) before A^T, and the
  three squared norms as per-rank fp64 partials gathered and summed in rank order
  (bitwise reproducible for a fixed world size).

Shards are equal-sized (the last one zero-padded), so the gathered buffer *is* the
full device layout and the CUDA kernels read it unchanged.  The driver is written
against two small interfaces -- a local operator (project_local / backproject_local)
and a vector backend -- so the same recurrences are exercised on CPU with gloo in
tests/test_distributed_cpu.py.
"""

from __future__ import annotations

import ctypes
import math
import time

import torch

from . import hostcopy
from ._lib import call
from .solvers import ConvergenceRecord, SolverReport, SolverConfig, _nvtx

__all__ = ["block", "ShardLayout", "ShardedOperator", "CudaVectors", "TorchComm", "DistCglsRun", "dist_cgls",
           "DistLsqrRun", "dist_lsqr", "DistClassicalRun", "dist_psirt", "dist_sirt", "gathered_report"]


def block(n: int, world: int, rank: int):
    """Equal-size contiguous block of n items for `rank`: (lo, hi, per); hi - lo may be < per."""
    per = -(-n // world)
    lo = min(n, rank * per)
    return lo, min(n, lo + per), per


class ShardLayout:
    """Which slice of the device layouts a rank owns (no CUDA needed: the CPU tests shard with it).

    Projection space: the view block [v0, v1) of [V][nu][nv] (``m_loc`` elements, the last rank's
    block zero-padded to equal size).  Volume space: the cell rows [y0, y1) of [ny][nx][zs]
    (``n_loc`` elements, zero-padded likewise), so an all_gather of equal blocks *is* the full
    device layout."""

    def __init__(self, vol_geom, trajectory, world: int, rank: int):
        from ._lib import zstride

        det = trajectory.detector
        self.world, self.rank = world, rank
        self.nx, self.ny, self.nz = vol_geom.nx, vol_geom.ny, vol_geom.nz
        self.zs = zstride(vol_geom.nz)
        self.nu, self.nv, self.n_views = det.nu, det.nv, trajectory.n_views
        self.v0, self.v1, self.vper = block(trajectory.n_views, world, rank)
        self.y0, self.y1, self.yper = block(vol_geom.ny, world, rank)
        self.view_elems = det.nu * det.nv
        self.row_elems = vol_geom.nx * self.zs
        self.m_loc = self.vper * self.view_elems
        self.n_loc = self.yper * self.row_elems
        self.m_full = world * self.m_loc
        self.n_full = world * self.n_loc

    def volume_mask(self, dtype, device):
        """1 on this rank's voxels, 0 on the z guards and on the zero-padded rows of its slab."""
        from ._lib import CBCT_ZPAD

        m = torch.zeros(self.yper, self.nx, self.zs, dtype=dtype, device=device)
        m[: self.y1 - self.y0, :, CBCT_ZPAD:CBCT_ZPAD + self.nz] = 1.0
        return m.view(-1)

    def proj_mask(self, dtype, device):
        m = torch.zeros(self.m_loc, dtype=dtype, device=device)
        m[: (self.v1 - self.v0) * self.view_elems] = 1.0
        return m


class TorchComm:
    """torch.distributed collectives used by the driver (NCCL on GPU, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, local: torch.Tensor, full: torch.Tensor) -> torch.Tensor:
        self.dist.all_gather_into_tensor(full, local, group=self.group)
        return full

    def allmax(self, value: float, device) -> float:
        t = torch.tensor([value], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def allsum(self, value: float, device) -> float:
        """Sum of per-rank fp64 partials in rank order (deterministic for a fixed world)."""
        t = torch.tensor([value], dtype=torch.float64, device=device)
        out = torch.empty(self.world, dtype=torch.float64, device=device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        acc = 0.0
        for v in out.cpu().tolist():
            acc += v
        return acc


class CudaVectors:
    """Vector backend on libcbct's fused kernels (deterministic fp64 partials)."""

    def __init__(self, op):
        from .solvers import _Dev

        self.dev = _Dev(op)

    def axpby(self, a, x, b, y, norm2=False):
        return self.dev.axpby(a, x, b, y, norm2=norm2)

    def sub(self, a, b, out, norm2=False):
        return self.dev.sub(a, b, out, norm2=norm2)

    def update2(self, x, d, r, a_prev, do_x, beta):
        self.dev.update2(x, d, r, a_prev, do_x, beta)

    def sumsq(self, y):
        return self.dev.sumsq(y)

    def div(self, y, d, norm2=False):
        return self.dev.div(y, d, norm2=norm2)

    def mul(self, a, b, out):
        self.dev.mul(a, b, out)

    def dot(self, x, y):
        return self.dev.dot(x, y)

    def clip(self, x, lo, hi, mask):
        """np.clip on this rank's voxels (guards and padded rows stay 0)."""
        torch.clamp(x, lo, hi, out=x)
        x.mul_(mask)


class ShardedOperator:
    """Rank-local A (own views, full volume in) and A^T (own cell rows, all views in) on one GPU."""

    def __init__(self, vol_geom, trajectory, comm, device=None):
        from .operator import CbctOperator

        self.comm = comm
        self.world, self.rank = comm.world, comm.rank
        self.layout = L = ShardLayout(vol_geom, trajectory, self.world, self.rank)
        # rank-local plan: the column table of this rank's views and the cell table of its cell
        # rows only (~1/world of the tables, cbct_plan_create_shard).  An empty block (more ranks
        # than views or rows) keeps one item, which is never launched.
        V, ny = trajectory.n_views, vol_geom.ny
        sv0 = min(L.v0, V - 1)
        sy0 = min(L.y0, ny - 1)
        shard = (sv0, max(L.v1, sv0 + 1), sy0, max(L.y1, sy0 + 1))
        full = shard == (0, V, 0, ny)
        self.op = CbctOperator(vol_geom, trajectory, device=device, _shard=None if full else shard)
        self.device = self.op.device
        det = trajectory.detector
        assert L.zs == self.op.zstride
        self.v0, self.v1, vper = L.v0, L.v1, L.vper
        self.y0, self.y1, yper = L.y0, L.y1, L.yper
        self.view_elems, self.row_elems = L.view_elems, L.row_elems
        self.m_loc, self.n_loc, self.m_full, self.n_full = L.m_loc, L.n_loc, L.m_full, L.n_full
        self.nu = det.nu
        self.nx = vol_geom.nx
        nparts = max(vper * det.nu, -(-vol_geom.nx // 16) * -(-yper // 16) * 256, 1)
        self._parts = torch.empty(nparts, dtype=torch.float64, device=self.device)
        self._scratch = self.op.new_bp_scratch()
        self._d_full = torch.zeros(self.n_full, dtype=torch.float32, device=self.device)
        self._e_full = torch.zeros(self.m_full, dtype=torch.float32, device=self.device)

    def _s(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _p(self, t):
        return ctypes.c_void_p(t.data_ptr()) if t is not None else None

    def _reduce(self, n, norm_out=None):
        if norm_out is not None:  # device scalar, no host round trip
            call("cbct_reduce_partials", self._p(self._parts), int(n), self._p(norm_out), None, self._s())
            return None
        call("cbct_reduce_partials", self._p(self._parts), int(n), self._p(self.op._red),
             ctypes.byref(self.op._host), self._s())
        return float(self.op._host.value)

    # ---------------------------------------------- fused updates over peer memory --
    def enable_p2p(self):
        """Allocate the full d / e buffers in symmetric memory (peer-addressable over NVLink) so
        the CGLS vector updates can store their new slab straight into every rank's buffer
        (cbct_cgls_*_update_p2p) and a device barrier replaces each all_gather."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        group = self.comm.group if self.comm.group is not None else dist.group.WORLD
        self._d_full = symm_mem.empty(self.n_full, dtype=torch.float32, device=self.device)
        self._e_full = symm_mem.empty(self.m_full, dtype=torch.float32, device=self.device)
        self._d_full.zero_()
        self._e_full.zero_()
        self._hd = symm_mem.rendezvous(self._d_full, group)
        self._he = symm_mem.rendezvous(self._e_full, group)
        self.p2p = True
        return self

    def d_slab(self):
        """This rank's slab of the full d buffer (its local d in the fused path)."""
        return self._d_full[self.rank * self.n_loc:(self.rank + 1) * self.n_loc]

    def e_slab(self):
        return self._e_full[self.rank * self.m_loc:(self.rank + 1) * self.m_loc]

    def gather_volume(self, local):
        return self.comm.all_gather(local, self._d_full)

    def gather_proj(self, local):
        return self.comm.all_gather(local, self._e_full)

    def project_local(self, d_full, p_local, norm2=False, norm_out=None):
        """p_local = (A d)[views v0..v1) ; returns the local ||p||^2 partial (or reduces it into the
        device scalar ``norm_out``)."""
        if self.v1 <= self.v0:
            if norm_out is not None:
                norm_out.zero_()
            return 0.0 if norm2 else None
        n = (self.v1 - self.v0) * self.nu
        want = norm2 or norm_out is not None
        call("cbct_project_views", self.op._plan, self._p(d_full), self._p(p_local), self.v0, self.v1,
             self._p(self._parts) if want else None, self._s())
        return self._reduce(n, norm_out) if want else None

    def backproject_local(self, e_full, r_local, norm2=False, norm_out=None, mode=1, col_scale=None):
        """r_local = (A^T e)[cell rows y0..y1) (mode 2: diag(A^T A) of those rows, e ignored), times
        the local ``col_scale`` slab if given; returns the local ||r||^2 partial (or reduces it into
        the device scalar ``norm_out``)."""
        if self.y1 <= self.y0:
            if norm_out is not None:
                norm_out.zero_()
            return 0.0 if norm2 else None
        n = -(-self.nx // 16) * -(-(self.y1 - self.y0) // 16) * 256
        want = norm2 or norm_out is not None
        call("cbct_backproject_rows", self.op._plan, self._p(e_full) if mode == 1 else None, self._p(r_local),
             self.y0, self.y1, int(mode), self._p(self._scratch), self._p(col_scale),
             self._p(self._parts) if want else None, self._s())
        return self._reduce(n, norm_out) if want else None


class DistCglsRun:
    """Sharded CGLS state (solvers.py:269-358 recurrences).  ``__init__`` runs the pre-loop
    (2 A + 1 A^T, first update folded in); ``step`` one loop iteration (1 A^T + 1 A, one
    all_gather each, two fused vector passes, three rank-ordered scalar reductions)."""

    def __init__(self, sop, vec, b_local: torch.Tensor, cfg: SolverConfig, record: bool = True, x0_local=None):
        self.sop, self.vec, self.cfg, self.record = sop, vec, cfg, record
        comm = sop.comm
        dev = b_local.device
        self.allsum = lambda v: comm.allsum(v, dev)  # noqa: E731
        self.t0 = time.perf_counter()
        self.b = b_local
        self.x = torch.zeros(sop.layout.n_loc, dtype=b_local.dtype, device=dev) if x0_local is None else \
            x0_local.clone()
        # fused path: d and e are this rank's slabs of the symmetric full buffers (the NCCL gathers of
        # the pre-loop below are then in place)
        self.p2p = getattr(sop, "p2p", False)
        self.d = sop.d_slab() if self.p2p else torch.zeros_like(self.x)
        self.r = torch.zeros_like(self.x)
        self.e = sop.e_slab() if self.p2p else torch.zeros_like(b_local)
        self.p = torch.zeros_like(b_local)
        self.nb0 = math.sqrt(self.allsum(vec.sumsq(b_local)))
        self.hist = []
        self.i = 0
        self.pending = 0.0
        self.done = self.breakdown = False
        sop.project_local(sop.gather_volume(self.x), self.p)
        vec.sub(b_local, self.p, self.e)
        self.nr2_old = self.allsum(sop.backproject_local(sop.gather_proj(self.e), self.r, norm2=True))
        self.nb = math.sqrt(self.allsum(vec.sumsq(self.e)))
        if self.nr2_old == 0.0:
            self._rec(0)
            self.done = self.breakdown = True
            return
        self.d.copy_(self.r)
        np2 = self.allsum(sop.project_local(sop.gather_volume(self.d), self.p, norm2=True))
        if np2 == 0.0:
            self._rec(0)
            self.done = self.breakdown = True
            return
        self.pending = self.nr2_old / np2
        self.nb = math.sqrt(self.allsum(vec.axpby(-self.pending, self.p, 1.0, self.e, norm2=True)))
        self._rec(0)

    def rel(self, v):
        return v / self.nb0 if self.nb0 > 0 else 0.0

    def _rec(self, i):
        if self.record:
            self.hist.append(ConvergenceRecord(i, time.perf_counter() - self.t0, self.rel(self.nb), None))

    def should_continue(self):
        return not self.done and self.rel(self.nb) > self.cfg.rel_discrepancy_tol and \
            self.i < self.cfg.max_iterations

    @_nvtx("cbct_dist_cgls_iteration")
    def step(self) -> bool:
        sop, vec = self.sop, self.vec
        nr2 = self.allsum(sop.backproject_local(sop.gather_proj(self.e), self.r, norm2=True))
        if nr2 == 0.0:
            self.done = self.breakdown = True
            return False
        beta = nr2 / self.nr2_old
        vec.update2(self.x, self.d, self.r, self.pending, self.pending != 0.0, beta)
        self.pending = 0.0
        self.nr2_old = nr2
        np2 = self.allsum(sop.project_local(sop.gather_volume(self.d), self.p, norm2=True))
        if np2 == 0.0:
            self.done = self.breakdown = True
            return False
        self.pending = self.nr2_old / np2
        self.nb = math.sqrt(self.allsum(vec.axpby(-self.pending, self.p, 1.0, self.e, norm2=True)))
        self.i += 1
        self._rec(self.i)
        return True

    # ------------------------------------------------- device-resident iterations --
    @_nvtx("cbct_dist_cgls_device_iterations")
    def run_device(self, k: int) -> None:
        """Up to k iterations with every scalar on the device (NCCL + libcbct only): the local norm
        partials are reduced into device scalars, all-gathered (8 bytes per rank) and summed in rank
        order by cbct_sum_ranks -- the same fp64 additions as ``TorchComm.allsum`` -- and
        cbct_cgls_scalars / the device-scalar updates run the recurrences as in the single-GPU loop
        (solvers.CglsRun.run_device).  One synchronisation at the end; iterates bit-identical to k
        calls of ``step``."""
        if self.done or k <= 0:
            return
        import torch

        from ._lib import call as _call

        sop, vec, dev = self.sop, self.vec, self.b.device
        if getattr(self, "_S", None) is None:
            self._S = torch.zeros(16 + self.cfg.max_iterations + 2, dtype=torch.float64, device=dev)
            self._loc = torch.zeros(1, dtype=torch.float64, device=dev)
            self._all = torch.zeros(sop.world, dtype=torch.float64, device=dev)
        S, loc, allv = self._S, self._loc, self._all
        S[:11].copy_(torch.tensor([self.nr2_old, 0.0, 0.0, self.pending, 0.0, 0.0, 0.0, float(self.i), self.nb0,
                                   float(self.cfg.rel_discrepancy_tol), 0.0], dtype=torch.float64))
        st = sop._s
        p = sop._p

        def allsum_into(slot):
            sop.comm.all_gather(loc, allv)
            _call("cbct_sum_ranks", p(allv), sop.world, p(S[slot:slot + 1]), st())

        i0 = self.i
        if self.p2p:
            sop.gather_proj(self.e)  # e_full current for the first A^T (the updates keep it so after)
        for _ in range(k):
            e_full = sop._e_full if self.p2p else sop.gather_proj(self.e)
            sop.backproject_local(e_full, self.r, norm_out=loc)
            allsum_into(1)
            _call("cbct_cgls_scalars", p(S), 1, st())
            if self.p2p:  # d update + its all-gather in one kernel, NVLink stores to every rank's buffer
                _call("cbct_cgls_volume_update_p2p", self.d.numel(), p(self.x), p(self.d), p(self.r), p(S),
                      ctypes.c_void_p(sop._hd.buffer_ptrs_dev), sop.world, sop.rank * sop.n_loc, st())
                sop._hd.barrier(channel=0)
                d_full = sop._d_full
            else:
                _call("cbct_cgls_volume_update_dev", self.d.numel(), p(self.x), p(self.d), p(self.r), p(S), st())
                d_full = sop.gather_volume(self.d)
            sop.project_local(d_full, self.p, norm_out=loc)
            allsum_into(2)
            _call("cbct_cgls_scalars", p(S), 2, st())
            if self.p2p:
                _call("cbct_cgls_proj_update_p2p", self.e.numel(), p(self.e), p(self.p), p(S),
                      p(vec.dev.partials), ctypes.c_void_p(sop._he.buffer_ptrs_dev), sop.world,
                      sop.rank * sop.m_loc, st())
            else:
                _call("cbct_cgls_proj_update_dev", self.e.numel(), p(self.e), p(self.p), p(S),
                      p(vec.dev.partials), st())
            _call("cbct_reduce_partials", p(vec.dev.partials), vec.dev.nblocks(self.e.numel()), p(loc), None, st())
            if self.p2p:
                sop._he.barrier(channel=0)
            allsum_into(5)
            _call("cbct_cgls_scalars", p(S), 3, st())
        h = S.cpu().numpy()
        self.nr2_old, self.pending = float(h[0]), float(h[3])
        it = int(h[7])
        for j in range(i0 + 1, it + 1):
            self.nb = math.sqrt(h[16 + j])
            self.i = j
            self._rec(j)
        self.i = it
        if h[6] == 1.0:
            self.done = self.breakdown = True

    def finish(self):
        if self.pending != 0.0:
            self.vec.axpby(self.pending, self.d, 1.0, self.x)
            self.pending = 0.0
        return {"iterations": self.i, "final_discrepancy_norm": self.nb, "history": self.hist,
                "breakdown": self.breakdown, "worker_count": self.sop.comm.world}, self.x


def dist_cgls(sop, vec, b_local: torch.Tensor, cfg: SolverConfig, record: bool = True, x0_local=None):
    """Run sharded CGLS to completion; returns (info dict, local x shard)."""
    run = DistCglsRun(sop, vec, b_local, cfg, record, x0_local)
    while run.should_continue():
        if not run.step():
            break
    return run.finish()


class DistLsqrRun:
    """Sharded LSQR (solvers.py:361-459) with optional Jacobi preconditioning (solvers.py:158-193):
    u and the projection temporaries live in view blocks, v, w, x and the Jacobi scale in cell-row
    slabs; A needs all_gather(scale * v), A^T all_gather(u); the two norms per iteration are
    rank-ordered fp64 sums.  Same vector kernels as the single-GPU ``solvers.LsqrRun``, so at one
    rank the iterates are bitwise those of ``lsqr``."""

    def __init__(self, sop, vec, b_local: torch.Tensor, cfg: SolverConfig, record: bool = True):
        self.sop, self.vec, self.cfg, self.record = sop, vec, cfg, record
        comm = sop.comm
        dev = b_local.device
        self.allsum = lambda v: comm.allsum(v, dev)  # noqa: E731
        self.t0 = time.perf_counter()
        L = sop.layout
        self.hist = []
        self.updates = 0
        self.done = self.breakdown = False
        self.scale = None
        if cfg.jacobi_precondition:
            diag = torch.zeros(L.n_loc, dtype=b_local.dtype, device=dev)
            sop.backproject_local(None, diag, mode=2)
            dmax = comm.allmax(float(diag.max()) if diag.numel() else 0.0, dev)
            if dmax <= 0:
                from .solvers import DegenerateOperatorError

                raise DegenerateOperatorError("normal-equation diagonal is identically zero")
            floored = torch.clamp(diag.double(), min=cfg.jacobi_floor * dmax)
            self.scale = (1.0 / torch.sqrt(floored)).to(b_local.dtype) * L.volume_mask(b_local.dtype, dev)
            self._sv = torch.zeros(L.n_loc, dtype=b_local.dtype, device=dev)
        self.b = b_local
        self.x = torch.zeros(L.n_loc, dtype=b_local.dtype, device=dev)
        self.nb0 = math.sqrt(self.allsum(vec.sumsq(b_local)))
        self.u = u = torch.empty_like(b_local)
        self._apply(self.x, u)
        beta = math.sqrt(self.allsum(vec.sub(b_local, u, u, norm2=True)))
        self.phibar = beta
        if beta == 0.0:
            self._rec(0, 0.0)
            self.done = self.breakdown = True
            return
        vec.div(u, beta)
        self.v = v = torch.empty_like(self.x)
        alpha = math.sqrt(self.allsum(self._applyT(u, v, norm2=True)))
        if alpha == 0.0:
            self._rec(0, self.rel(beta))
            self.done = self.breakdown = True
            return
        vec.div(v, alpha)
        self.w = v.clone()
        self.alpha = self.rhobar = alpha
        self.tmp_m = torch.empty_like(u)
        self.tmp_n = torch.empty_like(v)

    def _apply(self, z, out):
        """out = A (scale * z) on this rank's views."""
        sop = self.sop
        if self.scale is not None:
            self.vec.mul(z, self.scale, self._sv)
            z = self._sv
        sop.project_local(sop.gather_volume(z), out)

    def _applyT(self, y, out, norm2=False):
        """out = scale * A^T y on this rank's cell rows; the local ||out||^2 partial if norm2."""
        sop = self.sop
        return sop.backproject_local(sop.gather_proj(y), out, norm2=norm2, col_scale=self.scale)

    def rel(self, v):
        return v / self.nb0 if self.nb0 > 0 else 0.0

    def _rec(self, i, e):
        if self.record:
            self.hist.append(ConvergenceRecord(i, time.perf_counter() - self.t0, e, None))

    def should_continue(self):
        return not self.done and self.updates < self.cfg.max_iterations + 1

    @_nvtx("cbct_dist_lsqr_iteration")
    def step(self) -> None:
        vec, u, v = self.vec, self.u, self.v
        alpha = self.alpha
        self._apply(v, self.tmp_m)
        beta = math.sqrt(self.allsum(vec.axpby(1.0, self.tmp_m, -alpha, u, norm2=True)))  # u = A v - alpha u
        if beta > 0.0:
            vec.div(u, beta)
            self._applyT(u, self.tmp_n)
            alpha = math.sqrt(self.allsum(vec.axpby(1.0, self.tmp_n, -beta, v, norm2=True)))  # v = A^T u - beta v
            if alpha > 0.0:
                vec.div(v, alpha)
        rho = math.hypot(self.rhobar, beta)
        c, s = self.rhobar / rho, beta / rho
        theta = s * alpha
        self.rhobar = -c * alpha
        phi = c * self.phibar
        self.phibar = s * self.phibar
        self.alpha = alpha
        vec.update2(self.x, self.w, v, phi / rho, True, -(theta / rho))
        self._rec(self.updates, self.rel(self.phibar))
        self.updates += 1
        err = self.cfg.rel_discrepancy_tol
        if beta == 0.0 or alpha == 0.0:
            self.done = self.breakdown = True
        elif err > 0.0 and self.rel(self.phibar) <= err:
            self.done = True

    def finish(self):
        x = self.x
        if self.scale is not None:
            x = torch.empty_like(self.x)
            self.vec.mul(self.x, self.scale, x)
        return {"iterations": len(self.hist) - 1, "final_discrepancy_norm": self.phibar, "history": self.hist,
                "breakdown": self.breakdown, "worker_count": self.sop.comm.world}, x


def dist_lsqr(sop, vec, b_local: torch.Tensor, cfg: SolverConfig, record: bool = True):
    """Run sharded LSQR to completion; returns (info dict, local x shard)."""
    run = DistLsqrRun(sop, vec, b_local, cfg, record)
    while run.should_continue():
        run.step()
    return run.finish()


_PSIRT_SPECTRAL_SAFETY = 1.05  # solvers.py:496


def _inv_positive(t):
    return torch.where(t > 0, 1.0 / torch.where(t > 0, t, torch.ones_like(t)), torch.zeros_like(t))


class DistClassicalRun:
    """Sharded SIRT / PSIRT (solvers.py:462-587): the row sums (A 1) and R^-1 live in view blocks,
    the column sums (A^T 1), x and the update in cell-row slabs; the PSIRT step comes from the same
    10-step power iteration from all-ones as normal_spectral_radius (solvers.py:462-489), with
    rank-ordered norm and dot reductions.  Per iteration: all_gather(R^-1 r) before A^T and
    all_gather(x) before A."""

    def __init__(self, sop, vec, b_local: torch.Tensor, cfg: SolverConfig, method: str, record: bool = True):
        from .solvers import DegenerateOperatorError

        self.sop, self.vec, self.cfg, self.method, self.record = sop, vec, cfg, method, record
        comm = sop.comm
        dev = b_local.device
        dt = b_local.dtype
        self.allsum = lambda v: comm.allsum(v, dev)  # noqa: E731
        self.t0 = time.perf_counter()
        L = sop.layout
        self.mask = L.volume_mask(dt, dev)
        ones_p = L.proj_mask(dt, dev)
        row = torch.empty_like(b_local)
        sop.project_local(sop.gather_volume(self.mask), row)
        col = torch.empty_like(self.mask)
        sop.backproject_local(sop.gather_proj(ones_p), col)
        if self.allsum(float((row > 0).any())) == 0.0 or self.allsum(float((col > 0).any())) == 0.0:
            raise DegenerateOperatorError("operator never intersects the volume")
        self.inv_row = _inv_positive(row)
        del row
        if method == "sirt":
            self.step_vec = cfg.relaxation * _inv_positive(col)
            self.step_size = None
        else:
            self.step_vec = None
            self.step_size = 2.0 * cfg.relaxation / (_PSIRT_SPECTRAL_SAFETY * self._spectral(10))
        del col
        self.b = b_local
        self.x = torch.zeros_like(self.mask)
        self.nb0 = math.sqrt(self.allsum(vec.sumsq(b_local)))
        self.lo, self.hi = cfg.box_bounds if cfg.box_bounds is not None else (None, None)
        self.hist = []
        self.resid = torch.empty_like(b_local)
        self.weighted = torch.empty_like(b_local)
        self.upd = torch.empty_like(self.x)
        self._residual()
        self._rec(0)
        self.i = 0

    def _spectral(self, iters):
        """rho(A^T R^-1 A) by power iteration from all-ones (solvers.py:462-489)."""
        from .solvers import DegenerateOperatorError

        sop, vec = self.sop, self.vec
        proj = torch.empty_like(self.inv_row)
        v = self.mask.clone()
        w = torch.empty_like(v)
        for _ in range(iters):
            sop.project_local(sop.gather_volume(v), proj)
            vec.mul(proj, self.inv_row, proj)
            norm = math.sqrt(self.allsum(sop.backproject_local(sop.gather_proj(proj), w, norm2=True)))
            if norm == 0.0:
                raise DegenerateOperatorError("operator never intersects the volume")
            v.copy_(w)
            vec.div(v, norm)
        sop.project_local(sop.gather_volume(v), proj)
        vec.mul(proj, self.inv_row, proj)
        sop.backproject_local(sop.gather_proj(proj), w)
        return self.allsum(vec.dot(v, w))

    def _residual(self):
        sop = self.sop
        sop.project_local(sop.gather_volume(self.x), self.resid)
        self.e = self.rel(math.sqrt(self.allsum(self.vec.sub(self.b, self.resid, self.resid, norm2=True))))

    def rel(self, v):
        return v / self.nb0 if self.nb0 > 0 else 0.0

    def _rec(self, i):
        if self.record:
            self.hist.append(ConvergenceRecord(i, time.perf_counter() - self.t0, self.e, None))

    def should_continue(self):
        err = self.cfg.rel_discrepancy_tol
        return (err == 0.0 or self.e > err) and self.i < self.cfg.max_iterations

    @_nvtx("cbct_dist_classical_iteration")
    def step(self) -> None:
        sop, vec = self.sop, self.vec
        vec.mul(self.resid, self.inv_row, self.weighted)
        sop.backproject_local(sop.gather_proj(self.weighted), self.upd)
        if self.step_vec is not None:
            vec.mul(self.upd, self.step_vec, self.upd)
            vec.axpby(1.0, self.upd, 1.0, self.x)
        else:
            vec.axpby(self.step_size, self.upd, 1.0, self.x)
        if self.lo is not None:
            vec.clip(self.x, self.lo, self.hi, self.mask)
        self._residual()
        self.i += 1
        self._rec(self.i)

    def finish(self):
        return {"iterations": self.i, "final_discrepancy_norm": self.e * self.nb0, "history": self.hist,
                "breakdown": False, "worker_count": self.sop.comm.world}, self.x


def _dist_classical(sop, vec, b_local, cfg, method, record=True):
    run = DistClassicalRun(sop, vec, b_local, cfg, method, record)
    err = cfg.rel_discrepancy_tol
    while run.should_continue():
        run.step()
        if err > 0.0 and run.e <= err:
            break
    return run.finish()


def dist_psirt(sop, vec, b_local, cfg: SolverConfig, record: bool = True):
    """Run sharded PSIRT (solvers.py:581-587) to completion; returns (info dict, local x shard)."""
    return _dist_classical(sop, vec, b_local, cfg, "psirt", record)


def dist_sirt(sop, vec, b_local, cfg: SolverConfig, record: bool = True):
    """Run sharded SIRT (solvers.py:572-578) to completion; returns (info dict, local x shard)."""
    return _dist_classical(sop, vec, b_local, cfg, "sirt", record)


def gathered_report(sop, x_local, info) -> SolverReport:
    """Gather the volume shards and report like the single-GPU solvers (reference layout)."""
    from .phantom import Volume

    full = sop.gather_volume(x_local)[: sop.op.vol_elems]
    xr = hostcopy.to_host(sop.op.volume_from_internal(full, torch.float64))
    return SolverReport(Volume(sop.op.vol_geom, xr), info["iterations"], info["final_discrepancy_norm"],
                        info["history"], info["worker_count"], info["breakdown"])
