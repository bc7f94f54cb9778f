"""Multi-rank solver host logic on CPU: world_size 2 and 3 over gloo (no GPU needed).

The sharded drivers of paper_2110_13526_b200.distributed (dist_cgls, dist_lsqr with and without
Jacobi preconditioning, dist_psirt, dist_sirt) run against an oracle-backed local operator that
owns exactly what ShardedOperator owns on a GPU: the ShardLayout view block of the [V][nu][nv]
projection layout and the cell-row slab of the [ny][nx][zs] volume layout, zero guard slices and
zero-padded last blocks included.  Each rank applies the fp64 CPU oracle (the checker) and keeps
its block in the device layout; vectors are fp64 torch.  The drivers must reproduce the
single-process oracle solvers (oracle/oracle.py, a restatement of solvers.py:269-587) to 1e-11,
which exercises the partition, the all_gathers before A and A^T, the rank-ordered scalar sums and
the per-rank Jacobi / row-sum / column-sum slabs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _helpers import geom_from_golden, load_golden

ZPAD = 4


class TorchVectors:
    """fp64 CPU vector backend (test infrastructure), same interface as distributed.CudaVectors."""

    def axpby(self, a, x, b, y, norm2=False):
        y.mul_(b)
        if x is not None:
            y.add_(x, alpha=a)
        return float((y * y).sum()) if norm2 else None

    def sub(self, a, b, out, norm2=False):
        torch.sub(a, b, out=out)
        return float((out * out).sum()) if norm2 else None

    def update2(self, x, d, r, a_prev, do_x, beta):
        if do_x:
            x.add_(d, alpha=a_prev)
        d.mul_(beta).add_(r)

    def sumsq(self, y):
        return float((y * y).sum())

    def div(self, y, d, norm2=False):
        y.div_(d)
        return float((y * y).sum()) if norm2 else None

    def mul(self, a, b, out):
        torch.mul(a, b, out=out)

    def dot(self, x, y):
        return float((x * y).sum())

    def clip(self, x, lo, hi, mask):
        torch.clamp(x, lo, hi, out=x)
        x.mul_(mask)


class LayoutOracleShard:
    """Rank-local A / A^T in the device layouts of ShardedOperator, computed by the CPU oracle."""

    def __init__(self, vg, tr, comm):
        from oracle import oracle as O

        from paper_2110_13526_b200.distributed import ShardLayout

        self.comm = comm
        self.layout = L = ShardLayout(vg, tr, comm.world, comm.rank)
        self.ref = O.OracleOperator(vg, tr, workers=2, threads=2)
        self.L = L
        self._d_full = torch.zeros(L.n_full, dtype=torch.float64)
        self._e_full = torch.zeros(L.m_full, dtype=torch.float64)

    # device layout <-> reference layout (x-fastest volume, u-fastest projections)
    def _vol_ref(self, full):
        L = self.L
        v = full[: L.ny * L.row_elems].numpy().reshape(L.ny, L.nx, L.zs)[:, :, ZPAD:ZPAD + L.nz]
        return np.ascontiguousarray(v.transpose(2, 0, 1)).ravel()

    def _proj_ref(self, full):
        L = self.L
        p = full[: L.n_views * L.view_elems].numpy().reshape(L.n_views, L.nu, L.nv)
        return np.ascontiguousarray(p.transpose(0, 2, 1)).ravel()

    def gather_volume(self, local):
        return self.comm.all_gather(local, self._d_full)

    def gather_proj(self, local):
        return self.comm.all_gather(local, self._e_full)

    def project_local(self, d_full, p_local, norm2=False):
        L = self.L
        full = self.ref.project(self._vol_ref(d_full)).reshape(L.n_views, L.nv, L.nu).transpose(0, 2, 1)
        blk = np.ascontiguousarray(full[L.v0:L.v1]).ravel()
        p_local.zero_()
        p_local[: blk.size] = torch.from_numpy(blk)
        return float((p_local * p_local).sum()) if norm2 else None

    def backproject_local(self, e_full, r_local, norm2=False, mode=1, col_scale=None):
        L = self.L
        ref = self.ref.backproject(self._proj_ref(e_full)) if mode == 1 else self.ref.normal_diagonal()
        vol = ref.reshape(L.nz, L.ny, L.nx).transpose(1, 2, 0)  # (ny, nx, nz)
        out = np.zeros((L.yper, L.nx, L.zs))
        out[: L.y1 - L.y0, :, ZPAD:ZPAD + L.nz] = vol[L.y0:L.y1]
        r_local.copy_(torch.from_numpy(out.ravel()))
        if col_scale is not None:
            r_local.mul_(col_scale)
        return float((r_local * r_local).sum()) if norm2 else None


def _worker(rank, world, port, q, method):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O

        from paper_2110_13526_b200 import distributed as D
        from paper_2110_13526_b200.solvers import SolverConfig

        d = load_golden("adjoint_instance")
        vg, tr = geom_from_golden(d)
        comm = D.TorchComm()
        sop = LayoutOracleShard(vg, tr, comm)
        L = sop.L
        b = O.OracleOperator(vg, tr).project(O.shepp_logan_phantom(vg))
        bd = b.reshape(L.n_views, L.nv, L.nu).transpose(0, 2, 1)[L.v0:L.v1].ravel()
        b_local = torch.zeros(L.m_loc, dtype=torch.float64)
        b_local[: bd.size] = torch.from_numpy(np.ascontiguousarray(bd))
        K = 6
        vec = TorchVectors()
        if method == "cgls":
            info, x_local = D.dist_cgls(sop, vec, b_local, SolverConfig(method="cgls", max_iterations=K))
        elif method in ("lsqr", "lsqrj"):
            cfg = SolverConfig(method="lsqr", max_iterations=K, jacobi_precondition=method == "lsqrj")
            info, x_local = D.dist_lsqr(sop, vec, b_local, cfg)
        elif method == "psirt_box":
            info, x_local = D.dist_psirt(sop, vec, b_local,
                                         SolverConfig(method="psirt", max_iterations=K, box_bounds=(0.0, 0.9)))
        else:
            fn = {"psirt": D.dist_psirt, "sirt": D.dist_sirt}[method]
            info, x_local = fn(sop, vec, b_local, SolverConfig(method=method, max_iterations=K))
        full = sop._vol_ref(sop.gather_volume(x_local)).copy()
        q.put((rank, [h.rel_discrepancy for h in info["history"]], full if rank == 0 else None,
               info["iterations"]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_solution(method, K=6):
    from oracle import oracle as O

    d = load_golden("adjoint_instance")
    vg, tr = geom_from_golden(d)
    ref = O.OracleOperator(vg, tr)
    b = ref.project(O.shepp_logan_phantom(vg))
    if method == "cgls":
        return O.cgls(ref, b, K)
    if method in ("lsqr", "lsqrj"):
        scale = O.jacobi_scale(ref) if method == "lsqrj" else None
        return O.lsqr(ref, b, K, scale=scale)  # x = scale * z already
    if method == "psirt":
        return O.psirt(ref, b, K)
    if method == "psirt_box":
        return O.psirt(ref, b, K, box=(0.0, 0.9))
    # sirt: x += relaxation * C^-1 A^T R^-1 (b - A x)  (solvers.py:572-578, 505-569)
    row, col = ref.row_sums(), ref.col_sums()
    inv_row = np.where(row > 0, 1.0 / np.where(row > 0, row, 1.0), 0.0)
    inv_col = np.where(col > 0, 1.0 / np.where(col > 0, col, 1.0), 0.0)
    x = np.zeros(ref.n)
    nb0 = float(np.linalg.norm(b))
    resid = b - ref.project(x)
    hist = [float(np.linalg.norm(resid)) / nb0]
    for _ in range(K):
        x += inv_col * ref.backproject(resid * inv_row)
        resid = b - ref.project(x)
        hist.append(float(np.linalg.norm(resid)) / nb0)
    return x, hist


def _run(world, method):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, method)) for r in range(world)]
    import queue
    import time

    for p in procs:
        p.start()
    out, t0 = [], time.time()
    while len(out) < world:  # fail fast when a rank dies instead of waiting on the queue
        try:
            out.append(q.get(timeout=1.0))
        except queue.Empty:
            assert all(p.exitcode in (None, 0) for p in procs), [p.exitcode for p in procs]
            assert time.time() - t0 < 300, "sharded solve timed out"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    return out


@pytest.mark.parametrize("world", [2, 3])  # 3 ranks: uneven view blocks and cell-row slabs
@pytest.mark.parametrize("method", ["cgls", "lsqrj", "psirt"])
def test_sharded_solvers_match_single_process(world, method):
    x_ref, h_ref = _oracle_solution(method)
    out = _run(world, method)
    for rank, hist, _, iters in out:
        assert iters == 6
        np.testing.assert_allclose(hist, h_ref, rtol=1e-11)  # every rank sees the same reduced scalars
    x = out[0][2]
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-11


@pytest.mark.parametrize("method", ["lsqr", "sirt", "psirt_box"])
def test_sharded_solver_variants_world2(method):
    """Unpreconditioned LSQR, SIRT's per-voxel column scaling and PSIRT's box clip on the slabs."""
    x_ref, h_ref = _oracle_solution(method)
    out = _run(2, method)
    for _, hist, _, iters in out:
        assert iters == 6
        np.testing.assert_allclose(hist, h_ref, rtol=1e-11)
    x = out[0][2]
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-11
