"""Multi-rank CGLS host logic on CPU: world_size 2 and 3 over gloo (no GPU needed).

The sharded driver (paper_2110_13526_b200.distributed.dist_cgls) is run with an
oracle-backed local operator and fp64 torch vectors.  It must reproduce the
single-process oracle CGLS, which exercises the view / volume block partitioning,
the all_gathers before A and A^T, and the rank-ordered scalar reductions.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _helpers import geom_from_golden, load_golden


class TorchVectors:
    """fp64 CPU vector backend (test infrastructure)."""

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


class OracleShard:
    """Rank-local A / A^T on the CPU oracle: full operator, own block kept."""

    def __init__(self, vg, tr, comm):
        from oracle import oracle as O

        from paper_2110_13526_b200.distributed import block

        self.comm = comm
        self.ref = O.OracleOperator(vg, tr, workers=2, threads=2)
        self.n, self.m = self.ref.n, self.ref.m
        self.ve = tr.detector.nu * tr.detector.nv
        self.v0, self.v1, vper = block(tr.n_views, comm.world, comm.rank)
        _, _, nper = block(self.n, comm.world, comm.rank)
        self.n0 = comm.rank * nper
        self.n1 = min(self.n, self.n0 + nper)
        self.m_loc, self.n_loc = vper * self.ve, nper
        self._d_full = torch.zeros(comm.world * self.n_loc, dtype=torch.float64)
        self._e_full = torch.zeros(comm.world * self.m_loc, dtype=torch.float64)

    def gather_volume(self, local):
        return self.comm.all_gather(local, self._d_full)

    def gather_proj(self, local):
        return self.comm.all_gather(local, self._e_full)

    def project_local(self, d_full, p_local, norm2=False):
        full = self.ref.project(d_full[: self.n].numpy())
        blk = full[self.v0 * self.ve: self.v1 * self.ve]
        p_local.zero_()
        p_local[: blk.size] = torch.from_numpy(blk)
        return float((p_local * p_local).sum()) if norm2 else None

    def backproject_local(self, e_full, r_local, norm2=False):
        full = self.ref.backproject(e_full[: self.m].numpy())
        r_local.zero_()
        r_local[: self.n1 - self.n0] = torch.from_numpy(full[self.n0: self.n1])
        return float((r_local * r_local).sum()) if norm2 else None


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O

        from paper_2110_13526_b200.distributed import TorchComm, dist_cgls
        from paper_2110_13526_b200.solvers import SolverConfig

        d = load_golden("adjoint_instance")
        vg, tr = geom_from_golden(d)
        comm = TorchComm()
        sop = OracleShard(vg, tr, comm)
        b = O.OracleOperator(vg, tr).project(O.shepp_logan_phantom(vg))
        b_local = torch.zeros(sop.m_loc, dtype=torch.float64)
        blk = b[sop.v0 * sop.ve: sop.v1 * sop.ve]
        b_local[: blk.size] = torch.from_numpy(blk)
        info, x_local = dist_cgls(sop, TorchVectors(), b_local, SolverConfig(method="cgls", max_iterations=6))
        full = sop.gather_volume(x_local)[: sop.n].numpy().copy()
        q.put((rank, [h.rel_discrepancy for h in info["history"]], full if rank == 0 else None,
               info["iterations"]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])  # 3 ranks: uneven view and volume blocks
def test_sharded_cgls_matches_single_process(world):
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    d = load_golden("adjoint_instance")
    vg, tr = geom_from_golden(d)
    ref = O.OracleOperator(vg, tr)
    b = ref.project(O.shepp_logan_phantom(vg))
    x_ref, h_ref = O.cgls(ref, b, 6)
    for rank, hist, _, iters in out:
        assert iters == 6
        np.testing.assert_allclose(hist, h_ref, rtol=1e-11)  # both ranks see the same reduced scalars
    x = out[0][2]
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-11


def test_block_partition_covers_exactly():
    from paper_2110_13526_b200.distributed import block

    for n, w in ((360, 8), (361, 8), (7, 8), (256, 3), (1, 1)):
        seen = []
        for r in range(w):
            lo, hi, per = block(n, w, r)
            assert hi - lo <= per and per * w >= n
            seen.extend(range(lo, hi))
        assert seen == list(range(n))
