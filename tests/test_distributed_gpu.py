"""Sharded CUDA kernels and the sharded CGLS driver on one GPU.

Only one GPU is available, so multi-rank behaviour is covered by (a) evaluating every
rank's view block / cell-row slab in one process ("virtual ranks", no collectives) and
checking the assembled result bit-for-bit against the unsharded kernels, and (b) the
full NCCL driver at world size 1 against the single-GPU solver; the multi-rank
collectives are covered on CPU (tests/test_distributed_cpu.py).
"""

import os
import socket

import numpy as np
import pytest
import torch

from _helpers import baseline_geometry, geom_from_golden, load_golden

pytestmark = pytest.mark.gpu


class _VirtualComm:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_kernels_assemble_to_full(world):
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.distributed import ShardedOperator

    vg, tr = baseline_geometry(64, 90, 128, 96)
    full = P.CbctOperator(vg, tr)
    x = full.volume_to_internal(P.generate_phantom(P.shepp_logan_3d(), vg).data)
    y = torch.randn(full.m, device="cuda")
    p_full = full.new_projections()
    full.project_internal(x, p_full)
    r_full = full.new_volume()
    full.backproject_internal(y, r_full)
    p_parts, r_parts = [], []
    for rank in range(world):
        sop = ShardedOperator(vg, tr, _VirtualComm(world, rank))
        d_full = torch.zeros(sop.n_full, device="cuda")
        d_full[: full.vol_elems] = x
        e_full = torch.zeros(sop.m_full, device="cuda")
        e_full[: full.m] = y
        p_loc = torch.zeros(sop.m_loc, device="cuda")
        r_loc = torch.zeros(sop.n_loc, device="cuda")
        sop.project_local(d_full, p_loc)
        sop.backproject_local(e_full, r_loc)
        p_parts.append(p_loc)
        r_parts.append(r_loc)
    p_cat = torch.cat(p_parts)[: full.m]
    r_cat = torch.cat(r_parts)[: full.vol_elems]
    assert torch.equal(p_cat, p_full)
    assert torch.equal(r_cat, r_full)


@pytest.mark.parametrize("world", [3, 8])
def test_shard_plans_at_config3_geometry(world):
    """Rank-local plans (cbct_plan_create_shard) at BASELINE config-3 cell and detector sizes on a
    view subset and a z slab, where A^T runs the sided kernel: every rank's A on its views and
    A^T / diag(A^T A) on its cell rows reassemble bit-for-bit to the unsharded plan, and each
    rank's tables are ~1/world of the unsharded plan's (column table of its views, cell table of
    its rows)."""
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.distributed import ShardedOperator

    vg, tr = baseline_geometry(512, 720, 616, 480, views=(100, 24), zslab=(224, 64))
    full = P.CbctOperator(vg, tr)
    assert full.info.bp_sided_gs > 0
    x = full.volume_to_internal(P.generate_phantom(P.shepp_logan_3d(), vg).data)
    y = torch.randn(full.m, device="cuda")
    p_full, r_full, d_full = full.new_projections(), full.new_volume(), full.new_volume()
    full.project_internal(x, p_full)
    full.backproject_internal(y, r_full)
    full.backproject_internal(None, d_full, mode=2)
    parts = {"p": [], "r": [], "d": []}
    for rank in range(world):
        sop = ShardedOperator(vg, tr, _VirtualComm(world, rank))
        assert sop.op.shard is not None
        info = sop.op.info
        assert (info.proj_chunk, info.bp_groups, info.bp_view_batches, info.bp_sided_gs) == (
            full.info.proj_chunk, full.info.bp_groups, full.info.bp_view_batches, full.info.bp_sided_gs)
        # the column + cell tables scale with the shard; per-column headers and offsets do not
        assert info.table_bytes <= full.info.table_bytes * (1.0 / world + 0.12), (rank, info.table_bytes)
        dd = torch.zeros(sop.n_full, device="cuda")
        dd[: full.vol_elems] = x
        ee = torch.zeros(sop.m_full, device="cuda")
        ee[: full.m] = y
        p_loc = torch.zeros(sop.m_loc, device="cuda")
        r_loc, d_loc = torch.zeros(sop.n_loc, device="cuda"), torch.zeros(sop.n_loc, device="cuda")
        sop.project_local(dd, p_loc)
        sop.backproject_local(ee, r_loc)
        sop.backproject_local(None, d_loc, mode=2)
        parts["p"].append(p_loc)
        parts["r"].append(r_loc)
        parts["d"].append(d_loc)
    assert torch.equal(torch.cat(parts["p"])[: full.m], p_full)
    assert torch.equal(torch.cat(parts["r"])[: full.vol_elems], r_full)
    assert torch.equal(torch.cat(parts["d"])[: full.vol_elems], d_full)


def test_shard_plans_with_empty_blocks():
    """More ranks than views and than cell rows: the empty ranks still build a (one-item) plan and
    contribute nothing; the others reassemble the unsharded A, A^T bit for bit."""
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.distributed import ShardedOperator

    vg = P.VolumeGeometry(12, 3, 10, (2.0, 2.0, 2.0))
    tr = P.make_circular_trajectory(300.0, 500.0, 3, 0.1, 2.0, P.DetectorGeometry(20, 15, (3.0, 3.0)))
    full = P.CbctOperator(vg, tr)
    x = full.volume_to_internal(np.random.default_rng(0).random(full.n))
    y = torch.randn(full.m, device="cuda")
    p_full, r_full = full.new_projections(), full.new_volume()
    full.project_internal(x, p_full)
    full.backproject_internal(y, r_full)
    world = 4
    p_parts, r_parts = [], []
    for rank in range(world):
        sop = ShardedOperator(vg, tr, _VirtualComm(world, rank))
        dd = torch.zeros(sop.n_full, device="cuda")
        dd[: full.vol_elems] = x
        ee = torch.zeros(sop.m_full, device="cuda")
        ee[: full.m] = y
        p_loc, r_loc = torch.zeros(sop.m_loc, device="cuda"), torch.zeros(sop.n_loc, device="cuda")
        sop.project_local(dd, p_loc)
        sop.backproject_local(ee, r_loc)
        p_parts.append(p_loc)
        r_parts.append(r_loc)
    assert torch.equal(torch.cat(p_parts)[: full.m], p_full)
    assert torch.equal(torch.cat(r_parts)[: full.vol_elems], r_full)


def test_shard_plan_refuses_outside_its_blocks():
    import ctypes

    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200._lib import CbctError, call

    vg, tr = baseline_geometry(64, 90, 128, 96)
    op = P.CbctOperator(vg, tr, _shard=(30, 60, 16, 40))
    vol, proj = op.new_volume(), op.new_projections()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    with pytest.raises(CbctError, match="view block"):
        call("cbct_project_views", op._plan, ctypes.c_void_p(vol.data_ptr()), ctypes.c_void_p(proj.data_ptr()),
             0, 60, None, s)
    with pytest.raises(CbctError, match="row block"):
        call("cbct_backproject_rows", op._plan, ctypes.c_void_p(proj.data_ptr()), ctypes.c_void_p(vol.data_ptr()),
             10, 40, 1, ctypes.c_void_p(op.new_bp_scratch().data_ptr()), None, None, s)
    with pytest.raises(CbctError, match="view block"):
        op.project_internal(vol, proj)  # the whole-operator entry point needs every view
    with pytest.raises(ValueError, match="fp64"):
        P.CbctOperator(vg, tr, precision="f64", _shard=(0, 45, 0, 64))


def test_nccl_world1_driver_matches_cgls():
    import torch.distributed as dist

    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.distributed import CudaVectors, ShardedOperator, TorchComm, dist_cgls, gathered_report
    from paper_2110_13526_b200.solvers import SolverConfig

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        d = load_golden("adjoint_instance")
        vg, tr = geom_from_golden(d)
        sop = ShardedOperator(vg, tr, TorchComm())
        truth = P.generate_phantom(P.shepp_logan_3d(), vg).data
        b_int = sop.op.new_projections()
        sop.op.project_internal(sop.op.volume_to_internal(truth), b_int)
        b_local = torch.zeros(sop.m_loc, device="cuda")
        b_local[: b_int.numel()] = b_int
        cfg = SolverConfig(method="cgls", max_iterations=8)
        info, x_local = dist_cgls(sop, CudaVectors(sop.op), b_local, cfg)
        rep = gathered_report(sop, x_local, info)
        ref = P.cgls(sop.op, P.operator.InternalProjections(tr, b_int), cfg)
        np.testing.assert_allclose([h.rel_discrepancy for h in rep.history],
                                   [h.rel_discrepancy for h in ref.history], rtol=1e-5)
        xr = ref.final_x.data
        xr = xr.double().cpu().numpy() if hasattr(xr, "cpu") else xr
        assert np.linalg.norm(rep.final_x.data - xr) / np.linalg.norm(xr) <= 1e-5
    finally:
        dist.destroy_process_group()


def test_nccl_world1_device_resident_loop_is_bitwise_the_host_loop():
    """DistCglsRun.run_device (norm partials all-gathered on the device and summed in rank order by
    cbct_sum_ranks, scalars and stop tests on the GPU) equals DistCglsRun.step exactly."""
    import torch.distributed as dist

    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.distributed import CudaVectors, DistCglsRun, ShardedOperator, TorchComm
    from paper_2110_13526_b200.solvers import SolverConfig

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        d = load_golden("adjoint_instance")
        vg, tr = geom_from_golden(d)
        sop = ShardedOperator(vg, tr, TorchComm())
        b_int = sop.op.new_projections()
        sop.op.project_internal(sop.op.phantom_internal(P.shepp_logan_3d()), b_int)
        b_local = torch.zeros(sop.m_loc, device="cuda")
        b_local[: b_int.numel()] = b_int
        for tol, K in ((0.0, 9), (0.25, 30)):
            cfg = SolverConfig(method="cgls", max_iterations=K, rel_discrepancy_tol=tol)
            host = DistCglsRun(sop, CudaVectors(sop.op), b_local, cfg)
            while host.should_continue():
                if not host.step():
                    break
            devr = DistCglsRun(sop, CudaVectors(sop.op), b_local, cfg)
            while devr.should_continue():
                devr.run_device(min(4, K - devr.i))
            assert devr.i == host.i and devr.pending == host.pending
            assert [h.rel_discrepancy for h in devr.hist] == [h.rel_discrepancy for h in host.hist]
            assert torch.equal(devr.x, host.x) and torch.equal(devr.d, host.d) and torch.equal(devr.e, host.e)
    finally:
        dist.destroy_process_group()


def test_nccl_world1_fused_p2p_updates_are_bitwise_the_gathered_loop():
    """The fused update + all-gather kernels (stores into every rank's symmetric-memory buffer,
    device barrier instead of all_gather) give the same iterates as the NCCL-gathered loop.
    World size 1 here (one GPU): the store loop and the barrier path run, with one peer."""
    import torch.distributed as dist

    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.distributed import CudaVectors, DistCglsRun, ShardedOperator, TorchComm
    from paper_2110_13526_b200.solvers import SolverConfig

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        d = load_golden("adjoint_instance")
        vg, tr = geom_from_golden(d)
        ref_sop = ShardedOperator(vg, tr, TorchComm())
        b_int = ref_sop.op.new_projections()
        ref_sop.op.project_internal(ref_sop.op.phantom_internal(P.shepp_logan_3d()), b_int)
        b_local = torch.zeros(ref_sop.m_loc, device="cuda")
        b_local[: b_int.numel()] = b_int
        cfg = SolverConfig(method="cgls", max_iterations=9)
        base = DistCglsRun(ref_sop, CudaVectors(ref_sop.op), b_local, cfg)
        base.run_device(9)
        sop = ShardedOperator(vg, tr, TorchComm()).enable_p2p()
        fused = DistCglsRun(sop, CudaVectors(sop.op), b_local, cfg)
        assert fused.p2p
        fused.run_device(5)
        fused.run_device(4)
        assert fused.i == base.i == 9
        assert [h.rel_discrepancy for h in fused.hist] == [h.rel_discrepancy for h in base.hist]
        assert torch.equal(fused.x, base.x) and torch.equal(fused.d, base.d) and torch.equal(fused.e, base.e)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_mode2_and_col_scale_assemble_to_full(world):
    """The cell-row slabs of diag(A^T A) (the sharded Jacobi diagonal) and of A^T with a column
    scale (the sharded Jacobi applyT) reassemble bit-for-bit to the unsharded kernels."""
    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.distributed import ShardedOperator

    vg, tr = baseline_geometry(64, 90, 128, 96)
    full = P.CbctOperator(vg, tr)
    y = torch.randn(full.m, device="cuda")
    scale = torch.rand(full.vol_elems, device="cuda")
    d_full, r_full = full.new_volume(), full.new_volume()
    full.backproject_internal(None, d_full, mode=2)
    full.backproject_internal(y, r_full, col_scale=scale)
    d_parts, r_parts = [], []
    for rank in range(world):
        sop = ShardedOperator(vg, tr, _VirtualComm(world, rank))
        e_full = torch.zeros(sop.m_full, device="cuda")
        e_full[: full.m] = y
        sc = torch.zeros(sop.n_loc, device="cuda")
        lo = sop.y0 * sop.row_elems
        sc[: (sop.y1 - sop.y0) * sop.row_elems] = scale[lo: sop.y1 * sop.row_elems]
        d_loc, r_loc = torch.zeros(sop.n_loc, device="cuda"), torch.zeros(sop.n_loc, device="cuda")
        sop.backproject_local(None, d_loc, mode=2)
        sop.backproject_local(e_full, r_loc, col_scale=sc)
        d_parts.append(d_loc)
        r_parts.append(r_loc)
    assert torch.equal(torch.cat(d_parts)[: full.vol_elems], d_full)
    assert torch.equal(torch.cat(r_parts)[: full.vol_elems], r_full)


def test_nccl_world1_lsqr_and_psirt_drivers_match_single_gpu(monkeypatch):
    """dist_lsqr (Jacobi) and dist_psirt over NCCL at world size 1 run the same vector kernels and
    reductions as the single-GPU host loops of solvers.lsqr / solvers.psirt: identical histories
    and iterates (the single-GPU fp32 LSQR otherwise runs device-resident, in another rounding
    order -- compared in test_solvers_gpu.py)."""
    import paper_2110_13526_b200.solvers as S

    monkeypatch.setattr(S.LsqrRun, "device_capable", lambda self: False)
    import torch.distributed as dist

    import paper_2110_13526_b200 as P
    from paper_2110_13526_b200.distributed import (CudaVectors, ShardedOperator, TorchComm, dist_lsqr, dist_psirt,
                                                   gathered_report)
    from paper_2110_13526_b200.solvers import SolverConfig

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        d = load_golden("adjoint_instance")
        vg, tr = geom_from_golden(d)
        sop = ShardedOperator(vg, tr, TorchComm())
        b_int = sop.op.new_projections()
        sop.op.project_internal(sop.op.phantom_internal(P.shepp_logan_3d()), b_int)
        b_local = torch.zeros(sop.m_loc, device="cuda")
        b_local[: b_int.numel()] = b_int
        bi = P.operator.InternalProjections(tr, b_int)
        for cfg, fn, ref_fn in (
                (SolverConfig(method="lsqr", max_iterations=8, jacobi_precondition=True), dist_lsqr, P.lsqr),
                (SolverConfig(method="psirt", max_iterations=6), dist_psirt, P.psirt),
                (SolverConfig(method="psirt", max_iterations=6, box_bounds=(0.0, 0.5)), dist_psirt, P.psirt)):
            info, x_local = fn(sop, CudaVectors(sop.op), b_local, cfg)
            rep = gathered_report(sop, x_local, info)
            ref = ref_fn(sop.op, bi, cfg)
            assert rep.iterations == ref.iterations
            np.testing.assert_allclose([h.rel_discrepancy for h in rep.history],
                                       [h.rel_discrepancy for h in ref.history], rtol=1e-12)
            xr = ref.final_x.data
            xr = xr.double().cpu().numpy() if hasattr(xr, "cpu") else xr
            assert np.linalg.norm(rep.final_x.data - xr) <= 1e-12 * np.linalg.norm(xr)
    finally:
        dist.destroy_process_group()
