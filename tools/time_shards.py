"""Per-rank kernel time of the sharded operators (virtual ranks on one GPU):
python tools/time_shards.py cfg world"""
import pathlib, sys
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import torch
import bench
import paper_2110_13526_b200 as P
from paper_2110_13526_b200.distributed import ShardedOperator


class _V:
    def __init__(self, w, r):
        self.world, self.rank = w, r


cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
vg, tr = bench.geometry(cfg)
ta, tat = [], []
for r in range(world):
    sop = ShardedOperator(vg, tr, _V(world, r))
    d = torch.rand(sop.n_full, device="cuda")
    e = torch.randn(sop.m_full, device="cuda")
    p = torch.zeros(sop.m_loc, device="cuda")
    x = torch.zeros(sop.n_loc, device="cuda")
    for fn, out in ((lambda: sop.project_local(d, p), ta), (lambda: sop.backproject_local(e, x), tat)):
        fn()
        torch.cuda.synchronize()
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            fn()
        t.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(t) / 3)
    del sop
    torch.cuda.empty_cache()
mean = lambda v: sum(v) / len(v)  # noqa: E731
print(f"cfg{cfg} world {world}: A ms per rank {[round(v, 2) for v in ta]} max/mean {max(ta) / mean(ta):.3f}")
print(f"cfg{cfg} world {world}: AT ms per rank {[round(v, 2) for v in tat]} max/mean {max(tat) / mean(tat):.3f}")
