"""Plan tables per rank of the sharded operator (cbct_plan_create_shard) vs the unsharded plan at
BASELINE configs 3 and 5: table bytes and build time for every rank of worlds 2, 4 and 8.
python tools/shard_plan_sizes.py [cfg ...] > profiles/shard_plans_r2.json"""
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2110_13526_b200 as P  # noqa: E402
from paper_2110_13526_b200.distributed import ShardLayout  # noqa: E402


def build(vg, tr, shard=None):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = P.CbctOperator(vg, tr, _shard=shard)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tb = int(op.info.table_bytes)
    del op
    torch.cuda.empty_cache()
    return tb, dt


out = {}
for cfg in [int(a) for a in sys.argv[1:]] or [3, 5]:
    vg, tr = bench.geometry(cfg)
    full_b, full_t = build(vg, tr)
    rec = {"full": {"table_bytes": full_b, "build_s": round(full_t, 3)}}
    for world in (2, 4, 8):
        ranks = []
        for rank in range(world):
            L = ShardLayout(vg, tr, world, rank)
            b, t = build(vg, tr, (L.v0, L.v1, L.y0, L.y1))
            ranks.append({"rank": rank, "views": [L.v0, L.v1], "rows": [L.y0, L.y1], "table_bytes": b,
                          "build_s": round(t, 3), "frac_of_full": round(b / full_b, 4)})
        rec[f"world{world}"] = {"max_frac_of_full": max(r["frac_of_full"] for r in ranks), "ranks": ranks}
    out[f"config{cfg}"] = rec
    print(f"config {cfg}: full {full_b / 1e9:.2f} GB; max rank share " +
          ", ".join(f"N={w}: {rec[f'world{w}']['max_frac_of_full']:.3f}" for w in (2, 4, 8)), file=sys.stderr)
print(json.dumps(out, indent=1))
